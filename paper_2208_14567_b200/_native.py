"""ctypes binding of the C ABI in include/links_b200.h.

The library is REQUIRED: there is no CPU fallback anywhere in this package.
If ``_lib/liblinks_b200.so`` is missing it is built with nvcc on first use;
if that fails (or no CUDA device is present when a kernel is called) the call
raises.
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_lib" / "liblinks_b200.so"

LA_MAX_JOINTS = 20
LA_MAX_STEPS = 18
LA_MAX_TOPK = 32

LA_SIM_WRITE_TRAJ = 1
LA_SIM_FP64 = 2
LA_SIM_GATE_ONLY = 4
LA_SIM_NO_COARSE = 8
LA_SIM_TRAJ_F64 = 16
LA_SIM_DEFER = 32
LA_SIM_SCATTER = 64
LA_SIM_WRITE_ONLY = 128
LA_SIM_EXACT64 = 256
LA_SIM_LANE_SCREEN = 512
LA_SIM_STATIC_GRID = 1024
LA_CH_NO_MQ = 64
LA_CH_MQ_FINE = 128
LA_CH_NO_INDEX = 256
LA_CH_INDEX_MQ = 512
LA_PENDING = -3
ABI_VERSION = 4
LA_EINVAL = -1
LA_ERANGE = -2
LA_EWS = -3
LA_EHOST = -4

LA_CH_EXPANSION = 1
LA_CH_SCALAR_PIPE = 2
LA_CH_TENSOR = 8
LA_CH_NO_PRUNE = 16
LA_CH_SEED_SCAN = 32

EXPORTS = (
    "la_simulate",
    "la_plan_geometry",
    "la_dyad_solve",
    "la_compact_workspace",
    "la_compact_valid",
    "la_compact_rows_workspace",
    "la_compact_rows",
    "la_compact_rows_split_workspace",
    "la_compact_rows_split",
    "la_normalize",
    "la_circle_stats",
    "la_chamfer_workspace",
    "la_chamfer_topk",
    "la_chamfer_index",
    "la_merge_shard_lists",
    "la_sample_topologies",
    "la_sample_topology_rng",
    "la_sample_poses",
    "la_rng_draw",
    "la_coarse_descriptors",
    "la_coarse_workspace",
    "la_coarse_select",
    "la_curation_keep",
    "la_moving_joints",
    "la_gen_create",
    "la_gen_destroy",
    "la_gen_window",
    "la_gen_window_dev",
    "la_gen_poses",
    "la_gen_consume",
    "la_gen_count",
    "la_gen_records",
    "la_gen_negatives",
    "la_gen_stats",
    "la_abi_version",
    "la_last_error",
    "la_device_sm_count",
)


class LaPlan(C.Structure):
    _fields_ = [
        ("n", C.c_int16),
        ("nsteps", C.c_int16),
        ("fixed_mask", C.c_uint32),
        ("step", (C.c_int8 * 3) * LA_MAX_STEPS),
        ("_pad", C.c_int8 * 2),
    ]


assert C.sizeof(LaPlan) == 64


class LaGenBatch(C.Structure):
    _fields_ = [
        ("state_hi", C.c_uint64),
        ("state_lo", C.c_uint64),
        ("inc_hi", C.c_uint64),
        ("inc_lo", C.c_uint64),
        ("first", C.c_int64),
        ("k", C.c_int32),
        ("n", C.c_int32),
        ("plan", C.c_int32),
        ("_pad", C.c_int32),
    ]


assert C.sizeof(LaGenBatch) == 56


class LaGenCfg(C.Structure):
    _fields_ = [
        ("seed", C.c_int64),
        ("n_min", C.c_int32),
        ("n_max", C.c_int32),
        ("ng_prob", C.c_double),
        ("variants", C.c_int32),
        ("T_low", C.c_int32),
        ("T_high", C.c_int32),
        ("max_attempts", C.c_int32),
        ("retries", C.c_int32),
        ("batch", C.c_int32),
        ("negative_rate", C.c_double),
        ("threads", C.c_int32),
        ("_pad", C.c_int32),
    ]


class LaSimArgs(C.Structure):
    _fields_ = [
        ("pos0", C.c_void_p),
        ("topo", C.c_void_p),
        ("plans", C.c_void_p),
        ("crank_cs", C.c_void_p),
        ("B", C.c_int64),
        ("G", C.c_int32),
        ("pos_stride", C.c_int32),
        ("T", C.c_int32),
        ("traj_stride", C.c_int32),
        ("traj", C.c_void_p),
        ("traj_row", C.c_void_p),
        ("cand", C.c_void_p),
        ("n_cand", C.c_int64),
        ("cand_count", C.c_void_p),
        ("first_t", C.c_void_p),
        ("first_joint", C.c_void_p),
        ("low_t", C.c_void_p),
        ("low_joint", C.c_void_p),
        ("counters", C.c_void_p),
        ("fixup_tau", C.c_float),
        ("flags", C.c_uint32),
        ("traj2", C.c_void_p),
        ("traj_row2", C.c_void_p),
        ("screen_refill", C.c_int32),
        ("screen_replay", C.c_int32),
    ]


class LaNormArgs(C.Structure):
    _fields_ = [
        ("paths", C.c_void_p),
        ("in_f64", C.c_int32),
        ("src_row", C.c_void_p),
        ("M", C.c_int64),
        ("P", C.c_int32),
        ("out", C.c_void_p),
        ("out_f64", C.c_int32),
        ("pair", C.c_void_p),
        ("diameter", C.c_void_p),
        ("is_circle", C.c_void_p),
        ("circle_var", C.c_void_p),
        ("unstable", C.c_void_p),
        ("status", C.c_void_p),
        ("bbox", C.c_void_p),
        ("rel_tol", C.c_double),
        ("y_tol", C.c_double),
    ]


class LaChamferArgs(C.Structure):
    _fields_ = [
        ("db", C.c_void_p),
        ("N", C.c_int64),
        ("P", C.c_int32),
        ("queries", C.c_void_p),
        ("NQ", C.c_int32),
        ("Q", C.c_int32),
        ("order", C.c_void_p),
        ("pos_begin", C.c_int64),
        ("pos_end", C.c_int64),
        ("id_base", C.c_int64),
        ("pos_base", C.c_int64),
        ("pos_map", C.c_void_p),
        ("k", C.c_int32),
        ("threshold", C.c_float),
        ("exclude_id", C.c_int64),
        ("top_d", C.c_void_p),
        ("top_id", C.c_void_p),
        ("top_pos", C.c_void_p),
        ("hit_d", C.c_void_p),
        ("hit_id", C.c_void_p),
        ("hit_pos", C.c_void_p),
        ("n_hits", C.c_void_p),
        ("all_d", C.c_void_p),
        ("ws", C.c_void_p),
        ("ws_bytes", C.c_size_t),
        ("flags", C.c_uint32),
        ("fixup_below", C.c_float),
        ("n_full", C.c_void_p),
        ("n_stage", C.c_void_p),
        ("cells", C.c_void_p),
        ("coarse", C.c_void_p),
        ("fine", C.c_void_p),
    ]


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lock = threading.Lock()
_lib: C.CDLL | None = None


def _declare(lib: C.CDLL) -> None:
    vp, i32, i64, sz = C.c_void_p, C.c_int32, C.c_int64, C.c_size_t
    lib.la_simulate.argtypes = [C.POINTER(LaSimArgs), vp]
    lib.la_plan_geometry.argtypes = [vp, vp, vp, i64, i32, i32, vp, vp, vp, vp]
    lib.la_dyad_solve.argtypes = [vp, vp, vp, vp, vp, i64, vp, vp, vp]
    lib.la_compact_workspace.argtypes = [i64]
    lib.la_compact_workspace.restype = sz
    lib.la_compact_valid.argtypes = [vp, i64, i32, vp, vp, vp, sz, vp]
    lib.la_compact_rows_workspace.argtypes = [i64]
    lib.la_compact_rows_workspace.restype = sz
    lib.la_compact_rows.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.la_compact_rows_split_workspace.argtypes = [i64]
    lib.la_compact_rows_split_workspace.restype = sz
    lib.la_compact_rows_split.argtypes = [vp, i64, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp]
    lib.la_normalize.argtypes = [C.POINTER(LaNormArgs), vp]
    lib.la_circle_stats.argtypes = [vp, i32, i64, i32, vp, vp, vp]
    lib.la_chamfer_workspace.argtypes = [C.POINTER(LaChamferArgs)]
    lib.la_chamfer_workspace.restype = sz
    lib.la_chamfer_topk.argtypes = [C.POINTER(LaChamferArgs), vp]
    lib.la_chamfer_index.argtypes = [vp, i64, i32, vp, vp, vp, vp]
    lib.la_merge_shard_lists.argtypes = [vp, i32, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp]
    lib.la_sample_topologies.argtypes = [i64, i64, i64, i32, i32, C.c_double, i32, i32, vp, vp, vp, vp]
    lib.la_sample_topology_rng.argtypes = [vp, vp, i32, C.c_double, i32, vp, vp, vp]
    lib.la_sample_poses.argtypes = [i64, i64, i64, i32, vp, i32, i32, vp]
    lib.la_rng_draw.argtypes = [vp, i32, i32, i64, i64, vp, vp]
    lib.la_coarse_descriptors.argtypes = [vp, i64, i32, vp, vp, vp]
    lib.la_coarse_workspace.argtypes = [i64]
    lib.la_coarse_workspace.restype = sz
    lib.la_coarse_select.argtypes = [vp, i64, vp, i64, vp, vp, vp, vp, sz, vp]
    lib.la_moving_joints.argtypes = [vp, vp, vp, vp, i64, i32, vp, vp, vp, vp]
    lib.la_moving_joints.restype = i64
    lib.la_curation_keep.argtypes = [vp, vp, vp, i64, i64, C.c_double, vp, vp]
    lib.la_gen_create.argtypes = [C.POINTER(LaGenCfg), i64, i64]
    lib.la_gen_create.restype = vp
    lib.la_gen_destroy.argtypes = [vp]
    lib.la_gen_destroy.restype = None
    lib.la_gen_window.argtypes = [vp, i32, i64, i32, vp, vp, vp, vp]
    lib.la_gen_window.restype = i64
    lib.la_gen_window_dev.argtypes = [vp, i32, i64, vp, i64, vp, vp, vp]
    lib.la_gen_window_dev.restype = i64
    lib.la_gen_poses.argtypes = [vp, i64, i32, vp, vp, vp]
    lib.la_gen_consume.argtypes = [vp, vp, vp, vp]
    lib.la_gen_count.argtypes = [vp, i32]
    lib.la_gen_count.restype = i64
    lib.la_gen_records.argtypes = [vp, vp, vp, vp, vp, vp]
    lib.la_gen_negatives.argtypes = [vp, vp, vp, vp, vp]
    lib.la_gen_stats.argtypes = [vp, vp, vp]
    lib.la_abi_version.argtypes = []
    lib.la_last_error.argtypes = []
    lib.la_last_error.restype = C.c_char_p
    lib.la_device_sm_count.argtypes = []
    for name in EXPORTS:
        if name not in ("la_last_error", "la_compact_workspace", "la_compact_rows_workspace",
                        "la_compact_rows_split_workspace", "la_chamfer_workspace",
                        "la_coarse_workspace",
                        "la_gen_create",
                        "la_gen_destroy", "la_gen_window", "la_gen_window_dev", "la_gen_count", "la_moving_joints"):
            getattr(lib, name).restype = C.c_int


def load(build_if_missing: bool = True) -> C.CDLL:
    """Load (building once if needed) the CUDA library.  Never falls back."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if build_if_missing:
            from paper_2208_14567_b200 import build_lib

            # missing, or older than its sources (a stale library with another
            # struct layout must not be called): rebuild; if nvcc is not there
            # an existing library is still tried -- the ABI version check
            # below refuses one of another interface version
            if build_lib.needs_build():
                try:
                    build_lib.build()
                except Exception:
                    if not LIB_PATH.exists():
                        raise
        if not LIB_PATH.exists():
            raise NativeError(f"CUDA library missing: {LIB_PATH} (run python -m paper_2208_14567_b200.build_lib)")
        lib = C.CDLL(str(LIB_PATH))
        _declare(lib)
        if lib.la_abi_version() != ABI_VERSION:
            raise NativeError("ABI version mismatch")
        _lib = lib
    return _lib


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().la_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (status {rc}): {msg}")


def require_cuda():
    """Return torch with a CUDA device available, or raise (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise NativeError("a CUDA device (B200, sm_100a) is required: this package has no CPU path")
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t) -> int | None:
    return None if t is None else int(t.data_ptr())


def last_error() -> str:
    return load().la_last_error().decode(errors="replace")
