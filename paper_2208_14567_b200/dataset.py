"""Device dataset pipeline: generated mechanisms -> moving-joint curves ->
flags -> curation -> atlas, the CLI chain ``generate`` / ``normalize`` /
``curate`` / ``build-atlas`` (cli.py:56-93, 118-172) without leaving HBM.

* mech ids follow ``cli.generate``: ``slot * variants_per_topology +
  variant`` (cli.py:69-71);
* every non-Fixed joint's T_high path is normalised by ``la_normalize``
  (f64 in, f64 out, curves.py:45-71) with ``is_circle`` fused (curves.py:95);
* ``is_arc`` is the topology test of curves.py:87-92 (any Fixed neighbour);
* the keep rule (curves.py:104-110) runs per record on the device
  (``la_curation_keep``: numpy SeedSequence + PCG64 bit for bit).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from paper_2208_14567_b200 import _native as N
from paper_2208_14567_b200.curves import DegeneratePathError, normalize_tensors
from paper_2208_14567_b200.mechanism import JointType

NMAX = N.LA_MAX_JOINTS


@dataclass
class CurveBatch:
    """Curve records as arrays: points (M, T, 2) f64 on the device; ids and
    flags as host numpy arrays (record order = mechanism order, joints
    ascending, like cli.normalize)."""

    points: "torch.Tensor"
    mech_ids: np.ndarray
    joint_ids: np.ndarray
    is_arc: np.ndarray
    is_circle: np.ndarray

    def __len__(self) -> int:
        return len(self.mech_ids)

    def select(self, mask: np.ndarray) -> "CurveBatch":
        torch = N.require_cuda()
        idx = np.flatnonzero(mask)
        pts = self.points.index_select(0, torch.from_numpy(idx).to(self.points.device))
        return CurveBatch(pts, self.mech_ids[idx], self.joint_ids[idx], self.is_arc[idx], self.is_circle[idx])

    def records(self):
        from paper_2208_14567_b200.records import CurveRecord

        pts = self.points.cpu().numpy()
        return [CurveRecord(int(m), int(j), bool(a), bool(c), p.tolist())
                for m, j, a, c, p in zip(self.mech_ids, self.joint_ids, self.is_arc, self.is_circle, pts)]


def mechanisms_of_block(block, variants_per_topology: int) -> dict:
    """{mech_id: Mechanism} of a GeneratedBlock (ids as cli.generate)."""
    out = {}
    for i in range(block.R):
        slot, variant, _, n = (int(x) for x in block.meta[i])
        from paper_2208_14567_b200.mechanism import Mechanism

        out[slot * variants_per_topology + variant] = Mechanism(block.adjacency[i, :n, :n].copy(),
                                                                block.types[i, :n].copy(), block.pos0[i, :n].copy())
    return out


def moving_joint_rows(block, variants_per_topology: int):
    """(rows into block.traj, mech ids, joint ids, is_arc) of every non-Fixed
    joint of every record of a GeneratedBlock."""
    lib = N.load()
    meta = np.ascontiguousarray(block.meta, dtype=np.int64)
    types = np.ascontiguousarray(block.types, dtype=np.int8)
    adj = np.ascontiguousarray(block.adjacency, dtype=np.uint8)
    row0 = np.ascontiguousarray(block.row0, dtype=np.int64)
    R = len(meta)
    M = lib.la_moving_joints(meta.ctypes.data, types.ctypes.data, adj.ctypes.data, row0.ctypes.data, R,
                             int(variants_per_topology), None, None, None, None)
    rows = np.empty(M, dtype=np.int64)
    mech_ids = np.empty(M, dtype=np.int64)
    joint = np.empty(M, dtype=np.int64)
    arc = np.empty(M, dtype=np.uint8)
    lib.la_moving_joints(meta.ctypes.data, types.ctypes.data, adj.ctypes.data, row0.ctypes.data, R,
                         int(variants_per_topology), rows.ctypes.data, mech_ids.ctypes.data, joint.ctypes.data,
                         arc.ctypes.data)
    return rows, mech_ids, joint, arc.astype(bool)



def curves_from_block(block, variants_per_topology: int) -> CurveBatch:
    """cli.normalize over a GeneratedBlock (trajectories on the device)."""
    torch = N.require_cuda()
    traj = block.traj
    if isinstance(traj, np.ndarray):
        traj = torch.from_numpy(traj).cuda()
    rows, mech_ids, joint_ids, arc = moving_joint_rows(block, variants_per_topology)
    if len(rows) == 0:
        return CurveBatch(torch.empty((0, traj.shape[1], 2), dtype=torch.float64, device=traj.device), mech_ids,
                          joint_ids, arc, np.zeros(0, dtype=bool))
    res = normalize_tensors(traj, src_row=torch.from_numpy(rows).to(traj.device), out_f64=True)
    if bool((res["status"] != 0).any()):
        raise DegeneratePathError("all path points coincident")
    return CurveBatch(res["out"], mech_ids, joint_ids, arc, res["is_circle"].cpu().numpy().astype(bool))


def curation_keep_batch(mech_ids, joint_ids, flagged, keep_rate: float, seed: int) -> np.ndarray:
    """curation_keep (curves.py:104-110) for a batch, on the device."""
    torch = N.require_cuda()
    lib = N.load()
    m = torch.from_numpy(np.ascontiguousarray(mech_ids, dtype=np.int64)).cuda()
    j = torch.from_numpy(np.ascontiguousarray(joint_ids, dtype=np.int64)).cuda()
    f = torch.from_numpy(np.ascontiguousarray(flagged, dtype=np.uint8)).cuda()
    if bool((m < 0).any()) or bool((j < 0).any()) or seed < 0:
        raise ValueError("SeedSequence entropy must be non-negative")
    keep = torch.empty(m.numel(), dtype=torch.uint8, device="cuda")
    N.check(lib.la_curation_keep(m.data_ptr(), j.data_ptr(), f.data_ptr(), m.numel(), int(seed), float(keep_rate),
                                 keep.data_ptr(), N.stream_ptr()), "la_curation_keep")
    return keep.cpu().numpy().astype(bool)


def curate_batch(cb: CurveBatch, keep_rate: float = 0.005, seed: int = 0) -> CurveBatch:
    """cli.curate / curves.curate (curves.py:113-120) on a CurveBatch."""
    keep = curation_keep_batch(cb.mech_ids, cb.joint_ids, cb.is_arc | cb.is_circle, keep_rate, seed)
    return cb.select(keep)


def atlas_from_curves(cb: CurveBatch, mechanisms: dict, seed: int = 0):
    """Atlas.build (atlas.py:85-110, no resampling) from a CurveBatch; the
    device copy of the curves is reused for the scan."""
    from paper_2208_14567_b200.atlas import Atlas

    atlas = Atlas(cb.points.cpu().numpy(), cb.mech_ids, cb.joint_ids, mechanisms, seed)
    atlas._dev = cb.points.float().contiguous()
    return atlas
