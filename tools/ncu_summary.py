"""Summarise .ncu-rep captures into a compact text table for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep [...] > profiles/rNN_<name>.txt
"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active", "xu (MUFU) pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", "thread FFMA"),
    ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", "thread FADD"),
    ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", "thread FMUL"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
]


def summarise(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return f"{path}: no data\n"
    hdr, units = rows[0], rows[1]
    out = [f"# {path}"]
    for r in rows[2:]:
        out.append(f"## {r[hdr.index('Kernel Name')][:110]}")
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                out.append(f"  {label:30s} {r[i]:>18} {units[i]}")
        fl = 0.0
        for m, w in (("smsp__sass_thread_inst_executed_op_ffma_pred_on.sum", 2),
                     ("smsp__sass_thread_inst_executed_op_fadd_pred_on.sum", 1),
                     ("smsp__sass_thread_inst_executed_op_fmul_pred_on.sum", 1)):
            if m in hdr:
                try:
                    fl += w * float(r[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        if fl and "gpu__time_duration.sum" in hdr:
            dur = float(r[hdr.index("gpu__time_duration.sum")].replace(",", ""))
            unit = units[hdr.index("gpu__time_duration.sum")]
            sec = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(unit, 1e-9)
            out.append(f"  {'executed FP32 flops (scalar)':30s} {fl:18.4g}   -> {fl / sec / 1e12:.2f} TFLOP/s (FFMA2 counted per lane op)")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    for p in sys.argv[1:]:
        sys.stdout.write(summarise(p))
