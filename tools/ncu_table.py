"""Per-kernel achieved HBM GB/s and FP32/FP64 FLOP/s from an ncu metrics CSV.

    ncu --metrics <METRICS below> --csv --log-file gpurun_out/table.csv python tools/kernel_table.py
    python tools/ncu_table.py gpurun_out/table.csv > profiles/rNN_kernel_table.txt
"""
import csv
import io
import json
import sys
from collections import defaultdict

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__sass_thread_inst_executed_op_ffma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fmul_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]


def main(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = defaultdict(lambda: defaultdict(float))
    cnt = defaultdict(int)
    seen = set()
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("la::<unnamed>::", "")
        name = name.replace("(anonymous namespace)::", "")
        key = (r["ID"], name)
        if key not in seen:
            seen.add(key)
            cnt[name] += 1
        v = float(r["Metric Value"].replace(",", "")) if r["Metric Value"] not in ("", "n/a") else 0.0
        unit = r["Metric Unit"]
        if r["Metric Name"] == "gpu__time_duration.sum":
            v *= {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)
        elif "bytes" in r["Metric Name"]:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        agg[name][r["Metric Name"]] += v
    peaks = json.load(open("MEASURED_PEAKS.json")) if __import__("os").path.exists("MEASURED_PEAKS.json") else {}
    hbm = peaks.get("hbm_gbs", 6551.7)
    fp32 = 148 * 128 * 2 * 1.965e9 / 1e12
    print(f"# per-kernel totals over all launches (ncu metrics pass, --clock-control none); HBM peak {hbm} GB/s, "
          f"FP32 nominal {fp32:.1f} TFLOP/s")
    print(f"{'kernel':52s} {'launch':>6s} {'time ms':>9s} {'DRAM MB':>9s} {'GB/s':>8s} {'%HBM':>6s} "
          f"{'FP32 TF/s':>9s} {'%FP32':>6s} {'FP64 TF/s':>9s}")
    for name, m in sorted(agg.items(), key=lambda kv: -kv[1]["gpu__time_duration.sum"]):
        t = m["gpu__time_duration.sum"]
        by = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
        # packed f32x2 instructions (FFMA2/FADD2/FMUL2) carry two lanes' worth
        f32 = (2 * m["smsp__sass_thread_inst_executed_op_ffma_pred_on.sum"]
               + m["smsp__sass_thread_inst_executed_op_fadd_pred_on.sum"]
               + m["smsp__sass_thread_inst_executed_op_fmul_pred_on.sum"]
               + 4 * m["smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum"]
               + 2 * m["smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum"]
               + 2 * m["smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum"])
        f64 = (2 * m["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
               + m["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
               + m["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"])
        gbs = by / t / 1e9 if t else 0
        tf = f32 / t / 1e12 if t else 0
        print(f"{name[:52]:52s} {cnt[name]:6d} {t * 1e3:9.3f} {by / 1e6:9.1f} {gbs:8.0f} {gbs / hbm * 100:6.1f} "
              f"{tf:9.2f} {tf / fp32 * 100:6.1f} {f64 / t / 1e12 if t else 0:9.2f}")
    print("# FP32 = 2 FFMA + FADD + FMUL + 4 FFMA2 + 2 FADD2 + 2 FMUL2 thread instructions executed (all "
          "executed flops, including the error-model and padding work; bench.py reports algorithmic flops)")


if __name__ == "__main__":
    main(sys.argv[1])
