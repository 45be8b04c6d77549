"""One row per kernel launch of an ncu --set full report: duration, DRAM bytes, tensor-pipe and
SM / memory throughput (percent of peak).   python scripts/ncu_table.py report.ncu-rep"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "us", 1e-3),
        ("dram__bytes_read.sum", "DRAM rd MB", 1e-6), ("dram__bytes_write.sum", "DRAM wr MB", 1e-6),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe %", 1),
        ("sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed", "UTCHMMA bf16 %", 1),
        ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "HMMA subpipe %", 1),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %", 1),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem %", 1),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %", 1)]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units = rows[0], rows[1]
idx = {n: h.index(n) for n, _, _ in COLS if n in h}
print("| kernel | " + " | ".join(lbl for n, lbl, _ in COLS if n in idx) + " |")
print("|---" * (1 + len(idx)) + "|")
for r in rows[2:]:
    vals = []
    for n, lbl, sc in COLS:
        if n not in idx:
            continue
        v, u = r[idx[n]], units[idx[n]]
        try:
            x = float(v.replace(",", ""))
        except ValueError:
            vals.append(v)
            continue
        if n.startswith("gpu__time"):
            x = x * {"ns": 1e-3, "us": 1, "usecond": 1, "nsecond": 1e-3, "ms": 1e3}.get(u, 1)
        elif n.startswith("dram__bytes"):
            x = x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) * 1e-6
        vals.append(f"{x:.2f}")
    name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
    print(f"| {name} | " + " | ".join(vals) + " |")
