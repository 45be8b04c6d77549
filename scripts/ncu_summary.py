"""Summarise ncu artefacts into profiles/: launch-list shares (from the --metrics
gpu__time_duration.sum CSV) and per-kernel DRAM traffic / duration / tensor-pipe activity
(from a --set full report).
usage: python scripts/ncu_summary.py <launches.csv> <full.ncu-rep> [more.ncu-rep ...] > out.md"""
import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [r for r in rows if r and r[0] == "ID"][0]
    data = [r for r in rows if r and r[0].isdigit()]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in data:
        agg[r[ki].split("(")[0][:60]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = ["| kernel | launches | mean µs (cold, serialised) | share |", "|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| `{k}` | {len(v)} | {sum(v) / len(v) / 1000:.2f} | {sum(v) / tot:.3f} |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active"]


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
             "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
             "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9, "Kbyte": 1e3}
    res = []
    for r in data:
        d = {}
        for h, u, v in zip(hdr, units, r):
            if u in scale:
                try:
                    v = str(float(v.replace(",", "")) * scale[u])   # bytes / nanoseconds
                except ValueError:
                    pass
            d[h] = v
        res.append(d)
    return res


def main():
    print(f"## Launch list ({sys.argv[1]})\n")
    print(launches(sys.argv[1]))
    traffic = {}
    for rep in sys.argv[2:]:
        print(f"\n## ncu --set full: {rep}\n")
        print("| kernel | grid x block | regs | duration µs | DRAM read B | DRAM write B | tensor pipe % | FMA pipe % |")
        print("|---|---|---|---|---|---|---|---|")
        for d in full(rep):
            name = d.get("Kernel Name", "?").split("(")[0]
            rd = float(d.get("dram__bytes_read.sum", "0").replace(",", "") or 0)
            wr = float(d.get("dram__bytes_write.sum", "0").replace(",", "") or 0)
            dur = float(d.get("gpu__time_duration.sum", "0").replace(",", "") or 0)
            print(f"| `{name}` | {d.get('launch__grid_size')} x {d.get('launch__block_size')} | "
                  f"{d.get('launch__registers_per_thread')} | {dur / 1000:.2f} | {rd:.0f} | {wr:.0f} | "
                  f"{d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed', '-')} | "
                  f"{d.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', '-')} |")
            traffic.setdefault(name, []).append(rd + wr)
    json.dump({k: sum(v) / len(v) for k, v in traffic.items()}, open("/tmp/traffic_by_kernel.json", "w"), indent=1)
    print("\n(DRAM bytes are per launch from `ncu --set full`, which flushes caches between kernels: cold)")


if __name__ == "__main__":
    main()
