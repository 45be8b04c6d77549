"""Per-kernel DRAM bytes per launch from scripts/traffic_capture.sh's ncu CSVs (cold: ncu
flushes L2 before each kernel; warm: --cache-control none).
    python scripts/traffic_summary.py gpurun_out/traffic_b128_all.csv gpurun_out/traffic_b128_none.csv"""
import collections
import csv
import io
import sys


def load(path):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    per = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in rows:
        name = r["Kernel Name"].split("(")[0].replace("void ", "").replace("rpl::", "")
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "nsecond": 1e-3, "ns": 1e-3, "msecond": 1e3, "ms": 1e3}.get(unit, 1)
        per[name][r["Metric Name"]].append(v * scale)
    out = {}
    for k, m in per.items():
        n = len(m["gpu__time_duration.sum"])
        rd = sum(m["dram__bytes_read.sum"]) / n
        wr = sum(m["dram__bytes_write.sum"]) / n
        out[k] = {"launches": n, "bytes": rd + wr, "read": rd, "write": wr, "us": sum(m["gpu__time_duration.sum"]) / n}
    return out


if __name__ == "__main__":
    cold, warm = load(sys.argv[1]), load(sys.argv[2])
    tc = tw = 0.0
    print(f"{'kernel':32s} {'cold B':>12s} {'warm B':>12s} {'cold us':>8s} {'warm us':>8s}")
    for k in cold:
        c, w = cold[k], warm.get(k, {"bytes": float('nan'), "us": float('nan')})
        tc += c["bytes"]
        tw += w["bytes"]
        print(f"{k[:32]:32s} {c['bytes']:12.0f} {w['bytes']:12.0f} {c['us']:8.2f} {w['us']:8.2f}")
    print(f"{'step total':32s} {tc:12.0f} {tw:12.0f}   warm/cold = {tw / tc:.3f}")
