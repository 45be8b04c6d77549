"""Hottest CUDA source lines (warp-stall samples, with the top stall reasons) of one kernel
in an ncu report.   usage: python scripts/ncu_hot.py report.ncu-rep kernel_regex [n]"""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, fname, hdr = {}, "?", None
reasons = {}
def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr is None or len(r) < 5 or not r[0].isdigit():
        continue
    key = (fname, int(r[0]))
    v = f(r[4])
    old = agg.get(key, (0.0, r[1], {}))
    rs = dict(old[2])
    for i in st:
        rs[hdr[i][6:]] = rs.get(hdr[i][6:], 0.0) + f(r[i])
    agg[key] = (old[0] + v, r[1], rs)
tot = sum(v for v, _, _ in agg.values()) or 1
allr = {}
for _, _, rs in agg.values():
    for k, v in rs.items():
        allr[k] = allr.get(k, 0) + v
print(f"{tot:.0f} samples; stalls: " + ", ".join(f"{k} {v / tot:.0%}" for k, v in sorted(allr.items(), key=lambda kv: -kv[1])[:6]))
for (fn, ln), (v, src, rs) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    top = ", ".join(f"{k} {x / max(v, 1):.0%}" for k, x in sorted(rs.items(), key=lambda kv: -kv[1])[:2] if x > 0)
    print(f"{v / tot:6.1%} {fn}:{ln:<5} {src.strip()[:80]:80s} [{top}]")
