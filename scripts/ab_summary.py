"""Print batch / steps/s / per-kernel CUPTI means of bench.py JSON lines (A/B runs)."""
import json
import sys

for fn in sys.argv[1:]:
    print(fn)
    for line in open(fn):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        kc = d.get("roofline", {}).get("kernels_cupti", {})
        ks = " ".join(f"{k['kernel'].split('(')[0].split('::')[-1][:22]}={k['mean_us']:.1f}"
                      for k in kc.get("kernels", []))
        print(f"  B={d['config'].get('batch'):5d} {d['value']:9.0f} steps/s  {1e3 * d['ms_per_step']:7.1f} us  "
              f"frac={d['roofline'].get('frac', 0):.3f}  {ks}")
