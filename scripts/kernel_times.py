"""Warm per-kernel device times and inter-kernel gaps of the train step (CUPTI via
torch.profiler; no replay/serialisation, unlike ncu).  Run on the GPU box:
    python scripts/kernel_times.py [--batch 128] [--ddqn] [--steps 200] [--net dueling]
"""
import argparse
import collections
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ddqn", action="store_true")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--net", default="dueling")
    ap.add_argument("--capacity", type=int, default=1_000_000)
    ap.add_argument("--adds", type=int, default=4)
    a = ap.parse_args()
    import paper_1801_03138_b200.binding as b
    from inputs import experiences, init_params
    if a.net == "dueling":
        cfg = b.DQNConfig(double_dqn=a.ddqn, max_batch=a.batch)
    else:
        cfg = b.DQNConfig(dueling=False, hidden=(64, 64), double_dqn=a.ddqn, max_batch=a.batch)
    rp = b.Replay(a.capacity, 27, seed=2)
    rp.add_many(experiences(a.capacity, seed=1))
    dqn = b.DQN(cfg, init_params(27, 8, cfg.hidden, cfg.dueling, cfg.stream, seed=3))
    pool = {k: torch.from_numpy(v).cuda() for k, v in experiences(a.adds * 64, seed=7).items()}
    loss = torch.zeros(1, device="cuda")

    def step(i):
        if a.adds:
            j = (i % 64) * a.adds
            rp.add(**{k: v[j:j + a.adds] for k, v in pool.items()}, defer=True)
        dqn.train_step(rp, a.batch, loss)

    for i in range(50):
        step(i)
    torch.cuda.synchronize()
    import time
    t0 = time.perf_counter()
    for i in range(400):
        step(i)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"host enqueue {1e6 * (t1 - t0) / 400:.2f} us/step, wall incl. drain {1e6 * (t2 - t0) / 400:.2f} us/step")
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(a.steps):
            step(i)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    evs.sort(key=lambda e: e.time_range.start)
    per = collections.defaultdict(list)
    for e in evs:
        per[e.name[:50]].append(e.time_range.end - e.time_range.start)
    span = (evs[-1].time_range.end - evs[0].time_range.start) / a.steps
    print(f"batch {a.batch} ddqn {a.ddqn} net {a.net}: {span:.2f} us per step (first kernel start to last end / steps)")
    busy = 0.0
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        busy += sum(v)
        print(f"  {k:50s} n={len(v):5d} mean={np.mean(v):7.2f} us  p50={np.median(v):7.2f}  min={np.min(v):7.2f}")
    print(f"  busy {busy / a.steps:.2f} us/step, idle gaps {span - busy / a.steps:.2f} us/step")
    gaps = collections.defaultdict(list)
    for e0, e1 in zip(evs, evs[1:]):
        gaps[(e0.name[:20], e1.name[:20])].append(e1.time_range.start - e0.time_range.end)
    for k, v in sorted(gaps.items(), key=lambda kv: -len(kv[1]))[:8]:
        print(f"  gap {k[0]:20s} -> {k[1]:20s} mean {np.mean(v):6.2f} us")


def trace_main():
    """RPL_TRACE=1: per-CTA start/end of the four fast-path kernels of the last step, and the
    per-CTA phase marks (cycles after CTA start; for the tensor-core K3, accumulated phase
    cycles over all steps, printed per step)"""
    os.environ["RPL_TRACE"] = "1"
    ap = argparse.ArgumentParser()
    ap.add_argument("--trace", action="store_true")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--ddqn", action="store_true")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--accum", action="store_true", help="marks are per-phase cycle totals (tc kernels)")
    a = ap.parse_args()
    import paper_1801_03138_b200.binding as b
    from inputs import experiences, init_params
    cfg = b.DQNConfig(max_batch=a.batch, double_dqn=a.ddqn)
    rp = b.Replay(1_000_000, 27, seed=2)
    rp.add_many(experiences(1_000_000, seed=1))
    dqn = b.DQN(cfg, init_params(seed=3))
    loss = torch.zeros(1, device="cuda")
    for i in range(a.steps):
        dqn.train_step(rp, a.batch, loss)
    torch.cuda.synchronize()
    tr = dqn.debug(b.RPL_DBG_TRACE, a.batch).astype(np.int64)
    t0 = min(tr[k][tr[k][:, 0] > 0][:, 0].min() for k in range(4) if (tr[k][:, 0] > 0).any())
    names = ["K1 fwd", "K2 td", "K3 bwd1", "K4 bwd0+sgd"]
    for k in range(4):
        m = tr[k][:, 0] > 0
        if not m.any():
            continue
        st, en = (tr[k][m, 0] - t0) / 1000.0, (tr[k][m, 1] - t0) / 1000.0
        dur = en - st
        print(f"{names[k]:12s} ctas={m.sum():4d} start [{st.min():6.2f},{st.max():6.2f}] end [{en.min():6.2f},"
              f"{en.max():6.2f}] us  cta dur mean {dur.mean():5.2f} max {dur.max():5.2f} "
              f"(slowest cta {int(np.nonzero(m)[0][dur.argmax()])})")
        for ph in range(2, 8):
            mm = m & (tr[k][:, ph] > 0)
            if mm.any():
                rel = tr[k][mm, ph] / 1965.0   # SM cycles -> us at the 1965 MHz max clock
                if a.accum and (k == 2 or (k == 0 and ph >= 3)):   # accumulated phase totals (tc kernels)
                    rel = rel / a.steps
                    print(f"    phase {ph}: {rel.mean():6.2f} us per step per CTA (max {rel.max():6.2f}, n={mm.sum()})")
                else:
                    print(f"    mark {ph}: {rel.mean():6.2f} us after CTA start (max {rel.max():6.2f}, n={mm.sum()})")


if __name__ == "__main__":
    if "--trace" in sys.argv:
        trace_main()
    else:
        main()
