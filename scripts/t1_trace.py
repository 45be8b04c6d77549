"""Phase totals of the large-batch T1 kernel (tc_big.cuh tcb_fwd_kernel, RPL_TRACE=1, trace
kernel slot 4), per CTA per step.   python scripts/t1_trace.py [--batch 4096] [--ddqn]"""
import argparse
import os
import sys

import numpy as np

os.environ["RPL_TRACE"] = "1"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--ddqn", action="store_true")
    ap.add_argument("--steps", type=int, default=100)
    a = ap.parse_args()
    import torch
    import paper_1801_03138_b200.binding as b
    from inputs import experiences, init_params
    cfg = b.DQNConfig(max_batch=a.batch, double_dqn=a.ddqn)
    rp = b.Replay(1_000_000, 27, seed=2)
    rp.add_many(experiences(1_000_000, seed=1))
    dqn = b.DQN(cfg, init_params(seed=3))
    loss = torch.zeros(1, device="cuda")
    for _ in range(a.steps):
        dqn.train_step(rp, a.batch, loss)
    torch.cuda.synchronize()
    trall = dqn.debug(b.RPL_DBG_TRACE, a.batch).astype(np.int64)
    tr = trall[4]
    m = tr[:, 0] > 0
    dur = (tr[m, 1] - tr[m, 0]) / 1000.0
    print(f"T1 B={a.batch} ddqn={a.ddqn}: {m.sum()} CTAs, last-step CTA duration mean {dur.mean():.2f} max {dur.max():.2f} us")
    names = {2: "MMA waits for H0 slot", 3: "MMA waits for drained acc", 4: "epilogue waits for acc",
             5: "epilogue work", 6: "producer waits for free slot"}
    for w, nm in names.items():
        v = tr[m, w] / a.steps / 1965.0
        print(f"  {nm:30s} {v.mean():7.2f} us per step per CTA (max {v.max():7.2f})")
    tr = trall[5]
    m = tr[:, 0] > 0
    if m.any():
        dur = (tr[m, 1] - tr[m, 0]) / 1000.0
        print(f"T3a: {m.sum()} CTAs, last-step CTA duration mean {dur.mean():.2f} max {dur.max():.2f} us")
        for w, nm in {2: "chunk start (stage free + barrier)", 3: "dZ1 passes", 4: "barrier after passes",
                      5: "MMA issue waits for H0 chunk"}.items():
            v = tr[m, w] / a.steps / 1965.0
            print(f"  {nm:34s} {v.mean():7.2f} us per step per CTA (max {v.max():7.2f})")
        su, lo = tr[m, 6] / 1965.0, (tr[m, 7] - tr[m, 6]) / 1965.0
        print(f"  last step: setup {su.mean():6.2f} us (max {su.max():6.2f}), chunk loop {lo.mean():6.2f} (max {lo.max():6.2f}),"
              f" epilogue {(dur - su - lo).mean():6.2f} (max {(dur - su - lo).max():6.2f})")


if __name__ == "__main__":
    main()
