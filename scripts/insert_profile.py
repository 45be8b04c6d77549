"""Device-sourced replay_add blocks of k experiences into a 1M-slot ring, one call per k, for an
ncu capture of insert_kernel (achieved HBM GB/s of the insert):
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        -k regex:insert_kernel --csv python scripts/insert_profile.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_1801_03138_b200.binding as b
    from inputs import experiences
    ks = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "2000,10000,100000,1000000").split(",")]
    C = 1_000_000
    rp = b.Replay(C, 27, seed=2)
    e = {k: torch.from_numpy(v).cuda() for k, v in experiences(max(ks), seed=1).items()}
    for k in ks:
        rp.add(**{kk: v[:k] for kk, v in e.items()})
    torch.cuda.synchronize()
    assert rp.check() == b.RPL_OK
    print("inserted", ks)


if __name__ == "__main__":
    main()
