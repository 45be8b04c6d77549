#!/usr/bin/env python
"""Benchmark of the in-GPU replay DQN train step (BASELINE.json metric: DQN train steps/s at
batch 128 with a 1M replay, 1/2/4/8 B200s; gather GB/s vs HBM peak).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One "step" = the whole hot path over one batch: replay_add of
`--adds-per-step` fresh experiences + dqn_train_step (burn-in gate, Philox sample, gather,
forward online(s)/target(s'), TD target, Huber, backward, SGD, step/sync counters; NCCL
gradient all-reduce when N > 1).  Workload (N=1): BASELINE configs[1] -- 1,000,000-slot
replay pre-filled with synthetic 27-float Melee-shaped experiences, batch 128, the paper's
dueling DQN.  Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DQN train steps/s at batch 128, 1M replay (1/2/4/8 B200); gather GB/s vs HBM peak"
ROW_READ_BYTES = 228     # the paper's packed row: 57 fp32 values
ROW_WRITE_BYTES = 229    # unpacked s, s' (216 B), a (4), r (4), done (1) + idx (4)
EXP_INPUT_BYTES = 8 * 27 + 9   # one experience as replay_add input (SoA)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5000)
    ap.add_argument("--warmup", type=int, default=100)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--capacity", type=int, default=1_000_000)
    ap.add_argument("--net", choices=["dueling", "2x64"], default="dueling")
    ap.add_argument("--ddqn", action="store_true")
    ap.add_argument("--adds-per-step", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-gather", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--sweep", default="", help="comma list of batch sizes: one JSON line each")
    ap.add_argument("--avg-period", type=int, default=0,
                    help="N > 1: average parameters every K steps instead of gradients every step")
    ap.add_argument("--shared-state", action="store_true",
                    help="store one state per experience (P:141): s' = the next slot's s")
    ap.add_argument("--distinct", action="store_true",
                    help="sample distinct indices (RPL_SAMPLE_DISTINCT, P:75's planned switch)")
    ap.add_argument("--precision", choices=["fp32", "tf32", "bf16"], default="fp32",
                    help="tensor-core products: fp32 (FP32-accurate splits, the default and the "
                         "judged line) or one tf32 / bf16 product (reduced precision, parity 2e-2)")
    ap.add_argument("--dp", choices=["auto", "nccl", "p2p"], default="auto",
                    help="N > 1: gradient mean by the peer-memory mean + SGD kernel "
                         "(dqn_attach_peers) when every rank's GPU can map every other's (auto, "
                         "the default), or by ncclAllReduce")
    ap.add_argument("--ring", choices=["device", "host"], default="device",
                    help="host: the in-RAM comparison mode (SURVEY NEXT-1): ring rows in pinned host "
                         "memory, every batch read across PCIe by the same kernels")
    ap.add_argument("--config", choices=["c2", "c5"], default="c2",
                    help="c2: BASELINE configs[1] (default); c5: configs[4] 84x84x4 uint8 states, "
                         "batch 256 (other flags' defaults: --batch 256)")
    return ap.parse_args()


DTYPE = {"fp32": "f32", "tf32": "tf32", "bf16": "bf16"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_name(a, batch):
    net = ("dueling DQN 27-128-[V512|A512]-1+8 (P:92-94)" if a.net == "dueling"
           else "2x64 MLP 27-64-64-8")
    tgt = "Double-DQN" if a.ddqn else "DQN"
    where = (", ring rows in pinned host memory read across PCIe (in-RAM comparison mode)"
             if a.ring == "host" else "")
    return (f"BASELINE configs[1]: {a.capacity:,}-slot replay of 27-float states, batch {batch}, "
            f"{net}, {tgt} target, Huber, SGD, {a.adds_per_step} inserts/step{where}")


def make_cfg(a, binding, batch):
    if a.net == "dueling":
        return binding.DQNConfig(state_dim=27, n_actions=8, dueling=True, hidden=(128,), stream=512,
                                 double_dqn=a.ddqn, gamma=0.99, lr=1e-4, huber_kappa=1.0,
                                 sync_period=10_000, max_batch=max(batch, 128),
                                 avg_period=a.avg_period, precision=a.precision)
    return binding.DQNConfig(state_dim=27, n_actions=8, dueling=False, hidden=(64, 64),
                             double_dqn=a.ddqn, gamma=0.99, lr=1e-4, huber_kappa=1.0,
                             sync_period=10_000, max_batch=max(batch, 128), avg_period=a.avg_period,
                             precision=a.precision)


def oracle_net_of(cfg):
    import oracle
    return oracle.Net(cfg.state_dim, cfg.n_actions, cfg.dueling, tuple(cfg.hidden), cfg.stream)


# ------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for n, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def load_traffic():
    """dram bytes per launch of the train-step kernel from the committed ncu --set full capture"""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        try:
            return json.load(open(p))
        except Exception:
            return {}
    return {}


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def time_oracle(a, batch, seconds, max_steps=None, steps_wanted=None, warmup=0):
    import oracle
    from inputs import experiences, init_params
    import paper_1801_03138_b200.binding as binding  # host-only: DQNConfig / param count
    cfg = make_cfg(a, binding, batch)
    net = oracle_net_of(cfg)
    ring = oracle.Ring(a.capacity, 27)
    ring.add_many(experiences(a.capacity, seed=1))
    ln = oracle.Learner(net, init_params(27, 8, cfg.hidden, cfg.dueling, cfg.stream, seed=3),
                        gamma=float(np.float32(cfg.gamma)), kappa=1.0,
                        lr=float(np.float32(cfg.lr)), double_dqn=a.ddqn, burn_in=1,
                        sync_period=cfg.sync_period, seed=2)
    k = a.adds_per_step
    pool = experiences(max(k, 1) * 64, seed=11)

    def one(i):
        if k:
            j = (i % 64) * k
            ring.add(**{kk: v[j:j + k] for kk, v in pool.items()})
        rc, _, _ = ln.step(ring, batch)
        assert rc == oracle.OK

    for i in range(warmup):
        one(i)
    n, t0 = 0, time.perf_counter()
    while True:
        one(n)
        n += 1
        el = time.perf_counter() - t0
        if steps_wanted is not None and n >= steps_wanted:
            break
        if el >= seconds and n >= 3:
            break
        if max_steps is not None and n >= max_steps:
            break
    return n, el


def lscpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for l in out.splitlines():
            if l.startswith("Model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return "?"


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    batch = a.batch
    # bounded: the whole --steps K --warmup W run must end within a few minutes
    budget = 120.0
    n, el = time_oracle(a, batch, seconds=budget, steps_wanted=a.steps, warmup=min(a.warmup, 2))
    v = n / el
    sample = (f"{n} of the requested {a.steps} oracle steps (each: {a.adds_per_step} inserts + one "
              f"B={batch} train step from a {a.capacity:,}-row host ring), time-capped at "
              f"{budget:.0f} s; single thread, fp64 arithmetic")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "train_steps/s",
        "n_gpus": a.gpus, "steps": n, "warmup": min(a.warmup, 2), "ms_per_step": 1000 * el / n,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(a, batch), "batch": batch,
                                        "capacity": a.capacity, "parallelism": "none (CPU oracle)"},
        "cpu_baseline": {"value": v, "unit": "train_steps/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": lscpu_model()},
        "e2e": {"value": v, "unit": "train_steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def run_ours(a, batch, first_line=True):
    import torch
    import torch.distributed as dist
    import paper_1801_03138_b200.binding as binding
    from inputs import experiences, init_params

    rank, world, local = dist_env()
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    peaks, peaks_kind = load_peaks()

    cfg = make_cfg(a, binding, batch)
    rp = binding.Replay(a.capacity, 27, device=local, burn_in=1, seed=2, rank=rank,
                        sampling="distinct" if a.distinct else "uniform",
                        shared_state=a.shared_state, ring_memory=a.ring)
    # pre-fill the whole ring (startup excluded from timings); per-rank data stream
    rp.add_many(experiences(a.capacity, seed=1, rank=rank))
    dqn = binding.DQN(cfg, init_params(27, 8, cfg.hidden, cfg.dueling, cfg.stream, seed=3),
                      device=local)
    if world > 1:
        from paper_1801_03138_b200 import dp
        if a.avg_period:
            dp.attach(dqn)   # parameter averaging runs on NCCL
            a.dp_used = "nccl"
        elif a.dp == "auto":
            a.dp_used = dp.attach_auto(dqn)   # peer memory if possible, else NCCL
        elif a.dp == "p2p":
            dp.attach_peers(dqn)   # gradient mean + SGD over peer memory inside every step
            a.dp_used = "p2p"
        else:
            dp.attach(dqn)   # NCCL gradient all-reduce inside every dqn_train_step
            a.dp_used = "nccl"

    K, W, k = a.steps, a.warmup, a.adds_per_step
    npool = max(k, 1) * 256
    pool_h = experiences(npool, seed=7, rank=rank)
    pool_d = {kk: torch.from_numpy(v).to(dev) for kk, v in pool_h.items()}
    loss_dev = torch.zeros(1, device=dev)

    def add_dev(i):
        if k:
            j = (i % 256) * k
            rp.add(**{kk: v[j:j + k] for kk, v in pool_d.items()}, defer=True)

    launches0 = binding.kernel_launches()
    for i in range(W):
        add_dev(i)
        dqn.train_step(rp, batch, loss_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches_w = binding.kernel_launches()

    # ---- device-resident timed region (nothing but the steps between the two events) ------
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        for i in range(K):
            add_dev(W + i)
            dqn.train_step(rp, batch, loss_dev)
        end.record(stream)
        torch.cuda.synchronize()
    launches = binding.kernel_launches() - launches_w
    elapsed_ms = start.elapsed_time(end)
    # per-launch duration of the step's kernels for the roofline: a separate pass with CUDA
    # events around every dqn_train_step (the events add stream ops, so not the timed one)
    kr = min(K, 1000)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(kr)]
    for i in range(kr):
        add_dev(W + K + i)
        ev[i][0].record(stream)
        dqn.train_step(rp, batch, loss_dev)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    kern_ms = [s.elapsed_time(e) for s, e in ev]
    st = dqn.check()
    assert st == binding.RPL_OK, f"device error {st}: {binding.last_error()}"
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = t.item()
    ms_per_step = elapsed_ms / K
    value = world * K / (elapsed_ms / 1000.0)

    # ---- end to end: host inserts (pinned staging + H2D inside replay_add) + D2H loss ------
    e2e = None
    if not a.no_e2e:
        loss_host = torch.zeros(K, dtype=torch.float32, pin_memory=True)
        loss_slots = [loss_host[i:i + 1] for i in range(K)]   # one pinned result slot per step
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d0 = rp.state()["h2d_bytes"]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        s2.record(stream)
        for i in range(K):
            if k:
                j = (i % 256) * k
                rp.add(**{kk: v[j:j + k] for kk, v in pool_h.items()})
            # the step's loss is stored by the last kernel straight into pinned host memory
            # (a 4-byte device -> host write over PCIe; no copy op in the stream)
            dqn.train_step(rp, batch, loss_slots[i])
        e2.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_ms = s2.elapsed_time(e2)
        if world > 1:
            t = torch.tensor([e2e_ms, wall * 1000.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms, wall = t[0].item(), t[1].item() / 1000.0
        h2d = (rp.state()["h2d_bytes"] - h2d0) / K
        assert np.all(np.isfinite(loss_host.numpy()))
        e2e = {"value": world * K / (max(e2e_ms / 1000.0, wall)), "unit": "train_steps/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4,
               "us_per_step_device": e2e_ms * 1000.0 / K, "us_per_step_wall": wall * 1e6 / K,
               "note": "replay_add(RPL_HOST) from pageable numpy -> library pinned staging (read "
                       "by the device over PCIe when the step consumes the insert: zero-copy), "
                       "dqn_train_step whose last kernel writes the loss into pinned host memory, "
                       "every step; slower of CUDA-event and wall time"}

    # ---- roofline of the dominant kernel (the fused train step) --------------------------
    flops = binding.step_flops(cfg, batch)
    kern_avg_ms = float(np.mean(kern_ms))
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    peak_fp32 = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12   # FP32 FMA lanes x 2 x clock
    achieved = flops / (kern_avg_ms / 1000.0) / 1e12
    traffic = load_traffic().get(f"train_step_b{batch}_{a.net}_{'ddqn' if a.ddqn else 'dqn'}")
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_fp32, "unit": "TFLOP/s",
                "frac": achieved / peak_fp32, "traffic": traffic,
                "kernel": "the train-step CUDA graph (fwd / td / bwd1 / bwd0+sgd kernels) timed as one "
                          "unit with CUDA events around each dqn_train_step on the library stream",
                "kernel_avg_us": kern_avg_ms * 1000.0, "flops_per_launch": flops,
                "peak_note": "FP32 SIMT: 148 SMs x 128 FMA lanes x 2 FLOP x sm_max_mhz "
                             f"{sm_mhz:.0f} MHz (derived, {peaks_kind} clock); the forward runs its "
                             "products as 3xTF32 mma.sync, so this FP32 peak is the conservative "
                             "denominator for an FP32-accurate step"}

    # ---- gather bandwidth (metric part 2): explicit-index gather from the 1M ring --------
    gather = None
    if not a.no_gather and first_line:
        n_idx = 1 << 22
        idx = torch.randint(0, a.capacity, (n_idx,), dtype=torch.int32, device=dev)
        out = {"s": torch.empty(n_idx, 27, device=dev), "s_next": torch.empty(n_idx, 27, device=dev),
               "a": torch.empty(n_idx, dtype=torch.int32, device=dev),
               "r": torch.empty(n_idx, device=dev),
               "done": torch.empty(n_idx, dtype=torch.uint8, device=dev),
               "idx": torch.empty(n_idx, dtype=torch.int32, device=dev)}
        for _ in range(3):
            rp.gather(idx, out)
        reps = 20
        gs, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        gs.record(stream)
        for _ in range(reps):
            rp.gather(idx, out)
        ge.record(stream)
        torch.cuda.synchronize()
        g_ms = gs.elapsed_time(ge) / reps
        alg = n_idx * (ROW_READ_BYTES + ROW_WRITE_BYTES)
        gbs = alg / (g_ms / 1000.0) / 1e9
        gather = {"indices_per_launch": n_idx, "us_per_launch": g_ms * 1000.0,
                  "achieved_GBps": gbs, "peak_GBps": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"],
                  "bytes_per_index": ROW_READ_BYTES + ROW_WRITE_BYTES,
                  "note": "replay_gather of 4M uniform indices from the 256 MB ring (> L2); algorithmic "
                          "bytes = 228 B packed row read + 229 B unpacked write per index; peak = "
                          f"{peaks_kind} HBM copy bandwidth"}
        # the same gather across launch sizes (latency -> bandwidth bound)
        sweep = []
        for m in (128, 4096, 65536, 1 << 20, 1 << 22):
            sub = {kk: v[:m] for kk, v in out.items()}
            for _ in range(3):
                rp.gather(idx[:m], sub)
            reps_m = 50 if m <= 65536 else 10
            gs.record(stream)
            for _ in range(reps_m):
                rp.gather(idx[:m], sub)
            ge.record(stream)
            torch.cuda.synchronize()
            t_ms = gs.elapsed_time(ge) / reps_m
            sweep.append({"indices": m, "us": t_ms * 1000.0,
                          "GBps": m * (ROW_READ_BYTES + ROW_WRITE_BYTES) / (t_ms / 1000.0) / 1e9})
        gather["sweep"] = sweep
        rp.check()
        # insert cost vs block size k (the B200 version of P:119-125, Fig. 3),
        # host-sourced (one pinned H2D copy inside replay_add) and device-sourced
        ins = []
        big = experiences(10_000, seed=13, rank=rank)
        big_d = {kk: torch.from_numpy(v).to(dev) for kk, v in big.items()}
        for kk_ in (1, 10, 100, 2000, 10_000):
            row = {"k": kk_}
            for src, pool in (("host", big), ("device", big_d)):
                part = {kx: v[:kk_] for kx, v in pool.items()}
                for _ in range(3):
                    rp.add(**part)
                reps_i = 20
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                gs.record(stream)
                for _ in range(reps_i):
                    rp.add(**part)
                ge.record(stream)
                torch.cuda.synchronize()
                wall = (time.perf_counter() - t0) / reps_i
                dev_s = gs.elapsed_time(ge) / 1000.0 / reps_i
                t = max(wall, dev_s)
                row[f"{src}_us_per_experience"] = t * 1e6 / kk_
                row[f"{src}_GBps"] = kk_ * EXP_INPUT_BYTES / t / 1e9
            ins.append(row)
        gather["insert_sweep"] = ins
        rp.check()
        # P:73 / Fig. 3 proper: single host experiences through the update-size queue
        # (update_size U): wall time per replay_add call, block transfers included
        upd = []
        one = experiences(20_000, seed=14, rank=rank)
        for U in (1, 10, 100, 2000, 10_000):
            rq = binding.Replay(20_000, 27, device=local, update_size=U)
            rows = [{kx: v[i:i + 1] for kx, v in one.items()} for i in range(20_000)]
            for i in range(2000):
                rq.add(**rows[i])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i in range(20_000):
                rq.add(**rows[i])
            torch.cuda.synchronize()
            upd.append({"update_size": U, "us_per_add": (time.perf_counter() - t0) / 20_000 * 1e6})
            rq.close()
        gather["update_size_sweep"] = upd

    # ---- CPU oracle baseline (rank 0, N=1 only) ------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and first_line:
        n, el = time_oracle(a, batch, seconds=a.cpu_seconds)
        cpu = {"value": n / el, "unit": "train_steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{n} oracle steps ({a.adds_per_step} inserts + one B={batch} train step "
                         f"from a {a.capacity:,}-row host ring) in {el:.1f} s, single thread, fp64",
               "cpu": lscpu_model()}

    line = {
        "metric": METRIC, "value": value, "unit": "train_steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[a.precision], "data": "synthetic",
        "config": {"workload": workload_name(a, batch), "batch": batch, "capacity": a.capacity,
                   "net": a.net, "double_dqn": a.ddqn, "adds_per_step": k,
                   "sampling": "distinct" if a.distinct else "uniform (with replacement, P:75)",
                   "state_storage": "shared (s' = next slot's s, P:141)" if a.shared_state else "s and s' per row",
                   "ring_memory": "host (pinned, read across PCIe: in-RAM comparison)" if a.ring == "host" else "device (HBM)",
                   "parallelism": f"dp{world}" + (f", parameters averaged every {a.avg_period} steps"
                                                  if a.avg_period and world > 1 else "")
                                  + (", gradient mean over peer memory" if getattr(a, "dp_used", "") == "p2p"
                                     else ", NCCL gradient all-reduce" if world > 1 and not a.avg_period else ""),
                   "l2": "inputs larger than L2: the 256 MB ring (> 126 MB L2) is sampled uniformly;"
                         " the 0.56 MB weights stay L2-resident as in steady-state training"},
        "samples_per_s": value * batch,
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gather": gather,
        "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dqn.close()
    rp.close()
    return line


# ------------------------------------------------------------------------------------------
# config 5: 84x84x4 uint8 Atari-shaped states (BASELINE configs[4])
# ------------------------------------------------------------------------------------------
C5_D = 84 * 84 * 4
C5_ROW_BYTES = 56576      # device row: round_up(round_up(2 * C5_D, 16) + 12, 128)
C5_ROW_BYTES_SHARED = 28288   # one state per row: round_up(round_up(C5_D, 16) + 12, 128)


def c5_cfg(binding, batch, ddqn, precision="fp32"):
    return binding.DQNConfig(state_dim=C5_D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                             double_dqn=ddqn, gamma=0.99, lr=1e-4, huber_kappa=1.0,
                             sync_period=10_000, max_batch=batch, precision=precision)


def time_oracle_c5(batch, ddqn, seconds, pool):
    """The oracle on a bounded sample of config 5: a 1,024-row byte ring (the 56 GB ring does
    not fit in host RAM), its sampler + gather, u8 -> x, loss / gradient and SGD, composed
    as they stand (never tuned), single thread, fp64."""
    import oracle
    from inputs import init_params
    import paper_1801_03138_b200.binding as binding
    cfg = c5_cfg(binding, batch, ddqn)
    net = oracle_net_of(cfg)
    ring = oracle.RingU8(1024, C5_D)
    ring.add(**pool)
    online = init_params(C5_D, 8, (128,), True, 512, seed=3)
    target = online.copy()
    n, t0 = 0, time.perf_counter()
    while True:
        rc, ob = ring.sample(1, 2, 0, batch)
        ob = dict(ob, s=oracle.u8_input(ob["s"]), s_next=oracle.u8_input(ob["s_next"]))
        out = oracle.dqn_loss_grad(net, online, target, ob, float(np.float32(0.99)), 1.0, ddqn)
        online = oracle.sgd(online, out["grad"], float(np.float32(1e-4))).astype(np.float32)
        n += 1
        el = time.perf_counter() - t0
        if el >= seconds and n >= 2:
            return n, el


def run_c5(a):
    import torch
    import torch.distributed as dist
    import paper_1801_03138_b200.binding as binding
    from inputs import experiences_u8, init_params

    rank, world, local = dist_env()
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local)
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()
    peaks, peaks_kind = load_peaks()
    batch = a.batch if a.batch != 128 else 256
    cfg = c5_cfg(binding, batch, a.ddqn, a.precision)
    rp = binding.Replay(a.capacity, C5_D, device=local, burn_in=1, seed=2, rank=rank,
                        state_dtype="u8", shared_state=a.shared_state,
                        sampling="distinct" if a.distinct else "uniform")
    # device-side pre-fill (startup, excluded from timings): a 1,024-experience pool of
    # this rank's synthetic stream inserted round-robin until the ring is full
    npool = 1024
    pool_h = experiences_u8(npool, seed=1, rank=rank)
    pool_d = {kk: torch.from_numpy(v).to(dev) for kk, v in pool_h.items()}
    for i in range(0, a.capacity, npool):
        m = min(npool, a.capacity - i)
        rp.add(**{kk: v[:m] for kk, v in pool_d.items()})
    dqn = binding.DQN(cfg, init_params(C5_D, 8, (128,), True, 512, seed=3), device=local)
    if world > 1:
        from paper_1801_03138_b200 import dp
        if a.dp == "auto":
            a.dp_used = dp.attach_auto(dqn)
        elif a.dp == "p2p":
            dp.attach_peers(dqn)
            a.dp_used = "p2p"
        else:
            dp.attach(dqn)
            a.dp_used = "nccl"
    K, W, k = a.steps, a.warmup, a.adds_per_step
    loss_dev = torch.zeros(1, device=dev)

    def add_dev(i):
        if k:
            j = (i * k) % (npool - k)
            rp.add(**{kk: v[j:j + k] for kk, v in pool_d.items()})

    for i in range(W):
        add_dev(i)
        dqn.train_step(rp, batch, loss_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches_w = binding.kernel_launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        start.record(stream)
        for i in range(K):
            add_dev(W + i)
            dqn.train_step(rp, batch, loss_dev)
        end.record(stream)
        torch.cuda.synchronize()
    launches = binding.kernel_launches() - launches_w
    elapsed_ms = start.elapsed_time(end)
    kr = min(K, 200)   # per-step durations for the roofline, in a separate pass
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(kr)]
    for i in range(kr):
        add_dev(W + K + i)
        ev[i][0].record(stream)
        dqn.train_step(rp, batch, loss_dev)
        ev[i][1].record(stream)
    torch.cuda.synchronize()
    kern_ms = [s_.elapsed_time(e_) for s_, e_ in ev]
    assert dqn.check() == binding.RPL_OK, binding.last_error()
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = t.item()
    value = world * K / (elapsed_ms / 1000.0)

    e2e = None
    if not a.no_e2e:
        loss_host = torch.zeros(K, dtype=torch.float32, pin_memory=True)
        loss_slots = [loss_host[i:i + 1] for i in range(K)]   # one pinned result slot per step
        s2, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        h2d0 = rp.state()["h2d_bytes"]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        s2.record(stream)
        for i in range(K):
            if k:
                j = (i * k) % (npool - k)
                rp.add(**{kk: v[j:j + k] for kk, v in pool_h.items()})
            # the step's loss is stored by the last kernel straight into pinned host memory
            # (a 4-byte device -> host write over PCIe; no copy op in the stream)
            dqn.train_step(rp, batch, loss_slots[i])
        e2.record(stream)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        e2e_ms = s2.elapsed_time(e2)
        if world > 1:
            t = torch.tensor([e2e_ms, wall * 1000.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms, wall = t[0].item(), t[1].item() / 1000.0
        e2e = {"value": world * K / (max(e2e_ms / 1000.0, wall)), "unit": "train_steps/s",
               "h2d_bytes_per_step": (rp.state()["h2d_bytes"] - h2d0) / K,
               "d2h_bytes_per_step": 4,
               "us_per_step_device": e2e_ms * 1000.0 / K, "us_per_step_wall": wall * 1e6 / K,
               "note": "replay_add(RPL_HOST) of byte states -> pinned staging -> H2D on the replay's "
                       "copy stream (overlapping the previous step), insert kernel, dqn_train_step "
                       "whose last kernel writes the loss into pinned host memory, every step; "
                       "slower of CUDA-event and wall time"}

    flops = binding.step_flops(cfg, batch)
    kern_avg_ms = float(np.mean(kern_ms))
    # 97% of the step's FLOPs are layer 0, run as bf16 x3 tcgen05 MMAs (FP32-accurate): the
    # denominator is the measured bf16 dense peak / 3 (the FP32-emulation rate), the sustained
    # figure since the kernel runs inside a long step
    bf16 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1352.0)))
    peak_emu = bf16 / 3.0
    achieved = flops / (kern_avg_ms / 1000.0) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_emu, "unit": "TFLOP/s",
                "frac": achieved / peak_emu,
                "traffic": load_traffic().get(f"c5_step_b{batch}_{'ddqn' if a.ddqn else 'dqn'}"),
                "kernel": "the whole train step (Philox gather, wide_l0_kernel, the cooperative "
                          "train kernel for the layers above layer 0, wide_dw0_kernel + SGD) timed "
                          "with CUDA events around each dqn_train_step",
                "kernel_avg_us": kern_avg_ms * 1000.0, "flops_per_launch": flops,
                "peak_note": f"measured bf16 dense {bf16:.0f} TFLOP/s ({peaks_kind}) / 3: layer 0 runs "
                             "three bf16 MMAs per FP32 product (hi/mid/lo split of the fp32 operand, "
                             "exact u8 input)"}

    gather = None
    if not a.no_gather:
        n_idx = 4096
        idx = torch.randint(0, a.capacity, (n_idx,), dtype=torch.int32, device=dev)
        out = {"s": torch.empty(n_idx, C5_D, dtype=torch.uint8, device=dev),
               "s_next": torch.empty(n_idx, C5_D, dtype=torch.uint8, device=dev),
               "a": torch.empty(n_idx, dtype=torch.int32, device=dev),
               "r": torch.empty(n_idx, device=dev),
               "done": torch.empty(n_idx, dtype=torch.uint8, device=dev),
               "idx": torch.empty(n_idx, dtype=torch.int32, device=dev)}
        for _ in range(3):
            rp.gather(idx, out)
        reps = 20
        gs, ge = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        gs.record(stream)
        for _ in range(reps):
            rp.gather(idx, out)
        ge.record(stream)
        torch.cuda.synchronize()
        g_ms = gs.elapsed_time(ge) / reps
        per = (2 * C5_D + 12) + (2 * C5_D + 13)
        gbs = n_idx * per / (g_ms / 1000.0) / 1e9
        gather = {"indices_per_launch": n_idx, "us_per_launch": g_ms * 1000.0, "achieved_GBps": gbs,
                  "peak_GBps": peaks["hbm_gbs"], "frac": gbs / peaks["hbm_gbs"], "bytes_per_index": per,
                  "note": "replay_gather of 4,096 uniform indices from the byte ring (> L2): "
                          "56,460 B row read + 56,461 B unpacked write (+ idx) per index"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        n, el = time_oracle_c5(batch, a.ddqn, a.cpu_seconds, pool_h)
        cpu = {"value": n / el, "unit": "train_steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{n} oracle steps (sample + u8->x + loss/grad + SGD at B={batch}) from a "
                         f"1,024-row host byte ring in {el:.1f} s, single thread, fp64",
               "cpu": lscpu_model()}
    line = {
        "metric": "DQN train steps/s at batch 256, 84x84x4 uint8 states, 1M replay per GPU "
                  "(BASELINE configs[4]); gather GB/s vs HBM peak",
        "value": value, "unit": "train_steps/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": elapsed_ms / K, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[a.precision], "data": "synthetic",
        "config": {"workload": f"BASELINE configs[4]: {a.capacity:,}-slot replay of 84x84x4 uint8 "
                               f"states ({a.capacity * (C5_ROW_BYTES_SHARED if a.shared_state else C5_ROW_BYTES) / 1e9:.1f} GB ring"
                               f"{', shared states' if a.shared_state else ''}), "
                               f"batch {batch}, dueling DQN 28224-128-[V512|A512]-1+8 on x = u8/255, "
                               f"{'Double-DQN' if a.ddqn else 'DQN'} target, Huber, SGD, {k} "
                               "inserts/step",
                   "batch": batch, "capacity": a.capacity, "double_dqn": a.ddqn,
                   "adds_per_step": k, "parallelism": f"dp{world}" + (
                       ", gradient mean over peer memory" if getattr(a, "dp_used", "") == "p2p"
                       else ", NCCL gradient all-reduce" if world > 1 else ""),
                   "l2": "inputs larger than L2 (the byte ring is sampled uniformly)"},
        "samples_per_s": value * batch, "gpu_launches": launches, "roofline": roofline,
        "cpu_baseline": cpu, "e2e": e2e, "gather": gather, "clocks": clk.summary(),
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    dqn.close()
    rp.close()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
        return
    if a.config == "c5":
        run_c5(a)
    elif a.sweep:
        for i, bsz in enumerate(int(x) for x in a.sweep.split(",")):
            run_ours(a, bsz, first_line=(i == 0))
    else:
        run_ours(a, a.batch)
    import torch.distributed as dist
    if dist.is_initialized():
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
