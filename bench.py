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
import types
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
    ap.add_argument("--no-c5", action="store_true",
                    help="skip the config-5 (84x84x4 u8, 1M rows) measurement the default run embeds")
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
    ap.add_argument("--dp", choices=["nccl", "auto", "p2p"], default="nccl",
                    help="N > 1: gradient mean by ncclAllReduce inside every step (nccl, the "
                         "default: the north star's path), or by the peer-memory mean + SGD "
                         "kernel (dqn_attach_peers) when every rank's GPU can map every other's "
                         "(auto), or always (p2p)")
    ap.add_argument("--ring", choices=["device", "host", "host_batch"], default="device",
                    help="host_batch: the paper's in-RAM replay (SURVEY NEXT-1; P:15, P:50): CPU ring, "
                         "CPU sampler and gather, one H2D batch copy per step into the same kernels; "
                         "host: its zero-copy variant (ring rows in pinned host memory read across "
                         "PCIe by the kernels)")
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
    where = {"host": ", ring rows in pinned host memory read across PCIe (zero-copy in-RAM variant)",
             "host_batch": ", the paper's in-RAM replay: CPU ring + CPU sampler/gather, one H2D batch "
                           "copy per step (P:15, P:50)"}.get(a.ring, "")
    cfgi = config_index(a, batch)
    return (f"BASELINE configs[{cfgi}]: {a.capacity:,}-slot replay of 27-float states, batch {batch}, "
            f"{net}, {tgt} target, Huber, SGD, {a.adds_per_step} inserts/step{where}")


def config_index(a, batch):
    """Which BASELINE.json config a line measures: configs[1] is the paper setting (batch 128,
    DQN); a Double-DQN or other-batch line belongs to the configs[2] sweep; N > 1 is configs[3]."""
    if dist_env()[1] > 1:
        return 3
    return 1 if (batch == 128 and not a.ddqn) else 2


def metric_name(a, batch):
    """The headline metric string for the paper setting; sweep lines name their own batch."""
    if config_index(a, batch) == 2:
        tgt = "Double-DQN" if a.ddqn else "DQN"
        return f"{tgt} train steps/s at batch {batch}, 1M replay (BASELINE configs[2] batch sweep)"
    return METRIC


def cfg_fields(a, batch):
    """The learner configuration of the run as plain fields (no library import: the oracle arm
    uses these too)."""
    common = dict(state_dim=27, n_actions=8, double_dqn=a.ddqn, gamma=0.99, lr=1e-4, huber_kappa=1.0,
                  sync_period=10_000, max_batch=max(batch, 128), avg_period=a.avg_period,
                  precision=a.precision)
    if a.net == "dueling":
        return dict(common, dueling=True, hidden=(128,), stream=512)
    return dict(common, dueling=False, hidden=(64, 64), stream=0)


def make_cfg(a, binding, batch):
    return binding.DQNConfig(**cfg_fields(a, batch))


def oracle_net_of(cfg):
    import oracle
    return oracle.Net(cfg.state_dim, cfg.n_actions, cfg.dueling, tuple(cfg.hidden), cfg.stream)


# ------------------------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)
# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event reasons sampled through NVML every `poll_ms` from before the
    warm-up until after the extra passes; `mark_start` / `mark_end` bracket the timed region,
    whose samples (if any) the summary reports, else those of the whole loaded phase."""
    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, torch_device: int, poll_ms: float = 5.0):
        self.dev = torch_device
        self.poll = poll_ms / 1000.0
        self.rows = []          # (t, sm_mhz, reasons bitmask)
        self.win = [None, None]
        self.max_mhz = None
        self.err = None
        self._stop = threading.Event()
        self.t = None

    def _handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            pr = torch.cuda.get_device_properties(self.dev)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.dev)

    def start(self):
        try:
            nv, h = self._handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        except Exception as e:   # no NVML: the line says so
            self.err = f"{type(e).__name__}: {e}"
            return self

        def run():
            while not self._stop.is_set():
                try:
                    self.rows.append((time.perf_counter(), float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)),
                                      int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))))
                except Exception as e:
                    self.err = f"{type(e).__name__}: {e}"
                    return
                time.sleep(self.poll)

        self.t = threading.Thread(target=run, daemon=True)
        self.t.start()
        return self

    def mark_start(self):
        self.win[0] = time.perf_counter()

    def mark_end(self):
        self.win[1] = time.perf_counter()

    def stop(self):
        self._stop.set()
        if self.t:
            self.t.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"],
                    "error": self.err}
        t0, t1 = self.win
        timed = [r for r in self.rows if t0 is not None and t1 is not None and t0 <= r[0] <= t1]
        use = timed if timed else self.rows
        import pynvml as nv
        reasons = sorted({n for n, attr in self.REASONS for r in use
                          if r[2] & int(getattr(nv, attr, 0))})
        return {"sm_mhz": statistics.median(r[1] for r in use), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples_timed_region": len(timed), "samples": len(self.rows),
                "window": "timed region" if timed else
                          "warm-up + timed region + extra passes (the timed region was shorter than "
                          "one poll)",
                "poll_ms": self.poll * 1000.0, "source": "NVML"}


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


def step_traffic(key):
    """(warm, cold) DRAM bytes per step for a bench shape, or None when not captured"""
    t = load_traffic()
    return (t[key], t.get(key + "_cold")) if key in t else None


def kernel_breakdown(step, n):
    """Per-kernel device time of `n` calls of step(i), from CUPTI (torch.profiler): mean us per
    launch, launches per step and share of the summed kernel time; run after the timed region."""
    import collections
    import torch
    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(n):
            step(3 + i)
        torch.cuda.synchronize()
    per = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA:
            per[e.name].append(e.time_range.end - e.time_range.start)
    tot = sum(sum(v) for v in per.values()) or 1.0
    out = [{"kernel": k, "mean_us": float(np.mean(v)), "launches_per_step": len(v) / n,
            "share": sum(v) / tot} for k, v in per.items()]
    out.sort(key=lambda d: -d["share"])
    return {"steps": n, "busy_us_per_step": tot / n, "kernels": out}


def flop_parts(cfg, batch):
    """(forward, backward) FLOPs of one step (2 per multiply-add): forward = every net's pass
    (online on s, target on s', online on s' for Double DQN); backward = dW of every layer + dX
    of every layer but the first."""
    layers, k = [], cfg.state_dim
    for h in cfg.hidden:
        layers.append((h, k))
        k = h
    if cfg.dueling:
        layers += [(2 * cfg.stream, k), (1 + cfg.n_actions, cfg.stream)]
    else:
        layers.append((cfg.n_actions, k))
    fwd = sum(o * i for o, i in layers)
    dx = sum(o * i for o, i in layers[1:])
    nets = 3 if cfg.double_dqn else 2
    return 2 * batch * nets * fwd, 2 * batch * (fwd + dx)


def tensor_peak(peaks, precision):
    """The tensor-core roofline of the step's contractions: kind::tf32 tcgen05 MMAs (half the
    measured bf16 dense rate, the nominal tf32 / bf16 ratio), three products per FP32-accurate
    product (hi.hi + hi.lo + lo.hi) in the fp32 mode, one in the tf32 / bf16 modes; the
    sustained bf16 figure since the kernels run inside a long step."""
    bf16 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1352.0)))
    tf32 = bf16 * 0.5
    return (tf32 / 3.0 if precision == "fp32" else tf32), bf16


def step_roofline(cfg, binding, batch, flops, ms_per_step, kb, peaks, peaks_kind, traffic,
                  precision="fp32"):
    peak, bf16 = tensor_peak(peaks, precision)
    achieved = flops / (ms_per_step / 1000.0) / 1e12
    fwd, bwd = flop_parts(cfg, batch)
    kernels = []
    # the tensor-core kernels of the large-batch step (tc_big.cuh): their own contractions
    nets = 3 if cfg.double_dqn else 2
    n0, n1 = (cfg.hidden[0], 2 * cfg.stream) if cfg.dueling else (cfg.hidden[0], cfg.hidden[1] if len(cfg.hidden) > 1 else 0)
    tcb_flops = {"tcb_fwd": 2 * batch * nets * n1 * n0, "tcb_dw1": 2 * batch * n1 * n0,
                 "tcb_dh0": 2 * batch * n0 * n1 + 2 * batch * n0 * (cfg.state_dim + 1)}
    for d in kb["kernels"]:
        row = dict(d)
        name = d["kernel"]
        f = next((v for k, v in tcb_flops.items() if k in name), None)
        if f is None:
            f = fwd if "fast_fwd" in name else bwd if "bwd1" in name else None
        if f is not None and d["mean_us"] > 0:
            row["flops"] = f
            row["achieved_TFLOPs"] = f / (d["mean_us"] * 1e-6) / 1e12
            row["frac"] = row["achieved_TFLOPs"] / peak
        kernels.append(row)
    return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
            "frac": achieved / peak, "traffic": traffic[0] if traffic else None,
            "traffic_cold": traffic[1] if traffic else None,
            "traffic_note": "DRAM bytes per step from ncu (profiles/traffic.json, profiles/r02/traffic/): "
                            "traffic = warm (--cache-control none, the steady state), traffic_cold = "
                            "ncu's default cache flush per kernel" if traffic else None,
            "kernel": "the train step as one unit (one CUDA graph of the kernels listed in "
                      "kernels_cupti): its algorithmic FLOPs / the timed ms_per_step",
            "kernel_avg_us": ms_per_step * 1000.0, "flops_per_launch": flops,
            "peak_note": f"measured bf16 dense {bf16:.0f} TFLOP/s sustained ({peaks_kind}) x 0.5 "
                         "(nominal tf32 / bf16 ratio)"
                         + (" / 3 (three tf32 products per FP32-accurate product)" if precision == "fp32" else "")
                         + ": the tensor-core ceiling of the step's contractions on this GPU, whichever "
                           "MMA instructions the kernels of this batch size issue",
            "kernels_cupti": {"steps": kb["steps"], "busy_us_per_step": kb["busy_us_per_step"],
                              "kernels": kernels,
                              "note": "per-kernel CUPTI durations from a separate pass after the "
                                      "timed region; fwd = every net's forward FLOPs, bwd1 = the "
                                      "backward FLOPs"}}


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline and --impl reference)
# ------------------------------------------------------------------------------------------
def time_oracle(a, batch, seconds, max_steps=None, steps_wanted=None, warmup=0):
    import oracle
    from inputs import experiences, init_params
    cfg = types.SimpleNamespace(**cfg_fields(a, batch))
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
        "impl": "reference", "metric": metric_name(a, batch), "value": v, "unit": "train_steps/s",
        "n_gpus": a.gpus, "steps": n, "warmup": min(a.warmup, 2), "ms_per_step": 1000 * el / n,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": workload_name(a, batch), "batch": batch,
                                        "capacity": a.capacity, "parallelism": "none (CPU oracle)"},
        "cpu_baseline": {"value": v, "unit": "train_steps/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "cpu": lscpu_model(), "host_nproc": os.cpu_count(),
               "threads_used": 1},
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
            if a.ring == "host_batch":   # the in-RAM replay takes host inputs (CPU-written rows)
                rp.add(**{kk: v[j:j + k] for kk, v in pool_h.items()})
            else:
                rp.add(**{kk: v[j:j + k] for kk, v in pool_d.items()}, defer=True)

    clk = ClockSampler(local).start()   # before the warm-up, so a short timed region is covered
    for i in range(W):
        add_dev(i)
        dqn.train_step(rp, batch, loss_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches_w = binding.kernel_launches()

    # ---- device-resident timed region (nothing but the steps between the two events) ------
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.mark_start()
    start.record(stream)
    for i in range(K):
        add_dev(W + i)
        dqn.train_step(rp, batch, loss_dev)
    end.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    launches = binding.kernel_launches() - launches_w
    elapsed_ms = start.elapsed_time(end)
    # per-kernel device times (CUPTI through torch.profiler) in a separate pass after the timed
    # region: the roofline's kernel shares, never the timed number
    kb = kernel_breakdown(lambda i: (add_dev(W + K + i), dqn.train_step(rp, batch, loss_dev)),
                          min(max(K, 50), 400))
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
            # the step's loss is stored by a kernel of the step straight into pinned host memory
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
                       "dqn_train_step whose loss side branch (loss_out_kernel, forked after K3 / T3b) "
                       "writes the loss into pinned host memory, "
                       "every step; slower of CUDA-event and wall time"}

    # ---- roofline: the train step as one unit (its FLOPs / the timed ms_per_step) and each
    # tensor-core kernel on its own (its FLOPs / its CUPTI mean duration) ------------------
    flops = binding.step_flops(cfg, batch)
    roofline = step_roofline(cfg, binding, batch, flops, ms_per_step, kb, peaks, peaks_kind,
                             step_traffic(f"train_step_b{batch}_{a.net}_{'ddqn' if a.ddqn else 'dqn'}"))

    # ---- gather bandwidth (metric part 2): explicit-index gather from the 1M ring --------
    gather = None
    if not a.no_gather and first_line and a.ring != "host_batch":
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
        # insert cost vs block size k (the B200 version of P:119-125, Fig. 3):
        # replay_add timed inside the library (rpl_time_adds: no binding overhead per call),
        # host-sourced from pageable numpy (copied into pinned staging), from pinned memory (the
        # insert kernel reads it across PCIe, no staging copy, for k > 4096) and device-sourced;
        # the device rows also give the insert kernel's HBM rate (CUDA events around the calls)
        ins = []
        kmax = min(1_000_000, a.capacity)
        big = experiences(kmax, seed=13, rank=rank)
        big_p = {kk: torch.from_numpy(v).pin_memory() for kk, v in big.items()}
        big_d = {kk: v.to(dev) for kk, v in big_p.items()}
        for kk_ in (1, 10, 100, 2000, 10_000, 100_000, kmax):
            row = {"k": kk_}
            n_calls = max(3, min(2000, 2_000_000 // (kk_ * 10)))
            for src, pool in (("host", big), ("pinned", big_p), ("device", big_d)):
                if src == "host" and kk_ > 65_536:   # pageable adds go through the 64K staging
                    continue
                part = {kx: v[:kk_] for kx, v in pool.items()}
                rp.time_adds(part, 2)
                torch.cuda.synchronize()
                gs.record(stream)
                sec = rp.time_adds(part, n_calls)
                ge.record(stream)
                torch.cuda.synchronize()
                t = max(sec, gs.elapsed_time(ge) / 1000.0) / n_calls
                row[f"{src}_us_per_experience"] = t * 1e6 / kk_
                row[f"{src}_GBps"] = kk_ * EXP_INPUT_BYTES / t / 1e9
            # device-sourced: bytes the insert kernel moves (inputs read + 228 B algorithmic
            # row written) over the per-call time, against the HBM peak
            row["device_hbm_GBps"] = kk_ * (EXP_INPUT_BYTES + ROW_READ_BYTES) / (
                row["device_us_per_experience"] * kk_ * 1e-6) / 1e9
            row["device_hbm_frac"] = row["device_hbm_GBps"] / peaks["hbm_gbs"]
            ins.append(row)
        gather["insert_sweep"] = ins
        gather["insert_note"] = ("per-call time of replay_add from rpl_time_adds (C loop + stream sync, "
                                 "max of host wall and CUDA-event time); host = pageable numpy (memcpy "
                                 "into pinned staging, then H2D / zero-copy), pinned = torch pinned "
                                 "tensors (k > 4096: the insert kernel reads them across PCIe); GBps = "
                                 f"{EXP_INPUT_BYTES} input bytes per experience / time; device_hbm = "
                                 f"({EXP_INPUT_BYTES} read + {ROW_READ_BYTES} row bytes written) / time")
        del big_p, big_d
        rp.check()
        # P:73 / Fig. 3 proper: single host experiences through the update-size queue
        # (update_size U): per replay_add call, block transfers included, timed in the library
        upd = []
        one = experiences(1, seed=14, rank=rank)
        for U in (1, 10, 100, 2000, 10_000):
            rq = binding.Replay(20_000, 27, device=local, update_size=U)
            rq.time_adds(one, 2000)
            sec = rq.time_adds(one, 20_000)
            upd.append({"update_size": U, "us_per_add": sec / 20_000 * 1e6})
            rq.close()
        gather["update_size_sweep"] = upd

    # ---- CPU oracle baseline (rank 0, N=1 only) ------------------------------------------
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline and first_line:
        n, el = time_oracle(a, batch, seconds=a.cpu_seconds)
        cpu = {"value": n / el, "unit": "train_steps/s", "cores": 1, "kind": "oracle",
               "sample": f"{n} oracle steps ({a.adds_per_step} inserts + one B={batch} train step "
                         f"from a {a.capacity:,}-row host ring) in {el:.1f} s, single thread, fp64",
               "cpu": lscpu_model(), "host_nproc": os.cpu_count(),
               "threads_used": 1}

    # ---- N > 1: the peer-memory exchange (dp_peer.cuh) as a second measured arm ----------
    p2p_arm = None
    if world > 1 and a.dp == "nccl" and not a.avg_period and first_line:
        p2p_arm = time_p2p_arm(a, binding, cfg, rp, batch, add_dev, W + 2 * K + 400, stream, dev)

    line = {
        "metric": metric_name(a, batch), "value": value, "unit": "train_steps/s", "n_gpus": world, "steps": K,
        "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[a.precision], "data": "synthetic",
        "config": {"workload": workload_name(a, batch), "batch": batch, "capacity": a.capacity,
                   "net": a.net, "double_dqn": a.ddqn, "adds_per_step": k,
                   "sampling": "distinct" if a.distinct else "uniform (with replacement, P:75)",
                   "state_storage": "shared (s' = next slot's s, P:141)" if a.shared_state else "s and s' per row",
                   "ring_memory": {"host": "host (pinned, read across PCIe: zero-copy in-RAM variant)",
                                   "host_batch": "host (pageable; CPU sample + gather, one H2D batch copy "
                                                 "per step: the paper's in-RAM replay)"}.get(a.ring, "device (HBM)"),
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
        "dp_p2p_arm": p2p_arm,
        "clocks": (clk.stop(), clk.summary())[1],
    }
    default_run = (batch == 128 and not a.ddqn and a.net == "dueling" and a.ring == "device" and
                   not a.distinct and not a.shared_state and a.precision == "fp32" and not a.avg_period)
    if first_line and not a.sweep and world == 1 and not a.no_c5 and default_run:
        # BASELINE configs[4] measured in the same run (the driver's default invocation), on
        # its full 1M-row, 56.6 GB byte ring: a compact copy of the --config c5 line
        line["c5"] = c5_summary(a)
    if rank == 0:
        print(json.dumps(line), flush=True)
    dqn.close()
    rp.close()
    return line


def c5_summary(a):
    a5 = argparse.Namespace(**vars(a))
    a5.steps, a5.warmup = min(a.steps, 1000), max(3, min(a.warmup, 50))
    a5.batch, a5.capacity, a5.no_cpu_baseline, a5.no_gather = 256, 1_000_000, True, False
    a5.ddqn = False
    line = run_c5(a5, emit=False)
    keep = ("metric", "value", "unit", "steps", "warmup", "ms_per_step", "dtype", "config",
            "samples_per_s", "gpu_launches", "roofline", "e2e", "gather", "clocks")
    return {k: line[k] for k in keep}


def time_p2p_arm(a, binding, cfg, rp, batch, add_dev, i0, stream, dev):
    """A second learner on the same shards whose gradient mean + SGD runs in the peer-memory
    kernel (dqn_attach_peers) instead of NCCL: the same K steps, timed the same way (max over
    ranks).  Its failure mode is bounded: a missing peer ends the kernel's flag wait after ~10 s
    with RPL_ENCCL at the check, reported here instead of a number."""
    import torch
    import torch.distributed as dist
    from inputs import init_params
    from paper_1801_03138_b200 import dp
    K, W = a.steps, a.warmup
    dqn = binding.DQN(cfg, init_params(27, 8, cfg.hidden, cfg.dueling, cfg.stream, seed=3),
                      device=torch.cuda.current_device())
    try:
        used = dp.attach_auto(dqn)
        if used != "p2p":
            return {"unavailable": "peer mapping between the ranks' GPUs failed; NCCL used instead"}
        for i in range(W):
            add_dev(i0 + i)
            dqn.train_step(rp, batch)
        torch.cuda.synchronize()
        dist.barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        for i in range(K):
            add_dev(i0 + W + i)
            dqn.train_step(rp, batch)
        e.record(stream)
        torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        ok = dqn.check() == binding.RPL_OK
        t = torch.tensor([ms, 0.0 if ok else 1.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, bad = t[0].item(), t[1].item()
        if bad:
            return {"error": "a rank's exchange failed (sticky RPL_ENCCL)"}
        return {"value": dist.get_world_size() * K / (ms / 1000.0), "unit": "train_steps/s",
                "ms_per_step": ms / K, "steps": K,
                "note": "gradient mean + SGD over NVLink peer memory in one kernel per step "
                        "(dp_peer.cuh), same shards and batch as the NCCL line"}
    except Exception as ex:   # reported, never fatal to the NCCL line
        return {"error": f"{type(ex).__name__}: {ex}"}
    finally:
        dqn.close()


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
    import types
    import oracle
    from inputs import init_params
    # plain fields (no product import on the oracle arm)
    cfg = types.SimpleNamespace(state_dim=C5_D, n_actions=8, dueling=True, hidden=(128,), stream=512)
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


def run_c5(a, emit=True):
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

    clk = ClockSampler(local).start()   # before the warm-up, so a short timed region is covered
    for i in range(W):
        add_dev(i)
        dqn.train_step(rp, batch, loss_dev)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches_w = binding.kernel_launches()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk.mark_start()
    start.record(stream)
    for i in range(K):
        add_dev(W + i)
        dqn.train_step(rp, batch, loss_dev)
    end.record(stream)
    torch.cuda.synchronize()
    clk.mark_end()
    launches = binding.kernel_launches() - launches_w
    elapsed_ms = start.elapsed_time(end)
    # per-kernel CUPTI durations in a separate pass (the roofline's kernel shares)
    kb = kernel_breakdown(lambda i: (add_dev(W + K + i), dqn.train_step(rp, batch, loss_dev)),
                          min(max(K, 50), 200))
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
    ms_per_step = elapsed_ms / K
    # 97% of the step's FLOPs are layer 0, run as bf16 x3 tcgen05 MMAs (FP32-accurate): the
    # denominator is the measured bf16 dense peak / 3 (the FP32-emulation rate), the sustained
    # figure since the kernel runs inside a long step
    bf16 = float(peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops", 1352.0)))
    nterm = {"fp32": 3, "tf32": 2, "bf16": 1}[a.precision]
    peak_emu = bf16 / nterm
    achieved = flops / (ms_per_step / 1000.0) / 1e12
    roofline = {"bound": "tensor", "achieved": achieved, "peak": peak_emu, "unit": "TFLOP/s",
                "frac": achieved / peak_emu,
                "traffic": load_traffic().get(f"c5_step_b{batch}_{'ddqn' if a.ddqn else 'dqn'}"),
                "kernel": "the whole train step (one CUDA graph: Philox gather, wide_l0_kernel, "
                          "wide_reduce, the fast kernels for the layers above layer 0, wide_dw0_kernel "
                          "+ SGD): its algorithmic FLOPs / the timed ms_per_step",
                "kernel_avg_us": ms_per_step * 1000.0, "flops_per_launch": flops,
                "kernels_cupti": kb,
                "peak_note": f"measured bf16 dense {bf16:.0f} TFLOP/s ({peaks_kind}) / {nterm}: layer 0 runs "
                             f"{nterm} bf16 MMA(s) per product (hi/mid/lo split of the fp32 operand, "
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
               "cpu": lscpu_model(), "host_nproc": os.cpu_count(),
               "threads_used": 1}
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
        "cpu_baseline": cpu, "e2e": e2e, "gather": gather, "clocks": (clk.stop(), clk.summary())[1],
    }
    if rank == 0 and emit:
        print(json.dumps(line), flush=True)
    dqn.close()
    rp.close()
    return line


def spawn_ranks(n: int) -> int:
    """`--gpus N` without a torchrun environment: launch the N ranks here (one process per GPU,
    torch.distributed.run on 127.0.0.1, the driver's own launch form) and return their exit
    code; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    a = parse()
    if a.impl == "reference":   # rank 0 alone times the oracle (the other ranks exit at once)
        run_reference(a)
        return
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(a.gpus))
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
