"""Thin ctypes binding of ``include/ingpu_replay.h`` (argument marshalling only).

Every step of the path runs in ``lib/libingpu_replay.so`` (hand-written sm_100a CUDA).
There is no CPU fallback: if the library is missing this module raises at import, and
every call that needs a GPU fails loudly with the library's status and message.

torch is used only for device memory (CUDA tensors as caller-owned buffers) and streams.
Names follow the C-ABI: ``replay_create``, ``replay_add``, ``replay_sample``,
``dqn_train_step``, ``sync_target`` (+ the handle classes ``Replay`` and ``DQN``).
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libingpu_replay.so")

RPL_OK, RPL_NOT_READY = 0, 1
RPL_EINVAL, RPL_ENOMEM, RPL_ECORRUPT, RPL_ENUMERIC = -1, -2, -3, -4
RPL_ECUDA, RPL_ENCCL, RPL_ESTATE = -5, -6, -7
RPL_HOST, RPL_DEVICE, RPL_DEVICE_DEFER = 0, 1, 2
RPL_ONLINE, RPL_TARGET, RPL_GRAD = 0, 1, 2
RPL_F32, RPL_U8 = 0, 1
RPL_RING_DEVICE, RPL_RING_HOST, RPL_RING_HOST_BATCH = 0, 1, 2
RPL_PREC_FP32, RPL_PREC_TF32, RPL_PREC_BF16 = 0, 1, 2
(RPL_DBG_IDX, RPL_DBG_S, RPL_DBG_S_NEXT, RPL_DBG_A, RPL_DBG_R, RPL_DBG_DONE, RPL_DBG_Q,
 RPL_DBG_QT_NEXT, RPL_DBG_QO_NEXT, RPL_DBG_Y, RPL_DBG_ASTAR, RPL_DBG_H, RPL_DBG_LOSS,
 RPL_DBG_TRACE) = range(14)

EXPORTS = [
    "replay_create", "replay_destroy", "replay_add", "replay_sample", "replay_gather",
    "replay_size", "replay_state", "replay_flush_queue", "replay_queued", "replay_ring_bytes",
    "dqn_param_count",
    "dqn_create", "dqn_destroy",
    "dqn_train_step", "sync_target", "dqn_get_params", "dqn_set_params", "dqn_step_count",
    "dqn_debug_export", "rpl_nccl_unique_id", "dqn_attach_nccl", "dqn_peer_handle",
    "dqn_attach_peers", "dqn_detach_peers", "rpl_dp_emulate", "rpl_check",
    "rpl_last_error", "rpl_kernel_launches", "rpl_time_adds",
]


class RplError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"status {status}: {msg}")
        self.status = status


class _ReplayOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("cuda_stream", C.c_void_p), ("burn_in", C.c_int64),
                ("seed", C.c_uint64), ("rank", C.c_uint32), ("max_host_add", C.c_int64),
                ("state_dtype", C.c_int32), ("sampling", C.c_int32), ("state_sharing", C.c_int32),
                ("ring_memory", C.c_int32), ("update_size", C.c_int64), ("storage", C.c_void_p),
                ("storage_bytes", C.c_size_t)]


class _Batch(C.Structure):
    _fields_ = [("s", C.c_void_p), ("s_next", C.c_void_p), ("a", C.c_void_p), ("r", C.c_void_p),
                ("done", C.c_void_p), ("idx", C.c_void_p)]


class _DqnConfig(C.Structure):
    _fields_ = [("device", C.c_int32), ("cuda_stream", C.c_void_p), ("state_dim", C.c_int32),
                ("n_actions", C.c_int32), ("dueling", C.c_int32), ("n_hidden", C.c_int32),
                ("hidden", C.c_int32 * 4), ("stream", C.c_int32), ("double_dqn", C.c_int32),
                ("gamma", C.c_float), ("lr", C.c_float), ("huber_kappa", C.c_float),
                ("sync_period", C.c_int64), ("max_batch", C.c_int32), ("avg_period", C.c_int64),
                ("precision", C.c_int32)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_1801_03138_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "replay_create": (C.c_int, [i64, i32, C.POINTER(_ReplayOpts), C.POINTER(P)]),
        "replay_destroy": (C.c_int, [P]),
        "replay_add": (C.c_int, [P, i64, P, P, P, P, P, C.c_int]),
        "replay_sample": (C.c_int, [P, i32, C.POINTER(_Batch)]),
        "replay_gather": (C.c_int, [P, i64, P, C.POINTER(_Batch)]),
        "replay_size": (C.c_int, [P, C.POINTER(i64)]),
        "replay_flush_queue": (C.c_int, [P, C.POINTER(i64)]),
        "replay_ring_bytes": (C.c_int, [i64, i32, C.POINTER(_ReplayOpts), C.POINTER(C.c_size_t)]),
        "replay_queued": (C.c_int, [P, C.POINTER(i64)]),
        "replay_state": (C.c_int, [P, C.POINTER(i64), C.POINTER(i64), C.POINTER(u64),
                                   C.POINTER(u64), C.POINTER(u64)]),
        "dqn_param_count": (C.c_int, [C.POINTER(_DqnConfig), C.POINTER(i64)]),
        "dqn_create": (C.c_int, [C.POINTER(_DqnConfig), P, C.POINTER(P)]),
        "dqn_destroy": (C.c_int, [P]),
        "dqn_train_step": (C.c_int, [P, P, i32, P]),
        "sync_target": (C.c_int, [P]),
        "dqn_get_params": (C.c_int, [P, C.c_int, P, i64]),
        "dqn_set_params": (C.c_int, [P, C.c_int, P, i64]),
        "dqn_step_count": (C.c_int, [P, C.POINTER(i64)]),
        "dqn_debug_export": (C.c_int, [P, C.c_int, P, i64]),
        "rpl_nccl_unique_id": (C.c_int, [P]),
        "dqn_attach_nccl": (C.c_int, [P, i32, i32, P]),
        "dqn_peer_handle": (C.c_int, [P, P]),
        "dqn_attach_peers": (C.c_int, [P, i32, i32, P]),
        "dqn_detach_peers": (C.c_int, [P]),
        "rpl_dp_emulate": (C.c_int, [i32, i64, P, P, P, P, P, P, C.c_float, u64, i32]),
        "rpl_check": (C.c_int, [P, C.c_int]),
        "rpl_last_error": (C.c_char_p, []),
        "rpl_kernel_launches": (C.c_uint64, []),
        "rpl_time_adds": (C.c_int, [P, i64, i64, P, P, P, P, P, C.c_int, C.POINTER(C.c_double)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


_L = _load()


def lib():
    return _L


def last_error() -> str:
    return _L.rpl_last_error().decode(errors="replace")


def kernel_launches() -> int:
    return int(_L.rpl_kernel_launches())


def _ok(status: int, allow=(RPL_OK,)):
    if status not in allow:
        raise RplError(status, last_error())
    return status


def _dptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _host(x, dtype):
    """x as a C-contiguous numpy array of dtype (no copy when it already is one)."""
    if type(x) is np.ndarray and x.dtype == dtype and x.flags.c_contiguous:
        return x
    return np.ascontiguousarray(np.asarray(x), dtype)


def _torch():
    import torch
    return torch


def _stream_handle(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


# ==========================================================================================
# replay
# ==========================================================================================
class Replay:
    """Handle of the device FIFO replay (``replay_create``)."""

    def __init__(self, capacity: int, state_dim: int, *, device: int = 0, stream=None,
                 burn_in: int = 1, seed: int = 2, rank: int = 0, max_host_add: int = 0,
                 state_dtype: str = "f32", sampling: str = "uniform", shared_state: bool = False,
                 ring_memory: str = "device", update_size: int = 0, storage=None):
        """storage: optional caller-owned CUDA tensor holding the ring rows (at least
        Replay.ring_bytes(...) bytes; kept referenced by this object)."""
        torch = _torch()
        if not torch.cuda.is_available():
            raise RplError(RPL_ECUDA, "no CUDA device (the in-GPU replay has no CPU fallback)")
        self.device = device
        self.u8 = state_dtype == "u8"
        self.state_np = np.uint8 if self.u8 else np.float32
        self.state_torch = torch.uint8 if self.u8 else torch.float32
        with torch.cuda.device(device):
            self._stream = _stream_handle(stream)
        o = _ReplayOpts(device, self._stream, burn_in, seed, rank, max_host_add,
                        RPL_U8 if self.u8 else RPL_F32, 1 if sampling == "distinct" else 0,
                        1 if shared_state else 0,
                        {"device": RPL_RING_DEVICE, "host": RPL_RING_HOST,
                         "host_batch": RPL_RING_HOST_BATCH}[ring_memory], update_size,
                        None if storage is None else storage.data_ptr(),
                        0 if storage is None else storage.numel() * storage.element_size())
        self._storage = storage
        self.shared_state = shared_state
        self.ring_memory = ring_memory
        h = C.c_void_p()
        _ok(_L.replay_create(capacity, state_dim, C.byref(o), C.byref(h)))
        self._h = h
        self.capacity, self.state_dim, self.burn_in = capacity, state_dim, burn_in

    def close(self):
        if getattr(self, "_h", None):
            _L.replay_destroy(self._h)
            self._h = None
        self._storage = None

    @staticmethod
    def ring_bytes(capacity: int, state_dim: int, state_dtype: str = "f32", shared_state: bool = False) -> int:
        """replay_ring_bytes: the size a caller-provided `storage` tensor needs."""
        o = _ReplayOpts()
        o.state_dtype = RPL_U8 if state_dtype == "u8" else RPL_F32
        o.state_sharing = 1 if shared_state else 0
        n = C.c_size_t()
        _ok(_L.replay_ring_bytes(capacity, state_dim, C.byref(o), C.byref(n)))
        return n.value

    __del__ = close

    @property
    def handle(self):
        return self._h

    def add(self, s, a, r, s_next, done, defer: bool = False) -> int:
        """replay_add: numpy / CPU tensors -> RPL_HOST; CUDA tensors -> RPL_DEVICE, or
        RPL_DEVICE_DEFER with defer=True (the tensors must stay unchanged until the next
        call on this replay / the next train step on it; a reference is held until then)."""
        if type(s) is not np.ndarray and isinstance(s, _torch().Tensor) and s.is_cuda:
            torch = _torch()
            if s_next is None:   # shared-state replay: s' is the next experience's s
                s_next = s[:0]
            ts = [s.contiguous(), a.contiguous(), r.contiguous(), s_next.contiguous(),
                  done.contiguous()]
            assert ts[0].dtype == self.state_torch and ts[3].dtype == self.state_torch
            assert ts[1].dtype == torch.int32
            assert ts[2].dtype == torch.float32 and ts[4].dtype == torch.uint8
            k = ts[1].numel()
            ptrs = [_dptr(t) for t in ts]
            if ts[3].numel() == 0:
                ptrs[3] = None
            rc = _ok(_L.replay_add(self._h, k, *ptrs,
                                   RPL_DEVICE_DEFER if defer else RPL_DEVICE))
            self._deferred = ts if defer else None
            return rc
        sn = self.state_np
        arrs = (_host(s, sn), _host(a, np.int32), _host(r, np.float32),
                None if s_next is None else _host(s_next, sn), _host(done, np.uint8))
        k = arrs[1].size
        st = _L.replay_add(self._h, k, arrs[0].ctypes.data, arrs[1].ctypes.data, arrs[2].ctypes.data,
                           None if arrs[3] is None else arrs[3].ctypes.data, arrs[4].ctypes.data, RPL_HOST)
        return st if st == RPL_OK else _ok(st)

    def time_adds(self, e: dict, n_calls: int) -> float:
        """rpl_time_adds: wall seconds of n_calls replay_add calls of the experiences `e` (host
        numpy arrays -> RPL_HOST, CUDA tensors -> RPL_DEVICE), timed inside the library."""
        torch = _torch()
        if isinstance(e["a"], torch.Tensor) and e["a"].is_cuda:
            ts = [e[k].contiguous() for k in ("s", "a", "r", "s_next", "done")]
            ptrs, mem, keep = [_dptr(t) for t in ts], RPL_DEVICE, ts
        else:
            sn = self.state_np
            arrs = (_host(e["s"], sn), _host(e["a"], np.int32), _host(e["r"], np.float32),
                    _host(e["s_next"], sn), _host(e["done"], np.uint8))
            ptrs, mem, keep = [x.ctypes.data for x in arrs], RPL_HOST, arrs
        sec = C.c_double(0.0)
        _ok(_L.rpl_time_adds(self._h, n_calls, len(e["a"]), *ptrs, mem, C.byref(sec)))
        del keep
        return sec.value

    def add_many(self, e: dict, chunk: int = 65536):
        n = len(e["a"])
        chunk = min(chunk, self.capacity)
        for i in range(0, n, chunk):
            sl = slice(i, min(n, i + chunk))
            self.add(e["s"][sl], e["a"][sl], e["r"][sl], e["s_next"][sl], e["done"][sl])

    def _out(self, n, out):
        torch = _torch()
        if out is None:
            dev = torch.device("cuda", self.device)
            D = self.state_dim
            st = self.state_torch
            out = dict(s=torch.empty(n, D, dtype=st, device=dev),
                       s_next=torch.empty(n, D, dtype=st, device=dev),
                       a=torch.empty(n, dtype=torch.int32, device=dev),
                       r=torch.empty(n, device=dev),
                       done=torch.empty(n, dtype=torch.uint8, device=dev),
                       idx=torch.empty(n, dtype=torch.int32, device=dev))
        b = _Batch(*[_dptr(out.get(k)) for k in ("s", "s_next", "a", "r", "done", "idx")])
        return out, b

    def sample(self, batch: int, out: dict | None = None):
        """replay_sample -> dict of CUDA tensors, or None while burning in."""
        out, b = self._out(batch, out)
        st = _ok(_L.replay_sample(self._h, batch, C.byref(b)), (RPL_OK, RPL_NOT_READY))
        return None if st == RPL_NOT_READY else out

    def gather(self, idx, out: dict | None = None):
        n = idx.numel()
        out, b = self._out(n, out)
        _ok(_L.replay_gather(self._h, n, _dptr(idx), C.byref(b)))
        return out

    @property
    def size(self) -> int:
        v = C.c_int64()
        _ok(_L.replay_size(self._h, C.byref(v)))
        return v.value

    @property
    def queued(self) -> int:
        """Experiences waiting in the update-size queue (update_size > 0)."""
        v = C.c_int64()
        _ok(_L.replay_queued(self._h, C.byref(v)))
        return v.value

    def flush_queue(self) -> int:
        """replay_flush_queue: write the queued experiences as a partial block."""
        v = C.c_int64()
        _ok(_L.replay_flush_queue(self._h, C.byref(v)))
        return v.value

    def state(self) -> dict:
        c, s = C.c_int64(), C.c_int64()
        t, e, h = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _ok(_L.replay_state(self._h, C.byref(c), C.byref(s), C.byref(t), C.byref(e), C.byref(h)))
        return dict(cursor=c.value, size=s.value, total=t.value, events=e.value,
                    h2d_bytes=h.value)

    def check(self) -> int:
        return _L.rpl_check(self._h, 0)


# ==========================================================================================
# learner
# ==========================================================================================
@dataclass
class DQNConfig:
    state_dim: int = 27
    n_actions: int = 8
    dueling: bool = True
    hidden: tuple = (128,)
    stream: int = 512
    double_dqn: bool = False
    gamma: float = 0.99
    lr: float = 1e-4
    huber_kappa: float = 1.0
    sync_period: int = 10_000
    max_batch: int = 4096
    avg_period: int = 0       # DP: 0 = gradient mean every step; K = parameter mean every K steps
    precision: str = "fp32"   # "fp32" (FP32-accurate, default) | "tf32" | "bf16" (tensor-core products)

    def _c(self, device=0, stream=None) -> _DqnConfig:
        c = _DqnConfig()
        c.device = device
        c.cuda_stream = stream
        c.state_dim, c.n_actions = self.state_dim, self.n_actions
        c.dueling, c.n_hidden = int(self.dueling), len(self.hidden)
        for i, h in enumerate(self.hidden[:4]):
            c.hidden[i] = h
        c.stream = self.stream if self.dueling else 0
        c.double_dqn = int(self.double_dqn)
        c.gamma, c.lr, c.huber_kappa = self.gamma, self.lr, self.huber_kappa
        c.sync_period, c.max_batch = self.sync_period, self.max_batch
        c.avg_period = self.avg_period
        c.precision = {"fp32": RPL_PREC_FP32, "tf32": RPL_PREC_TF32, "bf16": RPL_PREC_BF16}[self.precision]
        return c

    @property
    def param_count(self) -> int:
        n = C.c_int64()
        _ok(_L.dqn_param_count(C.byref(self._c()), C.byref(n)))
        return n.value


class DQN:
    """Handle of the device learner (``dqn_create``)."""

    def __init__(self, cfg: DQNConfig, params, *, device: int = 0, stream=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise RplError(RPL_ECUDA, "no CUDA device (the fused train step has no CPU fallback)")
        self.cfg = cfg
        self.device = device
        with torch.cuda.device(device):
            self._stream = _stream_handle(stream)
        p = np.ascontiguousarray(np.asarray(params, np.float32))
        self.P = cfg.param_count
        if p.size != self.P:
            raise ValueError(f"params has {p.size} floats, the config needs {self.P}")
        h = C.c_void_p()
        _ok(_L.dqn_create(C.byref(cfg._c(device, self._stream)), p.ctypes.data_as(C.c_void_p),
                          C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            _L.dqn_destroy(self._h)
            self._h = None

    __del__ = close

    def train_step(self, replay: Replay, batch: int, loss_out=None) -> int:
        """dqn_train_step; returns RPL_OK or RPL_NOT_READY (burn-in)."""
        st = _L.dqn_train_step(self._h, replay._h, batch, None if loss_out is None else loss_out.data_ptr())
        if st != RPL_OK:
            _ok(st, (RPL_OK, RPL_NOT_READY))
        if st == RPL_OK:
            self._last_u8 = replay.u8
        return st

    def sync_target(self):
        _ok(_L.sync_target(self._h))

    def get_params(self, which: int = RPL_ONLINE) -> np.ndarray:
        out = np.empty(self.P, np.float32)
        _ok(_L.dqn_get_params(self._h, which, out.ctypes.data_as(C.c_void_p), self.P))
        return out

    def set_params(self, params, which: int = RPL_ONLINE):
        p = np.ascontiguousarray(np.asarray(params, np.float32))
        _ok(_L.dqn_set_params(self._h, which, p.ctypes.data_as(C.c_void_p), p.size))

    @property
    def steps(self) -> int:
        v = C.c_int64()
        _ok(_L.dqn_step_count(self._h, C.byref(v)))
        return v.value

    def debug(self, what: int, batch: int, hidden_units: int = 0) -> np.ndarray:
        D, A = self.cfg.state_dim, self.cfg.n_actions
        sd = np.uint8 if getattr(self, "_last_u8", False) else np.float32
        spec = {RPL_DBG_IDX: (np.int32, (batch,)), RPL_DBG_S: (sd, (batch, D)),
                RPL_DBG_S_NEXT: (sd, (batch, D)), RPL_DBG_A: (np.int32, (batch,)),
                RPL_DBG_R: (np.float32, (batch,)), RPL_DBG_DONE: (np.uint8, (batch,)),
                RPL_DBG_Q: (np.float32, (batch, A)), RPL_DBG_QT_NEXT: (np.float32, (batch, A)),
                RPL_DBG_QO_NEXT: (np.float32, (batch, A)), RPL_DBG_Y: (np.float32, (batch,)),
                RPL_DBG_ASTAR: (np.int32, (batch,)),
                RPL_DBG_H: (np.float32, (batch, hidden_units)),
                RPL_DBG_LOSS: (np.float32, (1,)),
                RPL_DBG_TRACE: (np.uint64, (8, 2048, 8))}[what]
        out = np.empty(spec[1], spec[0])
        _ok(_L.dqn_debug_export(self._h, what, out.ctypes.data_as(C.c_void_p), out.nbytes))
        return out

    def attach_nccl(self, rank: int, world: int, uid: bytes):
        buf = C.create_string_buffer(bytes(uid), 128)
        _ok(_L.dqn_attach_nccl(self._h, rank, world, buf))

    def peer_handle(self) -> bytes:
        """dqn_peer_handle: this learner's 64-byte exchange-buffer IPC handle."""
        buf = C.create_string_buffer(64)
        _ok(_L.dqn_peer_handle(self._h, buf))
        return buf.raw

    def attach_peers(self, rank: int, world: int, handles: bytes):
        """dqn_attach_peers: `handles` = every rank's peer_handle(), concatenated in rank order."""
        assert len(handles) == 64 * world
        buf = C.create_string_buffer(bytes(handles), 64 * world)
        _ok(_L.dqn_attach_peers(self._h, rank, world, buf))

    def detach_peers(self):
        _ok(_L.dqn_detach_peers(self._h))

    def check(self) -> int:
        return _L.rpl_check(self._h, 1)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _ok(_L.rpl_nccl_unique_id(buf))
    return buf.raw


# C-ABI names (functional spelling over the handle classes)
def replay_create(capacity: int, state_dim: int, **opts) -> Replay:
    return Replay(capacity, state_dim, **opts)


def replay_add(replay: Replay, s, a, r, s_next, done) -> int:
    return replay.add(s, a, r, s_next, done)


def replay_sample(replay: Replay, batch: int, out=None):
    return replay.sample(batch, out)


def dqn_train_step(dqn: DQN, replay: Replay, batch: int, loss_out=None) -> int:
    return dqn.train_step(replay, batch, loss_out)


def sync_target(dqn: DQN):
    dqn.sync_target()


def hidden_units(cfg: DQNConfig) -> int:
    return sum(cfg.hidden) + (2 * cfg.stream if cfg.dueling else 0)


def step_flops(cfg: DQNConfig, batch: int) -> int:
    """Algorithmic FLOPs of one train step (2 per multiply-add):
    forward(online, s) + forward(target, s') [+ forward(online, s') for Double DQN]
    + backward (dW of every layer, dX of every layer but the first)."""
    macs_fwd, macs_dx, k = 0, 0, cfg.state_dim
    layers = []
    for h in cfg.hidden:
        layers.append((h, k)); k = h
    if cfg.dueling:
        layers.append((2 * cfg.stream, k))
        layers.append((1 + cfg.n_actions, cfg.stream))  # block-diagonal head: S inputs each
    else:
        layers.append((cfg.n_actions, k))
    for i, (o, n_in) in enumerate(layers):
        macs_fwd += o * n_in
        if i > 0:
            macs_dx += o * n_in
    nets = 3 if cfg.double_dqn else 2
    return 2 * batch * (nets * macs_fwd + macs_fwd + macs_dx)
