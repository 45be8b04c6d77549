"""ctypes marshalling for ``oracle/liboracle.so`` (TEST INFRASTRUCTURE ONLY).

Argument marshalling only: all arithmetic is in ``oracle/oracle.c``.  Parity
unpinned: none -- every entry point here is pinned by ``tests/test_oracle_*.py``
(DESIGN.md "Oracle pins").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

OK, NOT_READY, EINVAL, ENOMEM, ECORRUPT, ENUMERIC = 0, 1, -1, -2, -3, -4


def build(force: bool = False) -> str:
    """Compile the oracle with plain ``gcc -O2`` (no -ffast-math)."""
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
        os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", src, "-o", _SO, "-lm"]
        )
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = C.CDLL(_SO)
        _declare(_lib)
    return _lib


class _Ring(C.Structure):
    _fields_ = [
        ("capacity", C.c_int64),
        ("state_dim", C.c_int32),
        ("row_width", C.c_int32),
        ("rows", C.POINTER(C.c_float)),
        ("cursor", C.c_int64),
        ("size", C.c_int64),
        ("total", C.c_uint64),
        ("events", C.c_uint64),
        ("distinct", C.c_int32),
        ("shared", C.c_int32),
    ]


class _RingU8(C.Structure):
    _fields_ = [
        ("capacity", C.c_int64),
        ("state_dim", C.c_int32),
        ("s", C.c_void_p),
        ("s_next", C.c_void_p),
        ("a", C.c_void_p),
        ("r", C.c_void_p),
        ("done", C.c_void_p),
        ("cursor", C.c_int64),
        ("size", C.c_int64),
        ("total", C.c_uint64),
        ("events", C.c_uint64),
        ("distinct", C.c_int32),
        ("shared", C.c_int32),
    ]


class _Net(C.Structure):
    _fields_ = [
        ("state_dim", C.c_int32),
        ("n_actions", C.c_int32),
        ("dueling", C.c_int32),
        ("n_hidden", C.c_int32),
        ("hidden", C.c_int32 * 4),
        ("stream", C.c_int32),
    ]


class _Learner(C.Structure):
    _fields_ = [
        ("net", _Net),
        ("online", C.POINTER(C.c_float)),
        ("target", C.POINTER(C.c_float)),
        ("gamma", C.c_double),
        ("kappa", C.c_double),
        ("lr", C.c_double),
        ("double_dqn", C.c_int32),
        ("burn_in", C.c_int64),
        ("sync_period", C.c_int64),
        ("seed", C.c_uint64),
        ("rank", C.c_uint32),
        ("step", C.c_int64),
    ]


_P = C.c_void_p


def _declare(L):
    L.oracle_philox4x32_10.argtypes = [_P, _P, _P]
    L.oracle_sample_indices.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int64, C.c_int32, _P]
    L.oracle_sample_distinct.argtypes = [C.c_uint64, C.c_uint32, C.c_uint64, C.c_int64, C.c_int32, _P]
    L.oracle_sample_distinct.restype = C.c_int
    L.oracle_ring_init.argtypes = [C.POINTER(_Ring), C.c_int64, C.c_int32]
    L.oracle_ring_init.restype = C.c_int
    L.oracle_ring_free.argtypes = [C.POINTER(_Ring)]
    L.oracle_ring_set_shared.argtypes = [C.POINTER(_Ring)]
    L.oracle_ring_set_shared.restype = C.c_int
    L.oracle_ring_add.argtypes = [C.POINTER(_Ring), C.c_int64, _P, _P, _P, _P, _P]
    L.oracle_ring_add.restype = C.c_int
    L.oracle_queue_init.argtypes = [C.POINTER(_Queue), C.c_int64, C.c_int32]
    L.oracle_queue_init.restype = C.c_int
    L.oracle_queue_free.argtypes = [C.POINTER(_Queue)]
    L.oracle_queue_add.argtypes = [C.POINTER(_Queue), C.POINTER(_Ring), C.c_int64, _P, _P, _P, _P, _P]
    L.oracle_queue_add.restype = C.c_int
    L.oracle_queue_flush.argtypes = [C.POINTER(_Queue), C.POINTER(_Ring)]
    L.oracle_queue_flush.restype = C.c_int64
    L.oracle_ring_gather.argtypes = [C.POINTER(_Ring), C.c_int32, _P, _P, _P, _P, _P, _P]
    L.oracle_ring_gather.restype = C.c_int
    L.oracle_ring_sample.argtypes = [C.POINTER(_Ring), C.c_int64, C.c_uint64, C.c_uint32,
                                     C.c_int32, _P, _P, _P, _P, _P, _P]
    L.oracle_ring_sample.restype = C.c_int
    L.oracle_ring_u8_init.argtypes = [C.POINTER(_RingU8), C.c_int64, C.c_int32]
    L.oracle_ring_u8_init.restype = C.c_int
    L.oracle_ring_u8_free.argtypes = [C.POINTER(_RingU8)]
    L.oracle_ring_u8_add.argtypes = [C.POINTER(_RingU8), C.c_int64, _P, _P, _P, _P, _P]
    L.oracle_ring_u8_add.restype = C.c_int
    L.oracle_ring_u8_gather.argtypes = [C.POINTER(_RingU8), C.c_int32, _P, _P, _P, _P, _P, _P]
    L.oracle_ring_u8_gather.restype = C.c_int
    L.oracle_ring_u8_sample.argtypes = [C.POINTER(_RingU8), C.c_int64, C.c_uint64, C.c_uint32,
                                        C.c_int32, _P, _P, _P, _P, _P, _P]
    L.oracle_ring_u8_sample.restype = C.c_int
    L.oracle_u8_input.argtypes = [C.c_int64, _P, _P]
    L.oracle_param_count.argtypes = [C.POINTER(_Net)]
    L.oracle_param_count.restype = C.c_int64
    L.oracle_hidden_units.argtypes = [C.POINTER(_Net)]
    L.oracle_hidden_units.restype = C.c_int64
    L.oracle_huber.argtypes = [C.c_double, C.c_double]
    L.oracle_huber.restype = C.c_double
    L.oracle_huber_grad.argtypes = [C.c_double, C.c_double]
    L.oracle_huber_grad.restype = C.c_double
    L.oracle_dqn_loss_grad.argtypes = [C.POINTER(_Net), _P, _P, C.c_int32, _P, _P, _P, _P, _P,
                                       C.c_double, C.c_double, C.c_int, _P, _P, _P, _P,
                                       _P, _P, _P, _P, _P, _P, _P]
    L.oracle_dqn_loss_grad.restype = C.c_int
    L.oracle_sgd.argtypes = [C.c_int64, _P, _P, C.c_double]
    L.oracle_dp_mean_sgd.argtypes = [C.c_int32, C.c_int64, _P, _P, C.c_double, _P]
    L.oracle_learner_step.argtypes = [C.POINTER(_Ring), C.POINTER(_Learner), C.c_int32, _P, _P]
    L.oracle_learner_step.restype = C.c_int
    L.oracle_sync_target.argtypes = [C.POINTER(_Learner)]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


# ------------------------------------------------------------------------------------
# Philox and the sampler
# ------------------------------------------------------------------------------------
def philox4x32_10(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32).copy()
    k = np.asarray(key, dtype=np.uint32).copy()
    out = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return out


def sample_indices(seed: int, rank: int, event: int, n: int, batch: int) -> np.ndarray:
    idx = np.zeros(batch, dtype=np.int32)
    lib().oracle_sample_indices(seed, rank, event, n, batch, _ptr(idx))
    return idx


def sample_distinct(seed: int, rank: int, event: int, n: int, batch: int) -> np.ndarray:
    """oracle_sample_distinct: the first `batch` distinct values of the index stream."""
    idx = np.zeros(batch, dtype=np.int32)
    rc = lib().oracle_sample_distinct(seed, rank, event, n, batch, _ptr(idx))
    if rc != OK:
        raise ValueError(f"oracle_sample_distinct rc={rc}")
    return idx


# ------------------------------------------------------------------------------------
# The replay ring (paper layout: packed 2D+3 floats per row)
# ------------------------------------------------------------------------------------
class _Queue(C.Structure):
    _fields_ = [
        ("update_size", C.c_int64),
        ("queued", C.c_int64),
        ("state_dim", C.c_int32),
        ("s", C.POINTER(C.c_float)),
        ("s_next", C.POINTER(C.c_float)),
        ("r", C.POINTER(C.c_float)),
        ("a", C.POINTER(C.c_int32)),
        ("done", C.POINTER(C.c_uint8)),
    ]


class Ring:
    def __init__(self, capacity: int, state_dim: int, distinct: bool = False,
                 shared: bool = False, update_size: int = 0):
        self._q = None
        if update_size:   # P:73 block updates through oracle_queue_*
            self._q = _Queue()
            rc = lib().oracle_queue_init(C.byref(self._q), update_size, state_dim)
            if rc != OK:
                raise ValueError(f"oracle_queue_init rc={rc}")
        self._r = _Ring()
        rc = lib().oracle_ring_init(C.byref(self._r), capacity, state_dim)
        if rc != OK:
            raise ValueError(f"oracle_ring_init rc={rc}")
        self._r.distinct = 1 if distinct else 0
        if shared:
            lib().oracle_ring_set_shared(C.byref(self._r))
        self.state_dim = state_dim

    def __del__(self):
        if getattr(self, "_r", None) is not None and self._r.rows:
            lib().oracle_ring_free(C.byref(self._r))
        if getattr(self, "_q", None) is not None and self._q.s:
            lib().oracle_queue_free(C.byref(self._q))

    @property
    def capacity(self):
        return self._r.capacity

    @property
    def queued(self):
        return self._q.queued if self._q is not None else 0

    def flush_queue(self) -> int:
        """Write the waiting experiences as a partial block; returns how many."""
        return lib().oracle_queue_flush(C.byref(self._q), C.byref(self._r)) if self._q is not None else 0

    @property
    def cursor(self):
        return self._r.cursor

    @property
    def size(self):
        return self._r.size

    @property
    def total(self):
        return self._r.total

    @property
    def events(self):
        return self._r.events

    @events.setter
    def events(self, v):
        self._r.events = v

    def rows(self) -> np.ndarray:
        """The packed rows (capacity x (2D+3) float32), a view."""
        n = self._r.capacity * self._r.row_width
        buf = np.ctypeslib.as_array(self._r.rows, shape=(n,))
        return buf.reshape(self._r.capacity, self._r.row_width)

    def add(self, s, a, r, s_next, done) -> int:
        D = self.state_dim
        s = _c(s, np.float32).reshape(-1, D)
        k = s.shape[0]
        a = _c(a, np.int32)
        r = _c(r, np.float32)
        s_next = _c(s_next, np.float32).reshape(-1, D) if s_next is not None else None
        done = _c(done, np.uint8)
        if self._q is not None:
            return lib().oracle_queue_add(C.byref(self._q), C.byref(self._r), k, _ptr(s), _ptr(a),
                                          _ptr(r), _ptr(s_next), _ptr(done))
        return lib().oracle_ring_add(C.byref(self._r), k, _ptr(s), _ptr(a), _ptr(r),
                                     _ptr(s_next), _ptr(done))

    def add_many(self, e: dict, chunk: int = 65536) -> None:
        n = len(e["a"])
        chunk = min(chunk, self.capacity)
        for i in range(0, n, chunk):
            rc = self.add(**{k: v[i:i + chunk] for k, v in e.items()})
            if rc != OK:
                raise ValueError(f"oracle_ring_add rc={rc}")

    def gather(self, idx):
        idx = _c(idx, np.int32)
        B, D = idx.shape[0], self.state_dim
        out = dict(s=np.zeros((B, D), np.float32), a=np.zeros(B, np.int32),
                   r=np.zeros(B, np.float32), s_next=np.zeros((B, D), np.float32),
                   done=np.zeros(B, np.uint8))
        rc = lib().oracle_ring_gather(C.byref(self._r), B, _ptr(idx), _ptr(out["s"]),
                                      _ptr(out["a"]), _ptr(out["r"]), _ptr(out["s_next"]),
                                      _ptr(out["done"]))
        if rc != OK:
            raise ValueError(f"oracle_ring_gather rc={rc}")
        out["idx"] = idx
        return out

    def sample(self, burn_in: int, seed: int, rank: int, batch: int):
        """Returns (rc, batch dict or None)."""
        D = self.state_dim
        out = dict(idx=np.zeros(batch, np.int32), s=np.zeros((batch, D), np.float32),
                   a=np.zeros(batch, np.int32), r=np.zeros(batch, np.float32),
                   s_next=np.zeros((batch, D), np.float32), done=np.zeros(batch, np.uint8))
        rc = lib().oracle_ring_sample(C.byref(self._r), burn_in, seed, rank, batch,
                                      _ptr(out["idx"]), _ptr(out["s"]), _ptr(out["a"]),
                                      _ptr(out["r"]), _ptr(out["s_next"]), _ptr(out["done"]))
        return rc, (out if rc == OK else None)


class RingU8:
    """Byte-state replay (SURVEY config 5): oracle_ring_u8_* (same FIFO / sampler / gather
    as Ring over uint8 states)."""

    def __init__(self, capacity: int, state_dim: int, distinct: bool = False,
                 shared: bool = False):
        self._r = _RingU8()
        rc = lib().oracle_ring_u8_init(C.byref(self._r), capacity, state_dim)
        if rc != OK:
            raise ValueError(f"oracle_ring_u8_init rc={rc}")
        self._r.distinct = 1 if distinct else 0
        self._r.shared = 1 if shared else 0
        self.state_dim = state_dim

    def __del__(self):
        if getattr(self, "_r", None) is not None and self._r.s:
            lib().oracle_ring_u8_free(C.byref(self._r))

    capacity = property(lambda self: self._r.capacity)
    cursor = property(lambda self: self._r.cursor)
    size = property(lambda self: self._r.size)
    total = property(lambda self: self._r.total)

    @property
    def events(self):
        return self._r.events

    @events.setter
    def events(self, v):
        self._r.events = v

    def add(self, s, a, r, s_next, done) -> int:
        D = self.state_dim
        s = _c(s, np.uint8).reshape(-1, D)
        return lib().oracle_ring_u8_add(C.byref(self._r), s.shape[0], _ptr(s), _ptr(_c(a, np.int32)),
                                        _ptr(_c(r, np.float32)),
                                        _ptr(_c(s_next, np.uint8).reshape(-1, D)) if s_next is not None else None,
                                        _ptr(_c(done, np.uint8)))

    def _batch(self, B):
        D = self.state_dim
        return dict(idx=np.zeros(B, np.int32), s=np.zeros((B, D), np.uint8),
                    a=np.zeros(B, np.int32), r=np.zeros(B, np.float32),
                    s_next=np.zeros((B, D), np.uint8), done=np.zeros(B, np.uint8))

    def gather(self, idx):
        idx = _c(idx, np.int32)
        out = self._batch(idx.shape[0])
        rc = lib().oracle_ring_u8_gather(C.byref(self._r), idx.shape[0], _ptr(idx), _ptr(out["s"]),
                                         _ptr(out["a"]), _ptr(out["r"]), _ptr(out["s_next"]),
                                         _ptr(out["done"]))
        if rc != OK:
            raise ValueError(f"oracle_ring_u8_gather rc={rc}")
        out["idx"] = idx
        return out

    def sample(self, burn_in: int, seed: int, rank: int, batch: int):
        """Returns (rc, batch dict or None)."""
        out = self._batch(batch)
        rc = lib().oracle_ring_u8_sample(C.byref(self._r), burn_in, seed, rank, batch,
                                         _ptr(out["idx"]), _ptr(out["s"]), _ptr(out["a"]),
                                         _ptr(out["r"]), _ptr(out["s_next"]), _ptr(out["done"]))
        return rc, (out if rc == OK else None)


def u8_input(u) -> np.ndarray:
    """oracle_u8_input: the network input x = u8 / 255 of byte states (reading Q27)."""
    u = _c(u, np.uint8)
    x = np.empty(u.shape, np.float32)
    lib().oracle_u8_input(u.size, _ptr(u), _ptr(x))
    return x


# ------------------------------------------------------------------------------------
# The network, the loss/gradient and the learner
# ------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Net:
    state_dim: int = 27
    n_actions: int = 8
    dueling: bool = True
    hidden: tuple = (128,)
    stream: int = 512

    def _c(self) -> _Net:
        n = _Net()
        n.state_dim = self.state_dim
        n.n_actions = self.n_actions
        n.dueling = int(self.dueling)
        n.n_hidden = len(self.hidden)
        for i, h in enumerate(self.hidden):
            n.hidden[i] = h
        n.stream = self.stream if self.dueling else 0
        return n

    @property
    def param_count(self) -> int:
        return int(lib().oracle_param_count(C.byref(self._c())))

    @property
    def hidden_units(self) -> int:
        return int(lib().oracle_hidden_units(C.byref(self._c())))


def huber(delta: float, kappa: float) -> float:
    return lib().oracle_huber(delta, kappa)


def huber_grad(delta: float, kappa: float) -> float:
    return lib().oracle_huber_grad(delta, kappa)


def dqn_loss_grad(net: Net, online, target, batch: dict, gamma: float, kappa: float,
                  double_dqn: bool, mask_override=None, argmax_override=None):
    """One loss/gradient evaluation (fp64).  Returns a dict with loss, grad, q_s,
    q_next_target, q_next_online, y, a_star, z (online pre-activations), on (masks)."""
    P, H, A = net.param_count, net.hidden_units, net.n_actions
    s = _c(batch["s"], np.float32)
    B = s.shape[0]
    on_w = _c(online, np.float64)
    tg_w = _c(target, np.float64)
    assert on_w.size == P and tg_w.size == P
    out = dict(grad=np.zeros(P), q_s=np.zeros((B, A)), q_next_target=np.zeros((B, A)),
               q_next_online=np.zeros((B, A)), y=np.zeros(B), a_star=np.zeros(B, np.int32),
               z=np.zeros((B, H)), on=np.zeros((B, H), np.uint8))
    loss = C.c_double(0.0)
    mo = _c(mask_override, np.uint8)
    ao = _c(argmax_override, np.int32)
    rc = lib().oracle_dqn_loss_grad(
        C.byref(net._c()), _ptr(on_w), _ptr(tg_w), B, _ptr(s), _ptr(_c(batch["a"], np.int32)),
        _ptr(_c(batch["r"], np.float32)), _ptr(_c(batch["s_next"], np.float32)),
        _ptr(_c(batch["done"], np.uint8)), gamma, kappa, int(double_dqn), _ptr(mo), _ptr(ao),
        C.byref(loss), _ptr(out["grad"]), _ptr(out["q_s"]), _ptr(out["q_next_target"]),
        _ptr(out["q_next_online"]), _ptr(out["y"]), _ptr(out["a_star"]), _ptr(out["z"]),
        _ptr(out["on"]))
    if rc != OK:
        raise ValueError(f"oracle_dqn_loss_grad rc={rc}")
    out["loss"] = loss.value
    if not double_dqn:
        out["a_star"] = None
        out["q_next_online"] = None
    return out


def sgd(w, g, lr: float) -> np.ndarray:
    w = np.array(w, dtype=np.float64)
    g = _c(g, np.float64)
    lib().oracle_sgd(w.size, _ptr(w), _ptr(g), lr)
    return w


def dp_mean_sgd(w, grads, lr: float):
    """O6: rank-order sum of the ranks' gradients / N, then SGD on the replica.
    Returns (new weights, mean gradient)."""
    w = np.array(w, dtype=np.float64)
    gs = [_c(g, np.float64) for g in grads]
    assert all(g.size == w.size for g in gs)
    arr = (C.c_void_p * len(gs))(*[g.ctypes.data for g in gs])
    mean = np.zeros_like(w)
    lib().oracle_dp_mean_sgd(len(gs), w.size, _ptr(w), C.cast(arr, C.c_void_p), lr, _ptr(mean))
    return w, mean


class Learner:
    """Burn-in gate + sample + loss/grad + SGD + periodic target sync (oracle_learner_step)."""

    def __init__(self, net: Net, params, *, gamma=0.99, kappa=1.0, lr=1e-4, double_dqn=False,
                 burn_in=1, sync_period=0, seed=2, rank=0):
        P = net.param_count
        self.net = net
        self.online = np.array(params, dtype=np.float32).reshape(P).copy()
        self.target = self.online.copy()
        self._l = _Learner()
        self._l.net = net._c()
        self._l.online = self.online.ctypes.data_as(C.POINTER(C.c_float))
        self._l.target = self.target.ctypes.data_as(C.POINTER(C.c_float))
        self._l.gamma, self._l.kappa, self._l.lr = gamma, kappa, lr
        self._l.double_dqn = int(double_dqn)
        self._l.burn_in = burn_in
        self._l.sync_period = sync_period
        self._l.seed = seed
        self._l.rank = rank
        self._l.step = 0

    @property
    def step_count(self):
        return self._l.step

    def step(self, ring: Ring, batch: int):
        loss = C.c_double(0.0)
        idx = np.zeros(batch, np.int32)
        rc = lib().oracle_learner_step(C.byref(ring._r), C.byref(self._l), batch,
                                       C.byref(loss), _ptr(idx))
        return rc, loss.value, idx

    def sync_target(self):
        lib().oracle_sync_target(C.byref(self._l))
