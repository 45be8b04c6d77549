"""GPU parity of the replay path (insert, Philox sample, gather, unpack) against the oracle.

Bit-exact: ring positions, sampled indices and every gathered value (BASELINE north star).
Calls go through the C-ABI (paper_1801_03138_b200.binding -> lib/libingpu_replay.so).
"""
import numpy as np
import pytest

import oracle
from inputs import experiences

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def B():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as b
    return b


def _np(out):
    return {k: v.cpu().numpy() for k, v in out.items()}


def _assert_batch_equal(g, o):
    for k in ("idx", "s", "s_next", "a", "r", "done"):
        assert g[k].dtype == o[k].dtype, k
        assert np.array_equal(g[k].view(np.uint8), o[k].view(np.uint8)), k  # bitwise


def test_c1_schedule_insert_sample_bit_exact(B):
    # C1 (BASELINE configs[0]): capacity 1000, D=27, 7 adds per iteration, burn-in 100, B=32;
    # the ring wraps mid-block in iteration 143
    D, C, Bt = 27, 1000, 32
    rp = B.Replay(C, D, burn_in=100, seed=2, rank=0)
    orc = oracle.Ring(C, D)
    e = experiences(214 * 7, state_dim=D, seed=1)
    executed = 0
    for it in range(1, 215):
        sl = slice((it - 1) * 7, it * 7)
        part = {k: v[sl] for k, v in e.items()}
        rp.add(**part)
        assert orc.add(**part) == oracle.OK
        st = rp.state()
        assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
        g = rp.sample(Bt)
        rc, o = orc.sample(100, 2, 0, Bt)
        if rc == oracle.NOT_READY:
            assert g is None and rp.state()["events"] == orc.events
            continue
        executed += 1
        _assert_batch_equal(_np(g), o)
        assert rp.state()["events"] == orc.events
    assert executed == 200
    assert rp.check() == B.RPL_OK


@pytest.mark.parametrize("D", [1, 5, 27, 31, 40])
def test_ragged_adds_and_batches(B, D):
    # state dims with and without the 256-byte row fast path; k = 0, k = C, ragged k;
    # batch sizes that are not multiples of the 64-entry warp group
    C = 97
    rp = B.Replay(C, D, burn_in=1, seed=9, rank=3)
    orc = oracle.Ring(C, D)
    e = experiences(600, state_dim=D, seed=5)
    o = 0
    for k in [0, 1, 13, 97, 0, 50, 96, 2, 64, 97, 31]:
        part = {kk: v[o:o + k] for kk, v in e.items()}
        o += k
        rp.add(**part)
        orc.add(**part)
        for bt in (1, 3, 63, 64, 65, 200):
            g = rp.sample(bt)
            rc, ob = orc.sample(1, 9, 3, bt)
            if orc.size == 0:
                continue
            _assert_batch_equal(_np(g), ob)
    st = rp.state()
    assert (st["cursor"], st["size"], st["total"], st["events"]) == (orc.cursor, orc.size,
                                                                       orc.total, orc.events)


def test_add_errors_have_no_side_effects(B):
    D, C = 4, 10
    rp = B.Replay(C, D)
    e = experiences(11, state_dim=D, seed=3)
    with pytest.raises(B.RplError) as ei:
        rp.add(**e)  # k > capacity (Q6)
    assert ei.value.status == B.RPL_EINVAL
    bad = {k: v[:3].copy() for k, v in e.items()}
    bad["done"][1] = 2
    with pytest.raises(B.RplError) as ei:
        rp.add(**bad)  # terminal must be 0/1
    assert ei.value.status == B.RPL_ECORRUPT
    assert rp.state()["size"] == 0 and rp.state()["total"] == 0
    assert rp.sample(4) is None  # burn_in = 1 but size 0: NOT_READY


def test_device_source_add_and_corrupt_flag(B):
    import torch
    D, C = 27, 300
    rp = B.Replay(C, D)
    orc = oracle.Ring(C, D)
    e = experiences(250, state_dim=D, seed=8)
    dev = {k: torch.from_numpy(v).cuda() for k, v in e.items()}
    rp.add(**dev)
    orc.add(**e)
    g = rp.sample(256)
    rc, o = orc.sample(1, 2, 0, 256)
    _assert_batch_equal(_np(g), o)
    assert rp.state()["h2d_bytes"] == 0  # device-sourced adds cross no PCIe
    bad = {k: v[:2].clone() for k, v in dev.items()}
    bad["done"][0] = 7
    rp.add(**bad)
    assert rp.check() == B.RPL_ECORRUPT
    assert rp.check() == B.RPL_OK  # cleared


def test_one_copy_h2d_accounting(B):
    # P:32/P:50 + S:462: only the single insert crosses PCIe: 225 B per Melee experience
    # (27+27 f32, a i32, r f32, done u8); sampling moves nothing
    rp = B.Replay(10_000, 27)
    e = experiences(2000, seed=4)
    rp.add(**e)
    assert rp.state()["h2d_bytes"] == 2000 * (8 * 27 + 9)
    for _ in range(50):
        rp.sample(128)
    assert rp.state()["h2d_bytes"] == 2000 * (8 * 27 + 9)


def test_full_1m_ring_sampled_rows(B):
    # BASELINE configs[1] size: 1,000,000-slot ring, 1.2M experiences inserted (wraps);
    # sampled rows checked against the host arrays through the FIFO closed form
    # t(i) = i + C*floor((T-1-i)/C)
    import torch
    C, D, T = 1_000_000, 27, 1_200_000
    rp = B.Replay(C, D, seed=2)
    e = experiences(T, state_dim=D, seed=1)
    rp.add_many(e)
    for ev in range(3):
        g = _np(rp.sample(4096))
        idx = oracle.sample_indices(2, 0, ev, C, 4096)
        assert np.array_equal(g["idx"], idx)
        t = idx.astype(np.int64) + C * ((T - 1 - idx.astype(np.int64)) // C)
        for k in ("s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k], e[k][t]), k
    # explicit-index gather over the whole ring (the gather-bandwidth kernel)
    idx = torch.randint(0, C, (1 << 20,), dtype=torch.int32, device="cuda")
    g = _np(rp.gather(idx))
    i = idx.cpu().numpy().astype(np.int64)
    t = i + C * ((T - 1 - i) // C)
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], e[k][t]), k
    assert rp.check() == B.RPL_OK


def test_caller_provided_ring_storage(B):
    # ring storage is library-allocated or caller-provided through opts.storage;
    # a torch tensor holds the rows, sampling is bit-exact with the oracle, destroy leaves it
    import torch
    C = 3000
    nbytes = B.Replay.ring_bytes(C, 27)
    assert nbytes == C * 256   # 256-byte rows for 27-float states
    buf = torch.full((nbytes,), 0xAB, dtype=torch.uint8, device="cuda")   # zeroed at create
    rp = B.Replay(C, 27, seed=12, storage=buf)
    orc = oracle.Ring(C, 27)
    e = experiences(C + 500, seed=13)
    for part in (slice(0, 2000), slice(2000, C + 500)):
        rp.add(**{k: v[part] for k, v in e.items()})
        orc.add(**{k: v[part] for k, v in e.items()})
    for _ in range(2):
        g = rp.sample(512)
        rc, o = orc.sample(1, 12, 0, 512)
        for k in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k].cpu().numpy(), o[k]), k
    rows = buf.view(torch.float32).view(C, 64)[:, :27].cpu().numpy()
    assert np.array_equal(rows, orc.rows()[:, :27])   # the rows really live in the tensor
    rp.close()
    assert buf.sum().item() != 0   # still allocated and intact after destroy
    with pytest.raises(B.RplError):
        B.Replay(C, 27, storage=buf[: nbytes - 256])   # too small
    with pytest.raises(B.RplError):
        B.Replay(C, 27, storage=buf[1:])               # misaligned


def test_staging_arena_wraps_with_many_adds_in_flight(B):
    # host adds take spans of a staging arena of 2 x max_host_add experiences (a ring): ragged
    # adds wrap it many times, with and without train steps consuming deferred (zero-copy)
    # inserts in between; the ring must hold exactly the oracle's rows
    import torch
    C = 5000
    rp = B.Replay(C, 27, seed=14, max_host_add=64)
    orc = oracle.Ring(C, 27)
    e = experiences(9000, seed=15)
    rng = np.random.default_rng(16)
    cfg = B.DQNConfig(max_batch=64)
    dqn = None
    t = 0
    for it in range(300):
        k = int(rng.integers(1, 65))
        part = {kk: v[t:t + k] for kk, v in e.items()}
        t += k
        rp.add(**part)
        orc.add(**part)
        if it == 100:
            from inputs import init_params
            dqn = B.DQN(cfg, init_params(27, 8, (128,), True, 512, seed=17))
        if dqn is not None and it % 3 == 0:
            assert dqn.train_step(rp, 64) == B.RPL_OK
            orc.events += 1   # the step consumed a sampler event
    st = rp.state()
    assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
    idx = torch.arange(orc.size, dtype=torch.int32, device="cuda")
    g = _np(rp.gather(idx))
    o = orc.gather(np.arange(orc.size, dtype=np.int32))
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], o[k]), k
    assert rp.check() == B.RPL_OK


@pytest.mark.parametrize("D,shared", [(27, False), (27, True), (40, False)])
def test_block_inserts_pinned_device_and_tiles(B, D, shared):
    # the tiled insert kernel (32 experiences per CTA iteration, 16-byte row stores; rows wider
    # than 64 words one warp per row) on blocks that are not multiples of the tile and wrap the
    # ring, from pinned host memory (k > 4096: read by the kernel across PCIe, no staging copy),
    # pageable host memory and device memory; the ring equals the oracle's row for row
    import torch
    C = 9000
    rp = B.Replay(C, D, seed=3, shared_state=shared)
    orc = oracle.Ring(C, D, shared=shared) if shared else oracle.Ring(C, D)
    e = experiences(30_000, state_dim=D, seed=21)
    t = 0
    h0 = rp.state()["h2d_bytes"]
    for src, k in [("pinned", 5003), ("host", 4097), ("device", 6001), ("pinned", 8999),
                   ("device", 33), ("pinned", 4100)]:
        part = {kk: v[t:t + k] for kk, v in e.items()}
        t += k
        if src == "pinned":
            rp.add(**{kk: torch.from_numpy(v).pin_memory() for kk, v in part.items()})
        elif src == "device":
            rp.add(**{kk: torch.from_numpy(v).cuda() for kk, v in part.items()})
        else:
            rp.add(**part)
        orc.add(**part)
        st = rp.state()
        assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
    per = (D if shared else 2 * D) * 4 + 9
    assert rp.state()["h2d_bytes"] - h0 == (5003 + 4097 + 8999 + 4100) * per
    ix = np.arange(orc.size, dtype=np.int32)
    if shared:   # the newest experience's s' is not stored yet (reading Q30)
        ix = ix[ix != (orc.cursor - 1) % C]
    g = {k: v.cpu().numpy() for k, v in rp.gather(torch.from_numpy(ix).cuda()).items()}
    o = orc.gather(ix)
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], o[k]), k
    assert rp.check() == B.RPL_OK


def test_time_adds_entry(B):
    # rpl_time_adds runs replay_add n times inside the library: same ring state as n adds
    rp = B.Replay(1000, 27, seed=3)
    orc = oracle.Ring(1000, 27)
    e = experiences(7, seed=5)
    sec = rp.time_adds(e, 300)
    for _ in range(300):
        orc.add(**e)
    assert sec > 0
    st = rp.state()
    assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
    g = {k: v.cpu().numpy() for k, v in rp.gather(
        __import__("torch").arange(1000, dtype=__import__("torch").int32, device="cuda")).items()}
    o = orc.gather(np.arange(1000, dtype=np.int32))
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], o[k]), k
