"""GPU parity of byte-state (RPL_U8) replays and the wide-input train step (SURVEY config 5:
84x84x4 uint8 Atari-shaped states, x = u8 / 255 per reading Q27) against the oracle.

Ring positions, sampled indices and gathered rows bit-exact; Q, y, loss, gradients and new
weights within 1e-5 normwise (FP32 path; BASELINE north star).
"""
import numpy as np
import pytest

import oracle
from inputs import ATARI_STATE_DIM, experiences_u8, init_params
from parity import f32, step_and_compare

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def b():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1801_03138_b200.binding as binding
    return binding


def _np(batch):
    return {k: v.cpu().numpy() for k, v in batch.items()}


@pytest.mark.parametrize("D", [ATARI_STATE_DIM, 37])
def test_u8_insert_sample_gather_bit_exact(b, D):
    # host- and device-sourced adds of ragged sizes wrap a small ring twice; every sample and
    # an explicit-index gather equal the oracle's byte for byte
    import torch
    C = 40
    rp = b.Replay(C, D, seed=7, burn_in=5, state_dtype="u8")
    orc = oracle.RingU8(C, D)
    e = experiences_u8(120, state_dim=D, seed=3)
    t = 0
    for i, k in enumerate([3, 9, 1, 17, 40, 5, 11, 2, 19, 13]):
        part = {key: v[t:t + k] for key, v in e.items()}
        t += k
        if i % 2:
            rp.add(**{key: torch.from_numpy(v).cuda() for key, v in part.items()})
        else:
            rp.add(**part)
        assert orc.add(**part) == oracle.OK
        st = rp.state()
        assert (st["cursor"], st["size"], st["total"]) == (orc.cursor, orc.size, orc.total)
        g = rp.sample(24)
        rc, o = orc.sample(5, 7, 0, 24)
        if rc == oracle.NOT_READY:
            assert g is None
            continue
        g = _np(g)
        for key in ("idx", "s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[key], o[key]), key
    idx = torch.arange(orc.size, dtype=torch.int32, device="cuda").flip(0)
    g = _np(rp.gather(idx))
    o = orc.gather(idx.cpu().numpy())
    for key in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[key], o[key]), key
    assert rp.state()["h2d_bytes"] == sum(k for k in [3, 1, 40, 11, 19]) * (2 * D + 9)
    assert rp.check() == b.RPL_OK


@pytest.mark.parametrize("path", ["tcgen05", "tcgen05-coop", "simt"])
@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_u8_wide_input_train_step(b, ddqn, path, monkeypatch):
    # config 5 network: the paper's dueling MLP on an 84x84x4 byte input (28,224 -> 128 ->
    # V 512 / A 512 -> 1 + 8); layer 0 runs on the tensor cores (wide.cuh: bf16x3 split of
    # the fp32 operands, exact u8) or split-K on FP32 SIMT tiles (RPL_NO_WIDE_TC=1)
    # tcgen05: layer 0 on the tensor cores, the layers above on the fast kernels;
    # tcgen05-coop: the layers above on the cooperative kernel; simt: all on the cooperative kernel
    if path == "simt":
        monkeypatch.setenv("RPL_NO_WIDE_TC", "1")
    if path == "tcgen05-coop":
        monkeypatch.setenv("RPL_NO_WIDE_FAST", "1")
    D = ATARI_STATE_DIM
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=ddqn, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=64)
    rp = b.Replay(96, D, seed=11, state_dtype="u8")
    orc = oracle.RingU8(96, D)
    e = experiences_u8(96, state_dim=D, seed=12)
    rp.add(**e)
    orc.add(**e)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=13))
    for batch in (64, 7):
        step_and_compare(b, cfg, dqn, rp, orc, batch, seed=11)
    assert np.array_equal(dqn.get_params(b.RPL_TARGET), dqn.get_params(b.RPL_ONLINE)) == (True)
    assert dqn.check() == b.RPL_OK


def test_u8_host_adds_through_a_small_staging_arena(b):
    # byte-state host adds are copied on the replay's copy stream into spans of a staging
    # arena of 2 x max_host_add experiences; ragged adds wrap it many times, interleaved with
    # wide train steps, and the ring must hold exactly the oracle's rows
    import torch
    D = 4096   # wide enough for the tcgen05 layer 0, small enough for a fast test
    C = 300
    rp = b.Replay(C, D, seed=21, state_dtype="u8", max_host_add=16)
    orc = oracle.RingU8(C, D)
    e = experiences_u8(900, state_dim=D, seed=22)
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      max_batch=32, sync_period=4)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=23))
    rng = np.random.default_rng(24)
    t = 0
    for it in range(60):
        k = int(rng.integers(1, 17))
        part = {kk: v[t:t + k] for kk, v in e.items()}
        t += k
        rp.add(**part)
        orc.add(**part)
        if it >= 10 and it % 2 == 0:
            assert dqn.train_step(rp, 32) == b.RPL_OK
            orc.events += 1
    idx = torch.arange(orc.size, dtype=torch.int32, device="cuda")
    g = {k: v.cpu().numpy() for k, v in rp.gather(idx).items()}
    o = orc.gather(np.arange(orc.size, dtype=np.int32))
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], o[k]), k
    assert rp.check() == b.RPL_OK and dqn.check() == b.RPL_OK


@pytest.mark.parametrize("path", ["tcgen05", "tcgen05-coop"])
@pytest.mark.parametrize("ddqn", [False, True], ids=["dqn", "ddqn"])
def test_u8_config5_batch_256_and_ragged_200(b, ddqn, path, monkeypatch):
    # BASELINE configs[4] at its configured batch (84x84x4 byte states, B = 256):
    # wide_l0 with UMMA N = 256 (one 256-column accumulator), wide_dw0 with four 64-sample
    # slices (mbarrier phase flips across slices), then a ragged 200 (the last slice partial);
    # both the fast layers-above kernels and the cooperative kernel
    if path == "tcgen05-coop":
        monkeypatch.setenv("RPL_NO_WIDE_FAST", "1")
    D = ATARI_STATE_DIM
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      double_dqn=ddqn, gamma=0.99, lr=1e-3, huber_kappa=1.0, sync_period=2,
                      max_batch=256)
    rp = b.Replay(300, D, seed=31, state_dtype="u8")
    orc = oracle.RingU8(300, D)
    e = experiences_u8(420, state_dim=D, seed=32)   # wraps the ring
    for part in (slice(0, 250), slice(250, 420)):
        rp.add(**{k: v[part] for k, v in e.items()})
        orc.add(**{k: v[part] for k, v in e.items()})
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=33))
    for batch in (256, 200, 256):
        assert step_and_compare(b, cfg, dqn, rp, orc, batch, seed=31) is not None
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK


def test_u8_ring_beyond_4gb_sampled_rows(b):
    # a byte ring whose row offsets pass 2^32 bytes: 80,000 rows x 56,576 B = 4.5 GB (configs[4]
    # rows); device-sourced adds wrap it, then the sampler's indices are bit-exact with the
    # oracle's and every sampled row -- replay_sample, an explicit gather, and the train
    # step's own in-step gather at B = 256 -- equals the generator's row t(i) of the FIFO
    # closed form t(i) = i + C floor((T - 1 - i) / C)
    import torch
    from inputs import u8_rows_np, u8_rows_torch
    C, D, T, K = 80_000, ATARI_STATE_DIM, 92_000, 2_000
    rp = b.Replay(C, D, seed=41, state_dtype="u8", max_host_add=16)
    assert b.Replay.ring_bytes(C, D, state_dtype="u8") > (1 << 32)
    for t0 in range(0, T, K):
        t = torch.arange(t0, t0 + K, dtype=torch.int64, device="cuda")
        rows = u8_rows_torch(t, D, 8)
        rp.add(**rows)
    torch.cuda.synchronize()
    st = rp.state()
    assert (st["size"], st["total"], st["cursor"]) == (C, T, T % C)

    def expect(idx):
        i = idx.astype(np.int64)
        return u8_rows_np(i + C * ((T - 1 - i) // C), D, 8)

    for ev in range(2):
        g = _np(rp.sample(256))
        idx = oracle.sample_indices(41, 0, ev, C, 256)
        assert np.array_equal(g["idx"], idx)
        ex = expect(idx)
        for k in ("s", "s_next", "a", "r", "done"):
            assert np.array_equal(g[k], ex[k]), k
    hi = torch.tensor([C - 1, C - 2, 76_000, 75_913, 0, 1], dtype=torch.int32, device="cuda")
    g = _np(rp.gather(hi))
    ex = expect(hi.cpu().numpy())
    for k in ("s", "s_next", "a", "r", "done"):
        assert np.array_equal(g[k], ex[k]), k
    # the wide train step's in-step gather (gather_u8_kernel) at the configured batch
    cfg = b.DQNConfig(state_dim=D, n_actions=8, dueling=True, hidden=(128,), stream=512,
                      lr=1e-4, sync_period=0, max_batch=256)
    dqn = b.DQN(cfg, init_params(D, 8, (128,), True, 512, seed=43))
    assert dqn.train_step(rp, 256) == b.RPL_OK
    idx = dqn.debug(b.RPL_DBG_IDX, 256)
    assert np.array_equal(idx, oracle.sample_indices(41, 0, 2, C, 256))
    ex = expect(idx)
    for what, key in [(b.RPL_DBG_S, "s"), (b.RPL_DBG_S_NEXT, "s_next"), (b.RPL_DBG_A, "a"),
                      (b.RPL_DBG_R, "r"), (b.RPL_DBG_DONE, "done")]:
        assert np.array_equal(dqn.debug(what, 256).view(np.uint8),
                              np.ascontiguousarray(ex[key]).view(np.uint8)), key
    assert dqn.check() == b.RPL_OK and rp.check() == b.RPL_OK
