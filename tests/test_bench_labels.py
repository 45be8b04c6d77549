"""bench.py's line labels (host logic, no GPU): the headline line is BASELINE configs[1]
(batch 128, DQN) under BASELINE.json's metric; Double-DQN and other-batch lines belong to the
configs[2] sweep and name their batch; the oracle arm uses plain fields (no product import)."""
import json
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _args(**kw):
    base = dict(ddqn=False, net="dueling", ring="device", capacity=1_000_000, adds_per_step=4,
                avg_period=0, precision="fp32")
    base.update(kw)
    return types.SimpleNamespace(**base)


def test_headline_line_is_baseline_metric(monkeypatch):
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    metric = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    a = _args()
    assert bench.config_index(a, 128) == 1
    assert bench.metric_name(a, 128) == metric
    assert bench.workload_name(a, 128).startswith("BASELINE configs[1]")


def test_sweep_lines_are_configs2_with_their_batch(monkeypatch):
    import bench
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    for ddqn, batch in ((True, 128), (True, 4096), (False, 32)):
        a = _args(ddqn=ddqn)
        assert bench.config_index(a, batch) == 2
        m = bench.metric_name(a, batch)
        assert f"batch {batch}" in m and "configs[2]" in m
        assert ("Double-DQN" in m) == ddqn
        assert bench.workload_name(a, batch).startswith("BASELINE configs[2]")


def test_multi_rank_lines_are_configs3(monkeypatch):
    import bench
    monkeypatch.setenv("WORLD_SIZE", "8")
    assert bench.config_index(_args(), 128) == 3


def test_oracle_arm_fields_need_no_product_library():
    import bench
    f = bench.cfg_fields(_args(ddqn=True), 128)
    assert f["double_dqn"] and f["hidden"] == (128,) and f["stream"] == 512 and f["max_batch"] == 128
    import inspect
    for fn in (bench.time_oracle, bench.time_oracle_c5):
        assert "binding" not in inspect.getsource(fn)
