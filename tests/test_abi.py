"""CPU checks of the C-ABI library: it loads, exports every symbol include/*.h declares, and
its host-only logic behaves (no compute call without a GPU)."""
import ctypes as C
import glob
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        src = open(h).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, re.M):
            names.add(m.group(1))
    return sorted(names)


def test_library_builds_and_exports_every_declared_symbol():
    from paper_1801_03138_b200 import build
    so = build.build()
    declared = _declared()
    assert {"replay_create", "replay_add", "replay_sample", "dqn_train_step", "sync_target"} <= set(declared)
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    missing = [n for n in declared if n not in exported]
    assert not missing, missing
    from paper_1801_03138_b200 import binding
    assert set(binding.EXPORTS) == set(declared)


def test_sm100a_code_in_library():
    from paper_1801_03138_b200 import build
    so = build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_param_count_host_only():
    from paper_1801_03138_b200 import DQNConfig
    assert DQNConfig().param_count == 140_297   # the paper's dueling net
    assert DQNConfig(dueling=False, hidden=(64, 64)).param_count == 6_472
    from paper_1801_03138_b200 import binding
    with pytest.raises(binding.RplError):
        DQNConfig(n_actions=0).param_count
    with pytest.raises(binding.RplError):
        DQNConfig(hidden=(1, 2, 3, 4, 5)).param_count


def test_param_count_matches_oracle_blob():
    import oracle
    from paper_1801_03138_b200 import DQNConfig
    for cfg in [DQNConfig(), DQNConfig(dueling=False, hidden=(64, 64)),
                DQNConfig(state_dim=5, n_actions=3, hidden=(6, 7), stream=11)]:
        net = oracle.Net(cfg.state_dim, cfg.n_actions, cfg.dueling, cfg.hidden, cfg.stream)
        assert cfg.param_count == net.param_count


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU path")
def test_no_gpu_fails_loudly():
    from paper_1801_03138_b200 import binding
    with pytest.raises(binding.RplError):
        binding.Replay(10, 27)
    lib = binding.lib()
    h = C.c_void_p()
    st = lib.replay_create(10, 27, None, C.byref(h))
    assert st == binding.RPL_ECUDA and not h.value
    assert "device" in binding.last_error()


def test_step_flops_matches_survey():
    from paper_1801_03138_b200 import DQNConfig, step_flops
    assert step_flops(DQNConfig(), 128) == 141_590_528   # 141.6 MFLOP
    assert step_flops(DQNConfig(dueling=False, hidden=(64, 64)), 128) == 6_045_696
