"""CPU checks of the C-ABI boundary: the library builds / loads and exports every
symbol include/fin.h declares.  No compute call is made without a GPU."""
import ctypes
import os
import re

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "fin.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fin_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_section8b_calls():
    d = _declared()
    for name in ("fin_env_create", "fin_env_reset", "fin_env_step", "fin_rollout", "fin_ensemble_act",
                 "fin_episode_metrics", "fin_env_get_state", "fin_env_check", "fin_policy_create"):
        assert name in d


def test_library_exports_every_declared_symbol():
    from paper_2501_10709_b200 import fin
    lib = ctypes.CDLL(fin.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_declared()) == set(fin.EXPORTS)
    assert fin.fin_abi_version() == 1


def test_library_is_sm100a_only():
    """The fatbin holds sm_100a SASS (cuobjdump), nothing for other arches."""
    import shutil
    import subprocess
    from paper_2501_10709_b200 import fin
    cob = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cob):
        return
    out = subprocess.run([cob, "--list-elf", fin.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_config_struct_layout_matches_header():
    from paper_2501_10709_b200 import fin
    # 16 int32, 3 double, 4 float, uint64, int64 with natural alignment
    assert ctypes.sizeof(fin.fin_env_config) == 16 * 4 + 3 * 8 + 4 * 4 + 8 + 8
    assert ctypes.sizeof(fin.fin_traj) == 13 * 8 + 8   # 13 pointers + ep_capacity (padded)
    assert ctypes.sizeof(fin.fin_noise) == 24


def test_tensor_marshalling_refuses_cpu_tensors():
    import pytest
    import torch
    from paper_2501_10709_b200 import fin
    with pytest.raises(ValueError):
        fin.make_traj(reward=torch.zeros(4))
