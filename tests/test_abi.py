"""CPU-side checks of the C ABI: the library builds, loads, exports every declared symbol,
and fails loudly (no CPU fallback) when there is no GPU."""

import ctypes
import os
import re

import pytest
import torch

from paper_2312_06126_b200 import spz

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "spz.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spz_[a-z0-9_]+)\s*\(", text)))


def test_header_declarations_match_binding_list():
    assert _declared_symbols() == sorted(spz.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = spz.lib()
    for name in _declared_symbols():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_library_is_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", spz.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_string():
    assert "sm_100a" in spz.spz_version()


def test_config_default_values():
    c = spz.spz_config_default(spz.SPZ_SAC, 22, 6)
    assert (c.gamma, c.tau, c.lr_actor, c.beta1, c.beta2, c.adam_eps) == (0.99, 0.005, 3e-4, 0.9, 0.999, 1e-8)
    assert c.target_entropy == -6.0 and c.alpha_auto == 1 and c.log_std_min == -20 and c.log_std_max == 2
    t = spz.spz_config_default(spz.SPZ_TD3, 44, 17)
    assert t.td3_noise == 0.2 and t.td3_noise_clip == 0.5 and t.td3_policy_delay == 2 and t.alpha_auto == 0
    dd = spz.spz_config_default(spz.SPZ_DDPG, 22, 6)  # f4: TD3 kernels, no delay, no target smoothing
    assert dd.td3_policy_delay == 1 and dd.td3_noise == 0.0 and dd.td3_noise_clip == 0.0 and dd.alpha_auto == 0
    v1 = spz.spz_config_default(spz.SPZ_SACV1, 22, 6)  # f4: SAC v1, fixed temperature by default
    assert v1.alpha_auto == 0 and v1.alpha_init == 0.2 and v1.target_entropy == -6.0
    assert spz.spz_stats().as_dict()["value_loss"] == 0.0
    with pytest.raises(spz.SpzError):
        spz.spz_config_default(spz.SPZ_SAC, 0, 6)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(spz.SpzError) as e:
        spz.spz_replay_create(3, 1, 100)
    assert e.value.status in (spz.SPZ_ECUDA,)
    with pytest.raises(spz.SpzError) as e:
        spz.Policy(3, 1, hidden=64, n_hidden=2)
    assert e.value.status in (spz.SPZ_ECUDA,)


def test_invalid_arguments_rejected_before_device_use():
    with pytest.raises(spz.SpzError) as e:
        spz.spz_replay_create(3, 1, 0)  # S:193 capacity 0 is an error
    assert e.value.status == spz.SPZ_EINVAL
