"""CPU checks of the C-ABI library: it loads, exports every symbol include/rnnlm.h
declares, and rejects bad arguments before touching a device."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1801_09866_b200 import _lib, build, redundancy_rate, hit_ratio
from synth.model import ModelDims, generate_model

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return _lib.load()


def header_functions():
    src = open(os.path.join(ROOT, "include", "rnnlm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rnnlm_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    names = header_functions()
    assert len(names) >= 15
    for n in names:
        assert hasattr(L, n), n
        assert n in _lib.SIGNATURES, f"binding lacks {n}"
    assert L.rnnlm_abi_version() == 3


def test_library_is_sm100a(L):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.library_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_status_strings(L):
    assert L.rnnlm_status_string(0) == b"ok"
    assert b"capacity" in L.rnnlm_status_string(6)


def _weights(d):
    m = generate_model(d, seed=1)
    arrs = {k: np.ascontiguousarray(m[k]) for k in _lib.WEIGHT_NAMES}
    return arrs, _lib.Weights(**{k: arrs[k].ctypes.data_as(ctypes.c_void_p) for k in arrs})


@pytest.mark.parametrize("field,value,status", [
    ("vocab", 1, 2), ("embed", 12, 2), ("hidden", 0, 2), ("maxent_order", 9, 2),
    ("maxent_order", 0, 2), ("max_histories_per_session", 1, 2), ("key_mode", 3, 1),
    ("round_digits", 5, 1), ("math", 7, 1), ("num_sessions", 0, 2)])
def test_create_rejects_bad_config_without_device(L, field, value, status):
    d = ModelDims(V=16, E=8, H=8, maxent_log2=4, N=3)
    arrs, w = _weights(d)
    cfg = _lib.Config(16, 8, 8, 4, 3, 1, 2, 0, 1, 1, 64, 64, 0)
    setattr(cfg, field, value)
    if field == "round_digits":
        cfg.key_mode = 1
    h = ctypes.c_void_p()
    assert L.rnnlm_create(ctypes.byref(cfg), ctypes.byref(w), ctypes.byref(h)) == status
    assert not h.value


def test_create_rejects_nonfinite_weights(L):
    d = ModelDims(V=16, E=8, H=8, maxent_log2=4, N=3)
    arrs, w = _weights(d)
    arrs["Uh"][3, 3] = np.inf
    cfg = _lib.Config(16, 8, 8, 4, 3, 0, 0, 0, 1, 1, 64, 64, 0)
    h = ctypes.c_void_p()
    assert L.rnnlm_create(ctypes.byref(cfg), ctypes.byref(w), ctypes.byref(h)) == 3


def test_null_handle_calls(L):
    assert L.rnnlm_query_batch(None, 1, None, None, None, None, None, None, None) == 1
    assert L.rnnlm_cache_stats(None, 0, None) == 1
    L.rnnlm_destroy(None)


def test_redundancy_rate_table1():
    # (103904, 102776) -> 1.09 %, (103904, 88749) -> 14.59 %
    assert redundancy_rate(103904, 102776) == 1.09
    assert redundancy_rate(103904, 88749) == 14.59
    assert redundancy_rate(5, 5) == 0.0
    with pytest.raises(ValueError):
        redundancy_rate(0, 0)


def test_hit_ratio_P111():
    assert hit_ratio(89, 100) == 0.89
    assert hit_ratio(0, 7) == 0.0 and hit_ratio(7, 7) == 1.0
