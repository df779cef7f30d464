"""The drop-in boundary: every symbol declared in include/spingp_c.h is exported by
the in-tree library and bound (with a signature) by the Python mirror; host-only
entry points work without a GPU; without a GPU the computing entry points fail
loudly (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import oracle_lib as O
import paper_1610_08035_b200 as P
from paper_1610_08035_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "spingp_c.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spingp_[a-z0-9_]+)\s*\(", src)))


def test_every_declared_symbol_is_exported_and_bound():
    syms = declared_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", P.lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (spingp_\w+)", out))
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    assert sorted(_capi.SIGNATURES) == syms


def test_library_links_only_the_cuda_runtime_no_fallback():
    out = subprocess.run(["ldd", P.lib_path], capture_output=True, text=True).stdout
    assert "libcudart" in out or "cudart" in out


def test_state_space_host_api_matches_oracle():
    for leaves, theta in [([P.MATERN12], [0.8, 1.7]), ([P.MATERN32], [1.3, 0.9]), ([P.MATERN52], [2.1, 1.2]),
                          ([(P.EQ, 6)], [1.1, 1.4]), ([(P.EQ, 10)], [1.1, 1.4]), ([P.MATERN32, P.MATERN12], [1, 0.7, 0.5, 2]),
                          ([(P.QP, 6)], [1.0, 1.0, 1.0, 20.0])]:
        a = P.state_space(leaves, theta)
        o = O.state_space(leaves, theta)
        assert a["b"] == o["b"]
        for k in ("F", "H", "dF"):
            assert np.abs(a[k] - o[k]).max() <= 1e-13 * max(1.0, np.abs(o[k]).max()), k
        for k in ("Pinf", "dPinf"):  # Lyapunov solve: algorithm-dependent rounding
            assert np.abs(a[k] - o[k]).max() <= 1e-9 * max(1.0, np.abs(o[k]).max()), k
        assert np.array_equal(a["f_constant"], o["f_constant"])


def test_kernel_dims_and_bad_leaves():
    assert P.kernel_dims([P.MATERN32, (P.QP, 6)]) == (16, 6)
    assert P.kernel_dims([(P.EQ, 10)]) == (10, 2)
    with pytest.raises(ValueError):
        P.state_space([P.MATERN32], [1.0])
    with pytest.raises(ValueError):
        P.state_space([(P.EQ, 3)], [1.0, 1.0])


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    with pytest.raises(P.DeviceError):
        P.Context(0)


def test_library_has_no_undefined_own_symbols():
    """Every template the launch code references is instantiated in some translation unit
    (a missing one only shows up when the library is loaded on the GPU box)."""
    import subprocess
    out = subprocess.run(["nm", "-D", "--undefined-only", P.lib_path], capture_output=True, text=True, check=True).stdout
    own = [ln for ln in out.splitlines() if "spingp" in ln]
    assert not own, own[:5]
