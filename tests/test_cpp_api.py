"""Builds and runs the C++ API tests (tests/cpp): the reference's kernel_ss suite
against include/spingp/kernels.hpp (host only), and the SPEC btd_core /
spingp_engine known answers through include/spingp/{btd,engine}.hpp on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CPP = os.path.join(ROOT, "tests", "cpp")
LIBDIR = os.path.join(ROOT, "paper_1610_08035_b200")


def build(name, link_lib):
    out = os.path.join(CPP, "build", name)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", CPP, os.path.join(CPP, name + ".cpp"),
           "-o", out]
    if link_lib:
        cmd += ["-L", LIBDIR, "-lspingp_b200", f"-Wl,-rpath,{LIBDIR}"]
    subprocess.run(cmd, check=True)
    return out


def test_reference_kernel_suite_against_cpp_api():
    exe = build("test_kernels_api", False)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:]


@pytest.mark.gpu
def test_spec_engine_api_on_gpu():
    exe = build("test_engine_api", True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_optimize_hyperparameters_api_on_gpu():
    """SPEC.md:307-315 examples through include/spingp/optimize.hpp (L-BFGS over the GPU
    loglik + gradient)."""
    exe = build("test_optimize_api", True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_btd_factor_api_on_gpu():
    """The device-resident BTDFactor: SPEC.md:135-140 reconstruction invariant, known
    answers, solve / selective_inverse on the kept factor (include/spingp/btd.hpp)."""
    exe = build("test_factor_api", True)
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
