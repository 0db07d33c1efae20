"""CPU: the C-ABI library loads, exports every symbol include/pcal_b200.h
declares, its host-side setup reproduces the reference's random stream, and
the product path fails loudly (no CPU fallback) when no CUDA device exists."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pcal_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden", "reference_small.npz")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(pcal_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported(pcal):
    out = subprocess.run(["nm", "-D", "--defined-only", pcal.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\sT\s(pcal_[a-z0-9_]+)", out))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert len(declared_functions()) >= 25


def test_library_is_sm100a(pcal):
    out = subprocess.run(["cuobjdump", "--list-elf", pcal.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_host_rng_matches_reference(pcal):
    g = np.load(GOLD)
    assert np.array_equal(pcal.random_normal(1001, 1, 1, threads=1)[:, 0], g["normal_seed1"])
    assert np.array_equal(pcal.random_normal(1001, 1, 1, threads=4)[:, 0], g["normal_seed1"])


def test_host_dense_operator_matches_reference(pcal, orc):
    a = pcal.gen_dense_operator(257, 3, threads=4)
    b = orc.sym_part(orc.random_normal(257, 257, 3))
    assert np.array_equal(a, b)
    assert np.array_equal(a, a.T)


def test_flops_estimate(pcal, orc):
    assert pcal.flops_estimate(1000, 20) == 2.8e6 == orc.flops_estimate_pcal(1000, 20)


def test_config_validation_is_host_side(pcal):
    with pytest.raises(pcal.ParameterError):
        pcal.SolverConfig(algorithm="lbfgs")._c()
    assert pcal.SolverConfig(algorithm="plam-da")._c().algorithm == 4
    c = pcal.SolverConfig(algorithm="alm", alm=pcal.AlmOptions(inner_max=7, outer_max=3))._c()
    assert (c.algorithm, c.alm_inner_max, c.alm_outer_max, c.alm_inner_tol_scale) == (2, 7, 3, 0.1)


def _has_cuda():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.mark.skipif(_has_cuda(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback(pcal):
    a = np.eye(8)
    x = np.zeros((8, 2)); x[0, 0] = x[1, 1] = 1.0
    with pytest.raises(pcal.NativeUnavailable):
        pcal.solve(pcal.QuadraticModel(a, 2, 1.0), pcal.SolverConfig(), x)
    with pytest.raises(pcal.NativeUnavailable):
        pcal.gram(x)


def test_initial_point_argument_checks_are_host_side(pcal):
    """initial_point's parameter_error cases (solver.cpp:137-138,144-146) fail
    before any device work."""
    with pytest.raises(pcal.ParameterError):
        pcal.initial_point(30, 16, 1)                       # 2p > n
    with pytest.raises(pcal.ParameterError):
        pcal.initial_point(30, 4, 1, mode="a2-i", sigma_lower=0.8)  # σ² > 1/2
    with pytest.raises(pcal.ParameterError):
        pcal.initial_point(30, 4, 1, mode="a2-i", sigma_lower=0.0)
    with pytest.raises(pcal.ParameterError):
        pcal.initial_point(30, 4, 1, mode="a3")
