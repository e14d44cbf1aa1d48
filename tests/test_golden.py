"""Golden fixtures (tests/golden/*.npz, produced from the unmodified reference
by tests/golden/make_golden.py). CPU tests pin the restatement to them
bit-for-bit; GPU tests hold the device path to the documented tolerances."""
from __future__ import annotations

import os

import numpy as np
import pytest

import pyoracle
from helpers import U32, U64, UDD, dd_diff, kappa_b, max_rel, north_star_gates, orth_err

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLD, name + ".npz")))


@pytest.mark.parametrize("name", ["stacked_diag", "graded_suite", "thread_invariance"])
def test_port_reproduces_reference_thin_svd(port, name):
    g = load(name)
    p = port.thin_svd(g["a"], threads=3)
    assert np.array_equal(p.u, g["u"]) and np.array_equal(p.v, g["v"]) and np.array_equal(p.sigma, g["sigma"])


def test_port_reproduces_reference_config_c1(port):
    import workloads as inputs

    g = load("config_c1")
    a = inputs.make(inputs.CONFIGS["c1"], seed=int(g["seed"]))
    assert np.array_equal(a.astype(np.float64).sum(axis=0), g["a_colsum"])  # same input bits
    p = port.thin_svd(a, threads=8)
    assert np.array_equal(p.sigma, g["sigma"]) and np.array_equal(p.v, g["v"])
    assert np.array_equal(p.u[:64], g["u_head"])
    assert np.array_equal(p.u.astype(np.float64).sum(axis=0), g["u_colsum"])


def test_port_golden_jacobi_and_dd(port):
    g = load("jacobi_2x2")
    lam, v, _, _ = port.twosided_jacobi(g["m"])
    assert np.array_equal(lam, g["lam"]) and np.array_equal(v, g["v"])
    for k in (4, 8):
        h = load(f"hilbert{k}")
        lam, _, _, _ = port.twosided_jacobi(h["m"])
        assert np.array_equal(lam, h["lam"])
        (lh, ll), _, _, _ = port.twosided_jacobi_dd(h["m"], sem=pyoracle.SEM_DEVICE)
        assert max_rel(lh, h["lam_dd"]) <= 16 * U64  # dd Jacobi vs dd bisection
    d = load("dd_gram")
    hi, lo = port.dd_gram(d["a"], threads=2)
    assert np.array_equal(hi, d["hi"]) and np.array_equal(lo, d["lo"])


# ---------------------------------------------------------------------------
@pytest.mark.gpu
def test_gpu_golden_cases():
    M = pytest.importorskip("paper_2603_11953_b200")
    if not M.device_available():
        pytest.skip("no CUDA device")
    g = load("stacked_diag")
    r = M.mp_thin_svd(g["a"])
    assert np.array_equal(r.u, g["u"]) and np.array_equal(r.v, g["v"]) and np.array_equal(r.sigma, g["sigma"])

    g = load("graded_suite")
    r = M.mp_thin_svd(g["a"])
    kb = float(g["kappa_b"])
    high_acc = 100.0 * (U32 + U64 * kb * kb)  # proj/tests/test_thinsvd.cpp:112
    assert max_rel(r.sigma, g["sigma_oracle"]) <= high_acc
    assert max_rel(r.sigma, g["sigma"]) <= 2 * high_acc
    assert orth_err(r.v) <= 100.0 * 64.0 * U64 + 64.0 * U32

    g = load("thread_invariance")
    rs = [M.mp_thin_svd(g["a"], threads=t) for t in (1, 2, 4)]
    for r in rs[1:]:  # thread count changes no bit (test_thinsvd.cpp:134-149)
        assert np.array_equal(r.u, rs[0].u) and np.array_equal(r.v, rs[0].v) and np.array_equal(r.sigma, rs[0].sigma)
    assert rs[0].gram_sync_events == 1 and rs[0].gram_blocks == int(g["gram_blocks"])
    kb = kappa_b(g["a"])
    gs, go = north_star_gates(24, U32, kb)
    assert max_rel(rs[0].sigma, g["sigma"]) <= gs

    h = load("hilbert8")
    lam, _, _, _ = M.twosided_jacobi_eig(h["m"])
    assert max_rel(lam, h["lam_dd"]) <= 1e3 * U64 * 1e10  # kappa of scaled Hilbert-8 ~ 1e10
    d = load("dd_gram")
    hi, lo = M.gram(d["a"])
    an = np.linalg.norm(d["a"], axis=0)
    assert np.all(dd_diff(hi, lo, d["hi"], d["lo"]) <= 4 * (40 * U64) ** 2 * np.outer(an, an) + 8 * UDD * np.abs(d["hi"]))
    r = M.mp_thin_svd_f64(d["a"])
    assert max_rel(r.sigma, d["sigma_dd"]) <= 8 * U64


@pytest.mark.gpu
def test_gpu_golden_config_c1():
    M = pytest.importorskip("paper_2603_11953_b200")
    if not M.device_available():
        pytest.skip("no CUDA device")
    import workloads as inputs

    g = load("config_c1")
    a = inputs.make(inputs.CONFIGS["c1"], seed=int(g["seed"]))
    r = M.mp_thin_svd(a)
    gs, go = north_star_gates(32, U32, kappa_b(a))
    assert max_rel(r.sigma, g["sigma"]) <= gs
    assert orth_err(r.u) <= go and orth_err(r.v) <= go
    assert np.max(np.abs(r.u[:64] - g["u_head"])) <= 1e3 * U32 * np.max(np.abs(g["u_head"]))
