"""CPU-only checks of the test oracles and of the host-side product logic.

* oracle/drot_oracle.c (the plain-C restatement) is bit-identical to the
  unmodified reference (oracle/_ref) on passes, drot_step and solves, and
  reproduces the committed golden digests (tests/golden/golden.json, made by
  tests/golden/make_golden.py from the reference);
* the product's host generators (probgen.cpp) are bit-identical to the
  reference's (gen_gaussian_problem, CounterRng fixtures);
* dyadic marginals pass the reference's own check_problem in fp32.
No CUDA call is made here.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from pyoracle import (PASS_FUSED, PASS_SKIP_COST, PASS_UNFUSED, LIB_PATHS, Oracle,
                      OracleError, default_config, dyadic_marginal)

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.json")
HAVE_REF = os.path.exists(LIB_PATHS["ref"])
needs_ref = pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@needs_ref
@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("kind,fold,folded,parity", [
    (PASS_FUSED, 0, 0, 0), (PASS_FUSED, 0, 0, 1), (PASS_SKIP_COST, 1, 0, 0),
    (PASS_SKIP_COST, 0, 1, 1), (PASS_UNFUSED, 0, 0, 1)])
@pytest.mark.parametrize("bs,ws", [(64, 4), (4, 2), (1, 1), (5, 3)])
def test_restatement_pass_bitwise(ref, orc, dt, kind, fold, folded, parity, bs, ws):
    m, n = 23, 17
    xy = ref.random_unit(4, m * n, -0.5, 1.0).astype(dt)
    cost = ref.random_unit(4 ^ 0xC0C0, m * n).astype(dt)
    sh = (ref.random_unit(4 ^ 0xFEED, m + n) - 0.5).astype(dt)
    a = ref.fused_pass(xy, cost, sh[:m], sh[m:], dt(0.2), m, n, bs=bs, ws=ws, workers=3,
                       kind=kind, fold=fold, folded=folded, parity=parity, want_dual=True,
                       want_dx=True)
    b = orc.fused_pass(xy, cost, sh[:m], sh[m:], dt(0.2), m, n, bs=bs, ws=ws, kind=kind,
                       fold=fold, folded=folded, parity=parity, want_dual=True, want_dx=True)
    for k in a:
        va, vb = np.asarray(a[k]), np.asarray(b[k])
        assert np.array_equal(va, vb) or (np.isnan(va).all() and np.isnan(vb).all()), k


@needs_ref
@pytest.mark.parametrize("kw", [{}, dict(skip_cost=0), dict(engine=0),
                                dict(relative_tolerances=1), dict(check_every=5, trace_every=4)])
def test_restatement_solve_bitwise(ref, orc, kw):
    m, n = 30, 26
    C = ref.random_unit(9, m * n)
    p, q = np.full(m, 1.0 / m), np.full(n, 1.0 / n)
    cfg = default_config(**kw)
    a, b = ref.solve(C, p, q, m, n, cfg), orc.solve(C, p, q, m, n, cfg)
    assert (a.iterations, a.status) == (b.iterations, b.status)
    assert np.array_equal(a.plan, b.plan) and np.array_equal(a.mu, b.mu)
    assert a.report == b.report
    assert len(a.trace) == len(b.trace)
    for ra, rb in zip(a.trace, b.trace):
        for k in ra:
            assert ra[k] == rb[k] or (np.isnan(ra[k]) and np.isnan(rb[k]))


@needs_ref
def test_restatement_steps_f32(ref, orc):
    m, n = 64, 48
    C, _, _ = ref.gen_gaussian(m, n, seed=0)
    C = C.astype(np.float32)
    p, q = dyadic_marginal(m, np.float32), dyadic_marginal(n, np.float32)
    s1 = ref.steps(C, p, q, m, n, 37)
    s2 = orc.steps(C, p, q, m, n, 37)
    for k in s1:
        assert (s1[k] == s2[k]) if k == "report" else np.array_equal(s1[k], s2[k]), k


def test_oracle_reproduces_golden_rect(orc):
    """The plain-C restatement reproduces the reference's committed digest
    (rect_f64: 600x300, random-simplex marginals, converged)."""
    gold = json.load(open(GOLDEN))["rect_f64"]
    sp = gold["spec"]
    m, n = sp["m"], sp["n"]
    C = orc.random_unit(sp["seed"], m * n)
    import ctypes as Cc
    f = orc.lib.orc_random_simplex
    f.argtypes = [Cc.c_int64, Cc.c_uint64, Cc.c_void_p]
    f.restype = None
    p, q = np.empty(m), np.empty(n)
    f(m, sp["seed"] ^ 0x1111, p.ctypes.data)
    f(n, sp["seed"] ^ 0x2222, q.ctypes.data)
    out = orc.solve(C, p, q, m, n, default_config())
    assert out.iterations == gold["iterations"]
    assert out.status == gold["status"]
    assert sha(out.plan) == gold["plan_sha256"]
    assert sha(out.mu) == gold["mu_sha256"]
    for k, v in gold["report"].items():
        assert float.fromhex(v) == out.report[k]


def test_golden_matches_survey_numbers():
    """The committed digests carry SURVEY §8(c)'s golden runs."""
    g = json.load(open(GOLDEN))
    assert g["c1_f64"]["iterations"] == 36041 and g["c1_f64"]["status"] == "converged"
    assert abs(g["c1_f64"]["report_float"]["objective"] - 0.00159626253482) < 1e-14
    assert g["gauss1000_f64"]["iterations"] == 52139
    assert abs(g["gauss1000_f64"]["report_float"]["objective"] - 0.236454396358) < 1e-12


@needs_ref
def test_validation_codes(ref, orc):
    m, n = 5, 4
    C = ref.random_unit(3, m * n)
    p, q = np.full(m, 1.0 / m), np.full(n, 1.0 / n)
    for mutate, name in [(lambda c, p, q: c.__setitem__(3, -1.0), "negative_cost"),
                         (lambda c, p, q: c.__setitem__(2, np.nan), "non_finite_entry"),
                         (lambda c, p, q: p.__setitem__(0, 0.9), "marginal_not_simplex")]:
        c2, p2, q2 = C.copy(), p.copy(), q.copy()
        mutate(c2, p2, q2)
        for o in (ref, orc):
            with pytest.raises(OracleError) as e:
                o.check_problem(c2, p2, q2, m, n)
            assert e.value.name == name


# ---- host logic of the product (no GPU) -----------------------------------------
@pytest.fixture(scope="module")
def drot_host():
    import paper_2110_11738_b200 as d
    return d


def test_generator_bit_identical(drot_host, orc):
    d = drot_host
    for (m, n, seed, dirich) in [(50, 30, 3, True), (33, 77, 0, False), (1, 5, 9, False)]:
        pr = d.gen_gaussian_problem(d.GaussianSpec(m, n, 5.0, seed, dirich))
        C, p, q = orc.gen_gaussian(m, n, seed=seed, dirichlet=dirich)
        assert np.array_equal(pr.cost.ravel(order="F"), C)
        assert np.array_equal(pr.p, p) and np.array_equal(pr.q, q)
    f = d.gen_gaussian_problem_as(d.GaussianSpec(64, 40, 5.0, 1), np.float32)
    C, _, _ = orc.gen_gaussian(64, 40, seed=1)
    assert np.array_equal(f.cost.ravel(order="F"), C.astype(np.float32))


def test_counter_uniform(drot_host, orc):
    assert np.array_equal(drot_host.counter_uniform(1, 4096), orc.random_unit(1, 4096))
    assert np.array_equal(drot_host.random_matrix(7, 9, 3, -0.5, 1.0).ravel(order="F"),
                          orc.random_unit(3, 63, -0.5, 1.0))


@pytest.mark.parametrize("length", [1, 3, 1000, 4096, 10000, 40000, 100000])
@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_dyadic_marginals_exact(drot_host, orc, length, dt):
    v = drot_host.dyadic_marginal(length, dt)
    assert v.dtype == dt and (v > 0).all()
    acc = 0.0
    for x in v.astype(np.float64):
        acc += x
    assert acc == 1.0  # exact, sequential double sum (problem.hpp:106-116)
    assert v.max() / v.min() < 1 + 1e-5
    assert np.array_equal(v, dyadic_marginal(length, dt))  # test-side twin


def test_dyadic_fp32_passes_reference_check(drot_host, orc):
    m, n = 1000, 10000
    C = np.zeros(m * n, np.float32)
    orc.check_problem(C, drot_host.dyadic_marginal(m, np.float32),
                      drot_host.dyadic_marginal(n, np.float32), m, n)
    with pytest.raises(OracleError):  # plain 1/m fails the 1e-12 check in fp32
        orc.check_problem(C, np.full(m, 1.0 / m, np.float32), np.full(n, 1.0 / n, np.float32), m, n)


def test_config_mirrors_reference_defaults(drot_host):
    c = drot_host.DrotConfig().to_c()
    ref = default_config()
    for k in ("rho0", "tol_primal", "tol_dual", "tol_gap", "max_iters", "check_every",
              "engine", "skip_cost", "deterministic", "record_trace", "block_rows",
              "work_size", "trace_every"):
        assert getattr(c, k) == getattr(ref, k), k
