"""Pins for the oracle's N_Vector operations (O1-O4), CPU only.

Each pin is independent of oracle.cpp's code: printed examples (golden
fixtures with citations), exact rational arithmetic (fractions.Fraction with
explicit single roundings via float(Fraction), which Python rounds
correctly), closed forms on dyadic data, and library routines (math.fsum:
correctly rounded sum; numpy max).
"""
import math
from fractions import Fraction as F

import numpy as np
import pytest
import torch

import oracle
import synth


def _rn(q: F) -> float:
    return float(q)          # correctly rounded (round-half-even)


def _bits(a):
    return np.asarray(a, dtype=np.float64).view(np.uint64)


def rand(stream, n, lo=-1.0, hi=1.0):
    return synth.uniform(stream, n, lo, hi).numpy()


# ------------------------------------------------------------ streaming
def test_linear_sum_golden(golden):
    for ex in golden["linear_sum"]:
        z = oracle.linear_sum(ex["a"], ex["x"], ex["b"], ex["y"])
        assert np.array_equal(_bits(z), _bits(ex["z"])), ex["cite"]


def test_linear_sum_exact_rational_no_contraction():
    # z_i = RN(RN(a x_i) + RN(b y_i)) evaluated in exact rationals.  With
    # random (non-dyadic) data an FMA or a reassociation changes some bits.
    n = 2000
    x, y = rand(1, n), rand(2, n)
    a, b = 0.3, -1.7
    z = oracle.linear_sum(a, x, b, y)
    exp = [_rn(F(_rn(F(a) * F(float(xi)))) + F(_rn(F(b) * F(float(yi))))) for xi, yi in zip(x, y)]
    assert np.array_equal(_bits(z), _bits(exp))
    fma_like = [_rn(F(a) * F(float(xi)) + F(_rn(F(b) * F(float(yi))))) for xi, yi in zip(x, y)]
    assert not np.array_equal(_bits(exp), _bits(fma_like))  # the pin can see an FMA


def test_linear_sum_dyadic_closed_form():
    n = 4097
    x, y = synth.dyadic(1, n).numpy(), synth.dyadic(2, n).numpy()
    z = oracle.linear_sum(1.25, x, -0.75, y)
    exact = [float(F(5, 4) * F(float(a)) - F(3, 4) * F(float(b))) for a, b in zip(x, y)]
    assert np.array_equal(z, np.array(exact))


def test_scale_prod_div_inv_abs_addconst():
    x = rand(1, 1000)
    # scale by -1 twice is the identity
    assert np.array_equal(_bits(oracle.scale(-1.0, oracle.scale(-1.0, x))), _bits(x))
    assert np.array_equal(oracle.prod([2, 3], [4, 5]), [8, 15])
    xd = synth.dyadic(3, 500).numpy()
    assert np.array_equal(oracle.scale(0.375, xd), np.array([float(F(3, 8) * F(float(v))) for v in xd]))
    # division / inverse: powers of two are exact; random vs exact-rational RN
    assert np.array_equal(oracle.inv([2.0, -0.25, 8.0]), [0.5, -4.0, 0.125])
    y = rand(2, 1000, 0.5, 1.5)
    dz = oracle.div(x, y)
    assert np.array_equal(dz, [_rn(F(float(a)) / F(float(b))) for a, b in zip(x, y)])
    iz = oracle.inv(y)
    assert np.array_equal(iz, [_rn(F(1) / F(float(b))) for b in y])
    assert np.array_equal(_bits(oracle.abs_(x)), _bits(np.abs(x)))
    assert np.array_equal(oracle.add_const(xd, 0.5), np.array([float(F(float(v)) + F(1, 2)) for v in xd]))
    c = oracle.const(3.5, 7)
    assert c.shape == (7,) and np.all(c == 3.5)
    assert oracle.const(0.0, 0).size == 0


def test_ewt_golden(golden):
    for ex in golden["ewt"]:
        y = np.array([ex["y"]])
        t = oracle.add_const(oracle.scale(ex["rtol"], oracle.abs_(y)), ex["atol"])
        assert oracle.inv(t)[0] == ex["ewt"], ex["cite"]


# ----------------------------------------------------------- reductions
def test_dot_golden_and_closed_forms(golden):
    for ex in golden["dot"]:
        assert oracle.dot(ex["x"], ex["y"]) == ex["d"], ex["cite"]
    n = 100003
    ones = np.ones(n)
    idx = np.arange(n, dtype=np.float64)
    assert oracle.dot(ones, idx) == n * (n - 1) // 2          # exact for n < 2^26
    assert oracle.dot([], []) == 0.0


@pytest.mark.parametrize("n", [1, 2, 3, 1000, 100001])
def test_dot_vs_fsum(n):
    # the terms are RN(x_i y_i); math.fsum returns their correctly rounded sum
    x, y = rand(1, n), rand(2, n)
    terms = x * y
    ref = math.fsum(terms.tolist())
    got = oracle.dot(x, y)
    tol = 2 ** -52 * abs(ref) + 1e-20 * float(np.sum(np.abs(terms)))   # Neumaier: 2u|S| + O(n u^2)Σ|t|
    assert abs(got - ref) <= tol
    # permutation invariance (to the same bound)
    perm = np.random.default_rng(5).permutation(n)
    got2 = oracle.dot(x[perm], y[perm])
    assert abs(got2 - ref) <= tol


def test_dot_beats_left_fold():
    # a cancelling sum where a plain left fold loses every digit
    x = np.array([1e16, 1.0, -1e16, 1.0])
    y = np.ones(4)
    assert oracle.dot(x, y) == 2.0


def test_wrms_golden(golden):
    for ex in golden["wrms"]:
        assert oracle.wrms(ex["x"], ex["w"]) == ex["r"], ex["cite"]
    for ex in golden["wrms_mask"]:
        r = oracle.wrms_mask(ex["x"], ex["w"], ex["id"])
        assert r == math.sqrt(ex["r_squared"]), ex["cite"]


@pytest.mark.parametrize("n", [1, 7, 1024, 99999])
def test_wrms_constant_closed_form(n):
    # WRMS(a·1, b·1) = |a b| exactly for dyadic a, b
    for a, b in [(3.0, 0.25), (-0.5, 1.5), (1.0, 1.0)]:
        assert oracle.wrms(np.full(n, a), np.full(n, b)) == abs(a * b)


def test_wrms_vs_fsum_and_mask():
    n = 50001
    x, w = rand(1, n), rand(3, n, 0.5, 1.5)
    p = x * w
    ref = math.sqrt(math.fsum((p * p).tolist()) / n)
    assert abs(oracle.wrms(x, w) - ref) <= 4e-16 * ref
    idv = (rand(4, n, 0, 1) > 0.5).astype(np.float64)
    refm = math.sqrt(math.fsum((p * p * idv).tolist()) / n)      # divisor N, not Σid (R5)
    assert abs(oracle.wrms_mask(x, w, idv) - refm) <= 4e-16 * refm
    assert abs(oracle.wsqrsum(x, w) - math.fsum((p * p).tolist())) <= 4e-16 * n
    assert math.isnan(oracle.wrms([], []))


def test_max_norm_min(golden):
    for ex in golden["max_norm"]:
        assert oracle.max_norm(ex["x"]) == ex["m"], ex["cite"]
    x = rand(1, 10007)
    assert oracle.max_norm(x) == np.max(np.abs(x))
    assert oracle.min_(x) == np.min(x)
    assert math.isnan(oracle.max_norm([]))
    assert oracle.min_([]) == math.inf


# ---------------------------------------------------------------- fused
def test_linear_combination_reduces_to_base_ops():
    n = 3001
    x, y = rand(1, n), rand(2, n)
    assert np.array_equal(_bits(oracle.linear_combination([0.7], [x])), _bits(oracle.scale(0.7, x)))
    assert np.array_equal(_bits(oracle.linear_combination([0.3, -1.7], [x, y])),
                          _bits(oracle.linear_sum(0.3, x, -1.7, y)))


def test_linear_combination_exact_rational_order():
    # z = RN(...RN(RN(c0 X0) + RN(c1 X1)) + ... + RN(c7 X7)): left to right (R4)
    n, nv = 300, 8
    X = [rand(32 + j, n) for j in range(nv)]
    c = [0.1 * (j + 1) - 0.35 for j in range(nv)]
    z = oracle.linear_combination(c, X)
    exp = []
    for i in range(n):
        acc = _rn(F(c[0]) * F(float(X[0][i])))
        for j in range(1, nv):
            acc = _rn(F(acc) + F(_rn(F(c[j]) * F(float(X[j][i])))))
        exp.append(acc)
    assert np.array_equal(_bits(z), _bits(exp))
    # dyadic closed form, coefficients c_j = (j+1)/8
    Xd = [synth.dyadic(32 + j, n).numpy() for j in range(nv)]
    cd = [(j + 1) / 8 for j in range(nv)]
    zd = oracle.linear_combination(cd, Xd)
    exact = [float(sum(F(j + 1, 8) * F(float(Xd[j][i])) for j in range(nv))) for i in range(n)]
    assert np.array_equal(zd, np.array(exact))


def test_scale_add_multi_and_dot_prod_multi():
    n, nv = 2049, 8
    x = rand(1, n)
    Y = [rand(16 + j, n) for j in range(nv)]
    a = [1 - j / 16 for j in range(nv)]
    Z = oracle.scale_add_multi(a, x, Y)
    for j in range(nv):
        assert np.array_equal(_bits(Z[j]), _bits(oracle.linear_sum(a[j], x, 1.0, Y[j])))
    d = oracle.dot_prod_multi(x, Y)
    for j in range(nv):
        ref = math.fsum((x * Y[j]).tolist())
        assert abs(d[j] - ref) <= 1e-15 * np.sum(np.abs(x * Y[j]))
        assert d[j] == oracle.dot(x, Y[j])


# -------------------------------------------------- partitioned (O4)
def test_partitioned_reduction_is_concatenation():
    # P slabs: the global reduction equals the reduction of the concatenation
    # (P:133-135); per-slab partials folded in rank order agree to 1e-15.
    n = 30001
    x, w = rand(1, n), rand(3, n, 0.5, 1.5)
    for P in (1, 2, 3, 8):
        cuts = np.linspace(0, n, P + 1).astype(int)
        parts = [oracle.wsqrsum(x[s:e], w[s:e]) for s, e in zip(cuts[:-1], cuts[1:])]
        glob = math.sqrt(sum(parts) / n)
        assert abs(glob - oracle.wrms(x, w)) <= 1e-15 * glob
        if P == 1:
            assert glob == oracle.wrms(x, w)
