"""GPU parity of the N_Vector kernels against the oracle (through the C ABI).

Streaming and fused linear ops: bit-exact.  Reductions: relative 1e-12 to
the oracle's compensated sum (signed dots: 1e-12 · Σ|x_i y_i|, DESIGN R6).
Sizes span several CTAs and grid-stride rounds, ragged tails and the
scalar head of misaligned views; 1e8 (the C2 bench size) on sampled
indices."""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from gpu_util import assert_bits_equal, needs_cuda, padded

pytestmark = [pytest.mark.gpu, needs_cuda]

LENGTHS = [0, 1, 2, 3, 5, 31, 32, 33, 1023, 4097, 65537, 1_000_001]


@pytest.fixture(scope="module")
def S():
    from paper_2011_12984_b200 import sunbw
    return sunbw


@pytest.fixture(scope="module")
def ctx(S):
    c = S.Context(0)
    yield c
    c.destroy()


def gen(stream, n, lo=-1.0, hi=1.0):
    return synth.uniform(stream, n, lo, hi, device="cuda")


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("n", LENGTHS)
@pytest.mark.parametrize("off", [0, 1, 3])
def test_streaming_bit_exact(S, ctx, n, off):
    x = padded(gen(1, n), off)
    y = padded(gen(2, n), off)
    yd = padded(gen(2, n, 0.5, 1.5), off)
    z = padded(torch.zeros(n, dtype=torch.float64, device="cuda"), off)
    vx, vy, vyd, vz = (S.NVector(ctx, t) for t in (x, y, yd, z))
    X, Y, YD = host(x), host(y), host(yd)
    cases = [
        (lambda: S.N_VLinearSum(1.25, vx, -0.75, vy, vz), oracle.linear_sum(1.25, X, -0.75, Y), "linear_sum"),
        (lambda: S.N_VLinearSum(0.3, vx, -1.7, vy, vz), oracle.linear_sum(0.3, X, -1.7, Y), "linear_sum2"),
        (lambda: S.N_VScale(-0.3, vx, vz), oracle.scale(-0.3, X), "scale"),
        (lambda: S.N_VProd(vx, vy, vz), oracle.prod(X, Y), "prod"),
        (lambda: S.N_VDiv(vx, vyd, vz), oracle.div(X, YD), "div"),
        (lambda: S.N_VConst(2.5, vz), oracle.const(2.5, n), "const"),
        (lambda: S.N_VAbs(vx, vz), oracle.abs_(X), "abs"),
        (lambda: S.N_VInv(vyd, vz), oracle.inv(YD), "inv"),
        (lambda: S.N_VAddConst(vx, 0.1, vz), oracle.add_const(X, 0.1), "add_const"),
    ]
    for run, ref, name in cases:
        z.fill_(float("nan"))
        run()
        ctx.check(name)
        assert_bits_equal(z, ref, f"{name} n={n} off={off}")


def test_streaming_mixed_alignment_and_aliasing(S, ctx):
    n = 10007
    x0, y0 = gen(1, n), gen(2, n)
    X, Y = host(x0), host(y0)
    # x 8-byte misaligned relative to z: falls back to the scalar path
    x = padded(x0, 1)
    z = padded(torch.zeros(n, dtype=torch.float64, device="cuda"), 0)
    S.N_VLinearSum(2.0, S.NVector(ctx, x), 0.5, S.NVector(ctx, y0), S.NVector(ctx, z))
    assert_bits_equal(z, oracle.linear_sum(2.0, X, 0.5, Y), "mixed alignment")
    # z == x and z == y
    a = x0.clone(); va = S.NVector(ctx, a)
    S.N_VLinearSum(0.7, va, -0.2, S.NVector(ctx, y0), va)
    assert_bits_equal(a, oracle.linear_sum(0.7, X, -0.2, Y), "z==x")
    b = y0.clone(); vb = S.NVector(ctx, b)
    S.N_VLinearSum(0.7, S.NVector(ctx, x0), -0.2, vb, vb)
    assert_bits_equal(b, oracle.linear_sum(0.7, X, -0.2, Y), "z==y")


@pytest.mark.parametrize("policy,block,grid", [(0, 0, 0), (0, 64, 3), (0, 1024, 0), (1, 128, 0), (1, 32, 0)])
def test_policy_invariance(S, ctx, policy, block, grid):
    n = 300001
    x, y = gen(1, n), gen(2, n)
    z = torch.empty_like(x)
    vx, vy, vz = S.NVector(ctx, x), S.NVector(ctx, y), S.NVector(ctx, z)
    for v in (vx, vy, vz):
        v.set_policy(policy, block, grid, block or 256)
    S.N_VLinearSum(0.3, vx, 1.1, vy, vz)
    assert_bits_equal(z, oracle.linear_sum(0.3, host(x), 1.1, host(y)), "policy")
    w = gen(3, n, 0.5, 1.5); vw = S.NVector(ctx, w); vw.set_policy(policy, block, grid, block or 256)
    r1, r2 = S.N_VWrmsNorm(vx, vw), S.N_VWrmsNorm(vx, vw)
    ref = oracle.wrms(host(x), host(w))
    assert r1 == r2                                        # deterministic
    assert abs(r1 - ref) <= 1e-12 * ref


@pytest.mark.parametrize("n", LENGTHS[1:])
@pytest.mark.parametrize("off", [0, 2])
def test_reductions(S, ctx, n, off):
    x = padded(gen(1, n), off)
    w = padded(gen(3, n, 0.5, 1.5), off)
    yp = padded(gen(2, n, 0.5, 1.5), off)
    idv = padded((gen(4, n, 0, 1) > 0.5).double(), off)
    vx, vw, vy, vid = (S.NVector(ctx, t) for t in (x, w, yp, idv))
    X, W, YP, ID = host(x), host(w), host(yp), host(idv)
    ref = oracle.wrms(X, W)
    assert abs(S.N_VWrmsNorm(vx, vw) - ref) <= 1e-12 * ref
    refm = oracle.wrms_mask(X, W, ID)
    assert abs(S.N_VWrmsNormMask(vx, vw, vid) - refm) <= 1e-12 * max(refm, 1e-300)
    assert abs(S.N_VWSqrSumLocal(vx, vw) - oracle.wsqrsum(X, W)) <= 1e-12 * oracle.wsqrsum(X, W)
    refd = oracle.dot(YP, W)                                # positive terms
    assert abs(S.N_VDotProd(vy, vw) - refd) <= 1e-12 * refd
    refs = oracle.dot(X, YP)                                # signed: condition-scaled bound
    assert abs(S.N_VDotProd(vx, vy) - refs) <= 1e-12 * float(np.sum(np.abs(X * YP)))
    assert abs(S.N_VDotProdLocal(vx, vy) - refs) <= 1e-12 * float(np.sum(np.abs(X * YP)))
    assert S.N_VMaxNorm(vx) == oracle.max_norm(X)           # exact: no reassociation
    assert S.N_VMin(vx) == oracle.min_(X)
    ctx.check("reductions")


def test_reduction_closed_forms_and_errors(S, ctx):
    n = 1 << 20
    a = torch.full((n,), 3.0, dtype=torch.float64, device="cuda")
    b = torch.full((n,), 0.25, dtype=torch.float64, device="cuda")
    assert S.N_VWrmsNorm(S.NVector(ctx, a), S.NVector(ctx, b)) == 0.75      # |a b| exactly
    ones = torch.ones(100003, dtype=torch.float64, device="cuda")
    idx = torch.arange(100003, dtype=torch.float64, device="cuda")
    assert S.N_VDotProd(S.NVector(ctx, ones), S.NVector(ctx, idx)) == 100003 * 100002 // 2
    e = torch.empty(0, dtype=torch.float64, device="cuda")
    ve = S.NVector(ctx, e)
    assert S.N_VDotProd(ve, ve) == 0.0
    assert math.isnan(S.N_VWrmsNorm(ve, ve))
    assert ctx.last_error() == -6                            # SUNBW_ERR_EMPTY
    assert math.isnan(S.N_VMaxNorm(ve))
    ctx.last_error()
    # length mismatch is reported, nothing is written
    x = torch.ones(10, dtype=torch.float64, device="cuda")
    z = torch.zeros(11, dtype=torch.float64, device="cuda")
    S.N_VScale(2.0, S.NVector(ctx, x), S.NVector(ctx, z))
    assert ctx.last_error() == -2 and float(z.abs().sum()) == 0.0


@pytest.mark.parametrize("n", [1, 33, 4097, 1_000_001])
@pytest.mark.parametrize("nv", [1, 2, 3, 4, 8, 11])
def test_fused_ops(S, ctx, n, nv):
    X = [gen(32 + j, n) for j in range(nv)]
    Xh = [host(t) for t in X]
    c = [0.1 * (j + 1) - 0.35 for j in range(nv)]
    z = torch.empty(n, dtype=torch.float64, device="cuda")
    vX = [S.NVector(ctx, t) for t in X]
    vz = S.NVector(ctx, z)
    assert S.N_VLinearCombination(c, vX, vz) == 0
    assert_bits_equal(z, oracle.linear_combination(c, Xh), f"LC nv={nv}")
    # z aliasing X[0]
    x0 = X[0].clone()
    assert S.N_VLinearCombination(c, [S.NVector(ctx, x0)] + vX[1:], S.NVector(ctx, x0)) == 0
    assert_bits_equal(x0, oracle.linear_combination(c, Xh), "LC z==X0")
    # ScaleAddMulti, including Z_j == Y_j
    x = gen(1, n)
    a = [1 - j / 16 for j in range(nv)]
    Z = [torch.empty_like(x) for _ in range(nv)]
    assert S.N_VScaleAddMulti(a, S.NVector(ctx, x), vX, [S.NVector(ctx, t) for t in Z]) == 0
    refZ = oracle.scale_add_multi(a, host(x), Xh)
    for j in range(nv):
        assert_bits_equal(Z[j], refZ[j], f"SAM j={j}")
    Yc = [t.clone() for t in X]
    vY = [S.NVector(ctx, t) for t in Yc]
    assert S.N_VScaleAddMulti(a, S.NVector(ctx, x), vY, vY) == 0
    for j in range(nv):
        assert_bits_equal(Yc[j], refZ[j], f"SAM Z==Y j={j}")
    # DotProdMulti
    d = S.N_VDotProdMulti(S.NVector(ctx, x), vX)
    refd = oracle.dot_prod_multi(host(x), Xh)
    for j in range(nv):
        bound = 1e-12 * float(np.sum(np.abs(host(x) * Xh[j])))
        assert abs(d[j] - refd[j]) <= bound, (j, d[j], refd[j])
    ctx.check("fused")


@pytest.mark.slow
def test_full_size_1e8_sampled(S, ctx):
    """C2 size (1e8), the launch configuration bench.py times: sampled
    elementwise parity (the oracle recomputes sampled indices one by one from
    the counter generator) and full reductions against the oracle."""
    n = 100_000_000
    x, y = gen(1, n), gen(2, n)
    z = torch.empty_like(x)
    vx, vy, vz = S.NVector(ctx, x), S.NVector(ctx, y), S.NVector(ctx, z)
    S.N_VLinearSum(1.25, vx, -0.75, vy, vz)
    idx = torch.cat([torch.arange(4096), torch.arange(n - 4096, n),
                     torch.randint(0, n, (200_000,), generator=torch.Generator().manual_seed(7))])
    xs = synth.uniform_at(1, idx, -1, 1).numpy()
    ys = synth.uniform_at(2, idx, -1, 1).numpy()
    assert_bits_equal(z[idx.cuda()], oracle.linear_sum(1.25, xs, -0.75, ys), "1e8 linear_sum")
    X8 = [gen(32 + j, n) for j in range(8)]
    c = [(j + 1) / 8 for j in range(8)]
    S.N_VLinearCombination(c, [S.NVector(ctx, t) for t in X8], vz)
    Xs = [synth.uniform_at(32 + j, idx, -1, 1).numpy() for j in range(8)]
    assert_bits_equal(z[idx.cuda()], oracle.linear_combination(c, Xs), "1e8 LC8")
    w = gen(3, n, 0.5, 1.5)
    got = S.N_VWrmsNorm(vx, S.NVector(ctx, w))
    ref = oracle.wrms(host(x), host(w))
    assert abs(got - ref) <= 1e-12 * ref
    d = S.N_VDotProdMulti(vx, [S.NVector(ctx, t) for t in X8])
    xh = host(x)
    for j in range(8):
        Xj = host(X8[j])
        assert abs(d[j] - oracle.dot(xh, Xj)) <= 1e-12 * float(np.sum(np.abs(xh * Xj)))


@pytest.mark.slow
def test_max_size_beyond_int32_sampled(S, ctx):
    """Largest size class: n = 2^31 + 37 elements (17.2 GB per vector), past
    32-bit element indices and byte offsets — the N_Vector ops must index
    with 64 bits (S:150 places no upper bound on n; SURVEY §8(d) C2 runs to
    1e9).  Streaming ops: sampled indices bit-exact against the oracle
    (counter generator, so the oracle draws the sampled inputs alone, the
    last 4096 included).  Reductions: WRMS/Dot/MaxNorm against the oracle's
    compensated sums taken over 2^27-element chunks and combined with
    math.fsum (exact combination of the chunk results; DESIGN R6 bounds)."""
    n = (1 << 31) + 37
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info()
    if free < 80 * (1 << 30):
        pytest.skip("needs ~75 GB of free device memory")
    x = gen(1, n)
    y = gen(2, n)
    z = torch.empty_like(x)
    vx, vy, vz = S.NVector(ctx, x), S.NVector(ctx, y), S.NVector(ctx, z)
    idx = torch.cat([torch.arange(4096), torch.arange(n - 4096, n),
                     torch.arange((1 << 31) - 2048, (1 << 31) + 37),
                     torch.randint(0, n, (200_000,), generator=torch.Generator().manual_seed(11))])
    xs = synth.uniform_at(1, idx, -1, 1).numpy()
    ys = synth.uniform_at(2, idx, -1, 1).numpy()
    S.N_VLinearSum(1.25, vx, -0.75, vy, vz)
    assert_bits_equal(z[idx.cuda()], oracle.linear_sum(1.25, xs, -0.75, ys), "2^31+37 linear_sum")
    S.N_VScale(-3.0, vx, vz)
    assert_bits_equal(z[idx.cuda()], oracle.scale(-3.0, xs), "2^31+37 scale")
    del y, vy
    w = z                                    # reuse the buffer for the weights
    w.copy_(gen(3, n, 0.5, 1.5))
    vw = S.NVector(ctx, w)
    got_w = S.N_VWrmsNorm(vx, vw)
    got_d = S.N_VDotProd(vx, vw)
    got_m = S.N_VMaxNorm(vx)
    ctx.check("2^31+37 reductions")
    ch = 1 << 27
    sq, dd, ad, mx = [], [], [], 0.0
    for s in range(0, n, ch):
        xc, wc = host(x[s:s + ch]), host(w[s:s + ch])
        sq.append(oracle.wsqrsum(xc, wc))
        dd.append(oracle.dot(xc, wc))
        ad.append(float(np.sum(np.abs(xc * wc))))
        mx = max(mx, oracle.max_norm(xc))
    ref_w = math.sqrt(math.fsum(sq) / n)
    assert abs(got_w - ref_w) <= 1e-12 * ref_w, (got_w, ref_w)
    assert abs(got_d - math.fsum(dd)) <= 1e-12 * math.fsum(ad), (got_d, math.fsum(dd))
    assert got_m == mx
    del x, z, w, vx, vz, vw
    torch.cuda.empty_cache()
