"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle,
element by element, bit-exact (integer work: no tolerance).

Small/medium sizes run the full oracle; the BASELINE configs at full size are
checked on sampled rows (computed one by one by the oracle) plus Freivalds'
test on the whole output.
"""
import os

import numpy as np
import pytest

import ffgen
import oracle

pytestmark = pytest.mark.gpu

CONFIG_PRIMES = [251, 65521, 8388593, 67108859]
SMALL_PRIMES = [2, 3, 5, 7, 257, 65279, 65537, 16711423, 2 ** 31 - 1]


@pytest.fixture(scope="module")
def env():
    import torch
    import paper_cs_0601133_b200 as ff
    assert torch.cuda.is_available()
    assert ff.ff_device_check(0) == 0, "device 0 is not sm_100"
    torch.cuda.set_device(0)
    return torch, ff


def _dev(torch, x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _stored(rng, rows, cols, p, ld_extra=0, lo=0):
    buf = rng.integers(lo, p, size=(rows, cols + ld_extra), dtype=np.int64).astype(np.int32)
    return buf


def _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, opts=None):
    """Run through the C ABI on device copies of the stored buffers (ld = buffer width)."""
    A, B, C = _dev(torch, Abuf), _dev(torch, Bbuf), _dev(torch, Cbuf)
    ff.ff_gemm_ex(p, tA, tB, m, n, k, alpha, A, Abuf.shape[1], B, Bbuf.shape[1], beta, C,
                  Cbuf.shape[1], opts)
    torch.cuda.synchronize()
    return C.cpu().numpy()


def _check(p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, got):
    a_cols = k if tA == "N" else m
    b_cols = n if tB == "N" else k
    want = oracle.fgemm(p, tA, tB, alpha, Abuf[:, :a_cols], Bbuf[:, :b_cols], beta,
                        Cbuf[:, :n], m=m, n=n, k=k)
    np.testing.assert_array_equal(got[:m, :n], want)
    # the leading-dimension padding of C is never written
    np.testing.assert_array_equal(got[:, n:], Cbuf[:, n:])


# ---------------------------------------------------------------- generator twin

def test_fill_uniform_matches_numpy_generator(env):
    torch, ff = env
    for p, seed, stream, rows, cols, ld, i0 in [(65521, 1, 0, 37, 53, 60, 0),
                                               (67108859, 5, 2, 300, 129, 129, 0),
                                               (251, 3, 1, 10, 1000, 1000, 777)]:
        X = torch.full((rows, ld), -7, dtype=torch.int32, device="cuda")
        ff.ff_fill_uniform(X, rows, cols, ld, p, seed, stream, i0)
        torch.cuda.synchronize()
        got = X.cpu().numpy()
        want = ffgen.uniform_flat(p, seed, stream, i0, rows * cols).reshape(rows, cols)
        np.testing.assert_array_equal(got[:, :cols], want)
        assert (got[:, cols:] == -7).all()


def _limb_opts(ff, p, k):
    """The limb scheme AUTO would pick if multi-modular were off (fewest limbs, S on ties)."""
    LS = ff.ff_plan_query(p, k, {"scheme": 1})["L"]
    LT = ff.ff_plan_query(p, k, {"scheme": 2})["L"]
    return {"scheme": 1 if LS <= LT else 2}


# ---------------------------------------------------------------- encoder

def _decode(limbs, info):
    """Host decode of limb planes: sum_i d_i 256^i with the plan's signedness."""
    L = info["L"]
    acc = np.zeros(limbs.shape[1:], dtype=np.int64)
    for i in range(L - 1, -1, -1):
        d = limbs[i].astype(np.int64)
        d = np.where(d < 0, d + 256, d) if not info["limb_signed"][i] else d
        acc = acc * 256 + d
    return acc


@pytest.mark.parametrize("p", CONFIG_PRIMES + [2, 3, 257, 65537, 2 ** 31 - 1])
@pytest.mark.parametrize("kmajor", [1, 0])
def test_encoder_roundtrip(env, p, kmajor):
    torch, ff = env
    rng = np.random.default_rng(p % 997 + kmajor)
    rows, k = 150, 333      # ragged: not multiples of the 64/16 encoder tiles
    lopt = _limb_opts(ff, p, k)
    info = ff.ff_plan_query(p, k, lopt)
    x = rng.integers(-2 ** 31, 2 ** 31, size=(rows, k), dtype=np.int64).astype(np.int32)
    x[0, :min(k, p)] = np.arange(min(k, p))                       # include 0..p-1 verbatim
    src = x if kmajor else np.ascontiguousarray(x.T)
    X = _dev(torch, src)
    limbs = torch.full((info["L"], rows, info["k_pad"]), 99, dtype=torch.int8, device="cuda")
    ff.ff_encode(p, k, lopt, kmajor, rows, X, src.shape[1], limbs)
    torch.cuda.synchronize()
    lb = limbs.cpu().numpy()
    r = np.mod(x.astype(np.int64), p)
    c = np.where(r > (p - 1) // 2, r - p, r)
    np.testing.assert_array_equal(_decode(lb, info)[:, :k], c)
    assert (lb[:, :, k:] == 0).all()                              # zero K padding
    for i in range(info["L"]):
        d = lb[i].astype(np.int64)
        if not info["limb_signed"][i]:
            d = np.where(d < 0, d + 256, d)
        assert np.abs(d).max() <= info["digit_max"][i]


@pytest.mark.parametrize("p", CONFIG_PRIMES + [65537])
@pytest.mark.parametrize("kmajor", [1, 0])
@pytest.mark.parametrize("scheme", ["limb", "crt"])
def test_encoder_mixed_canonical_groups(env, p, kmajor, scheme):
    """The encoders' short path for canonical groups (every value in [0, p): one
    compare, then centre) next to the Barrett path: mostly canonical inputs with
    ~2% of the values outside [0, p) (negative, = p, >= p, int32 extremes), so
    the groups of a warp mix both paths; limb and CRT planes, both source
    orientations, ragged sizes."""
    torch, ff = env
    rng = np.random.default_rng(p % 991 + 7 * kmajor + (scheme == "crt"))
    rows, k = 197, 1061
    x = rng.integers(0, p, size=(rows, k), dtype=np.int64)
    bad = rng.random((rows, k)) < 0.02
    specials = np.array([-1, p, p + 1, 2 * p - 1, -p, -2 ** 31, 2 ** 31 - 1, -(p - 1)], dtype=np.int64)
    x[bad] = rng.choice(specials, size=int(bad.sum()))
    x[5, :4] = [0, p - 1, (p - 1) // 2, (p + 1) // 2]
    x = x.astype(np.int32)
    src = x if kmajor else np.ascontiguousarray(x.T)
    X = _dev(torch, src)
    r = np.mod(x.astype(np.int64), p)
    c = np.where(r > (p - 1) // 2, r - p, r)
    if scheme == "limb":
        opt = _limb_opts(ff, p, k)
        info = ff.ff_plan_query(p, k, opt)
        out = torch.full((info["L"], rows, info["k_pad"]), 99, dtype=torch.int8, device="cuda")
        ff.ff_encode(p, k, opt, kmajor, rows, X, src.shape[1], out)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(_decode(out.cpu().numpy(), info)[:, :k], c)
    else:
        opt = {"scheme": 3}
        info = ff.ff_plan_query(p, k, opt)
        out = torch.full((info["L"], rows, info["k_pad"]), 99, dtype=torch.int8, device="cuda")
        ff.ff_encode(p, k, opt, kmajor, rows, X, src.shape[1], out)
        torch.cuda.synchronize()
        planes = out.cpu().numpy().astype(np.int64)
        for i, q in enumerate(info["moduli"]):
            np.testing.assert_array_equal(np.mod(planes[i, :, :k], q), np.mod(c, q), err_msg="modulus %d" % q)


@pytest.mark.parametrize("p", CONFIG_PRIMES)
def test_encoder_exhaustive_residues(env, p):
    """decode(encode(r)) = centre(r) for every residue r in [0, p) (p <= 2^26)."""
    torch, ff = env
    k = 4096
    rows = (p + k - 1) // k
    vals = np.arange(rows * k, dtype=np.int64) % p
    X = _dev(torch, vals.astype(np.int32).reshape(rows, k))
    lopt = _limb_opts(ff, p, k)
    info = ff.ff_plan_query(p, k, lopt)
    limbs = torch.empty((info["L"], rows, info["k_pad"]), dtype=torch.int8, device="cuda")
    ff.ff_encode(p, k, lopt, 1, rows, X, k, limbs)
    torch.cuda.synchronize()
    dec = _decode(limbs.cpu().numpy(), info).reshape(-1)
    want = np.where(vals > (p - 1) // 2, vals - p, vals)
    np.testing.assert_array_equal(dec, want)


# ---------------------------------------------------------------- GEMM parity, small/medium

SHAPES = [(1, 1, 1), (3, 5, 7), (128, 256, 128), (129, 257, 129), (200, 300, 1000),
          (256, 512, 640), (77, 600, 33)]


@pytest.mark.parametrize("scheme", ["limb", "crt"])
@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("p", CONFIG_PRIMES)
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_gemm_vs_oracle_shapes(env, p, tA, tB, cta_group, scheme):
    """Both kernels: 128x256 single-CTA and 256x256 CTA-pair (cta_group::2);
    both product schemes: limbs (Horner in TMEM) and multi-modular (CRT)."""
    torch, ff = env
    sopt = _limb_opts(ff, p, 1000) if scheme == "limb" else {"scheme": 3}
    rng = np.random.default_rng(p % 1009 + ord(tA) * 3 + ord(tB) + cta_group)
    for si, (m, n, k) in enumerate(SHAPES):
        ldx = si % 3
        Abuf = _stored(rng, *((m, k) if tA == "N" else (k, m)), p, ldx)
        Bbuf = _stored(rng, *((k, n) if tB == "N" else (n, k)), p, 2 * ldx)
        Cbuf = _stored(rng, m, n, p, ldx + 1)
        alpha = [1, p - 1, 3, int(rng.integers(0, p))][si % 4]
        beta = [0, 1, p - 1, int(rng.integers(0, p))][(si + 1) % 4]
        got = _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf,
                       dict(sopt, cta_group=cta_group))
        _check(p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, got)


@pytest.mark.parametrize("p", SMALL_PRIMES)
def test_gemm_other_primes_and_noncanonical_inputs(env, p):
    torch, ff = env
    rng = np.random.default_rng(p % 10007)
    m, n, k = 190, 300, 450
    Abuf = rng.integers(-2 ** 31, 2 ** 31, size=(m, k), dtype=np.int64).astype(np.int32)
    Bbuf = rng.integers(-2 ** 31, 2 ** 31, size=(k, n), dtype=np.int64).astype(np.int32)
    Cbuf = rng.integers(-2 ** 31, 2 ** 31, size=(m, n), dtype=np.int64).astype(np.int32)
    for alpha, beta in [(1, 0), (2 ** 32 - 1, 2 ** 32 - 1), (p - 1, 1)]:
        got = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf)
        _check(p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, got)


@pytest.mark.parametrize("korder", [1, 2])
@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("p,scheme", [(65521, 2), (65521, 1), (8388593, 1), (67108859, 1),
                                      (251, 1), (8388593, 2), (3, 1), (65537, 1),
                                      (67108859, 3), (65521, 3), (2 ** 31 - 1, 3), (3, 3)])
def test_kb_override_forces_mid_k_reductions(env, p, scheme, cta_group, korder):
    """Shrunk k-block ("overflow safety under shrunk gamma" analogue):
    several mid-k reductions per weight group must not change the result."""
    torch, ff = env
    rng = np.random.default_rng(11)
    m, n, k = 130, 260, 1000
    Abuf, Bbuf, Cbuf = _stored(rng, m, k, p), _stored(rng, k, n, p), _stored(rng, m, n, p)
    opts = {"kb_override": 128, "scheme": scheme, "cta_group": cta_group, "korder": korder}
    assert ff.ff_plan_query(p, k, opts)["num_kblocks"] == 8     # (CRT plans always run korder 1)
    got = _run_gpu(torch, ff, p, "N", "N", m, n, k, 5, Abuf, Bbuf, 7, Cbuf, opts)
    _check(p, "N", "N", m, n, k, 5, Abuf, Bbuf, 7, Cbuf, got)


def _adversarial_residue(p, info):
    """A residue whose limbs attain the digit bound of every limb (|d_i| = D_i)."""
    L = info["L"]
    if info["scheme"] == "T":
        # low bytes 255, top byte -128  (p = 65521: c = -32513, residue 33008)
        c = -128 * 256 ** (L - 1) + sum(255 * 256 ** i for i in range(L - 1))
    else:
        top = -info["digit_max"][-1]
        c = top * 256 ** (L - 1) + sum(-128 * 256 ** i for i in range(L - 1))
        while c < -((p - 1) // 2):       # stay inside the centred range
            top += 1
            c += 256 ** (L - 1)
    assert -((p - 1) // 2) <= c <= (p - 1) // 2
    return c % p


@pytest.mark.parametrize("p", CONFIG_PRIMES)
def test_accumulator_at_the_bound_closed_form(env, p):
    """All entries = a digit-extreme residue v, k = the planner's largest k-block
    (and 2 k-blocks + a ragged tail): every entry must be k v^2 mod p."""
    torch, ff = env
    lopt = _limb_opts(ff, p, 1)
    info = ff.ff_plan_query(p, 1, dict(lopt, korder=1))   # the safety k-block
    v = _adversarial_residue(p, info)
    if p == 65521:
        assert v == 33008
    for k in (info["kb"], 2 * info["kb"] + 45):
        m, n = 256, 512
        A = torch.full((m, k), v, dtype=torch.int32, device="cuda")
        B = torch.full((k, n), v, dtype=torch.int32, device="cuda")
        C = torch.empty((m, n), dtype=torch.int32, device="cuda")
        for sat, grp, ko in ((0, 1, 1), (1, 1, 1), (0, 2, 1), (1, 2, 1), (0, 2, 2), (1, 1, 2)):
            C.fill_(-1)
            kbo = info["kb"] if ko == 1 else 0      # k-outer: the locality k-block, several per k
            ff.ff_gemm_ex(p, "N", "N", m, n, k, 1, A, k, B, n, 0, C, n,
                          dict(lopt, debug_saturate=sat, cta_group=grp, korder=ko, kb_override=kbo))
            torch.cuda.synchronize()
            assert (C == (k * v * v) % p).all().item(), (p, k, sat, grp, ko)


# ---------------------------------------------------------------- multi-modular (CRT) specifics

@pytest.mark.parametrize("p", CONFIG_PRIMES + [2, 3, 65537, 2 ** 31 - 1])
@pytest.mark.parametrize("kmajor", [1, 0])
def test_crt_encoder_residue_planes(env, p, kmajor):
    """Plane i holds the centred residue of centre(x mod p) modulo q_i, as s8."""
    torch, ff = env
    rng = np.random.default_rng(p % 991 + 7 * kmajor)
    rows, k = 150, 333
    opts = {"scheme": 3}
    info = ff.ff_plan_query(p, k, opts)
    x = rng.integers(-2 ** 31, 2 ** 31, size=(rows, k), dtype=np.int64).astype(np.int32)
    x[0, :min(k, p)] = np.arange(min(k, p))
    src = x if kmajor else np.ascontiguousarray(x.T)
    planes = torch.full((info["L"], rows, info["k_pad"]), 99, dtype=torch.int8, device="cuda")
    ff.ff_encode(p, k, opts, kmajor, rows, _dev(torch, src), src.shape[1], planes)
    torch.cuda.synchronize()
    pl = planes.cpu().numpy().astype(np.int64)
    r = np.mod(x.astype(np.int64), p)
    c = np.where(r > (p - 1) // 2, r - p, r)
    for i, q in enumerate(info["moduli"]):
        d = pl[i, :, :k]
        assert ((d - c) % q == 0).all(), (p, q)
        assert d.min() >= -(q // 2) and d.max() <= (q - 1) // 2
        assert (pl[i, :, k:] == 0).all()


@pytest.mark.parametrize("p,k", [(67108859, 16384), (67108859, 333), (2 ** 31 - 1, 4096),
                                 (65521, 8192), (8388593, 4096), (65537, 1000)])
def test_crt_dot_product_at_the_bound(env, p, k):
    """|X| = k cmax^2, the largest exact dot product the moduli must recover
    (M >= 4 k cmax^2): all entries -cmax (X = +k cmax^2) and A = -cmax against
    B = +cmax (X = -k cmax^2); every entry must be X mod p."""
    torch, ff = env
    cm = (p - 1) // 2
    m, n = 256, 512
    for va, vb in ((p - cm, p - cm), (p - cm, cm), (cm, cm)):
        A = torch.full((m, k), va, dtype=torch.int32, device="cuda")
        B = torch.full((k, n), vb, dtype=torch.int32, device="cuda")
        C = torch.empty((m, n), dtype=torch.int32, device="cuda")
        X = k * ((va + cm) % p - cm) * ((vb + cm) % p - cm)
        assert abs(X) == k * cm * cm
        for grp in (1, 2):
            C.fill_(-1)
            ff.ff_gemm_ex(p, "N", "N", m, n, k, 1, A, k, B, n, 0, C, n, {"scheme": 3, "cta_group": grp})
            torch.cuda.synchronize()
            assert (C == X % p).all().item(), (p, k, va, vb, grp)


@pytest.mark.parametrize("p", [251, 65521, 8388593])
def test_wide_tiles_tiny_and_degenerate(env, p):
    """Forced 256 x 512 tiles on shapes far below one tile (1 x 1 x 1, a single row
    or column, k = 1, k = 129 across one k-slice boundary, n just past 256 and
    512), plus the quick returns (k = 0, alpha = 0), against the oracle and the
    square tiles."""
    torch, ff = env
    rng = np.random.default_rng(p % 101)
    for (m, n, k) in [(1, 1, 1), (1, 700, 33), (300, 1, 129), (5, 257, 1), (256, 513, 128), (257, 511, 255)]:
        A = _stored(rng, m, k, p, 1)
        B = _stored(rng, k, n, p, 2)
        C = _stored(rng, m, n, p, 3)
        alpha, beta = int(rng.integers(0, p)), int(rng.integers(0, p))
        opts = {"scheme": 1, "small_path": -1, "cta_group": 2}    # the pair kernel even for tiny outputs
        wide = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, A, B, beta, C, dict(opts, wide_tiles=1))
        square = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, A, B, beta, C, dict(opts, wide_tiles=-1))
        np.testing.assert_array_equal(wide, square, err_msg="m=%d n=%d k=%d" % (m, n, k))
        _check(p, "N", "N", m, n, k, alpha, A, B, beta, C, wide)
    C = _stored(rng, 40, 600, p)
    A = _stored(rng, 40, 8, p)
    B = _stored(rng, 8, 600, p)
    got = _run_gpu(torch, ff, p, "N", "N", 40, 600, 0, 3, A, B, 5, C, {"wide_tiles": 1, "cta_group": 2})
    np.testing.assert_array_equal(got[:, :600], (5 * C[:, :600].astype(np.int64)) % p)
    got = _run_gpu(torch, ff, p, "N", "N", 40, 600, 8, 0, A, B, 5, C, {"wide_tiles": 1, "cta_group": 2})
    np.testing.assert_array_equal(got[:, :600], (5 * C[:, :600].astype(np.int64)) % p)


def test_quick_returns_and_degenerate(env):
    torch, ff = env
    p = 65521
    rng = np.random.default_rng(3)
    Cbuf = _stored(rng, 70, 90, p, 3)
    A = _stored(rng, 70, 0 + 1, p)
    B = _stored(rng, 1, 90, p)
    # k = 0: C <- beta C
    got = _run_gpu(torch, ff, p, "N", "N", 70, 90, 0, 5, A, B, 3, Cbuf)
    np.testing.assert_array_equal(got[:, :90], (3 * Cbuf[:, :90].astype(np.int64)) % p)
    # alpha = 0: C <- beta C
    got = _run_gpu(torch, ff, p, "N", "N", 70, 90, 1, 0, A, B, 2, Cbuf)
    np.testing.assert_array_equal(got[:, :90], (2 * Cbuf[:, :90].astype(np.int64)) % p)
    # beta = 0: C is not read (garbage in, exact product out)
    junk = np.full_like(Cbuf, -1)
    got = _run_gpu(torch, ff, p, "N", "N", 70, 90, 1, 1, A, B, 0, junk)
    _check(p, "N", "N", 70, 90, 1, 1, A, B, 0, junk, got)
    # m = 0 / n = 0: no-op
    C = _dev(torch, Cbuf)
    ff.ff_gemm_ex(p, "N", "N", 0, 90, 5, 1, C, 5, C, 93, 1, C, 93)
    ff.ff_gemm_ex(p, "N", "N", 70, 0, 5, 1, C, 5, C, 1, 1, C, 93)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(C.cpu().numpy(), Cbuf)


def test_identity_permutation_on_gpu(env):
    torch, ff = env
    p = 67108859
    rng = np.random.default_rng(4)
    n = 300
    sigma = rng.permutation(n)
    P = np.zeros((n, n), dtype=np.int32)
    P[np.arange(n), sigma] = 1
    B = _stored(rng, n, 270, p)
    got = _run_gpu(torch, ff, p, "N", "N", n, 270, n, 1, P, B, 0, np.zeros((n, 270), np.int32))
    np.testing.assert_array_equal(got, B[sigma])


@pytest.mark.parametrize("tA,tB,beta,block,p", [("T", "N", 1, 0, 8388593), ("N", "N", 0, 256, 8388593),
                                                 ("T", "T", 5, 256, 8388593), ("N", "T", 0, 512, 8388593),
                                                 ("N", "N", 3, 256, 67108859), ("T", "N", 0, 0, 67108859),
                                                 ("T", "N", 1, 0, 251), ("N", "T", 0, 256, 251)])
def test_host_entry_point(env, tA, tB, beta, block, p):
    """ff_gemm_host: host buffers, pipelined over blocks of C (block=256 forces
    several row panels and column chunks, with ragged last blocks); p = 67108859
    runs the multi-modular (CRT) plan through the same pipeline."""
    torch, ff = env
    rng = np.random.default_rng(5 + block)
    m, n, k = 700, 900, 555
    A = _stored(rng, *((m, k) if tA == "N" else (k, m)), p, 1)
    B = _stored(rng, *((k, n) if tB == "N" else (n, k)), p, 2)
    C = _stored(rng, m, n, p, 3)
    out = C.copy()
    ff.ff_gemm_host(p, tA, tB, m, n, k, 3, A, A.shape[1], B, B.shape[1], beta, out, out.shape[1],
                    {"host_block": block})
    _check(p, tA, tB, m, n, k, 3, A, B, beta, C, out)


def test_host_entry_point_wide_blocks(env):
    """ff_gemm_host with blocks large enough for the 256 x 512 tiles (p = 251:
    one limb): sampled rows against the oracle, Freivalds on the whole output."""
    torch, ff = env
    p, m, n, k = 251, 5000, 4700, 1500
    rng = np.random.default_rng(17)
    A = _stored(rng, k, m, p)          # transA = T
    B = _stored(rng, k, n, p)
    C = _stored(rng, m, n, p)
    out = C.copy()
    ff.ff_gemm_host(p, "T", "N", m, n, k, 7, A, m, B, n, 2, out, n, None)
    rows = [0, 1, 2047, 4095, 4096, m - 1]
    want = oracle.fgemm_rows(p, "T", "N", 7, A, B, 2, C[rows], rows, m, n, k)
    np.testing.assert_array_equal(out[rows], want)
    x = rng.integers(0, p, size=n).astype(np.int32)
    lhs = oracle.matvec(p, "N", out, x).astype(np.int64)
    rhs = (7 * oracle.matvec(p, "T", A, oracle.matvec(p, "N", B, x)).astype(np.int64) +
           2 * oracle.matvec(p, "N", C, x).astype(np.int64)) % p
    np.testing.assert_array_equal(lhs, rhs)


def test_split_entry_points_chunked_B(env):
    """Encode once, multiply by column chunks of B (the multi-GPU building block)."""
    torch, ff = env
    p = 65521
    rng = np.random.default_rng(6)
    m, n, k = 300, 700, 900
    A, B, C = _stored(rng, m, k, p), _stored(rng, k, n, p), _stored(rng, m, n, p)
    info = ff.ff_plan_query(p, k)
    L, kp = info["L"], info["k_pad"]
    dA, dB, dC = _dev(torch, A), _dev(torch, B), _dev(torch, C)
    Al = torch.empty((L, m, kp), dtype=torch.int8, device="cuda")
    ff.ff_encode(p, k, None, 1, m, dA, k, Al)
    for n0, n1 in [(0, 256), (256, 300), (300, 700)]:
        Bl = torch.empty((L, n1 - n0, kp), dtype=torch.int8, device="cuda")
        ff.ff_encode(p, k, None, 0, n1 - n0, dB[:, n0:], n, Bl)
        ff.ff_gemm_limbs(p, m, n1 - n0, k, None, 7, Al, Bl, 2, dC[:, n0:], n)
    torch.cuda.synchronize()
    want = oracle.fgemm(p, "N", "N", 7, A, B, 2, C)
    np.testing.assert_array_equal(dC.cpu().numpy(), want)


# ---------------------------------------------------------------- BASELINE configs, full size

CONFIGS = {
    # name: (p, m, n, k, transA, transB, alpha, beta, seed)
    "c1": (65521, 512, 512, 512, "N", "N", 1, 0, 1),
    "c2": (8388593, 4096, 4096, 4096, "N", "N", 3, 1, 2),
    "c3": (251, 8192, 8192, 16384, "T", "N", 1, 0, 3),
    "c4": (65521, 32768, 32768, 8192, "N", "N", 1, 0, 4),
    "c5": (67108859, 16384, 16384, 16384, "N", "N", 67108858, 1, 5),
}


def _make_config(torch, ff, name):
    p, m, n, k, tA, tB, alpha, beta, seed = CONFIGS[name]
    ar, ac = (m, k) if tA == "N" else (k, m)
    br, bc = (k, n) if tB == "N" else (n, k)
    A = torch.empty((ar, ac), dtype=torch.int32, device="cuda")
    B = torch.empty((br, bc), dtype=torch.int32, device="cuda")
    C = torch.empty((m, n), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(A, ar, ac, ac, p, seed, ffgen.STREAM_A)
    ff.ff_fill_uniform(B, br, bc, bc, p, seed, ffgen.STREAM_B)
    if beta:
        ff.ff_fill_uniform(C, m, n, n, p, seed, ffgen.STREAM_C)
    return A, B, C


@pytest.mark.parametrize("p,tA,tB,m,n,k,opts", [
    (251, "N", "N", 3000, 3300, 1000, None),       # one limb; last tile: 2nd half empty
    (251, "T", "N", 3072, 3500, 1536, None),       # 2nd half partial
    (7, "N", "T", 2600, 3900, 777, None),
    (2, "T", "T", 3000, 3600, 2048, None),
    (127, "N", "N", 2560, 4096, 16500, None),      # long k
    (65521, "N", "N", 3000, 3300, 1000, None),     # 2 limbs (T): 3 weight groups, Horner write-backs
    (8388593, "T", "N", 3072, 3500, 1536, None),   # 3 limbs (S): 5 groups
    (65537, "N", "T", 2600, 3900, 777, {"scheme": 1}),                  # 3 limbs, ragged
    (65521, "N", "N", 3000, 3300, 1000, {"kb_override": 256, "korder": 1}),  # mid-k reductions
    (65521, "T", "N", 3000, 3300, 1000, {"kb_override": 256, "korder": 2}),  # k-outer: rescaled write-backs
    (8388593, "N", "N", 2600, 3600, 900, {"kb_override": 384, "korder": 2}),
])
def test_wide_tiles_vs_oracle(env, p, tA, tB, m, n, k, opts):
    """256 x 512 CTA-pair tiles (ff_opts.wide_tiles = 1; automatic for one limb):
    two N = 256 MMAs per A stage, the accumulator in all 512 TMEM columns, halves
    staggered through every write-back and the final output.  One to three limbs,
    forced k-blocks, ragged m, n (second 256-column half of the last tile empty or
    partial), all transposes, alpha/beta: bit-identical to the 256 x 256 tiles
    (wide_tiles = -1), sampled rows against the oracle, Freivalds on the whole output."""
    torch, ff = env
    rng = np.random.default_rng(m + n + k + p)
    Abuf = _stored(rng, *((m, k) if tA == "N" else (k, m)), p)
    Bbuf = _stored(rng, *((k, n) if tB == "N" else (n, k)), p)
    Cbuf = _stored(rng, m, n, p)
    alpha, beta = 3 % p, (p - 1) % p
    out = _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, dict(opts or {}, wide_tiles=1))
    square = _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, dict(opts or {}, wide_tiles=-1))
    np.testing.assert_array_equal(out, square)           # 256 x 512 and 256 x 256 tiles agree bit for bit
    rows = sorted(set([0, 1, 255, 256, 511, m // 2, m - 1] + rng.integers(0, m, size=4).tolist()))
    want = oracle.fgemm_rows(p, tA, tB, alpha, Abuf, Bbuf, beta, Cbuf[rows], rows, m, n, k)
    np.testing.assert_array_equal(out[rows], want)
    for t in range(3):
        x = rng.integers(0, p, size=n).astype(np.int32)
        lhs = oracle.matvec(p, "N", out, x).astype(np.int64)
        abx = oracle.matvec(p, tA, Abuf, oracle.matvec(p, tB, Bbuf, x)).astype(np.int64)
        rhs = (alpha * abx + beta * oracle.matvec(p, "N", Cbuf, x).astype(np.int64)) % p
        np.testing.assert_array_equal(lhs, rhs)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_baseline_config_sampled_rows_and_freivalds(env, name):
    torch, ff = env
    p, m, n, k, tA, tB, alpha, beta, seed = CONFIGS[name]
    A, B, C = _make_config(torch, ff, name)
    Cin = C.cpu().numpy() if beta else None
    ff.fgemm(p, A, B, C, alpha, beta, tA, tB)
    torch.cuda.synchronize()
    out = C.cpu().numpy()
    Ah, Bh = A.cpu().numpy(), B.cpu().numpy()
    # inputs are exactly the seeded generator's (no CUDA-side value is trusted)
    np.testing.assert_array_equal(Ah[:3], ffgen.uniform_matrix(p, seed, 0, *Ah.shape, row0=0, nrows=3))
    rng = np.random.default_rng(seed)
    rows = sorted(set([0, m - 1, 127, 128, m // 2] + rng.integers(0, m, size=5).tolist()))
    want = oracle.fgemm_rows(p, tA, tB, alpha, Ah, Bh, beta,
                             Cin[rows] if beta else None, rows, m, n, k)
    np.testing.assert_array_equal(out[rows], want)
    # Freivalds (t = 4): C_out x = alpha A (B x) + beta C_in x  (mod p), x random
    for t in range(4):
        x = ffgen.uniform_vector(p, seed, 8 + t, n)
        lhs = oracle.matvec(p, "N", out, x).astype(np.int64)
        bx = oracle.matvec(p, tB, Bh, x)
        abx = oracle.matvec(p, tA, Ah, bx).astype(np.int64)
        rhs = (alpha % p) * abx % p
        if beta:
            rhs = (rhs + (beta % p) * oracle.matvec(p, "N", Cin, x).astype(np.int64)) % p
        np.testing.assert_array_equal(lhs, rhs)
    assert out.min() >= 0 and out.max() < p


@pytest.mark.parametrize("world,name", [(2, "c1"), (4, "c1"), (3, "mixed"), (3, "c5int32"), (2, "c5wino"),
                                        (3, "c3planes")])
def test_row_panel_virtual_ranks_match_single_gpu(env, world, name):
    """The multi-GPU row-panel path run as `world` virtual ranks on one GPU (rank
    0's broadcast buffers -- encoded planes, or int32 chunks of B -- copied to the
    others, standing in for the NCCL broadcast): the concatenated panels must
    equal the single-GPU result bit for bit.  c5int32 / c5wino are c5-shaped
    (p = 2^26 - 5, CRT, alpha = -1, beta = 1): int32 broadcast with per-rank
    encoding, and (forced Winograd) one ff_gemm_ex per panel with the local
    one-level Winograd of SURVEY §8(e)."""
    torch, ff = env
    from paper_cs_0601133_b200.sharded import Problem, RowPanelGemm
    opts, mode = None, None
    if name == "c1":
        p, m, n, k, tA, tB, alpha, beta = 65521, 512, 512, 512, "N", "N", 1, 0
    elif name == "c5int32":
        p, m, n, k, tA, tB, alpha, beta = 67108859, 1000, 1300, 777, "N", "N", 67108858, 1
        mode = "int32"
    elif name == "c5wino":
        p, m, n, k, tA, tB, alpha, beta = 67108859, 2048, 1536, 1024, "N", "N", 67108858, 1
        opts, mode = {"winograd": 1}, "int32"
    elif name == "c3planes":
        p, m, n, k, tA, tB, alpha, beta = 251, 1024, 768, 2048, "T", "N", 1, 0
        mode = "planes"
    else:
        p, m, n, k, tA, tB, alpha, beta = 67108859, 700, 1100, 300, "T", "N", 67108858, 1
    rng = np.random.default_rng(world)
    A = _stored(rng, *((m, k) if tA == "N" else (k, m)), p)
    B = _stored(rng, *((k, n) if tB == "N" else (n, k)), p)
    C = _stored(rng, m, n, p)
    dA, dB = _dev(torch, A), _dev(torch, B)
    want = _dev(torch, C)
    ff.fgemm(p, dA, dB, want, alpha, beta, tA, tB)
    prob = Problem(p, m, n, k, tA, tB, alpha, beta)
    engs = [RowPanelGemm(prob, chunks=3, world=world, rank=r, opts=opts, mode=mode or "auto")
            for r in range(world)]
    if mode:
        assert all(e.mode == mode for e in engs)
    if name == "c5wino":
        assert all(e.whole for e in engs)
    out = _dev(torch, C)
    eng0 = engs[0]
    eng0.step(eng0.a_panel_view(dA), dB, out[eng0.row0:eng0.row1])
    torch.cuda.synchronize()
    for e in engs[1:]:
        for dst, src in zip(e.bcast_buffers(), eng0.bcast_buffers()):
            dst.copy_(src)                       # stands in for the NCCL broadcast
        e.step(e.a_panel_view(dA), None, out[e.row0:e.row1])
    torch.cuda.synchronize()
    assert torch.equal(out, want)
    got = out.cpu().numpy()
    np.testing.assert_array_equal(got, oracle.fgemm(p, tA, tB, alpha, A, B, beta, C))


# ---------------------------------------------------------------- one Winograd level (row a7)

@pytest.mark.parametrize("p", [251, 65521, 8388593, 65537])
def test_winograd_products_on_wide_tiles(env, p):
    """The Winograd products' multi-output epilogues (raw temporaries, addends,
    two read-modify-written quadrants) on the 256 x 512 tiles (wide_tiles = 1,
    limb schemes): bit-identical to the square tiles and to the classical path,
    and exact against the oracle."""
    torch, ff = env
    rng = np.random.default_rng(p % 997)
    m, n, k = 1536, 2048, 768
    Abuf = _stored(rng, m, k, p, 1)
    Bbuf = _stored(rng, k, n, p, 2)
    Cbuf = _stored(rng, m, n, p, 3)
    alpha, beta = p - 1, 1
    base = {"winograd": 1, "scheme": 1}
    wide = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, dict(base, wide_tiles=1))
    square = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, dict(base, wide_tiles=-1))
    np.testing.assert_array_equal(wide, square)
    classic = _run_gpu(torch, ff, p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, {"winograd": -1})
    np.testing.assert_array_equal(wide, classic)
    _check(p, "N", "N", m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, wide)


@pytest.mark.parametrize("p", CONFIG_PRIMES + [2, 3, 2 ** 31 - 1])
@pytest.mark.parametrize("tA,tB", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_winograd_level_vs_oracle(env, p, tA, tB):
    """One Winograd level (Table 2, A22 fix) fused into the GEMM
    epilogues: bit-exact against the oracle, and bit-identical to the classical
    path ("level invariance")."""
    torch, ff = env
    rng = np.random.default_rng(p % 991 + ord(tA) + 2 * ord(tB))
    for (m, n, k) in [(512, 512, 256), (768, 1024, 640), (1030, 514, 258)]:
        Abuf = _stored(rng, *((m, k) if tA == "N" else (k, m)), p, 3)
        Bbuf = _stored(rng, *((k, n) if tB == "N" else (n, k)), p, 1)
        Cbuf = _stored(rng, m, n, p, 2)
        for alpha, beta in [(1, 0), (p - 1, 1), (int(rng.integers(0, p)), int(rng.integers(0, p)))]:
            got = _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, {"winograd": 1})
            _check(p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, got)
            classic = _run_gpu(torch, ff, p, tA, tB, m, n, k, alpha, Abuf, Bbuf, beta, Cbuf, {"winograd": -1})
            np.testing.assert_array_equal(got, classic)


def test_winograd_rejects_odd_shapes(env):
    torch, ff = env
    A = torch.zeros((513, 256), dtype=torch.int32, device="cuda")
    B = torch.zeros((256, 512), dtype=torch.int32, device="cuda")
    C = torch.zeros((513, 512), dtype=torch.int32, device="cuda")
    with pytest.raises(ff.FFError):
        ff.fgemm(65521, A, B, C, opts={"winograd": 1})


def test_c5_full_size_crt_equals_limbs(env):
    """c5 at full size: the multi-modular path (the default there) and the
    4-limb Horner path give bit-identical outputs."""
    torch, ff = env
    p, m, n, k, tA, tB, alpha, beta, seed = CONFIGS["c5"]
    A, B, C = _make_config(torch, ff, "c5")
    assert ff.ff_plan_query(p, k)["scheme"] == "CRT"
    ref = C.clone()
    ff.fgemm(p, A, B, C, alpha, beta, tA, tB, opts={"scheme": 3, "winograd": -1})
    ff.fgemm(p, A, B, ref, alpha, beta, tA, tB, opts={"scheme": 1, "winograd": -1})
    torch.cuda.synchronize()
    assert torch.equal(C, ref)


@pytest.mark.parametrize("name", ["c2", "c5"])
def test_baseline_config_winograd_sampled_rows(env, name):
    torch, ff = env
    p, m, n, k, tA, tB, alpha, beta, seed = CONFIGS[name]
    A, B, C = _make_config(torch, ff, name)
    Cin = C.clone()
    ff.fgemm(p, A, B, C, alpha, beta, tA, tB, opts={"winograd": 1})
    ref = Cin.clone()
    ff.fgemm(p, A, B, ref, alpha, beta, tA, tB, opts={"winograd": -1})
    torch.cuda.synchronize()
    assert torch.equal(C, ref)                 # level invariance at full size
    out, Ah, Bh, Cinh = C.cpu().numpy(), A.cpu().numpy(), B.cpu().numpy(), Cin.cpu().numpy()
    rows = [0, 1, m // 2 - 1, m // 2, m - 1]
    want = oracle.fgemm_rows(p, tA, tB, alpha, Ah, Bh, beta, Cinh[rows], rows, m, n, k)
    np.testing.assert_array_equal(out[rows], want)


@pytest.mark.parametrize("p,opts", [(65521, None), (65521, {"scheme": 3}), (2 ** 31 - 1, None), (251, None)])
def test_huge_k_sampled_rows_and_freivalds(env, p, opts):
    """k = 2^20 + 37 (ragged last k-tile; dozens of delayed-reduction k-blocks
    per weight group for the large primes): sampled rows against the oracle
    and Freivalds' test on the whole output, adversarial inputs (every entry
    p - 1, the largest centred magnitude) in half of A."""
    torch, ff = env
    m, n, k = 300, 200, (1 << 20) + 37
    rng = np.random.default_rng(p % 1000 + (3 if opts else 0))
    A = rng.integers(0, p, size=(m, k), dtype=np.int64).astype(np.int32)
    A[: m // 2] = p - 1
    B = rng.integers(0, p, size=(k, n), dtype=np.int64).astype(np.int32)
    C = rng.integers(0, p, size=(m, n), dtype=np.int64).astype(np.int32)
    alpha, beta = p - 1, 1
    dA, dB, dC = (torch.from_numpy(x).cuda() for x in (A, B, C))
    ff.ff_gemm_ex(p, "N", "N", m, n, k, alpha, dA, k, dB, n, beta, dC, n, opts)
    torch.cuda.synchronize()
    out = dC.cpu().numpy()
    rows = [0, 1, m // 2 - 1, m // 2, m - 1]
    np.testing.assert_array_equal(out[rows], oracle.fgemm_rows(p, "N", "N", alpha, A, B, beta, C[rows], rows, m, n, k))
    for t in range(2):
        x = ffgen.uniform_vector(p, 99, 40 + t, n)
        lhs = oracle.matvec(p, "N", out, x).astype(np.int64)
        rhs = ((alpha % p) * oracle.matvec(p, "N", A, oracle.matvec(p, "N", B, x)).astype(np.int64)
               + beta * oracle.matvec(p, "N", C, x).astype(np.int64)) % p
        np.testing.assert_array_equal(lhs, rhs)


def test_more_than_2_31_elements_sampled_rows(env):
    """m = 3 * 2^26 rows, n = 16, k = 16: A and C hold 3 * 2^30 elements each
    (12 GiB; the limb planes, k padded to 128, 48 GiB), so every row past 2^27
    is addressed beyond 2^31 elements.  A comes from the
    device twin of the seeded generator; the sampled rows (around the 2^31-
    element boundary and at the end) are regenerated on the host by ffgen and
    checked against the oracle."""
    torch, ff = env
    p, m, n, k, seed = 65521, 3 << 26, 16, 16, 5
    A = torch.empty((m, k), dtype=torch.int32, device="cuda")
    ff.ff_fill_uniform(A, m, k, k, p, seed, 0)
    B = torch.from_numpy(ffgen.uniform_matrix(p, seed, 1, k, n)).cuda()
    C = torch.empty((m, n), dtype=torch.int32, device="cuda")
    ff.fgemm(p, A, B, C, 3, 0)
    torch.cuda.synchronize()
    edge = (1 << 31) // n
    rows = [0, edge - 1, edge, edge + 1, m - 2, m - 1]
    got = C[rows].cpu().numpy()
    Bh = B.cpu().numpy()
    for i, r in enumerate(rows):
        Ar = ffgen.uniform_matrix(p, seed, 0, m, k, row0=r, nrows=1)
        want = oracle.fgemm(p, "N", "N", 3, Ar, Bh, 0, None, m=1, n=n, k=k)
        np.testing.assert_array_equal(got[i:i + 1], want, err_msg="row %d" % r)
    del A, C
    torch.cuda.empty_cache()


# ---------------------------------------------------------------- instrumentation used by bench.py

def test_prof_events_and_launch_counts(env):
    """ff_prof_start/stop: one event pair per GEMM-kernel launch on its own stream,
    a count of every fgemm-path launch (encoders included), durations > 0; and
    ff_mma_ceiling returns a plausible tcgen05 int8 rate."""
    torch, ff = env
    p = 65521
    A = torch.randint(0, p, (2048, 2048), dtype=torch.int32, device="cuda")
    B = torch.randint(0, p, (2048, 2048), dtype=torch.int32, device="cuda")
    C = torch.zeros((2048, 2048), dtype=torch.int32, device="cuda")
    ff.fgemm(p, A, B, C)
    torch.cuda.synchronize()
    ff.ff_prof_start(16)
    for _ in range(3):
        ff.fgemm(p, A, B, C)                       # encode A, encode B, tcgen05 GEMM
    ms, launches = ff.ff_prof_stop(16)
    assert len(ms) == 3 and all(t > 0 for t in ms)
    assert launches == 9
    ff.ff_prof_start(4)
    ff.fgemm(p, A[:512, :512], B[:512, :512], C[:512, :512])   # one latency-kernel launch
    ms, launches = ff.ff_prof_stop(4)
    assert len(ms) == 1 and launches == 1
    tops = ff.ff_mma_ceiling(20000)
    assert 1000 < tops < 6000
