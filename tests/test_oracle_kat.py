"""CPU oracle against the reference's worked examples and properties.

SPEC.md:228-230 (compress KATs), 237-239 (decompress KATs), 268-273 (properties),
and the GLL operator identities of DESIGN.md 3.1-3.2 (north_star DLT).
"""
import math

import numpy as np
import pytest


@pytest.mark.parametrize("lx", range(2, 17))
def test_gll_identities(oracle, lx):
    x, w = oracle.gll(lx)
    F, B = oracle.matrices(lx)
    assert abs(w.sum() - 2.0) <= 4e-16 * lx                     # sum of weights
    assert np.all(x[:-1] < x[1:]) and x[0] == -1.0 and x[-1] == 1.0
    assert np.array_equal(x, -x[::-1]) and np.array_equal(w, w[::-1])  # exact mirroring
    assert np.abs(F @ B - np.eye(lx)).max() <= 8e-16 * lx     # F B = I (orthonormal DLT)
    sgn = np.array([(-1) ** k for k in range(lx)])
    assert np.array_equal(F[:, ::-1], F * sgn[:, None])        # parity, bitwise
    assert np.array_equal(B[::-1, :], B * sgn[None, :])
    # Q = diag(sqrt w) B orthogonal  (discrete GLL norm, gamma_N = 2/N)
    Q = np.sqrt(w)[:, None] * B
    assert np.abs(Q.T @ Q - np.eye(lx)).max() <= 8e-16 * lx


@pytest.mark.parametrize("lx", [2, 3, 6, 8, 11, 12])
def test_parseval_and_roundtrip(oracle, lx):
    rng = np.random.default_rng(lx)
    u = rng.standard_normal(lx ** 3)
    a = oracle.fwd_block(lx, u)
    x, w = oracle.gll(lx)
    W3 = np.einsum("i,j,k->ijk", w, w, w).reshape(-1)  # [z][y][x]
    assert abs((a * a).sum() / (W3 * u * u).sum() - 1.0) <= 1e-9
    ur = oracle.inv_block(lx, a)
    assert np.abs(ur - u).max() <= 1e-13 * np.abs(u).max()


def test_constant_field_one_coefficient(oracle):
    # constant c != 0 -> exactly 1 kept coefficient per element, and
    # the reconstruction is exact up to the fp64 transform (<= 8 ulp)
    for c in (1.0, -3.7, 1e-200, 7e300, 4e-310):
        u = np.full(8 * 512, c)
        rc, s, st = oracle.compress(u, 8, 1, 1e-3)
        assert rc == 0 and st.kept == 8
        rc, out, _ = oracle.decompress(s, 8, 1, 8)
        assert np.max(np.abs(out - c)) <= 8 * np.spacing(abs(c))


def test_zero_field(oracle):
    # all-zero element keeps 0 coefficients; exact reconstruction
    u = np.zeros(8 * 512)
    rc, s, st = oracle.compress(u, 8, 1, 1e-2)
    assert rc == 0 and st.kept == 0
    rc, out, st2 = oracle.decompress(s, 8, 1, 8, original=u)
    assert np.all(out == 0.0) and st2.err2 == 0.0


def test_tgv_kept_fraction_kat(oracle):
    # TGV, E=8, P=8, max_error=1e-2, RelativeL2 -> kept fraction <= 0.05
    u = oracle.gen_tgv(8, 8, 0)
    rc, s, st = oracle.compress(u, 8, 1, 1e-2)
    assert rc == 0
    assert st.kept / u.size <= 0.05
    # decompress(compress(tgv)) RelativeL2 error <= 1e-2
    rc, out, st2 = oracle.decompress(s, 8, 1, 512, original=u)
    assert math.sqrt(st2.err2 / st2.nrm2) <= 1e-2


@pytest.mark.parametrize("lx,eps", [(6, 1e-2), (8, 1e-3), (8, 1e-5), (10, 1e-4), (12, 1e-3)])
def test_error_guarantee(oracle, lx, eps):
    # reconstruct error <= max_error for randomized smooth fields; the
    # guarantee holds per element, hence also for the whole field
    u = oracle.gen_spectral(lx, 48, block0=lx * 1000)
    rc, s, st = oracle.compress(u, lx, 1, eps)
    rc, out, st2 = oracle.decompress(s, lx, 1, 48, original=u)
    assert math.sqrt(st2.err2 / st2.nrm2) <= eps * (1 + 1e-9)
    # coefficient-space (Parseval) estimate is an upper bound of the truncation error
    assert math.sqrt(st.disc2 / st.tot2) >= math.sqrt(st2.err2 / st2.nrm2) * (1 - 1e-6)
    n3 = lx ** 3
    x, w = oracle.gll(lx)
    W3 = np.einsum("i,j,k->ijk", w, w, w).reshape(-1)
    for b in range(48):
        ub, ob = u[b * n3:(b + 1) * n3], out[b * n3:(b + 1) * n3]
        e = math.sqrt((W3 * (ub - ob) ** 2).sum() / (W3 * ub * ub).sum())
        assert e <= eps * (1 + 1e-9)


def test_monotone_in_eps(oracle):
    # decreasing max_error never decreases the kept count
    u = oracle.gen_spectral(8, 64)
    kept_prev = None
    for eps in (0.5, 1e-1, 1e-2, 3e-3, 1e-3, 1e-4, 1e-5, 1e-6):
        co = oracle.forward_field(u, 8, 1)
        per_block = [oracle.select_block(8, co[b * 512:(b + 1) * 512], eps)[0] for b in range(64)]
        if kept_prev is not None:
            assert all(k >= p for k, p in zip(per_block, kept_prev))
        kept_prev = per_block


def test_tie_rule_index_order(oracle):
    # exact magnitude ties at the boundary: lower index kept first (stable order)
    a = np.zeros(512)
    a[0] = 1.0
    a[[5, 9, 300, 301]] = 0.01  # four equal magnitudes; budget allows dropping some
    a[7] = -0.01
    for eps in (0.012, 0.016, 0.019, 0.023):
        kept, mask, _ = oracle.select_block(8, a, eps)
        idx = [j for j in range(512) if (int(mask[j >> 6]) >> (j & 63)) & 1]
        assert idx[0] == 0
        ties = [j for j in (5, 7, 9, 300, 301) if j in idx]
        assert ties == sorted((5, 7, 9, 300, 301))[: len(ties)]  # prefix in index order


def test_eq1_compression_ratio_bitwise(oracle):
    # cr == (orig - comp)/orig in fp64 arithmetic
    u = oracle.gen_tgv(4, 8, 0)
    rc, s, st = oracle.compress(u, 8, 1, 1e-3)
    cr = (float(st.field_bytes) - float(st.stream_bytes)) / float(st.field_bytes)
    from paper_2407_20731_b200.lossy import CompressionReport
    assert CompressionReport.from_sizes(st.field_bytes, st.stream_bytes).cr == cr


def test_corrupt_stream_is_shape_mismatch(oracle):
    # an index >= P^3 / inconsistent block -> ShapeMismatch
    u = oracle.gen_tgv(4, 8, 0)
    rc, s, st = oracle.compress(u, 8, 1, 1e-3)
    bad = s.copy()
    bad[0] ^= 1  # count of block 0 no longer matches its mask
    rc, _, _ = oracle.decompress(bad, 8, 1, 64)
    assert rc == 13
    rc, _, _ = oracle.decompress(s[:-8], 8, 1, 64)
    assert rc == 13
    # a mask bit beyond P^3 (lx = 6: 216 bits in 4 words)
    v = oracle.gen_spectral(6, 4)
    rc, s6, _ = oracle.compress(v, 6, 1, 1e-3)
    _, masks, _ = oracle.parse_stream(s6, 6, 4)
    bad6 = s6.copy()
    mview = bad6[16:16 + 8 * 4 * 4].view(np.uint64)
    mview[3] |= np.uint64(1) << np.uint64(60)  # bit 252 >= 216
    rc, _, _ = oracle.decompress(bad6, 6, 1, 4)
    assert rc == 13


def test_nonfinite_rejected(oracle):
    u = np.zeros(512)
    u[17] = np.nan
    rc, _, st = oracle.compress(u, 8, 1, 1e-3)
    assert rc == 21 and st.status & 1


def test_vector_field_blocks(oracle):
    # components = 3: block b = element*3 + component, AoS within the element
    u = np.stack([oracle.gen_tgv(2, 8, w) for w in (0, 1, 3)], axis=-1).reshape(-1)
    rc, s, st = oracle.compress(u, 8, 3, 1e-3)
    assert rc == 0 and st.blocks == 8 * 3
    for c in range(3):
        rcc, sc, stc = oracle.compress(u.reshape(-1, 3)[:, c].copy(), 8, 1, 1e-3)
        cnt, _, _ = oracle.parse_stream(s, 8, 24)
        cntc, _, _ = oracle.parse_stream(sc, 8, 8)
        assert np.array_equal(cnt[c::3], cntc)
    rc, out, st2 = oracle.decompress(s, 8, 3, 8, original=u)
    assert math.sqrt(st2.err2 / st2.nrm2) <= 1e-3
