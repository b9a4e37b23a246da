"""The SPEC-literal truncation rule and the pinned integer rule v2 (CPU only).

SPEC.md:225 read in exact reals: sort by |a| descending (index ascending), keep the
smallest prefix whose discarded energy is <= max_error^2 times the block energy.
`oracle.select_block_literal` evaluates it in binary128 with a rigorous error
filter and falls back to `fractions.Fraction` when the filter cannot decide;
`oracle.select_block_literal_exact` is the all-rational restatement.  The pinned
rule v2 (exact integers at a block-total scale and a threshold-
relative scale) is what the GPU and the C oracle compute; these tests count where
it departs from the literal rule and check that every such block lies in SURVEY.md
8c's near-threshold band (the literal rule with eps^2*T scaled by 1 -+ 4*2^-52*lx^3
reproduces it)."""
from fractions import Fraction

import numpy as np
import pytest


def _rand_blocks(rng, lx, n):
    out = []
    for _ in range(n):
        a = rng.standard_normal(lx ** 3) * 10.0 ** rng.uniform(-3, 0, lx ** 3)
        a[rng.random(lx ** 3) < 0.1] = 0.0
        out.append(a)
    return out


@pytest.mark.parametrize("lx", [2, 3, 4])
def test_literal_filter_matches_exact(oracle, lx):
    rng = np.random.default_rng(7 + lx)
    for a in _rand_blocks(rng, lx, 40):
        for eps in (0.5, 1e-1, 1e-2, 1e-3):
            k1, m1 = oracle.select_block_literal(lx, a, eps)
            k2, m2 = oracle.select_block_literal_exact(lx, a, eps)
            assert k1 == k2 and np.array_equal(m1, m2)


def test_literal_exact_tie_goes_through_the_rational_path(oracle):
    # four equal coefficients, eps = 1/2: discarding one leaves exactly eps^2 * T
    # (1 == 1/4 * 4), so the literal rule keeps 3 -- the binary128 filter cannot
    # decide a zero margin and the rational fallback must
    a = np.zeros(8)
    a[[0, 3, 5, 6]] = 1.0
    import ctypes
    mask = np.zeros(1, dtype=np.uint64)
    amb = ctypes.c_int()
    oracle.lib().iso_select_block_literal(2, oracle._p(a), 0.5, 0.0, oracle._p(mask), ctypes.byref(amb))
    assert amb.value == 1
    k, m = oracle.select_block_literal(2, a, 0.5)
    assert k == 3
    assert int(m[0]) == (1 << 0) | (1 << 3) | (1 << 5)  # the largest index is discarded first
    # the integer rule keeps all four (its hi bounds are strict), which the
    # near-threshold band accepts: at eps^2 T (1 - 4 2^-52 8) the literal rule keeps 4
    kv2, _, _ = oracle.select_block(2, a, 0.5)
    assert kv2 == 4
    assert oracle.select_block_literal(2, a, 0.5, -4 * 2.0 ** -52 * 8)[0] == 4


@pytest.mark.parametrize("lx", [2, 3, 5, 8])
def test_v2_is_conservative_and_in_band(oracle, lx):
    """Per block: kept_v2 >= kept_literal, the discarded exact energy is <= eps^2 * T,
    and a differing block is accepted by the near-threshold band."""
    rng = np.random.default_rng(100 + lx)
    rel = 4 * 2.0 ** -52 * lx ** 3
    for a in _rand_blocks(rng, lx, 12 if lx == 8 else 40):
        for eps in (0.3, 1e-2, 1e-4, 1e-6):
            kv, mv, _ = oracle.select_block(lx, a, eps)
            kl, ml = oracle.select_block_literal(lx, a, eps)
            assert kv >= kl
            bits = np.unpackbits(mv.view(np.uint8), bitorder="little")[: lx ** 3].astype(bool)
            disc = sum((Fraction(float(x)) ** 2 for x in a[~bits]), Fraction(0))
            tot = sum((Fraction(float(x)) ** 2 for x in a), Fraction(0))
            assert disc <= Fraction(eps) ** 2 * tot
            if kv != kl:
                assert oracle.select_block_literal(lx, a, eps, -rel)[0] == kv


@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4, 1e-5])
def test_v2_vs_literal_tgv(oracle, eps):
    for which in (0, 1, 3):
        u = oracle.gen_tgv(8, 8, which)
        rc, s, _ = oracle.compress(u, 8, 1, eps)
        assert rc == 0
        r = oracle.literal_check(u, 8, 1, eps, s)
        assert r["far"] == 0, r
        assert r["kept_stream"] - r["kept_literal"] <= r["near_threshold"] * 8


@pytest.mark.parametrize("lx", [6, 8, 10, 12])
def test_v2_vs_literal_spectral(oracle, lx):
    u = oracle.gen_spectral(lx, 512)
    for eps in (1e-2, 1e-3, 1e-4, 1e-5):
        rc, s, _ = oracle.compress(u, lx, 1, eps)
        assert rc == 0
        r = oracle.literal_check(u, lx, 1, eps, s)
        assert r["far"] == 0, (eps, r)


def test_literal_check_flags_a_wrong_stream(oracle):
    """literal_check is a real checker: a stream with one extra kept coefficient far
    from the threshold is reported as a far difference."""
    u = oracle.gen_tgv(4, 8, 0)
    rc, s, _ = oracle.compress(u, 8, 1, 1e-2)
    B = 64
    counts, masks, _ = oracle.parse_stream(s, 8, B)
    s2 = s.copy()
    c2, m2, _ = oracle.parse_stream(s2, 8, B)
    # drop one kept coefficient of block 5 from the mask and the count (values are not
    # inspected by the checker)
    w = int(np.nonzero(m2[5])[0][0])
    bit = int(m2[5][w]) & -int(m2[5][w])
    m2[5][w] = np.uint64(int(m2[5][w]) ^ bit)
    c2[5] -= 1
    r = oracle.literal_check(u, 8, 1, 1e-2, s2)
    assert r["far"] == 1 and r["far_blocks"] == [5]
