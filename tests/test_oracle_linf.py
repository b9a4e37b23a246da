"""RelativeLInf truncation: the C oracle's rule pinned
against an independent exact Python restatement (fractions), and its guarantee
max|u - u~| <= eps * max|u| per block checked by full reconstruction."""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest


def _bits(x):
    return struct.unpack("<Q", struct.pack("<d", x))[0] & 0x7FFFFFFFFFFFFFFF


def _mul_dir(x, y, up):
    q = Fraction(x) * Fraction(y)
    p = float(q)
    if up and Fraction(p) < q:
        p = math.nextafter(p, math.inf)
    if not up and Fraction(p) > q:
        p = math.nextafter(p, -math.inf)
    return p


def linf_rule_py(lx, B, a, umax, eps):
    n3 = lx ** 3
    bm = [max(abs(B[i][k]) for i in range(lx)) for k in range(lx)]
    x = []
    for j in range(n3):
        kx, ky, kz = j % lx, (j // lx) % lx, j // (lx * lx)
        x.append(_mul_dir(abs(a[j]), _mul_dir(_mul_dir(bm[kx], bm[ky], True), bm[kz], True), True))
    m = max(x)
    mask = np.zeros(n3, dtype=bool)
    if m == 0.0:
        return 0, mask
    s = math.frexp(m)[1]
    k = (63 - math.ceil(math.log2(n3))) - s
    w = [0 if xj == 0.0 else max(1, math.ceil(Fraction(xj) * Fraction(2) ** k)) for xj in x]
    thr = math.floor(Fraction(_mul_dir(eps, umax, False)) * Fraction(2) ** k)
    thr = min(thr, 1 << 63)
    order = sorted(range(n3), key=lambda j: (_bits(a[j]), -j))
    acc, m_ = 0, 0
    while m_ < n3 and acc + w[order[m_]] <= thr:
        acc += w[order[m_]]
        m_ += 1
    for p in order[m_:]:
        mask[p] = True
    return n3 - m_, mask


def _mask_bits(words, n3):
    return np.unpackbits(words.view(np.uint8), bitorder="little")[:n3].astype(bool)


@pytest.mark.parametrize("lx,eps", [(4, 1e-2), (6, 1e-3), (8, 1e-2), (8, 1e-4), (5, 1e-1)])
def test_linf_rule_matches_python_restatement(oracle, lx, eps):
    _, B = oracle.matrices(lx)
    u = oracle.gen_spectral(lx, 6)
    n3 = lx ** 3
    for b in range(6):
        ub = u[b * n3:(b + 1) * n3]
        a = oracle.fwd_block(lx, ub)
        umax = float(np.max(np.abs(ub)))
        kept, words, nf = oracle.select_block_linf(lx, a, umax, eps)
        assert not nf
        kp, mp = linf_rule_py(lx, B, list(a), umax, eps)
        assert kept == kp
        assert np.array_equal(_mask_bits(words, n3), mp)


@pytest.mark.parametrize("lx", [4, 6, 8, 9])
@pytest.mark.parametrize("eps", [1e-1, 1e-2, 1e-4])
@pytest.mark.parametrize("kind", ["tgv", "spectral"])
def test_linf_guarantee_by_reconstruction(oracle, lx, eps, kind):
    E = 3
    n_el = E ** 3
    u = oracle.gen_tgv(E, lx, 3) if kind == "tgv" else oracle.gen_spectral(lx, n_el)
    rc, stream, _ = oracle.compress(u, lx, 1, eps, norm=1)
    assert rc == 0
    rc, back, _ = oracle.decompress(stream, lx, 1, n_el)
    assert rc == 0
    n3 = lx ** 3
    for b in range(n_el):
        ub, vb = u[b * n3:(b + 1) * n3], back[b * n3:(b + 1) * n3]
        umax = np.max(np.abs(ub))
        # the rule bounds the exact reconstruction; allow the fp64 transform rounding
        assert np.max(np.abs(ub - vb)) <= eps * umax + 1e-13 * umax


def test_linf_monotone_and_kats(oracle):
    lx = 8
    u = oracle.gen_spectral(lx, 8)
    kept = []
    for eps in (1e-1, 1e-2, 1e-3, 1e-4):
        rc, stream, st = oracle.compress(u, lx, 1, eps, norm=1)
        counts, _, _ = oracle.parse_stream(stream, lx, 8)
        kept.append(counts.astype(np.int64))
    for a, b in zip(kept, kept[1:]):
        assert np.all(b >= a)
    zero = np.zeros(2 * lx ** 3)
    rc, stream, _ = oracle.compress(zero, lx, 1, 1e-2, norm=1)
    assert np.all(oracle.parse_stream(stream, lx, 2)[0] == 0)
    const = np.full(2 * lx ** 3, 3.25)
    rc, stream, _ = oracle.compress(const, lx, 1, 1e-2, norm=1)
    counts, masks, _ = oracle.parse_stream(stream, lx, 2)
    assert np.all(counts == 1) and np.all(masks[:, 0] == 1)
