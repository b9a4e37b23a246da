#!/usr/bin/env python
"""Generate the golden fixtures of the lossy-compression hot path.

An INDEPENDENT restatement (pure Python, no oracle code) of the pinned
definitions in DESIGN.md 3 (SPEC.md:222-239 + north_star's Legendre DLT):

  * GLL nodes / weights and the Legendre matrices F, B in 40-digit `decimal`
    arithmetic (Newton on P'_N, mirrored), rounded once to binary64;
  * the three sweeps in the pinned order (forward z, y, x; even/odd split;
    first product then ascending fused multiply-adds), every fma evaluated
    exactly with `fractions.Fraction` and rounded once (float(Fraction) is
    correctly rounded), so the coefficients are bit-exact by construction;
  * the truncation rule (v2: exact integer energies at a block-total scale and
    a threshold-relative scale) with Python integers / fractions and an explicit
    stable sort (|a| descending, index ascending: "sort coefficients
    by magnitude descending ... smallest prefix");
  * the little-endian stream layout of include/isf_lossy.h.

The reference (/root/reference) has no implementation and no test vectors for
this path, so these fixtures pin the C oracle (tests/test_golden.py) and through
it the GPU kernels (tests/test_gpu_parity.py).  Run from the repo root:
    python tests/golden/make_golden.py
"""
from __future__ import annotations

import math
import os
import struct
from decimal import Decimal, getcontext
from fractions import Fraction

import numpy as np

getcontext().prec = 40
HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------- GLL operators
def _legendre(N, x):
    P = [Decimal(1), x]
    for k in range(2, N + 1):
        P.append(((2 * k - 1) * x * P[k - 1] - (k - 1) * P[k - 2]) / k)
    return P[: N + 1]


def gll_decimal(lx):
    N = lx - 1
    pi = Decimal("3.141592653589793238462643383279502884197")
    xs = []
    for i in range(N + 1):
        # cos via Taylor in Decimal
        a = pi * i / N
        c, term, n = Decimal(0), Decimal(1), 0
        while True:
            c += term
            n += 2
            term = -term * a * a / (n * (n - 1))
            if abs(term) < Decimal("1e-45"):
                break
        x = -c
        for _ in range(200):
            P = _legendre(N, x)
            dx = (x * P[N] - P[N - 1]) / ((N + 1) * P[N])
            x -= dx
            if abs(dx) < Decimal("1e-38"):
                break
        xs.append(x)
    xs[0], xs[N] = Decimal(-1), Decimal(1)
    for i in range(lx // 2):
        xs[N - i] = -xs[i]
    if lx % 2:
        xs[lx // 2] = Decimal(0)
    ws = []
    for i in range(N + 1):
        P = _legendre(N, xs[i])
        ws.append(Decimal(2) / (N * (N + 1) * P[N] * P[N]))
    for i in range(lx // 2):
        ws[N - i] = ws[i]
    return xs, ws


def matrices(lx):
    N = lx - 1
    xs, ws = gll_decimal(lx)
    F = [[0.0] * lx for _ in range(lx)]
    B = [[0.0] * lx for _ in range(lx)]
    for i in range((lx + 1) // 2):
        P = _legendre(N, xs[i])
        for k in range(lx):
            g = Decimal(2) / (2 * k + 1) if k < N else Decimal(2) / N
            rs = 1 / g.sqrt()
            f = float(ws[i] * P[k] * rs)
            b = float(P[k] * rs)
            if lx % 2 and i == lx // 2 and k % 2:
                f = b = 0.0
            F[k][i] = f
            B[i][k] = b
            if i != N - i:
                F[k][N - i] = -f if k % 2 else f
                B[N - i][k] = -b if k % 2 else b
    return F, B, [float(x) for x in xs], [float(w) for w in ws]


# ------------------------------------------------------------ pinned transforms
def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def _mul(a, b):
    return float(Fraction(a) * Fraction(b))


def fwd_line(F, u):
    n = len(u)
    h = n // 2
    s = [u[i] + u[n - 1 - i] for i in range(h)]
    d = [u[i] - u[n - 1 - i] for i in range(h)]
    out = []
    for k in range(n):
        v = d if k & 1 else s
        acc = _mul(F[k][0], v[0])
        for i in range(1, h):
            acc = _fma(F[k][i], v[i], acc)
        if n & 1 and not k & 1:
            acc = _fma(F[k][h], u[h], acc)
        out.append(acc)
    return out


def inv_line(B, a):
    n = len(a)
    h = n // 2
    out = [0.0] * n
    for i in range(h):
        E = _mul(B[i][0], a[0])
        for k in range(2, n, 2):
            E = _fma(B[i][k], a[k], E)
        O = _mul(B[i][1], a[1])
        for k in range(3, n, 2):
            O = _fma(B[i][k], a[k], O)
        out[i] = E + O
        out[n - 1 - i] = E - O
    if n & 1:
        E = _mul(B[h][0], a[0])
        for k in range(2, n, 2):
            E = _fma(B[h][k], a[k], E)
        out[h] = E
    return out


def fwd_block(F, u, n):
    a = np.array(u, dtype=float).reshape(n, n, n)  # [z][y][x]
    for y in range(n):
        for x in range(n):
            a[:, y, x] = fwd_line(F, list(a[:, y, x]))
    for z in range(n):
        for x in range(n):
            a[z, :, x] = fwd_line(F, list(a[z, :, x]))
    for z in range(n):
        for y in range(n):
            a[z, y, :] = fwd_line(F, list(a[z, y, :]))
    return a.reshape(-1)


# ------------------------------------------------------------ truncation rule
def _rd(q: Fraction) -> float:
    """Largest binary64 <= q (q >= 0, finite)."""
    f = float(q)  # correctly rounded to nearest
    if Fraction(f) > q:
        f = math.nextafter(f, 0.0)
    return f


def select(a, n3, eps):
    """Rule v2 of DESIGN.md 3.4 (two integer scales) with Python integers."""
    EM = min(52, 63 - math.ceil(math.log2(n3)))
    hm = EM // 2
    bits = [struct.unpack("<Q", struct.pack("<d", float(abs(x))))[0] for x in a]
    if max(bits) == 0:
        return [False] * n3
    _, s = math.frexp(max(abs(x) for x in a))
    k = hm - s
    e = [_rd(Fraction(math.ldexp(abs(x), k)) ** 2) for x in a]   # RD(x^2), x exact
    h = (EM - 2 * hm) + (1 if max(e) < 2.0 ** (2 * hm - 1) else 0)
    T = sum(int(Fraction(v) * 2 ** h) for v in e)                  # floor: values >= 0
    E2 = _rd(Fraction(eps) ** 2)
    m, ex = math.frexp(E2)
    M, Ee = int(math.ldexp(m, 53)), ex - 53
    P = T * M
    if P == 0:
        thr, G = 0, 0
    else:
        G = min(52 - P.bit_length() - Ee, 1023 - h)
        sh = G + Ee
        thr = P << sh if sh >= 0 else P >> (-sh)
    def hi(v):
        y = Fraction(v) * Fraction(2) ** (h + G)
        return 2 ** 52 if y >= 2 ** 52 else int(y) + 1
    order = sorted(range(n3), key=lambda j: (-bits[j], j))   # |a| desc, index asc (stable)
    disc = order[::-1]                                       # discard order
    acc, mm = 0, 0
    while mm < n3 and acc + hi(e[disc[mm]]) <= thr:
        acc += hi(e[disc[mm]])
        mm += 1
    kept = [True] * n3
    for j in disc[:mm]:
        kept[j] = False
    return kept


def encode(coeffs, n3, eps):
    B = len(coeffs) // n3
    W = (n3 + 63) // 64
    counts, masks, vals = [], [], []
    for b in range(B):
        a = coeffs[b * n3:(b + 1) * n3]
        kept = select(a, n3, eps)
        counts.append(sum(kept))
        words = [0] * W
        for j in range(n3):
            if kept[j]:
                words[j >> 6] |= 1 << (j & 63)
                vals.append(a[j])
        masks.extend(words)
    head = struct.pack(f"<{B}I", *counts)
    head += b"\0" * (((4 * B + 15) & ~15) - 4 * B)
    return head + struct.pack(f"<{len(masks)}Q", *masks) + struct.pack(f"<{len(vals)}d", *vals)


# ------------------------------------------------------------ inputs
def tgv_block(lx, E, ex, ey, ez, which, xs):
    h = 2 * math.pi / E
    X = [ex * h + (x + 1.0) * 0.5 * h for x in xs]
    Y = [ey * h + (x + 1.0) * 0.5 * h for x in xs]
    Z = [ez * h + (x + 1.0) * 0.5 * h for x in xs]
    out = []
    for pz in range(lx):
        for py in range(lx):
            for px in range(lx):
                x, y, z = X[px], Y[py], Z[pz]
                if which == 0:
                    out.append(math.cos(x) * math.sin(y) * math.sin(z))
                else:
                    out.append((math.cos(2.0 * x) + math.cos(2.0 * y)) * (math.cos(2.0 * z) + 2.0) / 16.0)
    return out


def main():
    out = {}
    for lx in range(2, 17):
        F, Bm, xs, ws = matrices(lx)
        out[f"F{lx}"] = np.array(F)
        out[f"B{lx}"] = np.array(Bm)
        out[f"x{lx}"] = np.array(xs)
        out[f"w{lx}"] = np.array(ws)
    cases = []
    # (name, lx, field values, eps)
    rng = np.random.default_rng(20240731)
    F8, B8, xs8, _ = matrices(8)
    tgv = []
    for e in range(2):
        tgv += tgv_block(8, 4, e, 1, 2, 0, xs8)
    cases.append(("tgv_u_lx8", 8, tgv, 1e-3))
    p = tgv_block(8, 4, 1, 2, 3, 3, xs8)
    cases.append(("tgv_p_lx8", 8, p, 1e-2))
    cases.append(("const_lx8", 8, [3.25] * 512, 1e-3))
    cases.append(("zero_lx8", 8, [0.0] * 512, 1e-3))
    for lx in (3, 5, 6):
        Fl, Bl, _, _ = matrices(lx)
        # smooth random block: inverse transform of decaying random coefficients
        vals = []
        for _b in range(2):
            co = [float(rng.uniform(-1, 1)) * 10.0 ** (-0.5 * math.sqrt(i * i + j * j + k * k))
                  for k in range(lx) for j in range(lx) for i in range(lx)]
            a = np.array(co).reshape(lx, lx, lx)
            for z in range(lx):
                for y in range(lx):
                    a[z, y, :] = inv_line(Bl, list(a[z, y, :]))
            for z in range(lx):
                for x in range(lx):
                    a[z, :, x] = inv_line(Bl, list(a[z, :, x]))
            for y in range(lx):
                for x in range(lx):
                    a[:, y, x] = inv_line(Bl, list(a[:, y, x]))
            vals += list(a.reshape(-1))
        cases.append((f"smooth_lx{lx}", lx, vals, 1e-4))
    names = []
    for name, lx, vals, eps in cases:
        Fm = matrices(lx)[0]
        n3 = lx ** 3
        co = []
        for b in range(len(vals) // n3):
            co += list(fwd_block(Fm, vals[b * n3:(b + 1) * n3], lx))
        stream = encode(co, n3, eps)
        out[f"{name}__field"] = np.array(vals)
        out[f"{name}__coeffs"] = np.array(co)
        out[f"{name}__stream"] = np.frombuffer(stream, dtype=np.uint8)
        out[f"{name}__meta"] = np.array([lx, eps])
        names.append(name)
    out["cases"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "golden_v2.npz"), **out)
    print("wrote", os.path.join(HERE, "golden_v2.npz"), names)


if __name__ == "__main__":
    main()
