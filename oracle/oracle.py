"""ctypes wrapper of the CPU ORACLE (oracle/isf_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` leg.  The product package never
imports this module.  See isf_oracle.h for what the oracle restates and its
parity-pinning status.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ISF_ORACLE_LIB: the -O3 -march=native build made on the benchmark host (bench.py)
_LIB_PATH = os.environ.get("ISF_ORACLE_LIB") or os.path.join(_HERE, "_build", "libisf_oracle.so")


class Stats(ctypes.Structure):
    _fields_ = [
        ("err2", ctypes.c_double), ("nrm2", ctypes.c_double),
        ("err_inf", ctypes.c_double), ("u_inf", ctypes.c_double),
        ("disc2", ctypes.c_double), ("tot2", ctypes.c_double),
        ("kept", ctypes.c_uint64), ("blocks", ctypes.c_uint64),
        ("stream_bytes", ctypes.c_uint64), ("field_bytes", ctypes.c_uint64),
        ("status", ctypes.c_uint64), ("reserved", ctypes.c_uint64),
    ]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def build(force: bool = False) -> str:
    if os.environ.get("ISF_ORACLE_LIB"):
        return _LIB_PATH
    if force or not os.path.exists(_LIB_PATH) or (
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "isf_oracle.c"))
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        u64, i32, f64 = ctypes.c_uint64, ctypes.c_int, ctypes.c_double
        L.iso_gll.argtypes = [i32, P, P]
        L.iso_matrices.argtypes = [i32, P, P]
        L.iso_fwd_block.argtypes = [i32, P, P, P]
        L.iso_inv_block.argtypes = [i32, P, P, P]
        L.iso_select_block.argtypes = [i32, P, f64, P, P, P, P, P]
        L.iso_select_block.restype = ctypes.c_uint32
        L.iso_select_block_perturbed.argtypes = [i32, P, f64, f64, P]
        L.iso_select_block_perturbed.restype = ctypes.c_uint32
        L.iso_stream_capacity.argtypes = [i32, u64]
        L.iso_stream_capacity.restype = u64
        L.iso_stream_header_bytes.argtypes = [i32, u64]
        L.iso_stream_header_bytes.restype = u64
        L.iso_compress.argtypes = [i32, i32, u64, P, f64, P, u64, P, P, i32]
        L.iso_compress_norm.argtypes = [i32, i32, u64, P, f64, i32, P, u64, P, P, i32]
        L.iso_select_block_literal.argtypes = [i32, P, f64, f64, P, P]
        L.iso_select_block_literal.restype = ctypes.c_uint32
        L.iso_literal_check.argtypes = [i32, i32, u64, P, f64, P, P, P, i32]
        L.iso_literal_check.restype = u64
        L.iso_select_block_linf.argtypes = [i32, P, P, f64, f64, P, P]
        L.iso_select_block_linf.restype = ctypes.c_uint32
        L.iso_decompress.argtypes = [i32, i32, u64, P, u64, P, P, P, i32]
        L.iso_forward_field.argtypes = [i32, i32, u64, P, P, i32]
        L.iso_gen_tgv.argtypes = [i32, i32, i32, ctypes.c_uint32, ctypes.c_uint32, f64, P, i32]
        L.iso_spectral_amplitudes.argtypes = [i32, f64, P]
        L.iso_gen_spectral.argtypes = [i32, u64, u64, u64, f64, P, i32]
        L.iso_philox4x32_10.argtypes = [P, P, P]
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def gll(lx: int):
    x = np.zeros(lx); w = np.zeros(lx)
    rc = lib().iso_gll(lx, _p(x), _p(w))
    if rc:
        raise ValueError(f"iso_gll rc={rc}")
    return x, w


def matrices(lx: int):
    F = np.zeros((lx, lx)); B = np.zeros((lx, lx))
    rc = lib().iso_matrices(lx, _p(F), _p(B))
    if rc:
        raise ValueError(f"iso_matrices rc={rc}")
    return F, B


def fwd_block(lx, u):
    F, _ = matrices(lx)
    u = np.ascontiguousarray(u, dtype=np.float64).reshape(-1)
    a = np.zeros_like(u)
    lib().iso_fwd_block(lx, _p(F), _p(u), _p(a))
    return a


def inv_block(lx, a):
    _, B = matrices(lx)
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    u = np.zeros_like(a)
    lib().iso_inv_block(lx, _p(B), _p(a), _p(u))
    return u


def select_block(lx, a, max_error):
    W = (lx ** 3 + 63) // 64
    mask = np.zeros(W, dtype=np.uint64)
    lt = ctypes.c_uint64(); ld = ctypes.c_uint64(); se = (ctypes.c_int * 2)(); nf = ctypes.c_int()
    a = np.ascontiguousarray(a, dtype=np.float64)
    kept = lib().iso_select_block(lx, _p(a), float(max_error), _p(mask), ctypes.byref(lt),
                                  ctypes.byref(ld), se, ctypes.byref(nf))
    return int(kept), mask, {"lo_total": lt.value, "lo_disc": ld.value, "scale_exp": se[0],
                             "disc_exp": se[1], "nonfinite": nf.value}


def select_block_perturbed(lx, a, max_error, rel):
    W = (lx ** 3 + 63) // 64
    mask = np.zeros(W, dtype=np.uint64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    kept = lib().iso_select_block_perturbed(lx, _p(a), float(max_error), float(rel), _p(mask))
    return int(kept), mask


def select_block_literal(lx, a, max_error, rel=0.0):
    """SPEC-literal rule (SPEC.md:225 in exact reals), binary128-filtered in C with
    an exact rational fallback: (kept, mask words)."""
    W = (lx ** 3 + 63) // 64
    mask = np.zeros(W, dtype=np.uint64)
    a = np.ascontiguousarray(a, dtype=np.float64)
    amb = ctypes.c_int()
    kept = lib().iso_select_block_literal(lx, _p(a), float(max_error), float(rel), _p(mask), ctypes.byref(amb))
    if amb.value:
        return select_block_literal_exact(lx, a, max_error, rel)
    return int(kept), mask


def select_block_literal_exact(lx, a, max_error, rel=0.0):
    """The same rule in exact rational arithmetic (fractions.Fraction): sort by
    (|a| descending, index ascending) and keep the smallest prefix whose discarded
    energy is <= eps^2 * total * (1 + rel)."""
    from fractions import Fraction
    n3 = lx ** 3
    a = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    e = [Fraction(float(x)) ** 2 for x in a]
    T = sum(e, Fraction(0))
    mask = np.zeros((n3 + 63) // 64, dtype=np.uint64)
    if T == 0:
        return 0, mask
    thr = Fraction(float(max_error)) ** 2 * T * (1 + Fraction(float(rel)))
    keys = np.abs(a).view(np.uint64)
    order = sorted(range(n3), key=lambda j: (int(keys[j]), -j))  # discard order
    acc, m = Fraction(0), 0
    while m < n3 and acc + e[order[m]] <= thr:
        acc += e[order[m]]
        m += 1
    for j in order[m:]:
        mask[j >> 6] |= np.uint64(1) << np.uint64(j & 63)
    return n3 - m, mask


def literal_check(field, lx, comps, max_error, stream, nthreads: int = 0):
    """Compare a stream's masks with the SPEC-literal rule block by block.

    Returns a dict: blocks, differ (blocks whose mask differs from the literal
    rule), near_threshold (those accepted by SURVEY.md 8c's rule: the literal rule
    with eps^2*T scaled by 1 -+ 4*2^-52*lx^3 reproduces the stream's kept count),
    far (differ beyond that), ambiguous_resolved (blocks binary128 could not decide,
    settled exactly), kept_literal, kept_stream, far_blocks (first 16 indices)."""
    field = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
    stream = np.ascontiguousarray(stream, dtype=np.uint8)
    n_el = field.size // (lx ** 3 * comps)
    B = n_el * comps
    cls = np.zeros(B, dtype=np.uint8)
    kl = ctypes.c_uint64()
    lib().iso_literal_check(lx, comps, n_el, _p(field), float(max_error), _p(stream), _p(cls), ctypes.byref(kl),
                            nthreads)
    counts, masks, _ = parse_stream(stream, lx, B)
    kept_lit = int(kl.value)
    amb = np.nonzero(cls == 3)[0]
    rel = 4 * 2.0 ** -52 * lx ** 3
    n3 = lx ** 3
    for b in amb:
        e, c = divmod(int(b), comps)
        blk = field[e * n3 * comps + c: (e + 1) * n3 * comps: comps]
        a = fwd_block(lx, blk)
        k, m = select_block_literal_exact(lx, a, max_error)
        kept_lit += 0  # the C pass already counted its (binary128) kept value for b
        if k == counts[b] and np.array_equal(m, masks[b]):
            cls[b] = 0
        elif any(select_block_literal_exact(lx, a, max_error, s * rel)[0] == counts[b] for s in (-1, 1)):
            cls[b] = 1
        else:
            cls[b] = 2
    far = np.nonzero(cls == 2)[0]
    return {"blocks": int(B), "differ": int(np.count_nonzero(cls)), "near_threshold": int(np.count_nonzero(cls == 1)),
            "far": int(far.size), "ambiguous_resolved": int(amb.size), "kept_literal": kept_lit,
            "kept_stream": int(counts.astype(np.int64).sum()), "far_blocks": [int(x) for x in far[:16]]}


def stream_capacity(lx, nblocks):
    return int(lib().iso_stream_capacity(lx, nblocks))


def stream_header_bytes(lx, nblocks):
    return int(lib().iso_stream_header_bytes(lx, nblocks))


def compress(field: np.ndarray, lx: int, comps: int, max_error: float, nthreads: int = 0, norm: int = 0):
    """Returns (rc, stream bytes as np.uint8 array, Stats).  norm: 0 RelativeL2, 1 RelativeLInf."""
    field = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
    n_el = field.size // (lx ** 3 * comps)
    cap = stream_capacity(lx, n_el * comps)
    buf = np.zeros(cap, dtype=np.uint8)
    nb = ctypes.c_uint64()
    st = Stats()
    rc = lib().iso_compress_norm(lx, comps, n_el, _p(field), float(max_error), int(norm), _p(buf), cap,
                                 ctypes.byref(nb), ctypes.byref(st), nthreads)
    return rc, buf[: nb.value].copy(), st


def select_block_linf(lx: int, a: np.ndarray, umax: float, max_error: float):
    """RelativeLInf rule on one block of coefficients: (kept, mask words)."""
    _, B = matrices(lx)[:2]
    B = np.ascontiguousarray(B, dtype=np.float64).reshape(-1)
    a = np.ascontiguousarray(a, dtype=np.float64)
    mask = np.zeros((lx ** 3 + 63) // 64, dtype=np.uint64)
    nf = ctypes.c_int()
    kept = lib().iso_select_block_linf(lx, _p(B), _p(a), float(umax), float(max_error), _p(mask), ctypes.byref(nf))
    return int(kept), mask, bool(nf.value)


def decompress(stream: np.ndarray, lx: int, comps: int, n_elements: int, original=None,
               nthreads: int = 0):
    out = np.zeros(n_elements * lx ** 3 * comps)
    st = Stats()
    stream = np.ascontiguousarray(stream, dtype=np.uint8)
    orig = None
    if original is not None:
        orig = np.ascontiguousarray(original, dtype=np.float64).reshape(-1)
    rc = lib().iso_decompress(lx, comps, n_elements, _p(stream), stream.size, _p(out),
                              _p(orig) if orig is not None else None, ctypes.byref(st), nthreads)
    return rc, out, st


def forward_field(field, lx, comps, nthreads: int = 0):
    field = np.ascontiguousarray(field, dtype=np.float64).reshape(-1)
    n_el = field.size // (lx ** 3 * comps)
    co = np.zeros(field.size)
    lib().iso_forward_field(lx, comps, n_el, _p(field), _p(co), nthreads)
    return co


def gen_tgv(E_ax: int, lx: int, which: int, ez0: int = 0, nz: int | None = None,
            domain: float = 2.0 * np.pi, nthreads: int = 0):
    nz = E_ax if nz is None else nz
    out = np.zeros(E_ax * E_ax * nz * lx ** 3)
    lib().iso_gen_tgv(E_ax, lx, which, ez0, nz, float(domain), _p(out), nthreads)
    return out


SPECTRAL_SEED = 0x240720731


def spectral_amplitudes(lx, decay_s=0.5):
    amp = np.zeros(lx ** 3)
    lib().iso_spectral_amplitudes(lx, float(decay_s), _p(amp))
    return amp


def gen_spectral(lx: int, nblocks: int, block0: int = 0, seed: int = SPECTRAL_SEED,
                 decay_s: float = 0.5, nthreads: int = 0):
    out = np.zeros(nblocks * lx ** 3)
    lib().iso_gen_spectral(lx, block0, nblocks, seed, float(decay_s), _p(out), nthreads)
    return out


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32); k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().iso_philox4x32_10(_p(c), _p(k), _p(o))
    return o


# ---- stream helpers (pure numpy; same format as DESIGN.md 3.5) ----
def parse_stream(stream: np.ndarray, lx: int, nblocks: int):
    W = (lx ** 3 + 63) // 64
    c_end = 4 * nblocks
    m0 = (c_end + 15) & ~15
    counts = stream[:c_end].view(np.uint32)
    masks = stream[m0:m0 + 8 * W * nblocks].view(np.uint64).reshape(nblocks, W)
    vals = stream[m0 + 8 * W * nblocks:].view(np.float64)
    return counts, masks, vals
