"""Which norm max_error bounds.

The truncation is exact in the GLL-quadrature norm ||v||_w^2 = sum w_x w_y w_z v^2
(Parseval for the orthonormal DLT), so per block rel_w(err) <= max_error.  The plain
point-sample norm is equivalent up to the weight ratio: min_w ||v||^2 <= ||v||_w^2 <=
max_w ||v||^2 gives rel_plain <= sqrt(max_w / min_w) * rel_w.  These tests pin both
facts on the oracle (CPU) for the SPEC acceptance field (TGV) and a spectral field, and
record that the plain norm can exceed max_error (so the docs must say which norm)."""
import numpy as np
import pytest

from oracle import oracle as O


def _norms(u, rec, lx):
    _, w = O.gll(lx)
    w3 = np.einsum("i,j,k->kji", w, w, w).reshape(-1)  # index x + lx (y + lx z)
    u = u.reshape(-1, lx ** 3)
    e = (u - rec.reshape(-1, lx ** 3))
    rel_w = np.sqrt((w3 * e * e).sum(1) / np.maximum((w3 * u * u).sum(1), 1e-300))
    rel_p = np.sqrt((e * e).sum(1) / np.maximum((u * u).sum(1), 1e-300))
    return rel_w, rel_p, np.sqrt(w3.max() / w3.min())


@pytest.mark.parametrize("lx,eps", [(8, 1e-2), (8, 1e-3), (6, 1e-2), (12, 1e-3)])
def test_weighted_bound_and_plain_equivalence(lx, eps):
    fields = [O.gen_spectral(lx, 64)]
    if lx == 8:
        fields.append(O.gen_tgv(4, lx, 0))
    for u in fields:
        n_el = u.size // lx ** 3
        rc, s, _ = O.compress(u, lx, 1, eps)
        assert rc == 0
        rc, rec, _ = O.decompress(s, lx, 1, n_el)
        assert rc == 0
        rel_w, rel_p, kappa = _norms(u, rec, lx)
        assert (rel_w <= eps * (1 + 1e-9)).all()            # the guarantee (per block)
        assert (rel_p <= kappa * rel_w * (1 + 1e-9) + 1e-300).all()  # norm equivalence


def test_plain_norm_can_exceed_max_error():
    # SPEC acceptance field (TGV E=8, P=8, 1e-2): weighted <= 1e-2 by construction, the
    # plain relative L2 of the whole field is above it -- the reason the headers say
    # "GLL-quadrature norm"
    u = O.gen_tgv(8, 8, 3)
    rc, s, _ = O.compress(u, 8, 1, 1e-2)
    rc, rec, _ = O.decompress(s, 8, 1, 512)
    _, w = O.gll(8)
    w3 = np.tile(np.einsum("i,j,k->kji", w, w, w).reshape(-1), 512)
    e = u - rec
    glob_w = np.sqrt((w3 * e * e).sum() / (w3 * u * u).sum())
    glob_p = np.sqrt((e * e).sum() / (u * u).sum())
    assert glob_w <= 1e-2
    assert glob_p > 1e-2
