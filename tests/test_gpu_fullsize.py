"""Full-size parity at BASELINE.json's configurations (GPU vs CPU oracle, whole fields).

cfg2 (configs[1]): the four TGV fields u, v, w, p of a 64^3-element lx = 8 mesh,
1 GiB each, RelativeL2 1e-3 and 1e-2.  cfg4 (configs[3]): 262,144 elements of the
turbulent-like spectral field at lx = 6, 8, 10, 12 and eps 1e-2 .. 1e-5.

For every case: the device stream is byte-identical to the oracle's stream of the
same input (every count, mask word and value record), the device reconstruction is
bit-identical to the oracle's, and the stream is checked against the SPEC-literal
rule (SPEC.md:225 in exact reals, oracle.literal_check): blocks that differ are
counted, and each must lie in SURVEY.md 8c's near-threshold band (far == 0).
The counts are printed (north_star: "counted and reported")."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _check_full(PK, oracle, vals, E, P, eps, n_el=None, decode=True):
    n = n_el if n_el is not None else E ** 3
    f = PK.Field(E, P, 1, vals, n_elements=n_el)
    blk = PK.lossy_compress(f, PK.LossyConfig(eps))
    got = blk.stream.cpu().numpy()
    host = vals.cpu().numpy()
    rc, ref, st = oracle.compress(host, P, 1, eps)
    assert rc == 0
    assert got.size == ref.size, (got.size, ref.size)
    if not np.array_equal(got, ref):
        d = np.nonzero(got != ref)[0]
        raise AssertionError(f"stream differs at {d.size} bytes, first {d[:8]}")
    lit = oracle.literal_check(host, P, 1, eps, ref)
    assert lit["far"] == 0, lit
    rep = None
    if decode:
        back, rep = PK.decompress_with_error(blk, f.shape, f)
        rc, ob, ost = oracle.decompress(ref, P, 1, n, original=host)
        assert rc == 0
        assert np.array_equal(back.values.cpu().numpy().view(np.uint64), ob.view(np.uint64))
        assert rep.rel_l2 <= eps * (1 + 1e-9)
        if ost.nrm2 > 0:
            assert abs(rep.err2 - ost.err2) <= 1e-9 * ost.err2 + 1e-300
            assert rep.err_inf == ost.err_inf and rep.u_inf == ost.u_inf
    print(f"\n[parity] lx={P} eps={eps:g} blocks={lit['blocks']} kept={lit['kept_stream']} "
          f"literal_kept={lit['kept_literal']} near_threshold={lit['near_threshold']} far={lit['far']}")
    return lit, rep


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_cfg2_full_field_parity(native, oracle, which):
    import paper_2407_20731_b200 as PK
    E, P = 64, 8
    plan = PK.get_plan(P, 1, 0)
    vals = torch.empty(E ** 3 * 512, dtype=torch.float64, device="cuda")
    plan.generate_tgv(vals, E, which)
    for eps in (1e-3, 1e-2):
        lit, rep = _check_full(PK, oracle, vals, E, P, eps, decode=(eps == 1e-3))
        if which == 2:
            assert lit["kept_stream"] == 0
    del vals
    torch.cuda.empty_cache()


@pytest.mark.parametrize("P", [6, 8, 10, 12])
def test_cfg4_full_field_parity(native, oracle, P):
    import paper_2407_20731_b200 as PK
    n = 262144
    plan = PK.get_plan(P, 1, 0)
    vals = torch.empty(n * P ** 3, dtype=torch.float64, device="cuda")
    plan.generate_spectral(vals, n, 0, oracle.SPECTRAL_SEED, oracle.spectral_amplitudes(P))
    for eps in (1e-2, 1e-3, 1e-4, 1e-5):
        _check_full(PK, oracle, vals, 64, P, eps, decode=(eps in (1e-2, 1e-5)))
    del vals
    torch.cuda.empty_cache()
