"""GPU parity: the sm_100a path (through the C ABI) against the CPU oracle.

Bar (north_star): coefficients / reconstructions within 1e-12 relative, masks
and streams identical except near-threshold blocks (counted; expected 0 because
the selection rule is exact integer arithmetic).
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL_TOL = 1e-12


def _field(P, comps, n_el, values):
    import paper_2407_20731_b200 as PK
    E = round(n_el ** (1 / 3))
    return PK.Field(E, P, comps, torch.from_numpy(values).cuda(),
                    n_elements=None if E ** 3 == n_el else n_el)


def _compress_both(native, oracle, values, P, comps, eps):
    n_el = values.size // (P ** 3 * comps)
    f = _field(P, comps, n_el, values)
    blk = native.lossy_compress(f, native.LossyConfig(eps))
    rc, ref, st = oracle.compress(values, P, comps, eps)
    assert rc == 0
    return f, blk, ref, st


def _assert_stream_parity(oracle, blk, ref, P, comps, eps, coeffs=None):
    got = blk.stream.cpu().numpy()
    B = blk.nblocks
    if got.size == ref.size and np.array_equal(got, ref):
        return 0
    # near-threshold acceptance rule: a differing block is accepted only if the
    # oracle with eps^2*T perturbed by +-4*2^-52*P^3 reproduces the GPU kept count.
    gc, gm, gv = oracle.parse_stream(got, P, B)
    rc_, rm, rv = oracle.parse_stream(ref, P, B)
    bad = np.nonzero((gc != rc_) | np.any(gm != rm, axis=1))[0]
    # every block with the oracle's count and mask carries bit-identical values
    go = np.concatenate([[0], np.cumsum(gc.astype(np.int64))])
    ro = np.concatenate([[0], np.cumsum(rc_.astype(np.int64))])
    ok_blk = np.ones(B, bool)
    ok_blk[bad] = False
    for b in np.nonzero(ok_blk)[0]:
        if gc[b]:
            assert np.array_equal(np.asarray(gv[go[b]:go[b + 1]]).view(np.uint64),
                                  np.asarray(rv[ro[b]:ro[b + 1]]).view(np.uint64)), f"block {b}: values differ"
    if bad.size == 0:
        assert got.size == ref.size and np.array_equal(got, ref), "stream bytes differ outside the value records"
    assert coeffs is not None, f"{bad.size} blocks differ"
    rel = 4 * 2.0 ** -52 * P ** 3
    for b in bad:
        a = coeffs[b * P ** 3:(b + 1) * P ** 3]
        ok = any(oracle.select_block_perturbed(P, a, eps, s * rel)[0] == gc[b] for s in (-1, 1))
        assert ok, f"block {b}: gpu kept {gc[b]} oracle {rc_[b]} (not a near-threshold case)"
    return bad.size


def test_operators_bitwise(native, oracle):
    for P in range(2, 17):
        plan = native.get_plan(P, 1, 0)
        F, B, x, w = plan.operators()
        Fo, Bo = oracle.matrices(P)
        xo, wo = oracle.gll(P)
        assert np.array_equal(F, Fo) and np.array_equal(B, Bo), P
        assert np.array_equal(x, xo) and np.array_equal(w, wo), P


@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-5])
def test_tgv_cfg1_stream_bitexact(native, oracle, eps):
    u = oracle.gen_tgv(16, 8, 0)
    f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, eps)
    assert blk.kept_total == st.kept
    assert _assert_stream_parity(oracle, blk, ref, 8, 1, eps) == 0
    assert blk.report.compressed_size == ref.size
    assert blk.report.cr == (float(st.field_bytes) - float(ref.size)) / float(st.field_bytes)


@pytest.mark.parametrize("which", [0, 1, 2, 3])
def test_tgv_fields_roundtrip(native, oracle, which):
    u = oracle.gen_tgv(8, 8, which)
    f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, 1e-3)
    assert _assert_stream_parity(oracle, blk, ref, 8, 1, 1e-3) == 0
    back, rep = native.decompress_with_error(blk, f.shape, f)
    rc, ob, ost = oracle.decompress(ref, 8, 1, 512, original=u)
    got = back.values.cpu().numpy()
    assert np.linalg.norm(got - ob) <= REL_TOL * max(np.linalg.norm(ob), 1e-300)
    if ost.nrm2 > 0:
        assert rep.rel_l2 <= 1e-3 * (1 + 1e-9)
        assert abs(rep.err2 - ost.err2) <= 1e-9 * ost.err2 + 1e-300
        assert abs(rep.nrm2 - ost.nrm2) <= 1e-12 * ost.nrm2
        assert rep.err_inf == ost.err_inf and rep.u_inf == ost.u_inf
    else:
        assert rep.rel_l2 == 0.0 and blk.kept_total == 0


@pytest.mark.parametrize("P", [2, 3, 4, 5, 6, 7, 9, 10, 11, 12, 13, 16])
def test_generic_lx_spectral(native, oracle, P):
    nb = 64 if P <= 12 else 16
    u = oracle.gen_spectral(P, nb)
    for eps in (1e-2, 1e-4):
        f, blk, ref, st = _compress_both(native, oracle, u, P, 1, eps)
        co = oracle.forward_field(u, P, 1)
        assert _assert_stream_parity(oracle, blk, ref, P, 1, eps, co) == 0
        back = native.lossy_decompress(blk, f.shape)
        rc, ob, _ = oracle.decompress(ref, P, 1, nb)
        assert np.linalg.norm(back.values.cpu().numpy() - ob) <= REL_TOL * np.linalg.norm(ob)


@pytest.mark.parametrize("eps", [1e-2, 1e-3, 1e-4, 1e-5])
def test_spectral_lx8_fast_path(native, oracle, eps):
    u = oracle.gen_spectral(8, 1000)  # ragged: 1000 blocks = 250 warp tiles
    f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, eps)
    co = oracle.forward_field(u, 8, 1)
    assert _assert_stream_parity(oracle, blk, ref, 8, 1, eps, co) == 0
    back = native.lossy_decompress(blk, f.shape)
    rc, ob, _ = oracle.decompress(ref, 8, 1, 1000)
    assert np.linalg.norm(back.values.cpu().numpy() - ob) <= REL_TOL * np.linalg.norm(ob)


def test_vector_field_components3(native, oracle):
    u = np.stack([oracle.gen_tgv(4, 8, w) for w in (0, 1, 3)], axis=-1)  # (E*512, 3)
    vals = u.reshape(-1)
    f, blk, ref, st = _compress_both(native, oracle, vals, 8, 3, 1e-3)
    assert _assert_stream_parity(oracle, blk, ref, 8, 3, 1e-3) == 0
    back = native.lossy_decompress(blk, f.shape)
    rc, ob, _ = oracle.decompress(ref, 8, 3, 64)
    assert np.linalg.norm(back.values.cpu().numpy() - ob) <= REL_TOL * np.linalg.norm(ob)


@pytest.mark.parametrize("eps,n_el", [(1e-2, 1000), (1e-5, 1000), (1e-3, 37)])
def test_vector_field_fast_path(native, oracle, eps, n_el):
    """components = 3 at lx = 8 runs on compress8 / compact8 / decompress8 (the stride-3
    block gather by cp.async): streams, reconstructions and the error report match the
    oracle exactly."""
    import paper_2407_20731_b200 as PK
    blocks = oracle.gen_spectral(8, 3 * n_el, block0=5).reshape(n_el, 3, 512)
    vals = np.ascontiguousarray(blocks.transpose(0, 2, 1)).reshape(-1)  # element -> point -> component
    f, blk, ref, st = _compress_both(native, oracle, vals, 8, 3, eps)
    assert PK.get_plan(8, 3, 0).last_launches() in (1, 2)   # single- or two-pass (auto schedule)
    assert _assert_stream_parity(oracle, blk, ref, 8, 3, eps) == 0
    back, rep = native.decompress_with_error(blk, f.shape, f)
    rc, ob, ost = oracle.decompress(ref, 8, 3, n_el, original=vals)
    assert rc == 0 and np.array_equal(back.values.cpu().numpy(), ob)  # bit-identical
    assert abs(rep.err2 - ost.err2) <= 1e-9 * max(ost.err2, 1e-300) and rep.err_inf == ost.err_inf


@pytest.mark.parametrize("n_el", [1, 3, 5, 7, 9, 33])
def test_ragged_small(native, oracle, n_el):
    u = oracle.gen_spectral(8, n_el, block0=77)
    f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, 1e-3)
    co = oracle.forward_field(u, 8, 1)
    assert _assert_stream_parity(oracle, blk, ref, 8, 1, 1e-3, co) == 0


def test_constant_and_zero_kat(native, oracle):
    # constant c != 0 -> exactly one kept coefficient per element
    for c in (3.7, -1e-200, 1e300, 5e-310):
        u = np.full(27 * 512, c)
        f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, 1e-3)
        assert blk.kept_total == 27 and st.kept == 27
        assert _assert_stream_parity(oracle, blk, ref, 8, 1, 1e-3) == 0
        back = native.lossy_decompress(blk, f.shape).values.cpu().numpy()
        assert np.max(np.abs(back - c)) <= 8 * np.spacing(abs(c))
    u = np.zeros(27 * 512)
    f, blk, ref, st = _compress_both(native, oracle, u, 8, 1, 1e-3)
    assert blk.kept_total == 0 and np.array_equal(blk.stream.cpu().numpy(), ref)
    assert np.all(native.lossy_decompress(blk, f.shape).values.cpu().numpy() == 0)


def test_nonfinite_rejected(native):
    import paper_2407_20731_b200 as PK
    u = torch.zeros(8 * 512, dtype=torch.float64, device="cuda")
    u[1234] = float("nan")
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_compress(PK.Field(2, 8, 1, u), PK.LossyConfig(1e-3))
    assert ei.value.code == PK.ErrorCode.InvalidArgument
    u[1234] = float("inf")
    with pytest.raises(PK.IsfError):
        PK.lossy_compress(PK.Field(2, 8, 1, u), PK.LossyConfig(1e-3))


def test_corrupt_stream_shape_mismatch(native, oracle):
    import paper_2407_20731_b200 as PK
    u = oracle.gen_tgv(4, 8, 0)
    f = _field(8, 1, 64, u)
    blk = PK.lossy_compress(f, PK.LossyConfig(1e-3))
    bad = PK.CompressedBlock(blk.stream.clone(), blk.n_elements, 8, 1, blk.kept_total, blk.report)
    bad.stream[0:4] = torch.tensor([255, 0, 0, 0], dtype=torch.uint8)  # count of block 0 wrong
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_decompress(bad, f.shape)
    assert ei.value.code == PK.ErrorCode.ShapeMismatch
    trunc = PK.CompressedBlock(blk.stream[:-8].clone(), blk.n_elements, 8, 1, blk.kept_total, blk.report)
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_decompress(trunc, f.shape)
    assert ei.value.code == PK.ErrorCode.ShapeMismatch
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_decompress(blk, (5, 8, 1))
    assert ei.value.code == PK.ErrorCode.ShapeMismatch


def test_determinism_and_launches(native, oracle):
    import paper_2407_20731_b200 as PK
    u = oracle.gen_spectral(8, 4096)
    f = _field(8, 1, 4096, u)
    plan = PK.get_plan(8, 1, 0)
    prev = plan.set_compress_mode(PK.LossyPlan.TWO_PASS)
    try:
        a = PK.lossy_compress(f, PK.LossyConfig(1e-3))
        b = PK.lossy_compress(f, PK.LossyConfig(1e-3))
        assert plan.last_launches() == 2                     # compress8 + compact8
        plan.set_compress_mode(PK.LossyPlan.SINGLE_PASS)
        c = PK.lossy_compress(f, PK.LossyConfig(1e-3))
        assert plan.last_launches() == 1
    finally:
        plan.set_compress_mode(prev)
    assert torch.equal(a.stream, b.stream) and torch.equal(a.stream, c.stream)


def test_host_entry_points(native, oracle):
    import paper_2407_20731_b200 as PK
    u = oracle.gen_tgv(8, 8, 3)
    plan = PK.get_plan(8, 1, 0)
    hs = np.zeros(plan.capacity(512), dtype=np.uint8)
    nb, st = plan.compress_host(u, 512, 1e-3, hs)
    rc, ref, ost = oracle.compress(u, 8, 1, 1e-3)
    assert nb == ref.size and np.array_equal(hs[:nb], ref)
    out = np.zeros_like(u)
    st2 = plan.decompress_host(hs, nb, 512, out, u)
    rc, ob, _ = oracle.decompress(ref, 8, 1, 512)
    assert np.linalg.norm(out - ob) <= REL_TOL * np.linalg.norm(ob)
    assert np.sqrt(st2.err2 / st2.nrm2) <= 1e-3


def test_device_generators_match_oracle(native, oracle):
    import paper_2407_20731_b200 as PK
    plan = PK.get_plan(8, 1, 0)
    out = torch.empty(256 * 512, dtype=torch.float64, device="cuda")
    plan.generate_spectral(out, 256, 1000, oracle.SPECTRAL_SEED, oracle.spectral_amplitudes(8))
    ref = oracle.gen_spectral(8, 256, block0=1000)
    assert np.array_equal(out.cpu().numpy(), ref)  # integer-exact coefficients + pinned inverse
    t = torch.empty(16 ** 3 * 512, dtype=torch.float64, device="cuda")
    plan.generate_tgv(t, 16, 0)
    tr = oracle.gen_tgv(16, 8, 0)
    assert np.max(np.abs(t.cpu().numpy() - tr)) <= 4e-15  # libm vs CUDA cos/sin: a few ulp


@pytest.mark.parametrize("kind", ["spectral", "tgv"])
def test_determinism_stress(native, oracle, kind):
    """Repeated runs must give identical streams and statistics (no races in the TMA
    ring, the parked coefficients, the compaction or the fused finalize)."""
    import paper_2407_20731_b200 as PK
    if kind == "spectral":
        u = oracle.gen_spectral(8, 20000)
        n_el = 20000
    else:
        u = oracle.gen_tgv(32, 8, 3)
        n_el = 32 ** 3
    f = _field(8, 1, n_el, u)
    ref = None
    refd = None
    for it in range(6):
        blk = PK.lossy_compress(f, PK.LossyConfig(1e-3))
        back, rep = PK.decompress_with_error(blk, f.shape, f)
        s = blk.stream.cpu().numpy()
        d = back.values.cpu().numpy()
        if ref is None:
            ref, refd, refrep = s, d, rep
            rc, os_, st = oracle.compress(u, 8, 1, 1e-3)
            assert np.array_equal(s, os_)
        else:
            assert np.array_equal(s, ref), f"stream differs on run {it}"
            assert np.array_equal(d, refd), f"reconstruction differs on run {it}"
            assert (rep.err2, rep.nrm2, rep.err_inf, rep.u_inf) == (refrep.err2, refrep.nrm2, refrep.err_inf, refrep.u_inf)


def test_c_abi_allreduce_single_rank(native):
    """isf_lossy_allreduce over a 1-rank NCCL communicator: sums/max are identities
    and every status bit survives the lane spread/fold (NCCL has no OR)."""
    import ctypes
    import glob
    import os
    from paper_2407_20731_b200 import _native
    libs = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "nccl", "lib", "libnccl.so*"))
    if not libs:
        pytest.skip("no libnccl")
    nccl = ctypes.CDLL(libs[0], mode=ctypes.RTLD_GLOBAL)
    comm = ctypes.c_void_p()
    torch.cuda.set_device(0)
    assert nccl.ncclCommInitAll(ctypes.byref(comm), 1, (ctypes.c_int * 1)(0)) == 0
    try:
        L = _native.lib()
        for status in (0, 1, 2, 5, 7):
            st = torch.zeros(12, dtype=torch.float64)
            st[:6] = torch.tensor([1.5, 2.0, 0.25, 3.0, 0.125, 4.0], dtype=torch.float64)
            st = st.cuda()
            su = st.view(torch.int64)
            su[6:11] = torch.tensor([11, 22, 33, 44, status], dtype=torch.int64, device="cuda")
            ref = st.clone()
            s = torch.cuda.current_stream()
            assert L.isf_lossy_allreduce(ctypes.c_void_p(st.data_ptr()), comm, ctypes.c_void_p(s.cuda_stream)) == 0
            torch.cuda.synchronize()
            assert torch.equal(st.view(torch.int64)[:11], ref.view(torch.int64)[:11]), status
    finally:
        nccl.ncclCommDestroy(comm)


@pytest.mark.parametrize("P", [3, 4, 6, 10, 12])
def test_generic_decompress_bitexact(native, oracle, P):
    """The generic (lx != 8) decode + inverse DLT is bit-identical to the oracle's."""
    nb = 64
    u = oracle.gen_spectral(P, nb)
    for eps in (1e-2, 1e-6):
        f, blk, ref, st = _compress_both(native, oracle, u, P, 1, eps)
        back = native.lossy_decompress(blk, f.shape)
        rc, ob, _ = oracle.decompress(blk.stream.cpu().numpy(), P, 1, nb)
        assert rc == 0
        assert np.array_equal(back.values.cpu().numpy().view(np.uint64), ob.view(np.uint64)), (P, eps)


@pytest.mark.parametrize("P", [4, 5, 6, 10, 12])
def test_warp_decompress_shape_and_bits(native, oracle, P):
    """The warp-per-block decode (lx 4/5/6/10/12, dlt_warp.cuh): a wrong count, a
    truncated value region and a stray mask bit past lx^3 raise ShapeMismatch; tiny
    (subnormal) coefficients and all-(-0) blocks reconstruct bit-identically to the
    oracle (+0 canonicalisation)."""
    import paper_2407_20731_b200 as PK
    n = 27
    u = oracle.gen_spectral(P, n)
    f = _field(P, 1, n, u)
    blk = PK.lossy_compress(f, PK.LossyConfig(1e-3))
    # count of block 3 off by one
    bad = PK.CompressedBlock(blk.stream.clone(), blk.n_elements, P, 1, blk.kept_total, blk.report)
    c3 = int(bad.stream[12:16].cpu().numpy().view(np.uint32)[0])
    bad.stream[12:16] = torch.from_numpy(np.array([c3 + 1], dtype=np.uint32).view(np.uint8)).cuda()
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_decompress(bad, f.shape)
    assert ei.value.code == PK.ErrorCode.ShapeMismatch
    trunc = PK.CompressedBlock(blk.stream[:-16].clone(), blk.n_elements, P, 1, blk.kept_total, blk.report)
    with pytest.raises(PK.IsfError) as ei:
        PK.lossy_decompress(trunc, f.shape)
    assert ei.value.code == PK.ErrorCode.ShapeMismatch
    N3, W = P ** 3, (P ** 3 + 63) // 64
    if N3 % 64:
        stray = PK.CompressedBlock(blk.stream.clone(), blk.n_elements, P, 1, blk.kept_total, blk.report)
        mask_off = (4 * n + 15) & ~15
        o = mask_off + 8 * (0 * W + W - 1) + 7  # last mask word of block 0, bit 63
        stray.stream[o] = int(stray.stream[o].item()) | 0x80
        with pytest.raises(PK.IsfError) as ei:
            PK.lossy_decompress(stray, f.shape)
        assert ei.value.code == PK.ErrorCode.ShapeMismatch
    # subnormal coefficients and an all -0 block
    v = (u * 1e-305).reshape(n, N3)
    v[5] = -0.0
    v = v.reshape(-1)
    f2, blk2, ref2, _ = _compress_both(native, oracle, v, P, 1, 1e-2)
    assert _assert_stream_parity(oracle, blk2, ref2, P, 1, 1e-2) == 0
    back = native.lossy_decompress(blk2, f2.shape)
    rc, ob, _ = oracle.decompress(ref2, P, 1, n)
    assert rc == 0
    assert np.array_equal(back.values.cpu().numpy().view(np.uint64), ob.view(np.uint64))
    assert not np.any(back.values.cpu().numpy().view(np.uint64)[5 * N3:6 * N3])  # +0, not -0


@pytest.mark.parametrize("case", ["tgv", "spectral_dense", "tiny_values", "signed_zeros", "mixed"])
def test_decompress_bitexact(native, oracle, case):
    """Reconstructions are bit-identical to the oracle's (incl. +0 canonicalisation,
    DESIGN.md 3.3), also for streams whose values are subnormal, zero or -0 and
    whose occupied index planes are sparse (the lx=8 kernel skips empty planes)."""
    import paper_2407_20731_b200 as PK
    P, E = 8, 4
    n_el = E ** 3
    if case == "tgv":
        u = oracle.gen_tgv(E, P, 3)
        eps = 1e-3
    elif case == "mixed":  # sparse TGV blocks interleaved with dense spectral ones
        t = oracle.gen_tgv(E, P, 0).reshape(n_el, P ** 3)
        sp = oracle.gen_spectral(P, n_el).reshape(n_el, P ** 3)
        u = np.where((np.arange(n_el) % 3 == 1)[:, None], sp, t).reshape(-1).copy()
        eps = 1e-5
    else:
        u = oracle.gen_spectral(P, n_el)
        eps = 1e-2 if case != "spectral_dense" else 1e-6
    rc, ref, _ = oracle.compress(u, P, 1, eps)
    assert rc == 0
    ref = ref.copy()
    counts, masks, vals = oracle.parse_stream(ref, P, n_el)
    vals = vals.copy()
    rng = np.random.default_rng(7)
    if case == "tiny_values":
        sel = rng.random(vals.size) < 0.5
        vals[sel] *= 2.0 ** -1070          # subnormal products underflow inside the sweeps
    if case == "signed_zeros":
        sel = rng.random(vals.size)
        vals[sel < 0.2] = 0.0
        vals[(sel >= 0.2) & (sel < 0.4)] = -0.0
    ref[ref.size - vals.size * 8:] = vals.view(np.uint8)
    rc, ob, _ = oracle.decompress(ref, P, 1, n_el)
    assert rc == 0
    plan = PK.get_plan(P, 1, 0)
    d_stream = torch.from_numpy(ref).cuda()
    out = torch.empty(n_el * P ** 3, dtype=torch.float64, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    plan.decompress_async(d_stream, ref.size, n_el, out, stats)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert int(stats.view(torch.int64)[10].item()) == 0
    assert np.array_equal(got.view(np.uint64), ob.view(np.uint64))
    assert not np.any(got.view(np.uint64) == np.uint64(1 << 63))  # no -0 in the output


@pytest.mark.parametrize("P,eps,kind", [(8, 1e-2, "tgv"), (8, 1e-4, "spectral"), (6, 1e-3, "spectral"),
                                        (4, 1e-1, "spectral"), (12, 1e-3, "spectral"), (16, 1e-2, "spectral")])
def test_linf_stream_bitexact_and_bound(native, oracle, P, eps, kind):
    """RelativeLInf truncation: GPU stream byte-identical to the oracle,
    reconstruction within eps * max|u| (global) through the error report."""
    import paper_2407_20731_b200 as PK
    E = 3 if P >= 12 else 4
    n_el = E ** 3
    u = oracle.gen_tgv(E, P, 0) if kind == "tgv" else oracle.gen_spectral(P, n_el)
    f = _field(P, 1, n_el, u)
    cfg = PK.LossyConfig(eps, PK.ErrorNorm.RelativeLInf)
    blk = native.lossy_compress(f, cfg)
    rc, ref, _ = oracle.compress(u, P, 1, eps, norm=1)
    assert rc == 0
    assert np.array_equal(blk.stream.cpu().numpy(), ref)
    back, rep = native.decompress_with_error(blk, f.shape, f)
    assert rep.rel_linf <= eps * (1 + 1e-9)


def test_linf_vector_field(native, oracle):
    import paper_2407_20731_b200 as PK
    P, E = 8, 3
    u = np.concatenate([oracle.gen_spectral(P, E ** 3, block0=b) for b in (0, 100, 200)])
    v = u.reshape(3, -1, P ** 3).transpose(1, 2, 0).copy().reshape(-1)  # element, point, component
    f = _field(P, 3, E ** 3, v)
    blk = native.lossy_compress(f, PK.LossyConfig(1e-3, PK.ErrorNorm.RelativeLInf))
    rc, ref, _ = oracle.compress(v, P, 3, 1e-3, norm=1)
    assert rc == 0 and np.array_equal(blk.stream.cpu().numpy(), ref)


def test_plan_reuse_varying_sizes(native, oracle):
    """One plan, block counts that grow and shrink across calls: the double-buffered
    per-chunk kept sums (compress8 -> compact8) must be clean for every call."""
    P = 8
    plan = native.get_plan(P, 1, 0)
    for n_el in (5000, 1100, 70, 1100, 5000, 3000, 5000):
        u = oracle.gen_spectral(P, n_el)
        f = _field(P, 1, n_el, u)
        blk = native.lossy_compress(f, native.LossyConfig(1e-3), plan=plan)
        rc, ref, _ = oracle.compress(u, P, 1, 1e-3)
        assert rc == 0 and np.array_equal(blk.stream.cpu().numpy(), ref), n_el


@pytest.mark.parametrize("kind", ["tgv", "spectral_dense", "spectral"])
def test_single_pass_schedule(native, oracle, kind):
    """The single-pass lx = 8 compress (values written in place two rounds after their
    selection, behind per-round CTA aggregates) gives the two-pass streams byte for byte,
    including dense blocks, partial last rounds and repeated calls on one plan."""
    import paper_2407_20731_b200 as PK
    P = 8
    plan = PK.LossyPlan(P, 1, 0)
    assert plan.set_compress_mode(PK.LossyPlan.SINGLE_PASS) == PK.LossyPlan.AUTO  # the default
    try:
        if kind == "tgv":
            u, n_el, eps = oracle.gen_tgv(24, P, 0), 24 ** 3, 1e-3
        elif kind == "spectral_dense":
            u, n_el, eps = oracle.gen_spectral(P, 7001), 7001, 1e-5
        else:
            u, n_el, eps = oracle.gen_spectral(P, 3333), 3333, 1e-2
        f = _field(P, 1, n_el, u)
        rc, ref, _ = oracle.compress(u, P, 1, eps)
        assert rc == 0
        for _ in range(3):
            blk = native.lossy_compress(f, native.LossyConfig(eps), plan=plan)
            assert plan.last_launches() == 1
            assert np.array_equal(blk.stream.cpu().numpy(), ref)
        back = native.lossy_decompress(blk, f.shape)
        rc, ob, _ = oracle.decompress(ref, P, 1, n_el)
        assert np.allclose(back.values.cpu().numpy(), ob, rtol=0, atol=0)
    finally:
        plan.set_compress_mode(PK.LossyPlan.AUTO)
    with pytest.raises(PK.IsfError):
        plan.set_compress_mode(7)


def test_auto_schedule_follows_density(native, oracle):
    """AUTO (default) runs the two-pass schedule after sparse calls and the single-pass
    one after a call that kept more than half of the coefficients; streams equal the
    oracle's on every call."""
    import paper_2407_20731_b200 as PK
    plan = PK.LossyPlan(8, 1, 0)
    dense = oracle.gen_spectral(8, 2000)
    sparse = oracle.gen_tgv(12, 8, 0)
    seq = [(sparse, 12 ** 3, 1e-3, 2), (dense, 2000, 1e-5, 2), (dense, 2000, 1e-5, 1), (sparse, 12 ** 3, 1e-3, 1),
           (sparse, 12 ** 3, 1e-3, 2)]
    for u, n_el, eps, launches in seq:
        blk = native.lossy_compress(_field(8, 1, n_el, u), native.LossyConfig(eps), plan=plan)
        torch.cuda.synchronize()
        assert plan.last_launches() == launches, (n_el, eps)
        rc, ref, _ = oracle.compress(u, 8, 1, eps)
        assert np.array_equal(blk.stream.cpu().numpy(), ref)


@pytest.mark.parametrize("P,mode", [(8, 0), (8, 1), (6, 0), (12, 0)])
def test_status_flags_all_schedules(native, oracle, P, mode):
    """Non-finite input and a stream capacity that cannot hold the kept values raise
    the same status bits on every compress schedule (two-pass lx=8, single-pass lx=8,
    generic slots + compact_generic), and a good call afterwards is clean again."""
    import paper_2407_20731_b200 as PK
    plan = PK.LossyPlan(P, 1, 0)
    plan.set_compress_mode(mode) if P == 8 else None
    n_el = 3000
    u = oracle.gen_spectral(P, n_el)
    x = torch.from_numpy(u).cuda()
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    hdr = plan.header_bytes(n_el)
    # 1. capacity: header plus room for 10 values only (the spectrum keeps far more)
    small = torch.zeros(hdr + 80, dtype=torch.uint8, device="cuda")
    plan.compress_async(x, n_el, 1e-5, small, stats)
    torch.cuda.synchronize()
    assert int(stats.view(torch.int64)[10].item()) & 4, "overflow not flagged"
    # 2. non-finite input
    bad = x.clone()
    bad[777] = float("nan")
    st = torch.zeros(plan.capacity(n_el), dtype=torch.uint8, device="cuda")
    plan.compress_async(bad, n_el, 1e-3, st, stats)
    torch.cuda.synchronize()
    assert int(stats.view(torch.int64)[10].item()) & 1, "non-finite not flagged"
    # 3. a good call right after: clean status, oracle-identical stream
    plan.compress_async(x, n_el, 1e-3, st, stats)
    torch.cuda.synchronize()
    si = stats.view(torch.int64)
    assert int(si[10].item()) == 0
    rc, ref, _ = oracle.compress(u, P, 1, 1e-3)
    assert np.array_equal(st[: int(si[8].item())].cpu().numpy(), ref)


@pytest.mark.parametrize("P", [6, 12])
def test_generic_large_sampled_parity(native, oracle, P):
    """cfg4-sized generic path (32,768 elements): deterministic streams, the L2 bound,
    plain decode == decode with error report, and the first / last 128 blocks of the
    stream (counts, masks, value records) bit-identical to the oracle's stream of the
    same blocks (offsets at full size)."""
    import paper_2407_20731_b200 as PK
    n, S = 32768, 128
    plan = PK.get_plan(P, 1, 0)
    vals = torch.empty(n * P ** 3, dtype=torch.float64, device="cuda")
    plan.generate_spectral(vals, n, 0, oracle.SPECTRAL_SEED, oracle.spectral_amplitudes(P))
    f = PK.Field(32, P, 1, vals)
    eps = 1e-3
    a = PK.lossy_compress(f, PK.LossyConfig(eps))
    b = PK.lossy_compress(f, PK.LossyConfig(eps))
    assert torch.equal(a.stream, b.stream)
    back, rep = PK.decompress_with_error(a, f.shape, f)
    plain = PK.lossy_decompress(a, f.shape)
    assert torch.equal(back.values.view(torch.int64), plain.values.view(torch.int64))
    assert 0 < rep.rel_l2 <= eps * (1 + 1e-9)
    got = a.stream.cpu().numpy()
    gc, gm, gv = oracle.parse_stream(got, P, n)
    go = np.concatenate([[0], np.cumsum(gc.astype(np.int64))])
    for b0 in (0, n - S):
        u = oracle.gen_spectral(P, S, block0=b0)
        rc, ref, _ = oracle.compress(u, P, 1, eps)
        assert rc == 0
        rc_, rm, rv = oracle.parse_stream(ref, P, S)
        assert np.array_equal(gc[b0:b0 + S], rc_) and np.array_equal(gm[b0:b0 + S], rm)
        assert np.array_equal(np.asarray(gv[go[b0]:go[b0 + S]]).view(np.uint64), np.asarray(rv).view(np.uint64))
