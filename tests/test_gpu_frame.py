"""Device CRC-32 and kind-1 framing against zlib and the frame
codec that mirrors the reference build_frame (proj/src/core/frame.cpp:9-25)."""
import zlib

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [0, 1, 7, 16, 127, 128, 4095, 4096, 4097, 8192, 12345, 1 << 20,
                               (1 << 22) + 13, 3 * (1 << 22) * 1024 // 1024 + 4095])
@pytest.mark.parametrize("offset", [0, 3])
def test_crc32_matches_zlib(native, n, offset):
    import paper_2407_20731_b200 as PK
    rng = np.random.default_rng(n + offset)
    host = rng.integers(0, 256, n + offset, dtype=np.uint8)
    d = torch.from_numpy(host).cuda()
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    plan = PK.get_plan(8, 1, 0)
    plan.crc32_async(d[offset:], n, out)
    torch.cuda.synchronize()
    got = int(out.item()) & 0xFFFFFFFF
    assert got == zlib.crc32(host[offset:].tobytes()) & 0xFFFFFFFF


def test_crc32_large_chunk_tree(native):
    """> 1024 * 4 KiB so that the per-thread runs of the final fold are longer than one."""
    import paper_2407_20731_b200 as PK
    n = 4096 * 5000 + 1234
    d = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
    out = torch.zeros(1, dtype=torch.int32, device="cuda")
    PK.get_plan(8, 1, 0).crc32_async(d, n, out)
    torch.cuda.synchronize()
    assert int(out.item()) & 0xFFFFFFFF == zlib.crc32(d.cpu().numpy().tobytes()) & 0xFFFFFFFF


@pytest.mark.parametrize("which,eps", [(0, 1e-3), (2, 1e-3), (3, 1e-5)])
def test_device_frame_equals_host_frame(native, oracle, which, eps):
    """The device frame (SPEC.md:282 payload converted on the device) equals the host
    framing of the oracle's stream, and parses back to exactly that stream."""
    import paper_2407_20731_b200 as PK
    from paper_2407_20731_b200 import frame as FR
    E, P = 8, 8
    u = oracle.gen_tgv(E, P, which)
    f = PK.Field(E, P, 1, torch.from_numpy(u).cuda())
    fr, rep, kept = PK.lossy_compress_frame(f, PK.LossyConfig(eps), step_index=42, sim_time=0.125)
    got = fr.cpu().numpy().tobytes()
    rc, ref, _ = oracle.compress(u, P, 1, eps)
    assert rc == 0
    payload = FR.spec_payload(ref, E ** 3, P, 1)
    want = FR.build_frame(FR.FrameHeader(FR.KIND_COMPRESSED_BLOCK, 42, 0.125, E, P, 1), payload)
    assert got == want
    h, stream, codec, coded = FR.parse_block_frame(got)
    assert stream == ref.tobytes() and codec == 0 and coded == b""
    assert h.payload_len == 4 * E ** 3 + 12 * kept + 10
    assert rep.compressed_size == len(ref)


@pytest.mark.parametrize("P,comps,n", [(6, 1, 27), (8, 3, 8), (12, 1, 8)])
def test_device_frame_generic_lx_and_vector(native, oracle, P, comps, n):
    import paper_2407_20731_b200 as PK
    from paper_2407_20731_b200 import frame as FR
    u = np.random.default_rng(P * comps).standard_normal(n * P ** 3 * comps)
    E = round(n ** (1 / 3))
    f = PK.Field(E, P, comps, torch.from_numpy(u).cuda())
    fr, rep, kept = PK.lossy_compress_frame(f, PK.LossyConfig(1e-2))
    rc, ref, _ = oracle.compress(u, P, comps, 1e-2)
    got = fr.cpu().numpy().tobytes()
    assert got == FR.build_frame(FR.FrameHeader(FR.KIND_COMPRESSED_BLOCK, 0, 0.0, E, P, comps),
                                 FR.spec_payload(ref, n, P, comps))
    assert FR.parse_block_frame(got, n)[1] == ref.tobytes()


def test_device_frame_overflow_flag(native, oracle):
    import paper_2407_20731_b200 as PK
    E, P = 4, 8
    u = oracle.gen_tgv(E, P, 0)
    plan = PK.get_plan(P, 1, 0)
    n_el = E ** 3
    stream = torch.zeros(plan.capacity(n_el), dtype=torch.uint8, device="cuda")
    stats = torch.zeros(12, dtype=torch.float64, device="cuda")
    plan.compress_async(torch.from_numpy(u).cuda(), n_el, 1e-3, stream, stats)
    small = torch.zeros(64, dtype=torch.uint8, device="cuda")  # far too small for header + payload
    plan.frame_async(small, stream, n_el, stats, E)
    torch.cuda.synchronize()
    assert int(stats.view(torch.int64)[10].item()) & 4
