"""Kind-1 frames of a compressed block against the REFERENCE's own build_frame /
parse_frame (proj/src/core/frame.cpp:9-71), compiled from /root/reference into
oracle/_ref/ by `make -C oracle ref`.  Skipped where the reference is absent (the
GPU box); the pure-Python framing checks still run."""
import ctypes
import os
import struct
import zlib

import numpy as np
import pytest

from paper_2407_20731_b200 import frame as FR
from paper_2407_20731_b200.lossy import ErrorCode, IsfError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libisf_ref.so")


@pytest.fixture(scope="module")
def ref():
    if os.path.isdir("/root/reference/proj"):
        import subprocess
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
    if not os.path.exists(REF_SO):
        pytest.skip("reference core not built here (no /root/reference)")
    L = ctypes.CDLL(REF_SO)
    L.ref_build_frame.restype = ctypes.c_ulonglong
    L.ref_build_frame.argtypes = [ctypes.c_uint, ctypes.c_ulonglong, ctypes.c_double, ctypes.c_uint,
                                  ctypes.c_uint, ctypes.c_uint, ctypes.c_void_p, ctypes.c_ulonglong,
                                  ctypes.c_void_p, ctypes.c_ulonglong]
    L.ref_parse_frame.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong, ctypes.POINTER(ctypes.c_ulonglong),
                                  ctypes.POINTER(ctypes.c_ulonglong), ctypes.POINTER(ctypes.c_uint)]
    L.ref_crc32.restype = ctypes.c_uint
    L.ref_crc32.argtypes = [ctypes.c_void_p, ctypes.c_ulonglong]
    L.ref_field_validate.argtypes = [ctypes.c_uint, ctypes.c_uint, ctypes.c_uint, ctypes.c_void_p,
                                     ctypes.c_ulonglong]
    L.ref_error_code_name.restype = ctypes.c_char_p
    return L


def _ref_frame(L, h, payload: bytes) -> bytes:
    buf = ctypes.create_string_buffer(len(payload) + 64)
    n = L.ref_build_frame(h.kind, h.step_index, h.sim_time, h.elements_per_axis, h.points_per_element_axis,
                          h.components, payload, len(payload), buf, len(buf))
    return buf.raw[:n]


def test_kind1_frame_bytes_equal_reference(ref, oracle):
    u = oracle.gen_tgv(4, 8, 0)
    rc, s, st = oracle.compress(u, 8, 1, 1e-3)
    payload = FR.spec_payload(s, 64, 8, 1)
    h = FR.FrameHeader(FR.KIND_COMPRESSED_BLOCK, 42, 0.125, 4, 8, 1, len(payload))
    mine = FR.build_frame(h, payload)
    assert mine == _ref_frame(ref, h, payload)
    off, ln, kind = ctypes.c_ulonglong(), ctypes.c_ulonglong(), ctypes.c_uint()
    assert ref.ref_parse_frame(mine, len(mine), ctypes.byref(off), ctypes.byref(ln), ctypes.byref(kind)) == 0
    assert kind.value == 1 and off.value == 48 and ln.value == len(payload)
    hh, stream, codec, coded = FR.parse_block_frame(mine)
    assert stream == s.tobytes() and codec == 0 and coded == b""
    # SPEC.md:282 layout: kept_count u32 per element | index u32 | value f64 | trailer
    K = int(st.kept)
    assert len(payload) == 4 * 64 + 12 * K + 10
    per_el = np.frombuffer(payload, dtype="<u4", count=64)
    assert int(per_el.sum()) == K


def test_crc_and_error_codes_match_reference(ref):
    for data in (b"123456789", bytes(range(256)) * 7):
        assert ref.ref_crc32(data, len(data)) == zlib.crc32(data)
    assert zlib.crc32(b"123456789") == 0xCBF43926
    frame = FR.build_frame(FR.FrameHeader(payload_len=3), b"abc")
    bad = bytearray(frame)
    bad[50] ^= 1
    off, ln, kind = ctypes.c_ulonglong(), ctypes.c_ulonglong(), ctypes.c_uint()
    rc = ref.ref_parse_frame(bytes(bad), len(bad), ctypes.byref(off), ctypes.byref(ln), ctypes.byref(kind))
    assert rc == 1 + ErrorCode.ChecksumMismatch
    with pytest.raises(IsfError) as ei:
        FR.parse_frame(bytes(bad))
    assert ei.value.code == ErrorCode.ChecksumMismatch
    rc = ref.ref_parse_frame(frame[:30], 30, ctypes.byref(off), ctypes.byref(ln), ctypes.byref(kind))
    assert rc == 1 + ErrorCode.LengthMismatch
    for code in ErrorCode:
        assert ref.ref_error_code_name(int(code)).decode() == code.name


def test_field_validation_matches_reference(ref):
    # proj/src/core/types.cpp:58-74: the codes our API returns for the same defects
    ok = np.zeros(8 * 8 * 8 * 8)
    assert ref.ref_field_validate(2, 8, 1, ok.ctypes.data, ok.size) == 0
    assert ref.ref_field_validate(2, 8, 4, ok.ctypes.data, ok.size) == 1 + ErrorCode.InvalidArgument
    bad = ok.copy()
    bad[3] = np.inf
    assert ref.ref_field_validate(2, 8, 1, bad.ctypes.data, bad.size) == 1 + ErrorCode.InvalidArgument


def test_python_frame_errors():
    f = FR.build_frame(FR.FrameHeader(payload_len=2), b"xy")
    assert len(f) == 48 + 2 + 4
    with pytest.raises(IsfError) as e:
        FR.parse_frame(b"ISF2" + f[4:])
    assert e.value.code == ErrorCode.BadMagic
    with pytest.raises(IsfError) as e:
        FR.parse_frame(f[:4] + struct.pack("<H", 2) + f[6:])
    assert e.value.code == ErrorCode.UnsupportedVersion
    with pytest.raises(IsfError) as e:
        FR.parse_frame(f[:-1])
    assert e.value.code == ErrorCode.LengthMismatch
