"""ISF1 core frame around a compressed block (payload_kind = 1).

Byte-compatible with the reference's framing (proj/include/isf/core/frame.hpp:3-11,
proj/src/core/frame.cpp:9-71): little-endian 48-byte header
``"ISF1" | version u16 = 1 | payload_kind u16 | step u64 | sim_time f64 | E u32 |
P u32 | components u32 | reserved u32 = 0 | payload_len u64`` followed by the payload
and an IEEE CRC-32 (zlib polynomial) of header + payload.  Errors mirror
parse_frame / parse_frame_header (BadMagic, UnsupportedVersion, LengthMismatch,
ChecksumMismatch).  The payload of a kind-1 frame is SPEC.md:282's:
``kept_count u32[n_elements] | index u32[K] | value f64[K] | codec id u16 | coded
length u64 | coded bytes`` with index = component * P^3 + j (ascending inside each
element), converted from / to the mask stream of include/isf_lossy.h.
The device builds the same bytes (isf_lossy_frame_async).
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

import numpy as np

from .lossy import ErrorCode, IsfError

MAGIC = b"ISF1"
VERSION = 1
HEADER_SIZE = 48   # frame.hpp:23
TRAILER_SIZE = 4   # frame.hpp:24
KIND_FIELD_SNAPSHOT = 0
KIND_COMPRESSED_BLOCK = 1
_HDR = struct.Struct("<4sHHQdIIIIQ")


@dataclass
class FrameHeader:
    kind: int = KIND_COMPRESSED_BLOCK
    step_index: int = 0
    sim_time: float = 0.0
    elements_per_axis: int = 0
    points_per_element_axis: int = 0
    components: int = 0
    payload_len: int = 0


def build_frame(h: FrameHeader, payload: bytes) -> bytes:
    """frame.cpp:9-25."""
    head = _HDR.pack(MAGIC, VERSION, h.kind, h.step_index, h.sim_time, h.elements_per_axis,
                     h.points_per_element_axis, h.components, 0, len(payload))
    body = head + bytes(payload)
    return body + struct.pack("<I", zlib.crc32(body) & 0xFFFFFFFF)


def parse_frame_header(b: bytes) -> FrameHeader:
    """frame.cpp:27-55."""
    if len(b) < HEADER_SIZE:
        raise IsfError(ErrorCode.LengthMismatch, f"frame header needs {HEADER_SIZE} bytes, got {len(b)}")
    magic, ver, kind, step, t, E, P, C, _res, plen = _HDR.unpack_from(b, 0)
    for i in range(4):
        if magic[i] != MAGIC[i]:
            raise IsfError(ErrorCode.BadMagic, f"magic mismatch at byte {i}")
    if ver != VERSION:
        raise IsfError(ErrorCode.UnsupportedVersion, f"frame version {ver}, expected {VERSION}")
    if kind > 1:
        raise IsfError(ErrorCode.UnsupportedVersion, f"unknown payload_kind {kind}")
    return FrameHeader(kind, step, t, E, P, C, plen)


def parse_frame(b: bytes):
    """frame.cpp:57-71: validates length and CRC, returns (header, payload)."""
    h = parse_frame_header(b)
    expected = HEADER_SIZE + h.payload_len + TRAILER_SIZE
    if len(b) != expected:
        raise IsfError(ErrorCode.LengthMismatch, f"frame length {len(b)}, header implies {expected}")
    body = b[: HEADER_SIZE + h.payload_len]
    (crc,) = struct.unpack_from("<I", b, HEADER_SIZE + h.payload_len)
    if (zlib.crc32(body) & 0xFFFFFFFF) != crc:
        raise IsfError(ErrorCode.ChecksumMismatch, "CRC mismatch")
    return h, b[HEADER_SIZE: HEADER_SIZE + h.payload_len]


def _stream_parts(stream: np.ndarray, n_el: int, P: int, comps: int):
    B = n_el * comps
    W = (P ** 3 + 63) // 64
    m0 = (4 * B + 15) & ~15
    counts = stream[: 4 * B].view(np.uint32)
    masks = stream[m0: m0 + 8 * W * B].view(np.uint64).reshape(B, W)
    vals = stream[m0 + 8 * W * B:].view(np.float64)
    return counts, masks, vals


def spec_payload(stream, n_el: int, P: int, comps: int, codec: int = 0, coded: bytes = b"") -> bytes:
    """SPEC.md:282 kind-1 payload from the mask stream (host restatement of the
    device conversion in csrc/crc32.cuh spec_frame_kernel)."""
    stream = np.frombuffer(bytes(stream), dtype=np.uint8) if not isinstance(stream, np.ndarray) else stream
    P3 = P ** 3
    counts, masks, vals = _stream_parts(stream, n_el, P, comps)
    B = n_el * comps
    W = masks.shape[1]
    bits = np.unpackbits(masks.view(np.uint8).reshape(B, W * 8), axis=1, bitorder="little")[:, :P3]
    bi, ji = np.nonzero(bits)
    idx = (bi % comps).astype(np.uint32) * np.uint32(P3) + ji.astype(np.uint32)
    per_el = counts.reshape(n_el, comps).sum(axis=1).astype("<u4")
    return (per_el.tobytes() + idx.astype("<u4").tobytes() + vals.astype("<f8").tobytes() +
            struct.pack("<HQ", codec, len(coded)) + bytes(coded))


def stream_from_spec_payload(payload: bytes, n_el: int, P: int, comps: int):
    """Inverse of spec_payload: (mask stream bytes, codec id, coded bytes).  Raises
    LengthMismatch / ShapeMismatch for payloads that do not describe n_el elements."""
    P3 = P ** 3
    if len(payload) < 4 * n_el + 10:
        raise IsfError(ErrorCode.LengthMismatch, "kind-1 payload shorter than its counts + codec trailer")
    per_el = np.frombuffer(payload, dtype="<u4", count=n_el)
    K = int(per_el.sum(dtype=np.uint64))
    body = 4 * n_el + 12 * K
    if len(payload) < body + 10:
        raise IsfError(ErrorCode.LengthMismatch, "kind-1 payload shorter than its index and value arrays")
    codec, n = struct.unpack_from("<HQ", payload, body)
    if body + 10 + n != len(payload):
        raise IsfError(ErrorCode.LengthMismatch, "codec trailer length mismatch")
    idx = np.frombuffer(payload, dtype="<u4", count=K, offset=4 * n_el).astype(np.int64)
    vals = np.frombuffer(payload, dtype="<f8", count=K, offset=4 * n_el + 4 * K)
    el = np.repeat(np.arange(n_el), per_el.astype(np.int64))
    if K and (idx.max() >= comps * P3 or bool(np.any((np.diff(idx) <= 0) & (np.diff(el) == 0)))):
        raise IsfError(ErrorCode.ShapeMismatch, "kind-1 payload: index out of range or not ascending")
    blk = el * comps + idx // P3
    j = idx % P3
    B = n_el * comps
    W = (P3 + 63) // 64
    counts = np.bincount(blk, minlength=B).astype("<u4")
    masks = np.zeros((B, W), dtype=np.uint64)
    np.bitwise_or.at(masks, (blk, j // 64), np.left_shift(np.uint64(1), (j % 64).astype(np.uint64)))
    m0 = (4 * B + 15) & ~15
    out = bytearray(m0 + 8 * W * B + 8 * K)
    out[: 4 * B] = counts.tobytes()
    out[m0: m0 + 8 * W * B] = masks.astype("<u8").tobytes()
    out[m0 + 8 * W * B:] = vals.astype("<f8").tobytes()
    return bytes(out), codec, payload[body + 10:]


def frame_block(block, step_index: int = 0, sim_time: float = 0.0, elements_per_axis: int | None = None) -> bytes:
    """Wrap a CompressedBlock as a kind-1 frame with the SPEC.md:282 payload (the
    StageWriter::write_frame payload, proj/include/isf/staging/staging.hpp:59-60)."""
    E = elements_per_axis if elements_per_axis is not None else round(block.n_elements ** (1 / 3))
    payload = spec_payload(block.stream.detach().cpu().numpy(), block.n_elements, block.points_per_element_axis,
                           block.components, block.lossless_codec, block.coded_bytes)
    h = FrameHeader(KIND_COMPRESSED_BLOCK, step_index, sim_time, E, block.points_per_element_axis,
                    block.components, len(payload))
    return build_frame(h, payload)


def parse_block_frame(frame: bytes, n_elements: int | None = None):
    """A kind-1 frame back to (header, mask stream bytes, codec id, coded bytes);
    n_elements defaults to E^3 (a cubic mesh; slabs pass their element count)."""
    h, payload = parse_frame(frame)
    if h.kind != KIND_COMPRESSED_BLOCK:
        raise IsfError(ErrorCode.ShapeMismatch, "not a compressed-block frame")
    n_el = n_elements if n_elements is not None else h.elements_per_axis ** 3
    stream, codec, coded = stream_from_spec_payload(bytes(payload), n_el, h.points_per_element_axis, h.components)
    return h, stream, codec, coded
