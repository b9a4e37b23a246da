"""ISF1 core frame around a compressed block (payload_kind = 1).

Byte-compatible with the reference's framing (proj/include/isf/core/frame.hpp:3-11,
proj/src/core/frame.cpp:9-71): little-endian 48-byte header
``"ISF1" | version u16 = 1 | payload_kind u16 | step u64 | sim_time f64 | E u32 |
P u32 | components u32 | reserved u32 = 0 | payload_len u64`` followed by the payload
and an IEEE CRC-32 (zlib polynomial) of header + payload.  Errors mirror
parse_frame / parse_frame_header (BadMagic, UnsupportedVersion, LengthMismatch,
ChecksumMismatch).  The payload of a kind-1 frame produced here is the device
stream of include/isf_lossy.h followed by SPEC.md:282's codec trailer
(codec id u16 | coded length u64 | coded bytes), see DESIGN.md 3.5.
"""
from __future__ import annotations

import struct
import zlib
from dataclasses import dataclass

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


def block_payload(stream: bytes, codec: int = 0, coded: bytes = b"") -> bytes:
    """Kind-1 payload: device stream | codec id u16 | coded length u64 | coded bytes."""
    return bytes(stream) + struct.pack("<HQ", codec, len(coded)) + bytes(coded)


def split_block_payload(payload: bytes, stream_len: int):
    if len(payload) < stream_len + 10:
        raise IsfError(ErrorCode.LengthMismatch, "payload shorter than stream + codec trailer")
    codec, n = struct.unpack_from("<HQ", payload, stream_len)
    coded = payload[stream_len + 10: stream_len + 10 + n]
    if len(coded) != n or stream_len + 10 + n != len(payload):
        raise IsfError(ErrorCode.LengthMismatch, "codec trailer length mismatch")
    return payload[:stream_len], codec, coded


def frame_block(block, step_index: int = 0, sim_time: float = 0.0, elements_per_axis: int | None = None) -> bytes:
    """Wrap a CompressedBlock as a kind-1 frame (the StageWriter::write_frame payload,
    proj/include/isf/staging/staging.hpp:59-60)."""
    E = elements_per_axis if elements_per_axis is not None else round(block.n_elements ** (1 / 3))
    stream = block.stream.detach().cpu().numpy().tobytes()
    payload = block_payload(stream, block.lossless_codec, block.coded_bytes)
    h = FrameHeader(KIND_COMPRESSED_BLOCK, step_index, sim_time, E, block.points_per_element_axis,
                    block.components, len(payload))
    return build_frame(h, payload)
