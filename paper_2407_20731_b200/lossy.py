"""Python host API of the in-situ lossy-compression task (SPEC.md MODULE tasks).

Mirrors the reference's task interface for this path -- the same names,
argument meaning and error behaviour as SPEC.md:204-239 and the reference's
``isf::Error{ErrorCode}`` convention (proj/include/isf/core/errors.hpp:8-52) --
on top of the C ABI in include/isf_lossy.h.  PyTorch is used only to own device
memory and CUDA streams; all compute is the sm_100a kernels of libisf_lossy.so.

    cfg   = LossyConfig(max_error=1e-3)
    block = lossy_compress(field, cfg)
    back  = lossy_decompress(block, field.shape)
    back, rep = decompress_with_error(block, field.shape, field)   # L2 / Linf report
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field as dc_field
from enum import IntEnum

import numpy as np
import torch

from . import _native
from ._native import Stats

DEFAULT_DOMAIN_LENGTH = 2.0 * math.pi  # proj/include/isf/core/types.hpp:18


class ErrorCode(IntEnum):
    """proj/include/isf/core/errors.hpp:8-38 (same order, same values)."""
    BadMagic = 0
    UnsupportedVersion = 1
    LengthMismatch = 2
    ChecksumMismatch = 3
    SerializationFailed = 4
    ConnectFailed = 5
    VersionMismatch = 6
    InvalidCapacity = 7
    ReaderGone = 8
    WriterGone = 9
    StagingError = 10
    CalibrationFailed = 11
    ShapeMismatch = 12
    UnknownCodec = 13
    DegenerateRange = 14
    InvalidCadence = 15
    DegenerateSamples = 16
    TaskFailed = 17
    ConsumerCrashed = 18
    ConfigError = 19
    InvalidArgument = 20


class IsfError(RuntimeError):
    """``isf::Error``: message prefixed by the code name (errors.hpp:43-52)."""

    def __init__(self, code: ErrorCode, message: str):
        self.code = ErrorCode(code)
        prefix = f"{self.code.name}: "
        super().__init__(message if message.startswith(prefix) else prefix + message)


def _check(rc: int) -> None:
    if rc != 0:
        raise IsfError(ErrorCode(rc - 1), _native.last_error())


class ErrorNorm(IntEnum):
    """LossyConfig.error_norm."""
    RelativeL2 = 0
    RelativeLInf = 1


@dataclass(frozen=True)
class LossyConfig:
    """SPEC.md:204-207.  The transform is the per-element Legendre/GLL DLT (north_star).

    RelativeL2 bounds the error in the GLL-quadrature norm (sum of w_x w_y w_z v^2: the
    L2 norm of the element polynomials), which is the norm Parseval holds in for this
    transform; the plain point-sample relative L2 is bounded only up to
    sqrt(max w / min w) per element (tests/test_oracle_norms.py)."""
    max_error: float = 1e-2
    error_norm: ErrorNorm = ErrorNorm.RelativeL2

    def __post_init__(self):
        if not (0.0 < float(self.max_error) < 1.0):
            raise IsfError(ErrorCode.InvalidArgument,
                           f"LossyConfig: max_error must be in (0,1), got {self.max_error}")
        try:
            ErrorNorm(self.error_norm)
        except ValueError:
            raise IsfError(ErrorCode.InvalidArgument, f"LossyConfig: unknown error_norm {self.error_norm}") from None


@dataclass(frozen=True)
class CompressionReport:
    """cr == (original - compressed)/original in fp64 (Eq. 1)."""
    original_size: int
    compressed_size: int
    cr: float

    @staticmethod
    def from_sizes(original_size: int, compressed_size: int) -> "CompressionReport":
        cr = (float(original_size) - float(compressed_size)) / float(original_size)
        return CompressionReport(int(original_size), int(compressed_size), cr)


@dataclass
class Field:
    """proj/include/isf/core/types.hpp:20-66.  ``values`` is an fp64 tensor (device or
    host) of length elements * P^3 * components, element-major then point-major
    (px fastest) then component.  ``n_elements`` overrides E^3 for rank slabs."""
    elements_per_axis: int
    points_per_element_axis: int
    components: int
    values: torch.Tensor
    domain_length: float = DEFAULT_DOMAIN_LENGTH
    n_elements: int | None = None

    def __post_init__(self):
        self.validate_shape()

    def element_count(self) -> int:
        return self.n_elements if self.n_elements is not None else self.elements_per_axis ** 3

    def points_per_element(self) -> int:
        return self.points_per_element_axis ** 3

    def value_count(self) -> int:
        return self.element_count() * self.points_per_element() * self.components

    @property
    def shape(self) -> tuple:
        return (self.elements_per_axis, self.points_per_element_axis, self.components, self.element_count())

    def validate_shape(self) -> None:
        """Shape part of Field::validate (types.cpp:58-70); finiteness is checked by
        the compress kernel (fused flag -> InvalidArgument)."""
        if self.elements_per_axis < 1:
            raise IsfError(ErrorCode.InvalidArgument, "Field: elements_per_axis must be >= 1")
        if self.points_per_element_axis < 2:
            raise IsfError(ErrorCode.InvalidArgument, "Field: points_per_element_axis must be >= 2")
        if self.components not in (1, 3):
            raise IsfError(ErrorCode.InvalidArgument, "Field: components must be 1 or 3")
        if not (self.domain_length > 0.0):
            raise IsfError(ErrorCode.InvalidArgument, "Field: domain_length must be positive")
        if self.values.dtype != torch.float64:
            raise IsfError(ErrorCode.InvalidArgument, "Field: values must be float64")
        if self.values.numel() != self.value_count():
            raise IsfError(ErrorCode.InvalidArgument,
                           f"Field: values length {self.values.numel()} != expected {self.value_count()}")


@dataclass
class ErrorReport:
    """GLL-weighted relative L2 and relative Linf errors (north_star "L2/Linf")."""
    err2: float
    nrm2: float
    err_inf: float
    u_inf: float

    @property
    def rel_l2(self) -> float:
        if self.nrm2 == 0.0:
            return 0.0 if self.err2 == 0.0 else math.inf
        return math.sqrt(self.err2 / self.nrm2)

    @property
    def rel_linf(self) -> float:
        if self.u_inf == 0.0:
            return 0.0 if self.err_inf == 0.0 else math.inf
        return self.err_inf / self.u_inf


@dataclass
class CompressedBlock:
    """SPEC.md:208-211 in the mask + packed-value layout of include/isf_lossy.h.
    ``stream`` is a uint8 tensor (device) holding exactly ``compressed_size`` bytes."""
    stream: torch.Tensor
    n_elements: int
    points_per_element_axis: int
    components: int
    kept_total: int
    report: CompressionReport
    lossless_codec: int = 0
    coded_bytes: bytes = b""
    estimate: dict = dc_field(default_factory=dict)

    @property
    def nblocks(self) -> int:
        return self.n_elements * self.components

    def _parts(self):
        P = self.points_per_element_axis
        B = self.nblocks
        W = (P ** 3 + 63) // 64
        s = self.stream
        m0 = (4 * B + 15) & ~15
        counts = s[: 4 * B].view(torch.int32)
        masks = s[m0: m0 + 8 * W * B].view(torch.int64).reshape(B, W)
        vals = s[m0 + 8 * W * B:].view(torch.float64)
        return counts, masks, vals

    def kept_counts(self) -> torch.Tensor:
        return self._parts()[0]

    def masks(self) -> torch.Tensor:
        return self._parts()[1]

    def values(self) -> torch.Tensor:
        return self._parts()[2]

    def spec_payload(self) -> bytes:
        """SPEC.md:282 kind-1 payload: kept_count u32 per element | index u32 | value f64 |
        codec u16 | coded length u64 | coded bytes (indices are component*P^3 + j inside
        the element, derived from the masks; frame.spec_payload)."""
        from .frame import spec_payload
        return spec_payload(self.stream.detach().cpu().numpy(), self.n_elements, self.points_per_element_axis,
                            self.components, self.lossless_codec, self.coded_bytes)


class LossyPlan:
    """Owns an ``isf_lossy_plan`` (GLL operators in constant memory, look-back
    descriptors, reduction workspace) for one (device, P, components)."""

    def __init__(self, points_per_element_axis: int, components: int = 1, device: int | None = None):
        L = _native.lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = int(device)
        self.P = int(points_per_element_axis)
        self.components = int(components)
        h = ctypes.c_void_p()
        _check(L.isf_lossy_plan_create(ctypes.byref(h), self.P, self.components, self.device))
        self._h = h
        self._lib = L

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.isf_lossy_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def capacity(self, n_elements: int) -> int:
        return int(self._lib.isf_lossy_stream_capacity(self.P, self.components, n_elements))

    def header_bytes(self, n_elements: int) -> int:
        return int(self._lib.isf_lossy_stream_header_bytes(self.P, self.components, n_elements))

    def operators(self):
        n = self.P
        F = np.zeros((n, n)); B = np.zeros((n, n)); x = np.zeros(n); w = np.zeros(n)
        p = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        _check(self._lib.isf_lossy_plan_operators(self._h, p(F), p(B), p(x), p(w)))
        return F, B, x, w

    def last_launches(self) -> int:
        return int(self._lib.isf_lossy_plan_last_launches(self._h))

    TWO_PASS, SINGLE_PASS, AUTO = 0, 1, 2

    def set_compress_mode(self, mode: int) -> int:
        """lx = 8 compress schedule (isf_lossy_plan_set_compress_mode): TWO_PASS (slots +
        packing kernel), SINGLE_PASS (values written in place two rounds after their
        selection; faster for weakly compressible data) or AUTO (default: single-pass
        when the plan's last completed compress kept more than half of the
        coefficients).  Returns the previous mode; the streams are identical either way."""
        rc = int(self._lib.isf_lossy_plan_set_compress_mode(self._h, int(mode)))
        if rc < 0:
            raise IsfError(ErrorCode.InvalidArgument, f"unknown compress mode {mode}")
        return rc

    # ---- raw device entry points (bench / in-situ use) ----
    def compress_async(self, values: torch.Tensor, n_elements: int, max_error: float,
                       stream_buf: torch.Tensor, stats_buf: torch.Tensor, cuda_stream=None):
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        _check(self._lib.isf_lossy_compress_async(
            self._h, ctypes.c_void_p(values.data_ptr()), n_elements, float(max_error), 0,
            ctypes.c_void_p(stream_buf.data_ptr()), stream_buf.numel(),
            ctypes.c_void_p(stats_buf.data_ptr()), ctypes.c_void_p(cs.cuda_stream)))

    def crc32_async(self, data: torch.Tensor, nbytes: int, out: torch.Tensor, cuda_stream=None):
        """Device CRC-32 (zlib) of the first nbytes of a CUDA tensor into out (int32/uint32[1])."""
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        _check(self._lib.isf_lossy_crc32(self._h, ctypes.c_void_p(data.data_ptr()), int(nbytes),
                                         ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(cs.cuda_stream)))

    def frame_async(self, frame_buf: torch.Tensor, stream_buf: torch.Tensor, n_elements: int, stats_buf: torch.Tensor,
                    elements_per_axis: int, step_index: int = 0, sim_time: float = 0.0, cuda_stream=None):
        """Kind-1 frame with the SPEC.md:282 payload, converted on the device from the stream
        in stream_buf (stats_buf = that compress call's stats)."""
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        _check(self._lib.isf_lossy_frame_async(self._h, ctypes.c_void_p(frame_buf.data_ptr()), frame_buf.numel(),
                                               ctypes.c_void_p(stream_buf.data_ptr()), int(n_elements),
                                               ctypes.c_void_p(stats_buf.data_ptr()), int(elements_per_axis),
                                               int(step_index), float(sim_time), ctypes.c_void_p(cs.cuda_stream)))

    def frame_capacity(self, n_elements: int) -> int:
        return int(self._lib.isf_lossy_frame_capacity(self.P, self.components, n_elements))

    def decompress_async(self, stream_buf: torch.Tensor, stream_bytes: int, n_elements: int,
                         out: torch.Tensor, stats_buf: torch.Tensor, original: torch.Tensor | None = None,
                         cuda_stream=None):
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        _check(self._lib.isf_lossy_decompress_async(
            self._h, ctypes.c_void_p(stream_buf.data_ptr()), int(stream_bytes), n_elements,
            ctypes.c_void_p(out.data_ptr()),
            ctypes.c_void_p(original.data_ptr()) if original is not None else None,
            ctypes.c_void_p(stats_buf.data_ptr()), ctypes.c_void_p(cs.cuda_stream)))

    def compress_host(self, h_field: np.ndarray, n_elements: int, max_error: float, h_stream: np.ndarray):
        nb = ctypes.c_uint64()
        st = Stats()
        _check(self._lib.isf_lossy_compress_host(
            self._h, ctypes.c_void_p(h_field.ctypes.data), n_elements, float(max_error), 0,
            ctypes.c_void_p(h_stream.ctypes.data), h_stream.nbytes, ctypes.byref(nb), ctypes.byref(st)))
        return nb.value, st

    def decompress_host(self, h_stream: np.ndarray, stream_bytes: int, n_elements: int, h_out: np.ndarray,
                        h_original: np.ndarray | None = None):
        st = Stats()
        _check(self._lib.isf_lossy_decompress_host(
            self._h, ctypes.c_void_p(h_stream.ctypes.data), int(stream_bytes), n_elements,
            ctypes.c_void_p(h_out.ctypes.data),
            ctypes.c_void_p(h_original.ctypes.data) if h_original is not None else None,
            ctypes.byref(st)))
        return st

    def generate_tgv(self, out: torch.Tensor, E_ax: int, which: int, ez0: int = 0, nz: int | None = None,
                     domain: float = DEFAULT_DOMAIN_LENGTH, cuda_stream=None):
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        nz = E_ax if nz is None else nz
        _check(self._lib.isf_lossy_generate_tgv(self._h, ctypes.c_void_p(out.data_ptr()), E_ax, ez0, nz, which,
                                                float(domain), ctypes.c_void_p(cs.cuda_stream)))

    def generate_spectral(self, out: torch.Tensor, nblocks: int, block0: int, seed: int, amp: np.ndarray,
                          cuda_stream=None):
        cs = torch.cuda.current_stream(self.device) if cuda_stream is None else cuda_stream
        amp = np.ascontiguousarray(amp, dtype=np.float64)
        _check(self._lib.isf_lossy_generate_spectral(self._h, ctypes.c_void_p(out.data_ptr()), block0, nblocks,
                                                     seed, ctypes.c_void_p(amp.ctypes.data),
                                                     ctypes.c_void_p(cs.cuda_stream)))


_plans: dict = {}


def get_plan(P: int, components: int, device: int) -> LossyPlan:
    key = (int(P), int(components), int(device))
    if key not in _plans:
        _plans[key] = LossyPlan(P, components, device)
    return _plans[key]


def _device_values(field: Field) -> torch.Tensor:
    v = field.values
    if not v.is_cuda:
        v = v.cuda()
    if not v.is_contiguous():
        v = v.contiguous()
    if v.data_ptr() % 16:
        v = v.clone()
    return v


def lossy_compress(field: Field, cfg: LossyConfig, *, plan: LossyPlan | None = None) -> CompressedBlock:
    """SPEC.md:222-230 on the device.  Raises IsfError(InvalidArgument) for a
    non-finite value (types.cpp:71-73) or an invalid config."""
    field.validate_shape()
    v = _device_values(field)
    dev = v.device.index
    plan = plan or get_plan(field.points_per_element_axis, field.components, dev)
    n_el = field.element_count()
    cap = plan.capacity(n_el)
    buf = torch.empty(cap, dtype=torch.uint8, device=v.device)
    nb = ctypes.c_uint64()
    st = Stats()
    cs = torch.cuda.current_stream(dev)
    _check(plan._lib.isf_lossy_compress(plan.handle, ctypes.c_void_p(v.data_ptr()), n_el, float(cfg.max_error),
                                        int(cfg.error_norm), ctypes.c_void_p(buf.data_ptr()), cap,
                                        ctypes.byref(nb), ctypes.byref(st), ctypes.c_void_p(cs.cuda_stream)))
    rep = CompressionReport.from_sizes(st.field_bytes, nb.value)
    est = {"disc2": st.disc2, "tot2": st.tot2,
           "rel_l2_estimate": math.sqrt(st.disc2 / st.tot2) if st.tot2 > 0 else 0.0}
    # right-sized result: the worst-case capacity buffer (F + masks + counts) goes back
    # to the allocator instead of being kept alive by a view of its first C bytes
    return CompressedBlock(buf[: nb.value].clone(), n_el, field.points_per_element_axis, field.components,
                           int(st.kept), rep, estimate=est)


def lossy_compress_frame(field: Field, cfg: LossyConfig, step_index: int = 0, sim_time: float = 0.0, *,
                         plan: LossyPlan | None = None):
    """Compress and build a staging-ready kind-1 frame on the device:
    the SPEC.md:282 payload (kept_count u32 per element | index u32 | value f64 | codec
    trailer), header and CRC-32 are all written by kernels, so the only host work left
    is one D2H copy of the frame (StageWriter::write_frame,
    proj/include/isf/staging/staging.hpp:59-60).  Returns (frame uint8 CUDA tensor of
    exactly the frame bytes, CompressionReport of the stream, kept count)."""
    field.validate_shape()
    v = _device_values(field)
    dev = v.device.index
    plan = plan or get_plan(field.points_per_element_axis, field.components, dev)
    n_el = field.element_count()
    stream = torch.empty(plan.capacity(n_el), dtype=torch.uint8, device=v.device)
    frame = torch.empty(plan.frame_capacity(n_el), dtype=torch.uint8, device=v.device)
    stats = torch.zeros(12, dtype=torch.float64, device=v.device)
    cs = torch.cuda.current_stream(dev)
    _check(plan._lib.isf_lossy_compress_async(plan.handle, ctypes.c_void_p(v.data_ptr()), n_el,
                                              float(cfg.max_error), int(cfg.error_norm),
                                              ctypes.c_void_p(stream.data_ptr()), stream.numel(),
                                              ctypes.c_void_p(stats.data_ptr()), ctypes.c_void_p(cs.cuda_stream)))
    plan.frame_async(frame, stream, n_el, stats, field.elements_per_axis, step_index, sim_time, cuda_stream=cs)
    st = stats.view(torch.int64).cpu()
    status = int(st[10])
    if status & 1:
        raise IsfError(ErrorCode.InvalidArgument, "Field: non-finite value (types.cpp:71-73)")
    if status:
        raise IsfError(ErrorCode.SerializationFailed, f"frame assembly failed (status {status})")
    sb, kept = int(st[8]), int(st[6])
    rep = CompressionReport.from_sizes(int(st[9]), sb)
    return frame[: _native.FRAME_OVERHEAD + 4 * n_el + 12 * kept], rep, kept


def _decompress(block: CompressedBlock, shape, original: torch.Tensor | None):
    if shape is not None:
        E, P, C = shape[0], shape[1], shape[2]
        n_el = shape[3] if len(shape) > 3 else E ** 3
        if (P, C, n_el) != (block.points_per_element_axis, block.components, block.n_elements):
            raise IsfError(ErrorCode.ShapeMismatch,
                           f"block holds {block.n_elements} elements of P={block.points_per_element_axis} "
                           f"x{block.components}, requested shape {tuple(shape)}")
    else:
        E = round(block.n_elements ** (1 / 3))
    s = block.stream
    dev = s.device.index
    plan = get_plan(block.points_per_element_axis, block.components, dev)
    n = block.n_elements * block.points_per_element_axis ** 3 * block.components
    out = torch.empty(n, dtype=torch.float64, device=s.device)
    if s.data_ptr() % 16:
        s = s.clone()
    st = Stats()
    cs = torch.cuda.current_stream(dev)
    orig = None
    if original is not None:
        if original.dtype != torch.float64 or original.numel() != n:
            raise IsfError(ErrorCode.ShapeMismatch,
                           f"original: {original.numel()} {original.dtype} values, the block decodes to {n} float64")
        orig = original if original.is_cuda else original.cuda()
        orig = orig.contiguous()
        if orig.data_ptr() % 16:
            orig = orig.clone()
    _check(plan._lib.isf_lossy_decompress(plan.handle, ctypes.c_void_p(s.data_ptr()), s.numel(),
                                          block.n_elements, ctypes.c_void_p(out.data_ptr()),
                                          ctypes.c_void_p(orig.data_ptr()) if orig is not None else None,
                                          ctypes.byref(st), ctypes.c_void_p(cs.cuda_stream)))
    f = Field(E, block.points_per_element_axis, block.components, out,
              n_elements=None if E ** 3 == block.n_elements else block.n_elements)
    return f, st


def lossy_decompress(block: CompressedBlock, shape=None) -> Field:
    """SPEC.md:231-239.  ``shape`` = Field.shape of the original (E, P, components[, n_elements]);
    an inconsistent stream raises IsfError(ShapeMismatch)."""
    return _decompress(block, shape, None)[0]


def decompress_with_error(block: CompressedBlock, shape, original: Field | torch.Tensor):
    """Decompress and measure the GLL-weighted relative L2 and the relative Linf error
    against ``original`` in the same kernel."""
    ov = original.values if isinstance(original, Field) else original
    f, st = _decompress(block, shape, ov)
    return f, ErrorReport(st.err2, st.nrm2, st.err_inf, st.u_inf)


def compression_ratio(original_size: int, compressed_size: int) -> float:
    """Eq. 1 through the C ABI (bit-identical to CompressionReport.from_sizes)."""
    return float(_native.lib().isf_lossy_compression_ratio(original_size, compressed_size))
