#pragma once

// isf/tasks/lossy.hpp -- the in-situ lossy-compression task of the reference
// framework, the header that proj/include/isf/core/frame.hpp:11 refers to
// ("payload_kind 1 carries a compressed block (see tasks/lossy.hpp)") but that
// the reference never shipped.  Header-only C++ host API with the SPEC.md
// signatures and the reference's conventions (owned values, isf::Error with an
// isf::ErrorCode, proj/include/isf/core/errors.hpp:43-52), implemented by the
// B200 kernels behind the C ABI of include/isf_lossy.h (libisf_lossy.so).
//
//   SPEC.md:204-207  LossyConfig          SPEC.md:212-215  CompressionReport (Eq. 1)
//   SPEC.md:208-211  CompressedBlock      SPEC.md:222-230  lossy_compress
//   SPEC.md:231-239  lossy_decompress     SPEC.md:282      kind-1 frame payload
//
// Drop-in: put this file at proj/include/isf/tasks/lossy.hpp, add include/ to the
// include path and link libisf_lossy.so.  The transform is the
// per-element Legendre/GLL DLT of north_star (SPEC.md:205 says DCT-II).

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <memory>
#include <vector>

#include <cuda_runtime.h>

#include "isf/core/errors.hpp"
#include "isf/core/frame.hpp"
#include "isf/core/types.hpp"
#include "isf_lossy.h"

namespace isf::tasks {

enum class ErrorNorm { RelativeL2 = ISF_NORM_RELATIVE_L2, RelativeLInf = ISF_NORM_RELATIVE_LINF };

struct LossyConfig {
    // SPEC.md:205 paper value.  RelativeL2 bounds the GLL-quadrature (polynomial) L2
    // norm of the error per block, not the plain point-sample norm (isf_lossy.h,
    // DESIGN.md 3.8).
    double max_error = 1e-2;
    ErrorNorm error_norm = ErrorNorm::RelativeL2;

    void validate() const {
        if (!(max_error > 0.0 && max_error < 1.0))
            throw Error(ErrorCode::InvalidArgument, "LossyConfig: max_error must be in (0,1)");
        if (error_norm != ErrorNorm::RelativeL2 && error_norm != ErrorNorm::RelativeLInf)
            throw Error(ErrorCode::InvalidArgument, "LossyConfig: unknown error_norm");
    }
};

struct CompressionReport {
    std::uint64_t original_size = 0;
    std::uint64_t compressed_size = 0;
    double cr = 0.0;  // == (original - compressed) / original in fp64 (Eq. 1)

    static CompressionReport from_sizes(std::uint64_t orig, std::uint64_t comp) {
        return {orig, comp, isf_lossy_compression_ratio(orig, comp)};
    }
};

struct ErrorReport {
    double err2 = 0, nrm2 = 0, err_inf = 0, u_inf = 0;
    double rel_l2() const { return nrm2 == 0.0 ? (err2 == 0.0 ? 0.0 : 1.0 / 0.0) : __builtin_sqrt(err2 / nrm2); }
    double rel_linf() const { return u_inf == 0.0 ? (err_inf == 0.0 ? 0.0 : 1.0 / 0.0) : err_inf / u_inf; }
};

namespace detail {
/// SPEC.md:282 payload body (kept_count u32 per element | index u32 | value f64, index =
/// component * P^3 + j ascending inside the element) from the mask stream; the host
/// restatement of the device conversion (csrc/crc32.cuh spec_frame_kernel).
inline Bytes spec_body_from_stream(std::span<const std::byte> stream, std::uint64_t n_el, std::uint32_t P,
                                   std::uint32_t comps) {
    const std::uint64_t P3 = std::uint64_t(P) * P * P, W = (P3 + 63) / 64, B = n_el * comps;
    const std::uint64_t m0 = (4 * B + 15) & ~std::uint64_t(15), v0 = m0 + 8 * W * B;
    if (stream.size() < v0) throw Error(ErrorCode::ShapeMismatch, "stream shorter than its header");
    const std::uint64_t K = (stream.size() - v0) / 8;
    Bytes out(4 * n_el + 12 * K);
    std::uint64_t k = 0;
    for (std::uint64_t e = 0; e < n_el; ++e) {
        std::uint32_t ce = 0;
        for (std::uint32_t c = 0; c < comps; ++c) {
            const std::uint64_t b = e * comps + c;
            std::uint32_t cnt;
            std::memcpy(&cnt, stream.data() + 4 * b, 4);
            ce += cnt;
            for (std::uint64_t w = 0; w < W; ++w) {
                std::uint64_t m;
                std::memcpy(&m, stream.data() + m0 + 8 * (b * W + w), 8);
                for (; m; m &= m - 1) {
                    if (k >= K) throw Error(ErrorCode::ShapeMismatch, "stream masks exceed its values");
                    const std::uint32_t idx = std::uint32_t(c * P3 + 64 * w + std::uint64_t(__builtin_ctzll(m)));
                    std::memcpy(out.data() + 4 * n_el + 4 * k, &idx, 4);
                    ++k;
                }
            }
        }
        std::memcpy(out.data() + 4 * e, &ce, 4);
    }
    if (k != K) throw Error(ErrorCode::ShapeMismatch, "stream masks and values disagree");
    std::memcpy(out.data() + 4 * n_el + 4 * K, stream.data() + v0, 8 * K);
    return out;
}
/// Inverse: the mask stream from a SPEC.md:282 payload body (ShapeMismatch when the
/// indices are out of range or not ascending inside an element).
inline Bytes stream_from_spec_body(std::span<const std::byte> body, std::uint64_t n_el, std::uint32_t P,
                                   std::uint32_t comps) {
    const std::uint64_t P3 = std::uint64_t(P) * P * P, W = (P3 + 63) / 64, B = n_el * comps;
    if (body.size() < 4 * n_el) throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its counts");
    std::uint64_t K = 0;
    for (std::uint64_t e = 0; e < n_el; ++e) {
        std::uint32_t c;
        std::memcpy(&c, body.data() + 4 * e, 4);
        K += c;
    }
    if (body.size() != 4 * n_el + 12 * K) throw Error(ErrorCode::LengthMismatch, "kind-1 payload body length");
    const std::uint64_t m0 = (4 * B + 15) & ~std::uint64_t(15), v0 = m0 + 8 * W * B;
    Bytes out(v0 + 8 * K, std::byte{0});
    std::uint64_t k = 0;
    for (std::uint64_t e = 0; e < n_el; ++e) {
        std::uint32_t ce;
        std::memcpy(&ce, body.data() + 4 * e, 4);
        std::int64_t prev = -1;
        for (std::uint32_t q = 0; q < ce; ++q, ++k) {
            std::uint32_t idx;
            std::memcpy(&idx, body.data() + 4 * n_el + 4 * k, 4);
            if (idx >= comps * P3 || std::int64_t(idx) <= prev)
                throw Error(ErrorCode::ShapeMismatch, "kind-1 payload: index out of range or not ascending");
            prev = idx;
            const std::uint64_t b = e * comps + idx / P3, j = idx % P3;
            std::uint32_t cnt;
            std::memcpy(&cnt, out.data() + 4 * b, 4);
            ++cnt;
            std::memcpy(out.data() + 4 * b, &cnt, 4);
            std::uint64_t m;
            std::memcpy(&m, out.data() + m0 + 8 * (b * W + j / 64), 8);
            m |= std::uint64_t(1) << (j % 64);
            std::memcpy(out.data() + m0 + 8 * (b * W + j / 64), &m, 8);
        }
    }
    std::memcpy(out.data() + v0, body.data() + 4 * n_el + 4 * K, 8 * K);
    return out;
}
}  // namespace detail

/// SPEC.md:208-211.  `stream` is the device encoding of include/isf_lossy.h
/// (counts | masks | values) copied to the host; codec 0 / empty coded bytes
/// until a lossless stage runs.  The kind-1 payload it frames as
/// is SPEC.md:282's (payload()).
struct CompressedBlock {
    std::uint32_t elements_per_axis = 0;
    std::uint32_t points_per_element_axis = 0;
    std::uint32_t components = 0;
    std::uint64_t n_elements = 0;
    std::uint64_t kept_total = 0;
    Bytes stream;
    std::uint16_t lossless_codec = 0;
    Bytes coded_bytes;
    std::uint64_t coded_source_bytes = 0;  // bytes the lossless codec coded (the SPEC payload body)
    CompressionReport report;

    /// SPEC.md:282 kind-1 payload: kept_count u32 per element | index u32 | value f64 |
    /// codec id u16 | coded length u64 | coded bytes
    Bytes payload() const {
        Bytes out = detail::spec_body_from_stream(stream, n_elements, points_per_element_axis, components);
        put_u16(out, lossless_codec);
        put_u64(out, coded_bytes.size());
        out.insert(out.end(), coded_bytes.begin(), coded_bytes.end());
        return out;
    }
    /// core frame with payload_kind = 1, ready for StageWriter::write_frame
    Bytes frame(std::uint64_t step_index = 0, double sim_time = 0.0) const {
        FrameHeader h;
        h.kind = PayloadKind::CompressedBlock;
        h.step_index = step_index;
        h.sim_time = sim_time;
        h.elements_per_axis = elements_per_axis;
        h.points_per_element_axis = points_per_element_axis;
        h.components = components;
        auto p = payload();
        h.payload_len = p.size();
        return build_frame(h, p);
    }
};

namespace detail {
inline void check(int rc) {
    if (rc != 0) throw Error(static_cast<ErrorCode>(rc - 1), isf_lossy_last_error());
}
/// One plan per (device, P, components), created on first use on this thread.
class Plan {
  public:
    Plan(std::uint32_t P, std::uint32_t comps, int device) { check(isf_lossy_plan_create(&p_, P, comps, device)); }
    ~Plan() { isf_lossy_plan_destroy(p_); }
    Plan(const Plan&) = delete;
    Plan& operator=(const Plan&) = delete;
    isf_lossy_plan* get() const { return p_; }

  private:
    isf_lossy_plan* p_ = nullptr;
};
inline isf_lossy_plan* plan_for(std::uint32_t P, std::uint32_t comps) {
    int dev = 0;
    cudaGetDevice(&dev);
    struct Key { std::uint32_t P, c; int d; };
    // owned by the thread: destroyed (isf_lossy_plan_destroy) when the thread exits
    thread_local std::vector<std::pair<Key, std::unique_ptr<Plan>>> plans;
    for (auto& kv : plans)
        if (kv.first.P == P && kv.first.c == comps && kv.first.d == dev) return kv.second->get();
    plans.emplace_back(Key{P, comps, dev}, std::make_unique<Plan>(P, comps, dev));
    return plans.back().second->get();
}
}  // namespace detail

/// compress a host Field (H2D, kernels, D2H inside the call).
inline CompressedBlock lossy_compress(const Field& f, const LossyConfig& cfg) {
    f.validate();
    cfg.validate();
    auto* plan = detail::plan_for(f.points_per_element_axis, f.components);
    CompressedBlock b;
    b.elements_per_axis = f.elements_per_axis;
    b.points_per_element_axis = f.points_per_element_axis;
    b.components = f.components;
    b.n_elements = f.element_count();
    const std::uint64_t cap = isf_lossy_stream_capacity(f.points_per_element_axis, f.components, b.n_elements);
    // worst-case scratch without value-initialisation (F + masks + counts), then a
    // right-sized owned copy of the C bytes actually produced
    std::unique_ptr<std::byte[]> scratch(new std::byte[cap]);
    std::uint64_t n = 0;
    isf_lossy_stats st{};
    detail::check(isf_lossy_compress_host(plan, f.values.data(), b.n_elements, cfg.max_error,
                                          static_cast<int>(cfg.error_norm), scratch.get(), cap, &n, &st));
    b.stream.assign(scratch.get(), scratch.get() + n);
    b.kept_total = st.kept;
    b.report = CompressionReport::from_sizes(st.field_bytes, n);
    return b;
}

/// decompress to a host Field of the original shape.
inline Field lossy_decompress(const CompressedBlock& b, const Field& shape, ErrorReport* report = nullptr,
                              const Field* original = nullptr) {
    if (b.points_per_element_axis != shape.points_per_element_axis || b.components != shape.components ||
        b.n_elements != shape.element_count())
        throw Error(ErrorCode::ShapeMismatch, "compressed block does not match the requested field shape");
    if (original && original->values.size() != shape.value_count())
        throw Error(ErrorCode::ShapeMismatch, "original field does not match the requested field shape");
    auto* plan = detail::plan_for(b.points_per_element_axis, b.components);
    std::vector<double> out(shape.value_count());
    isf_lossy_stats st{};
    detail::check(isf_lossy_decompress_host(plan, b.stream.data(), b.stream.size(), b.n_elements, out.data(),
                                            original ? original->values.data() : nullptr, &st));
    if (report) *report = ErrorReport{st.err2, st.nrm2, st.err_inf, st.u_inf};
    return Field(shape.elements_per_axis, shape.points_per_element_axis, shape.components, std::move(out),
                 shape.domain_length);
}

/// Device-resident in-situ use (the field already lives in HBM): asynchronous on
/// `stream`; the field must not be overwritten until the work completed
/// (handoff rule, proj/include/isf/staging/staging.hpp:5-9).
inline void lossy_compress_device(const double* d_field, std::uint64_t n_elements, std::uint32_t P,
                                  std::uint32_t comps, const LossyConfig& cfg, void* d_stream,
                                  std::uint64_t capacity, isf_lossy_stats* d_stats, cudaStream_t stream) {
    cfg.validate();
    detail::check(isf_lossy_compress_async(detail::plan_for(P, comps), d_field, n_elements, cfg.max_error,
                                           static_cast<int>(cfg.error_norm), d_stream, capacity, d_stats, stream));
}

/// Device-resident kind-1 frame: compresses into d_stream, then
/// converts it on the device into the SPEC.md:282 payload and writes header, codec
/// trailer and CRC-32 (isf_lossy_frame_async).  d_frame holds
/// isf_lossy_frame_capacity bytes; the frame is ISF_FRAME_OVERHEAD + 4 n_elements +
/// 12 d_stats->kept bytes long.
inline void lossy_compress_frame_device(const double* d_field, std::uint64_t n_elements, std::uint32_t E_ax,
                                        std::uint32_t P, std::uint32_t comps, const LossyConfig& cfg,
                                        void* d_stream, std::uint64_t stream_cap, void* d_frame,
                                        std::uint64_t frame_cap, isf_lossy_stats* d_stats, std::uint64_t step_index,
                                        double sim_time, cudaStream_t stream) {
    cfg.validate();
    auto* plan = detail::plan_for(P, comps);
    detail::check(isf_lossy_compress_async(plan, d_field, n_elements, cfg.max_error,
                                           static_cast<int>(cfg.error_norm), d_stream, stream_cap, d_stats, stream));
    detail::check(isf_lossy_frame_async(plan, d_frame, frame_cap, d_stream, n_elements, d_stats, E_ax, step_index,
                                        sim_time, stream));
}

/// Synchronous prefix of the hybrid mode (SPEC.md run_hybrid):
/// the device frame copied to an owned host frame for StageWriter::write_frame
/// (staging.hpp:59-60).  Only the compressed frame crosses PCIe.
inline Bytes lossy_compress_frame(const double* d_field, std::uint64_t n_elements, std::uint32_t E_ax,
                                  std::uint32_t P, std::uint32_t comps, const LossyConfig& cfg,
                                  std::uint64_t step_index = 0, double sim_time = 0.0,
                                  cudaStream_t stream = nullptr) {
    struct Bufs {
        void* frame = nullptr;
        std::uint64_t cap = 0;
        void* stream = nullptr;
        std::uint64_t scap = 0;
        isf_lossy_stats* stats = nullptr;
        std::byte* pinned = nullptr;  // page-locked staging of the frame (full-speed D2H)
        std::uint64_t pinned_cap = 0;
        ~Bufs() { cudaFree(frame); cudaFree(stream); cudaFree(stats); cudaFreeHost(pinned); }
    };
    thread_local Bufs b;
    const std::uint64_t cap = isf_lossy_frame_capacity(P, comps, n_elements);
    const std::uint64_t scap = isf_lossy_stream_capacity(P, comps, n_elements);
    if (cap > b.cap) {
        cudaFree(b.frame);
        b.frame = nullptr;
        if (cudaMalloc(&b.frame, cap) != cudaSuccess) throw Error(ErrorCode::TaskFailed, "cudaMalloc frame");
        b.cap = cap;
    }
    if (scap > b.scap) {
        cudaFree(b.stream);
        b.stream = nullptr;
        if (cudaMalloc(&b.stream, scap) != cudaSuccess) throw Error(ErrorCode::TaskFailed, "cudaMalloc stream");
        b.scap = scap;
    }
    if (!b.stats && cudaMalloc(&b.stats, sizeof(isf_lossy_stats)) != cudaSuccess)
        throw Error(ErrorCode::TaskFailed, "cudaMalloc stats");
    lossy_compress_frame_device(d_field, n_elements, E_ax, P, comps, cfg, b.stream, b.scap, b.frame, b.cap, b.stats,
                                step_index, sim_time, stream);
    isf_lossy_stats st{};
    if (cudaMemcpyAsync(&st, b.stats, sizeof st, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        throw Error(ErrorCode::TaskFailed, "frame statistics copy failed");
    if (st.status & ISF_STATUS_NONFINITE) throw Error(ErrorCode::InvalidArgument, "Field: non-finite value");
    if (st.status) throw Error(ErrorCode::SerializationFailed, "frame assembly failed");
    const std::uint64_t fbytes = ISF_FRAME_OVERHEAD + 4 * n_elements + 12 * st.kept;
    if (fbytes > b.pinned_cap) {  // grows (x1.5 headroom) with the frames seen, not to the capacity bound
        cudaFreeHost(b.pinned);
        b.pinned = nullptr;
        b.pinned_cap = 0;
        const std::uint64_t want = std::min<std::uint64_t>(b.cap, fbytes + fbytes / 2);
        if (cudaMallocHost(reinterpret_cast<void**>(&b.pinned), want) != cudaSuccess)
            throw Error(ErrorCode::TaskFailed, "cudaMallocHost frame staging");
        b.pinned_cap = want;
    }
    if (cudaMemcpyAsync(b.pinned, b.frame, fbytes, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        throw Error(ErrorCode::TaskFailed, "frame copy failed");
    return Bytes(b.pinned, b.pinned + fbytes);  // the owned frame StageWriter::write_frame takes
}

/// Length of the SPEC.md:282 body (counts, indices, values) at the front of a kind-1
/// payload; the codec trailer (codec id u16 | coded length u64 | coded) follows.
inline std::size_t kind1_body_bytes(std::span<const std::byte> payload, std::uint64_t n_elements) {
    if (payload.size() < 4 * n_elements + 10)
        throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its counts + codec trailer");
    std::uint64_t K = 0;
    for (std::uint64_t e = 0; e < n_elements; ++e) {
        std::uint32_t c = 0;
        std::memcpy(&c, payload.data() + 4 * e, 4);
        K += c;
    }
    const std::size_t body = 4 * n_elements + 12 * K;
    if (payload.size() < body + 10) throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its arrays");
    std::uint64_t coded = 0;
    std::memcpy(&coded, payload.data() + body + 2, 8);
    if (body + 10 + coded != payload.size()) throw Error(ErrorCode::LengthMismatch, "kind-1 payload length mismatch");
    return body;
}

/// Inverse of CompressedBlock::payload(): a block from a kind-1 payload (SPEC.md:282
/// body converted back into the mask stream).  keep_stream = false leaves the stream
/// out (metadata, codec trailer and report only).
inline CompressedBlock block_from_payload(std::span<const std::byte> payload, const FrameHeader& h,
                                          std::uint64_t n_elements, bool keep_stream = true) {
    CompressedBlock b;
    b.elements_per_axis = h.elements_per_axis;
    b.points_per_element_axis = h.points_per_element_axis;
    b.components = h.components;
    b.n_elements = n_elements;
    const std::size_t body = kind1_body_bytes(payload, n_elements);
    std::uint64_t coded = 0;
    std::memcpy(&coded, payload.data() + body + 2, 8);
    b.kept_total = (body - 4 * n_elements) / 12;
    const std::uint64_t W = (std::uint64_t(h.points_per_element_axis) * h.points_per_element_axis *
                                 h.points_per_element_axis + 63) / 64;
    const std::uint64_t B = n_elements * h.components;
    const std::uint64_t sb = ((4 * B + 15) & ~std::uint64_t(15)) + 8 * W * B + 8 * b.kept_total;
    if (keep_stream)
        b.stream = detail::stream_from_spec_body(payload.first(body), n_elements, h.points_per_element_axis,
                                                 h.components);
    b.lossless_codec = std::uint16_t(std::to_integer<std::uint8_t>(payload[body])) |
                       std::uint16_t(std::uint16_t(std::to_integer<std::uint8_t>(payload[body + 1])) << 8);
    b.coded_bytes.assign(payload.begin() + body + 10, payload.begin() + body + 10 + coded);
    b.report = CompressionReport::from_sizes(n_elements * h.points_per_element_axis * h.points_per_element_axis *
                                                 h.points_per_element_axis * h.components * 8,
                                             sb);
    return b;
}

inline void lossy_decompress_device(const void* d_stream, std::uint64_t stream_bytes, std::uint64_t n_elements,
                                    std::uint32_t P, std::uint32_t comps, double* d_out, const double* d_original,
                                    isf_lossy_stats* d_stats, cudaStream_t stream) {
    detail::check(isf_lossy_decompress_async(detail::plan_for(P, comps), d_stream, stream_bytes, n_elements, d_out,
                                             d_original, d_stats, stream));
}

}  // namespace isf::tasks
