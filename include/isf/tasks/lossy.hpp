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

/// SPEC.md:208-211.  `stream` is the device encoding of include/isf_lossy.h
/// (counts | masks | values) copied to the host; codec 0 / empty coded bytes
/// until a lossless stage runs on it.
struct CompressedBlock {
    std::uint32_t elements_per_axis = 0;
    std::uint32_t points_per_element_axis = 0;
    std::uint32_t components = 0;
    std::uint64_t n_elements = 0;
    std::uint64_t kept_total = 0;
    Bytes stream;
    std::uint16_t lossless_codec = 0;
    Bytes coded_bytes;
    CompressionReport report;

    /// kind-1 payload (SPEC.md:282 codec trailer appended to the stream)
    Bytes payload() const {
        Bytes out(stream);
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

/// Device-resident kind-1 frame: compresses straight into
/// d_frame + 48 and writes header, codec trailer and CRC-32 on the device
/// (isf_lossy_frame_async).  d_frame holds stream capacity + ISF_FRAME_OVERHEAD
/// bytes; the frame is d_stats->stream_bytes + ISF_FRAME_OVERHEAD bytes long.
inline void lossy_compress_frame_device(const double* d_field, std::uint64_t n_elements, std::uint32_t E_ax,
                                        std::uint32_t P, std::uint32_t comps, const LossyConfig& cfg,
                                        void* d_frame, std::uint64_t frame_cap, isf_lossy_stats* d_stats,
                                        std::uint64_t step_index, double sim_time, cudaStream_t stream) {
    cfg.validate();
    auto* plan = detail::plan_for(P, comps);
    detail::check(isf_lossy_compress_async(plan, d_field, n_elements, cfg.max_error,
                                           static_cast<int>(cfg.error_norm), static_cast<char*>(d_frame) + 48,
                                           frame_cap - 48, d_stats, stream));
    detail::check(isf_lossy_frame_async(plan, d_frame, frame_cap, d_stats, E_ax, step_index, sim_time, stream));
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
        isf_lossy_stats* stats = nullptr;
        std::byte* pinned = nullptr;  // page-locked staging of the frame (full-speed D2H)
        std::uint64_t pinned_cap = 0;
        ~Bufs() { cudaFree(frame); cudaFree(stats); cudaFreeHost(pinned); }
    };
    thread_local Bufs b;
    const std::uint64_t cap = isf_lossy_stream_capacity(P, comps, n_elements) + ISF_FRAME_OVERHEAD;
    if (cap > b.cap) {
        cudaFree(b.frame);
        b.frame = nullptr;
        if (cudaMalloc(&b.frame, cap) != cudaSuccess) throw Error(ErrorCode::TaskFailed, "cudaMalloc frame");
        b.cap = cap;
    }
    if (!b.stats && cudaMalloc(&b.stats, sizeof(isf_lossy_stats)) != cudaSuccess)
        throw Error(ErrorCode::TaskFailed, "cudaMalloc stats");
    lossy_compress_frame_device(d_field, n_elements, E_ax, P, comps, cfg, b.frame, b.cap, b.stats, step_index,
                                sim_time, stream);
    isf_lossy_stats st{};
    if (cudaMemcpyAsync(&st, b.stats, sizeof st, cudaMemcpyDeviceToHost, stream) != cudaSuccess ||
        cudaStreamSynchronize(stream) != cudaSuccess)
        throw Error(ErrorCode::TaskFailed, "frame statistics copy failed");
    if (st.status & ISF_STATUS_NONFINITE) throw Error(ErrorCode::InvalidArgument, "Field: non-finite value");
    if (st.status) throw Error(ErrorCode::SerializationFailed, "frame assembly failed");
    const std::uint64_t fbytes = st.stream_bytes + ISF_FRAME_OVERHEAD;
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

/// Length of the stream at the front of a kind-1 payload: its header plus 8 bytes
/// per stored value (the counts say how many); the SPEC.md:282 codec trailer follows.
inline std::size_t kind1_stream_bytes(std::span<const std::byte> payload, const FrameHeader& h,
                                      std::uint64_t n_elements) {
    if (payload.size() < 10) throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its trailer");
    const std::uint64_t B = n_elements * h.components;
    const std::uint64_t hdr = isf_lossy_stream_header_bytes(h.points_per_element_axis, h.components, n_elements);
    if (payload.size() < hdr + 10) throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its header");
    std::uint64_t total = 0;
    for (std::uint64_t i = 0; i < B; ++i) {
        std::uint32_t c = 0;
        std::memcpy(&c, payload.data() + 4 * i, 4);
        total += c;
    }
    const std::size_t sb = hdr + 8 * total;
    if (payload.size() < sb + 10) throw Error(ErrorCode::LengthMismatch, "kind-1 payload shorter than its stream");
    std::uint64_t coded = 0;
    std::memcpy(&coded, payload.data() + sb + 2, 8);
    if (sb + 10 + coded != payload.size()) throw Error(ErrorCode::LengthMismatch, "kind-1 payload length mismatch");
    return sb;
}

/// Inverse of CompressedBlock::payload(): a block from a kind-1 payload (the
/// stream is everything before the SPEC.md:282 codec trailer).  keep_stream = false
/// leaves the stream out (metadata, codec trailer and report only).
inline CompressedBlock block_from_payload(std::span<const std::byte> payload, const FrameHeader& h,
                                          std::uint64_t n_elements, bool keep_stream = true) {
    CompressedBlock b;
    b.elements_per_axis = h.elements_per_axis;
    b.points_per_element_axis = h.points_per_element_axis;
    b.components = h.components;
    b.n_elements = n_elements;
    const std::size_t sb = kind1_stream_bytes(payload, h, n_elements);
    std::uint64_t coded = 0;
    std::memcpy(&coded, payload.data() + sb + 2, 8);
    if (keep_stream) b.stream.assign(payload.begin(), payload.begin() + sb);
    b.lossless_codec = std::uint16_t(std::to_integer<std::uint8_t>(payload[sb])) |
                       std::uint16_t(std::uint16_t(std::to_integer<std::uint8_t>(payload[sb + 1])) << 8);
    b.coded_bytes.assign(payload.begin() + sb + 10, payload.begin() + sb + 10 + coded);
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
