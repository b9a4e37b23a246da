#pragma once

// isf/tasks/lossless.hpp -- the lossless stage of the reference framework's task
// chain (SPEC.md:240-248 lossless_encode / decode, codec ids pluggable) and the
// asynchronous suffix of the hybrid mode (SPEC.md:318-321 run_hybrid; PAPER.md:
// 277-278): a consumer that reads the kind-1 frames the synchronous device prefix
// staged (reference StageReader, proj/include/isf/staging/staging.hpp:78-95, CRC
// validated) and lossless-codes each block's stream on a pool of host threads.
//
// Header-only, compiled with the reference core + staging sources and zlib (the
// reference's own dependency, proj/CMakeLists.txt:14).  Codec ids: 0 none, 1 RLE,
// 2 Deflate (one zlib stream, level 6), 3 chunked Deflate (the stream cut into
// 1 MiB chunks deflated in parallel at level 1; coded = u32 n | u64 chunk size |
// n x u64 coded length | chunks), which is what lets one CPU suffix keep up with a
// B200 prefix.

#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <functional>
#include <span>
#include <thread>
#include <vector>

#include "isf/core/bytes.hpp"
#include "isf/core/errors.hpp"
#include "isf/staging/staging.hpp"
#include "isf/tasks/lossy.hpp"

namespace isf::tasks {

enum class LosslessCodec : std::uint16_t { None = 0, Rle = 1, Deflate = 2, DeflateChunked = 3 };

struct LosslessResult {
    Bytes coded;
    CompressionReport report;  // Eq. 1 over (input bytes, coded bytes)
};

namespace detail {
inline void put64(Bytes& b, std::size_t at, std::uint64_t v) { std::memcpy(b.data() + at, &v, 8); }
inline std::uint64_t get64(std::span<const std::byte> b, std::size_t at) {
    std::uint64_t v;
    std::memcpy(&v, b.data() + at, 8);
    return v;
}
inline int pool_size(int threads) {
    if (threads > 0) return threads;
    const unsigned h = std::thread::hardware_concurrency();
    return h ? int(h) : 1;
}
// run f(i) for i in [0, n) on up to `threads` threads (the caller's thread included)
inline void parallel_for(std::size_t n, int threads, const std::function<void(std::size_t)>& f) {
    const int t = std::max(1, std::min<int>(pool_size(threads), int(n)));
    std::atomic<std::size_t> next{0};
    auto work = [&] {
        for (std::size_t i; (i = next.fetch_add(1)) < n;) f(i);
    };
    std::vector<std::thread> pool;
    for (int k = 1; k < t; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
}
inline std::size_t deflate_into(std::span<const std::byte> in, Bytes& out, int level) {
    uLongf len = compressBound(in.size());
    out.resize(len);
    if (compress2(reinterpret_cast<Bytef*>(out.data()), &len, reinterpret_cast<const Bytef*>(in.data()), in.size(),
                  level) != Z_OK)
        throw Error(ErrorCode::SerializationFailed, "zlib deflate failed");
    out.resize(len);
    return len;
}
inline void inflate_exact(std::span<const std::byte> in, std::byte* out, std::size_t n) {
    uLongf len = n;
    if (uncompress(reinterpret_cast<Bytef*>(out), &len, reinterpret_cast<const Bytef*>(in.data()), in.size()) != Z_OK ||
        len != n)
        throw Error(ErrorCode::SerializationFailed, "zlib inflate failed");
}
constexpr std::size_t kChunk = std::size_t(1) << 20;
}  // namespace detail

/// codec output + Eq. 1 report; UnknownCodec for an unregistered id.
inline LosslessResult lossless_encode(std::span<const std::byte> in, LosslessCodec codec, int threads = 0) {
    Bytes out;
    switch (codec) {
        case LosslessCodec::None:
            out.assign(in.begin(), in.end());
            break;
        case LosslessCodec::Rle:  // (run length u8 1..255, byte) pairs
            out.reserve(in.size() / 8 + 16);
            for (std::size_t i = 0; i < in.size();) {
                std::size_t j = i + 1;
                while (j < in.size() && j - i < 255 && in[j] == in[i]) ++j;
                out.push_back(std::byte(j - i));
                out.push_back(in[i]);
                i = j;
            }
            break;
        case LosslessCodec::Deflate:
            detail::deflate_into(in, out, 6);
            break;
        case LosslessCodec::DeflateChunked: {
            const std::size_t n = (in.size() + detail::kChunk - 1) / detail::kChunk;
            std::vector<Bytes> parts(n);
            detail::parallel_for(n, threads, [&](std::size_t i) {
                const std::size_t b = i * detail::kChunk, e = std::min(in.size(), b + detail::kChunk);
                detail::deflate_into(in.subspan(b, e - b), parts[i], 1);
            });
            std::size_t total = 12 + 8 * n;
            for (auto& p : parts) total += p.size();
            out.resize(total);
            const std::uint32_t n32 = std::uint32_t(n);
            std::memcpy(out.data(), &n32, 4);
            detail::put64(out, 4, detail::kChunk);
            std::size_t at = 12 + 8 * n;
            for (std::size_t i = 0; i < n; ++i) {
                detail::put64(out, 12 + 8 * i, parts[i].size());
                std::memcpy(out.data() + at, parts[i].data(), parts[i].size());
                at += parts[i].size();
            }
            break;
        }
        default:
            throw Error(ErrorCode::UnknownCodec, "lossless codec " + std::to_string(unsigned(codec)));
    }
    const CompressionReport rep = CompressionReport::from_sizes(in.size(), out.size());
    return {std::move(out), rep};
}

/// Inverse of lossless_encode (decode(encode(x)) == x).
inline Bytes lossless_decode(std::span<const std::byte> in, LosslessCodec codec, std::size_t original_size,
                             int threads = 0) {
    Bytes out;
    switch (codec) {
        case LosslessCodec::None:
            out.assign(in.begin(), in.end());
            break;
        case LosslessCodec::Rle:
            out.reserve(original_size);
            for (std::size_t i = 0; i + 1 < in.size(); i += 2) out.insert(out.end(), std::size_t(in[i]), in[i + 1]);
            break;
        case LosslessCodec::Deflate:
            out.resize(original_size);
            detail::inflate_exact(in, out.data(), original_size);
            break;
        case LosslessCodec::DeflateChunked: {
            if (in.size() < 12) throw Error(ErrorCode::LengthMismatch, "chunked deflate: short header");
            std::uint32_t n;
            std::memcpy(&n, in.data(), 4);
            const std::uint64_t chunk = detail::get64(in, 4);
            if (in.size() < 12 + 8ull * n) throw Error(ErrorCode::LengthMismatch, "chunked deflate: short table");
            std::vector<std::size_t> off(n + 1, 12 + 8ull * n);
            for (std::uint32_t i = 0; i < n; ++i) off[i + 1] = off[i] + detail::get64(in, 12 + 8ull * i);
            if (off[n] != in.size()) throw Error(ErrorCode::LengthMismatch, "chunked deflate: length mismatch");
            out.resize(original_size);
            detail::parallel_for(n, threads, [&](std::size_t i) {
                const std::size_t b = i * chunk, e = std::min<std::size_t>(original_size, b + chunk);
                detail::inflate_exact(in.subspan(off[i], off[i + 1] - off[i]), out.data() + b, e - b);
            });
            break;
        }
        default:
            throw Error(ErrorCode::UnknownCodec, "lossless codec " + std::to_string(unsigned(codec)));
    }
    if (out.size() != original_size) throw Error(ErrorCode::LengthMismatch, "lossless decode: size mismatch");
    return out;
}

/// Asynchronous suffix of the hybrid mode: drain `reader` (CRC-validated kind-1
/// frames from the device prefix), lossless-code every block's SPEC.md:282 payload
/// body with `codec` on `threads` host threads (straight from the frame, no copy) and
/// hand the block (metadata, codec id, coded bytes and coded_source_bytes; the mask
/// stream too if keep_stream) to `sink`.  Returns the number of frames consumed.  Runs
/// on the caller's (consumer) thread.
inline std::uint64_t run_lossless_suffix(staging::StageReader& reader, std::uint64_t n_elements, LosslessCodec codec,
                                         int threads, const std::function<void(std::uint64_t, CompressedBlock&&)>& sink,
                                         bool keep_stream = false) {
    std::uint64_t frames = 0;
    while (auto fr = reader.read_frame()) {
        const auto& h = fr->header;
        if (h.kind != PayloadKind::CompressedBlock)
            throw Error(ErrorCode::InvalidArgument, "hybrid suffix: frame is not a compressed block");
        const auto payload = fr->payload();
        CompressedBlock blk = block_from_payload(payload, h, n_elements, keep_stream);
        const std::size_t body = kind1_body_bytes(payload, n_elements);
        LosslessResult r = lossless_encode(payload.first(body), codec, threads);  // the SPEC.md:282 body
        blk.coded_source_bytes = body;
        blk.lossless_codec = static_cast<std::uint16_t>(codec);
        blk.coded_bytes = std::move(r.coded);
        sink(h.step_index, std::move(blk));
        ++frames;
    }
    return frames;
}

}  // namespace isf::tasks
