// SPEC.md:240-248 lossless_encode / lossless_decode examples and properties for the
// product's codecs (include/isf/tasks/lossless.hpp); CPU only.  Prints one JSON line.
#include <cstdio>
#include <random>

#include "isf/tasks/lossless.hpp"

using namespace isf;
using tasks::LosslessCodec;

int main() {
    bool ok = true;
    auto check = [&](bool c, const char* what) {
        if (!c) {
            std::fprintf(stderr, "FAIL: %s\n", what);
            ok = false;
        }
    };
    // 1 MiB of zero bytes under Rle -> cr >= 0.99
    Bytes zeros(1 << 20, std::byte{0});
    auto r = tasks::lossless_encode(zeros, LosslessCodec::Rle);
    check(r.report.cr >= 0.99, "rle zeros cr");
    check(tasks::lossless_decode(r.coded, LosslessCodec::Rle, zeros.size()) == zeros, "rle zeros round trip");
    // decode(encode(x)) == x for random x, every codec, sizes around the chunk size
    std::mt19937_64 g(20240731);
    for (std::size_t sz : {std::size_t(0), std::size_t(1), std::size_t(1000), std::size_t(1 << 20),
                           std::size_t((3 << 20) + 17)}) {
        Bytes x(sz);
        for (auto& b : x) b = std::byte(g() % 7 == 0 ? g() & 255 : 0);  // compressible random bytes
        for (auto c : {LosslessCodec::None, LosslessCodec::Rle, LosslessCodec::Deflate, LosslessCodec::DeflateChunked}) {
            auto e = tasks::lossless_encode(x, c, 4);
            check(tasks::lossless_decode(e.coded, c, x.size(), 4) == x, "round trip");
            check(e.report.original_size == x.size() && e.report.compressed_size == e.coded.size(), "report sizes");
        }
    }
    // compressed_size == original_size -> cr == 0.0 (Eq. 1)
    check(tasks::CompressionReport::from_sizes(4096, 4096).cr == 0.0, "eq1 equal sizes");
    // unknown codec -> UnknownCodec
    bool threw = false;
    try {
        (void)tasks::lossless_encode(zeros, LosslessCodec(9));
    } catch (const Error& e) {
        threw = e.code() == ErrorCode::UnknownCodec;
    }
    check(threw, "unknown codec");
    std::printf("{\"ok\": %s}\n", ok ? "true" : "false");
    return ok ? 0 : 1;
}
