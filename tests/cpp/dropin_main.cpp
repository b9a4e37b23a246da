// Drop-in check: the reference's own core types (compiled from /root/reference by
// oracle/Makefile `ref`) + include/isf/tasks/lossy.hpp + libisf_lossy.so.
// Builds a TGV Field with the reference Field type, compresses / decompresses it
// through the SPEC-shaped C++ API, frames the block with the reference
// build_frame (kind 1) and parses it back with the reference parse_frame.
#include <cmath>
#include <cstdio>

#include "isf/tasks/lossy.hpp"

int main() {
    using namespace isf;
    const std::uint32_t E = 8, P = 8;
    std::vector<double> x(P), w(P);
    {
        isf_lossy_plan* p = tasks::detail::plan_for(P, 1);
        isf_lossy_plan_operators(p, nullptr, nullptr, x.data(), w.data());
    }
    std::vector<double> v(E * E * E * P * P * P);
    const double h = 2 * M_PI / E;
    for (std::uint32_t ez = 0; ez < E; ++ez)
        for (std::uint32_t ey = 0; ey < E; ++ey)
            for (std::uint32_t ex = 0; ex < E; ++ex)
                for (std::uint32_t pz = 0; pz < P; ++pz)
                    for (std::uint32_t py = 0; py < P; ++py)
                        for (std::uint32_t px = 0; px < P; ++px) {
                            const double X = ex * h + (x[px] + 1) * 0.5 * h, Y = ey * h + (x[py] + 1) * 0.5 * h,
                                         Z = ez * h + (x[pz] + 1) * 0.5 * h;
                            const std::uint64_t el = ex + E * (ey + E * ez), pt = px + P * (py + P * pz);
                            v[el * P * P * P + pt] = std::cos(X) * std::sin(Y) * std::sin(Z);
                        }
    Field f(E, P, 1, v);
    tasks::LossyConfig cfg{1e-2};
    auto blk = tasks::lossy_compress(f, cfg);
    tasks::ErrorReport rep;
    Field back = tasks::lossy_decompress(blk, f, &rep, &f);
    auto fr = blk.frame(7, 0.5);
    auto parsed = parse_frame({fr.data(), fr.size()});
    bool ok = parsed.header.kind == PayloadKind::CompressedBlock && parsed.payload.size() == blk.payload().size();
    // SPEC.md:282 payload: 4 B count per element + 12 B per kept value + codec trailer,
    // and it parses back to the identical mask stream
    ok = ok && parsed.payload.size() == 4 * f.element_count() + 12 * blk.kept_total + 10;
    auto blk2 = tasks::block_from_payload(parsed.payload, parsed.header, f.element_count());
    ok = ok && blk2.stream == blk.stream && blk2.kept_total == blk.kept_total;
    ok = ok && rep.rel_l2() <= 1e-2 && blk.kept_total <= v.size() / 20;
    bool threw = false;
    try {
        tasks::LossyConfig bad{1.5};
        tasks::lossy_compress(f, bad);
    } catch (const Error& e) {
        threw = e.code() == ErrorCode::InvalidArgument;
    }
    std::printf("dropin kept=%llu cr=%.4f relL2=%.3e relLinf=%.3e frame=%zu ok=%d threw=%d\n",
                (unsigned long long)blk.kept_total, blk.report.cr, rep.rel_l2(), rep.rel_linf(), fr.size(), ok, threw);
    return (ok && threw) ? 0 : 1;
}
