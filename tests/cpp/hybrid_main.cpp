// Hybrid in-situ mode (SPEC.md run_hybrid) through
// the reference's own staging layer: the synchronous prefix (device lossy
// compression + device kind-1 frame, include/isf/tasks/lossy.hpp) runs inline with
// a device-resident producer; only the compressed frame crosses PCIe and goes to
// the reference StageWriter (InProcess backend, staging.hpp:59-60); an
// asynchronous consumer thread reads validated frames with the reference
// StageReader (its CRC check is the reference's zlib one), applies the lossless
// suffix (zlib deflate of the stream, codec id 2 = Deflate) and decodes the block
// back to check the error bound.  Prints one JSON line.
//
// Built by oracle/Makefile `hybrid` from the reference sources (never copied).
#include <zlib.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <thread>

#include "isf/staging/staging.hpp"
#include "isf/tasks/lossy.hpp"

using namespace isf;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const std::uint32_t E = argc > 1 ? std::atoi(argv[1]) : 16, P = 8;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 6;
    const double eps = 1e-3;
    const std::uint64_t n_el = std::uint64_t(E) * E * E, n = n_el * P * P * P;
    double* d_field = nullptr;
    if (cudaMalloc(&d_field, n * 8) != cudaSuccess) return 2;
    isf_lossy_plan* gen = tasks::detail::plan_for(P, 1);

    staging::Options opt;
    opt.capacity = 2;
    auto [writer, reader] = staging::open_pair(staging::Backend::InProcess, opt);

    bool ok = true;
    double worst_rel = 0.0, consumer_s = 0.0;
    std::uint64_t staged = 0, coded_total = 0, frames = 0;
    std::thread consumer([&, &reader = reader] {
        const auto t0 = clk::now();
        isf_lossy_plan* gen_c = tasks::detail::plan_for(P, 1);  // this thread's plan
        std::vector<double> host_orig(n);
        while (auto fr = reader.read_frame()) {  // CRC-validated by the reference
            ++frames;
            const auto& h = fr->header;
            if (h.kind != PayloadKind::CompressedBlock || h.points_per_element_axis != P) ok = false;
            auto blk = tasks::block_from_payload(fr->payload(), h, n_el);
            // lossless suffix: deflate the stream
            uLongf clen = compressBound(blk.stream.size());
            Bytes coded(clen);
            if (compress2(reinterpret_cast<Bytef*>(coded.data()), &clen,
                          reinterpret_cast<const Bytef*>(blk.stream.data()), blk.stream.size(), 6) != Z_OK)
                ok = false;
            coded.resize(clen);
            uLongf back_len = blk.stream.size();
            Bytes back(back_len);
            if (uncompress(reinterpret_cast<Bytef*>(back.data()), &back_len,
                           reinterpret_cast<const Bytef*>(coded.data()), clen) != Z_OK ||
                back_len != blk.stream.size() || back != blk.stream)
                ok = false;
            coded_total += clen;
            blk.lossless_codec = 2;
            blk.coded_bytes = std::move(coded);
            // decode and check against the producer's field of that step (regenerated on the host side
            // from the device generator: same call, same bytes)
            double* d_tmp = nullptr;
            cudaMalloc(&d_tmp, n * 8);
            isf_lossy_generate_tgv(gen_c, d_tmp, E, 0, E, int(h.step_index % 4), 2 * M_PI, nullptr);
            cudaMemcpy(host_orig.data(), d_tmp, n * 8, cudaMemcpyDeviceToHost);
            cudaFree(d_tmp);
            Field orig(E, P, 1, host_orig);
            tasks::ErrorReport rep;
            (void)tasks::lossy_decompress(blk, orig, &rep, &orig);
            const double rel = rep.rel_l2();
            worst_rel = rel > worst_rel ? rel : worst_rel;
            if (!(rel <= eps * (1 + 1e-9))) ok = false;
        }
        consumer_s = std::chrono::duration<double>(clk::now() - t0).count();
    });

    double prefix_s = 0.0, handoff_s = 0.0;
    for (int s = 0; s < steps; ++s) {
        // device-resident producer step: the TGV component s % 4
        isf_lossy_generate_tgv(gen, d_field, E, 0, E, s % 4, 2 * M_PI, nullptr);
        cudaDeviceSynchronize();
        const auto t0 = clk::now();
        Bytes fr = tasks::lossy_compress_frame(d_field, n_el, E, P, 1, tasks::LossyConfig{eps}, s, 0.1 * s);
        prefix_s += std::chrono::duration<double>(clk::now() - t0).count();
        staged += fr.size();
        handoff_s += writer.write_frame(std::move(fr));
    }
    writer.close();
    consumer.join();
    cudaFree(d_field);
    const double raw = double(n) * 8 * steps;
    // SPEC.md run_hybrid example: TGV with kept fraction <= 5% -> staged bytes <= 10% of raw
    ok = ok && frames == std::uint64_t(steps) && staged <= 0.10 * raw;
    std::printf("{\"ok\": %s, \"steps\": %d, \"raw_bytes\": %.0f, \"staged_bytes\": %llu, \"staged_fraction\": %.5f, "
                "\"deflated_bytes\": %llu, \"worst_rel_l2\": %.3e, \"prefix_ms_per_step\": %.3f, "
                "\"handoff_ms_per_step\": %.3f, \"consumer_s\": %.3f}\n",
                ok ? "true" : "false", steps, raw, (unsigned long long)staged, staged / raw,
                (unsigned long long)coded_total, worst_rel, 1e3 * prefix_s / steps, 1e3 * handoff_s / steps,
                consumer_s);
    return ok ? 0 : 1;
}
