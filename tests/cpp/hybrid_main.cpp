// Hybrid in-situ mode (SPEC.md run_hybrid) through
// the reference's own staging layer: the synchronous prefix (device lossy
// compression + device kind-1 frame + pinned D2H, include/isf/tasks/lossy.hpp) runs
// inline with a device-resident producer; only the compressed frame crosses PCIe and
// goes to the reference StageWriter (InProcess backend, staging.hpp:59-60).  The
// asynchronous suffix is the product's (include/isf/tasks/lossless.hpp
// run_lossless_suffix): a consumer thread reads the frames with the reference
// StageReader (its CRC check is the reference's zlib one) and lossless-codes each
// block's stream on a host thread pool (codec 3, chunked Deflate).  After the timed
// run every coded block is decoded back (SPEC payload body -> mask stream) and decompressed against the
// producer's field of that step (exact round trip: the error bound and the stream
// parser both need every byte).  Prints one JSON line.
//
// Built by oracle/Makefile `hybrid` from the reference sources (never copied).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <map>
#include <thread>

#include "isf/staging/staging.hpp"
#include "isf/tasks/lossless.hpp"
#include "isf/tasks/lossy.hpp"

using namespace isf;
using clk = std::chrono::steady_clock;

int main(int argc, char** argv) {
    const std::uint32_t E = argc > 1 ? std::atoi(argv[1]) : 16, P = 8;
    const int steps = argc > 2 ? std::atoi(argv[2]) : 6;
    const int threads = argc > 3 ? std::atoi(argv[3]) : 0;  // suffix pool (0: all host threads)
    const double eps = 1e-3;
    const std::uint64_t n_el = std::uint64_t(E) * E * E, n = n_el * P * P * P;
    double* d_field = nullptr;
    if (cudaMalloc(&d_field, n * 8) != cudaSuccess) return 2;
    isf_lossy_plan* gen = tasks::detail::plan_for(P, 1);

    staging::Options opt;
    opt.capacity = 2;
    auto [writer, reader] = staging::open_pair(staging::Backend::InProcess, opt);

    std::map<std::uint64_t, tasks::CompressedBlock> done;
    double consumer_s = 0.0;
    std::uint64_t frames = 0;
    bool consumer_ok = true;
    std::thread consumer([&, &reader = reader] {
        const auto t0 = clk::now();
        try {
            frames = tasks::run_lossless_suffix(reader, n_el, tasks::LosslessCodec::DeflateChunked, threads,
                                                [&](std::uint64_t step, tasks::CompressedBlock&& b) {
                                                    done.emplace(step, std::move(b));
                                                });
        } catch (const std::exception& e) {
            std::fprintf(stderr, "consumer: %s\n", e.what());
            consumer_ok = false;
        }
        consumer_s = std::chrono::duration<double>(clk::now() - t0).count();
    });

    double prefix_s = 0.0, handoff_s = 0.0, prefix_warm_s = 0.0, handoff_warm_s = 0.0;
    std::uint64_t staged = 0;
    const auto run0 = clk::now();
    for (int s = 0; s < steps; ++s) {
        // device-resident producer step: the TGV component s % 4
        isf_lossy_generate_tgv(gen, d_field, E, 0, E, s % 4, 2 * M_PI, nullptr);
        cudaDeviceSynchronize();
        const auto t0 = clk::now();
        Bytes fr = tasks::lossy_compress_frame(d_field, n_el, E, P, 1, tasks::LossyConfig{eps}, s, 0.1 * s);
        const double pf = std::chrono::duration<double>(clk::now() - t0).count();
        prefix_s += pf;
        staged += fr.size();
        const double hf = writer.write_frame(std::move(fr));
        handoff_s += hf;
        if (s > 0) {  // after the first step's allocations (device frame, pinned staging)
            prefix_warm_s += pf;
            handoff_warm_s += hf;
        }
    }
    writer.close();
    consumer.join();
    const double run_s = std::chrono::duration<double>(clk::now() - run0).count();

    // validation (outside the timed run): lossless round trip + lossy error bound
    bool ok = consumer_ok && frames == std::uint64_t(steps) && done.size() == std::size_t(steps);
    double worst_rel = 0.0;
    std::uint64_t coded_total = 0;
    std::vector<double> host_orig(n);
    for (auto& [step, blk] : done) {
        coded_total += blk.coded_bytes.size();
        // the suffix kept only the coded bytes: decode them back into the SPEC payload body
        // and that into the block's mask stream
        const Bytes body = tasks::lossless_decode(blk.coded_bytes, tasks::LosslessCodec(blk.lossless_codec),
                                                  blk.coded_source_bytes, threads);
        blk.stream = tasks::detail::stream_from_spec_body(body, n_el, P, 1);
        if (blk.stream.size() != blk.report.compressed_size) ok = false;
        isf_lossy_generate_tgv(gen, d_field, E, 0, E, int(step % 4), 2 * M_PI, nullptr);
        cudaMemcpy(host_orig.data(), d_field, n * 8, cudaMemcpyDeviceToHost);
        Field orig(E, P, 1, host_orig);
        tasks::ErrorReport rep;
        (void)tasks::lossy_decompress(blk, orig, &rep, &orig);
        const double rel = rep.rel_l2();
        worst_rel = rel > worst_rel ? rel : worst_rel;
        if (!(rel <= eps * (1 + 1e-9))) ok = false;
    }
    cudaFree(d_field);
    const double raw = double(n) * 8 * steps;
    // SPEC.md run_hybrid example: TGV with kept fraction <= 5% -> staged bytes <= 10% of raw
    ok = ok && staged <= 0.10 * raw;
    std::printf("{\"ok\": %s, \"steps\": %d, \"raw_bytes\": %.0f, \"staged_bytes\": %llu, \"staged_fraction\": %.5f, "
                "\"coded_bytes\": %llu, \"codec\": \"deflate-chunked (1 MiB, level 1)\", \"suffix_threads\": %d, "
                "\"worst_rel_l2\": %.3e, \"prefix_ms_per_step\": %.3f, \"handoff_ms_per_step\": %.3f, "
                "\"consumer_ms_per_frame\": %.3f, \"run_ms_per_step\": %.3f, \"prefix_ms_per_step_warm\": %.3f, "
                "\"handoff_ms_per_step_warm\": %.3f}\n",
                ok ? "true" : "false", steps, raw, (unsigned long long)staged, staged / raw,
                (unsigned long long)coded_total, tasks::detail::pool_size(threads), worst_rel,
                1e3 * prefix_s / steps, 1e3 * handoff_s / steps, 1e3 * consumer_s / steps, 1e3 * run_s / steps,
                steps > 1 ? 1e3 * prefix_warm_s / (steps - 1) : 0.0, steps > 1 ? 1e3 * handoff_warm_s / (steps - 1) : 0.0);
    return ok ? 0 : 1;
}
