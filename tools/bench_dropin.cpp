// bench_dropin — the reference's own entry point, timed: sspread::DetectPipeline<
// uint8_t>::process_slice (pipeline.hpp:110-129) through the drop-in headers
// (include/sspread), on BASELINE.json's C2 workload with HOST records.
//
// Each slice of the C2 trace is generated on the device (srla_generate_slice,
// byte-identical to the reference generator) and copied into a pinned host
// buffer outside the timed region; the timed call is process_slice(span of
// host records, sink): host->device copy, scan, fused report + slide, report
// hand-off into the sink. After k - 1 prefill slices and `warmup` steps,
// `steps` steps are timed. Prints one JSON line.
//
//   bench_dropin <steps> <warmup> [packets_per_slice]
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <span>
#include <vector>

#include "sspread/pipeline.hpp"

using namespace sspread;

namespace {
void check(srla_status s, const char* what) {
    if (s != SRLA_OK) {
        std::fprintf(stderr, "%s: %s\n", what, srla_last_error());
        std::exit(1);
    }
}
}  // namespace

int main(int argc, char** argv) {
    const int steps = argc > 1 ? std::atoi(argv[1]) : 10;
    const int warmup = argc > 2 ? std::atoi(argv[2]) : 3;
    const uint32_t pairs = argc > 3 ? static_cast<uint32_t>(std::atoll(argv[3])) : 100000000u;
    RunConfig rc;  // C2: u=4 v=2^20 g=8 g'=1024 z=4 k=10 theta=1024 (paper_1803_10369_b200/workloads.py)
    rc.sea.rows = 4;
    rc.sea.cols = 1u << 20;
    rc.sea.rough_slots = 8;
    rc.sea.linear_slots = 1024;
    rc.sea.recorder_bits = 4;
    rc.sea.window = 10;
    rc.sea.theta = 1024;
    rc.sea.seed = 0x5EA00001;
    rc.slice_seconds = 1;
    std::vector<srla_plant> plants;
    for (int i = 0; i < 50; ++i)
        plants.push_back({0x0AC80001u + i,
                          static_cast<uint32_t>(std::floor(1152.0 * std::pow(16384.0 / 1152.0, i / 49.0) + 0.5)), 0,
                          0xFFFFFFFFu});
    const int total = static_cast<int>(rc.sea.window) - 1 + warmup + steps;
    srla_trace_spec spec{1, 1700000000u, 1, static_cast<uint32_t>(total), 10, 0x0A100000u, 0x64400000u, 4194304u,
                         1u << 22, pairs, 50, 1.0, plants.data()};
    srla_generator* gen = nullptr;
    check(srla_generator_create(&spec, 0, &gen), "srla_generator_create");
    uint64_t cap = 0;
    check(srla_generate_slice(gen, 0, nullptr, 0, &cap, nullptr), "srla_generate_slice");
    cap += 1024;
    void* d_recs = nullptr;
    void* h_recs = nullptr;
    check(srla_device_alloc(0, cap * sizeof(srla_record), &d_recs), "srla_device_alloc");
    check(srla_host_alloc(cap * sizeof(srla_record), &h_recs), "srla_host_alloc");  // pinned: DMA-able

    DetectPipeline<uint8_t> pipe(rc);
    uint64_t entries = 0;
    double timed_ms = 0.0, packets = 0.0;
    std::vector<double> eos;
    for (int s = 0; s < total; ++s) {
        uint64_t n = 0;
        check(srla_generate_slice(gen, s, static_cast<srla_record*>(d_recs), cap, &n, nullptr), "srla_generate_slice");
        check(srla_copy_to_host(0, h_recs, d_recs, n * sizeof(srla_record)), "srla_copy_to_host");
        const std::span<const TraceRecord> recs(static_cast<const TraceRecord*>(h_recs), n);
        const auto t0 = std::chrono::steady_clock::now();
        pipe.process_slice(static_cast<uint64_t>(s), recs, [&](const WindowReport& r) {
            entries = r.entries.size();
            eos.push_back(r.estimate_ms);
        });
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        if (s >= total - steps) {
            timed_ms += ms;
            packets += static_cast<double>(n);
        }
    }
    std::vector<double> tail(eos.end() - std::min<size_t>(eos.size(), static_cast<size_t>(steps)), eos.end());
    std::sort(tail.begin(), tail.end());
    std::printf(
        "{\"api\": \"sspread::DetectPipeline<uint8_t>::process_slice (host records, pinned)\", \"value\": %.6g, "
        "\"unit\": \"packets/s\", \"ms_per_step\": %.4f, \"steps\": %d, \"warmup\": %d, \"packets_per_slice\": %u, "
        "\"report_entries\": %llu, \"report_slide_ms_median\": %.4f, \"h2d_bytes_per_step\": %.0f}\n",
        packets / (timed_ms / 1e3), timed_ms / steps, steps, warmup, pairs, static_cast<unsigned long long>(entries),
        tail.empty() ? 0.0 : tail[tail.size() / 2], packets / steps * 12.0);
    srla_host_free(h_recs);
    srla_device_free(0, d_recs);
    srla_generator_destroy(gen);
    return 0;
}
