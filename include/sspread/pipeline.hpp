// sspread/pipeline.hpp — drop-in for the reference's detection driver
// (/root/reference/proj/include/sspread/pipeline.hpp) on the B200 engine.
//
// process_slice keeps the reference contract (scan, report when the window is
// full and a sink is set, slide; pipeline.hpp:110-129) but the record batch
// crosses to the device once and the candidate list stays in HBM between
// slices. process_slice_device() is an addition for records already resident
// on the GPU. Exact-cardinality ground truth (run_oracle) runs on the device
// store of oracle.hpp.
#pragma once

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <functional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "oracle.hpp"
#include "sea.hpp"
#include "trace.hpp"

namespace sspread {

class ConfigError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

class InternalError : public std::runtime_error {
  public:
    using std::runtime_error::runtime_error;
};

struct RunConfig {
    SeaConfig sea;
    uint32_t slice_seconds = 300;
    CidrPrefix a_network{0x0A000000, 8};
    uint32_t workers = 1;  // host threads for host-side helpers; the sketch runs on the GPU
    int device = 0;        // addition: CUDA device of the sketch

    void validate() const {  // pipeline.hpp:38-48
        try {
            sea.validate();
            if (slice_seconds == 0) throw std::invalid_argument("slice duration must be >= 1 second");
            if (workers == 0 || workers > 256) throw std::invalid_argument("workers must be in [1, 256]");
            if (sea.cols & (sea.cols - 1)) throw std::invalid_argument("cols must be a power of two");
        } catch (const std::invalid_argument& e) {
            throw ConfigError(e.what());
        }
    }
};

// fn over near-equal subranges of [0, total) on `workers` threads (pipeline.hpp:54-68)
inline void parallel_ranges(uint64_t total, uint32_t workers, const std::function<void(uint64_t, uint64_t)>& fn) {
    if (!total) return;
    const uint64_t n = std::min<uint64_t>(std::max<uint32_t>(workers, 1), total);
    std::vector<std::thread> pool;
    for (uint64_t w = 1; w < n; ++w) pool.emplace_back([&, w] { fn(total * w / n, total * (w + 1) / n); });
    fn(0, total / n);
    for (auto& t : pool) t.join();
}

inline ChunkRunner chunked(uint32_t workers) {
    return [workers](uint64_t total, const std::function<void(uint64_t, uint64_t)>& fn) {
        parallel_ranges(total, workers, fn);
    };
}

template <RecorderWord W>
class DetectPipeline {
  public:
    using ReportSink = std::function<void(const WindowReport&)>;

    explicit DetectPipeline(const RunConfig& cfg) : cfg_((cfg.validate(), cfg)), sea_(cfg.sea, cfg.device) {}

    EstimatorArray<W>& sketch() noexcept { return sea_; }
    const OrientStats& orient_stats() const noexcept { return stats_; }
    uint64_t pairs_scanned() const noexcept { return pairs_; }
    uint64_t slices_seen() const noexcept { return slices_; }
    double total_scan_ms() const noexcept { return total_scan_ms_; }
    double total_estimate_ms() const noexcept { return total_estimate_ms_; }

    // pipeline.hpp:96-106. Binary (SRLT) traces take the device front end:
    // the file crosses to HBM once; parsing, orientation and the slice
    // boundaries run on the GPU (srla_parse_srlt / srla_orient_records /
    // srla_slice_bounds) and every slice is scanned where it lies. CSV traces
    // take the host path, and so do binary traces above kDeviceTraceBytes
    // (SRLA_DEVICE_TRACE_MAX overrides it): the device front end holds the
    // file and two record copies in HBM, the host path streams the file one
    // slice at a time, as the reference does.
    static constexpr uint64_t kDeviceTraceBytes = 8ull << 30;
    void run(const std::string& trace_path, const ReportSink& sink) {
        uint64_t limit = kDeviceTraceBytes;
        if (const char* v = std::getenv("SRLA_DEVICE_TRACE_MAX")) limit = std::strtoull(v, nullptr, 0);
        std::error_code ec;
        const auto fsize = std::filesystem::file_size(trace_path, ec);
        if (sniff_trace_format(trace_path) == TraceFormat::binary && (ec || fsize <= limit)) {
            run_device(trace_path, sink);
            return;
        }
        SlicePartitioner partitioner(cfg_.slice_seconds);
        const auto on_slice = [&](uint64_t id, std::vector<TraceRecord>&& records) {
            process_slice(id, records, sink);
        };
        for_each_record(trace_path, [&](const TraceRecord& r) {
            if (const auto o = orient_record(r, cfg_.a_network, stats_)) partitioner.push(*o, on_slice);
        });
        partitioner.finish(on_slice);
    }

    void process_slice(uint64_t slice_id, std::span<const TraceRecord> records, const ReportSink& sink) {
        process(slice_id, records.data(), records.size(), 0, sink);
    }

    // Addition: `d_records` points to `n` records in device memory on the
    // sketch's GPU (e.g. a capture ring already in HBM).
    void process_slice_device(uint64_t slice_id, const TraceRecord* d_records, uint64_t n, const ReportSink& sink) {
        process(slice_id, d_records, n, 1, sink);
    }

    const CandidateList& candidates() const {
        if (!csip_valid_) {
            csip_.clear();
            const std::vector<uint32_t> v =
                sea_.st_->pipeline_owns_list ? sea_.engine_list() : sea_.st_->saved_pipeline_list;
            for (uint32_t h : v) csip_.insert(h);
            csip_valid_ = true;
        }
        return csip_;
    }

  private:
    void run_device(const std::string& path, const ReportSink& sink) {
        std::ifstream in(path, std::ios::binary | std::ios::ate);
        if (!in) throw InputError("cannot open trace: " + path);
        const uint64_t nbytes = static_cast<uint64_t>(in.tellg());
        std::vector<char> bytes(nbytes);
        in.seekg(0);
        in.read(bytes.data(), static_cast<std::streamsize>(nbytes));
        const int dev = cfg_.device;
        struct DevMem {
            int dev;
            void* p = nullptr;
            ~DevMem() { if (p) srla_device_free(dev, p); }
        } d_bytes{dev}, d_raw{dev}, d_recs{dev};
        const uint64_t cap = nbytes >= 5 ? (nbytes - 5) / 12 + 1 : 1;
        detail::check(srla_device_alloc(dev, std::max<uint64_t>(nbytes, 1), &d_bytes.p), "srla_device_alloc");
        detail::check(srla_device_alloc(dev, cap * sizeof(srla_record), &d_raw.p), "srla_device_alloc");
        detail::check(srla_device_alloc(dev, cap * sizeof(srla_record), &d_recs.p), "srla_device_alloc");
        detail::check(srla_copy_to_device(dev, d_bytes.p, bytes.data(), nbytes), "srla_copy_to_device");
        uint64_t n = 0;
        const srla_status ps = srla_parse_srlt(d_bytes.p, nbytes, static_cast<srla_record*>(d_raw.p), &n, nullptr);
        std::string input_error;
        if (ps == SRLA_E_INPUT) input_error = reference_input_error(srla_last_error(), path, bytes, n);
        else detail::check(ps, "srla_parse_srlt");
        uint64_t m = 0;
        srla_orient_stats os{};
        detail::check(srla_orient_records(static_cast<const srla_record*>(d_raw.p), n, cfg_.a_network.addr,
                                          cfg_.a_network.bits, static_cast<srla_record*>(d_recs.p), &m, &os, nullptr),
                      "srla_orient_records");
        stats_.kept += os.kept;
        stats_.flipped += os.flipped;
        stats_.dropped_both += os.dropped_both;
        stats_.dropped_neither += os.dropped_neither;
        uint64_t ns = 0;
        detail::check(srla_slice_bounds(static_cast<const srla_record*>(d_recs.p), m, cfg_.slice_seconds, nullptr, 0,
                                        &ns, nullptr),
                      "srla_slice_bounds");
        std::vector<uint64_t> off(ns + 1);
        if (ns)
            detail::check(srla_slice_bounds(static_cast<const srla_record*>(d_recs.p), m, cfg_.slice_seconds,
                                            off.data(), off.size(), &ns, nullptr),
                          "srla_slice_bounds");
        // a failed read leaves the last, unfinished slice unprocessed (the
        // partitioner is never finished), as for_each_record's throw does
        const uint64_t done = input_error.empty() ? ns : (ns ? ns - 1 : 0);
        const auto* d = static_cast<const TraceRecord*>(d_recs.p);
        for (uint64_t sid = 0; sid < done; ++sid) process_slice_device(sid, d + off[sid], off[sid + 1] - off[sid], sink);
        if (!input_error.empty()) throw InputError(input_error);
    }

    // for_each_record's InputError text (trace.hpp:109-170) for a device
    // parse failure: the record index comes from the device, the timestamps of
    // a regression from the file bytes still on the host
    static std::string reference_input_error(const std::string& msg, const std::string& path,
                                             const std::vector<char>& bytes, uint64_t bad) {
        auto ts_at = [&](uint64_t i) {
            uint32_t v = 0;
            std::memcpy(&v, bytes.data() + 5 + 12 * i, 4);  // x86: little-endian
            return v;
        };
        if (msg.rfind("timestamp regression", 0) == 0 && bad > 0 && 5 + 12 * (bad + 1) <= bytes.size())
            return "timestamp regression at record " + std::to_string(bad) + " of " + path + " (" +
                   std::to_string(ts_at(bad)) + " after " + std::to_string(ts_at(bad - 1)) + ")";
        if (msg.rfind("not a binary trace", 0) == 0) return "not a binary trace (bad magic): " + path;
        if (msg.rfind("unsupported trace version", 0) == 0) return "unsupported trace version in " + path;
        return msg + " in " + path;  // "truncated record N in PATH"
    }

    void process(uint64_t slice_id, const TraceRecord* recs, uint64_t n, int on_device, const ReportSink& sink) {
        sea_.pipeline_mode();
        sea_.to_device();
        const auto t0 = std::chrono::steady_clock::now();
        detail::check(srla_scan_batch(sea_.eng(), reinterpret_cast<const srla_record*>(recs), n, on_device, nullptr,
                                      0, nullptr),
                      "srla_scan_batch");
        const double scan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        total_scan_ms_ += scan_ms;
        pairs_ += n;
        ++slices_;
        // report + slide as ONE fused end-of-slice (srla_end_slice: the
        // window's fill counts come out of the same pass that ages the table,
        // and the entries are mapped on the device). The report handed to the
        // sink is the reference's; the sketch it could be queried through has
        // already slid.
        const uint32_t k = cfg_.sea.window;
        const bool due = slice_id + 1 >= k && static_cast<bool>(sink);
        const auto t1 = std::chrono::steady_clock::now();
        // the hand-off buffer is sized from the first try: srla_end_slice
        // rejects a short buffer (reporting the count) before doing any work
        uint64_t n_out = 0, kept = 0;
        srla_status es = srla_end_slice(sea_.eng(), slice_id, due ? 1 : 0, entries_.data(), entries_.size(), &n_out,
                                        &kept);
        if (es == SRLA_E_CAPACITY && due) {
            entries_.reserve(n_out);
            es = srla_end_slice(sea_.eng(), slice_id, 1, entries_.data(), entries_.size(), &n_out, &kept);
        }
        detail::check(es, "srla_end_slice");
        sea_.st_->mirror_valid = false;
        csip_valid_ = false;
        if (due) {
            // one report object reused across slices: its entry storage stays
            // mapped (a fresh 18 MB vector per slice costs ~9 ms of page faults at C2)
            WindowReport& report = report_;
            report.window_start = slice_id + 1 - k;
            report.window = k;
            detail::fill_entries(report.entries, entries_.data(), n_out);
            report.scan_ms = scan_ms;
            report.estimate_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
            total_estimate_ms_ += report.estimate_ms;
            sink(report);
        }
    }

    RunConfig cfg_;
    EstimatorArray<W> sea_;
    detail::PinnedEntries entries_;  // report hand-off buffer (pinned: entries mapped on the device, one DMA)
    WindowReport report_;            // handed to the sink by const reference
    mutable CandidateList csip_;
    mutable bool csip_valid_ = false;
    OrientStats stats_;
    uint64_t pairs_ = 0;
    uint64_t slices_ = 0;
    double total_scan_ms_ = 0;
    double total_estimate_ms_ = 0;
};

/// Ground-truth record for one window (pipeline.hpp:183-187).
struct TruthEntry {
    uint64_t window_start = 0;
    uint32_t host = 0;
    uint64_t cardinality = 0;
};

enum class OracleEngine { ring, pair_recorders, both };

inline constexpr uint64_t kOraclePairGuard = 100'000'000;

/// pipeline.hpp:189-247: exact sliding-window cardinalities over a trace —
/// per complete window, every host reaching `min_cardinality`, sorted by
/// address. Both reference engines are the same device store here
/// (oracle.hpp), so OracleEngine::both has nothing to cross-check; the pair
/// guard and its message are the reference's.
inline void run_oracle(const RunConfig& cfg, const std::string& trace_path, OracleEngine engine,
                       uint64_t min_cardinality, const std::function<void(const TruthEntry&)>& sink,
                       uint64_t max_pairs = kOraclePairGuard) {
    cfg.validate();
    const uint32_t k = cfg.sea.window;
    if (engine != OracleEngine::ring) RecorderModel::with_bits(cfg.sea.recorder_bits).validate_window(k);
    SliceRingStore store(k, cfg.device);
    OrientStats stats;
    uint64_t observed = 0;
    const auto on_slice = [&](uint64_t id, std::vector<TraceRecord>&& records) {
        for (const auto& r : records) store.observe(r.src, r.dst);
        if (id + 1 >= k) {
            const uint64_t t = id + 1 - k;
            for (const auto& [host, n] : store.cardinalities(t, k))  // ascending by address
                if (n >= min_cardinality) sink(TruthEntry{t, host, n});
        }
        store.end_slice();
    };
    SlicePartitioner partitioner(cfg.slice_seconds);
    for_each_record(trace_path, [&](const TraceRecord& r) {
        const auto oriented = orient_record(r, cfg.a_network, stats);
        if (!oriented) return;
        if (++observed > max_pairs)
            throw InputError("trace exceeds the oracle pair guard (" + std::to_string(max_pairs) +
                             " records); raise --max-pairs for a machine that can hold it");
        partitioner.push(*oriented, on_slice);
    });
    partitioner.finish(on_slice);
}

// Runtime width -> storage word (pipeline.hpp:173-180).
template <typename Fn>
decltype(auto) with_recorder_word(uint32_t recorder_bits, Fn&& fn) {
    switch (recorder_word_bytes(recorder_bits)) {
        case 1: return fn(uint8_t{0});
        case 2: return fn(uint16_t{0});
        default: return fn(uint32_t{0});
    }
}

}  // namespace sspread
