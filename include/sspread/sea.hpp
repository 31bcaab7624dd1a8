// sspread/sea.hpp — drop-in for the reference's estimator array
// (/root/reference/proj/include/sspread/sea.hpp), backed by the B200 engine.
//
// Same namespace, types and member signatures. The sketch state lives in HBM
// and every call goes through the C ABI in srla.h (libsrla_b200.so); nothing
// here computes on the CPU except the reference's own host-side helpers.
//
// Differences a caller can observe:
//  * construction takes an optional CUDA device index;
//  * the raw row spans (indicator_row / rough_row / linear_row) alias a host
//    mirror that is pulled from the device on access and pushed back before
//    the next device operation if a mutable span was handed out — a span kept
//    across a later scan/slide is stale (the reference's spans alias live
//    storage);
//  * scan_records() is an addition: the batched form of scan_ip_pair;
//  * ChunkRunner arguments are accepted and ignored (bulk passes run on the
//    device).
#pragma once

#include <algorithm>
#include <chrono>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../srla.h"
#include "estimators.hpp"
#include "hash.hpp"
#include "recorders.hpp"
#include "trace.hpp"

namespace sspread {

inline constexpr uint32_t kIndicatorBits = 16;

using ChunkRunner = std::function<void(uint64_t, const std::function<void(uint64_t, uint64_t)>&)>;

inline void serial_chunks(uint64_t total, const std::function<void(uint64_t, uint64_t)>& fn) { fn(0, total); }

struct SeaConfig {
    uint32_t rows = 4;
    uint32_t cols = 65536;
    uint32_t rough_slots = 8;
    uint32_t linear_slots = 1024;
    uint32_t recorder_bits = 1;
    uint32_t window = 1;
    uint32_t theta = 1024;
    double fill_ratio = kSuperTestRatio;
    uint64_t seed = 0x00C0FFEEull;

    void validate() const {  // sea.hpp:44-51
        if (rows == 0) throw std::invalid_argument("rows must be >= 1");
        if (cols == 0) throw std::invalid_argument("cols must be >= 1");
        if (rough_slots == 0) throw std::invalid_argument("rough_slots must be >= 1");
        if (linear_slots < 2) throw std::invalid_argument("linear_slots must be >= 2");
        if (theta == 0) throw std::invalid_argument("theta must be >= 1");
        RecorderModel::with_bits(recorder_bits).validate_window(window);
    }
};

// Deduplicated, first-insertion order (sea.hpp:56-76).
class CandidateList {
  public:
    bool insert(uint32_t host) {
        if (!seen_.insert(host).second) return false;
        hosts_.push_back(host);
        return true;
    }
    bool contains(uint32_t host) const { return seen_.count(host) != 0; }
    size_t size() const noexcept { return hosts_.size(); }
    bool empty() const noexcept { return hosts_.empty(); }
    const std::vector<uint32_t>& hosts() const noexcept { return hosts_; }
    void clear() {
        hosts_.clear();
        seen_.clear();
    }

  private:
    std::vector<uint32_t> hosts_;
    std::unordered_set<uint32_t> seen_;
};

template <RecorderWord W>
struct UnionView {
    uint16_t indicator = 0;
    std::vector<W> rough;
    std::vector<W> linear;
};

struct WindowEntry {
    uint32_t host = 0;
    uint32_t union_weight = 0;
    std::optional<double> estimate;
    bool is_super = false;
};

struct WindowReport {
    uint64_t window_start = 0;
    uint32_t window = 1;
    std::vector<WindowEntry> entries;  // sorted by host address
    double scan_ms = 0.0;
    double estimate_ms = 0.0;
};

namespace detail {

[[noreturn]] inline void raise_status(srla_status st, const char* call);

// Page-locked buffer of report entries (srla_host_alloc): the engine maps
// (host, weight) to entries on the device and hands them off in one DMA.
class PinnedEntries {
  public:
    PinnedEntries() = default;
    PinnedEntries(const PinnedEntries&) = delete;
    PinnedEntries& operator=(const PinnedEntries&) = delete;
    ~PinnedEntries() { srla_host_free(p_); }
    void reserve(uint64_t n) {
        if (n <= cap_) return;
        srla_host_free(p_);
        p_ = nullptr;
        cap_ = 0;
        void* q = nullptr;
        const uint64_t c = std::max<uint64_t>(n + n / 4, 1024);
        const srla_status s = srla_host_alloc(c * sizeof(srla_entry), &q);
        if (s != SRLA_OK) raise_status(s, "srla_host_alloc");
        p_ = static_cast<srla_entry*>(q);
        cap_ = c;
    }
    srla_entry* data() const noexcept { return p_; }
    uint64_t size() const noexcept { return cap_; }
    const srla_entry& operator[](uint64_t i) const noexcept { return p_[i]; }

  private:
    srla_entry* p_ = nullptr;
    uint64_t cap_ = 0;
};

[[noreturn]] inline void raise_status(srla_status st, const char* call) {
    const std::string msg = srla_last_error();
    if (st == SRLA_E_INVALID) throw std::invalid_argument(msg);
    if (st == SRLA_E_RANGE) throw std::out_of_range(msg);
    throw std::runtime_error(std::string(call) + ": " + msg);
}
inline void check(srla_status st, const char* call) {
    if (st != SRLA_OK) raise_status(st, call);
}
struct EngineDeleter {
    void operator()(srla_engine* e) const noexcept { srla_destroy(e); }
};
inline srla_config to_c(const SeaConfig& c) {
    srla_config x{};
    x.rows = c.rows;
    x.cols = c.cols;
    x.rough_slots = c.rough_slots;
    x.linear_slots = c.linear_slots;
    x.recorder_bits = c.recorder_bits;
    x.window = c.window;
    x.theta = c.theta;
    x.fill_ratio = c.fill_ratio;
    x.seed = c.seed;
    return x;
}
inline WindowEntry to_entry(const srla_entry& e) {
    WindowEntry w;
    w.host = e.host;
    w.union_weight = e.union_weight;
    if (e.has_estimate) w.estimate = e.estimate;
    w.is_super = e.is_super != 0;
    return w;
}

// Entries handed from the engine's buffer into a report: a single thread is
// host-memory bound (~10 ns per entry: 24 B read + 32 B written), so large
// reports (C2: ~750k entries) are converted on up to 16 threads.
inline void fill_entries(std::vector<WindowEntry>& out, const srla_entry* in, uint64_t n) {
    out.resize(n);
    const uint64_t per = 65536;
    const uint64_t hw = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t t = std::min<uint64_t>({16, hw, (n + per - 1) / per});
    auto run = [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) out[i] = to_entry(in[i]);
    };
    if (t <= 1) return run(0, n);
    std::vector<std::thread> pool;
    for (uint64_t w = 1; w < t; ++w) pool.emplace_back(run, n * w / t, n * (w + 1) / t);
    run(0, n / t);
    for (auto& th : pool) th.join();
}

}  // namespace detail

template <RecorderWord W>
class DetectPipeline;

template <RecorderWord W>
class EstimatorArray {
  public:
    explicit EstimatorArray(const SeaConfig& cfg, int device = 0)
        : cfg_(cfg),
          model_(RecorderModel::with_bits(cfg.recorder_bits)),
          hashes_(cfg.seed),
          params_(DetectionParams::make(cfg.theta, cfg.rough_slots, cfg.window, cfg.fill_ratio)),
          st_(std::make_unique<State>()) {
        cfg_.validate();
        if (!model_.template fits<W>()) throw std::invalid_argument("recorder width exceeds the array's storage word");
        if (recorder_word_bytes(cfg_.recorder_bits) != sizeof(W))
            throw std::invalid_argument("storage word does not match the recorder width (use with_recorder_word)");
        if (cfg_.rows > 64) throw std::invalid_argument("at most 64 rows supported");
        const srla_config c = detail::to_c(cfg_);
        srla_engine* e = nullptr;
        detail::check(srla_create(&c, device, &e), "srla_create");
        eng_.reset(e);
        uint32_t tau = 0, wb = 0;
        detail::check(srla_params(e, &tau, &threshold_, &wb), "srla_params");
    }

    EstimatorArray(EstimatorArray&&) noexcept = default;
    EstimatorArray& operator=(EstimatorArray&&) noexcept = default;

    const SeaConfig& config() const noexcept { return cfg_; }
    const RecorderModel& model() const noexcept { return model_; }
    const HashFamily& hashes() const noexcept { return hashes_; }
    const DetectionParams& params() const noexcept { return params_; }
    uint32_t weight_threshold() const noexcept { return threshold_; }

    uint32_t column_of(uint32_t row, uint32_t aip) const { return hashes_.reduce(kRowHashBase + row, aip, cfg_.cols); }

    // sea.hpp:150-196 — one pair; pushes (if any) appended to the sink.
    void scan_ip_pair(uint32_t aip, uint32_t bip, std::vector<uint32_t>& candidate_sink) {
        const TraceRecord r{0, aip, bip};
        scan_records(std::span<const TraceRecord>(&r, 1), candidate_sink);
    }

    // Batched scan_ip_pair over records in order (host memory).
    void scan_records(std::span<const TraceRecord> records, std::vector<uint32_t>& candidate_sink) {
        std::lock_guard<std::mutex> lk(st_->scan_mu);
        user_mode();
        to_device();
        const size_t at = candidate_sink.size();
        candidate_sink.resize(at + records.size());
        uint64_t n = 0;
        detail::check(srla_scan_batch(eng(), reinterpret_cast<const srla_record*>(records.data()), records.size(), 0,
                                      candidate_sink.data() + at, records.size(), &n),
                      "srla_scan_batch");
        candidate_sink.resize(at + n);
        st_->mirror_valid = false;
    }

    UnionView<W> union_view(uint32_t aip, bool include_linear) const {
        to_device();
        UnionView<W> u;
        std::vector<uint32_t> r(cfg_.rough_slots), l(include_linear ? cfg_.linear_slots : 0);
        detail::check(srla_union_view(eng(), aip, &u.indicator, r.data(), include_linear ? l.data() : nullptr),
                      "srla_union_view");
        u.rough.assign(r.begin(), r.end());
        if (include_linear) u.linear.assign(l.begin(), l.end());
        return u;
    }

    uint32_t union_rough_weight(uint32_t aip) const {
        to_device();
        uint32_t w = 0;
        detail::check(srla_union_weights(eng(), &aip, 1, &w, nullptr), "srla_union_weights");
        return w;
    }

    uint32_t union_linear_weight(uint32_t aip) const {
        to_device();
        uint32_t w = 0;
        detail::check(srla_union_weights(eng(), &aip, 1, nullptr, &w), "srla_union_weights");
        return w;
    }

    double row_fill_fraction(uint32_t row, const ChunkRunner& = serial_chunks) const {
        if (row >= cfg_.rows) throw std::invalid_argument("row index out of range");
        const auto a = row_active();
        return static_cast<double>(a[row]) / static_cast<double>(uint64_t(cfg_.cols) * cfg_.linear_slots);
    }

    double union_fill_product(const ChunkRunner& = serial_chunks) const {
        const auto a = row_active();
        const double words = static_cast<double>(uint64_t(cfg_.cols) * cfg_.linear_slots);
        double p = 1.0;
        for (uint32_t i = 0; i < cfg_.rows; ++i) p *= static_cast<double>(a[i]) / words;
        return p;
    }

    std::optional<double> corrected_estimate_from(uint32_t weight, double fill_product) const {
        double v = 0.0;
        int has = 0;
        detail::check(srla_estimate_from(eng(), weight, fill_product, &v, &has), "srla_estimate_from");
        return has ? std::optional<double>(v) : std::nullopt;
    }

    std::optional<double> corrected_estimate(uint32_t aip, const ChunkRunner& chunks = serial_chunks) const {
        return corrected_estimate_from(union_linear_weight(aip), union_fill_product(chunks));
    }

    // sea.hpp:288-309
    WindowReport report_window(const CandidateList& csip, uint64_t window_start,
                               const ChunkRunner& = serial_chunks) const {
        user_mode();
        to_device();
        set_list(csip.hosts());
        return engine_report(window_start);
    }

    // sea.hpp:316-338
    CandidateList slide(const CandidateList& csip, const ChunkRunner& = serial_chunks) {
        user_mode();
        to_device();
        set_list(csip.hosts());
        uint64_t n = 0;
        detail::check(srla_slide(eng(), &n), "srla_slide");
        st_->mirror_valid = false;
        CandidateList out;
        for (uint32_t h : engine_list()) out.insert(h);
        return out;
    }

    // Raw rows (sea.hpp:341-346), through the host mirror.
    std::span<const uint16_t> indicator_row(uint32_t i) const { return pull().ind.at(i); }
    std::span<uint16_t> indicator_row(uint32_t i) { return {touch().ind.at(i)}; }
    std::span<const W> rough_row(uint32_t i) const { return pull().rough.at(i); }
    std::span<W> rough_row(uint32_t i) { return {touch().rough.at(i)}; }
    std::span<const W> linear_row(uint32_t i) const { return pull().lin.at(i); }
    std::span<W> linear_row(uint32_t i) { return {touch().lin.at(i)}; }

    // The engine handle (for callers that drive the C ABI directly).
    srla_engine* engine_handle() const noexcept { return eng_.get(); }

  private:
    friend class DetectPipeline<W>;
    template <RecorderWord V>
    friend void save_snapshot(const EstimatorArray<V>&, const CandidateList&, const std::string&);
    template <RecorderWord V>
    friend std::pair<EstimatorArray<V>, CandidateList> load_snapshot(const std::string&, int);

    struct Mirror {
        std::vector<std::vector<uint16_t>> ind;
        std::vector<std::vector<W>> rough, lin;
    };
    struct State {
        std::mutex scan_mu;
        Mirror mirror;
        bool mirror_valid = false;
        bool mirror_dirty = false;
        bool pipeline_owns_list = true;  // the engine's candidate list belongs to a DetectPipeline
        std::vector<uint32_t> saved_pipeline_list;
    };

    srla_engine* eng() const noexcept { return eng_.get(); }

    std::vector<uint64_t> row_active() const {
        to_device();
        std::vector<uint64_t> a(cfg_.rows);
        detail::check(srla_row_active(eng(), a.data()), "srla_row_active");
        return a;
    }

    std::vector<uint32_t> engine_list() const {
        uint64_t n = 0;
        srla_status s = srla_candidates(eng(), nullptr, 0, &n);
        if (s != SRLA_OK && s != SRLA_E_CAPACITY) detail::raise_status(s, "srla_candidates");
        std::vector<uint32_t> v(n);
        detail::check(srla_candidates(eng(), v.data(), n, &n), "srla_candidates");
        return v;
    }
    void set_list(const std::vector<uint32_t>& h) const {
        detail::check(srla_set_candidates(eng(), h.data(), h.size()), "srla_set_candidates");
    }
    // the reference keeps a DetectPipeline's list outside the sketch; the
    // engine keeps it on the device, so direct sketch calls park it first
    void user_mode() const {
        if (st_->pipeline_owns_list) {
            st_->saved_pipeline_list = engine_list();
            st_->pipeline_owns_list = false;
        }
    }
    void pipeline_mode() const {
        if (!st_->pipeline_owns_list) {
            set_list(st_->saved_pipeline_list);
            st_->saved_pipeline_list.clear();
            st_->pipeline_owns_list = true;
        }
    }

    WindowReport engine_report(uint64_t window_start) const {
        const auto t0 = std::chrono::steady_clock::now();
        WindowReport rep;
        rep.window_start = window_start;
        rep.window = cfg_.window;
        uint64_t n = 0;
        srla_status s = srla_candidates(eng(), nullptr, 0, &n);
        if (s != SRLA_OK && s != SRLA_E_CAPACITY) detail::raise_status(s, "srla_candidates");
        std::vector<srla_entry> buf(n);
        double fp = 0.0;
        detail::check(srla_report(eng(), buf.data(), buf.size(), &n, &fp), "srla_report");
        detail::fill_entries(rep.entries, buf.data(), n);
        rep.estimate_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        return rep;
    }

    uint64_t words(int kind) const {
        uint64_t b = 0;
        detail::check(srla_row_bytes(eng(), kind, &b), "srla_row_bytes");
        return b / (kind == SRLA_INDICATOR ? 2 : sizeof(W));
    }

    Mirror& pull() const {
        Mirror& m = st_->mirror;
        if (!st_->mirror_valid && !st_->mirror_dirty) {
            m.ind.resize(cfg_.rows);
            m.rough.resize(cfg_.rows);
            m.lin.resize(cfg_.rows);
            for (uint32_t i = 0; i < cfg_.rows; ++i) {
                m.ind[i].resize(words(SRLA_INDICATOR));
                m.rough[i].resize(words(SRLA_ROUGH));
                m.lin[i].resize(words(SRLA_LINEAR));
                detail::check(srla_export_row(eng(), i, SRLA_INDICATOR, m.ind[i].data(), m.ind[i].size() * 2), "export");
                detail::check(srla_export_row(eng(), i, SRLA_ROUGH, m.rough[i].data(), m.rough[i].size() * sizeof(W)), "export");
                detail::check(srla_export_row(eng(), i, SRLA_LINEAR, m.lin[i].data(), m.lin[i].size() * sizeof(W)), "export");
            }
            st_->mirror_valid = true;
        }
        return m;
    }
    Mirror& touch() {
        Mirror& m = pull();
        st_->mirror_dirty = true;
        return m;
    }
    void to_device() const {
        if (!st_->mirror_dirty) return;
        const Mirror& m = st_->mirror;
        for (uint32_t i = 0; i < cfg_.rows; ++i) {
            detail::check(srla_import_row(eng(), i, SRLA_INDICATOR, m.ind[i].data(), m.ind[i].size() * 2), "import");
            detail::check(srla_import_row(eng(), i, SRLA_ROUGH, m.rough[i].data(), m.rough[i].size() * sizeof(W)), "import");
            detail::check(srla_import_row(eng(), i, SRLA_LINEAR, m.lin[i].data(), m.lin[i].size() * sizeof(W)), "import");
        }
        st_->mirror_dirty = false;
        st_->mirror_valid = true;
    }

    SeaConfig cfg_;
    RecorderModel model_;
    HashFamily hashes_;
    DetectionParams params_;
    uint32_t threshold_ = 0;
    std::unique_ptr<State> st_;
    std::unique_ptr<srla_engine, detail::EngineDeleter> eng_;
};

}  // namespace sspread
