// sspread/oracle.hpp — drop-in exact ground truth
// (/root/reference/proj/include/sspread/oracle.hpp) on the B200.
//
// The reference's "precise method" keeps a hash-map entry per live pair on the
// host. Both of its stores are served here by one device store (srla_exact_*,
// csrc/exact.cu): each slice a sorted, deduplicated array of pair keys in HBM,
// a window query a radix sort + unique + run-length encode over its slices.
// observe() only appends to a host buffer; the buffer crosses to the device in
// batches. Results equal the reference's on every query (tests/test_exact*).
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <optional>
#include <set>
#include <utility>
#include <vector>

#include "sea.hpp"

namespace sspread {

/// Detection quality (oracle.hpp:17-26): of N true super points the detector
/// reported N' hosts, N+ of them wrong, and missed N-.
struct AccuracyMetrics {
    uint64_t truth_size = 0;       // N
    uint64_t detected_size = 0;    // N'
    uint64_t false_positives = 0;  // N+
    uint64_t false_negatives = 0;  // N-
    double fpr = 0;
    double fnr = 0;
    double tfr = 0;
};

/// oracle.hpp:30-43: undefined (empty) for an empty truth set.
inline std::optional<AccuracyMetrics> score(const std::set<uint32_t>& detected, const std::set<uint32_t>& truth) {
    if (truth.empty()) return std::nullopt;
    AccuracyMetrics m;
    m.truth_size = truth.size();
    m.detected_size = detected.size();
    // both sets are ordered: one merge pass counts the two differences
    auto d = detected.begin();
    auto t = truth.begin();
    while (d != detected.end() || t != truth.end()) {
        if (t == truth.end() || (d != detected.end() && *d < *t)) {
            ++m.false_positives;
            ++d;
        } else if (d == detected.end() || *t < *d) {
            ++m.false_negatives;
            ++t;
        } else {
            ++d;
            ++t;
        }
    }
    const double n = static_cast<double>(m.truth_size);
    m.fpr = static_cast<double>(m.false_positives) / n;
    m.fnr = static_cast<double>(m.false_negatives) / n;
    m.tfr = m.fpr + m.fnr;
    return m;
}

namespace detail {

// The device store behind both reference stores, with a host-side batch of
// observed pairs and a cache of the last window queried.
class ExactStore {
  public:
    ExactStore(uint32_t max_window, int device) {
        srla_exact* x = nullptr;
        check(srla_exact_create(max_window, device, &x), "srla_exact_create");
        x_.reset(x);
    }

    void observe(uint32_t aip, uint32_t bip) {
        batch_.push_back(srla_record{0, aip, bip});
        cache_valid_ = false;
        if (batch_.size() >= kBatch) flush();
    }
    void end_slice() {
        flush();
        check(srla_exact_end_slice(x_.get()), "srla_exact_end_slice");
        cache_valid_ = false;
    }
    uint64_t current_slice() const {
        uint64_t s = 0;
        check(srla_exact_current_slice(x_.get(), &s), "srla_exact_current_slice");
        return s;
    }
    uint64_t pair_count() {
        flush();
        uint64_t n = 0;
        check(srla_exact_pair_count(x_.get(), &n), "srla_exact_pair_count");
        return n;
    }
    // (host, distinct count) of every host with a nonzero count, ascending
    const std::vector<std::pair<uint32_t, uint64_t>>& window(uint64_t t, uint32_t k) {
        flush();
        if (cache_valid_ && cache_t_ == t && cache_k_ == k) return cache_;
        uint64_t n = 0;
        srla_status s = srla_exact_cardinalities(x_.get(), t, k, nullptr, nullptr, 0, &n);
        if (s != SRLA_OK && s != SRLA_E_CAPACITY) raise_status(s, "srla_exact_cardinalities");
        std::vector<uint32_t> hosts(n);
        std::vector<uint64_t> counts(n);
        check(srla_exact_cardinalities(x_.get(), t, k, hosts.data(), counts.data(), n, &n), "srla_exact_cardinalities");
        cache_.resize(n);
        for (uint64_t i = 0; i < n; ++i) cache_[i] = {hosts[i], counts[i]};
        cache_t_ = t;
        cache_k_ = k;
        cache_valid_ = true;
        return cache_;
    }
    uint64_t cardinality(uint32_t aip, uint64_t t, uint32_t k) {
        const auto& w = window(t, k);
        const auto it = std::lower_bound(w.begin(), w.end(), std::make_pair(aip, uint64_t{0}));
        return it != w.end() && it->first == aip ? it->second : 0;
    }
    std::set<uint32_t> super_points(uint64_t t, uint32_t k, uint32_t theta) {
        std::set<uint32_t> out;
        for (const auto& [host, n] : window(t, k))
            if (n >= theta) out.insert(out.end(), host);
        return out;
    }

  private:
    static constexpr size_t kBatch = size_t(1) << 20;
    struct Deleter {
        void operator()(srla_exact* x) const { srla_exact_destroy(x); }
    };
    void flush() {
        if (batch_.empty()) return;
        check(srla_exact_observe(x_.get(), batch_.data(), batch_.size(), 0), "srla_exact_observe");
        batch_.clear();
    }
    std::unique_ptr<srla_exact, Deleter> x_;
    std::vector<srla_record> batch_;
    std::vector<std::pair<uint32_t, uint64_t>> cache_;
    uint64_t cache_t_ = 0;
    uint32_t cache_k_ = 0;
    bool cache_valid_ = false;
};

}  // namespace detail

/// oracle.hpp:48-133: exact per-pair sliding cardinalities. The recorder
/// width bounds the window as the reference's does (validate_window).
class PairRecorderStore {
  public:
    explicit PairRecorderStore(uint32_t recorder_bits, uint32_t max_window, int device = 0)
        : store_((RecorderModel::with_bits(recorder_bits).validate_window(max_window), max_window), device) {}

    void observe(uint32_t aip, uint32_t bip) { store_.observe(aip, bip); }
    void end_slice() { store_.end_slice(); }
    uint64_t current_slice() const { return store_.current_slice(); }
    uint64_t pair_count() const { return store_.pair_count(); }
    uint64_t cardinality(uint32_t aip, uint64_t t, uint32_t k) const { return store_.cardinality(aip, t, k); }
    std::set<uint32_t> super_points(uint64_t t, uint32_t k, uint32_t theta) const {
        return store_.super_points(t, k, theta);
    }
    std::vector<std::pair<uint32_t, uint64_t>> cardinalities(uint64_t t, uint32_t k) const { return store_.window(t, k); }

  private:
    mutable detail::ExactStore store_;  // queries flush the host-side batch
};

/// oracle.hpp:136-203: the independent ring-of-slices implementation; here the
/// same device store (the reference cross-checks its two stores against each
/// other; tests/test_exact_gpu.py checks this one against both of them).
class SliceRingStore {
  public:
    explicit SliceRingStore(uint32_t max_window, int device = 0)
        : store_((max_window < 1 ? throw std::invalid_argument("window must be >= 1") : max_window), device) {}

    void observe(uint32_t aip, uint32_t bip) { store_.observe(aip, bip); }
    void end_slice() { store_.end_slice(); }
    uint64_t current_slice() const { return store_.current_slice(); }
    uint64_t cardinality(uint32_t aip, uint64_t t, uint32_t k) const { return store_.cardinality(aip, t, k); }
    std::set<uint32_t> super_points(uint64_t t, uint32_t k, uint32_t theta) const {
        return store_.super_points(t, k, theta);
    }
    std::vector<std::pair<uint32_t, uint64_t>> cardinalities(uint64_t t, uint32_t k) const { return store_.window(t, k); }

  private:
    mutable detail::ExactStore store_;  // queries flush the host-side batch
};

}  // namespace sspread
