// ref_capi.cpp — C ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include/sspread/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libsspread_ref.so. TEST INFRASTRUCTURE ONLY: it pins the C
// restatement (srla_oracle.c) against the real reference, generates the golden
// fixtures under tests/golden/, and is the CPU baseline of bench.py's
// reference arm. No reference source is copied here; this file only calls the
// reference's public API with the same entry points as srla_oracle.h
// (prefix `ref_` instead of `orc_`).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sspread/generator.hpp"
#include "sspread/oracle.hpp"
#include "sspread/pipeline.hpp"
#include "sspread/sea.hpp"
#include "sspread/snapshot.hpp"
#include "sspread/trace.hpp"

#include "srla_oracle.h"  // shared struct layouts (orc_config, orc_spec, kinds)

using namespace sspread;

namespace {

SeaConfig to_sea(const orc_config* c) {
    SeaConfig s;
    s.rows = c->rows;
    s.cols = c->cols;
    s.rough_slots = c->rough_slots;
    s.linear_slots = c->linear_slots;
    s.recorder_bits = c->recorder_bits;
    s.window = c->window;
    s.theta = c->theta;
    s.fill_ratio = c->fill_ratio;
    s.seed = c->seed;
    return s;
}

void set_err(char* err, size_t errlen, const char* msg) {
    if (err && errlen) std::snprintf(err, errlen, "%s", msg);
}

struct SeaBase {
    virtual ~SeaBase() = default;
    virtual uint32_t tau() = 0;
    virtual uint32_t threshold() = 0;
    virtual uint32_t word_bytes() = 0;
    virtual uint32_t column_of(uint32_t row, uint32_t aip) = 0;
    virtual uint64_t row_len(int kind) = 0;
    virtual void scan(const uint32_t* recs, uint64_t n, uint32_t* sink, uint64_t* nsink) = 0;
    virtual uint32_t urw(uint32_t) = 0;
    virtual uint32_t ulw(uint32_t) = 0;
    virtual uint16_t view(uint32_t aip, uint32_t* rough, uint32_t* linear) = 0;
    virtual uint64_t row_active(uint32_t row) = 0;
    virtual double rff(uint32_t row) = 0;
    virtual double ufp() = 0;
    virtual int cef(uint32_t w, double fp, double* out) = 0;
    virtual void report(const uint32_t* csip, uint64_t n, uint32_t* hosts, uint32_t* weights,
                        double* est, uint8_t* has, uint8_t* sup) = 0;
    virtual uint64_t slide(const uint32_t* csip, uint64_t n, uint32_t* retained) = 0;
    virtual void export_row(uint32_t row, int kind, void* buf) = 0;
    virtual void import_row(uint32_t row, int kind, const void* buf) = 0;
};

CandidateList to_list(const uint32_t* csip, uint64_t n) {
    CandidateList l;
    for (uint64_t i = 0; i < n; ++i) l.insert(csip[i]);
    return l;
}

void put_report(const WindowReport& r, uint32_t* hosts, uint32_t* weights, double* est,
                uint8_t* has, uint8_t* sup) {
    for (size_t e = 0; e < r.entries.size(); ++e) {
        hosts[e] = r.entries[e].host;
        weights[e] = r.entries[e].union_weight;
        has[e] = r.entries[e].estimate.has_value();
        est[e] = r.entries[e].estimate.value_or(0.0);
        sup[e] = r.entries[e].is_super;
    }
}

template <RecorderWord W>
struct Sea final : SeaBase {
    EstimatorArray<W>* a;  // not owned when borrowed from a pipeline
    std::unique_ptr<EstimatorArray<W>> own;
    explicit Sea(const SeaConfig& c) : own(std::make_unique<EstimatorArray<W>>(c)) { a = own.get(); }
    explicit Sea(EstimatorArray<W>* borrowed) : a(borrowed) {}
    uint32_t tau() override { return a->params().tau; }
    uint32_t threshold() override { return a->weight_threshold(); }
    uint32_t word_bytes() override { return sizeof(W); }
    uint32_t column_of(uint32_t row, uint32_t aip) override { return a->column_of(row, aip); }
    uint64_t row_len(int kind) override {
        if (kind == ORC_INDICATOR) return a->indicator_row(0).size();
        if (kind == ORC_ROUGH) return a->rough_row(0).size();
        return a->linear_row(0).size();
    }
    void scan(const uint32_t* recs, uint64_t n, uint32_t* sink, uint64_t* nsink) override {
        std::vector<uint32_t> s;
        for (uint64_t r = 0; r < n; ++r) a->scan_ip_pair(recs[3 * r + 1], recs[3 * r + 2], s);
        std::memcpy(sink, s.data(), s.size() * sizeof(uint32_t));
        *nsink = s.size();
    }
    uint32_t urw(uint32_t h) override { return a->union_rough_weight(h); }
    uint32_t ulw(uint32_t h) override { return a->union_linear_weight(h); }
    uint16_t view(uint32_t aip, uint32_t* rough, uint32_t* linear) override {
        const auto u = a->union_view(aip, linear != nullptr);
        for (size_t j = 0; j < u.rough.size(); ++j) rough[j] = u.rough[j];
        if (linear)
            for (size_t j = 0; j < u.linear.size(); ++j) linear[j] = u.linear[j];
        return u.indicator;
    }
    uint64_t row_active(uint32_t row) override {
        return count_active(a->linear_row(row), a->config().window);
    }
    double rff(uint32_t row) override { return a->row_fill_fraction(row); }
    double ufp() override { return a->union_fill_product(); }
    int cef(uint32_t w, double fp, double* out) override {
        const auto e = a->corrected_estimate_from(w, fp);
        if (e) *out = *e;
        return e.has_value();
    }
    void report(const uint32_t* csip, uint64_t n, uint32_t* hosts, uint32_t* weights, double* est,
                uint8_t* has, uint8_t* sup) override {
        put_report(a->report_window(to_list(csip, n), 0), hosts, weights, est, has, sup);
    }
    uint64_t slide(const uint32_t* csip, uint64_t n, uint32_t* retained) override {
        const auto out = a->slide(to_list(csip, n));
        std::memcpy(retained, out.hosts().data(), out.size() * sizeof(uint32_t));
        return out.size();
    }
    void export_row(uint32_t row, int kind, void* buf) override {
        if (kind == ORC_INDICATOR) {
            const auto r = a->indicator_row(row);
            std::memcpy(buf, r.data(), r.size() * 2);
        } else {
            const auto r = kind == ORC_ROUGH ? a->rough_row(row) : a->linear_row(row);
            std::memcpy(buf, r.data(), r.size() * sizeof(W));  // x86: little-endian
        }
    }
    void import_row(uint32_t row, int kind, const void* buf) override {
        if (kind == ORC_INDICATOR) {
            auto r = a->indicator_row(row);
            std::memcpy(r.data(), buf, r.size() * 2);
        } else {
            auto r = kind == ORC_ROUGH ? a->rough_row(row) : a->linear_row(row);
            std::memcpy(r.data(), buf, r.size() * sizeof(W));
        }
    }
};

struct PipeBase {
    virtual ~PipeBase() = default;
    std::unique_ptr<SeaBase> sea;
    virtual void process(uint64_t id, const uint32_t* recs, uint64_t n, int want, int* reported,
                         uint64_t* ne, uint32_t* hosts, uint32_t* weights, double* est,
                         uint8_t* has, uint8_t* sup) = 0;
    virtual uint64_t ncand() = 0;
    virtual void cands(uint32_t* out) = 0;
    virtual double scan_ms() = 0;
    virtual double est_ms() = 0;
    virtual void save(const char* path) = 0;
};

template <RecorderWord W>
struct Pipe final : PipeBase {
    DetectPipeline<W> p;
    std::vector<TraceRecord> buf;
    explicit Pipe(const RunConfig& rc) : p(rc) { sea = std::make_unique<Sea<W>>(&p.sketch()); }
    void process(uint64_t id, const uint32_t* recs, uint64_t n, int want, int* reported,
                 uint64_t* ne, uint32_t* hosts, uint32_t* weights, double* est, uint8_t* has,
                 uint8_t* sup) override {
        static_assert(sizeof(TraceRecord) == 12);
        const std::span<const TraceRecord> records(reinterpret_cast<const TraceRecord*>(recs), n);
        *reported = 0;
        *ne = 0;
        typename DetectPipeline<W>::ReportSink sink;
        if (want)
            sink = [&](const WindowReport& r) {
                *reported = 1;
                *ne = r.entries.size();
                if (hosts) put_report(r, hosts, weights, est, has, sup);
            };
        p.process_slice(id, records, sink);
    }
    uint64_t ncand() override { return p.candidates().size(); }
    void cands(uint32_t* out) override {
        const auto& h = p.candidates().hosts();
        std::memcpy(out, h.data(), h.size() * sizeof(uint32_t));
    }
    double scan_ms() override { return p.total_scan_ms(); }
    double est_ms() override { return p.total_estimate_ms(); }
    void save(const char* path) override { save_snapshot(p.sketch(), p.candidates(), path); }  // snapshot.hpp:109-136
};

SeaBase* S(void* h) { return static_cast<SeaBase*>(h); }

PlantSpec to_spec(const orc_spec* s) {
    PlantSpec spec;
    spec.seed = s->seed;
    spec.start_ts = s->start_ts;
    spec.slice_seconds = s->slice_seconds;
    spec.slices = s->slices;
    spec.window = s->window;
    spec.a_base = s->a_base;
    spec.b_base = s->b_base;
    spec.background = {s->a_hosts, s->b_hosts, s->pairs_per_slice, s->skew};
    for (uint32_t i = 0; i < s->n_plants; ++i)
        spec.plants.push_back({s->plants[i].host, s->plants[i].cardinality, s->plants[i].first_slice,
                               s->plants[i].last_slice});
    return spec;
}

// Records the plants contribute to slice s (generator.hpp:127-139).
uint64_t plant_records(const PlantSpec& spec, uint64_t s) {
    uint64_t n = 0;
    for (const auto& p : spec.plants) {
        if (!p.active_in(s)) continue;
        const uint32_t r = static_cast<uint32_t>((s - p.first_slice) % spec.window);
        const auto [lo, hi] = detail::rotation_chunk(p.cardinality, spec.window, r);
        n += hi - lo;
    }
    return n;
}

// Block digest of a little-endian byte row: per 1 MiB block, the wrapping sum
// over its 8-byte words w (zero-padded) of avalanche64(w ^ avalanche64(i + 1)),
// i = the word's index within the row. The engine computes the same sums on
// the device (srla_state_blocks); tests compare sha256 over them.
constexpr uint64_t kDigestBlock = 1ull << 20;

void block_sums(const uint8_t* p, uint64_t bytes, uint32_t threads, uint64_t* out) {
    const uint64_t nb = (bytes + kDigestBlock - 1) / kDigestBlock;
    parallel_ranges(nb, std::max<uint32_t>(threads, 1), [&](uint64_t b0, uint64_t b1) {
        for (uint64_t b = b0; b < b1; ++b) {
            const uint64_t lo = b * kDigestBlock, hi = std::min(bytes, lo + kDigestBlock);
            uint64_t acc = 0;
            for (uint64_t o = lo; o < hi; o += 8) {
                uint64_t w = 0;
                std::memcpy(&w, p + o, std::min<uint64_t>(8, hi - o));
                acc += avalanche64(w ^ avalanche64(o / 8 + 1));
            }
            out[b] = acc;
        }
    });
}

// One sketch + candidate list driven like DetectPipeline::process_slice with
// ONE scan worker (pipeline.hpp:110-139: record order, the parity definition
// of SURVEY.md §8c), its bulk passes (report_window's fill product, slide)
// chunked over `threads` — ChunkRunner splits do not change results
// (sea.hpp:23-26).
struct FlowBase {
    virtual ~FlowBase() = default;
    virtual uint64_t scan(const uint32_t* recs, uint64_t n, std::vector<uint32_t>& pushes) = 0;
    virtual const std::vector<uint32_t>& cands() = 0;
    virtual uint64_t report(uint64_t window_start, uint32_t* hosts, uint32_t* weights, double* est, uint8_t* has,
                            uint8_t* sup) = 0;
    virtual uint64_t slide() = 0;
    virtual void state_blocks(uint32_t row, int kind, uint64_t* out) = 0;
    virtual uint64_t row_bytes(int kind) = 0;
    std::vector<uint32_t> pushes;
};

template <RecorderWord W>
struct Flow final : FlowBase {
    EstimatorArray<W> a;
    CandidateList csip;
    uint32_t threads;
    Flow(const SeaConfig& c, uint32_t t) : a(c), threads(t) {}
    uint64_t scan(const uint32_t* recs, uint64_t n, std::vector<uint32_t>& sink) override {
        sink.clear();
        for (uint64_t r = 0; r < n; ++r) a.scan_ip_pair(recs[3 * r + 1], recs[3 * r + 2], sink);
        for (uint32_t h : sink) csip.insert(h);
        return sink.size();
    }
    const std::vector<uint32_t>& cands() override { return csip.hosts(); }
    uint64_t report(uint64_t ws, uint32_t* hosts, uint32_t* weights, double* est, uint8_t* has,
                    uint8_t* sup) override {
        const auto r = a.report_window(csip, ws, chunked(threads));
        if (hosts) put_report(r, hosts, weights, est, has, sup);
        return r.entries.size();
    }
    uint64_t slide() override {
        csip = a.slide(csip, chunked(threads));
        return csip.size();
    }
    uint64_t row_bytes(int kind) override {
        if (kind == ORC_INDICATOR) return a.indicator_row(0).size() * 2;
        if (kind == ORC_ROUGH) return a.rough_row(0).size() * sizeof(W);
        return a.linear_row(0).size() * sizeof(W);
    }
    void state_blocks(uint32_t row, int kind, uint64_t* out) override {
        const uint8_t* p = kind == ORC_INDICATOR ? reinterpret_cast<const uint8_t*>(a.indicator_row(row).data())
                           : kind == ORC_ROUGH   ? reinterpret_cast<const uint8_t*>(a.rough_row(row).data())
                                                 : reinterpret_cast<const uint8_t*>(a.linear_row(row).data());
        block_sums(p, row_bytes(kind), threads, out);  // x86: words already little-endian
    }
};

}  // namespace

extern "C" {

uint64_t ref_avalanche64(uint64_t x) { return avalanche64(x); }
uint32_t ref_hash_u32(uint64_t seed, uint32_t index, uint32_t key) { return HashFamily(seed).u32(index, key); }
uint32_t ref_hash_reduce(uint64_t seed, uint32_t index, uint32_t key, uint32_t range) {
    return HashFamily(seed).reduce(index, key, range);
}
uint32_t ref_sampling_exponent(uint64_t theta, uint64_t slots) { return sampling_exponent(theta, slots); }
uint32_t ref_super_weight_threshold(double ratio, uint32_t slots) { return super_weight_threshold(ratio, slots); }
double ref_super_test_ratio(void) { return kSuperTestRatio; }
int ref_linear_estimate(uint32_t weight, uint32_t slots, double* out) {
    const auto e = linear_estimate(weight, slots);
    if (e) *out = *e;
    return e.has_value();
}

void* ref_create(const orc_config* cfg, char* err, size_t errlen) {
    try {
        const SeaConfig c = to_sea(cfg);
        return with_recorder_word(c.recorder_bits, [&](auto word) -> void* {
            using Word = decltype(word);
            return static_cast<SeaBase*>(new Sea<Word>(c));
        });
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
void ref_destroy(void* h) { delete S(h); }
uint32_t ref_tau(void* h) { return S(h)->tau(); }
uint32_t ref_threshold(void* h) { return S(h)->threshold(); }
uint32_t ref_word_bytes(void* h) { return S(h)->word_bytes(); }
uint32_t ref_column_of(void* h, uint32_t row, uint32_t aip) { return S(h)->column_of(row, aip); }
uint64_t ref_row_len(void* h, int kind) { return S(h)->row_len(kind); }
void ref_scan(void* h, const uint32_t* recs, uint64_t n, uint32_t* sink, uint64_t* nsink) {
    S(h)->scan(recs, n, sink, nsink);
}
uint32_t ref_union_rough_weight(void* h, uint32_t aip) { return S(h)->urw(aip); }
uint32_t ref_union_linear_weight(void* h, uint32_t aip) { return S(h)->ulw(aip); }
uint16_t ref_union_view(void* h, uint32_t aip, uint32_t* rough, uint32_t* linear) {
    return S(h)->view(aip, rough, linear);
}
uint64_t ref_row_active(void* h, uint32_t row) { return S(h)->row_active(row); }
double ref_row_fill_fraction(void* h, uint32_t row) { return S(h)->rff(row); }
double ref_union_fill_product(void* h) { return S(h)->ufp(); }
int ref_corrected_estimate_from(void* h, uint32_t w, double fp, double* out) { return S(h)->cef(w, fp, out); }
void ref_report(void* h, const uint32_t* csip, uint64_t n, uint32_t* hosts, uint32_t* weights,
                double* est, uint8_t* has, uint8_t* sup) {
    S(h)->report(csip, n, hosts, weights, est, has, sup);
}
uint64_t ref_slide(void* h, const uint32_t* csip, uint64_t n, uint32_t* retained) {
    return S(h)->slide(csip, n, retained);
}
void ref_export_row(void* h, uint32_t row, int kind, void* buf) { S(h)->export_row(row, kind, buf); }
void ref_import_row(void* h, uint32_t row, int kind, const void* buf) { S(h)->import_row(row, kind, buf); }

void* ref_pipeline_create(const orc_config* cfg, uint32_t workers, char* err, size_t errlen) {
    try {
        RunConfig rc;
        rc.sea = to_sea(cfg);
        rc.workers = workers;
        rc.validate();
        return with_recorder_word(rc.sea.recorder_bits, [&](auto word) -> void* {
            using Word = decltype(word);
            return static_cast<PipeBase*>(new Pipe<Word>(rc));
        });
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
void ref_pipeline_destroy(void* p) { delete static_cast<PipeBase*>(p); }
void* ref_pipeline_sketch(void* p) { return static_cast<PipeBase*>(p)->sea.get(); }
void ref_pipeline_process_slice(void* p, uint64_t slice_id, const uint32_t* recs, uint64_t n,
                                int want_report, int* reported, uint64_t* n_entries,
                                uint32_t* hosts, uint32_t* weights, double* estimates,
                                uint8_t* has_estimate, uint8_t* is_super) {
    static_cast<PipeBase*>(p)->process(slice_id, recs, n, want_report, reported, n_entries, hosts,
                                       weights, estimates, has_estimate, is_super);
}
uint64_t ref_pipeline_ncand(void* p) { return static_cast<PipeBase*>(p)->ncand(); }
void ref_pipeline_candidates(void* p, uint32_t* out) { static_cast<PipeBase*>(p)->cands(out); }
double ref_pipeline_scan_ms(void* p) { return static_cast<PipeBase*>(p)->scan_ms(); }
double ref_pipeline_estimate_ms(void* p) { return static_cast<PipeBase*>(p)->est_ms(); }
// the reference's own save_snapshot of the pipeline's sketch and candidate list
int ref_pipeline_save_snapshot(void* p, const char* path, char* err, size_t errlen) {
    try {
        static_cast<PipeBase*>(p)->save(path);
        return 0;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return 1;
    }
}

uint64_t ref_generate(const orc_spec* s, uint32_t* out, char* err, size_t errlen) {
    try {
        PlantSpec spec;
        spec.seed = s->seed;
        spec.start_ts = s->start_ts;
        spec.slice_seconds = s->slice_seconds;
        spec.slices = s->slices;
        spec.window = s->window;
        spec.a_base = s->a_base;
        spec.b_base = s->b_base;
        spec.background = {s->a_hosts, s->b_hosts, s->pairs_per_slice, s->skew};
        for (uint32_t i = 0; i < s->n_plants; ++i)
            spec.plants.push_back({s->plants[i].host, s->plants[i].cardinality,
                                   s->plants[i].first_slice, s->plants[i].last_slice});
        const auto recs = generate_trace(spec);
        if (out) std::memcpy(out, recs.data(), recs.size() * sizeof(TraceRecord));
        return recs.size();
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return UINT64_MAX;
    }
}

// Slice `slice` of generate_trace (generator.hpp:117-161), produced in
// parallel from the reference's own SplitMix64 / ZipfSampler / rotation
// helpers. The generator's draws are counter-based (hash.hpp:21-24: state +=
// phi per draw) and fixed per record (plant record: ts; background record:
// src, dst, ts), so record j of a slice starts at a known stream offset.
// slice_seconds == 1 only: every ts of a slice equals its base, so the
// per-slice stable sort and the anchoring are identities. out = NULL counts.
uint64_t ref_generate_slice(const orc_spec* s, uint64_t slice, uint32_t threads, uint32_t* out, char* err,
                            size_t errlen) {
    try {
        const PlantSpec spec = to_spec(s);
        spec.validate();
        if (spec.slice_seconds != 1) throw std::invalid_argument("ref_generate_slice needs slice_seconds == 1");
        if (slice >= spec.slices) throw std::invalid_argument("slice out of range");
        uint64_t draws = 0;  // stream position at the start of the slice
        for (uint64_t t = 0; t < slice; ++t) draws += plant_records(spec, t) + 3ull * spec.background.pairs_per_slice;
        const uint64_t np = plant_records(spec, slice);
        const uint64_t n = np + spec.background.pairs_per_slice;
        if (!out) return n;
        constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;
        const uint32_t ts = spec.start_ts + static_cast<uint32_t>(slice) * spec.slice_seconds;
        uint64_t at = 0;
        for (size_t pi = 0; pi < spec.plants.size(); ++pi) {  // one draw (ts) per plant record
            const auto& p = spec.plants[pi];
            if (!p.active_in(slice)) continue;
            const uint32_t r = static_cast<uint32_t>((slice - p.first_slice) % spec.window);
            const auto [lo, hi] = detail::rotation_chunk(p.cardinality, spec.window, r);
            const uint32_t off = detail::plant_pool_offset(pi, spec.background.b_hosts);
            for (uint32_t j = lo; j < hi; ++j, ++at) {
                out[3 * at] = ts;
                out[3 * at + 1] = p.host;
                out[3 * at + 2] = spec.b_base + (off + j) % spec.background.b_hosts;
            }
        }
        const detail::ZipfSampler zipf(spec.background.b_hosts, spec.background.skew);
        const uint64_t base = draws + np;
        parallel_ranges(spec.background.pairs_per_slice, std::max<uint32_t>(threads, 1), [&](uint64_t i0, uint64_t i1) {
            SplitMix64 rng(spec.seed + kPhi * (base + 3 * i0));
            for (uint64_t i = i0; i < i1; ++i) {
                uint32_t* r = out + 3 * (np + i);
                r[1] = spec.a_base + static_cast<uint32_t>(rng.next_below(spec.background.a_hosts));
                r[2] = spec.b_base + zipf.draw(rng);
                r[0] = ts + static_cast<uint32_t>(rng.next_below(spec.slice_seconds));
            }
        });
        return n;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return UINT64_MAX;
    }
}

// ---- record-order flow (the parity definition) at full size
void* ref_flow_create(const orc_config* cfg, uint32_t threads, char* err, size_t errlen) {
    try {
        const SeaConfig c = to_sea(cfg);
        c.validate();
        return with_recorder_word(c.recorder_bits, [&](auto word) -> void* {
            using Word = decltype(word);
            return static_cast<FlowBase*>(new Flow<Word>(c, threads));
        });
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
void ref_flow_destroy(void* f) { delete static_cast<FlowBase*>(f); }
// scan in record order; returns the sink pushes (pushes() reads them)
uint64_t ref_flow_scan(void* f, const uint32_t* recs, uint64_t n) {
    auto* F = static_cast<FlowBase*>(f);
    return F->scan(recs, n, F->pushes);
}
void ref_flow_pushes(void* f, uint32_t* out) {
    const auto& p = static_cast<FlowBase*>(f)->pushes;
    std::memcpy(out, p.data(), p.size() * 4);
}
uint64_t ref_flow_ncand(void* f) { return static_cast<FlowBase*>(f)->cands().size(); }
void ref_flow_candidates(void* f, uint32_t* out) {
    const auto& c = static_cast<FlowBase*>(f)->cands();
    std::memcpy(out, c.data(), c.size() * 4);
}
uint64_t ref_flow_report(void* f, uint64_t window_start, uint32_t* hosts, uint32_t* weights, double* est,
                         uint8_t* has, uint8_t* sup) {
    return static_cast<FlowBase*>(f)->report(window_start, hosts, weights, est, has, sup);
}
uint64_t ref_flow_slide(void* f) { return static_cast<FlowBase*>(f)->slide(); }
uint64_t ref_flow_row_bytes(void* f, int kind) { return static_cast<FlowBase*>(f)->row_bytes(kind); }
void ref_flow_state_blocks(void* f, uint32_t row, int kind, uint64_t* out) {
    static_cast<FlowBase*>(f)->state_blocks(row, kind, out);
}
// the same block sums over any byte buffer (records, exported rows)
void ref_block_sums(const void* p, uint64_t bytes, uint32_t threads, uint64_t* out) {
    block_sums(static_cast<const uint8_t*>(p), bytes, threads, out);
}

// ---- the reference's exact stores (oracle.hpp): ring (engine 0) or pair recorders (engine 1)
struct ExactRef {
    std::unique_ptr<SliceRingStore> ring;
    std::unique_ptr<PairRecorderStore> pairs;
};
void* ref_exact_create(int engine, uint32_t recorder_bits, uint32_t max_window, char* err, size_t errlen) {
    try {
        auto* x = new ExactRef();
        if (engine == 0) x->ring = std::make_unique<SliceRingStore>(max_window);
        else x->pairs = std::make_unique<PairRecorderStore>(recorder_bits, max_window);
        return x;
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return nullptr;
    }
}
void ref_exact_destroy(void* h) { delete static_cast<ExactRef*>(h); }
void ref_exact_observe(void* h, const uint32_t* recs, uint64_t n) {
    auto* x = static_cast<ExactRef*>(h);
    for (uint64_t i = 0; i < n; ++i) {
        if (x->ring) x->ring->observe(recs[3 * i + 1], recs[3 * i + 2]);
        else x->pairs->observe(recs[3 * i + 1], recs[3 * i + 2]);
    }
}
void ref_exact_end_slice(void* h) {
    auto* x = static_cast<ExactRef*>(h);
    if (x->ring) x->ring->end_slice();
    else x->pairs->end_slice();
}
uint64_t ref_exact_pair_count(void* h) {
    auto* x = static_cast<ExactRef*>(h);
    return x->pairs ? x->pairs->pair_count() : 0;
}
// cardinalities(t, k) sorted by host; returns the count (-1 as UINT64_MAX on a throw: err holds the message)
uint64_t ref_exact_cardinalities(void* h, uint64_t t, uint32_t k, uint32_t* hosts, uint64_t* counts, char* err,
                                 size_t errlen) {
    auto* x = static_cast<ExactRef*>(h);
    try {
        auto c = x->ring ? x->ring->cardinalities(t, k) : x->pairs->cardinalities(t, k);
        std::sort(c.begin(), c.end());
        if (hosts)
            for (size_t i = 0; i < c.size(); ++i) {
                hosts[i] = c[i].first;
                counts[i] = c[i].second;
            }
        return c.size();
    } catch (const std::exception& e) {
        set_err(err, errlen, e.what());
        return UINT64_MAX;
    }
}

// ---- ingest front end: the reference's own orient_record / SlicePartitioner / for_each_record
uint64_t ref_orient(const uint32_t* recs, uint64_t n, uint32_t prefix_addr, uint32_t prefix_bits, uint32_t* out,
                    uint64_t* stats) {
    const CidrPrefix net{prefix_addr & CidrPrefix::mask_of(prefix_bits), prefix_bits};
    OrientStats st;
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i) {
        if (const auto o = orient_record(TraceRecord{recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]}, net, st)) {
            out[3 * m] = o->ts;
            out[3 * m + 1] = o->src;
            out[3 * m + 2] = o->dst;
            ++m;
        }
    }
    stats[0] = st.kept;
    stats[1] = st.flipped;
    stats[2] = st.dropped_both;
    stats[3] = st.dropped_neither;
    return m;
}

uint64_t ref_slice_bounds(const uint32_t* recs, uint64_t n, uint32_t slice_seconds, uint64_t* offsets) {
    SlicePartitioner part(slice_seconds);
    uint64_t slices = 0, at = 0;
    const auto sink = [&](uint64_t id, std::vector<TraceRecord>&& batch) {
        if (offsets) offsets[id] = at;
        at += batch.size();
        slices = id + 1;
    };
    for (uint64_t i = 0; i < n; ++i) part.push(TraceRecord{recs[3 * i], recs[3 * i + 1], recs[3 * i + 2]}, sink);
    part.finish(sink);
    if (offsets && slices) offsets[slices] = at;
    return slices;
}

uint64_t ref_parse_srlt(const uint8_t* bytes, uint64_t nbytes, uint32_t* out, int* err, uint64_t* err_index) {
    *err = 0;
    *err_index = 0;
    char path[] = "/tmp/srla_ref_srlt_XXXXXX";
    const int fd = mkstemp(path);
    if (fd < 0) throw std::runtime_error("mkstemp");
    FILE* f = fdopen(fd, "wb");
    fwrite(bytes, 1, nbytes, f);
    fclose(f);
    uint64_t n = 0;
    try {
        for_each_record(path, TraceFormat::binary, [&](const TraceRecord& r) {
            if (out) {
                out[3 * n] = r.ts;
                out[3 * n + 1] = r.src;
                out[3 * n + 2] = r.dst;
            }
            ++n;
        });
    } catch (const InputError& e) {
        const std::string m = e.what();
        *err = m.find("truncated") != std::string::npos ? 2 : m.find("regression") != std::string::npos ? 3 : 1;
        *err_index = n;
    }
    std::remove(path);
    return n;
}

}  // extern "C"
