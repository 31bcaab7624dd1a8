// ref_capi.cpp — C ABI over the UNMODIFIED reference headers
// (/root/reference/proj/include/sspread/*.hpp), compiled by oracle/Makefile into
// oracle/_ref/libsspread_ref.so. TEST INFRASTRUCTURE ONLY: it pins the C
// restatement (srla_oracle.c) against the real reference, generates the golden
// fixtures under tests/golden/, and is the CPU baseline of bench.py's
// reference arm. No reference source is copied here; this file only calls the
// reference's public API with the same entry points as srla_oracle.h
// (prefix `ref_` instead of `orc_`).
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sspread/generator.hpp"
#include "sspread/pipeline.hpp"
#include "sspread/sea.hpp"
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
};

SeaBase* S(void* h) { return static_cast<SeaBase*>(h); }

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
