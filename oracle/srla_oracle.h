/*
 * srla_oracle.h — CPU restatement of the SRLA hot path, TEST INFRASTRUCTURE ONLY.
 *
 * This is the parity checker for the B200 engine: plain C, serial, record-order
 * semantics, restating /root/reference/proj/include/sspread/{hash,recorders,
 * estimators,sea,pipeline,generator}.hpp function by function (each definition
 * in srla_oracle.c cites the reference file:line it follows).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * arm may load this library, and only as the checker — never as the product
 * path. The engine (paper_1803_10369_b200/csrc) never links it.
 *
 * Parity pinning: tests/test_oracle_golden.py checks every entry point against
 * golden vectors produced by the unmodified reference headers compiled into
 * oracle/_ref/libsspread_ref.so (recipe: oracle/Makefile, generator script:
 * tests/golden/make_golden.py), and against the reference's own KATs.
 *
 * The same ABI (prefix `ref_` instead of `orc_`) is exported by
 * oracle/ref_capi.cpp over the reference classes, so tests can swap the two.
 */
#ifndef SRLA_ORACLE_H
#define SRLA_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Mirrors sspread::SeaConfig (sea.hpp:33-52) field for field. */
typedef struct orc_config {
    uint32_t rows;
    uint32_t cols;
    uint32_t rough_slots;
    uint32_t linear_slots;
    uint32_t recorder_bits;
    uint32_t window;
    uint32_t theta;
    uint32_t _pad;
    double fill_ratio;
    uint64_t seed;
} orc_config;

/* Mirrors sspread::PlantSpec + BackgroundSpec + PlantedHost (generator.hpp:16-64). */
typedef struct orc_plant {
    uint32_t host;
    uint32_t cardinality;
    uint32_t first_slice;
    uint32_t last_slice;
} orc_plant;

typedef struct orc_spec {
    uint64_t seed;
    uint32_t start_ts;
    uint32_t slice_seconds;
    uint32_t slices;
    uint32_t window;
    uint32_t a_base;
    uint32_t b_base;
    uint32_t a_hosts;
    uint32_t b_hosts;
    uint32_t pairs_per_slice;
    uint32_t n_plants;
    double skew;
    const orc_plant* plants;
} orc_spec;

/* kinds for export/import */
enum { ORC_INDICATOR = 0, ORC_ROUGH = 1, ORC_LINEAR = 2 };

/* Library-level helpers (hash.hpp, estimators.hpp). */
uint64_t orc_avalanche64(uint64_t x);
uint32_t orc_hash_u32(uint64_t seed, uint32_t index, uint32_t key);
uint32_t orc_hash_reduce(uint64_t seed, uint32_t index, uint32_t key, uint32_t range);
uint32_t orc_sampling_exponent(uint64_t theta, uint64_t slots);
uint32_t orc_super_weight_threshold(double ratio, uint32_t slots);
double orc_super_test_ratio(void);
int orc_linear_estimate(uint32_t weight, uint32_t slots, double* out);

/* Sketch (EstimatorArray<W>, sea.hpp:113-359). Returns NULL and fills err on a
 * configuration the reference rejects. */
void* orc_create(const orc_config* cfg, char* err, size_t errlen);
void orc_destroy(void* h);
uint32_t orc_tau(void* h);
uint32_t orc_threshold(void* h);
uint32_t orc_word_bytes(void* h);
uint32_t orc_column_of(void* h, uint32_t row, uint32_t aip);
uint64_t orc_row_len(void* h, int kind);

/* Scan `n` records laid out as TraceRecord {ts, src, dst} triples, in order.
 * Candidate pushes go to `sink` (capacity n); *nsink receives the count. */
void orc_scan(void* h, const uint32_t* recs, uint64_t n, uint32_t* sink, uint64_t* nsink);

uint32_t orc_union_rough_weight(void* h, uint32_t aip);
uint32_t orc_union_linear_weight(void* h, uint32_t aip);
/* union_view: indicator AND, rough max (g words as u32), linear max (g' as u32) */
uint16_t orc_union_view(void* h, uint32_t aip, uint32_t* rough, uint32_t* linear);
uint64_t orc_row_active(void* h, uint32_t row);
double orc_row_fill_fraction(void* h, uint32_t row);
double orc_union_fill_product(void* h);
int orc_corrected_estimate_from(void* h, uint32_t weight, double fill_product, double* out);

/* report_window over csip[0..n): outputs n entries sorted by host. */
void orc_report(void* h, const uint32_t* csip, uint64_t n, uint32_t* hosts, uint32_t* weights,
                double* estimates, uint8_t* has_estimate, uint8_t* is_super);
/* slide: retained (capacity n) in csip order; returns count. */
uint64_t orc_slide(void* h, const uint32_t* csip, uint64_t n, uint32_t* retained);

/* Rows as little-endian W-byte (u16 for the indicator) words. */
void orc_export_row(void* h, uint32_t row, int kind, void* buf);
void orc_import_row(void* h, uint32_t row, int kind, const void* buf);

/* DetectPipeline<W> with workers = 1 (pipeline.hpp:110-158): an
 * EstimatorArray plus its CandidateList. */
void* orc_pipeline_create(const orc_config* cfg, uint32_t workers, char* err, size_t errlen);
void orc_pipeline_destroy(void* p);
void* orc_pipeline_sketch(void* p);
/* process_slice; if a report is produced, *reported = 1 and the entries are
 * written (capacity = current csip size, query with orc_pipeline_ncand first). */
void orc_pipeline_process_slice(void* p, uint64_t slice_id, const uint32_t* recs, uint64_t n,
                                int want_report, int* reported, uint64_t* n_entries,
                                uint32_t* hosts, uint32_t* weights, double* estimates,
                                uint8_t* has_estimate, uint8_t* is_super);
uint64_t orc_pipeline_ncand(void* p);
void orc_pipeline_candidates(void* p, uint32_t* out);
double orc_pipeline_scan_ms(void* p);
double orc_pipeline_estimate_ms(void* p);

/* generate_trace (generator.hpp:117-161). Returns the record count; writes
 * triples into out when out != NULL (capacity must be >= the count). */
uint64_t orc_generate(const orc_spec* spec, uint32_t* out, char* err, size_t errlen);

/* Ingest front end (trace.hpp), records as (ts, src, dst) u32 triples.
 * orient: orient_record over a batch (trace.hpp:223-238) against the prefix
 * addr/bits (CidrPrefix, addr masked as CidrPrefix::parse does); kept/flipped
 * records to `out` in input order; stats = {kept, flipped, dropped_both,
 * dropped_neither}; returns the records written. */
uint64_t orc_orient(const uint32_t* recs, uint64_t n, uint32_t prefix_addr, uint32_t prefix_bits, uint32_t* out,
                    uint64_t* stats);
/* SlicePartitioner over an ordered batch (trace.hpp:243-281): offsets[s] =
 * first record of slice s for s in [0, nslices], origin = the first record's
 * ts, empty slices included. Returns nslices (0 for an empty batch);
 * offsets == NULL only counts. */
uint64_t orc_slice_bounds(const uint32_t* recs, uint64_t n, uint32_t slice_seconds, uint64_t* offsets);
/* SRLT v1 file bytes (for_each_record binary branch, trace.hpp:148-170):
 * returns the records parsed into `out` (NULL: count only); *err = 0 ok,
 * 1 bad magic/version, 2 truncated record, 3 timestamp regression, with the
 * record index in *err_index. */
uint64_t orc_parse_srlt(const uint8_t* bytes, uint64_t nbytes, uint32_t* out, int* err, uint64_t* err_index);

#ifdef __cplusplus
}
#endif
#endif
