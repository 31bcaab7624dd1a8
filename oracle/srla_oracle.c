/*
 * srla_oracle.c — serial CPU restatement of the SRLA hot path.
 * TEST INFRASTRUCTURE ONLY (see srla_oracle.h): the parity checker, never the
 * product path. Reference paths are relative to /root/reference/proj/include/sspread/.
 *
 * Recorder words are held as uint32_t internally and masked to the storage
 * width W (1/2/4 bytes, recorders.hpp:64-66) wherever the reference's
 * arithmetic would wrap in W, so out-of-model values poked through the row
 * accessors behave exactly as in the reference.
 */
#define _GNU_SOURCE
#include "srla_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ hash.hpp */

/* hash.hpp:9-13 — splitmix64 finalizer */
uint64_t orc_avalanche64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* hash.hpp:53-56 — HashFamily::u32 */
uint32_t orc_hash_u32(uint64_t seed, uint32_t index, uint32_t key) {
    const uint64_t sub = orc_avalanche64(seed + 0x9E3779B97F4A7C15ull * (uint64_t)(index + 1u));
    return (uint32_t)orc_avalanche64(sub ^ (uint64_t)key);
}

/* hash.hpp:60-62 — HashFamily::reduce, multiply-shift */
uint32_t orc_hash_reduce(uint64_t seed, uint32_t index, uint32_t key, uint32_t range) {
    return (uint32_t)(((uint64_t)orc_hash_u32(seed, index, key) * range) >> 32);
}

enum { kSampleHash = 0, kRoughSlotHash = 1, kIndicatorHash = 2, kRowHashBase = 8 }; /* hash.hpp:70-73 */
#define kIndicatorBits 16u                                                         /* sea.hpp:21 */
#define kMaxRows 64u                                                               /* sea.hpp:349 */

/* hash.hpp:17-39 — SplitMix64 */
typedef struct { uint64_t state; } splitmix64;
static uint64_t sm_next(splitmix64* r) {
    r->state += 0x9E3779B97F4A7C15ull;
    return orc_avalanche64(r->state);
}
static uint64_t sm_next_below(splitmix64* r, uint64_t bound) {
    return (uint64_t)(((unsigned __int128)sm_next(r) * bound) >> 64);
}
static double sm_next_double(splitmix64* r) { return (double)(sm_next(r) >> 11) * 0x1.0p-53; }

/* ------------------------------------------------------------ estimators.hpp */

/* estimators.hpp:19 */
double orc_super_test_ratio(void) { return 0.99 * (1.0 - exp(-1.0 / 3.0)); }

/* estimators.hpp:24-29 — integer ceil-log2 of ceil(theta/slots) */
uint32_t orc_sampling_exponent(uint64_t theta, uint64_t slots) {
    if (theta < 1 || slots < 1) return 0;
    const uint64_t ratio = (theta + slots - 1) / slots;
    if (ratio <= 1) return 0;
    return (uint32_t)(64 - __builtin_clzll(ratio - 1)); /* std::bit_width */
}

/* estimators.hpp:33-35 */
uint32_t orc_super_weight_threshold(double ratio, uint32_t slots) {
    return (uint32_t)ceil(ratio * slots - 1e-9);
}

/* estimators.hpp:141-146 — returns 0 for "nullopt" (saturated) */
int orc_linear_estimate(uint32_t weight, uint32_t slots, double* out) {
    if (weight >= slots) return 0;
    *out = -(double)slots * log1p(-(double)weight / (double)slots);
    return 1;
}

/* ------------------------------------------------------------- candidate list */

/* sea.hpp:56-76 — CandidateList: dedup, first-insertion order */
typedef struct {
    uint32_t* hosts;
    uint64_t n, cap;
    uint64_t* table; /* open addressing over host+1 (0 = empty) */
    uint64_t tcap;
} cand_list;

static void cl_init(cand_list* c) { memset(c, 0, sizeof(*c)); }
static void cl_free(cand_list* c) {
    free(c->hosts);
    free(c->table);
    cl_init(c);
}
static uint64_t cl_slot(uint32_t host, uint64_t tcap) { return orc_avalanche64(host) & (tcap - 1); }
static int cl_contains(const cand_list* c, uint32_t host) {
    if (!c->tcap) return 0;
    const uint64_t key = (uint64_t)host + 1u;
    for (uint64_t s = cl_slot(host, c->tcap);; s = (s + 1) & (c->tcap - 1)) {
        if (c->table[s] == 0) return 0;
        if (c->table[s] == key) return 1;
    }
}
static void cl_place(uint64_t* table, uint64_t tcap, uint32_t host) {
    uint64_t s = cl_slot(host, tcap);
    while (table[s]) s = (s + 1) & (tcap - 1);
    table[s] = (uint64_t)host + 1u;
}
static int cl_insert(cand_list* c, uint32_t host) {
    if (cl_contains(c, host)) return 0;
    if (c->n == c->cap) {
        c->cap = c->cap ? c->cap * 2 : 64;
        c->hosts = (uint32_t*)realloc(c->hosts, c->cap * sizeof(uint32_t));
    }
    c->hosts[c->n++] = host;
    if ((c->n + 1) * 2 > c->tcap) {
        free(c->table);
        c->tcap = c->tcap ? c->tcap * 2 : 128;
        c->table = (uint64_t*)calloc(c->tcap, sizeof(uint64_t));
        for (uint64_t i = 0; i < c->n; ++i) cl_place(c->table, c->tcap, c->hosts[i]);
    } else {
        cl_place(c->table, c->tcap, host);
    }
    return 1;
}

/* ---------------------------------------------------------------- sea.hpp */

typedef struct {
    orc_config cfg;
    uint32_t expired;    /* recorders.hpp:39-42 */
    uint32_t word_bytes; /* recorders.hpp:64-66 */
    uint32_t wmask;
    uint32_t tau;        /* estimators.hpp:24-29 via DetectionParams::make */
    uint32_t threshold;  /* sea.hpp:121 */
    uint64_t sub_row[kMaxRows];
    uint16_t** indicator; /* indicator[i][col]       sea.hpp:356 */
    uint32_t** rough;     /* rough[i][col*g + slot]  sea.hpp:357 */
    uint32_t** linear;    /* linear[i][col*g' + slot] sea.hpp:358 */
} orc_sea;

static int fail(char* err, size_t errlen, const char* msg) {
    if (err && errlen) snprintf(err, errlen, "%s", msg);
    return 0;
}

/* SeaConfig::validate (sea.hpp:44-51) + RecorderModel (recorders.hpp:33-54)
 * + EstimatorArray ctor checks (sea.hpp:122-126). */
static int validate(const orc_config* c, char* err, size_t errlen) {
    if (c->rows < 1) return fail(err, errlen, "rows must be >= 1");
    if (c->cols < 1) return fail(err, errlen, "cols must be >= 1");
    if (c->rough_slots < 1) return fail(err, errlen, "rough_slots must be >= 1");
    if (c->linear_slots < 2) return fail(err, errlen, "linear_slots must be >= 2");
    if (c->theta < 1) return fail(err, errlen, "theta must be >= 1");
    if (c->recorder_bits < 1 || c->recorder_bits > 32)
        return fail(err, errlen, "recorder width must be in [1, 32] bits");
    const uint32_t e = c->recorder_bits == 32 ? 0xFFFFFFFFu : (1u << c->recorder_bits) - 1u;
    if (c->window < 1 || c->window > e) return fail(err, errlen, "window does not fit the recorder");
    if (c->rows > kMaxRows) return fail(err, errlen, "at most 64 rows supported");
    return 1;
}

void* orc_create(const orc_config* cfg, char* err, size_t errlen) {
    if (!validate(cfg, err, errlen)) return NULL;
    orc_sea* s = (orc_sea*)calloc(1, sizeof(orc_sea));
    s->cfg = *cfg;
    s->expired = cfg->recorder_bits == 32 ? 0xFFFFFFFFu : (1u << cfg->recorder_bits) - 1u;
    s->word_bytes = cfg->recorder_bits <= 8 ? 1 : cfg->recorder_bits <= 16 ? 2 : 4;
    s->wmask = s->word_bytes == 4 ? 0xFFFFFFFFu : (1u << (8 * s->word_bytes)) - 1u;
    s->tau = orc_sampling_exponent(cfg->theta, cfg->rough_slots);
    s->threshold = orc_super_weight_threshold(cfg->fill_ratio, cfg->rough_slots);
    for (uint32_t i = 0; i < cfg->rows; ++i)
        s->sub_row[i] = orc_avalanche64(cfg->seed + 0x9E3779B97F4A7C15ull * (uint64_t)(kRowHashBase + i + 1u));
    s->indicator = (uint16_t**)calloc(cfg->rows, sizeof(void*));
    s->rough = (uint32_t**)calloc(cfg->rows, sizeof(void*));
    s->linear = (uint32_t**)calloc(cfg->rows, sizeof(void*));
    const uint64_t nr = (uint64_t)cfg->cols * cfg->rough_slots;
    const uint64_t nl = (uint64_t)cfg->cols * cfg->linear_slots;
    for (uint32_t i = 0; i < cfg->rows; ++i) { /* sea.hpp:130-134 */
        s->indicator[i] = (uint16_t*)calloc(cfg->cols, sizeof(uint16_t));
        s->rough[i] = (uint32_t*)malloc(nr * sizeof(uint32_t));
        s->linear[i] = (uint32_t*)malloc(nl * sizeof(uint32_t));
        for (uint64_t j = 0; j < nr; ++j) s->rough[i][j] = s->expired;
        for (uint64_t j = 0; j < nl; ++j) s->linear[i][j] = s->expired;
    }
    return s;
}

void orc_destroy(void* h) {
    orc_sea* s = (orc_sea*)h;
    if (!s) return;
    for (uint32_t i = 0; i < s->cfg.rows; ++i) {
        free(s->indicator[i]);
        free(s->rough[i]);
        free(s->linear[i]);
    }
    free(s->indicator);
    free(s->rough);
    free(s->linear);
    free(s);
}

uint32_t orc_tau(void* h) { return ((orc_sea*)h)->tau; }
uint32_t orc_threshold(void* h) { return ((orc_sea*)h)->threshold; }
uint32_t orc_word_bytes(void* h) { return ((orc_sea*)h)->word_bytes; }

/* sea.hpp:143-145 */
static uint32_t column_of(const orc_sea* s, uint32_t row, uint32_t aip) {
    const uint32_t hv = (uint32_t)orc_avalanche64(s->sub_row[row] ^ (uint64_t)aip);
    return (uint32_t)(((uint64_t)hv * s->cfg.cols) >> 32);
}
uint32_t orc_column_of(void* h, uint32_t row, uint32_t aip) { return column_of((orc_sea*)h, row, aip); }

uint64_t orc_row_len(void* h, int kind) {
    const orc_sea* s = (orc_sea*)h;
    if (kind == ORC_INDICATOR) return s->cfg.cols;
    if (kind == ORC_ROUGH) return (uint64_t)s->cfg.cols * s->cfg.rough_slots;
    return (uint64_t)s->cfg.cols * s->cfg.linear_slots;
}

static inline uint32_t rjoin(uint32_t a, uint32_t b) { return a > b ? a : b; } /* recorders.hpp:90-93 */
static inline int ractive(uint32_t r, uint32_t k) { return r < k; }            /* recorders.hpp:97-100 */

/* sea.hpp:150-196 — EstimatorArray::scan_ip_pair, serial */
static void scan_pair(orc_sea* s, uint32_t aip, uint32_t bip, uint32_t* sink, uint64_t* nsink) {
    const orc_config* c = &s->cfg;
    uint32_t cols[kMaxRows];
    for (uint32_t i = 0; i < c->rows; ++i) cols[i] = column_of(s, i, aip);

    const uint32_t sample = orc_hash_u32(c->seed, kSampleHash, bip);
    const uint32_t lslot = sample % c->linear_slots; /* modulo, not reduce: sea.hpp:157 */
    for (uint32_t i = 0; i < c->rows; ++i) s->linear[i][(uint64_t)cols[i] * c->linear_slots + lslot] = 0;

    /* lowest_set_bit(0) = 32 (recorders.hpp:14-16) */
    const uint32_t lsb = sample ? (uint32_t)__builtin_ctz(sample) : 32u;
    if (lsb < s->tau) return; /* sea.hpp:164 */
    const uint32_t rslot = orc_hash_reduce(c->seed, kRoughSlotHash, bip, c->rough_slots);
    for (uint32_t i = 0; i < c->rows; ++i) s->rough[i][(uint64_t)cols[i] * c->rough_slots + rslot] = 0;

    uint32_t weight = 0; /* sea.hpp:172-182 */
    for (uint32_t j = 0; j < c->rough_slots; ++j) {
        uint32_t joined = 0;
        for (uint32_t i = 0; i < c->rows; ++i)
            joined = rjoin(joined, s->rough[i][(uint64_t)cols[i] * c->rough_slots + j]);
        weight += ractive(joined, c->window);
    }
    if (weight < s->threshold) return;

    const uint16_t bit = (uint16_t)(1u << orc_hash_reduce(c->seed, kIndicatorHash, aip, kIndicatorBits));
    uint16_t joined_si = 0xFFFF; /* sea.hpp:185-190 */
    for (uint32_t i = 0; i < c->rows; ++i) joined_si &= s->indicator[i][cols[i]];
    if (joined_si & bit) return;

    sink[(*nsink)++] = aip; /* sea.hpp:192-195 */
    for (uint32_t i = 0; i < c->rows; ++i) s->indicator[i][cols[i]] |= bit;
}

void orc_scan(void* h, const uint32_t* recs, uint64_t n, uint32_t* sink, uint64_t* nsink) {
    orc_sea* s = (orc_sea*)h;
    *nsink = 0;
    for (uint64_t r = 0; r < n; ++r) scan_pair(s, recs[3 * r + 1], recs[3 * r + 2], sink, nsink);
}

/* sea.hpp:219-230 */
static uint32_t union_rough_weight(const orc_sea* s, uint32_t aip) {
    const orc_config* c = &s->cfg;
    uint32_t weight = 0;
    for (uint32_t j = 0; j < c->rough_slots; ++j) {
        uint32_t joined = 0;
        for (uint32_t i = 0; i < c->rows; ++i)
            joined = rjoin(joined, s->rough[i][(uint64_t)column_of(s, i, aip) * c->rough_slots + j]);
        weight += ractive(joined, c->window);
    }
    return weight;
}
uint32_t orc_union_rough_weight(void* h, uint32_t aip) { return union_rough_weight((orc_sea*)h, aip); }

/* sea.hpp:232-243 */
static uint32_t union_linear_weight(const orc_sea* s, uint32_t aip) {
    const orc_config* c = &s->cfg;
    const uint32_t* cells[kMaxRows];
    for (uint32_t i = 0; i < c->rows; ++i)
        cells[i] = &s->linear[i][(uint64_t)column_of(s, i, aip) * c->linear_slots];
    uint32_t weight = 0;
    for (uint32_t j = 0; j < c->linear_slots; ++j) {
        uint32_t joined = 0;
        for (uint32_t i = 0; i < c->rows; ++i) joined = rjoin(joined, cells[i][j]);
        weight += ractive(joined, c->window);
    }
    return weight;
}
uint32_t orc_union_linear_weight(void* h, uint32_t aip) { return union_linear_weight((orc_sea*)h, aip); }

/* sea.hpp:199-217 */
uint16_t orc_union_view(void* h, uint32_t aip, uint32_t* rough, uint32_t* linear) {
    const orc_sea* s = (orc_sea*)h;
    const orc_config* c = &s->cfg;
    uint16_t ind = 0xFFFF;
    for (uint32_t j = 0; j < c->rough_slots; ++j) rough[j] = 0;
    if (linear)
        for (uint32_t j = 0; j < c->linear_slots; ++j) linear[j] = 0;
    for (uint32_t i = 0; i < c->rows; ++i) {
        const uint32_t col = column_of(s, i, aip);
        ind &= s->indicator[i][col];
        for (uint32_t j = 0; j < c->rough_slots; ++j)
            rough[j] = rjoin(rough[j], s->rough[i][(uint64_t)col * c->rough_slots + j]);
        if (linear)
            for (uint32_t j = 0; j < c->linear_slots; ++j)
                linear[j] = rjoin(linear[j], s->linear[i][(uint64_t)col * c->linear_slots + j]);
    }
    return ind;
}

/* recorders.hpp:119-129 count_active over one linear row */
uint64_t orc_row_active(void* h, uint32_t row) {
    const orc_sea* s = (orc_sea*)h;
    const uint64_t n = (uint64_t)s->cfg.cols * s->cfg.linear_slots;
    uint64_t a = 0;
    for (uint64_t j = 0; j < n; ++j) a += s->linear[row][j] < s->cfg.window;
    return a;
}

/* sea.hpp:248-257 */
double orc_row_fill_fraction(void* h, uint32_t row) {
    const orc_sea* s = (orc_sea*)h;
    const uint64_t n = (uint64_t)s->cfg.cols * s->cfg.linear_slots;
    return (double)orc_row_active(h, row) / (double)n;
}

/* sea.hpp:261-265 — product in row order */
double orc_union_fill_product(void* h) {
    const orc_sea* s = (orc_sea*)h;
    double p = 1.0;
    for (uint32_t i = 0; i < s->cfg.rows; ++i) p *= orc_row_fill_fraction(h, i);
    return p;
}

/* sea.hpp:270-279 — Eq. 9; returns 0 for nullopt */
int orc_corrected_estimate_from(void* h, uint32_t weight, double fill_product, double* out) {
    const orc_sea* s = (orc_sea*)h;
    const double slots = s->cfg.linear_slots;
    if (fill_product >= 1.0 - 1e-12) return orc_linear_estimate(weight, s->cfg.linear_slots, out);
    const double contaminated = slots * fill_product;
    const double numerator = (double)weight - contaminated;
    if (numerator < 0) {
        *out = 0.0;
        return 1;
    }
    const double x = numerator / (slots * (1.0 - fill_product));
    if (x >= 1.0) return 0;
    *out = -slots * log1p(-x);
    return 1;
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

/* sea.hpp:288-309 — report_window: sorted by host, Eq. 9 estimate, theta cut */
void orc_report(void* h, const uint32_t* csip, uint64_t n, uint32_t* hosts, uint32_t* weights,
                double* estimates, uint8_t* has_estimate, uint8_t* is_super) {
    orc_sea* s = (orc_sea*)h;
    memcpy(hosts, csip, n * sizeof(uint32_t));
    qsort(hosts, n, sizeof(uint32_t), cmp_u32);
    const double fp = orc_union_fill_product(h);
    for (uint64_t e = 0; e < n; ++e) {
        weights[e] = union_linear_weight(s, hosts[e]);
        double est = 0;
        has_estimate[e] = (uint8_t)orc_corrected_estimate_from(h, weights[e], fp, &est);
        estimates[e] = has_estimate[e] ? est : 0.0;
        is_super[e] = (uint8_t)(!has_estimate[e] || est >= (double)s->cfg.theta);
    }
}

/* sea.hpp:316-338 — slide: clear SI, age rough then linear per row, retain */
uint64_t orc_slide(void* h, const uint32_t* csip, uint64_t n, uint32_t* retained) {
    orc_sea* s = (orc_sea*)h;
    const orc_config* c = &s->cfg;
    for (uint32_t i = 0; i < c->rows; ++i) memset(s->indicator[i], 0, c->cols * sizeof(uint16_t));
    const uint64_t nr = (uint64_t)c->cols * c->rough_slots;
    const uint64_t nl = (uint64_t)c->cols * c->linear_slots;
    for (uint32_t i = 0; i < c->rows; ++i) { /* slide_recorders, recorders.hpp:113-116 */
        for (uint64_t j = 0; j < nr; ++j) {
            const uint32_t r = s->rough[i][j];
            s->rough[i][j] = (r + (r != s->expired)) & s->wmask;
        }
        for (uint64_t j = 0; j < nl; ++j) {
            const uint32_t r = s->linear[i][j];
            s->linear[i][j] = (r + (r != s->expired)) & s->wmask;
        }
    }
    cand_list out;
    cl_init(&out);
    for (uint64_t e = 0; e < n; ++e) {
        const uint32_t host = csip[e];
        if (union_rough_weight(s, host) < s->threshold) continue;
        cl_insert(&out, host);
        const uint16_t bit = (uint16_t)(1u << orc_hash_reduce(c->seed, kIndicatorHash, host, kIndicatorBits));
        for (uint32_t i = 0; i < c->rows; ++i) s->indicator[i][column_of(s, i, host)] |= bit;
    }
    memcpy(retained, out.hosts, out.n * sizeof(uint32_t));
    const uint64_t m = out.n;
    cl_free(&out);
    return m;
}

void orc_export_row(void* h, uint32_t row, int kind, void* buf) {
    const orc_sea* s = (orc_sea*)h;
    const uint64_t n = orc_row_len(h, kind);
    if (kind == ORC_INDICATOR) {
        memcpy(buf, s->indicator[row], n * sizeof(uint16_t));
        return;
    }
    const uint32_t* src = kind == ORC_ROUGH ? s->rough[row] : s->linear[row];
    uint8_t* out = (uint8_t*)buf;
    for (uint64_t j = 0; j < n; ++j)
        for (uint32_t b = 0; b < s->word_bytes; ++b) out[j * s->word_bytes + b] = (uint8_t)(src[j] >> (8 * b));
}

void orc_import_row(void* h, uint32_t row, int kind, const void* buf) {
    orc_sea* s = (orc_sea*)h;
    const uint64_t n = orc_row_len(h, kind);
    if (kind == ORC_INDICATOR) {
        memcpy(s->indicator[row], buf, n * sizeof(uint16_t));
        return;
    }
    uint32_t* dst = kind == ORC_ROUGH ? s->rough[row] : s->linear[row];
    const uint8_t* in = (const uint8_t*)buf;
    for (uint64_t j = 0; j < n; ++j) {
        uint32_t v = 0;
        for (uint32_t b = 0; b < s->word_bytes; ++b) v |= (uint32_t)in[j * s->word_bytes + b] << (8 * b);
        dst[j] = v;
    }
}

/* ------------------------------------------------------------ pipeline.hpp */

typedef struct {
    orc_sea* sea;
    cand_list csip;
    uint32_t* sink;
    uint64_t sink_cap;
    double scan_ms, estimate_ms;
} orc_pipe;

void* orc_pipeline_create(const orc_config* cfg, uint32_t workers, char* err, size_t errlen) {
    (void)workers; /* the oracle is the 1-worker (record-order) path */
    if (cfg->cols & (cfg->cols - 1)) { /* RunConfig::validate, pipeline.hpp:43-44 */
        fail(err, errlen, "cols must be a power of two");
        return NULL;
    }
    orc_sea* s = (orc_sea*)orc_create(cfg, err, errlen);
    if (!s) return NULL;
    orc_pipe* p = (orc_pipe*)calloc(1, sizeof(orc_pipe));
    p->sea = s;
    cl_init(&p->csip);
    return p;
}

void orc_pipeline_destroy(void* pp) {
    orc_pipe* p = (orc_pipe*)pp;
    if (!p) return;
    orc_destroy(p->sea);
    cl_free(&p->csip);
    free(p->sink);
    free(p);
}

void* orc_pipeline_sketch(void* p) { return ((orc_pipe*)p)->sea; }
uint64_t orc_pipeline_ncand(void* p) { return ((orc_pipe*)p)->csip.n; }
void orc_pipeline_candidates(void* p, uint32_t* out) {
    orc_pipe* q = (orc_pipe*)p;
    memcpy(out, q->csip.hosts, q->csip.n * sizeof(uint32_t));
}
double orc_pipeline_scan_ms(void* p) { return ((orc_pipe*)p)->scan_ms; }
double orc_pipeline_estimate_ms(void* p) { return ((orc_pipe*)p)->estimate_ms; }

static double now_ms(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
}

/* pipeline.hpp:110-129 process_slice + :134-139 scan_records (1 worker) */
void orc_pipeline_process_slice(void* pp, uint64_t slice_id, const uint32_t* recs, uint64_t n,
                                int want_report, int* reported, uint64_t* n_entries,
                                uint32_t* hosts, uint32_t* weights, double* estimates,
                                uint8_t* has_estimate, uint8_t* is_super) {
    orc_pipe* p = (orc_pipe*)pp;
    const double t0 = now_ms();
    if (n > p->sink_cap) {
        free(p->sink);
        p->sink_cap = n;
        p->sink = (uint32_t*)malloc(n * sizeof(uint32_t));
    }
    uint64_t ns = 0;
    orc_scan(p->sea, recs, n, p->sink, &ns);
    for (uint64_t i = 0; i < ns; ++i) cl_insert(&p->csip, p->sink[i]);
    p->scan_ms += now_ms() - t0;

    const uint32_t k = p->sea->cfg.window;
    *reported = 0;
    *n_entries = 0;
    if (slice_id + 1 >= k && want_report) {
        const double t1 = now_ms();
        orc_report(p->sea, p->csip.hosts, p->csip.n, hosts, weights, estimates, has_estimate, is_super);
        p->estimate_ms += now_ms() - t1;
        *reported = 1;
        *n_entries = p->csip.n;
    }
    uint32_t* retained = (uint32_t*)malloc((p->csip.n + 1) * sizeof(uint32_t));
    const uint64_t m = orc_slide(p->sea, p->csip.hosts, p->csip.n, retained);
    cl_free(&p->csip);
    cl_init(&p->csip);
    for (uint64_t i = 0; i < m; ++i) cl_insert(&p->csip, retained[i]);
    free(retained);
}

/* ------------------------------------------------------------ generator.hpp */

/* generator.hpp:98-109 */
static uint32_t plant_pool_offset(uint64_t plant_index, uint32_t pool) {
    return (uint32_t)((plant_index * 2654435761ull) % pool);
}

typedef struct {
    uint32_t ts, src, dst;
} rec3;

/* stable merge sort by ts (std::stable_sort, generator.hpp:153-154) */
static void stable_sort_ts(rec3* a, rec3* tmp, uint64_t n) {
    if (n < 2) return;
    for (uint64_t w = 1; w < n; w *= 2) {
        for (uint64_t lo = 0; lo < n; lo += 2 * w) {
            uint64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            uint64_t i = lo, j = mid, k = lo;
            while (i < mid && j < hi) tmp[k++] = (a[j].ts < a[i].ts) ? a[j++] : a[i++];
            while (i < mid) tmp[k++] = a[i++];
            while (j < hi) tmp[k++] = a[j++];
        }
        memcpy(a, tmp, n * sizeof(rec3));
    }
}

/* generator.hpp:45-63 PlantSpec::validate */
static int spec_validate(const orc_spec* s, char* err, size_t errlen) {
    if (s->slices < 1) return fail(err, errlen, "trace needs at least one slice");
    if (s->window < 1) return fail(err, errlen, "window must be >= 1");
    if (s->slice_seconds < 1) return fail(err, errlen, "slice duration must be >= 1");
    if (s->b_hosts < 1) return fail(err, errlen, "destination pool is empty");
    for (uint32_t i = 0; i < s->n_plants; ++i) {
        const orc_plant* p = &s->plants[i];
        if (p->cardinality < 1) return fail(err, errlen, "planted cardinality must be >= 1");
        if (p->cardinality > s->b_hosts) return fail(err, errlen, "planted cardinality exceeds the destination pool");
        if (p->host >= s->a_base && p->host < s->a_base + s->a_hosts)
            return fail(err, errlen, "planted host collides with the background source pool");
        if (p->first_slice > p->last_slice) return fail(err, errlen, "empty active span");
    }
    return 1;
}

/* generator.hpp:117-161 generate_trace */
uint64_t orc_generate(const orc_spec* spec, uint32_t* out, char* err, size_t errlen) {
    if (!spec_validate(spec, err, errlen)) return (uint64_t)-1;
    /* record count is independent of the random draws */
    uint64_t total = 0;
    for (uint64_t s = 0; s < spec->slices; ++s) {
        for (uint32_t pi = 0; pi < spec->n_plants; ++pi) {
            const orc_plant* p = &spec->plants[pi];
            if (!(s >= p->first_slice && s <= p->last_slice)) continue;
            const uint32_t r = (uint32_t)((s - p->first_slice) % spec->window);
            const uint64_t lo = (uint64_t)p->cardinality * r / spec->window;
            const uint64_t hi = (uint64_t)p->cardinality * (r + 1) / spec->window;
            total += hi - lo;
        }
        total += spec->pairs_per_slice;
    }
    if (!out) return total;

    /* ZipfSampler (generator.hpp:72-96) */
    double* cdf = NULL;
    if (spec->skew > 0.0) {
        cdf = (double*)malloc((size_t)spec->b_hosts * sizeof(double));
        double acc = 0;
        for (uint32_t r = 0; r < spec->b_hosts; ++r) {
            acc += 1.0 / pow((double)(r + 1), spec->skew);
            cdf[r] = acc;
        }
        for (uint32_t r = 0; r < spec->b_hosts; ++r) cdf[r] /= acc;
    }
    splitmix64 rng = {spec->seed};
    rec3* recs = (rec3*)out;
    rec3* tmp = NULL;
    uint64_t tmp_cap = 0;
    uint64_t n = 0;
    int anchored = 0;
    for (uint64_t s = 0; s < spec->slices; ++s) {
        const uint64_t slice_start = n;
        const uint32_t ts_base = spec->start_ts + (uint32_t)s * spec->slice_seconds;
        for (uint32_t pi = 0; pi < spec->n_plants; ++pi) {
            const orc_plant* p = &spec->plants[pi];
            if (!(s >= p->first_slice && s <= p->last_slice)) continue;
            const uint32_t r = (uint32_t)((s - p->first_slice) % spec->window);
            const uint32_t lo = (uint32_t)((uint64_t)p->cardinality * r / spec->window);
            const uint32_t hi = (uint32_t)((uint64_t)p->cardinality * (r + 1) / spec->window);
            const uint32_t offset = plant_pool_offset(pi, spec->b_hosts);
            for (uint32_t j = lo; j < hi; ++j) {
                const uint32_t dst = spec->b_base + (uint32_t)(((uint64_t)offset + j) % spec->b_hosts);
                recs[n].ts = ts_base + (uint32_t)sm_next_below(&rng, spec->slice_seconds);
                recs[n].src = p->host;
                recs[n].dst = dst;
                ++n;
            }
        }
        for (uint32_t i = 0; i < spec->pairs_per_slice; ++i) {
            const uint32_t src = spec->a_base + (uint32_t)sm_next_below(&rng, spec->a_hosts);
            uint32_t rank;
            if (spec->skew <= 0.0) {
                rank = (uint32_t)sm_next_below(&rng, spec->b_hosts);
            } else {
                const double u = sm_next_double(&rng);
                uint32_t lo = 0, hi = spec->b_hosts; /* std::lower_bound */
                while (lo < hi) {
                    const uint32_t mid = lo + (hi - lo) / 2;
                    if (cdf[mid] < u) lo = mid + 1;
                    else hi = mid;
                }
                rank = lo == spec->b_hosts ? spec->b_hosts - 1 : lo;
            }
            recs[n].ts = ts_base + (uint32_t)sm_next_below(&rng, spec->slice_seconds);
            recs[n].src = src;
            recs[n].dst = spec->b_base + rank;
            ++n;
        }
        const uint64_t m = n - slice_start;
        if (spec->slice_seconds > 1 && m > 1) {
            if (m > tmp_cap) {
                free(tmp);
                tmp_cap = m;
                tmp = (rec3*)malloc(m * sizeof(rec3));
            }
            stable_sort_ts(recs + slice_start, tmp, m);
        }
        if (!anchored && n > slice_start) {
            recs[slice_start].ts = ts_base;
            anchored = 1;
        }
    }
    free(tmp);
    free(cdf);
    return n;
}

/* ------------------------------------------------------------------ ingest (trace.hpp) */

/* CidrPrefix::mask_of (trace.hpp:73-75) */
static uint32_t cidr_mask(uint32_t bits) { return bits == 0 ? 0u : 0xFFFFFFFFu << (32 - bits); }

/* orient_record (trace.hpp:223-238) applied to a batch */
uint64_t orc_orient(const uint32_t* recs, uint64_t n, uint32_t prefix_addr, uint32_t prefix_bits, uint32_t* out,
                    uint64_t* stats) {
    const uint32_t mask = cidr_mask(prefix_bits), addr = prefix_addr & mask; /* CidrPrefix::parse */
    uint64_t m = 0;
    stats[0] = stats[1] = stats[2] = stats[3] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint32_t ts = recs[3 * i], src = recs[3 * i + 1], dst = recs[3 * i + 2];
        const int src_in = (src & mask) == addr, dst_in = (dst & mask) == addr; /* contains, :77 */
        if (src_in && !dst_in) {
            ++stats[0];
            out[3 * m] = ts; out[3 * m + 1] = src; out[3 * m + 2] = dst;
            ++m;
        } else if (!src_in && dst_in) {
            ++stats[1];
            out[3 * m] = ts; out[3 * m + 1] = dst; out[3 * m + 2] = src;
            ++m;
        } else if (src_in) {
            ++stats[2];
        } else {
            ++stats[3];
        }
    }
    return m;
}

/* SlicePartitioner::push / finish (trace.hpp:248-271): id = (ts - origin) /
   seconds with the first record's ts as origin; every id up to the last is a
   slice, empty or not */
uint64_t orc_slice_bounds(const uint32_t* recs, uint64_t n, uint32_t slice_seconds, uint64_t* offsets) {
    if (n == 0) return 0;
    const uint64_t origin = recs[0];
    uint64_t current = 0;
    if (offsets) offsets[0] = 0;
    for (uint64_t i = 0; i < n; ++i) {
        const uint64_t id = ((uint64_t)recs[3 * i] - origin) / slice_seconds;
        while (current < id) {
            ++current;
            if (offsets) offsets[current] = i;
        }
    }
    if (offsets) offsets[current + 1] = n;
    return current + 1;
}

/* for_each_record, binary branch (trace.hpp:148-170): magic "SRLT", version 1,
   packed little-endian (u32 ts, u32 src, u32 dst), non-decreasing ts */
uint64_t orc_parse_srlt(const uint8_t* bytes, uint64_t nbytes, uint32_t* out, int* err, uint64_t* err_index) {
    *err = 0;
    *err_index = 0;
    if (nbytes < 5 || memcmp(bytes, "SRLT", 4) != 0 || bytes[4] != 1) {
        *err = 1;
        return 0;
    }
    const uint8_t* p = bytes + 5;
    const uint64_t body = nbytes - 5, n = body / 12;
    uint32_t last = 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t v[3];
        for (int k = 0; k < 3; ++k) {
            const uint8_t* q = p + 12 * i + 4 * k;
            v[k] = (uint32_t)q[0] | (uint32_t)q[1] << 8 | (uint32_t)q[2] << 16 | (uint32_t)q[3] << 24;
        }
        if (i > 0 && v[0] < last) { /* check_order, trace.hpp:113-119 */
            *err = 3;
            *err_index = i;
            return i;
        }
        last = v[0];
        if (out) { out[3 * i] = v[0]; out[3 * i + 1] = v[1]; out[3 * i + 2] = v[2]; }
    }
    if (body % 12) {
        *err = 2;
        *err_index = n;
    }
    return n;
}
