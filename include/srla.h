/*
 * srla.h — C ABI of the B200-native SRLA engine (libsrla_b200.so).
 *
 * The reference (`sspread`, /root/reference/proj/include/sspread) is a
 * header-only C++ library with no FFI; its hot path is the EstimatorArray /
 * DetectPipeline API. Every entry point below replaces one reference call (the
 * cite is on each declaration) and is what the drop-in headers in
 * include/sspread/ (*.hpp) bind. Plain pointers and sizes only; no CUDA or torch
 * types cross this boundary. One CUDA stream per engine; an engine is not
 * re-entrant (the drop-in wrapper serialises calls, matching the reference's
 * "exclusive access outside the scan phase" contract, sea.hpp:108-112).
 *
 * Error convention: every call returns an srla_status. The message of the
 * last failure on the calling thread is srla_last_error(). The C++ wrapper maps
 * SRLA_E_INVALID to std::invalid_argument and SRLA_E_RANGE to
 * std::out_of_range, as the reference throws them (sea.hpp:44-51,125-126,
 * 249,341-346; recorders.hpp:35-53).
 */
#ifndef SRLA_H
#define SRLA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum srla_status {
    SRLA_OK = 0,
    SRLA_E_INVALID = 1,  /* bad argument / configuration (std::invalid_argument) */
    SRLA_E_RANGE = 2,    /* row index out of range (std::out_of_range) */
    SRLA_E_CAPACITY = 3, /* output buffer too small; *n_out holds the size needed */
    SRLA_E_CUDA = 4,     /* CUDA runtime / device failure */
    SRLA_E_INTERNAL = 5,
    SRLA_E_INPUT = 6     /* malformed trace input (sspread::InputError) */
} srla_status;

/* sspread::SeaConfig (sea.hpp:33-52), field for field. */
typedef struct srla_config {
    uint32_t rows;          /* u: estimator rows, <= 64 (sea.hpp:125-126,349) */
    uint32_t cols;          /* v: estimators per row */
    uint32_t rough_slots;   /* g */
    uint32_t linear_slots;  /* g' */
    uint32_t recorder_bits; /* z: 1..32; storage word 1/2/4 B (recorders.hpp:64-66) */
    uint32_t window;        /* k: 1..2^z-1 */
    uint32_t theta;
    uint32_t flags;         /* SRLA_FLAG_*; 0 = automatic (not part of SeaConfig) */
    double fill_ratio;      /* kSuperTestRatio by default (estimators.hpp:19) */
    uint64_t seed;
} srla_config;

/* Linear-recorder representation (results are identical either way):
 * literal distances with an O(table) slide, or epoch stamps with an O(1)
 * slide. Default: stamps for linear tables of 16 GiB and more. */
enum { SRLA_FLAG_EPOCH = 1u, SRLA_FLAG_LITERAL = 2u };

/* sspread::TraceRecord (trace.hpp:20-26): 12 bytes, host byte order. */
typedef struct srla_record {
    uint32_t ts;
    uint32_t src; /* aip: the monitored-side host */
    uint32_t dst; /* bip: the opposite host */
} srla_record;

/* sspread::WindowEntry (sea.hpp:88-93). has_estimate == 0 is the reference's
 * empty std::optional ("saturated"). */
typedef struct srla_entry {
    uint32_t host;
    uint32_t union_weight;
    double estimate;
    uint8_t has_estimate;
    uint8_t is_super;
    uint8_t reserved[6];
} srla_entry;

/* Row kinds for export/import (the raw spans of sea.hpp:341-346). */
enum { SRLA_INDICATOR = 0, SRLA_ROUGH = 1, SRLA_LINEAR = 2 };

typedef struct srla_engine srla_engine;

typedef struct srla_stats {
    uint64_t packets;         /* records scanned since create */
    uint64_t sampled_events;  /* rough-estimator updates (1 in 2^tau) */
    uint64_t crossings;       /* sampled updates that passed the rho*g test */
    uint64_t first_crossings; /* distinct hosts crossing, per chunk, summed */
    uint64_t flagged;         /* hosts needing ordered SI resolution */
    uint64_t pushed;          /* candidate-sink pushes */
    uint64_t kernel_launches; /* launches of this library's own kernels */
    uint64_t library_launches;/* CUB sort/scan/select launches (approximate) */
    uint64_t chunks;
    uint64_t slides;
    uint64_t overlapped_chunks; /* K1 run under a pending asynchronous end-of-slice */
} srla_stats;

/* Last failure message on this thread ("" if none). */
const char* srla_last_error(void);
/* Library version / build string ("srla_b200 <ver> sm_100a"). */
const char* srla_version(void);

/* EstimatorArray<W>::EstimatorArray (sea.hpp:116-135): validates, allocates
 * u*v*(g+g')*W + u*v*2 bytes of HBM on `device`, all recorders expired. */
srla_status srla_create(const srla_config* cfg, int device, srla_engine** out);
srla_status srla_destroy(srla_engine* e);

/* params().tau, weight_threshold(), storage word bytes (sea.hpp:140-141). */
srla_status srla_params(const srla_engine* e, uint32_t* tau, uint32_t* threshold,
                        uint32_t* word_bytes);
/* EstimatorArray::column_of (sea.hpp:143-145); host-side hash. */
srla_status srla_column_of(const srla_engine* e, uint32_t row, uint32_t aip, uint32_t* col);

/* Scan records in order: EstimatorArray::scan_ip_pair applied to each record
 * (sea.hpp:150-196), as DetectPipeline::scan_records does with one worker
 * (pipeline.hpp:134-139). `recs` is host memory (on_device = 0) or device
 * memory on the engine's GPU (on_device = 1). May be called repeatedly within
 * a slice. Hosts the reference would push to its candidate sink are appended,
 * in push order, to the engine's candidate list (deduplicated, like
 * CandidateList::insert, sea.hpp:58-62) and, if `pushed` != NULL, copied out
 * (up to `cap`; *n_pushed always receives the true count). */
srla_status srla_scan_batch(srla_engine* e, const srla_record* recs, uint64_t n, int on_device,
                            uint32_t* pushed, uint64_t cap, uint64_t* n_pushed);

/* srla_scan_batch over device records with an explicit producer: the engine's
 * streams wait (device-side) for everything queued on `producer_stream` (a
 * cudaStream_t; NULL = the legacy default stream) before reading `d_recs`.
 * srla_scan_batch(on_device = 1) is this call with the legacy default stream,
 * so records written by work on another non-blocking stream need this form.
 * `d_recs` must be device memory on the engine's GPU (SRLA_E_INVALID
 * otherwise). The records may be reused once the call returns. */
srla_status srla_scan_device(srla_engine* e, const srla_record* d_recs, uint64_t n, void* producer_stream,
                             uint32_t* pushed, uint64_t cap, uint64_t* n_pushed);

/* The engine-owned candidate list (DetectPipeline::candidates, pipeline.hpp:131),
 * insertion order. */
srla_status srla_candidates(srla_engine* e, uint32_t* out, uint64_t cap, uint64_t* n);
/* Replace it (the CandidateList argument of report_window / slide);
 * duplicates are dropped keeping first occurrences. */
srla_status srla_set_candidates(srla_engine* e, const uint32_t* hosts, uint64_t n);

/* EstimatorArray::report_window over the engine's candidate list
 * (sea.hpp:288-309): entries sorted by host, union_linear_weight, Eq. 9
 * estimate (host LUT of corrected_estimate_from, sea.hpp:270-279), theta cut.
 * *fill_product receives union_fill_product() (sea.hpp:261-265). */
srla_status srla_report(srla_engine* e, srla_entry* out, uint64_t cap, uint64_t* n_out,
                        double* fill_product);

/* EstimatorArray::slide over the engine's candidate list (sea.hpp:316-338);
 * the list becomes the retained list. */
srla_status srla_slide(srla_engine* e, uint64_t* n_retained);

/* DetectPipeline::process_slice after the scan (pipeline.hpp:119-128): report
 * if want_report and slice_id + 1 >= window, then slide. *n_out = 0 when no
 * report is due. */
srla_status srla_end_slice(srla_engine* e, uint64_t slice_id, int want_report, srla_entry* out,
                           uint64_t cap, uint64_t* n_out, uint64_t* n_retained);

/* The same as srla_end_slice, split in two: _async starts the end-of-slice
 * work and returns; a following srla_scan_batch with host records stages its
 * host->device copies while it runs (the copies are the bound of a host-fed
 * scan). `out` must stay valid until srla_end_slice_wait, which returns the
 * report size and retained-candidate count. Any other call waits for it too. */
srla_status srla_end_slice_async(srla_engine* e, uint64_t slice_id, int want_report, srla_entry* out,
                                 uint64_t cap);
srla_status srla_end_slice_wait(srla_engine* e, uint64_t* n_out, uint64_t* n_retained);

/* srla_end_slice with the report handed off compactly: hosts (ascending) and
 * union weights (8 bytes per entry instead of 24; host or device memory) plus this window's Eq. 9
 * table over the g'+1 possible weights: estimate = est_lut[w], has_estimate =
 * flags_lut[w] & 1, is_super = (flags_lut[w] >> 1) & 1. Same results as the
 * srla_entry form (sea.hpp:296-305). */
srla_status srla_end_slice_compact(srla_engine* e, uint64_t slice_id, int want_report, uint32_t* hosts,
                                   uint32_t* weights, uint64_t cap, uint64_t* n_out, double* est_lut,
                                   uint8_t* flags_lut, uint64_t* n_retained);

/* union_rough_weight / union_linear_weight (sea.hpp:219-243) per host; either
 * output may be NULL. */
srla_status srla_union_weights(srla_engine* e, const uint32_t* hosts, uint64_t n,
                               uint32_t* rough_w, uint32_t* linear_w);
/* union_view (sea.hpp:199-217); linear may be NULL (include_linear = false).
 * rough / linear receive g / g' words widened to uint32. */
srla_status srla_union_view(srla_engine* e, uint32_t aip, uint16_t* indicator, uint32_t* rough,
                            uint32_t* linear);
/* count_active over each linear row (the numerators of row_fill_fraction,
 * sea.hpp:248-257); `counts` has `rows` entries. */
srla_status srla_row_active(srla_engine* e, uint64_t* counts);
/* corrected_estimate_from (sea.hpp:270-279), host arithmetic, bit-identical. */
srla_status srla_estimate_from(const srla_engine* e, uint32_t weight, double fill_product,
                               double* estimate, int* has_estimate);

/* Raw rows (indicator_row / rough_row / linear_row, sea.hpp:341-346) as
 * little-endian W-byte words (u16 for the indicator). `bytes` must equal the
 * row size. */
srla_status srla_row_bytes(const srla_engine* e, int kind, uint64_t* bytes);
srla_status srla_export_row(srla_engine* e, uint32_t row, int kind, void* buf, uint64_t bytes);
srla_status srla_import_row(srla_engine* e, uint32_t row, int kind, const void* buf,
                            uint64_t bytes);
/* Byte range [offset, offset + bytes) of a raw row in the same layout, so a
 * 16 GiB row (2^24 columns) streams to or from a snapshot file in bounded
 * pieces (snapshot.hpp:117-120, 176-181). Packed 4-bit tables need an even
 * offset and size. Pinned buffers (srla_host_alloc) are copied by DMA
 * directly, pageable ones through the engine's pinned staging. Epoch-stamp
 * rows keep their histograms exact across a partial import. */
srla_status srla_export_range(srla_engine* e, uint32_t row, int kind, uint64_t offset, void* buf, uint64_t bytes);
srla_status srla_import_range(srla_engine* e, uint32_t row, int kind, uint64_t offset, const void* buf,
                              uint64_t bytes);
/* Page-locked host memory (cudaMallocHost) for callers without CUDA headers. */
srla_status srla_host_alloc(uint64_t bytes, void** out);
srla_status srla_host_free(void* p);

/* Block digests of one raw row (indicator_row / rough_row / linear_row,
 * sea.hpp:341-346) in the reference's little-endian byte layout, computed on
 * the device: per 1 MiB block, the wrapping sum over its 8-byte words w_i
 * (zero-padded) of avalanche64(w_i ^ avalanche64(i + 1)), i = the word's index
 * in the row. Parity at 2^24 columns compares these against the reference's
 * rows (oracle/ref_capi.cpp block_sums) instead of exporting 64 GiB per slice.
 * out = NULL queries *n_blocks. */
srla_status srla_state_blocks(srla_engine* e, uint32_t row, int kind, uint64_t* out, uint64_t cap,
                              uint64_t* n_blocks);
/* The same block sums over `bytes` of any device buffer (e.g. a record batch);
 * `out` is host memory with room for ceil(bytes / 2^20) sums. */
srla_status srla_block_sums(const void* d_buf, uint64_t bytes, uint64_t* out, uint64_t cap, void* stream);

srla_status srla_stats_get(const srla_engine* e, srla_stats* out);

/* Device time of the dominant kernel (K1 scan, CUDA events on the engine
 * stream around each launch) and of end-of-slice (report + slide: device
 * events, and host wall time including the report hand-off). */
typedef struct srla_timing {
    double scan_kernel_ms;
    uint64_t scan_kernel_launches;
    uint64_t scan_kernel_records;
    double end_slice_device_ms;
    double end_slice_wall_ms;
    double last_end_slice_device_ms;
    double last_end_slice_wall_ms;
    uint64_t end_slices;
    double order_wall_ms;   /* K2..K5 + candidate append, per-chunk host wall, summed */
    double report_wall_ms;  /* report_window part of end-of-slice */
    double slide_wall_ms;   /* slide part of end-of-slice */
    /* device time (CUDA events on the engine stream) of the other hot kernels */
    double split_kernel_ms;       /* k_split: region bins -> fine slice bins */
    uint64_t split_kernel_launches;
    uint64_t split_entries;       /* linear marks re-binned */
    double apply_kernel_ms;       /* k_slice_apply(_bulk) / k_slice_stamp */
    uint64_t apply_kernel_launches;
    uint64_t apply_entries;       /* linear marks applied */
    uint64_t apply_stream_bytes;  /* table bytes read + written by whole-slice passes */
    double gather_kernel_ms;      /* k_union_linear(_epoch): report union weights */
    uint64_t gather_kernel_launches;
    uint64_t gather_bytes;        /* candidates x rows x g' x W */
    double sync_wait_ms;          /* host time blocked on engine-stream synchronisation (scan ordering) */
    uint64_t syncs;
    double alloc_ms;              /* process-wide device/pinned (re)allocation host time */
    uint64_t allocs;
    double serial_kernel_ms;      /* k_serial: ordered indicator resolution of flagged hosts */
    uint64_t serial_kernel_launches;
    uint64_t flagged_hosts;       /* hosts resolved by k_serial */
} srla_timing;
srla_status srla_timing_get(const srla_engine* e, srla_timing* out);
srla_status srla_timing_reset(srla_engine* e);
srla_status srla_synchronize(srla_engine* e);
/* The engine's cudaStream_t (as void*), for callers that time on it. */
srla_status srla_stream(srla_engine* e, void** stream);

/* Synthetic trace on the device: generate_trace (generator.hpp:117-161),
 * byte-identical to the reference, one slice at a time. `out` is device
 * memory with room for *n_out records (query with out = NULL). Valid for
 * slice_seconds == 1 (no in-slice reordering); other specs return
 * SRLA_E_INVALID. */
typedef struct srla_plant {
    uint32_t host;
    uint32_t cardinality;
    uint32_t first_slice;
    uint32_t last_slice;
} srla_plant;

typedef struct srla_trace_spec {
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
    const srla_plant* plants;
} srla_trace_spec;

typedef struct srla_generator srla_generator;
srla_status srla_generator_create(const srla_trace_spec* spec, int device, srla_generator** out);
srla_status srla_generator_destroy(srla_generator* g);
/* Records in slice `slice` (0-based); out = NULL just reports the count. */
srla_status srla_generate_slice(srla_generator* g, uint64_t slice, srla_record* out_device,
                                uint64_t cap, uint64_t* n_out, void* stream);

/* Multi-GPU ingest: keep the records (device memory) whose monitored host is
 * owned by shard `part` of `nparts`, in their original order. Ownership is
 * HashFamily(seed).reduce(3, src, nparts) — function index 3 is unused by the
 * reference (hash.hpp:70-73), so shards are independent of every sketch hash.
 * *n_out receives the kept count; d_out has room for n records. */
srla_status srla_partition_records(const srla_record* d_in, uint64_t n, uint64_t seed, uint32_t nparts,
                                   uint32_t part, srla_record* d_out, uint64_t* n_out, void* stream);
/* Host-side owner of one address (same function). */
uint32_t srla_owner_of(uint64_t seed, uint32_t aip, uint32_t nparts);

/* ---- sharded pipeline: one rank of an owner-partitioned
 * DetectPipeline. The reference is single-node and has no counterpart
 * (multi-node sharding is its non-goal); each shard equals a reference
 * DetectPipeline fed the owner-filtered sub-trace in order
 * (pipeline.hpp:110-129), and the merged report equals the concatenation of
 * the shards' reports sorted by host (report_window's order, sea.hpp:294-295).
 *
 * The collectives go through a transport: NCCL over NVLink/NVSwitch
 * (srla_transport_nccl, libnccl.so.2 loaded at first use), or caller
 * callbacks (e.g. gloo for tests). Every rank calls every collective in the
 * same order. */
typedef struct srla_transport {
    void* ctx;
    uint32_t rank, world;
    /* 1: the callbacks receive host memory (the library stages device data
     * through pinned buffers); 0: device memory, ordered on `stream`. */
    int host_memory;
    /* every rank contributes `bytes` at `send`; `recv` receives world * bytes, rank-major */
    int (*allgather)(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream);
    /* send_bytes[j] bytes at send + send_off[j] go to rank j; recv_bytes[i]
     * bytes from rank i land at recv + recv_off[i] */
    int (*alltoallv)(void* ctx, const void* send, const uint64_t* send_bytes, const uint64_t* send_off, void* recv,
                     const uint64_t* recv_bytes, const uint64_t* recv_off, void* stream);
} srla_transport;

/* ncclGetUniqueId (128 bytes): rank 0 creates it and broadcasts it out of band. */
srla_status srla_nccl_unique_id(void* id128);
/* An NCCL communicator for (rank, world) on `device`, wrapped as a transport
 * (device memory, the shard's stream). */
srla_status srla_transport_nccl(const void* id128, uint32_t rank, uint32_t world, int device, srla_transport* out);
srla_status srla_transport_nccl_destroy(srla_transport* t);

typedef struct srla_shard srla_shard;
/* The rank's engine (srla_create(cfg, device)) behind a transport (copied). */
srla_status srla_shard_create(const srla_config* cfg, int device, const srla_transport* t, srla_shard** out);
srla_status srla_shard_destroy(srla_shard* s);
/* The rank's engine (stats, timing, rows, candidates). Owned by the shard. */
srla_status srla_shard_engine(srla_shard* s, srla_engine** e);

/* How srla_shard_process_slice's records arrive. */
enum {
    SRLA_SHARD_OWNED = 0, /* already owner-partitioned (e.g. NIC RSS by host hash): scanned as given */
    SRLA_SHARD_RANGE = 1  /* this rank's contiguous range of the slice (ranges in rank order): partitioned
                           * by owner on the device and exchanged all-to-all, sources concatenated in rank
                           * order so every owner sees its records in slice order */
};

/* DetectPipeline::process_slice for one slice across the ranks: scan, then
 * if want_report and slice_id + 1 >= window the report all-gather (entry
 * counts, (host, weight) words and each shard's Eq. 9 table) merged by host
 * on the device into `out` (host memory, cap entries; *n_out = the merged
 * size, 0 when no report is due), then slide. *n_scanned = records this rank
 * scanned. Collective: every rank calls it for every slice. A report larger
 * than `cap` returns SRLA_E_CAPACITY with *n_out set, after the slice has
 * completed (fetch it with srla_shard_last_report). */
srla_status srla_shard_process_slice(srla_shard* s, uint64_t slice_id, const srla_record* recs, uint64_t n,
                                     int on_device, int input_mode, int want_report, srla_entry* out, uint64_t cap,
                                     uint64_t* n_out, uint64_t* n_scanned);
/* The last merged report again (e.g. after SRLA_E_CAPACITY from
 * srla_shard_process_slice, which still completed the slice). */
srla_status srla_shard_last_report(srla_shard* s, srla_entry* out, uint64_t cap, uint64_t* n_out);

/* Device memory for callers without CUDA headers (the drop-in C++ API). */
srla_status srla_device_alloc(int device, uint64_t bytes, void** out);
srla_status srla_device_free(int device, void* p);
srla_status srla_copy_to_device(int device, void* dst, const void* src, uint64_t bytes);
srla_status srla_copy_to_host(int device, void* dst, const void* src, uint64_t bytes);

/* ---- ingest front end on the device (trace.hpp) ----
 * All buffers are device memory; `stream` is a cudaStream_t (NULL: default). */

/* for_each_record's binary branch (trace.hpp:109-170, replaces
 * read_trace/for_each_record for SRLT files): `d_bytes` is the whole file
 * ("SRLT", version 1, packed little-endian u32 ts/src/dst). Bad magic or
 * version, a truncated last record and a timestamp regression return
 * SRLA_E_INPUT with the reference's message; *n_out = the records before the
 * failure, as the reference delivers them. d_out has room for
 * (nbytes - 5) / 12 records. */
srla_status srla_parse_srlt(const void* d_bytes, uint64_t nbytes, srla_record* d_out, uint64_t* n_out, void* stream);

/* orient_record over a batch (trace.hpp:223-238, OrientStats :212-221): src in
 * the prefix and dst outside -> kept; the reverse -> flipped (src <-> dst);
 * both / neither -> dropped and counted. Output in input order. */
typedef struct srla_orient_stats {
    uint64_t kept, flipped, dropped_both, dropped_neither;
} srla_orient_stats;
srla_status srla_orient_records(const srla_record* d_in, uint64_t n, uint32_t prefix_addr, uint32_t prefix_bits,
                                srla_record* d_out, uint64_t* n_out, srla_orient_stats* stats, void* stream);

/* SlicePartitioner (trace.hpp:243-281) over an ordered batch: the origin is
 * the first record's ts; offsets[s] (host memory, n_slices + 1 entries) is the
 * first record of slice s, empty slices included. offsets == NULL queries
 * *n_slices. A timestamp regression returns SRLA_E_INPUT. */
srla_status srla_slice_bounds(const srla_record* d_recs, uint64_t n, uint32_t slice_seconds, uint64_t* offsets,
                              uint64_t cap, uint64_t* n_slices, void* stream);

/* ---- exact sliding-window cardinalities on the device (ground truth;
 * oracle.hpp:45-203). SliceRingStore semantics: pairs
 * observed in the current slice, a ring of the last max_window slices, a
 * window [t, t+k) observable only at the end of slice t+k-1 (SRLA_E_RANGE
 * with the reference's message otherwise). */
typedef struct srla_exact srla_exact;
srla_status srla_exact_create(uint32_t max_window, int device, srla_exact** out);
srla_status srla_exact_destroy(srla_exact* x);
/* SliceRingStore::observe for a batch: (src = aip, dst = bip) of every record
 * joins the current slice (host or device records, like srla_scan_batch). */
srla_status srla_exact_observe(srla_exact* x, const srla_record* recs, uint64_t n, int on_device);
srla_status srla_exact_end_slice(srla_exact* x);
srla_status srla_exact_current_slice(srla_exact* x, uint64_t* slice);
/* PairRecorderStore::pair_count: distinct pairs live in the ring. */
srla_status srla_exact_pair_count(srla_exact* x, uint64_t* n);
/* cardinalities(t, k): every host with a nonzero distinct count, ascending by
 * address, and its count. hosts = NULL (or cap too small) returns
 * SRLA_E_CAPACITY with *n_out = the number of hosts. */
srla_status srla_exact_cardinalities(srla_exact* x, uint64_t window_start, uint32_t window, uint32_t* hosts,
                                     uint64_t* counts, uint64_t cap, uint64_t* n_out);

#ifdef __cplusplus
}
#endif
#endif /* SRLA_H */
