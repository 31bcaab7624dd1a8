// engine.cu — the SRLA engine behind the C ABI (include/srla.h).
//
// One engine = one EstimatorArray's state resident in HBM plus the
// DetectPipeline's candidate list, driven on one CUDA stream. The scan is
// processed in chunks; each chunk runs K1 scan -> K2 crossing -> K5 rough
// commit -> K3 first crossings -> K4 ordered indicator resolution, which
// reproduces the reference's record-order semantics exactly (kernels.cuh).
#include <cub/cub.cuh>
#include <thrust/iterator/counting_iterator.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <thread>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "host_math.h"
#include "kernels.cuh"
#include "scan_binned.cuh"
#include "epoch.cuh"
#include "nibble.cuh"
#include "digest.cuh"
#include "order.cuh"
#include "srla.h"

namespace srla {

struct Error : std::runtime_error {
    srla_status code;
    Error(srla_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define CK(x)                                                                                 \
    do {                                                                                      \
        cudaError_t e_ = (x);                                                                 \
        if (e_ != cudaSuccess)                                                                \
            throw ::srla::Error(SRLA_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

// device/pinned (re)allocations: count and host time (srla_timing)
inline double g_alloc_ms = 0.0;
inline uint64_t g_allocs = 0;
struct AllocTimer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    AllocTimer(size_t bytes = 0, size_t cap = 0) {
        static const bool verbose = [] { const char* v = std::getenv("SRLA_TRACE_ALLOC"); return v && v[0] == '1'; }();
        if (verbose) std::fprintf(stderr, "[srla] alloc %zu bytes (had %zu)\n", bytes, cap);
    }
    ~AllocTimer() {
        g_alloc_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++g_allocs;
    }
};

struct PairHash {
    size_t operator()(const std::pair<int, const void*>& k) const {
        return std::hash<const void*>()(k.second) ^ (static_cast<size_t>(k.first) * 0x9E3779B97F4A7C15ull);
    }
};

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    ~DevBuf() {
        if (p) cudaFree(p);
    }
    void ensure(size_t n) {
        if (n <= cap) return;
        AllocTimer at(n * sizeof(T), cap * sizeof(T));
        if (p) CK(cudaFree(p));
        p = nullptr;
        const size_t c = std::max<size_t>({n + n / 4, cap * 2, 256});
        CK(cudaMalloc(&p, c * sizeof(T)));
        cap = c;
    }
    // grow keeping the first `keep` elements (stream-ordered copy)
    void ensure_keep(size_t n, size_t keep, cudaStream_t st) {
        if (n <= cap) return;
        AllocTimer at(n * sizeof(T), cap * sizeof(T) + 2);
        const size_t c = std::max<size_t>({n, cap * 2, 256});
        T* q = nullptr;
        CK(cudaMalloc(&q, c * sizeof(T)));
        if (keep) CK(cudaMemcpyAsync(q, p, keep * sizeof(T), cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
        if (p) CK(cudaFree(p));
        p = q;
        cap = c;
    }
};

template <typename T>
struct PinBuf {
    T* p = nullptr;
    size_t cap = 0;
    PinBuf() = default;
    PinBuf(const PinBuf&) = delete;
    ~PinBuf() {
        if (p) cudaFreeHost(p);
    }
    // pinned allocations cost milliseconds: grow geometrically (x2) so a
    // candidate list that creeps up over the first window reallocates rarely
    void ensure(size_t n) {
        if (n <= cap) return;
        AllocTimer at(n * sizeof(T), cap * sizeof(T) + 1);
        if (p) CK(cudaFreeHost(p));
        p = nullptr;
        const size_t c = std::max<size_t>({n + n / 4, cap * 2, 4096});
        CK(cudaMallocHost(&p, c * sizeof(T)));
        cap = c;
    }
};

// Dynamic shared-memory caps are per kernel, shared by every engine on a
// device: only ever raise them (a smaller engine created later must not lower
// the cap a larger one launches with).
inline std::mutex g_smem_mu;
template <typename K>
void raise_smem_cap(K* kernel, size_t bytes) {
    static std::unordered_map<std::pair<int, const void*>, size_t, PairHash>* seen = nullptr;
    std::lock_guard<std::mutex> lk(g_smem_mu);
    if (!seen) seen = new std::unordered_map<std::pair<int, const void*>, size_t, PairHash>();
    int dev = 0;
    CK(cudaGetDevice(&dev));
    size_t& cur = (*seen)[{dev, reinterpret_cast<const void*>(kernel)}];
    if (bytes <= cur) return;
    CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)));
    cur = bytes;
}

struct Engine {
    // compact report hand-off (srla_end_slice_compact)
    struct Compact {
        uint32_t* hosts;
        uint32_t* weights;
        double* est;
        uint8_t* flags;
    };

    srla_config cfg{};
    int device = 0;
    cudaStream_t st = nullptr;
    DevCfg dc{};
    uint32_t tau = 0, thr = 0, wb = 1;
    uint64_t lin_words = 0, rough_words = 0;  // per row
    void* d_lin = nullptr;
    void* d_rough = nullptr;
    uint16_t* d_si = nullptr;
    uint32_t* d_stamp = nullptr;
    int sms = 148;

    static constexpr uint32_t kChunk = 1u << 27;      // records per ordered chunk (a C2 slice in one)
    static constexpr uint32_t kHostStage = 1u << 24;  // records per host->device hop

    DevBuf<uint32_t> ev;
    uint32_t ev_cap = 0;
    DevBuf<uint32_t> ctr;  // device counters
    PinBuf<uint32_t> pin_ctr;
    DevBuf<uint64_t> xkeys, xsorted, hp, hps, fmask, tkey, skey;
    DevBuf<uint32_t> cnt, off, hosts, tval, sval, towner, posof, flagged, pushed, newhosts;
    DevBuf<uint8_t> status, definite, fl_und, fl_ins, isnew, keep, temp;
    DevBuf<uint32_t> csip, csip2, qhosts, sorted_hosts, weights, rweights;
    uint64_t ncsip = 0;
    DevBuf<unsigned long long> cset;
    uint64_t cset_cap = 0;
    DevBuf<unsigned long long> d_counts;
    DevBuf<uint32_t> dstage[2];
    PinBuf<uint32_t> pstage[2], pin_hosts, pin_w;
    cudaStream_t cs = nullptr;  // host->device copy stream
    cudaStream_t st2 = nullptr; // end-of-slice side stream (rough aging overlaps the report)
    cudaEvent_t ev_eos_start = nullptr, ev_reported = nullptr, ev_retained = nullptr;
    bool slide_begun = false;
    // report hand-off: device->host copies on their own stream
    static constexpr uint32_t kReportParts = 4;
    cudaEvent_t ev_counts_ready = nullptr, ev_counts = nullptr;
    // the retained candidate list sorted by host (built on st2 by the slide)
    DevBuf<uint32_t> sorted_ret, newsorted, sorted_tmp;
    uint64_t nsorted_ret = 0;
    bool sorted_ret_valid = true;  // the empty list is sorted
    uint64_t last_sort_new = 0;  // hosts sorted at the last report (all of them without a sorted prefix)
    cudaStream_t ds = nullptr;
    cudaEvent_t ev_sorted = nullptr, ev_d2h = nullptr, ev_part[kReportParts] = {};
    // table maintenance queued on st2 by slide_finish (join_maint)
    cudaEvent_t ev_maint_lin = nullptr, ev_maint = nullptr;
    bool maint_lin_pending = false, maint_pending = false;
    DevBuf<uint8_t> temp2;  // CUB scratch of the side stream
    cudaEvent_t ev_copied[2] = {}, ev_scanned[2] = {};
    cudaEvent_t t_scan0 = nullptr, t_scan1 = nullptr, t_eos0 = nullptr, t_eos1 = nullptr;
    srla_timing timing{};
    PinBuf<unsigned long long> pin_counts;
    std::vector<uint32_t> host_pushed;
    // asynchronous end-of-slice (srla_end_slice_async / srla_end_slice_wait)
    std::thread eos_thread;
    struct EosResult {
        bool pending = false;
        srla_status code = SRLA_OK;
        std::string msg;
        uint64_t n = 0, nret = 0;
    } eos;
    PinBuf<uint8_t> pin_lut;
    DevBuf<uint8_t> d_lut;
    DevBuf<unsigned long long> d_entries;
    std::vector<double> lut_est;
    std::vector<uint8_t> lut_has, lut_sup;
    bool collect_pushed = false;
    srla_stats stats{};

    // ordering phase on device counts (order.cuh); SRLA_ORDER=legacy selects
    // the sorted, host-synchronised path (kernels.cuh K2..K4f) throughout
    bool fast_order = [] { const char* v = std::getenv("SRLA_ORDER"); return !(v && std::string(v) == "legacy"); }();
    DevBuf<uint32_t> octr, ht_vals, tt_vals, hl, tl, host_a, host_p, host_cols, flist, bm_new, bm_push, bits_cnt, newlist,
        pushlist;
    DevBuf<unsigned long long> ht_keys, tt_keys;
    DevBuf<uint64_t> host_f;
    DevBuf<uint8_t> ostatus;
    PinBuf<uint32_t> pin_octr;
    uint32_t order_cap = 0;
    uint64_t ht_mask = 0, tt_mask = 0;

    void setup_order(uint32_t cap) {
        if (cap <= order_cap) return;
        uint64_t hs = 1024, ts = 1024;
        while (hs < 2ull * cap) hs <<= 1;
        while (ts < 2ull * cap * std::min<uint32_t>(cfg.rows, 8)) ts <<= 1;
        octr.ensure(kOcCount);
        pin_octr.ensure(kOcCount);
        ht_keys.ensure(hs); ht_vals.ensure(hs); tt_keys.ensure(ts); tt_vals.ensure(ts);
        hl.ensure(cap); tl.ensure(uint64_t(cap) * std::min<uint32_t>(cfg.rows, 8));
        host_a.ensure(cap); host_p.ensure(cap); host_f.ensure(cap); ostatus.ensure(cap);
        host_cols.ensure(uint64_t(cap) * kOrderRows); flist.ensure(cap);
        newlist.ensure(cap); pushlist.ensure(cap);
        xkeys.ensure(cap);
        // the sorted fallback's scratch (order_tail), sized once: a regrowth is
        // a cudaFree, a device-wide synchronisation
        const size_t m = std::min<size_t>(cap, size_t(1) << 21);
        xsorted.ensure(m); hp.ensure(m); hps.ensure(m); fmask.ensure(m); cnt.ensure(m); off.ensure(m);
        hosts.ensure(m); status.ensure(m); definite.ensure(m); fl_und.ensure(m); fl_ins.ensure(m);
        flagged.ensure(m); pushed.ensure(m); newhosts.ensure(m); isnew.ensure(m);
        const size_t t = m * std::min<uint32_t>(cfg.rows, 8);
        tkey.ensure(t); skey.ensure(t); tval.ensure(t); sval.ensure(t); towner.ensure(t); posof.ensure(t);
        const uint64_t words = (uint64_t(kChunk) + 31) / 32;
        bm_new.ensure(words); bm_push.ensure(words);
        bits_cnt.ensure((words + kBitsWords - 1) / kBitsWords + 1);
        CK(cudaMemsetAsync(ht_keys.p, 0, ht_keys.cap * 8, st));
        CK(cudaMemsetAsync(ht_vals.p, 0xFF, ht_vals.cap * 4, st));
        CK(cudaMemsetAsync(tt_keys.p, 0, tt_keys.cap * 8, st));
        CK(cudaMemsetAsync(tt_vals.p, 0xFF, tt_vals.cap * 4, st));
        CK(cudaMemsetAsync(bm_new.p, 0, bm_new.cap * 4, st));
        CK(cudaMemsetAsync(bm_push.p, 0, bm_push.cap * 4, st));
        ht_mask = hs - 1;
        tt_mask = ts - 1;
        order_cap = cap;
    }

    OrderBufs order_bufs(bool collect) {
        return OrderBufs{octr.p, ht_keys.p, ht_vals.p, ht_mask, hl.p, tt_keys.p, tt_vals.p, tt_mask, tl.p,
                         host_a.p, host_p.p, host_f.p, host_cols.p, flist.p, ostatus.p, bm_new.p,
                         collect ? bm_push.p : nullptr, order_cap};
    }

    // ordered compaction of a packet bitmap into `out` (device count -> octr[ctr_idx])
    void emit_bitmap(uint32_t* bm, uint32_t n, const uint32_t* d_recs, uint32_t* out, uint32_t ctr_idx) {
        const uint32_t words = (n + 31) / 32;
        const uint32_t nb = (words + kBitsWords - 1) / kBitsWords;
        k_bits_count<<<nb, kBitsThreads, 0, st>>>(bm, words, bits_cnt.p);
        k_bits_scan<<<1, 1024, 0, st>>>(bits_cnt.p, nb, octr.p + ctr_idx);
        k_bits_emit<<<nb, kBitsThreads, 0, st>>>(bm, words, bits_cnt.p, d_recs, out);
        check_launch();
        launched(3);
    }

    // binned linear marks (scan_binned.cuh), for tables larger than L2
    bool use_bins = false;
    bool nib = false;  // linear recorders packed two per byte (nibble.cuh)
    BinCfg bcfg{};
    DevBuf<uint32_t> bins, bin_count, tile_prefix, fine_count;
    DevBuf<uint16_t> fine_bins;
    FineCfg fcfg{};
    bool bulk_ok = false;
    uint32_t bulk_end = 0;
    size_t split_smem = 0;

    // epoch-stamp linear table (epoch.cuh): u8 stamps, O(1) slide
    bool epoch = false;
    uint32_t stamp_sparse_max = 1024;  // SRLA_STAMP_SPARSE, read per engine at setup
    int dedup_mode = -1;               // SRLA_K1_DEDUP: 1 on, 0 off, -1 on after the first bin overflow
    uint32_t split_threads = 512;      // k_split block (SRLA_SPLIT_THREADS)
    uint32_t cur_epoch = 0;
    DevBuf<unsigned long long> hist;  // rows x 256
    PinBuf<unsigned long long> pin_hist;
    uint64_t sweep_pos = 0;
    EpochCfg ecfg() const { return EpochCfg{epoch ? 1u : 0u, cur_epoch, hist.p, lin_words}; }
    PinBuf<uint32_t> pin_bc;
    uint64_t pending_entries = 0;  // marks in the region bins
    uint64_t fine_pending = 0;     // marks split into the fine bins, not yet applied
    // Early split: right after K1 the region bins are split on stream ssplit,
    // concurrent with the scan's ordering phase (K2..K5, latency-bound); the
    // apply waits for it (flush_linear), as does the next K1.
    cudaStream_t ssplit = nullptr;
    cudaEvent_t ev_split_done = nullptr, ev_k1_done = nullptr;
    bool split_in_flight = false;
    bool early_split = [] { const char* v = std::getenv("SRLA_EARLY_SPLIT"); return !(v && v[0] == '0'); }();
    // Second region-bin set: a slice's K1 bins into it on stream sk while the
    // previous slice's asynchronous end-of-slice still flushes the first
    // (srla_end_slice_async followed by srla_scan_batch of device records).
    DevBuf<uint32_t> bins_alt, bin_count_alt, ctr_k1;
    PinBuf<uint32_t> pin_k1;
    cudaStream_t sk = nullptr;
    cudaEvent_t ev_scan_done = nullptr;
    // the overlapped K1 starts once the end-of-slice has queued its split
    // (K1 and the split are both SM-bound; the apply and gather that follow
    // are HBM-bound and co-run with K1)
    cudaEvent_t ev_k1_gate = nullptr;
    std::atomic<bool> k1_gate{false};
    bool in_async_eos = false;
    // Measured on B200 (C2): K1 co-running with the end-of-slice slows both
    // (K1 and the split are SM-bound; K1's shared memory and the apply's
    // slices cannot co-reside), 6.4 vs 6.1 ms per slice, so it is opt-in.
    bool overlap_on = [] { const char* v = std::getenv("SRLA_OVERLAP"); return v && v[0] == '1'; }();
    bool prefetch_next = false;  // bulk-prefetch region r+1 while applying r (measured slower; off)

    // ------------------------------------------------------------ kernel timers
    // Device time of the split / apply / gather kernels: event pairs on the
    // engine stream, resolved after the stream has passed them.
    enum TimerKind { kTimeSplit = 0, kTimeApply = 1, kTimeGather = 2, kTimeSerial = 3 };
    struct PendingTimer {
        cudaEvent_t a, b;
        int kind;
    };
    std::vector<cudaEvent_t> ev_pool;
    std::vector<PendingTimer> timers;
    DevBuf<unsigned long long> d_streamed;  // FineCfg::streamed
    PinBuf<unsigned long long> pin_streamed;
    cudaEvent_t take_event() {
        if (ev_pool.empty()) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            return e;
        }
        cudaEvent_t e = ev_pool.back();
        ev_pool.pop_back();
        return e;
    }
    cudaEvent_t timer_start(cudaStream_t s = nullptr) {
        cudaEvent_t a = take_event();
        CK(cudaEventRecord(a, s ? s : st));
        return a;
    }
    void timer_stop(cudaEvent_t a, int kind, cudaStream_t s = nullptr) {
        cudaEvent_t b = take_event();
        CK(cudaEventRecord(b, s ? s : st));
        timers.push_back({a, b, kind});
        if (timers.size() > 256) resolve_timers(true);
    }
    void resolve_timers(bool wait) {
        size_t keep = 0;
        for (size_t i = 0; i < timers.size(); ++i) {
            PendingTimer& t = timers[i];
            if (!wait && cudaEventQuery(t.b) != cudaSuccess) {
                cudaGetLastError();
                timers[keep++] = t;
                continue;
            }
            CK(cudaEventSynchronize(t.b));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, t.a, t.b));
            (t.kind == kTimeSplit    ? timing.split_kernel_ms
             : t.kind == kTimeApply  ? timing.apply_kernel_ms
             : t.kind == kTimeSerial ? timing.serial_kernel_ms
                                     : timing.gather_kernel_ms) += ms;
            ev_pool.push_back(t.a);
            ev_pool.push_back(t.b);
        }
        timers.resize(keep);
    }
    // Non-blocking: timers the stream has not reached yet are reported later
    // (the streamed-slice count is the device counter as of the last flush).
    void timing_snapshot(srla_timing* out) {
        resolve_timers(false);
        *out = timing;
        out->alloc_ms = g_alloc_ms;
        out->allocs = g_allocs;
        if (pin_streamed.p) out->apply_stream_bytes = 2ull * pin_streamed.p[0];
    }
    void timing_clear() {
        resolve_timers(true);
        timing = srla_timing{};
        if (d_streamed.p) {
            CK(cudaMemsetAsync(d_streamed.p, 0, sizeof(unsigned long long), st));
            CK(cudaStreamSynchronize(st));
            pin_streamed.p[0] = 0;
        }
    }

    // ------------------------------------------------------------ lifecycle
    explicit Engine(const srla_config& c, int dev) : cfg(c), device(dev) {
        validate();
        CK(cudaSetDevice(device));
        // the engine stream outranks the side stream: queued slide maintenance
        // and the candidate re-validation must not hold SMs the report needs
        int prio_low = 0, prio_high = 0;
        CK(cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high));
        CK(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, prio_high));
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&st2, cudaStreamNonBlocking, prio_low));
        CK(cudaEventCreateWithFlags(&ev_eos_start, cudaEventDisableTiming));
        for (cudaEvent_t* e : {&ev_reported, &ev_retained, &ev_maint_lin, &ev_maint, &ev_sorted, &ev_d2h, &ev_counts_ready,
                               &ev_counts})
            CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        for (cudaEvent_t& e : ev_part) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaStreamCreateWithFlags(&ds, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithPriority(&sk, cudaStreamNonBlocking, prio_low));
        CK(cudaEventCreateWithFlags(&ev_scan_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_k1_gate, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_split_done, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&ev_k1_done, cudaEventDisableTiming));
        // the early split yields to the ordering phase on the engine stream: the
        // split-first order measured 5.46 vs 5.19 ms per C2 step
        CK(cudaStreamCreateWithPriority(&ssplit, cudaStreamNonBlocking, prio_low));
        CK(cudaEventRecord(ev_scan_done, st));
        ctr_k1.ensure(4);
        pin_k1.ensure(4);
        for (int b = 0; b < 2; ++b) {
            CK(cudaEventCreateWithFlags(&ev_copied[b], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ev_scanned[b], cudaEventDisableTiming));
            CK(cudaEventRecord(ev_copied[b], cs));
            CK(cudaEventRecord(ev_scanned[b], st));
        }
        CK(cudaEventCreate(&t_scan0));
        CK(cudaEventCreate(&t_scan1));
        CK(cudaEventCreate(&t_eos0));
        CK(cudaEventCreate(&t_eos1));
        CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
        const uint32_t bits = cfg.recorder_bits;
        wb = bits <= 8 ? 1 : bits <= 16 ? 2 : 4;
        tau = srla_host::sampling_exponent(cfg.theta, cfg.rough_slots);
        thr = srla_host::super_weight_threshold(cfg.fill_ratio, cfg.rough_slots);
        dc.rows = cfg.rows;
        dc.cols = cfg.cols;
        dc.g = cfg.rough_slots;
        dc.gl = cfg.linear_slots;
        dc.k = cfg.window;
        dc.expired = bits == 32 ? 0xFFFFFFFFu : (1u << bits) - 1u;
        dc.tau_mask = tau >= 32 ? 0xFFFFFFFFu : (1u << tau) - 1u;
        dc.thr = thr;
        dc.gl_mask = (cfg.linear_slots & (cfg.linear_slots - 1)) == 0 ? cfg.linear_slots - 1 : 0;
        dc.wbytes = wb;
        dc.sub_sample = sub_key(cfg.seed, kSampleHash);
        dc.sub_rslot = sub_key(cfg.seed, kRoughSlotHash);
        dc.sub_ind = sub_key(cfg.seed, kIndicatorHash);
        for (uint32_t i = 0; i < kMaxRows; ++i) dc.sub_row[i] = sub_key(cfg.seed, kRowHashBase + i);
        dc.kh_sample = sub_hi_term(dc.sub_sample);
        dc.kh_rslot = sub_hi_term(dc.sub_rslot);
        for (uint32_t i = 0; i < kMaxRows; ++i) dc.kh_row[i] = sub_hi_term(dc.sub_row[i]);
        lin_words = static_cast<uint64_t>(cfg.cols) * cfg.linear_slots;
        rough_words = static_cast<uint64_t>(cfg.cols) * cfg.rough_slots;
        const uint64_t rows = cfg.rows;
        ctr.ensure(16);
        pin_ctr.ensure(16);
        setup_bins();  // decides the linear table's packing (nibble.cuh)
        CK(cudaMalloc(&d_lin, lin_bytes(rows * lin_words)));
        CK(cudaMalloc(&d_rough, rows * rough_words * wb));
        CK(cudaMalloc(&d_si, rows * cfg.cols * sizeof(uint16_t)));
        CK(cudaMalloc(&d_stamp, rows * rough_words * sizeof(uint32_t)));
        if (nib) {
            CK(cudaMemsetAsync(d_lin, static_cast<int>(dc.expired * 0x11u), lin_bytes(rows * lin_words), st));
        } else {
            fill_expired(d_lin, rows * lin_words);
        }
        fill_expired(d_rough, rows * rough_words);
        CK(cudaMemsetAsync(d_si, 0, rows * cfg.cols * sizeof(uint16_t), st));
        CK(cudaMemsetAsync(d_stamp, 0xFF, rows * rough_words * sizeof(uint32_t), st));
        setup_epoch();
        if (use_bins) reserve_candidates(size_t(1) << 21);
        rebuild_cset(1024);
        CK(cudaStreamSynchronize(st));
    }

    ~Engine() {
        if (eos_thread.joinable()) eos_thread.join();
        if (st) cudaStreamSynchronize(st);
        if (st2) cudaStreamSynchronize(st2);  // queued slide maintenance
        if (ds) cudaStreamSynchronize(ds);
        if (d_lin) cudaFree(d_lin);
        if (d_rough) cudaFree(d_rough);
        if (d_si) cudaFree(d_si);
        if (d_stamp) cudaFree(d_stamp);
        if (cs) cudaStreamSynchronize(cs);
        for (int b = 0; b < 2; ++b) {
            if (ev_copied[b]) cudaEventDestroy(ev_copied[b]);
            if (ev_scanned[b]) cudaEventDestroy(ev_scanned[b]);
        }
        for (cudaEvent_t e : {t_scan0, t_scan1, t_eos0, t_eos1})
            if (e) cudaEventDestroy(e);
        for (const PendingTimer& t : timers) {
            cudaEventDestroy(t.a);
            cudaEventDestroy(t.b);
        }
        for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
        if (cs) cudaStreamDestroy(cs);
        if (st2) {
            cudaStreamSynchronize(st2);
            cudaStreamDestroy(st2);
        }
        for (cudaEvent_t e : {ev_eos_start, ev_reported, ev_retained, ev_maint_lin, ev_maint, ev_sorted, ev_d2h,
                              ev_counts_ready, ev_counts})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_part)
            if (e) cudaEventDestroy(e);
        if (ds) {
            cudaStreamSynchronize(ds);
            cudaStreamDestroy(ds);
        }
        if (sk) {
            cudaStreamSynchronize(sk);
            cudaStreamDestroy(sk);
        }
        if (ev_scan_done) cudaEventDestroy(ev_scan_done);
        if (ev_k1_gate) cudaEventDestroy(ev_k1_gate);
        if (ssplit) {
            cudaStreamSynchronize(ssplit);
            cudaStreamDestroy(ssplit);
        }
        for (cudaEvent_t e : {ev_split_done, ev_k1_done, ev_input})
            if (e) cudaEventDestroy(e);
        if (st) cudaStreamDestroy(st);
    }

    // SeaConfig::validate (sea.hpp:44-51), RecorderModel (recorders.hpp:33-54),
    // EstimatorArray ctor (sea.hpp:122-126).
    void validate() const {
        auto bad = [](const char* m) { throw Error(SRLA_E_INVALID, m); };
        if (cfg.rows < 1) bad("rows must be >= 1");
        if (cfg.cols < 1) bad("cols must be >= 1");
        if (cfg.rough_slots < 1) bad("rough_slots must be >= 1");
        if (cfg.linear_slots < 2) bad("linear_slots must be >= 2");
        if (cfg.theta < 1) bad("theta must be >= 1");
        if (cfg.recorder_bits < 1 || cfg.recorder_bits > 32)
            throw Error(SRLA_E_INVALID, "recorder width must be in [1, 32] bits, got " +
                                            std::to_string(cfg.recorder_bits));
        const uint32_t e = cfg.recorder_bits == 32 ? 0xFFFFFFFFu : (1u << cfg.recorder_bits) - 1u;
        if (cfg.window < 1 || cfg.window > e)
            throw Error(SRLA_E_INVALID, "window of " + std::to_string(cfg.window) +
                                            " slices does not fit a " +
                                            std::to_string(cfg.recorder_bits) +
                                            "-bit recorder (valid range [1, " + std::to_string(e) + "])");
        if (cfg.rows > kMaxRows) bad("at most 64 rows supported");
        if (cfg.flags & ~uint32_t(SRLA_FLAG_EPOCH | SRLA_FLAG_LITERAL)) bad("unknown srla_config.flags bits");
        if ((cfg.flags & SRLA_FLAG_EPOCH) && (cfg.flags & SRLA_FLAG_LITERAL)) bad("conflicting srla_config.flags");
    }

    uint32_t blocks(uint64_t work, uint32_t per = 256, uint32_t waves = 8) const {
        const uint64_t b = (work + per - 1) / per;
        return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(b, uint64_t(sms) * waves)));
    }

    void launched(uint64_t n = 1) { stats.kernel_launches += n; }
    void lib_launched(uint64_t n = 1) { stats.library_launches += n; }
    void check_launch() { CK(cudaGetLastError()); }

    template <typename Fn>
    void with_w(Fn&& fn) {
        switch (wb) {
            case 1: fn(uint8_t{}); break;
            case 2: fn(uint16_t{}); break;
            default: fn(uint32_t{}); break;
        }
    }

    void fill_expired(void* t, uint64_t words) {
        with_w([&](auto w) {
            using W = decltype(w);
            k_fill<W><<<blocks(words, 256, 16), 256, 0, st>>>(static_cast<W*>(t), words, static_cast<W>(dc.expired));
        });
        check_launch();
        launched();
    }

    uint32_t read_ctr(uint32_t idx) {
        CK(cudaMemcpyAsync(pin_ctr.p + idx, ctr.p + idx, 4, cudaMemcpyDeviceToHost, st));
        sync_st();
        return pin_ctr.p[idx];
    }
    // engine-stream synchronisation with the host wait accounted (srla_timing)
    void sync_st() {
        const auto t0 = std::chrono::steady_clock::now();
        CK(cudaStreamSynchronize(st));
        timing.sync_wait_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        timing.syncs += 1;
    }

    // ------------------------------------------------------------ CUB helpers
    template <typename Fn>
    void cub_call(Fn&& fn, DevBuf<uint8_t>* tbuf = nullptr) {
        DevBuf<uint8_t>& t = tbuf ? *tbuf : temp;
        size_t bytes = 0;
        CK(fn(static_cast<void*>(nullptr), bytes));
        t.ensure(bytes + 16);
        CK(fn(static_cast<void*>(t.p), bytes));
        lib_launched();
    }

    static int bit_length(uint64_t x) { return x ? 64 - __builtin_clzll(x) : 1; }

    // Large sketches: size the candidate-list buffers for 2M candidates up
    // front, so the list creeping up over the first windows never reallocates
    // (a cudaFree synchronises the whole device) inside a running pipeline.
    void reserve_candidates(size_t n) {
        csip.ensure_keep(n, 0, st);
        csip2.ensure(n); sorted_hosts.ensure(n); weights.ensure(n); keep.ensure(n); sorted_ret.ensure(n);
        sorted_tmp.ensure(n);
        newsorted.ensure(n); d_entries.ensure(3 * n);
        size_t cap = 1024;
        while (cap < 2 * n) cap <<= 1;
        cset.ensure(cap);
    }

    // ------------------------------------------------------------ candidate set
    void rebuild_cset(uint64_t want, cudaStream_t s = nullptr) {
        if (!s) s = st;
        uint64_t cap = 1024;
        while (cap < 2 * want) cap <<= 1;
        if (cap != cset_cap) {
            cset.ensure(cap);
            cset_cap = cap;
        }
        CK(cudaMemsetAsync(cset.p, 0, cset_cap * sizeof(unsigned long long), s));
        if (ncsip) {
            k_cset_insert<<<blocks(ncsip), 256, 0, s>>>(csip.p, static_cast<uint32_t>(ncsip), cset.p, cset_cap - 1);
            check_launch();
            launched();
        }
    }

    // Append hosts (distinct, in order) to the candidate list unless present.
    void append_candidates(const uint32_t* d_hosts, uint32_t n) {
        if (!n) return;
        isnew.ensure(n);
        newhosts.ensure(n);
        k_cset_lookup<<<blocks(n), 256, 0, st>>>(d_hosts, n, cset.p, cset_cap - 1, isnew.p);
        check_launch();
        launched();
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, d_hosts, isnew.p, newhosts.p, ctr.p + 7, static_cast<int>(n), st);
        });
        append_new(newhosts.p, read_ctr(7));
    }

    // Append `nn` hosts already known to be new (distinct, in order).
    void append_new(const uint32_t* d_new, uint32_t nn) {
        if (!nn) return;
        csip.ensure_keep(ncsip + nn, ncsip, st);
        CK(cudaMemcpyAsync(csip.p + ncsip, d_new, nn * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st));
        // keep the sorted view of the list current: sort the newcomers, merge
        if (sorted_ret_valid && nsorted_ret == ncsip) {
            newsorted.ensure(nn);
            sorted_tmp.ensure(ncsip + nn);
            sorted_ret.ensure_keep(ncsip + nn, ncsip, st);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceRadixSort::SortKeys(t, b, d_new, newsorted.p, static_cast<int>(nn), 0, 32, st);
            });
            k_merge_sorted<<<blocks((ncsip + nn + 7) / 8), 256, 0, st>>>(sorted_ret.p, static_cast<uint32_t>(ncsip),
                                                                       newsorted.p, nn, sorted_tmp.p);
            check_launch();
            launched();
            std::swap(sorted_ret.p, sorted_tmp.p);
            std::swap(sorted_ret.cap, sorted_tmp.cap);
            nsorted_ret = ncsip + nn;
        }
        ncsip += nn;
        if (2 * ncsip > cset_cap) {
            rebuild_cset(ncsip);
        } else {
            k_cset_insert<<<blocks(nn), 256, 0, st>>>(d_new, nn, cset.p, cset_cap - 1);
            check_launch();
            launched();
        }
    }

    // ------------------------------------------------------------ binned linear marks
    // k_slice_apply_nib: two stages of (packed slice + its mark list)
    uint64_t nib_apply_smem() const { return 2 * (lin_bytes(1ull << fcfg.shift) + uint64_t(fcfg.cap) * 2); }

    // Bytes of `words` linear recorders in the device layout.
    uint64_t lin_bytes(uint64_t words) const { return nib ? words / 2 : words * wb; }

    // Epoch stamps (epoch.cuh) for this config: tables of 16 GiB and more, or
    // srla_config.flags / SRLA_EPOCH (setup_epoch may still decline).
    bool epoch_wanted() const {
        const char* env = std::getenv("SRLA_EPOCH");
        bool want = uint64_t(cfg.rows) * lin_words * wb >= (16ull << 30);
        if (cfg.flags & SRLA_FLAG_EPOCH) want = true;
        if (cfg.flags & SRLA_FLAG_LITERAL) want = false;
        if (env) want = env[0] == '1';
        return want;
    }

    void setup_bins() {
        const char* direct = std::getenv("SRLA_DIRECT_MARKS");  // A/B switch for measurements
        if (cfg.rows > kBinRows || (direct && direct[0] == '1')) return;
        // literal recorders of z <= 4 bits packed two per byte when the table
        // geometry allows it (every slice whole and 16-byte aligned)
        const char* ne = std::getenv("SRLA_NIBBLE");
        nib = wb == 1 && cfg.recorder_bits <= 4 && !epoch_wanted() && !(ne && ne[0] == '0');
        if (nib && !setup_bins_geometry()) nib = false;
        if (!nib) setup_bins_geometry();
    }

    bool setup_bins_geometry() {
        const uint64_t total_words = uint64_t(cfg.rows) * lin_words;
        const char* force = std::getenv("SRLA_FORCE_BINS");     // exercise the binned path on small tables (tests)
        const bool forced = force && force[0] == '1';
        const bool small = total_words * wb < (256ull << 20);
        if (!forced && small) return false;
        uint32_t shift = 0;
        // 8 MB coarse regions: K1's fan-out (regions per tile) against the
        // split's (fine slices per region); measured best on C2 with the
        // device-count ordering and a full-GPU early split (4-64 MB swept,
        // profiles/r02/ab_region_waves.txt)
        uint64_t region_bytes = 8ull << 20;
        const char* rm = std::getenv("SRLA_REGION_MB");
        if (rm) region_bytes = std::strtoull(rm, nullptr, 10) << 20;
        while (lin_bytes(1ull << (shift + 1)) <= region_bytes) ++shift;
        if (forced)
            while (shift > 4 && (total_words >> shift) < 8) --shift;  // ~8 regions even for tiny tables
        // at most 1024 regions by default (more costs K1 coalescing: C3 with 4096 regions
        // 4.9 ms vs 2.6 ms with 1024, profiles/r02/ab_region_waves.txt); kMaxRegions if asked for
        const uint64_t max_regions = rm ? kMaxRegions : 1024;
        while (((total_words + (1ull << shift) - 1) >> shift) > max_regions) ++shift;
        // fine slices (u16 offsets): 32 KB, or larger so one region splits into <= 4096
        uint32_t fs = 0;
        uint64_t fine_bytes = 32ull << 10;  // 32 KB: two buffers per block
        if (const char* fk = std::getenv("SRLA_FINE_KB")) fine_bytes = std::strtoull(fk, nullptr, 10) << 10;
        while (lin_bytes(1ull << (fs + 1)) <= fine_bytes) ++fs;
        if (nib) fs = std::min<uint32_t>(fs, 16);  // u16 offsets within a slice
        fs = std::min(fs, shift);
        if (forced && small) fs = std::max<uint32_t>(std::min<uint32_t>(shift, 4), shift > 3 ? shift - 3 : 0);
        while (shift - fs > 12) ++fs;  // split fan-out <= 4096 slices per region
        if (lin_bytes(1ull << fs) > (64ull << 10) || fs > 16) return false;  // slices fit twice in shared memory
        if (nib) {  // nibble tables: whole, 16-byte slices; rows of whole 16-byte vectors (bulk kernel only)
            const uint64_t slice_words = 1ull << fs;
            if (lin_bytes(slice_words) % 16 || (lin_words % 32) || lin_words < slice_words || total_words % slice_words)
                return false;
        }
        bcfg.region_shift = shift;
        bcfg.nregions = static_cast<uint32_t>((total_words + (1ull << shift) - 1) >> shift);
        // K1 stages (region, offset) as one word when the table has <= 2^32 recorders (C2: exactly)
        bcfg.pack = shift < 32 && (uint64_t(bcfg.nregions) << shift) <= (1ull << 32) ? 1u : 0u;
        if (const char* pk = std::getenv("SRLA_K1_PACK"); pk && pk[0] == '0') bcfg.pack = 0;
        // K1's duplicate-mark filter: off until a region bin overflows (then on
        // for the engine's life); SRLA_K1_DEDUP=1 / 0 forces it
        const char* dd = std::getenv("SRLA_K1_DEDUP");
        dedup_mode = dd ? (dd[0] == '1' ? 1 : 0) : -1;
        bcfg.dedup = bcfg.pack && dedup_mode == 1 ? 1u : 0u;
        bcfg.ab_nohoist = std::getenv("SRLA_K1_HOIST") && std::getenv("SRLA_K1_HOIST")[0] == '0' ? 1u : 0u;
        bcfg.seen_ovf = nullptr;  // set where K1 runs with the ordering counters
        // forced-binned small tables (tests): tiny bins, so the overflow paths run
        uint64_t coarse_total = small ? (1ull << 16) : (1ull << 29);
        if (const char* be = std::getenv("SRLA_SMALL_BIN_ENTRIES"); be && small) coarse_total = std::strtoull(be, nullptr, 10);
        bcfg.cap = static_cast<uint32_t>(std::min<uint64_t>(coarse_total / bcfg.nregions, 0xFFFFFFF0ull)) & ~3u;
        bins.ensure(uint64_t(bcfg.cap) * bcfg.nregions + 4);  // + 16 bytes: k_split bulk-loads whole 16-byte units
        bin_count.ensure(bcfg.nregions);
        if (overlap_on) {
            bins_alt.ensure(uint64_t(bcfg.cap) * bcfg.nregions + 4);
            bin_count_alt.ensure(bcfg.nregions);
            CK(cudaMemsetAsync(bin_count_alt.p, 0, bcfg.nregions * sizeof(uint32_t), st));
        }
        pin_bc.ensure(2 * bcfg.nregions + 2);
        tile_prefix.ensure(2 * bcfg.nregions + 2);
        CK(cudaMemsetAsync(bin_count.p, 0, bcfg.nregions * sizeof(uint32_t), st));
        bcfg.bins = bins.p;
        bcfg.count = bin_count.p;
        fcfg.shift = fs;
        fcfg.per_region = 1u << (shift - fs);
        fcfg.nfine = static_cast<uint32_t>((total_words + (1ull << fs) - 1) >> fs);
        fcfg.cap = static_cast<uint32_t>(std::max<uint64_t>(64, (coarse_total * 3 / 2 / fcfg.nfine + 7) & ~7ull));
        // Large sparse-active tables (many slices, marks clustered on the
        // active sources' cells) overflow an average-sized fine bin; give
        // each slice room for 1024 marks while that stays within 4 GB.
        if (!small && fcfg.cap < 1024 && uint64_t(fcfg.nfine) * 1024 * 2 <= (4ull << 30)) fcfg.cap = 1024;
        if (uint64_t(fcfg.cap) * fcfg.nfine >= (1ull << 32)) throw Error(SRLA_E_INTERNAL, "fine bin index overflow");
        fine_bins.ensure(uint64_t(fcfg.nfine) * fcfg.cap);
        fine_count.ensure(fcfg.nfine);
        fcfg.bins = fine_bins.p;
        fcfg.count = fine_count.p;
        d_streamed.ensure(1);
        pin_streamed.ensure(1);
        pin_streamed.p[0] = 0;
        CK(cudaMemsetAsync(d_streamed.p, 0, sizeof(unsigned long long), st));
        fcfg.streamed = d_streamed.p;
        CK(cudaMemsetAsync(fine_count.p, 0, fine_count.cap * sizeof(uint32_t), st));
        const int smem = static_cast<int>(lin_bytes(1ull << fs));
        // 1024-thread split blocks (16384-entry tiles) for wide fan-outs: twice the
        // entries per fine slice per tile, half the bin reservations (C3: 2048 slices per region)
        split_threads = fcfg.per_region >= 1024 ? 1024u : 512u;
        if (const char* v = std::getenv("SRLA_SPLIT_THREADS")) split_threads = std::atoi(v) == 1024 ? 1024u : 512u;
        split_smem = 2 * uint64_t(split_threads) * kSplitPerThread * 4 + fcfg.per_region * 16;  // two tile stages + per-slice tables
        with_w([&](auto w) {
            using W = decltype(w);
            raise_smem_cap(k_split<W, 512>, static_cast<int>(split_smem));
            raise_smem_cap(k_split<W, 1024>, static_cast<int>(split_smem));
            raise_smem_cap(k_slice_apply<W>, std::max(smem, 16));
            raise_smem_cap(k_slice_apply_bulk<W>, std::max(2 * smem, 32));
        });
        if (const char* v = std::getenv("SRLA_STAMP_SPARSE")) stamp_sparse_max = static_cast<uint32_t>(std::atoi(v));
        raise_smem_cap(k_stamp_warp, static_cast<int>(stamp_claim_bytes(fs)));
        if (nib) {
            if (nib_apply_smem() > 200 * 1024) return false;  // two stages must fit in shared memory
            raise_smem_cap(k_slice_apply_nib, static_cast<int>(nib_apply_smem()));
        }
        with_w([&](auto w) {
            using W = decltype(w);
            raise_smem_cap(k_scan_bin<W, 4>, bin_smem(bcfg.nregions));
            raise_smem_cap(k_scan_bin<W, 0>, bin_smem(bcfg.nregions));
        });
        // bulk (TMA) slices need 16-byte slices and rows at least one slice long
        const uint64_t slice_words = 1ull << fs;
        bulk_ok = lin_bytes(slice_words) % 16 == 0 && lin_bytes(lin_words) % 16 == 0 && lin_words >= slice_words;
        bulk_end = lin_bytes(total_words % slice_words) % 16 == 0 ? fcfg.nfine : fcfg.nfine - 1;
        if (total_words % slice_words) bulk_end = fcfg.nfine - 1;  // partial last slice: plain kernel
        bcfg.nib = fcfg.nib = nib ? 1u : 0u;
        use_bins = true;
        return true;
    }

    // Epoch stamps replace the O(table) slide by O(1) + a 1/(255-expired)
    // sweep, at the price of a CAS per mark. Chosen for tables of 16 GiB and
    // more (the 2^24-column sketch), or by srla_config.flags / SRLA_EPOCH.
    void setup_epoch() {
        if (!epoch_wanted() || nib || !use_bins || wb != 1 || dc.expired > 127) return;
        if (lin_words < (1ull << fcfg.shift)) return;  // a slice may span at most two rows
        epoch = true;
        cur_epoch = 0;
        hist.ensure(uint64_t(cfg.rows) * 256);
        pin_hist.ensure(uint64_t(cfg.rows) * 256);
        CK(cudaMemsetAsync(hist.p, 0, uint64_t(cfg.rows) * 256 * sizeof(unsigned long long), st));
        const uint64_t words = uint64_t(cfg.rows) * lin_words;
        k_fill<uint8_t><<<blocks(words, 256, 16), 256, 0, st>>>(static_cast<uint8_t*>(d_lin), words,
                                                                static_cast<uint8_t>((256 - dc.expired) & 0xFF));
        check_launch();
        launched();
        raise_smem_cap(k_slice_stamp, std::max<int>(32, int(2u << fcfg.shift)));
    }

    // Unpack a nibble table to a byte per recorder (an import carried values
    // above 15); the bin geometry is rebuilt for the byte layout.
    void leave_nibble() {
        if (!nib) return;
        flush_linear();
        const uint64_t words = uint64_t(cfg.rows) * lin_words;
        void* wide = nullptr;
        CK(cudaMalloc(&wide, words));
        k_unpack_nib<<<blocks(words / 2, 256, 16), 256, 0, st>>>(static_cast<const uint8_t*>(d_lin), words / 2,
                                                                 static_cast<uint8_t*>(wide));
        check_launch();
        launched();
        CK(cudaStreamSynchronize(st));
        CK(cudaFree(d_lin));
        d_lin = wide;
        nib = false;
        if (!setup_bins_geometry()) use_bins = false;
        CK(cudaStreamSynchronize(st));
    }

    // Literal recorder value of a stamp (recorders.hpp:84-87 applied cur - s times).
    uint32_t stamp_value(uint32_t s) const {
        const uint32_t a = (cur_epoch - s) & 0xFFu;
        return a < dc.expired ? a : dc.expired;
    }

    // Convert the table back to literal recorders (an import carried values
    // outside [0, expired], which stamps cannot hold).
    void leave_epoch() {
        if (!epoch) return;
        flush_linear();
        const uint64_t words = uint64_t(cfg.rows) * lin_words;
        k_epoch_to_literal<<<blocks(words / 16 + 1, 256, 16), 256, 0, st>>>(static_cast<uint8_t*>(d_lin), words, cur_epoch,
                                                                           dc.expired);
        check_launch();
        launched();
        epoch = false;
    }

    // counts_active per row from the stamp histograms (already on the host)
    void counts_from_hist(uint64_t* counts) const { counts_from_hist(counts, cur_epoch); }
    void counts_from_hist(uint64_t* counts, uint32_t ep) const {
        for (uint32_t i = 0; i < cfg.rows; ++i) {
            uint64_t s = 0;
            for (uint32_t j = 0; j < cfg.window; ++j) s += pin_hist.p[uint64_t(i) * 256 + ((ep - j) & 0xFFu)];
            counts[i] = s;
        }
    }

    // Age (and optionally count) linear words [w0, w1) — split at row
    // boundaries so each piece counts into its own row (non-binned tables).
    template <typename W>
    void count_age_range(uint64_t w0, uint64_t w1, bool count) {
        while (w0 < w1) {
            const uint64_t row = w0 / lin_words;
            const uint64_t end = std::min(w1, (row + 1) * lin_words);
            k_count_age<W><<<blocks((end - w0) * sizeof(W) / 16 + 1, 256, 8), 256, 0, st>>>(
                static_cast<W*>(d_lin) + w0, end - w0, cfg.window, dc.expired, count ? 1 : 0, d_counts.p + row);
            check_launch();
            launched();
            w0 = end;
        }
    }

    // Apply pending linear marks. mode 0: apply only (slices without marks
    // untouched); 1: apply + age the whole table; 2: apply + count active per
    // row into d_counts (pre-age) + age. One streaming pass over the table.
    // Split the region bins into the fine bins on stream `s` (the region bins
    // and their counts are free again when ev_split_done fires).
    void split_now(cudaStream_t s) {
        if (!pending_entries) return;
        const uint32_t R = bcfg.nregions;
        // the tile table is built on the device (k_split_prefix): no host round trip
        if (s != st) {
            CK(cudaEventRecord(ev_k1_done, st));
            CK(cudaStreamWaitEvent(s, ev_k1_done, 0));
        }
        if (split_in_flight) CK(cudaStreamWaitEvent(s, ev_split_done, 0));  // tile_prefix reuse
        split_in_flight = false;
        const uint32_t tile = split_threads * kSplitPerThread;
        k_split_prefix<<<1, 1024, 0, s>>>(bin_count.p, R, bcfg.cap, tile, tile_prefix.p);
        check_launch();
        launched();
        const cudaEvent_t t0 = timer_start(s);
        with_w([&](auto w) {
            using W = decltype(w);
            // an early split leaves room for the ordering phase's kernels
            static const uint32_t waves = [] { const char* v = std::getenv("SRLA_SPLIT_WAVES"); return v ? static_cast<uint32_t>(std::atoi(v)) : 16u; }();
            const uint64_t max_tiles = pending_entries / tile + R;
            const uint32_t grid = static_cast<uint32_t>(std::min<uint64_t>(max_tiles, sms * (s == st ? 8u : waves)));
            if (split_threads == 1024)
                k_split<W, 1024><<<grid, 1024, split_smem, s>>>(bins.p, bcfg.cap, tile_prefix.p, tile_prefix.p + R + 1, R,
                                                                bcfg.region_shift, fcfg, ecfg(), static_cast<W*>(d_lin));
            else
                k_split<W, 512><<<grid, 512, split_smem, s>>>(bins.p, bcfg.cap, tile_prefix.p, tile_prefix.p + R + 1, R,
                                                              bcfg.region_shift, fcfg, ecfg(), static_cast<W*>(d_lin));
        });
        check_launch();
        launched();
        timer_stop(t0, kTimeSplit, s);
        timing.split_kernel_launches += 1;
        timing.split_entries += pending_entries;
        CK(cudaMemsetAsync(bin_count.p, 0, R * sizeof(uint32_t), s));
        if (s != st) {
            CK(cudaEventRecord(ev_split_done, s));
            split_in_flight = true;
        }
        fine_pending += pending_entries;
        pending_entries = 0;
    }
    // the engine stream waits for an early split (device-side)
    void join_split() {
        if (!split_in_flight) return;
        CK(cudaStreamWaitEvent(st, ev_split_done, 0));
        split_in_flight = false;
    }

    void flush_linear(int mode = 0) {
        if (!use_bins) return;
        join_maint_lin();
        split_now(st);
        join_split();
        if (fine_pending == 0 && mode == 0) return;
        const uint64_t total = uint64_t(cfg.rows) * lin_words;
        open_k1_gate();
        const cudaEvent_t t_apply = timer_start();
        timing.apply_entries += fine_pending;
        if (epoch) {
            if (fine_pending) {
                // sparse slices warp by warp in place, dense ones through shared memory
                const uint32_t sparse_max = stamp_sparse_max;
                const uint32_t sp = cfg.rows <= kStampWarpRows && lin_words % 4 == 0 ? sparse_max : 0u;
                if (sp) {
                    // 5 blocks fit an SM; 40 per SM make the warp-strided slice assignment
                    // finer (C3: 3.28 vs 3.35 ms with 5; profiles/r02/ab_region_waves.txt)
                    static const uint32_t stamp_per_sm = [] { const char* v = std::getenv("SRLA_STAMP_BLOCKS"); return v ? static_cast<uint32_t>(std::atoi(v)) : 40u; }();
                    k_stamp_warp<<<sms * stamp_per_sm, 256, stamp_claim_bytes(fcfg.shift), st>>>(static_cast<uint8_t*>(d_lin), lin_words, fcfg, sp, cur_epoch,
                                                         cfg.window, cfg.rows, hist.p);
                    check_launch();
                    launched();
                }
                k_slice_stamp<<<std::min<uint32_t>(fcfg.nfine, sms * 3), 256, 2u << fcfg.shift, st>>>(
                    static_cast<uint8_t*>(d_lin), total, lin_words, fcfg, 0, bulk_ok ? 1 : 0, cur_epoch, cfg.window, hist.p,
                    sp);
                check_launch();
                launched();
                timer_stop(t_apply, kTimeApply);
                timing.apply_kernel_launches += 1;
                CK(cudaMemcpyAsync(pin_streamed.p, d_streamed.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
                CK(cudaMemsetAsync(fine_count.p, 0, fcfg.nfine * sizeof(uint32_t), st));
            } else {
                ev_pool.push_back(t_apply);
            }
            fine_pending = 0;
            return;
        }
        if (nib) {
            // 512 threads per slice block: 1.09 vs 1.12 ms (256) and 1.27 ms (1024) per C2 slice.
            // Two blocks fit an SM (112 KB of stages); the grid is 16 per SM so the
            // strided slice assignment balances: 1.00 ms vs 1.09 ms with 3 per SM
            // (2: 1.07, 4: 1.03, 8: 1.01, 24: 1.00; profiles/r02/ab_region_waves.txt)
            static const uint32_t apply_threads = [] { const char* v = std::getenv("SRLA_APPLY_THREADS"); return v ? static_cast<uint32_t>(std::atoi(v)) : 512u; }();
            static const uint32_t apply_per_sm = [] { const char* v = std::getenv("SRLA_APPLY_BLOCKS"); return v ? static_cast<uint32_t>(std::atoi(v)) : 16u; }();
            k_slice_apply_nib<<<std::min<uint32_t>(fcfg.nfine, sms * apply_per_sm), apply_threads, nib_apply_smem(), st>>>(
                static_cast<uint8_t*>(d_lin), lin_words, fcfg, fcfg.nfine, mode, cfg.window, dc.expired, d_counts.p);
            check_launch();
            launched();
        } else with_w([&](auto w) {
            using W = decltype(w);
            const size_t smem = (1ull << fcfg.shift) * sizeof(W);
            uint32_t begin = 0;
            if (bulk_ok && bulk_end) {
                k_slice_apply_bulk<W><<<std::min<uint32_t>(bulk_end, sms * 3), 256, 2 * smem, st>>>(
                    static_cast<W*>(d_lin), lin_words, fcfg, bulk_end, mode, cfg.window, dc.expired, d_counts.p);
                check_launch();
                launched();
                begin = bulk_end;
            }
            if (begin < fcfg.nfine) {
                k_slice_apply<W><<<std::min<uint32_t>(fcfg.nfine - begin, sms * 3), 256, smem, st>>>(
                    static_cast<W*>(d_lin), total, lin_words, fcfg, begin, mode, cfg.window, dc.expired, d_counts.p);
                check_launch();
                launched();
            }
        });
        timer_stop(t_apply, kTimeApply);
        timing.apply_kernel_launches += 1;
        CK(cudaMemcpyAsync(pin_streamed.p, d_streamed.p, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaMemsetAsync(fine_count.p, 0, fcfg.nfine * sizeof(uint32_t), st));
        fine_pending = 0;
    }

    // ------------------------------------------------------------ scan
    void open_k1_gate_final() {  // end-of-slice over without a split: gate on its end
        if (k1_gate.load(std::memory_order_relaxed)) return;
        cudaEventRecord(ev_k1_gate, st);
        k1_gate.store(true, std::memory_order_release);
    }
    void open_k1_gate() {
        if (!in_async_eos || k1_gate.load(std::memory_order_relaxed)) return;
        CK(cudaEventRecord(ev_k1_gate, st));
        k1_gate.store(true, std::memory_order_release);
    }

    // current <-> alternate region-bin set
    void swap_bin_sets() {
        std::swap(bins.p, bins_alt.p);
        std::swap(bins.cap, bins_alt.cap);
        std::swap(bin_count.p, bin_count_alt.p);
        std::swap(bin_count.cap, bin_count_alt.cap);
        bcfg.bins = bins.p;
        bcfg.count = bin_count.p;
    }

    // K1 of the first chunk of a slice while the previous slice's
    // end-of-slice runs on its worker thread: bins into the alternate set on
    // stream sk (never marking the table directly), then joins the
    // end-of-slice and makes that set current. Returns false (after joining)
    // when the chunk has to be scanned the ordinary way.
    template <typename W>
    bool scan_k1_overlapped(const uint32_t* d_recs, uint32_t n, int vec, uint32_t& n_ev) {
        BinCfg b2 = bcfg;
        b2.bins = bins_alt.p;
        b2.count = bin_count_alt.p;
        b2.no_direct = 1;
        b2.overflow = ctr_k1.p + 1;
        const uint64_t add = uint64_t(n) * cfg.rows;
        if (add / bcfg.nregions * 13 / 10 + 8192 > bcfg.cap) {
            join_eos();
            return false;
        }
        // the alternate set was zeroed, and the stamps reset, before the last scan ended
        CK(cudaStreamWaitEvent(sk, ev_scan_done, 0));
        if (!std::getenv("SRLA_K1_EARLY")) {
            while (!k1_gate.load(std::memory_order_acquire)) std::this_thread::yield();
            CK(cudaStreamWaitEvent(sk, ev_k1_gate, 0));
        }
        CK(cudaMemsetAsync(ctr_k1.p, 0, 4 * sizeof(uint32_t), sk));
        CK(cudaEventRecord(t_scan0, sk));
        const uint32_t tiles = (n + kBinTile - 1) / kBinTile;
        if (cfg.rows == 4)
            k_scan_bin<W, 4><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), sk>>>(
                d_recs, n, dc, b2, EpochCfg{0u, 0u, nullptr, 0ull}, static_cast<W*>(d_lin), d_stamp, ev.p, ev_cap, ctr_k1.p, vec);
        else
            k_scan_bin<W, 0><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), sk>>>(
                d_recs, n, dc, b2, EpochCfg{0u, 0u, nullptr, 0ull}, static_cast<W*>(d_lin), d_stamp, ev.p, ev_cap, ctr_k1.p, vec);
        CK(cudaGetLastError());
        CK(cudaEventRecord(t_scan1, sk));
        CK(cudaMemcpyAsync(pin_k1.p, ctr_k1.p, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost, sk));
        join_eos();  // the end-of-slice has flushed (and zeroed) the current set
        CK(cudaStreamSynchronize(sk));
        launched();
        swap_bin_sets();
        pending_entries = add;
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, t_scan0, t_scan1));
        timing.scan_kernel_ms += ms;
        timing.scan_kernel_launches += 1;
        timing.scan_kernel_records += n;
        n_ev = pin_k1.p[0];
        if (pin_k1.p[1] || n_ev > ev_cap) {  // a bin or the event list overflowed: drop and rescan
            CK(cudaMemsetAsync(bin_count.p, 0, bcfg.nregions * sizeof(uint32_t), st));
            pending_entries = 0;
            return false;
        }
        CK(cudaMemsetAsync(ctr.p, 0, 16 * sizeof(uint32_t), st));
        ++stats.overlapped_chunks;
        return true;
    }

    // The sorted, ordered resolution from the chunk's X crossing keys
    // (xkeys): K3 first crossings, K4 indicator resolution, sink pushes,
    // candidate append (kernels.cuh).
    void order_tail(uint32_t X) {
        // K3: first crossing per host, then order hosts by P
        xsorted.ensure(X);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, xkeys.p, xsorted.p, static_cast<int>(X), 0, 64, st);
        });
        hp.ensure(X);
        k_first<<<blocks(X), 256, 0, st>>>(xsorted.p, X, hp.p, ctr.p + 2);
        check_launch();
        launched();
        const uint32_t Hn = read_ctr(2);
        trace("scan: sort+first");
        stats.first_crossings += Hn;
        hps.ensure(Hn);
        cub_call([&](void* t, size_t& b) {
            // by P alone (bits 32..): P (< kChunk) is distinct per host
            return cub::DeviceRadixSort::SortKeys(t, b, hp.p, hps.p, static_cast<int>(Hn), 32, 32 + bit_length(kChunk - 1), st);
        });

        // K4: ordered indicator resolution
        fmask.ensure(Hn);
        cnt.ensure(Hn);
        off.ensure(Hn);
        hosts.ensure(Hn);
        status.ensure(Hn);
        definite.ensure(Hn);
        fl_und.ensure(Hn);
        fl_ins.ensure(Hn);
        k_si_check<<<blocks(Hn), 256, 0, st>>>(hps.p, Hn, dc, d_si, fmask.p, cnt.p, hosts.p, status.p);
        check_launch();
        launched();
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceScan::ExclusiveSum(t, b, cnt.p, off.p, static_cast<int>(Hn), st);
        });
        CK(cudaMemcpyAsync(pin_ctr.p + 8, off.p + (Hn - 1), 4, cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(pin_ctr.p + 9, cnt.p + (Hn - 1), 4, cudaMemcpyDeviceToHost, st));
        sync_st();
        const uint32_t T = pin_ctr.p[8] + pin_ctr.p[9];
        CK(cudaMemsetAsync(definite.p, 0, Hn, st));
        if (T) {
            tkey.ensure(T);
            skey.ensure(T);
            tval.ensure(T);
            sval.ensure(T);
            towner.ensure(T);
            posof.ensure(T);
            k_tuples<<<blocks(Hn), 256, 0, st>>>(hosts.p, Hn, dc, fmask.p, off.p, tkey.p, tval.p, towner.p);
            check_launch();
            launched();
            const int end_bit = bit_length(uint64_t(cfg.rows) * cfg.cols * kIndicatorBits - 1);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceRadixSort::SortPairs(t, b, tkey.p, skey.p, tval.p, sval.p, static_cast<int>(T), 0, end_bit, st);
            });
            k_first_key<<<blocks(T), 256, 0, st>>>(skey.p, sval.p, T, towner.p, definite.p, posof.p);
            check_launch();
            launched();
        }
        k_classify<<<blocks(Hn), 256, 0, st>>>(Hn, status.p, definite.p, fl_und.p, fl_ins.p);
        check_launch();
        launched();
        flagged.ensure(Hn);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, thrust::counting_iterator<uint32_t>(0), fl_und.p, flagged.p,
                                              ctr.p + 3, static_cast<int>(Hn), st);
        });
        const uint32_t nf = read_ctr(3);
        trace("scan: K4 resolve");
        stats.flagged += nf;
        if (nf) {
            const cudaEvent_t ts = timer_start();
            k_serial<<<1, 32, 0, st>>>(flagged.p, nf, fmask.p, off.p, posof.p, skey.p, sval.p, towner.p, status.p, fl_ins.p);
            check_launch();
            launched();
            timer_stop(ts, kTimeSerial);
            timing.serial_kernel_launches += 1;
            timing.flagged_hosts += nf;
        }
        k_si_set<<<blocks(Hn), 256, 0, st>>>(hosts.p, Hn, status.p, dc, d_si);
        check_launch();
        launched();
        pushed.ensure(Hn);
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Flagged(t, b, hosts.p, fl_ins.p, pushed.p, ctr.p + 4, static_cast<int>(Hn), st);
        });
        const uint32_t np = read_ctr(4);
        stats.pushed += np;
        if (collect_pushed && np) {
            const size_t at = host_pushed.size();
            host_pushed.resize(at + np);
            pin_hosts.ensure(np);
            CK(cudaMemcpyAsync(pin_hosts.p, pushed.p, np * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            std::memcpy(host_pushed.data() + at, pin_hosts.p, np * sizeof(uint32_t));
        }
        trace("scan: K4 set+select");
        append_candidates(pushed.p, np);
        trace("scan: append");
    }

    // A few records: the reference's scan_ip_pair loop on one device thread
    // (k_scan_serial), one launch and one synchronisation per call.
    template <typename W, int MAXR>
    void scan_chunk_serial(const uint32_t* d_recs, uint32_t n) {
        join_maint();
        join_split();
        setup_order(std::max<uint32_t>(n, 1024));
        CK(cudaMemsetAsync(octr.p, 0, kOcCount * sizeof(uint32_t), st));
        k_scan_serial<W, MAXR><<<1, 32, 0, st>>>(d_recs, n, dc, static_cast<W*>(d_lin), nib ? 1 : 0, ecfg(),
                                                 static_cast<W*>(d_rough), d_si, cset.p, cset_cap - 1, pushlist.p,
                                                 newlist.p, octr.p);
        check_launch();
        launched();
        CK(cudaMemcpyAsync(pin_octr.p, octr.p, kOcCount * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
        sync_st();
        const uint32_t np = pin_octr.p[kOcPushList], nn = pin_octr.p[kOcNew];
        stats.sampled_events += pin_octr.p[kOcEvents];
        stats.pushed += np;
        if (collect_pushed && np) {
            const size_t at = host_pushed.size();
            host_pushed.resize(at + np);
            CK(cudaMemcpy(host_pushed.data() + at, pushlist.p, np * sizeof(uint32_t), cudaMemcpyDeviceToHost));
        }
        append_new(newlist.p, nn);
    }

    // One chunk with the ordering phase on device counts (order.cuh): K1, the
    // early split, K2h/K5, K4h, classify and the ordered compaction of new
    // candidates all queue back to back; the host synchronises once, reads
    // the counters and appends. Flagged hosts (rare) fall back to the sorted
    // resolution (order_tail) from the intact crossing keys and indicators.
    template <typename W, int MAXR>
    void scan_chunk_fast(const uint32_t* d_recs, uint32_t n) {
        W* lin = static_cast<W*>(d_lin);
        W* rough = static_cast<W*>(d_rough);
        const int vec = (reinterpret_cast<uintptr_t>(d_recs) & 15) == 0;
        if (!ev_cap) {
            ev_cap = static_cast<uint32_t>(std::min<uint64_t>(kChunk, (uint64_t(kChunk) >> tau) + (uint64_t(kChunk) >> (tau + 3)) + 65536));
            ev.ensure(3ull * ev_cap);
        }
        join_maint_lin();  // K1 may stamp the linear table directly (bin overflow)
        join_split();      // the region bins must have been split and zeroed
        uint32_t* pc = nullptr;
        while (true) {
            setup_order(ev_cap);
            CK(cudaMemsetAsync(octr.p, 0, kOcCount * sizeof(uint32_t), st));
            bcfg.seen_ovf = octr.p + kOcBinOvf;
            if (use_bins) {
                const uint64_t add = uint64_t(n) * cfg.rows;
                if ((pending_entries + add) / bcfg.nregions * 13 / 10 + 8192 > bcfg.cap) flush_linear();
            }
            CK(cudaEventRecord(t_scan0, st));
            uint32_t* evc = octr.p + kOcEvents;
            if (use_bins && MAXR <= kBinRows) {
                const uint32_t tiles = (n + kBinTile - 1) / kBinTile;
                if (cfg.rows == 4)
                    k_scan_bin<W, 4><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), st>>>(d_recs, n, dc, bcfg, ecfg(), lin, d_stamp, ev.p, ev_cap, evc, vec);
                else
                    k_scan_bin<W, 0><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), st>>>(d_recs, n, dc, bcfg, ecfg(), lin, d_stamp, ev.p, ev_cap, evc, vec);
            } else {
                k_scan<W, MAXR><<<blocks((n + 3) / 4, 256, 16), 256, 0, st>>>(d_recs, n, dc, lin, d_stamp, ev.p, ev_cap, evc, vec);
            }
            check_launch();
            launched();
            CK(cudaEventRecord(t_scan1, st));
            if (use_bins) pending_entries += uint64_t(n) * cfg.rows;
            timing.scan_kernel_launches += 1;
            timing.scan_kernel_records += n;
            // split the region bins now, concurrent with the ordering phase below
            if (use_bins && early_split && !overlap_on) split_now(ssplit);
            const auto w_order = std::chrono::steady_clock::now();
            join_maint();  // rough aging, indicators and the candidate hash of the last slide
            const OrderBufs ob = order_bufs(collect_pushed);
            const uint32_t g = blocks(ev_cap, 256, 4);
            k_cross_ht<W, MAXR><<<g, 256, 0, st>>>(ev.p, ev_cap, dc, rough, d_stamp, xkeys.p, ob);
            k_commit_dev<W, MAXR><<<g, 256, 0, st>>>(ev.p, ev_cap, dc, rough, d_stamp, ob);
            k_si_open<<<g, 256, 0, st>>>(dc, d_si, ob);
            k_order_classify<<<g, 256, 0, st>>>(dc, cset.p, cset_cap - 1, ob);
            const cudaEvent_t tf = timer_start();
            k_resolve_flagged<<<1, 1024, 0, st>>>(dc, cset.p, cset_cap - 1, ob);
            timer_stop(tf, kTimeSerial);
            check_launch();
            launched(5);
            emit_bitmap(bm_new.p, n, d_recs, newlist.p, kOcNew);
            if (collect_pushed) emit_bitmap(bm_push.p, n, d_recs, pushlist.p, kOcPushList);
            CK(cudaMemcpyAsync(pin_octr.p, octr.p, kOcCount * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
            sync_st();  // the chunk's one host synchronisation
            pc = pin_octr.p;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, t_scan0, t_scan1));
            timing.scan_kernel_ms += ms;
            timing.order_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w_order).count();
            if (pc[kOcBinOvf] && dedup_mode < 0 && bcfg.pack) bcfg.dedup = 1;
            if (pc[kOcEvents] <= ev_cap) break;
            // event overflow: the ordering kernels did nothing; marks and rough
            // stamps are idempotent, so K1 reruns with room
            ev_cap = static_cast<uint32_t>(std::min<uint64_t>(uint64_t(pc[kOcEvents]) * 5 / 4 + 4096, 0xFFFFFFF0ull));
            ev.ensure(3ull * ev_cap);
        }
        const uint32_t n_ev = pc[kOcEvents], X = pc[kOcCross], Hn = pc[kOcHosts], nf = pc[kOcFlagged];
        const uint32_t np = pc[kOcPushed], nn = pc[kOcNew], Tn = pc[kOcTuples];
        stats.sampled_events += n_ev;
        stats.crossings += X;
        const OrderBufs ob = order_bufs(false);
        if (pc[kOcFallback]) {  // many flagged hosts: the sorted path from the crossing keys
            const auto w = std::chrono::steady_clock::now();
            CK(cudaMemsetAsync(ctr.p, 0, 16 * sizeof(uint32_t), st));
            order_tail(X);
            timing.order_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w).count();
        } else {
            stats.first_crossings += Hn;
            stats.flagged += nf;
            timing.serial_kernel_launches += 1;
            timing.flagged_hosts += nf;
            stats.pushed += np;
            if (Hn) {
                k_order_si_set<<<blocks(Hn), 256, 0, st>>>(dc, d_si, ob, Hn);
                check_launch();
                launched();
            }
            if (collect_pushed && pc[kOcPushList]) {
                const uint32_t m = pc[kOcPushList];
                const size_t at = host_pushed.size();
                host_pushed.resize(at + m);
                pin_hosts.ensure(m);
                CK(cudaMemcpyAsync(pin_hosts.p, pushlist.p, m * sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                std::memcpy(host_pushed.data() + at, pin_hosts.p, m * sizeof(uint32_t));
            }
            append_new(newlist.p, nn);
        }
        if (Hn || Tn) {
            k_order_clear<<<blocks(std::max(Hn, Tn)), 256, 0, st>>>(ob, Hn, Tn);
            check_launch();
            launched();
        }
        trace("scan: fast order");
    }

    template <typename W, int MAXR>
    void scan_chunk_t(const uint32_t* d_recs, uint32_t n, bool overlap) {
        W* lin = static_cast<W*>(d_lin);
        W* rough = static_cast<W*>(d_rough);
        const int vec = (reinterpret_cast<uintptr_t>(d_recs) & 15) == 0;
        if (!ev_cap) {
            ev_cap = static_cast<uint32_t>(std::min<uint64_t>(kChunk, (uint64_t(kChunk) >> tau) + (uint64_t(kChunk) >> (tau + 3)) + 65536));
            ev.ensure(3ull * ev_cap);
            // the ordering scratch is bounded by the sampled events of a chunk:
            // size it once instead of creeping up (each regrowth is a cudaFree,
            // a device-wide synchronisation)
            const size_t m = std::min<size_t>(ev_cap, size_t(1) << 21);
            xkeys.ensure(m); xsorted.ensure(m); hp.ensure(m); hps.ensure(m); fmask.ensure(m);
            cnt.ensure(m); off.ensure(m); hosts.ensure(m); status.ensure(m); definite.ensure(m);
            fl_und.ensure(m); fl_ins.ensure(m); flagged.ensure(m); pushed.ensure(m); newhosts.ensure(m);
            isnew.ensure(m);
            const size_t t = m * std::min<uint32_t>(cfg.rows, 8);
            tkey.ensure(t); skey.ensure(t); tval.ensure(t); sval.ensure(t); towner.ensure(t); posof.ensure(t);
        }
        uint32_t n_ev = 0;
        bool k1_done = false;
        if (overlap) {
            if (use_bins && MAXR <= kBinRows && bins_alt.p) k1_done = scan_k1_overlapped<W>(d_recs, n, vec, n_ev);
            else join_eos();
        }
        join_maint_lin();  // K1 may stamp the linear table directly (bin overflow)
        join_split();      // the region bins must have been split and zeroed
        while (!k1_done) {
            CK(cudaMemsetAsync(ctr.p, 0, 16 * sizeof(uint32_t), st));
            if (use_bins) {
                const uint64_t add = uint64_t(n) * cfg.rows;
                if ((pending_entries + add) / bcfg.nregions * 13 / 10 + 8192 > bcfg.cap) flush_linear();
            }
            CK(cudaEventRecord(t_scan0, st));
            if (use_bins && MAXR <= kBinRows) {
                const uint32_t tiles = (n + kBinTile - 1) / kBinTile;
                if (cfg.rows == 4)
                    k_scan_bin<W, 4><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), st>>>(d_recs, n, dc, bcfg, ecfg(), lin, d_stamp, ev.p, ev_cap, ctr.p, vec);
                else
                    k_scan_bin<W, 0><<<std::min<uint32_t>(tiles, sms * 2), kBinThreads, bin_smem(bcfg.nregions, bcfg.dedup), st>>>(d_recs, n, dc, bcfg, ecfg(), lin, d_stamp, ev.p, ev_cap, ctr.p, vec);
            } else {
                k_scan<W, MAXR><<<blocks((n + 3) / 4, 256, 16), 256, 0, st>>>(d_recs, n, dc, lin, d_stamp, ev.p, ev_cap, ctr.p, vec);
            }
            check_launch();
            launched();
            CK(cudaEventRecord(t_scan1, st));
            n_ev = read_ctr(0);
            if (use_bins) pending_entries += uint64_t(n) * cfg.rows;
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, t_scan0, t_scan1));
            timing.scan_kernel_ms += ms;
            timing.scan_kernel_launches += 1;
            timing.scan_kernel_records += n;
            if (n_ev <= ev_cap) break;
            // capacity overflow: marks and stamps are idempotent, rerun with room
            ev_cap = static_cast<uint32_t>(std::min<uint64_t>(uint64_t(n_ev) * 5 / 4 + 4096, 0xFFFFFFF0ull));
            ev.ensure(3ull * ev_cap);
        }
        stats.sampled_events += n_ev;
        // split the region bins now, concurrent with the ordering phase below
        if (use_bins && early_split && !overlap_on) split_now(ssplit);
        trace("scan: K1");
        if (!n_ev) return;
        const auto w_order = std::chrono::steady_clock::now();
        struct OrderTimer {
            srla_timing& t;
            std::chrono::steady_clock::time_point t0;
            ~OrderTimer() { t.order_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
        } order_timer{timing, w_order};

        join_maint();  // rough aging, indicators and the candidate hash of the last slide
        xkeys.ensure(n_ev);
        k_cross<W, MAXR><<<blocks(n_ev), 256, 0, st>>>(ev.p, ev_cap, n_ev, dc, rough, d_stamp, xkeys.p, ctr.p + 1);
        check_launch();
        launched();
        k_commit<W, MAXR><<<blocks(n_ev), 256, 0, st>>>(ev.p, ev_cap, n_ev, dc, rough, d_stamp);
        check_launch();
        launched();
        const uint32_t X = read_ctr(1);
        trace("scan: K2+K5");
        stats.crossings += X;
        if (!X) return;

        order_tail(X);
    }

    void scan_chunk(const uint32_t* d_recs, uint32_t n, bool overlap = false) {
        if (!n) {
            if (overlap) join_eos();
            return;
        }
        trace(nullptr);
        stats.chunks++;
        stats.packets += n;
        with_w([&](auto w) {
            using W = decltype(w);
            static const uint32_t serial_max = [] { const char* v = std::getenv("SRLA_SERIAL_MAX"); return v ? static_cast<uint32_t>(std::atoi(v)) : 64u; }();
            if (n <= serial_max && !overlap && cfg.rows <= 8) {
                if (cfg.rows <= 4) scan_chunk_serial<W, 4>(d_recs, n);
                else scan_chunk_serial<W, 8>(d_recs, n);
            } else if (fast_order && !overlap && cfg.rows <= kOrderRows) {
                if (cfg.rows <= 4) scan_chunk_fast<W, 4>(d_recs, n);
                else scan_chunk_fast<W, 8>(d_recs, n);
            } else if (cfg.rows <= 4) {
                scan_chunk_t<W, 4>(d_recs, n, overlap);
            } else {
                scan_chunk_t<W, 64>(d_recs, n, overlap);
            }
        });
    }

    // SRLA_TRACE=1: synchronise and print per-phase wall times (diagnostics only)
    bool tracing = [] { const char* t = std::getenv("SRLA_TRACE"); return t && t[0] == '1'; }();
    std::chrono::steady_clock::time_point trace_t0{};
    void trace(const char* what) {
        if (!tracing) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        if (what) std::fprintf(stderr, "[srla] %-28s %8.3f ms\n", what, std::chrono::duration<double, std::milli>(now - trace_t0).count());
        trace_t0 = now;
    }

    // SRLA_EOS_TRACE=1: device-event marks on the engine stream through the
    // end-of-slice, printed after it (no extra synchronisation)
    bool eos_tracing = [] { const char* t = std::getenv("SRLA_EOS_TRACE"); return t && t[0] == '1'; }();
    std::vector<std::pair<const char*, cudaEvent_t>> eos_marks;
    std::vector<std::pair<const char*, double>> eos_host_marks;
    std::chrono::steady_clock::time_point eos_host_t0{};
    void eos_mark(const char* what) {
        if (!eos_tracing) return;
        cudaEvent_t e = take_event();
        CK(cudaEventRecord(e, st));
        eos_marks.push_back({what, e});
        eos_host_marks.push_back({what, std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - eos_host_t0).count()});
    }
    void eos_dump() {
        if (!eos_tracing || eos_marks.empty()) return;
        std::string line = "[srla eos] n=" + std::to_string(ncsip) + " sorted_new=" + std::to_string(last_sort_new);
        for (size_t i = 1; i < eos_marks.size(); ++i) {
            float ms = 0.f;
            CK(cudaEventSynchronize(eos_marks[i].second));
            CK(cudaEventElapsedTime(&ms, eos_marks[i - 1].second, eos_marks[i].second));
            char b[128];
            std::snprintf(b, sizeof b, " %s %.3f(h%.3f)", eos_marks[i].first, ms, eos_host_marks[i].second);
            line += b;
        }
        std::fprintf(stderr, "%s\n", line.c_str());
        for (auto& m : eos_marks) ev_pool.push_back(m.second);
        eos_marks.clear();
        eos_host_marks.clear();
    }

    void join_eos() {
        if (eos_thread.joinable()) eos_thread.join();
    }

    // Run end_slice on a worker thread; the caller's next scan_batch stages its
    // host->device copies meanwhile. `out` must stay valid until the wait.
    void end_slice_async(uint64_t slice_id, bool want_report, srla_entry* out, uint64_t cap) {
        join_eos();
        if (eos.pending) throw Error(SRLA_E_INVALID, "previous srla_end_slice_async not collected");
        const bool due = want_report && slice_id + 1 >= cfg.window;
        if (due && (ncsip > cap || (!out && ncsip)))
            throw Error(SRLA_E_CAPACITY, "report buffer holds " + std::to_string(cap) + " entries, " +
                                             std::to_string(ncsip) + " needed");
        eos = EosResult{};
        eos.pending = true;
        eos.n = due ? ncsip : 0;
        k1_gate.store(false);
        eos_thread = std::thread([this, slice_id, want_report, out] {
            try {
                CK(cudaSetDevice(device));
                in_async_eos = true;
                timed_end_slice(slice_id, want_report, out);
                in_async_eos = false;
                open_k1_gate_final();
                eos.nret = ncsip;
            } catch (const Error& x) {
                eos.code = x.code;
                eos.msg = x.what();
                open_k1_gate_final();
            } catch (const std::exception& x) {
                eos.code = SRLA_E_INTERNAL;
                eos.msg = x.what();
                open_k1_gate_final();
            }
        });
    }

    void timed_end_slice(uint64_t slice_id, bool want_report, srla_entry* out, const Compact* compact = nullptr) {
        const auto w0 = std::chrono::steady_clock::now();
        CK(cudaEventRecord(t_eos0, st));
        end_slice(slice_id, want_report, out, compact);
        CK(cudaEventRecord(t_eos1, st));
        CK(cudaEventSynchronize(t_eos1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, t_eos0, t_eos1));
        timing.end_slice_device_ms += ms;
        timing.last_end_slice_device_ms = ms;
        timing.last_end_slice_wall_ms =
            std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
        timing.end_slice_wall_ms += timing.last_end_slice_wall_ms;
        timing.end_slices += 1;
    }

    // Device records are read on the engine's non-blocking streams: first
    // wait (device-side) for the work the producer stream has queued.
    cudaEvent_t ev_input = nullptr;
    void wait_producer(cudaStream_t producer) {
        if (!ev_input) CK(cudaEventCreateWithFlags(&ev_input, cudaEventDisableTiming));
        CK(cudaEventRecord(ev_input, producer));
        CK(cudaStreamWaitEvent(st, ev_input, 0));
        CK(cudaStreamWaitEvent(sk, ev_input, 0));
    }

    void scan_batch(const srla_record* recs, uint64_t n, int on_device, cudaStream_t producer = cudaStreamLegacy) {
        if (!n) {
            join_eos();
            return;
        }
        if (on_device) {
            cudaPointerAttributes pa{};
            if (cudaPointerGetAttributes(&pa, recs) != cudaSuccess || pa.type != cudaMemoryTypeDevice ||
                pa.device != device) {
                cudaGetLastError();
                throw Error(SRLA_E_INVALID, "on_device records must be device memory on the engine's GPU");
            }
            wait_producer(producer);
            // a pending asynchronous end-of-slice overlaps this batch's first K1
            const bool overlap = overlap_on && eos_thread.joinable() && ev_cap != 0;
            if (!overlap) join_eos();
            const uint32_t* base = reinterpret_cast<const uint32_t*>(recs);
            for (uint64_t o = 0; o < n; o += kChunk)
                scan_chunk(base + 3 * o, static_cast<uint32_t>(std::min<uint64_t>(kChunk, n - o)), overlap && o == 0);
        } else {
            scan_host(reinterpret_cast<const uint32_t*>(recs), n);
        }
        // epoch stamps: apply this batch's marks now, so end-of-slice only
        // reads histograms and the candidates' cells
        if (epoch) flush_linear();
        CK(cudaEventRecord(ev_scan_done, st));
    }

    // Host records: double-buffered H2D on a copy stream overlapping the scan
    // of the previous chunk. Pinned caller memory is DMA'd directly; pageable
    // memory is bounced through pinned staging.
    void scan_host(const uint32_t* src, uint64_t n) {
        cudaPointerAttributes attr{};
        bool pinned = cudaPointerGetAttributes(&attr, src) == cudaSuccess && attr.type == cudaMemoryTypeHost;
        cudaGetLastError();
        const uint32_t step = static_cast<uint32_t>(std::min<uint64_t>(kHostStage, n));
        const uint64_t nchunks = (n + step - 1) / step;
        for (int b = 0; b < 2; ++b) {
            dstage[b].ensure(3ull * step);
            if (!pinned) pstage[b].ensure(3ull * step);
        }
        auto len = [&](uint64_t j) { return static_cast<uint32_t>(std::min<uint64_t>(step, n - j * step)); };
        auto issue = [&](uint64_t j) {
            const int b = static_cast<int>(j & 1);
            const uint32_t* from = src + 3ull * j * step;
            if (!pinned) {
                CK(cudaEventSynchronize(ev_copied[b]));
                std::memcpy(pstage[b].p, from, 12ull * len(j));
                from = pstage[b].p;
            }
            CK(cudaStreamWaitEvent(cs, ev_scanned[b], 0));
            CK(cudaMemcpyAsync(dstage[b].p, from, 12ull * len(j), cudaMemcpyHostToDevice, cs));
            CK(cudaEventRecord(ev_copied[b], cs));
        };
        issue(0);
        if (nchunks > 1) issue(1);
        join_eos();  // copies above overlap a pending asynchronous end-of-slice
        for (uint64_t j = 0; j < nchunks; ++j) {
            if (j >= 1 && j + 1 < nchunks) issue(j + 1);
            const int b = static_cast<int>(j & 1);
            CK(cudaStreamWaitEvent(st, ev_copied[b], 0));
            scan_chunk(dstage[b].p, len(j));
            CK(cudaEventRecord(ev_scanned[b], st));
        }
    }

    // ------------------------------------------------------------ report
    template <typename W, int MAXR>
    void union_linear_t(const uint32_t* d_hosts, uint32_t n, uint32_t* d_out, uint32_t kthr) {
        k_union_linear<W, MAXR><<<blocks(uint64_t(n) * 32, 256, 16), 256, 0, st>>>(d_hosts, n, dc, static_cast<const W*>(d_lin), kthr, d_out);
        check_launch();
        launched();
    }
    void union_linear(const uint32_t* d_hosts, uint32_t n, uint32_t* d_out, uint32_t kthr) {
        if (!n) return;
        if (nib) {
            k_union_linear_nib<4><<<blocks(uint64_t(n) * 32, 256, 16), 256, 0, st>>>(d_hosts, n, dc, static_cast<const uint8_t*>(d_lin), kthr, d_out);
            check_launch();
            launched();
            return;
        }
        if (epoch) {
            if (cfg.rows <= 4)
                k_union_linear_epoch<4><<<blocks(uint64_t(n) * 32, 256, 16), 256, 0, st>>>(d_hosts, n, dc, static_cast<const uint8_t*>(d_lin), cur_epoch, d_out);
            else
                k_union_linear_epoch<64><<<blocks(uint64_t(n) * 32, 256, 16), 256, 0, st>>>(d_hosts, n, dc, static_cast<const uint8_t*>(d_lin), cur_epoch, d_out);
            check_launch();
            launched();
            return;
        }
        with_w([&](auto w) {
            using W = decltype(w);
            if (cfg.rows <= 4) union_linear_t<W, 4>(d_hosts, n, d_out, kthr);
            else union_linear_t<W, 64>(d_hosts, n, d_out, kthr);
        });
    }

    void row_active_async() {
        d_counts.ensure(cfg.rows);
        CK(cudaMemsetAsync(d_counts.p, 0, cfg.rows * sizeof(unsigned long long), st));
        if (nib) {
            dim3 grid(blocks(lin_bytes(lin_words) / 4, 256, std::max(1u, 16u / std::min(16u, cfg.rows))), cfg.rows);
            k_row_active_nib<<<grid, 256, 0, st>>>(static_cast<const uint8_t*>(d_lin), lin_words, cfg.window, d_counts.p);
        } else with_w([&](auto w) {
            using W = decltype(w);
            const uint64_t vecs = lin_words * sizeof(W) / 16 + 1;
            dim3 grid(blocks(vecs, 256, std::max(1u, 16u / std::min(16u, cfg.rows))), cfg.rows);
            k_row_active<W><<<grid, 256, 0, st>>>(static_cast<const W*>(d_lin), lin_words, cfg.window, d_counts.p);
        });
        check_launch();
        launched();
    }

    void row_active(uint64_t* out) {
        flush_linear();
        if (epoch) {
            CK(cudaMemcpyAsync(pin_hist.p, hist.p, uint64_t(cfg.rows) * 256 * 8, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            counts_from_hist(out);
            return;
        }
        row_active_async();
        pin_counts.ensure(cfg.rows);
        CK(cudaMemcpyAsync(pin_counts.p, d_counts.p, cfg.rows * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (uint32_t i = 0; i < cfg.rows; ++i) out[i] = pin_counts.p[i];
    }

    // Candidates in ascending host order into sorted_hosts (or the sorted
    // retained list itself). The retained prefix of the list was sorted in the
    // background by the last slide; only the hosts appended since are sorted
    // here and merged in.
    const uint32_t* sort_candidates(uint32_t n) {
        last_sort_new = n;
        if (sorted_ret_valid && nsorted_ret == n) return sorted_ret.p;  // kept up to date by append_candidates
        if (sorted_ret_valid && nsorted_ret <= n && nsorted_ret > 0) {
            const uint32_t m = n - static_cast<uint32_t>(nsorted_ret);
            last_sort_new = m;
            if (m == 0) return sorted_ret.p;
            newsorted.ensure(m);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceRadixSort::SortKeys(t, b, csip.p + nsorted_ret, newsorted.p, static_cast<int>(m), 0, 32, st);
            });
            eos_mark("sort-new");
            k_merge_sorted<<<blocks((uint64_t(n) + 7) / 8), 256, 0, st>>>(sorted_ret.p, static_cast<uint32_t>(nsorted_ret),
                                                                        newsorted.p, m, sorted_hosts.p);
            check_launch();
            launched();
            return sorted_hosts.p;
        }
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, csip.p, sorted_hosts.p, static_cast<int>(n), 0, 32, st);
        });
        return sorted_hosts.p;
    }

    // report_window (sea.hpp:288-309). With counts_ready, d_counts already
    // holds the per-row active counts and the table has been aged by the fused
    // count+age pass, so union activity is tested with r < k+1 (exact while
    // k < expired: an aged recorder r' = r+1 for every r < expired).
    // `between` runs once the report's device work is queued, before the host
    // waits for it (end_slice queues the slide maintenance there).
    void report(srla_entry* out, double* fp_out, bool counts_ready = false, const Compact* compact = nullptr,
                const std::function<void()>& between = {}) {
        const auto w0 = std::chrono::steady_clock::now();
        const uint32_t n = static_cast<uint32_t>(ncsip);
        cudaPointerAttributes oa{};
        const bool out_pinned = !compact && n >= (1u << 14) && cudaPointerGetAttributes(&oa, out) == cudaSuccess &&
                                oa.type == cudaMemoryTypeHost;
        cudaGetLastError();
        const uint32_t kthr = counts_ready ? cfg.window + 1 : cfg.window;
        if (!counts_ready) {
            flush_linear();
            if (!epoch) row_active_async();
        }
        // the fill counts go to the host first (copy stream), so the Eq. 9
        // table is built while the gather runs
        CK(cudaEventRecord(ev_counts_ready, st));
        CK(cudaStreamWaitEvent(ds, ev_counts_ready, 0));
        pin_counts.ensure(cfg.rows);
        if (epoch) CK(cudaMemcpyAsync(pin_hist.p, hist.p, uint64_t(cfg.rows) * 256 * 8, cudaMemcpyDeviceToHost, ds));
        else CK(cudaMemcpyAsync(pin_counts.p, d_counts.p, cfg.rows * sizeof(unsigned long long), cudaMemcpyDeviceToHost, ds));
        CK(cudaEventRecord(ev_counts, ds));
        const uint32_t* sh = sorted_hosts.p;  // report order: hosts ascending (sea.hpp:294-295)
        if (n) {
            sorted_hosts.ensure(n);
            weights.ensure(n);
            eos_mark("pre-sort");
            sh = sort_candidates(n);
            eos_mark("sorted");
            // (host, weight) pairs go to the host on the copy stream ds: the
            // sorted hosts while the gather runs, the weights part by part as
            // the gather finishes them (the hand-off trails by one part)
            uint32_t* hdst = compact ? compact->hosts : nullptr;
            uint32_t* wdst = compact ? compact->weights : nullptr;
            if (!compact && !out_pinned) {
                pin_hosts.ensure(n);
                pin_w.ensure(n);
                hdst = pin_hosts.p;
                wdst = pin_w.p;
            }
            if (hdst) {
                CK(cudaEventRecord(ev_sorted, st));
                CK(cudaStreamWaitEvent(ds, ev_sorted, 0));
                CK(cudaMemcpyAsync(hdst, sh, n * 4ull, cudaMemcpyDefault, ds));  // host, or device (srla_shard)
            }
            const uint32_t parts = hdst && n >= (1u << 16) ? kReportParts : 1u;
            for (uint32_t c = 0; c < parts; ++c) {
                const uint32_t lo = static_cast<uint32_t>(uint64_t(n) * c / parts);
                const uint32_t hi = static_cast<uint32_t>(uint64_t(n) * (c + 1) / parts);
                const cudaEvent_t tg = timer_start();
                union_linear(sh + lo, hi - lo, weights.p + lo, kthr);
                timer_stop(tg, kTimeGather);
                timing.gather_kernel_launches += 1;
                timing.gather_bytes += uint64_t(hi - lo) * cfg.rows * lin_bytes(cfg.linear_slots);
                if (hdst) {
                    CK(cudaEventRecord(ev_part[c], st));
                    CK(cudaStreamWaitEvent(ds, ev_part[c], 0));
                    CK(cudaMemcpyAsync(wdst + lo, weights.p + lo, (hi - lo) * 4ull, cudaMemcpyDefault, ds));
                }
            }
            eos_mark("gathered");
            if (hdst) {
                CK(cudaEventRecord(ev_d2h, ds));
                CK(cudaStreamWaitEvent(st, ev_d2h, 0));
            }
            eos_mark("d2h");
        }
        const uint32_t report_epoch = cur_epoch;  // `between` may slide it
        if (between) between();
        CK(cudaEventSynchronize(ev_counts));
        eos_mark("counts");
        std::vector<uint64_t> counts(pin_counts.p, pin_counts.p + cfg.rows);
        if (epoch) counts_from_hist(counts.data(), report_epoch);
        const double fp = srla_host::fill_product(counts.data(), cfg.rows, lin_words);
        if (fp_out) *fp_out = fp;
        lut_est.resize(cfg.linear_slots + 1);
        lut_has.resize(cfg.linear_slots + 1);
        lut_sup.resize(cfg.linear_slots + 1);
        srla_host::estimate_lut(cfg.linear_slots, fp, cfg.theta, lut_est.data(), lut_has.data(), lut_sup.data());
        eos_mark("lut");
        CK(cudaStreamSynchronize(st));
        eos_mark("synced");
        trace("  report: sort+gather+d2h");
        // (host, weight) -> entries: on the device straight into a pinned
        // caller buffer, else on the host into pageable memory
        if (compact) {
            for (uint32_t w = 0; w <= cfg.linear_slots; ++w) {
                compact->est[w] = lut_est[w];
                compact->flags[w] = static_cast<uint8_t>(lut_has[w] | (lut_sup[w] << 1));
            }
        } else if (out_pinned) {
            const uint32_t L = cfg.linear_slots + 1;
            pin_lut.ensure(L * 10ull);
            double* le = reinterpret_cast<double*>(pin_lut.p);
            uint8_t* lh = pin_lut.p + 8ull * L;
            std::memcpy(le, lut_est.data(), 8ull * L);
            std::memcpy(lh, lut_has.data(), L);
            std::memcpy(lh + L, lut_sup.data(), L);
            d_lut.ensure(L * 10ull);
            CK(cudaMemcpyAsync(d_lut.p, pin_lut.p, L * 10ull, cudaMemcpyHostToDevice, st));
            d_entries.ensure(3ull * n);
            k_map_entries<<<blocks(n), 256, 0, st>>>(sh, weights.p, n, reinterpret_cast<const double*>(d_lut.p),
                                                     d_lut.p + 8ull * L, d_lut.p + 9ull * L, d_entries.p);
            check_launch();
            launched();
            // one DMA into the caller's pinned buffer (kernel stores over PCIe are scattered)
            CK(cudaMemcpyAsync(out, d_entries.p, 24ull * n, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
        } else {
            auto fill = [&](uint32_t lo, uint32_t hi) {
                for (uint32_t e = lo; e < hi; ++e) {
                    const uint32_t w = pin_w.p[e];
                    srla_entry x{};
                    x.host = pin_hosts.p[e];
                    x.union_weight = w;
                    x.estimate = lut_est[w];
                    x.has_estimate = lut_has[w];
                    x.is_super = lut_sup[w];
                    out[e] = x;
                }
            };
            const uint32_t nt = n >= (1u << 16) ? 8u : 1u;
            if (nt == 1) {
                fill(0, n);
            } else {
                std::vector<std::thread> pool;
                for (uint32_t t = 1; t < nt; ++t) pool.emplace_back(fill, uint64_t(n) * t / nt, uint64_t(n) * (t + 1) / nt);
                fill(0, n / nt);
                for (auto& th : pool) th.join();
            }
        }
        timing.report_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
    }

    // ------------------------------------------------------------ slide (sea.hpp:316-338)
    // The slide is split so that only what the report hand-off needs sits on
    // the engine stream:
    //  * slide_begin (side stream st2, at end-of-slice start, concurrent with
    //    the report): re-validate the candidates on the NOT yet aged rough
    //    table.
    //    union_rough_weight after aging counts r + (r != expired) < k, i.e.
    //    r < k - 1 (k <= expired), so the retain test runs with k - 1.
    //  * slide_finish: swap in the retained list, then queue the table
    //    maintenance on st2 — indicator clear + re-set for the kept hosts,
    //    rough aging, the epoch sweep, the candidate hash rebuild and sorted view. It overlaps the next slice's K1 (which touches none of it);
    //    the engine stream joins it before the first reader (join_maint).
    template <typename W, int MAXR>
    void slide_begin_t() {
        CK(cudaEventRecord(ev_eos_start, st));
        CK(cudaStreamWaitEvent(st2, ev_eos_start, 0));
        if (ncsip) {
            const uint32_t n = static_cast<uint32_t>(ncsip);
            keep.ensure(n);
            csip2.ensure(n);
            DevCfg aged = dc;
            aged.k = dc.k - 1;  // retain on the pre-aging table (see above)
            // a quarter of the GPU: the retain has the whole report to finish
            k_retain<W, MAXR><<<blocks(n, 256, 2), 256, 0, st2>>>(csip.p, n, aged, static_cast<const W*>(d_rough), keep.p);
            check_launch();
            launched();
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceSelect::Flagged(t, b, csip.p, keep.p, csip2.p, ctr.p + 6, static_cast<int>(n), st2);
            }, &temp2);
            CK(cudaMemcpyAsync(pin_ctr.p + 6, ctr.p + 6, 4, cudaMemcpyDeviceToHost, st2));
        }
        CK(cudaEventRecord(ev_retained, st2));
        slide_begun = true;
    }
    void slide_begin() {
        with_w([&](auto w) {
            using W = decltype(w);
            if (cfg.rows <= 4) slide_begin_t<W, 4>();
            else slide_begin_t<W, 64>();
        });
    }

    template <typename W>
    void slide_finish_t(bool age_linear) {
        const uint64_t rows = cfg.rows;
        // the report (and anything else on st) has finished reading the
        // linear table and the old candidate list
        CK(cudaEventRecord(ev_reported, st));
        CK(cudaStreamWaitEvent(st2, ev_reported, 0));
        if (epoch) {
            cur_epoch = (cur_epoch + 1) & 0xFFu;
            k_zero_hist_bin<<<1, 64, 0, st>>>(hist.p, cfg.rows, cur_epoch);
            check_launch();
            launched();
            sweep_t(st2);
            CK(cudaEventRecord(ev_maint_lin, st2));
            maint_lin_pending = true;
        } else if (age_linear) {
            k_age<W><<<blocks(rows * lin_words * sizeof(W) / 16 + 1, 256, 16), 256, 0, st>>>(static_cast<W*>(d_lin), rows * lin_words, dc.expired);
            check_launch();
            launched();
        }
        k_age<W><<<blocks(rows * rough_words * sizeof(W) / 16 + 1, 256, 16), 256, 0, st2>>>(static_cast<W*>(d_rough), rows * rough_words, dc.expired);
        check_launch();
        launched();
        // the retained count gates the host-side list swap; the engine stream
        // also waits for it, so the end-of-slice device time covers the retain
        CK(cudaEventSynchronize(ev_retained));
        CK(cudaStreamWaitEvent(st, ev_retained, 0));
        slide_begun = false;
        if (ncsip) {
            ncsip = pin_ctr.p[6];
            std::swap(csip.p, csip2.p);
            std::swap(csip.cap, csip2.cap);
        }
        // indicators: clear all, re-set the retained hosts' bit in every row
        // (sea.hpp:318, 333-335); read again only by the next slice's K4
        CK(cudaMemsetAsync(d_si, 0, rows * cfg.cols * sizeof(uint16_t), st2));
        if (ncsip) {
            k_si_mark<<<blocks(ncsip), 256, 0, st2>>>(csip.p, static_cast<uint32_t>(ncsip), dc, d_si);
            check_launch();
            launched();
        }
        rebuild_cset(ncsip, st2);
        if (ncsip) {  // into the spare buffer: a queued report may still read the current view
            sorted_tmp.ensure(ncsip);
            cub_call([&](void* t, size_t& b) {
                return cub::DeviceRadixSort::SortKeys(t, b, csip.p, sorted_tmp.p, static_cast<int>(ncsip), 0, 32, st2);
            }, &temp2);
            std::swap(sorted_ret.p, sorted_tmp.p);
            std::swap(sorted_ret.cap, sorted_tmp.cap);
        }
        nsorted_ret = ncsip;
        sorted_ret_valid = true;
        CK(cudaEventRecord(ev_maint, st2));
        maint_pending = true;
        trace("  slide: finish (maintenance queued)");
    }

    // one slide's share of the epoch sweep (epoch.cuh: every byte at least
    // once per 255 - expired slides)
    void sweep_t(cudaStream_t s) {
        const uint64_t total = uint64_t(cfg.rows) * lin_words;
        const uint64_t period = 255 - dc.expired;
        const uint64_t chunk = ((total + period - 1) / period + 15) & ~15ull;
        const uint64_t end = std::min(total, sweep_pos + chunk);
        k_sweep<<<blocks((end - sweep_pos) / 16 + 1, 256, 8), 256, 0, s>>>(static_cast<uint8_t*>(d_lin), sweep_pos,
                                                                          end - sweep_pos, cur_epoch, dc.expired);
        check_launch();
        launched();
        sweep_pos = end >= total ? 0 : end;
    }

    // The engine stream waits for queued maintenance (device-side wait).
    void join_maint_lin() {
        if (!maint_lin_pending) return;
        CK(cudaStreamWaitEvent(st, ev_maint_lin, 0));
        maint_lin_pending = false;
    }
    void join_maint() {
        join_maint_lin();
        if (!maint_pending) return;
        CK(cudaStreamWaitEvent(st, ev_maint, 0));
        maint_pending = false;
    }

    void slide_finish(bool age_linear) {
        with_w([&](auto w) { slide_finish_t<decltype(w)>(age_linear); });
    }

    // EstimatorArray::slide (sea.hpp:316-338) on its own
    void slide(bool age_linear = true) {
        const auto w0 = std::chrono::steady_clock::now();
        stats.slides++;
        join_maint();
        flush_linear(use_bins && !epoch && age_linear ? 1 : 0);
        if (use_bins && !epoch) age_linear = false;  // aged by the flush
        if (!slide_begun) slide_begin();
        slide_finish(age_linear);
        CK(cudaStreamSynchronize(st));
        timing.slide_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w0).count();
    }

    // process_slice tail (pipeline.hpp:119-128). When a report is due and
    // k < expired, one fused pass counts and ages the linear table, and the
    // report reads the aged table (see report()).
    void end_slice(uint64_t slice_id, bool want_report, srla_entry* out, const Compact* compact = nullptr) {
        const bool due = want_report && slice_id + 1 >= cfg.window;
        trace(nullptr);
        eos_host_t0 = std::chrono::steady_clock::now();
        eos_mark("start");
        join_maint();
        stats.slides++;
        // the candidate re-validation reads only the rough table: with a
        // streamed apply in this end-of-slice it starts after the apply
        // (overlapping the gather) instead of competing with it
        static const bool retain_late = [] { const char* v = std::getenv("SRLA_RETAIN_LATE"); return !(v && v[0] == '0'); }();
        const bool late = retain_late && !epoch && use_bins && due && dc.k < dc.expired;
        if (!late) slide_begin();
        eos_mark("begin");
        const auto w0 = std::chrono::steady_clock::now();
        bool age_linear = false, finished = false;
        // the slide maintenance is queued while the report's gather runs
        auto finish = [&] {
            eos_mark("reported");
            slide_finish(false);
            eos_mark("slid");
            finished = true;
        };
        if (epoch) {
            flush_linear();
            if (due) report(out, nullptr, false, compact, finish);
            trace("eos: report (epoch)");
        } else if (due && dc.k < dc.expired && use_bins) {
            d_counts.ensure(cfg.rows);
            CK(cudaMemsetAsync(d_counts.p, 0, cfg.rows * sizeof(unsigned long long), st));
            flush_linear(2);
            if (late) slide_begin();
            trace("eos: split+apply+count+age");
            report(out, nullptr, true, compact, finish);
            trace("eos: report");
        } else if (due && dc.k < dc.expired) {
            d_counts.ensure(cfg.rows);
            CK(cudaMemsetAsync(d_counts.p, 0, cfg.rows * sizeof(unsigned long long), st));
            with_w([&](auto w) { count_age_range<decltype(w)>(0, uint64_t(cfg.rows) * lin_words, true); });
            report(out, nullptr, true, compact, finish);
            trace("eos: report");
        } else if (!due && use_bins) {
            flush_linear(1);
        } else {
            if (due) report(out, nullptr, false, compact);
            age_linear = !use_bins;
            if (use_bins) flush_linear(1);
        }
        const auto w1 = std::chrono::steady_clock::now();
        if (!finished) {
            eos_mark("reported");
            slide_finish(age_linear);
            eos_mark("slid");
        }
        CK(cudaStreamSynchronize(st));
        eos_dump();
        timing.slide_wall_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - w1).count();
        (void)w0;
        resolve_timers(false);
        trace("eos: slide");
    }

    // ------------------------------------------------------------ queries
    void set_candidates(const uint32_t* h, uint64_t n) {
        sorted_ret_valid = false;
        std::vector<uint32_t> uniq;
        uniq.reserve(n);
        std::unordered_set<uint32_t> seen;
        for (uint64_t i = 0; i < n; ++i)
            if (seen.insert(h[i]).second) uniq.push_back(h[i]);
        ncsip = 0;
        csip.ensure(std::max<size_t>(uniq.size(), 1));
        if (!uniq.empty())
            CK(cudaMemcpyAsync(csip.p, uniq.data(), uniq.size() * 4, cudaMemcpyHostToDevice, st));
        ncsip = uniq.size();
        rebuild_cset(ncsip);
        CK(cudaStreamSynchronize(st));
    }

    void candidates(std::vector<uint32_t>& out) {
        out.resize(ncsip);
        if (ncsip) CK(cudaMemcpyAsync(out.data(), csip.p, ncsip * 4, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }

    void union_weights(const uint32_t* h, uint64_t n, uint32_t* rw, uint32_t* lw) {
        if (!n) return;
        const uint32_t m = static_cast<uint32_t>(n);
        qhosts.ensure(m);
        weights.ensure(m);
        rweights.ensure(m);
        CK(cudaMemcpyAsync(qhosts.p, h, n * 4, cudaMemcpyHostToDevice, st));
        if (rw) {
            with_w([&](auto w) {
                using W = decltype(w);
                if (cfg.rows <= 4)
                    k_union_rough<W, 4><<<blocks(m), 256, 0, st>>>(qhosts.p, m, dc, static_cast<const W*>(d_rough), rweights.p);
                else
                    k_union_rough<W, 64><<<blocks(m), 256, 0, st>>>(qhosts.p, m, dc, static_cast<const W*>(d_rough), rweights.p);
            });
            check_launch();
            launched();
            CK(cudaMemcpyAsync(rw, rweights.p, n * 4, cudaMemcpyDeviceToHost, st));
        }
        if (lw) {
            flush_linear();
            union_linear(qhosts.p, m, weights.p, cfg.window);
            CK(cudaMemcpyAsync(lw, weights.p, n * 4, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
    }

    uint32_t host_column(uint32_t row, uint32_t aip) const {
        return static_cast<uint32_t>((static_cast<uint64_t>(hash_u32(dc.sub_row[row], aip)) * cfg.cols) >> 32);
    }

    uint32_t word_at(const std::vector<uint8_t>& b, uint64_t j) const {
        uint32_t v = 0;
        for (uint32_t q = 0; q < wb; ++q) v |= static_cast<uint32_t>(b[j * wb + q]) << (8 * q);
        return v;
    }

    // union_view (sea.hpp:199-217)
    void union_view(uint32_t aip, uint16_t* ind, uint32_t* rough, uint32_t* linear) {
        flush_linear();
        uint16_t acc = 0xFFFF;
        std::fill(rough, rough + cfg.rough_slots, 0u);
        if (linear) std::fill(linear, linear + cfg.linear_slots, 0u);
        std::vector<uint8_t> rb(uint64_t(cfg.rough_slots) * wb), lb(uint64_t(cfg.linear_slots) * wb);
        for (uint32_t i = 0; i < cfg.rows; ++i) {
            const uint64_t col = host_column(i, aip);
            uint16_t s = 0;
            CK(cudaMemcpyAsync(&s, d_si + uint64_t(i) * cfg.cols + col, 2, cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(rb.data(), static_cast<uint8_t*>(d_rough) + (uint64_t(i) * rough_words + col * cfg.rough_slots) * wb, rb.size(), cudaMemcpyDeviceToHost, st));
            if (linear && nib) {  // gl is a multiple of 32 in nibble mode: whole bytes
                std::vector<uint8_t> pk(cfg.linear_slots / 2);
                CK(cudaMemcpyAsync(pk.data(), static_cast<uint8_t*>(d_lin) + lin_bytes(uint64_t(i) * lin_words + col * cfg.linear_slots),
                                   pk.size(), cudaMemcpyDeviceToHost, st));
                CK(cudaStreamSynchronize(st));
                for (uint32_t j = 0; j < cfg.linear_slots; ++j) lb[j] = (pk[j >> 1] >> (4 * (j & 1))) & 0xF;
            } else if (linear)
                CK(cudaMemcpyAsync(lb.data(), static_cast<uint8_t*>(d_lin) + (uint64_t(i) * lin_words + col * cfg.linear_slots) * wb, lb.size(), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            acc &= s;
            for (uint32_t j = 0; j < cfg.rough_slots; ++j) rough[j] = std::max(rough[j], word_at(rb, j));
            if (linear)
                for (uint32_t j = 0; j < cfg.linear_slots; ++j)
                    linear[j] = std::max(linear[j], epoch ? stamp_value(lb[j]) : word_at(lb, j));
        }
        *ind = acc;
    }

    uint64_t row_bytes(int kind) const {
        if (kind == SRLA_INDICATOR) return uint64_t(cfg.cols) * 2;
        if (kind == SRLA_ROUGH) return rough_words * wb;
        if (kind == SRLA_LINEAR) return lin_words * wb;
        throw Error(SRLA_E_INVALID, "unknown row kind");
    }

    uint8_t* row_ptr(uint32_t row, int kind) {
        if (row >= cfg.rows) throw Error(SRLA_E_RANGE, "row index out of range");
        const uint64_t b = row_bytes(kind);
        if (kind == SRLA_INDICATOR) return reinterpret_cast<uint8_t*>(d_si) + row * b;
        if (kind == SRLA_ROUGH) return static_cast<uint8_t*>(d_rough) + row * b;
        return static_cast<uint8_t*>(d_lin) + lin_bytes(uint64_t(row) * lin_words);
    }

    // Row export/import (the raw spans of sea.hpp:341-346; snapshot.hpp
    // writes and reads them). Epoch-stamp and nibble tables convert to and
    // from the reference's layout on the device, chunk by chunk through a
    // staging buffer, so a 16 GiB row moves at copy speed.
    static constexpr uint64_t kXferChunk = 1ull << 26;  // reference-layout bytes per hop
    DevBuf<uint8_t> xfer;

    void export_row(uint32_t row, int kind, void* buf, uint64_t bytes) {
        if (bytes != row_bytes(kind)) throw Error(SRLA_E_INVALID, "buffer size does not match the row");
        export_range(row, kind, 0, buf, bytes);
    }

    // Reference-layout bytes [off, off + bytes) of a row, chunk by chunk:
    // converted on the device (nibble / epoch tables) and copied through a
    // pinned staging buffer unless the caller's buffer is pinned itself.
    PinBuf<uint8_t> xpin;
    static bool is_pinned(const void* p) {
        cudaPointerAttributes a{};
        const bool pinned = cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeHost;
        cudaGetLastError();
        return pinned;
    }
    void check_range(uint32_t row, int kind, uint64_t off, uint64_t bytes) {
        (void)row_ptr(row, kind);  // row / kind checks
        if (off > row_bytes(kind) || bytes > row_bytes(kind) - off) throw Error(SRLA_E_RANGE, "byte range outside the row");
        if (kind == SRLA_LINEAR && nib && ((off | bytes) & 1))
            throw Error(SRLA_E_INVALID, "packed linear rows move in whole bytes pairs: even offset and size");
    }
    void export_range(uint32_t row, int kind, uint64_t off, void* buf, uint64_t bytes) {
        flush_linear();
        check_range(row, kind, off, bytes);
        uint8_t* p = row_ptr(row, kind);
        uint8_t* b = static_cast<uint8_t*>(buf);
        const bool convert = kind == SRLA_LINEAR && (nib || epoch);
        const bool direct = is_pinned(buf);
        if (convert) xfer.ensure(std::min(bytes, kXferChunk));
        if (!direct) xpin.ensure(std::min(bytes, kXferChunk));
        for (uint64_t j0 = 0; j0 < bytes; j0 += kXferChunk) {
            const uint64_t m = std::min(kXferChunk, bytes - j0);  // reference-layout bytes of this hop
            const uint8_t* src = p + off + j0;
            if (convert) {
                if (nib)
                    k_unpack_nib<<<blocks(m / 2, 256, 16), 256, 0, st>>>(p + (off + j0) / 2, m / 2, xfer.p);
                else
                    k_stamps_to_values<<<blocks(m, 256, 16), 256, 0, st>>>(p + off + j0, m, cur_epoch, dc.expired, xfer.p);
                check_launch();
                launched();
                src = xfer.p;
            }
            CK(cudaMemcpyAsync(direct ? b + j0 : xpin.p, src, m, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            if (!direct) std::memcpy(b + j0, xpin.p, m);
        }
    }

    // Block digests of one row in the reference layout (digest.cuh), on the device.
    DevBuf<uint64_t> d_digest;
    uint64_t state_blocks(uint32_t row, int kind, uint64_t* out, uint64_t cap) {
        flush_linear();
        join_maint();
        uint8_t* p = row_ptr(row, kind);
        const uint64_t bytes = row_bytes(kind);
        const uint64_t nb = (bytes + (1ull << kDigestBlockShift) - 1) >> kDigestBlockShift;
        if (!out) return nb;
        if (cap < nb) throw Error(SRLA_E_CAPACITY, "digest buffer holds " + std::to_string(cap) + " blocks, " +
                                                       std::to_string(nb) + " needed");
        DigestSrc src{p, bytes, kDigestRaw, cur_epoch, dc.expired};
        if (kind == SRLA_LINEAR && nib) src.layout = kDigestNibble;
        if (kind == SRLA_LINEAR && epoch) src.layout = kDigestEpoch;
        d_digest.ensure(nb);
        if (nb) {
            k_block_sums<<<static_cast<uint32_t>(nb), kDigestThreads, 0, st>>>(src, d_digest.p);
            check_launch();
            launched();
            CK(cudaMemcpyAsync(out, d_digest.p, nb * 8, cudaMemcpyDeviceToHost, st));
        }
        CK(cudaStreamSynchronize(st));
        return nb;
    }

    void import_row(uint32_t row, int kind, const void* buf, uint64_t bytes) {
        if (bytes != row_bytes(kind)) throw Error(SRLA_E_INVALID, "buffer size does not match the row");
        import_range(row, kind, 0, buf, bytes);
    }

    void import_range(uint32_t row, int kind, uint64_t off, const void* buf, uint64_t bytes) {
        flush_linear();
        check_range(row, kind, off, bytes);
        uint8_t* p = row_ptr(row, kind);
        const uint8_t* v = static_cast<const uint8_t*>(buf);
        const bool convert = kind == SRLA_LINEAR && (nib || epoch);
        if (convert) {
            uint8_t vmax = 0;  // vectorisable reduction (no early exit)
            for (uint64_t j = 0; j < bytes; ++j) vmax = std::max(vmax, v[j]);
            if (vmax > (nib ? 0xFu : dc.expired)) {  // beyond the packed / stamp model: a byte per value
                if (nib) leave_nibble();
                else leave_epoch();
                import_range(row, kind, off, buf, bytes);
                return;
            }
            xfer.ensure(std::min(bytes, kXferChunk));
        }
        const bool direct = is_pinned(buf);
        if (!direct) xpin.ensure(std::min(bytes, kXferChunk));
        unsigned long long* h = epoch && kind == SRLA_LINEAR ? hist.p + uint64_t(row) * 256 : nullptr;
        for (uint64_t j0 = 0; j0 < bytes; j0 += kXferChunk) {
            const uint64_t m = std::min(kXferChunk, bytes - j0);
            const uint8_t* src = v + j0;
            if (!direct) {
                std::memcpy(xpin.p, v + j0, m);
                src = xpin.p;
            }
            if (h) {  // the row's stamp histogram loses the overwritten stamps ...
                k_row_hist<<<blocks(m, 256, 4), 256, 0, st>>>(p + off + j0, m, h, -1);
                check_launch();
                launched();
            }
            if (convert) {
                CK(cudaMemcpyAsync(xfer.p, src, m, cudaMemcpyHostToDevice, st));
                if (nib)
                    k_pack_nib<<<blocks(m / 2, 256, 16), 256, 0, st>>>(xfer.p, m / 2, p + (off + j0) / 2);
                else
                    k_values_to_stamps<<<blocks(m, 256, 16), 256, 0, st>>>(xfer.p, m, cur_epoch, p + off + j0);
                check_launch();
                launched();
            } else {
                CK(cudaMemcpyAsync(p + off + j0, src, m, cudaMemcpyHostToDevice, st));
            }
            if (h) {  // ... and gains the new ones
                k_row_hist<<<blocks(m, 256, 4), 256, 0, st>>>(p + off + j0, m, h, 1);
                check_launch();
                launched();
            }
            CK(cudaStreamSynchronize(st));  // the staging buffers are reused
        }
    }
};

}  // namespace srla

// ====================================================================== C ABI
struct srla_engine {
    srla::Engine* impl;
    std::mutex mu;
};

namespace {
thread_local std::string g_last_error;

template <typename Fn>
srla_status guard(Fn&& fn) {
    try {
        fn();
        g_last_error.clear();
        return SRLA_OK;
    } catch (const srla::Error& e) {
        g_last_error = e.what();
        return e.code;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return SRLA_E_INTERNAL;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return SRLA_E_INTERNAL;
    }
}

// the engine's call mutex (a null engine is an argument error, not a crash)
std::mutex& lock_of(srla_engine* e) {
    if (!e || !e->impl) throw srla::Error(SRLA_E_INVALID, "null engine");
    return e->mu;
}

srla::Engine& E(srla_engine* e, bool join = true) {
    if (!e || !e->impl) throw srla::Error(SRLA_E_INVALID, "null engine");
    CK(cudaSetDevice(e->impl->device));
    if (join) {
        e->impl->join_eos();
        e->impl->join_maint();
    }
    return *e->impl;
}
const srla::Engine& CE(const srla_engine* e) {
    if (!e || !e->impl) throw srla::Error(SRLA_E_INVALID, "null engine");
    return *e->impl;
}

void check_capacity(uint64_t need, srla_entry* out, uint64_t cap, uint64_t* n_out) {
    if (n_out) *n_out = need;
    if (need > cap || (!out && need))
        throw srla::Error(SRLA_E_CAPACITY, "report buffer holds " + std::to_string(cap) + " entries, " +
                                               std::to_string(need) + " needed");
}
}  // namespace

extern "C" {

const char* srla_last_error(void) { return g_last_error.c_str(); }

srla_status srla_internal_set_error(srla_status code, const char* msg) {
    g_last_error = msg ? msg : "";
    return code;
}
const char* srla_version(void) { return "srla_b200 0.1 sm_100a"; }

srla_status srla_create(const srla_config* cfg, int device, srla_engine** out) {
    return guard([&] {
        if (!cfg || !out) throw srla::Error(SRLA_E_INVALID, "null argument");
        *out = nullptr;
        auto* e = new srla_engine;
        try {
            e->impl = new srla::Engine(*cfg, device);
        } catch (...) {
            delete e;
            throw;
        }
        *out = e;
    });
}

srla_status srla_destroy(srla_engine* e) {
    return guard([&] {
        if (!e) return;
        if (e->impl) {
            cudaSetDevice(e->impl->device);
            delete e->impl;
        }
        delete e;
    });
}

srla_status srla_params(const srla_engine* e, uint32_t* tau, uint32_t* threshold, uint32_t* word_bytes) {
    return guard([&] {
        const auto& x = CE(e);
        if (tau) *tau = x.tau;
        if (threshold) *threshold = x.thr;
        if (word_bytes) *word_bytes = x.wb;
    });
}

srla_status srla_column_of(const srla_engine* e, uint32_t row, uint32_t aip, uint32_t* col) {
    return guard([&] {
        const auto& x = CE(e);
        if (row >= x.cfg.rows) throw srla::Error(SRLA_E_RANGE, "row index out of range");
        *col = x.host_column(row, aip);
    });
}

namespace {
srla_status scan_batch_impl(srla_engine* e, const srla_record* recs, uint64_t n, int on_device, cudaStream_t producer,
                            uint32_t* pushed, uint64_t cap, uint64_t* n_pushed) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e, /*join=*/false);  // joins a pending async end-of-slice after staging copies
        if (n && !recs) throw srla::Error(SRLA_E_INVALID, "null records");
        x.collect_pushed = pushed != nullptr || n_pushed != nullptr;
        x.host_pushed.clear();
        x.scan_batch(recs, n, on_device, producer);
        CK(cudaStreamSynchronize(x.st));
        if (n_pushed) *n_pushed = x.host_pushed.size();
        if (pushed)
            std::memcpy(pushed, x.host_pushed.data(), std::min<uint64_t>(cap, x.host_pushed.size()) * 4);
        x.collect_pushed = false;
    });
}
}  // namespace

srla_status srla_scan_batch(srla_engine* e, const srla_record* recs, uint64_t n, int on_device,
                            uint32_t* pushed, uint64_t cap, uint64_t* n_pushed) {
    return scan_batch_impl(e, recs, n, on_device, cudaStreamLegacy, pushed, cap, n_pushed);
}

srla_status srla_scan_device(srla_engine* e, const srla_record* d_recs, uint64_t n, void* producer_stream,
                             uint32_t* pushed, uint64_t cap, uint64_t* n_pushed) {
    return scan_batch_impl(e, d_recs, n, 1, producer_stream ? static_cast<cudaStream_t>(producer_stream) : cudaStreamLegacy,
                           pushed, cap, n_pushed);
}

srla_status srla_candidates(srla_engine* e, uint32_t* out, uint64_t cap, uint64_t* n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e);
        std::vector<uint32_t> v;
        x.candidates(v);
        if (n) *n = v.size();
        if (v.size() > cap || (!out && !v.empty()))
            throw srla::Error(SRLA_E_CAPACITY, "candidate buffer too small");
        if (!v.empty()) std::memcpy(out, v.data(), v.size() * 4);
    });
}

srla_status srla_set_candidates(srla_engine* e, const uint32_t* hosts, uint64_t n) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (n && !hosts) throw srla::Error(SRLA_E_INVALID, "null hosts");
        E(e).set_candidates(hosts, n);
    });
}

srla_status srla_report(srla_engine* e, srla_entry* out, uint64_t cap, uint64_t* n_out, double* fill_product) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e);
        check_capacity(x.ncsip, out, cap, n_out);
        x.report(out, fill_product);
    });
}

srla_status srla_slide(srla_engine* e, uint64_t* n_retained) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e);
        x.slide();
        if (n_retained) *n_retained = x.ncsip;
    });
}

srla_status srla_end_slice(srla_engine* e, uint64_t slice_id, int want_report, srla_entry* out,
                           uint64_t cap, uint64_t* n_out, uint64_t* n_retained) {
    srla_status s = srla_end_slice_async(e, slice_id, want_report, out, cap);
    if (s != SRLA_OK) {
        if (s == SRLA_E_CAPACITY && n_out && e && e->impl) *n_out = e->impl->ncsip;
        return s;
    }
    return srla_end_slice_wait(e, n_out, n_retained);
}

srla_status srla_end_slice_compact(srla_engine* e, uint64_t slice_id, int want_report, uint32_t* hosts,
                                   uint32_t* weights, uint64_t cap, uint64_t* n_out, double* est_lut,
                                   uint8_t* flags_lut, uint64_t* n_retained) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e);
        const bool due = want_report && slice_id + 1 >= x.cfg.window;
        if (n_out) *n_out = due ? x.ncsip : 0;
        if (due && (x.ncsip > cap || ((!hosts || !weights) && x.ncsip)))
            throw srla::Error(SRLA_E_CAPACITY, "report buffers too small");
        if (due && (!est_lut || !flags_lut)) throw srla::Error(SRLA_E_INVALID, "null estimate table");
        const srla::Engine::Compact c{hosts, weights, est_lut, flags_lut};
        x.timed_end_slice(slice_id, want_report != 0, nullptr, &c);
        if (n_retained) *n_retained = x.ncsip;
    });
}

srla_status srla_end_slice_async(srla_engine* e, uint64_t slice_id, int want_report, srla_entry* out,
                                 uint64_t cap) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        E(e).end_slice_async(slice_id, want_report != 0, out, cap);
    });
}

srla_status srla_end_slice_wait(srla_engine* e, uint64_t* n_out, uint64_t* n_retained) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        auto& x = E(e);
        if (!x.eos.pending) throw srla::Error(SRLA_E_INVALID, "no srla_end_slice_async pending");
        x.eos.pending = false;
        if (x.eos.code != SRLA_OK) throw srla::Error(x.eos.code, x.eos.msg);
        if (n_out) *n_out = x.eos.n;
        if (n_retained) *n_retained = x.eos.nret;
    });
}

srla_status srla_union_weights(srla_engine* e, const uint32_t* hosts, uint64_t n, uint32_t* rough_w,
                               uint32_t* linear_w) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (n && !hosts) throw srla::Error(SRLA_E_INVALID, "null hosts");
        E(e).union_weights(hosts, n, rough_w, linear_w);
    });
}

srla_status srla_union_view(srla_engine* e, uint32_t aip, uint16_t* indicator, uint32_t* rough, uint32_t* linear) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (!indicator || !rough) throw srla::Error(SRLA_E_INVALID, "null output");
        E(e).union_view(aip, indicator, rough, linear);
    });
}

srla_status srla_row_active(srla_engine* e, uint64_t* counts) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (!counts) throw srla::Error(SRLA_E_INVALID, "null output");
        E(e).row_active(counts);
    });
}

srla_status srla_estimate_from(const srla_engine* e, uint32_t weight, double fill_product, double* estimate,
                               int* has_estimate) {
    return guard([&] {
        const auto& x = CE(e);
        if (fill_product >= 1.0 - 1e-12 && weight > x.cfg.linear_slots)  // linear_estimate (estimators.hpp:142)
            throw srla::Error(SRLA_E_INVALID, "weight exceeds slot count");
        double v = 0.0;
        const bool h = srla_host::corrected_estimate(x.cfg.linear_slots, weight, fill_product, &v);
        if (estimate) *estimate = h ? v : 0.0;
        if (has_estimate) *has_estimate = h;
    });
}

srla_status srla_row_bytes(const srla_engine* e, int kind, uint64_t* bytes) {
    return guard([&] { *bytes = CE(e).row_bytes(kind); });
}

srla_status srla_export_row(srla_engine* e, uint32_t row, int kind, void* buf, uint64_t bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        E(e).export_row(row, kind, buf, bytes);
    });
}

srla_status srla_import_row(srla_engine* e, uint32_t row, int kind, const void* buf, uint64_t bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        E(e).import_row(row, kind, buf, bytes);
    });
}

srla_status srla_state_blocks(srla_engine* e, uint32_t row, int kind, uint64_t* out, uint64_t cap, uint64_t* n_blocks) {
    return guard([&] {
        const uint64_t nb = E(e).state_blocks(row, kind, out, cap);
        if (n_blocks) *n_blocks = nb;
    });
}

srla_status srla_block_sums(const void* d_buf, uint64_t bytes, uint64_t* out, uint64_t cap, void* stream) {
    return guard([&] {
        using namespace srla;
        const uint64_t nb = (bytes + (1ull << kDigestBlockShift) - 1) >> kDigestBlockShift;
        if (cap < nb) throw Error(SRLA_E_CAPACITY, "digest buffer too small");
        if (!nb) return;
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        uint64_t* d = nullptr;
        CK(cudaMallocAsync(&d, nb * 8, s));
        k_block_sums<<<static_cast<uint32_t>(nb), kDigestThreads, 0, s>>>(
            DigestSrc{static_cast<const uint8_t*>(d_buf), bytes, kDigestRaw, 0, 0}, d);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(out, d, nb * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaFreeAsync(d, s));
        CK(cudaStreamSynchronize(s));
    });
}

srla_status srla_export_range(srla_engine* e, uint32_t row, int kind, uint64_t offset, void* buf, uint64_t bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (bytes && !buf) throw srla::Error(SRLA_E_INVALID, "null buffer");
        E(e).export_range(row, kind, offset, buf, bytes);
    });
}

srla_status srla_import_range(srla_engine* e, uint32_t row, int kind, uint64_t offset, const void* buf, uint64_t bytes) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        if (bytes && !buf) throw srla::Error(SRLA_E_INVALID, "null buffer");
        E(e).import_range(row, kind, offset, buf, bytes);
    });
}

srla_status srla_host_alloc(uint64_t bytes, void** out) {
    return guard([&] {
        if (!out) throw srla::Error(SRLA_E_INVALID, "null output");
        *out = nullptr;
        CK(cudaMallocHost(out, std::max<uint64_t>(bytes, 1)));
    });
}

srla_status srla_host_free(void* p) {
    return guard([&] {
        if (p) CK(cudaFreeHost(p));
    });
}

srla_status srla_stats_get(const srla_engine* e, srla_stats* out) {
    return guard([&] { *out = CE(e).stats; });
}

srla_status srla_timing_get(const srla_engine* e, srla_timing* out) {
    return guard([&] {
        if (!out) throw srla::Error(SRLA_E_INVALID, "null output");
        // resolving the pending kernel timers mutates only timing bookkeeping
        auto* m = const_cast<srla_engine*>(e);
        std::lock_guard<std::mutex> lk(m->mu);
        E(m, false).timing_snapshot(out);
    });
}

srla_status srla_timing_reset(srla_engine* e) {
    return guard([&] {
        std::lock_guard<std::mutex> lk(lock_of(e));
        E(e).timing_clear();
    });
}

srla_status srla_synchronize(srla_engine* e) {
    return guard([&] { CK(cudaStreamSynchronize(E(e).st)); });
}

srla_status srla_stream(srla_engine* e, void** stream) {
    return guard([&] { *stream = static_cast<void*>(E(e).st); });
}

}  // extern "C"
