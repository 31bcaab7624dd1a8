// scan_binned.cuh — the linear-mark path for tables larger than L2.
//
// Measured on B200 (tools/membench.cu, profiles/): scattered 1-byte stores into
// a 4 GiB table sustain ~23 G/s (every store is a DRAM sector read-modify-
// write), the same stores confined to an L2-resident 64 MB region ~129 G/s and
// 32-bit atomicAnd ~212 G/s. The linear marks of a slice (u per packet,
// store 0) commute with each other and with every other hot-path step except
// reads of the linear table, so K1 only *bins* them: a block multi-split by
// table region (64 MB slabs) with one global reservation per region per tile
// and coalesced bin writes. At flush time the region bins are split into
// 64 KB table slices and each slice is applied in shared memory (below), so
// the table streams through HBM once per flush instead of one sector
// read-modify-write per mark. Any reader of the linear table flushes first
// (Engine::flush_linear).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace srla {

// ---- bulk-copy (TMA engine) + mbarrier helpers, sm_90+/sm_100a PTX
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}
// global -> shared, completion counted on the mbarrier in bytes
__device__ __forceinline__ void bulk_load(void* dst_smem, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst_smem)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
// shared -> global, tracked by the issuing thread's bulk groups
__device__ __forceinline__ void bulk_store(void* dst, const void* src_smem, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
                 "r"(bytes)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_all() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

struct BinCfg {
    uint32_t* bins;         // nregions x cap offsets (words within the region)
    uint32_t* count;        // reserved entries per region (may exceed cap: overflow applied directly)
    uint32_t nregions;
    uint32_t cap;
    uint32_t region_shift;  // log2(words per region)
    uint32_t nib;           // linear recorders packed two per byte (nibble.cuh)
    uint32_t no_direct;     // a bin overflow sets *overflow instead of marking the table directly
    uint32_t* overflow;
    uint32_t pack;          // region << region_shift | offset fits 32 bits (tables of <= 2^32 words)
    uint32_t dedup;         // drop marks this block staged before (needs pack; see k_scan_bin)
    uint32_t* seen_ovf;     // set when a bin overflowed (the engine then turns dedup on)
    uint32_t ab_nohoist;    // A/B (SRLA_K1_HOIST=0): the filter's branch inside the mark loop
};

constexpr int kBinThreads = 512;
constexpr int kBinPerThread = 4;                            // packets per thread per tile
constexpr int kBinTile = kBinThreads * kBinPerThread;       // packets per tile
constexpr int kBinRows = 4;                                 // rows handled by the binned path
constexpr int kBinEntries = kBinTile * kBinRows;
constexpr int kMaxRegions = 4096;
// duplicate-mark filter: a direct-mapped cache of 2^kDedupBits mark words per block
constexpr int kDedupBits = 13;
// k_scan_bin dynamic shared memory for `nregions` regions (2 blocks per SM up to kMaxRegions)
constexpr int bin_smem(uint32_t nregions, uint32_t dedup = 1) {
    return static_cast<int>(nregions) * 16 + kBinEntries * 6 + (dedup ? (4 << kDedupBits) : 0);
}

// Epoch-stamp mode of the linear table (epoch.cuh): marks write the current
// epoch instead of 0 and keep per-row stamp histograms.
struct EpochCfg {
    uint32_t on;
    uint32_t cur;
    unsigned long long* hist;  // rows x 256
    uint64_t row_words;
};

// set byte `off` of the 32-bit-aligned table to `cur`; returns the old byte
__device__ __forceinline__ uint32_t stamp_byte_global(uint8_t* base, uint64_t off, uint32_t cur) {
    unsigned int* w = reinterpret_cast<unsigned int*>(base + (off & ~3ull));
    const uint32_t sh = 8u * static_cast<uint32_t>(off & 3u);
    unsigned int old = *w, assumed;
    do {
        assumed = old;
        if (((assumed >> sh) & 0xFFu) == cur) return cur;
        old = atomicCAS(w, assumed, (assumed & ~(0xFFu << sh)) | (cur << sh));
    } while (old != assumed);
    return (old >> sh) & 0xFFu;
}

// Overflow path (bin full): stamp directly in HBM and account the histogram.
__device__ __forceinline__ void mark_epoch_global(uint8_t* lin, uint64_t word, uint64_t row_words, uint32_t cur,
                                                  unsigned long long* hist) {
    const uint32_t old = stamp_byte_global(lin, word, cur);
    if (old != cur) {
        unsigned long long* h = hist + (word / row_words) * 256;
        atomicAdd(h + old, ~0ull);  // -1
        atomicAdd(h + cur, 1ull);
    }
}

// "store 0" into packed recorder w (two per byte, low nibble for even w)
__device__ __forceinline__ void mark_nibble_global(uint8_t* lin, uint64_t w) {
    atomicAnd(reinterpret_cast<unsigned int*>(lin + ((w >> 1) & ~3ull)), ~(0xFu << (4u * static_cast<uint32_t>(w & 7u))));
}

// "store 0" into one recorder word (recorder_mark) as a 32-bit AND, which the
// L2 executes ~1.6x faster than a byte store.
template <typename W>
__device__ __forceinline__ void mark_word(W* base, uint32_t off) {
    if constexpr (sizeof(W) == 1) {
        atomicAnd(reinterpret_cast<unsigned int*>(base + (off & ~3u)), ~(0xFFu << (8u * (off & 3u))));
    } else if constexpr (sizeof(W) == 2) {
        atomicAnd(reinterpret_cast<unsigned int*>(base + (off & ~1u)), ~(0xFFFFu << (16u * (off & 1u))));
    } else {
        base[off] = W(0);
    }
}

// K1 (binned): per record the u column hashes and the sample hash; linear
// marks are binned by region; sampled packets stamp their rough entries and
// append events exactly as k_scan does.
//
// ROWS = 4 (the configs of BASELINE.json) fixes the row loop at compile time;
// ROWS = 0 reads c.rows (<= kBinRows). Tiles where every thread has its four
// records take a path without per-record liveness tests.
template <typename W, int ROWS>
__global__ void __launch_bounds__(kBinThreads, 2) k_scan_bin(const uint32_t* __restrict__ recs, uint32_t n, DevCfg c,
                                                         BinCfg b, EpochCfg ep, W* __restrict__ lin,
                                                         uint32_t* __restrict__ stamp, uint32_t* __restrict__ ev,
                                                         uint32_t ev_cap, uint32_t* __restrict__ ev_count, int vec) {
    // dynamic shared memory (bin_smem(nregions, dedup) bytes):
    //   win[nregions] (uint2) | cnt[nregions] | lbase[nregions] | off[kBinEntries] | reg[kBinEntries] (u16)
    //   | seen[2^kDedupBits]
    // win: per region {bin slot of staging entry idx = x + idx (mod 2^32; nregions * cap < 2^32),
    //                  first staging index that no longer fits the region's bin}
    extern __shared__ __align__(16) uint8_t s_bin_raw[];
    uint2* s_win = reinterpret_cast<uint2*>(s_bin_raw);
    uint32_t* s_cnt = reinterpret_cast<uint32_t*>(s_win + b.nregions);
    uint32_t* s_lbase = s_cnt + b.nregions;
    uint32_t* s_off = s_lbase + b.nregions;
    uint16_t* s_reg = reinterpret_cast<uint16_t*>(s_off + kBinEntries);
    // Duplicate marks (same recorder word) are idempotent: with b.dedup a
    // mark whose word this block staged earlier in the launch is dropped
    // (adversarial skew: one host's 1e7 packets per slice hit the same 4
    // cells and would overflow their region bins). The cache only ever holds
    // words already staged, so a dropped mark is applied by its twin.
    uint32_t* s_seen = reinterpret_cast<uint32_t*>(s_reg + kBinEntries);
    __shared__ uint32_t s_warp[kBinThreads / 32];
    if (b.dedup)
        for (uint32_t q = threadIdx.x; q < (1u << kDedupBits); q += kBinThreads) s_seen[q] = 0xFFFFFFFFu;

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    const uint32_t rmask = (1u << b.region_shift) - 1u;
    const uint32_t ntiles = (n + kBinTile - 1) / kBinTile;
    const uint32_t regs_per_thread = (b.nregions + kBinThreads - 1) / kBinThreads;
    for (uint32_t r = tid; r < b.nregions; r += kBinThreads) s_cnt[r] = 0;
    __syncthreads();

    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        // s_cnt is zero here: cleared before the loop and by each region's
        // owner thread once it has read the count (below)
        const uint32_t base = tile * kBinTile + tid * kBinPerThread;
        uint32_t src[kBinPerThread], dst[kBinPerThread];
        uint32_t valid = 0;
        if (base < n) {
            if (vec && base + kBinPerThread <= n) {  // 4 records = three 16-byte vectors
                const uint4* q = reinterpret_cast<const uint4*>(recs + 3ull * base);
                const uint4 x = __ldcs(q), y = __ldcs(q + 1), z = __ldcs(q + 2);
                src[0] = x.y; dst[0] = x.z;
                src[1] = y.x; dst[1] = y.y;
                src[2] = y.w; dst[2] = z.x;
                src[3] = z.z; dst[3] = z.w;
                valid = kBinPerThread;
            } else {
                valid = min(static_cast<uint32_t>(kBinPerThread), n - base);
                for (uint32_t q = 0; q < kBinPerThread; ++q) {
                    src[q] = q < valid ? __ldcs(recs + 3ull * (base + q) + 1) : 0u;
                    dst[q] = q < valid ? __ldcs(recs + 3ull * (base + q) + 2) : 0u;
                }
            }
        }
        // per mark: offset in its region, and (region << 16 | rank in the tile's
        // region bucket); 0xFFFFFFFF = no mark (dead record or row)
        uint32_t off[kBinPerThread][kBinRows], rr[kBinPerThread][kBinRows];
        uint32_t smask = 0, rsl[kBinPerThread];
        const uint32_t nrows = ROWS ? static_cast<uint32_t>(ROWS) : c.rows;
        auto place = [&](auto full_tag, auto dedup_tag) {
            constexpr bool kFull = decltype(full_tag)::value;
            constexpr bool kDedup = decltype(dedup_tag)::value;
#pragma unroll
            for (uint32_t q = 0; q < kBinPerThread; ++q) {
                rsl[q] = 0;
                const bool live = kFull || q < valid;
                const uint32_t sample = hash_u32k(c.sub_sample, c.kh_sample, dst[q]);
                const uint32_t lslot = c.gl_mask ? (sample & c.gl_mask) : (sample % c.gl);
                uint32_t cols[kBinRows];
#pragma unroll
                for (int i = 0; i < kBinRows; ++i) {
                    rr[q][i] = 0xFFFFFFFFu;
                    if (live && (ROWS ? i < ROWS : static_cast<uint32_t>(i) < nrows)) {
                        const uint32_t col = column_of(c, i, src[q]);
                        cols[i] = col;
                        const uint64_t w = i * lrow + static_cast<uint64_t>(col) * c.gl + lslot;
                        const uint32_t r = static_cast<uint32_t>(w >> b.region_shift);
                        off[q][i] = static_cast<uint32_t>(w) & rmask;
                        bool dup = false;
                        if (kDedup && b.dedup) {  // w < 2^32 (pack)
                            const uint32_t key = static_cast<uint32_t>(w);
                            uint32_t* slot = s_seen + ((key * 0x9E3779B1u) >> (32 - kDedupBits));
                            dup = *slot == key;
                            if (!dup) *slot = key;
                        }
                        if (!kDedup || !dup) rr[q][i] = (r << 16) | atomicAdd(&s_cnt[r], 1u);
                    }
                }
                if (live && (sample & c.tau_mask) == 0u) {  // sampled (1 in 2^tau): rough stamps
                    const uint32_t rslot = reduce32(hash_u32k(c.sub_rslot, c.kh_rslot, dst[q]), c.g);
                    for (uint32_t i = 0; i < nrows; ++i)
                        atomicMin(stamp + i * rrow + static_cast<uint64_t>(cols[i < kBinRows ? i : 0]) * c.g + rslot,
                                  base + q);
                    smask |= 1u << q;
                    rsl[q] = rslot;
                }
            }
        };
        // the filter's branch hoisted out of the mark loop (it is off unless bins overflowed)
        if (b.dedup || b.ab_nohoist) {
            if (valid == kBinPerThread) place(std::true_type{}, std::true_type{});
            else place(std::false_type{}, std::true_type{});
        } else {
            if (valid == kBinPerThread) place(std::true_type{}, std::false_type{});
            else place(std::false_type{}, std::false_type{});
        }
        if (__any_sync(0xFFFFFFFFu, smask != 0)) {
            uint32_t pos = warp_append(ev_count, __popc(smask));
#pragma unroll
            for (uint32_t q = 0; q < kBinPerThread; ++q) {
                if (smask & (1u << q)) {
                    if (pos < ev_cap) {
                        ev[pos] = base + q;
                        ev[ev_cap + pos] = src[q];
                        ev[2ull * ev_cap + pos] = rsl[q];
                    }
                    ++pos;
                }
            }
        }
        __syncthreads();

        // exclusive scan of the region counts (each thread owns a run of regions)
        uint32_t mine = 0;
        const uint32_t r0 = tid * regs_per_thread;
        for (uint32_t r = r0; r < min(r0 + regs_per_thread, b.nregions); ++r) mine += s_cnt[r];
        uint32_t incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= static_cast<uint32_t>(o)) incl += t;
        }
        if (lane == 31) s_warp[warp] = incl;
        __syncthreads();
        uint32_t wbase = 0;
        for (uint32_t w2 = 0; w2 < warp; ++w2) wbase += s_warp[w2];
        uint32_t run = wbase + incl - mine;
        // Each region's global bin reservation is issued here and its window
        // stored only after the scatter below, which hides the atomic's round
        // trip (owners of <= 2 regions; more regions per thread store at once).
        // The owner clears its counts for the next tile once read.
        constexpr int kDefer = 2;
        uint32_t dg[kDefer], dcn[kDefer], dlb[kDefer];
        const bool defer = regs_per_thread <= static_cast<uint32_t>(kDefer);
        if (defer) {
#pragma unroll
            for (int j = 0; j < kDefer; ++j) {
                const uint32_t r = r0 + j;
                dcn[j] = 0;
                if (static_cast<uint32_t>(j) < regs_per_thread && r < b.nregions) {
                    const uint32_t cn = s_cnt[r];
                    s_cnt[r] = 0;
                    s_lbase[r] = run;
                    dlb[j] = run;
                    dcn[j] = cn;
                    if (cn) dg[j] = atomicAdd(b.count + r, cn);
                    run += cn;
                }
            }
        } else {
            for (uint32_t r = r0; r < min(r0 + regs_per_thread, b.nregions); ++r) {
                const uint32_t cn = s_cnt[r];
                s_cnt[r] = 0;
                s_lbase[r] = run;
                if (cn) {
                    const uint32_t g = atomicAdd(b.count + r, cn);
                    const uint32_t fit = g >= b.cap ? 0u : min(cn, b.cap - g);
                    s_win[r] = make_uint2(r * b.cap + g - run, run + fit);
                }
                run += cn;
            }
        }
        uint32_t total = 0;
        for (uint32_t w2 = 0; w2 < kBinThreads / 32; ++w2) total += s_warp[w2];
        __syncthreads();

        // branch-free when every mark of the tile is staged (4 rows, full tile, no filter)
        auto scatter = [&](auto all_tag, auto pack_tag) {
            constexpr bool kAll = decltype(all_tag)::value;
            constexpr bool kPack = decltype(pack_tag)::value;
#pragma unroll
            for (uint32_t q = 0; q < kBinPerThread; ++q)
#pragma unroll
                for (int i = 0; i < kBinRows; ++i)
                    if (kAll || rr[q][i] != 0xFFFFFFFFu) {
                        const uint32_t reg = rr[q][i] >> 16;
                        const uint32_t p = s_lbase[reg] + (rr[q][i] & 0xFFFFu);
                        if constexpr (kPack) {  // region and offset in one word: the write pass loads one value
                            s_off[p] = (reg << b.region_shift) | off[q][i];
                        } else {
                            s_off[p] = off[q][i];
                            s_reg[p] = static_cast<uint16_t>(reg);
                        }
                    }
        };
        const bool all_marks = ROWS == kBinRows && !b.dedup && !b.ab_nohoist &&
                               (tile + 1) * static_cast<uint64_t>(kBinTile) <= n;
        if (b.pack) {
            if (all_marks) scatter(std::true_type{}, std::true_type{});
            else scatter(std::false_type{}, std::true_type{});
        } else {
            if (all_marks) scatter(std::true_type{}, std::false_type{});
            else scatter(std::false_type{}, std::false_type{});
        }
        if (defer) {
#pragma unroll
            for (int j = 0; j < kDefer; ++j)
                if (dcn[j]) {
                    const uint32_t r = r0 + j, g = dg[j], cn = dcn[j];
                    const uint32_t fit = g >= b.cap ? 0u : min(cn, b.cap - g);
                    s_win[r] = make_uint2(r * b.cap + g - dlb[j], dlb[j] + fit);
                }
        }
        __syncthreads();

        // coalesced bin writes: consecutive staging entries of a region go to
        // consecutive bin slots
        // four entries per thread per round, every shared load before the
        // global stores (a generic-pointer store would otherwise order them)
        bool ovf = false;
        constexpr int kWU = 4;
        for (uint32_t idx0 = tid; idx0 < total; idx0 += kWU * kBinThreads) {
            uint32_t v[kWU], r[kWU];
            uint2 wv[kWU];
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
                const uint32_t idx = idx0 + u * kBinThreads;
                v[u] = idx < total ? s_off[idx] : 0u;
                if (b.pack) {
                    r[u] = v[u] >> b.region_shift;
                    v[u] &= rmask;
                } else {
                    r[u] = idx < total ? s_reg[idx] : 0u;
                }
            }
#pragma unroll
            for (int u = 0; u < kWU; ++u) wv[u] = s_win[r[u]];
#pragma unroll
            for (int u = 0; u < kWU; ++u) {
                const uint32_t idx = idx0 + u * kBinThreads;
                if (idx >= total) break;
                if (idx < wv[u].y) __stcg(b.bins + (wv[u].x + idx), v[u]);
                else ovf = true;
            }
        }
        if (__syncthreads_or(ovf)) {  // a bin is full: mark the rest directly (marks commute)
            if (tid == 0 && b.seen_ovf) atomicOr(b.seen_ovf, 1u);
            if (b.no_direct) {  // the table is busy elsewhere: the caller reruns this scan
                if (tid == 0) atomicOr(b.overflow, 1u);
                __syncthreads();
                continue;
            }
            for (uint32_t idx = tid; idx < total; idx += kBinThreads) {
                const uint32_t r = b.pack ? s_off[idx] >> b.region_shift : s_reg[idx];
                if (idx < s_win[r].y) continue;
                const uint32_t o = b.pack ? s_off[idx] & rmask : s_off[idx];
                if (ep.on)
                    mark_epoch_global(reinterpret_cast<uint8_t*>(lin), (static_cast<uint64_t>(r) << b.region_shift) + o,
                                      ep.row_words, ep.cur, ep.hist);
                else if (b.nib)
                    mark_nibble_global(reinterpret_cast<uint8_t*>(lin), (static_cast<uint64_t>(r) << b.region_shift) + o);
                else
                    mark_word<W>(lin + (static_cast<uint64_t>(r) << b.region_shift), o);
            }
            __syncthreads();
        }
    }
}

// Fused end-of-slice pass over a range of one linear row: optionally count
// the recorders active in the window (count_active, recorders.hpp:119-129)
// into counts[row], then age them (slide_recorders, recorders.hpp:113-116) in
// the same read+write.
template <typename W>
__global__ void __launch_bounds__(256) k_count_age(W* __restrict__ base, uint64_t words, uint32_t k,
                                                   uint32_t expired, int count,
                                                   unsigned long long* __restrict__ counter) {
    const uint32_t kk = sizeof(W) == 1 ? k * 0x01010101u : sizeof(W) == 2 ? k * 0x00010001u : k;
    const uint32_t ee = sizeof(W) == 1 ? expired * 0x01010101u : sizeof(W) == 2 ? expired * 0x00010001u : expired;
    const uint32_t one = sizeof(W) == 1 ? 0x01010101u : sizeof(W) == 2 ? 0x00010001u : 1u;
    unsigned long long acc = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t bytes = words * sizeof(W);
    auto age = [&](uint32_t x) -> uint32_t {
        if constexpr (sizeof(W) == 1) return __vadd4(x, __vcmpne4(x, ee) & one);
        else if constexpr (sizeof(W) == 2) return __vadd2(x, __vcmpne2(x, ee) & one);
        else return x + (x != ee ? 1u : 0u);
    };
    if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(base) & 15) == 0) {
        uint4* v = reinterpret_cast<uint4*>(base);
        const uint64_t nv = bytes / 16;
        for (uint64_t q = tid; q < nv; q += stride) {
            uint4 x = v[q];
            if (count)
                acc += count_lt_word<W>(x.x, kk, k) + count_lt_word<W>(x.y, kk, k) + count_lt_word<W>(x.z, kk, k) +
                       count_lt_word<W>(x.w, kk, k);
            x.x = age(x.x);
            x.y = age(x.y);
            x.z = age(x.z);
            x.w = age(x.w);
            v[q] = x;
        }
        if constexpr (sizeof(W) == 1) acc >>= 3;
        else if constexpr (sizeof(W) == 2) acc >>= 4;
    } else {
        for (uint64_t q = tid; q < words; q += stride) {
            const W x = base[q];
            acc += static_cast<uint32_t>(x) < k;
            base[q] = static_cast<W>(x + (static_cast<uint32_t>(x) != expired ? 1 : 0));
        }
    }
    if (!count) return;
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ unsigned long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += part[w];
        if (s) atomicAdd(counter, s);
    }
}

}  // namespace srla

namespace srla {

// ----------------------------------------------------------------------------
// Two-level apply: coarse region bins -> fine 64 KB slices -> shared memory.
//
// k_split re-bins each region's marks by 64 KB table slice (u16 offsets, one
// block-level multi-split per 4096 entries); k_slice_apply then gives every
// slice to one block, which loads it into shared memory with 16-byte coalesced
// loads, applies its marks there, optionally counts active recorders and ages
// them (the end-of-slice work), and writes the slice back coalesced. The table
// is streamed once at full bandwidth instead of fetched one sector at a time.

struct FineCfg {
    uint16_t* bins;       // nfine x cap
    uint32_t* count;      // per fine slice
    uint32_t cap;
    uint32_t shift;       // log2(words per fine slice)
    uint32_t per_region;  // fine slices per coarse region = 2^(region_shift - shift)
    uint32_t nfine;       // total fine slices covering the table
    unsigned long long* streamed;  // table bytes read (= written) by the apply kernels (statistics)
    uint32_t nib;                  // linear recorders packed two per byte (nibble.cuh)
};

constexpr int kSplitThreads = 512;  // default block; 1024 for fan-outs >= 1024 (Engine::setup_bins)
constexpr int kSplitPerThread = 16;
constexpr int kSplitTile = kSplitThreads * kSplitPerThread;  // 8192 entries
template <int T>
constexpr int split_tile_entries() { return T * kSplitPerThread; }

// One k_split tile: the n entries of region r staged at s_sorted (loaded
// there; sorted in place) -> fine-slice bins. s_cnt must be zero on entry.
// Ends with a block barrier.
template <typename W, int T>
__device__ __forceinline__ void split_tile(uint32_t* s_sorted, uint32_t r, uint32_t n, uint32_t* s_cnt,
                                           uint32_t* s_lbase, uint2* s_win, uint32_t* s_warp,
                                           uint32_t region_shift, const FineCfg& f, const EpochCfg& ep,
                                           W* __restrict__ lin) {
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint32_t fmask = (1u << f.shift) - 1u;
    const uint32_t per_thread = (f.per_region + T - 1) / T;
    uint32_t off[kSplitPerThread];
    // entries 4 * (q * T + tid) .. + 3: consecutive lanes read consecutive
    // 16-byte vectors (no bank conflicts); which thread ranks an entry is free
    const uint4* v = reinterpret_cast<const uint4*>(s_sorted);
#pragma unroll
    for (int q = 0; q < kSplitPerThread / 4; ++q) {
        const uint32_t e0 = 4u * (q * T + tid);
        const uint4 x = v[q * T + tid];
        off[4 * q] = e0 < n ? x.x : 0xFFFFFFFFu;
        off[4 * q + 1] = e0 + 1 < n ? x.y : 0xFFFFFFFFu;
        off[4 * q + 2] = e0 + 2 < n ? x.z : 0xFFFFFFFFu;
        off[4 * q + 3] = e0 + 3 < n ? x.w : 0xFFFFFFFFu;
    }
    // full tiles (all but a region's last) rank and scatter without per-entry tests
    const bool full = n == static_cast<uint32_t>(T * kSplitPerThread);
    uint32_t rank[kSplitPerThread];
    if (full) {
#pragma unroll
        for (int k = 0; k < kSplitPerThread; ++k) rank[k] = atomicAdd(&s_cnt[off[k] >> f.shift], 1u);
    } else {
#pragma unroll
        for (int k = 0; k < kSplitPerThread; ++k)
            if (off[k] != 0xFFFFFFFFu) rank[k] = atomicAdd(&s_cnt[off[k] >> f.shift], 1u);
    }
    __syncthreads();
    uint32_t mine = 0;
    const uint32_t b0 = tid * per_thread;
    for (uint32_t b = b0; b < min(b0 + per_thread, f.per_region); ++b) mine += s_cnt[b];
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += v;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    uint32_t run = incl - mine;
    for (uint32_t w2 = 0; w2 < warp; ++w2) run += s_warp[w2];
    const uint32_t fine0 = r * f.per_region;
    for (uint32_t b = b0; b < min(b0 + per_thread, f.per_region); ++b) {
        const uint32_t cn = s_cnt[b];
        s_lbase[b] = run;
        if (cn) {
            const uint32_t g = atomicAdd(f.count + fine0 + b, cn);
            const uint32_t fit = g >= f.cap ? 0u : min(cn, f.cap - g);
            s_win[b] = make_uint2((fine0 + b) * f.cap + g - run, run + fit);
        }
        run += cn;
    }
    __syncthreads();
    if (full) {
#pragma unroll
        for (int k = 0; k < kSplitPerThread; ++k) {
            const uint32_t b = off[k] >> f.shift;
            s_sorted[s_lbase[b] + rank[k]] = (b << 16) | (off[k] & fmask);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kSplitPerThread; ++k)
            if (off[k] != 0xFFFFFFFFu) {
                const uint32_t b = off[k] >> f.shift;
                s_sorted[s_lbase[b] + rank[k]] = (b << 16) | (off[k] & fmask);
            }
    }
    __syncthreads();
    bool ovf = false;
    for (uint32_t i = tid; i < n; i += T) {
        const uint32_t v = s_sorted[i];
        const uint2 wv = s_win[v >> 16];
        if (i < wv.y) f.bins[wv.x + i] = static_cast<uint16_t>(v);
        else ovf = true;
    }
    if (__syncthreads_or(ovf)) {  // a fine bin is full: mark in place (marks commute)
        for (uint32_t i = tid; i < n; i += T) {
            const uint32_t v = s_sorted[i];
            const uint32_t b = v >> 16;
            if (i < s_win[b].y) continue;
            if (ep.on)
                mark_epoch_global(reinterpret_cast<uint8_t*>(lin),
                                  (static_cast<uint64_t>(r) << region_shift) + (static_cast<uint64_t>(b) << f.shift) +
                                      (v & 0xFFFFu),
                                  ep.row_words, ep.cur, ep.hist);
            else if (f.nib)
                mark_nibble_global(reinterpret_cast<uint8_t*>(lin), (static_cast<uint64_t>(r) << region_shift) +
                                                                        (static_cast<uint64_t>(b) << f.shift) + (v & 0xFFFFu));
            else
                mark_word<W>(lin + (static_cast<uint64_t>(r) << region_shift) + (static_cast<uint64_t>(b) << f.shift),
                             v & 0xFFFFu);
        }
    }
    __syncthreads();
}

// Re-bin coarse region bins by fine slice. One tile = 8192 consecutive entries
// of one region: shared-memory counting sort by slice (ranks from shared
// atomics), one global reservation per slice per tile, coalesced u16 writes.
template <typename W, int T>
__global__ void __launch_bounds__(T, 1024 / T) k_split(const uint32_t* __restrict__ coarse, uint32_t coarse_cap,
                                                         const uint32_t* __restrict__ tile_prefix,
                                                         const uint32_t* __restrict__ coarse_n, uint32_t nregions,
                                                         uint32_t region_shift, FineCfg f, EpochCfg ep,
                                                         W* __restrict__ lin) {
    // dynamic shared memory, sized by the fan-out f.per_region (<= 4096):
    //   stage[2][T * kSplitPerThread] | cnt[P] | lbase[P] | win[P] (uint2)
    // A tile's entries are bulk-loaded into its stage while the block sorts
    // the previous tile (the coarse bins have >= 16 bytes of slack at the end);
    // once read into registers, the stage holds the tile's sorted entries.
    constexpr uint32_t kTile = split_tile_entries<T>();
    extern __shared__ __align__(128) uint32_t s_dyn[];
    uint32_t* s_stage = s_dyn;
    uint32_t* s_cnt = s_dyn + 2 * kTile;
    uint32_t* s_lbase = s_cnt + f.per_region;
    // per fine slice: {bin slot of sorted entry i = x + i (mod 2^32; nfine * cap < 2^32 by
    // construction, Engine::setup_bins), first sorted index that no longer fits its bin}
    uint2* s_win = reinterpret_cast<uint2*>(s_lbase + f.per_region);
    __shared__ uint32_t s_warp[T / 32];
    __shared__ uint32_t s_region[2], s_n[2];
    __shared__ __align__(8) uint64_t s_bar[2];
    const uint32_t tid = threadIdx.x;
    const uint32_t total_tiles = tile_prefix[nregions];
    // thread 0: locate tile t (region r with tile_prefix[r] <= t < tile_prefix[r+1]) and load it
    auto issue = [&](uint32_t t, uint32_t b) {
        uint32_t lo = 0, hi = nregions;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (tile_prefix[mid] <= t) lo = mid;
            else hi = mid;
        }
        const uint32_t begin = (t - tile_prefix[lo]) * kTile;
        const uint32_t n = min(coarse_n[lo] - begin, kTile);
        s_region[b] = lo;
        s_n[b] = n;
        const uint32_t bytes = (n * 4u + 15u) & ~15u;
        mbar_expect_tx(&s_bar[b], bytes);
        bulk_load(s_stage + b * kTile, coarse + static_cast<uint64_t>(lo) * coarse_cap + begin, bytes, &s_bar[b]);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    __syncthreads();
    if (tid == 0 && blockIdx.x < total_tiles) issue(blockIdx.x, 0);
    uint32_t it = 0;
    for (uint32_t t = blockIdx.x; t < total_tiles; t += gridDim.x, ++it) {
        const uint32_t sb = it & 1u;
        // the other stage was last read by the previous tile, finished at its final barrier
        if (tid == 0 && t + gridDim.x < total_tiles) issue(t + gridDim.x, sb ^ 1u);
        for (uint32_t i = tid; i < f.per_region; i += T) s_cnt[i] = 0;
        mbar_wait(&s_bar[sb], (it >> 1) & 1u);
        __syncthreads();
        const uint32_t r = s_region[sb];
        const uint32_t n = s_n[sb];
        split_tile<W, T>(s_stage + sb * kTile, r, n, s_cnt, s_lbase, s_win, s_warp, region_shift, f, ep, lin);
    }
}

// k_split's tile table on the device (no host round trip): per region the
// clamped entry count n_r = min(count, cap) (overflow was marked directly)
// and the exclusive prefix of its `tile`-entry tiles; prefix[R] = total
// tiles, which k_split reads. Out: prefix[0..R], n_r at prefix + R + 1.
__global__ void __launch_bounds__(1024) k_split_prefix(const uint32_t* __restrict__ count, uint32_t nregions,
                                                       uint32_t cap, uint32_t tile, uint32_t* __restrict__ prefix) {
    __shared__ uint32_t s_w[32];
    const uint32_t per = (nregions + 1023) / 1024;  // regions per thread (nregions <= kMaxRegions)
    const uint32_t r0 = threadIdx.x * per;
    uint32_t mine = 0;
    for (uint32_t r = r0; r < min(r0 + per, nregions); ++r) mine += (min(count[r], cap) + tile - 1) / tile;
    uint32_t incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((threadIdx.x & 31) >= static_cast<uint32_t>(o)) incl += t;
    }
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint32_t run = incl - mine;
    for (uint32_t j = 0; j < (threadIdx.x >> 5); ++j) run += s_w[j];
    for (uint32_t r = r0; r < min(r0 + per, nregions); ++r) {
        const uint32_t n = min(count[r], cap);
        prefix[r] = run;
        prefix[nregions + 1 + r] = n;
        run += (n + tile - 1) / tile;
    }
    if (threadIdx.x == 1023) prefix[nregions] = run;
}

// mode 0: apply marks (slices without marks are skipped); 1: apply + age;
// 2: apply + count active (counts[row], pre-age) + age.
template <typename W>
__global__ void __launch_bounds__(256) k_slice_apply(W* __restrict__ lin, uint64_t total_words, uint64_t row_words,
                                                     FineCfg f, uint32_t f_begin, int mode, uint32_t k,
                                                     uint32_t expired, unsigned long long* __restrict__ counts) {
    extern __shared__ uint4 s_slice[];
    W* sw = reinterpret_cast<W*>(s_slice);
    const uint32_t tid = threadIdx.x;
    const uint32_t kk = sizeof(W) == 1 ? k * 0x01010101u : sizeof(W) == 2 ? k * 0x00010001u : k;
    const uint32_t ee = sizeof(W) == 1 ? expired * 0x01010101u : sizeof(W) == 2 ? expired * 0x00010001u : expired;
    const uint32_t one = sizeof(W) == 1 ? 0x01010101u : sizeof(W) == 2 ? 0x00010001u : 1u;
    auto age = [&](uint32_t x) -> uint32_t {
        if constexpr (sizeof(W) == 1) return __vadd4(x, __vcmpne4(x, ee) & one);
        else if constexpr (sizeof(W) == 2) return __vadd2(x, __vcmpne2(x, ee) & one);
        else return x + (x != ee ? 1u : 0u);
    };
    __shared__ unsigned long long s_part[8];
    // 16-byte vectors only when slices and rows are 16-byte aligned
    const bool vec = ((row_words * sizeof(W)) & 15) == 0 && (((1ull << f.shift) * sizeof(W)) & 15) == 0;
    for (uint32_t fb = f_begin + blockIdx.x; fb < f.nfine; fb += gridDim.x) {
        const uint32_t n = min(f.count[fb], f.cap);
        if (mode == 0 && n == 0) continue;
        const uint64_t w0 = static_cast<uint64_t>(fb) << f.shift;
        const uint32_t nw = static_cast<uint32_t>(min(static_cast<uint64_t>(1u << f.shift), total_words - w0));
        if (tid == 0) atomicAdd(f.streamed, static_cast<unsigned long long>(nw) * sizeof(W));
        const uint32_t nv = vec ? static_cast<uint32_t>((static_cast<uint64_t>(nw) * sizeof(W)) / 16) : 0u;
        const uint32_t tail0 = nv * 16 / sizeof(W);
        uint4* g = reinterpret_cast<uint4*>(lin + w0);
        for (uint32_t q = tid; q < nv; q += blockDim.x) s_slice[q] = __ldcs(g + q);
        for (uint32_t q = tail0 + tid; q < nw; q += blockDim.x) sw[q] = lin[w0 + q];
        __syncthreads();
        const uint16_t* e = f.bins + static_cast<uint64_t>(fb) * f.cap;
        for (uint32_t i = tid; i < n; i += blockDim.x) sw[__ldcs(e + i)] = W(0);
        __syncthreads();
        if (mode == 0) {
            for (uint32_t q = tid; q < nv; q += blockDim.x) __stcs(g + q, s_slice[q]);
            for (uint32_t q = tail0 + tid; q < nw; q += blockDim.x) lin[w0 + q] = sw[q];
            __syncthreads();
            continue;
        }
        const uint64_t row_a = w0 / row_words, row_b = (w0 + nw - 1) / row_words;
        unsigned long long acc_a = 0, acc_b = 0;
        for (uint32_t q = tid; q < nv; q += blockDim.x) {
            uint4 x = s_slice[q];
            if (mode == 2) {
                const uint32_t c = count_lt_word<W>(x.x, kk, k) + count_lt_word<W>(x.y, kk, k) +
                                   count_lt_word<W>(x.z, kk, k) + count_lt_word<W>(x.w, kk, k);
                if (row_a == row_b || (w0 + static_cast<uint64_t>(q) * 16 / sizeof(W)) / row_words == row_a) acc_a += c;
                else acc_b += c;  // a 16-byte vector never straddles rows when row bytes % 16 == 0
            }
            x.x = age(x.x);
            x.y = age(x.y);
            x.z = age(x.z);
            x.w = age(x.w);
            __stcs(g + q, x);
        }
        if constexpr (sizeof(W) == 1) {
            acc_a >>= 3;
            acc_b >>= 3;
        } else if constexpr (sizeof(W) == 2) {
            acc_a >>= 4;
            acc_b >>= 4;
        }
        for (uint32_t q = tail0 + tid; q < nw; q += blockDim.x) {
            const W x = sw[q];
            if (mode == 2 && static_cast<uint32_t>(x) < k) ((w0 + q) / row_words == row_a ? acc_a : acc_b) += 1;
            lin[w0 + q] = static_cast<W>(x + (static_cast<uint32_t>(x) != expired ? 1 : 0));
        }
        if (mode == 2) {
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                acc_a += __shfl_xor_sync(0xFFFFFFFFu, acc_a, o);
                acc_b += __shfl_xor_sync(0xFFFFFFFFu, acc_b, o);
            }
            if ((tid & 31) == 0) s_part[tid >> 5] = acc_a;
            __syncthreads();
            if (tid == 0) {
                unsigned long long s = 0;
                for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += s_part[w];
                if (s) atomicAdd(counts + row_a, s);
            }
            __syncthreads();
            if ((tid & 31) == 0) s_part[tid >> 5] = acc_b;
            __syncthreads();
            if (tid == 0) {
                unsigned long long s = 0;
                for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += s_part[w];
                if (s) atomicAdd(counts + row_b, s);
            }
        }
        __syncthreads();
    }
}

}  // namespace srla

namespace srla {

// Same contract as k_slice_apply for slices [f_begin, f_end) whose bytes are
// a multiple of 16 and 16-byte aligned (and rows are 16-byte multiples):
// each block walks its slices through two shared-memory buffers; slice i+1 is
// bulk-loaded while slice i is marked, counted and aged, and each finished
// slice is bulk-stored back — the table streams through HBM once.
template <typename W>
__global__ void __launch_bounds__(256) k_slice_apply_bulk(W* __restrict__ lin, uint64_t row_words, FineCfg f,
                                                          uint32_t f_end, int mode, uint32_t k, uint32_t expired,
                                                          unsigned long long* __restrict__ counts) {
    extern __shared__ __align__(128) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ unsigned long long s_part[2][8];
    const uint32_t tid = threadIdx.x;
    const uint32_t slice_bytes = (1u << f.shift) * sizeof(W);
    uint8_t* buf[2] = {s_raw, s_raw + slice_bytes};
    const uint32_t kk = sizeof(W) == 1 ? k * 0x01010101u : sizeof(W) == 2 ? k * 0x00010001u : k;
    const uint32_t ee = sizeof(W) == 1 ? expired * 0x01010101u : sizeof(W) == 2 ? expired * 0x00010001u : expired;
    const uint32_t one = sizeof(W) == 1 ? 0x01010101u : sizeof(W) == 2 ? 0x00010001u : 1u;
    auto age = [&](uint32_t x) -> uint32_t {
        if constexpr (sizeof(W) == 1) return __vadd4(x, __vcmpne4(x, ee) & one);
        else if constexpr (sizeof(W) == 2) return __vadd2(x, __vcmpne2(x, ee) & one);
        else return x + (x != ee ? 1u : 0u);
    };
    // slices of this block: blockIdx.x + j*gridDim.x, skipping mark-free ones in mode 0
    auto next_slice = [&](uint32_t from) -> uint32_t {
        for (uint32_t fb = from; fb < f_end; fb += gridDim.x)
            if (mode != 0 || f.count[fb] != 0) return fb;
        return f_end;
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    __syncthreads();
    uint32_t cur = next_slice(blockIdx.x);
    if (tid == 0 && cur < f_end) {
        mbar_expect_tx(&s_bar[0], slice_bytes);
        bulk_load(buf[0], lin + (static_cast<uint64_t>(cur) << f.shift), slice_bytes, &s_bar[0]);
    }
    for (uint32_t i = 0; cur < f_end; ++i) {
        const uint32_t b = i & 1u;
        const uint32_t nxt = next_slice(cur + gridDim.x);
        if (tid == 0 && nxt < f_end) {
            bulk_wait_read_all();  // the other buffer's store (slice i-1) has left shared memory
            mbar_expect_tx(&s_bar[b ^ 1u], slice_bytes);
            bulk_load(buf[b ^ 1u], lin + (static_cast<uint64_t>(nxt) << f.shift), slice_bytes, &s_bar[b ^ 1u]);
        }
        mbar_wait(&s_bar[b], (i >> 1) & 1u);
        if (tid == 0) atomicAdd(f.streamed, static_cast<unsigned long long>(slice_bytes));
        W* sw = reinterpret_cast<W*>(buf[b]);
        const uint32_t n = min(f.count[cur], f.cap);
        const uint16_t* e = f.bins + static_cast<uint64_t>(cur) * f.cap;
        const uint4* ev = reinterpret_cast<const uint4*>(e);
        for (uint32_t q = tid; q < n / 8; q += blockDim.x) {
            const uint4 x = __ldcs(ev + q);
            sw[x.x & 0xFFFF] = W(0); sw[x.x >> 16] = W(0);
            sw[x.y & 0xFFFF] = W(0); sw[x.y >> 16] = W(0);
            sw[x.z & 0xFFFF] = W(0); sw[x.z >> 16] = W(0);
            sw[x.w & 0xFFFF] = W(0); sw[x.w >> 16] = W(0);
        }
        for (uint32_t q = (n / 8) * 8 + tid; q < n; q += blockDim.x) sw[e[q]] = W(0);
        __syncthreads();
        if (mode != 0) {
            const uint64_t w0 = static_cast<uint64_t>(cur) << f.shift;
            const uint64_t row_a = w0 / row_words;
            const uint64_t split = (row_a + 1) * row_words;  // first word of the next row
            unsigned long long acc_a = 0, acc_b = 0;
            uint4* sv = reinterpret_cast<uint4*>(buf[b]);
            const uint32_t nv = slice_bytes / 16;
            for (uint32_t q = tid; q < nv; q += blockDim.x) {
                uint4 x = sv[q];
                if (mode == 2) {
                    const uint32_t c = count_lt_word<W>(x.x, kk, k) + count_lt_word<W>(x.y, kk, k) +
                                       count_lt_word<W>(x.z, kk, k) + count_lt_word<W>(x.w, kk, k);
                    if (w0 + static_cast<uint64_t>(q) * (16 / sizeof(W)) < split) acc_a += c;
                    else acc_b += c;
                }
                x.x = age(x.x);
                x.y = age(x.y);
                x.z = age(x.z);
                x.w = age(x.w);
                sv[q] = x;
            }
            if (mode == 2) {
                if constexpr (sizeof(W) == 1) {
                    acc_a >>= 3;
                    acc_b >>= 3;
                } else if constexpr (sizeof(W) == 2) {
                    acc_a >>= 4;
                    acc_b >>= 4;
                }
#pragma unroll
                for (int o = 16; o; o >>= 1) {
                    acc_a += __shfl_xor_sync(0xFFFFFFFFu, acc_a, o);
                    acc_b += __shfl_xor_sync(0xFFFFFFFFu, acc_b, o);
                }
                if ((tid & 31) == 0) {
                    s_part[0][tid >> 5] = acc_a;
                    s_part[1][tid >> 5] = acc_b;
                }
            }
            fence_proxy_async_smem();
            __syncthreads();
            if (mode == 2 && tid == 0) {
                unsigned long long sa = 0, sb = 0;
                for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                    sa += s_part[0][w];
                    sb += s_part[1][w];
                }
                if (sa) atomicAdd(counts + row_a, sa);
                if (sb) atomicAdd(counts + row_a + 1, sb);
            }
        } else {
            fence_proxy_async_smem();
            __syncthreads();
        }
        if (tid == 0) bulk_store(lin + (static_cast<uint64_t>(cur) << f.shift), buf[b], slice_bytes);
        cur = nxt;
    }
    if (tid == 0) bulk_wait_all();
}

}  // namespace srla
