// scan_binned.cuh — the linear-mark path for tables larger than L2.
//
// Measured on B200 (tools/membench.cu, profiles/): scattered 1-byte stores into
// a 4 GiB table sustain ~23 G/s (every store is a DRAM sector read-modify-
// write), the same stores confined to an L2-resident 64 MB region ~129 G/s and
// 32-bit atomicAnd ~212 G/s. The linear marks of a slice (u per packet,
// store 0) commute with each other and with every other hot-path step except
// reads of the linear table, so K1 only *bins* them: a block multi-split by
// table region (64 MB slabs) with one global reservation per region per tile
// and coalesced bin writes. The apply pass then replays one region at a time
// while it is L2-resident, so each touched sector costs one DRAM read and one
// write per flush instead of one of each per mark. Any reader of the linear
// table flushes first (Engine::flush_linear).
#pragma once

#include "common.cuh"

namespace srla {

struct BinCfg {
    uint32_t* bins;         // nregions x cap offsets (words within the region)
    uint32_t* count;        // reserved entries per region (may exceed cap: overflow applied directly)
    uint32_t nregions;
    uint32_t cap;
    uint32_t region_shift;  // log2(words per region)
};

constexpr int kBinThreads = 256;
constexpr int kBinPerThread = 4;                            // packets per thread per tile
constexpr int kBinTile = kBinThreads * kBinPerThread;       // packets per tile
constexpr int kBinRows = 4;                                 // rows handled by the binned path
constexpr int kBinEntries = kBinTile * kBinRows;
constexpr int kMaxRegions = 1024;

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
template <typename W>
__global__ void __launch_bounds__(kBinThreads) k_scan_bin(const uint32_t* __restrict__ recs, uint32_t n, DevCfg c,
                                                         BinCfg b, W* __restrict__ lin,
                                                         uint32_t* __restrict__ stamp, uint32_t* __restrict__ ev,
                                                         uint32_t ev_cap, uint32_t* __restrict__ ev_count, int vec) {
    __shared__ uint32_t s_cnt[kMaxRegions];
    __shared__ uint32_t s_lbase[kMaxRegions];
    __shared__ uint32_t s_gbase[kMaxRegions];
    __shared__ uint32_t s_off[kBinEntries];
    __shared__ uint16_t s_reg[kBinEntries];
    __shared__ uint32_t s_warp[kBinThreads / 32];

    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    const uint32_t rmask = (1u << b.region_shift) - 1u;
    const uint32_t ntiles = (n + kBinTile - 1) / kBinTile;
    const uint32_t regs_per_thread = (b.nregions + kBinThreads - 1) / kBinThreads;

    for (uint32_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        for (uint32_t r = tid; r < b.nregions; r += kBinThreads) s_cnt[r] = 0;
        __syncthreads();

        const uint32_t base = tile * kBinTile + tid * kBinPerThread;
        uint32_t src[4], dst[4];
        uint32_t valid = 0;
        if (base < n) {
            if (vec && base + 4 <= n) {
                const uint4* q = reinterpret_cast<const uint4*>(recs + 3ull * base);
                const uint4 x = __ldcs(q), y = __ldcs(q + 1), z = __ldcs(q + 2);
                src[0] = x.y; dst[0] = x.z;
                src[1] = y.x; dst[1] = y.y;
                src[2] = y.w; dst[2] = z.x;
                src[3] = z.z; dst[3] = z.w;
                valid = 4;
            } else {
                valid = min(4u, n - base);
                for (uint32_t q = 0; q < 4; ++q) {
                    src[q] = q < valid ? __ldcs(recs + 3ull * (base + q) + 1) : 0u;
                    dst[q] = q < valid ? __ldcs(recs + 3ull * (base + q) + 2) : 0u;
                }
            }
        }
        uint32_t off[4][kBinRows], rank[4][kBinRows];
        uint16_t reg[4][kBinRows];
        uint32_t smask = 0, rsl[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            rsl[q] = 0;
            const bool live = q < valid;
            const uint32_t sample = hash_u32(c.sub_sample, dst[q]);
            const uint32_t lslot = c.gl_mask ? (sample & c.gl_mask) : (sample % c.gl);
            const bool smp = live && (sample & c.tau_mask) == 0u;
            const uint32_t rslot = smp ? reduce32(hash_u32(c.sub_rslot, dst[q]), c.g) : 0u;
#pragma unroll
            for (int i = 0; i < kBinRows; ++i) {
                reg[q][i] = 0xFFFF;
                const bool on = live && i < static_cast<int>(c.rows);
                if (on) {
                    const uint32_t col = column_of(c, i, src[q]);
                    const uint64_t w = i * lrow + static_cast<uint64_t>(col) * c.gl + lslot;
                    const uint32_t r = static_cast<uint32_t>(w >> b.region_shift);
                    reg[q][i] = static_cast<uint16_t>(r);
                    off[q][i] = static_cast<uint32_t>(w) & rmask;
                    rank[q][i] = atomicAdd(&s_cnt[r], 1u);  // slot within the tile's region bucket
                    if (smp) atomicMin(stamp + i * rrow + static_cast<uint64_t>(col) * c.g + rslot, base + q);
                }
            }
            if (smp) {
                smask |= 1u << q;
                rsl[q] = rslot;
            }
        }
        if (__any_sync(0xFFFFFFFFu, smask != 0)) {
            uint32_t pos = warp_append(ev_count, __popc(smask));
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) {
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
        for (uint32_t r = r0; r < min(r0 + regs_per_thread, b.nregions); ++r) {
            const uint32_t cn = s_cnt[r];
            s_lbase[r] = run;
            if (cn) s_gbase[r] = atomicAdd(b.count + r, cn);
            run += cn;
        }
        uint32_t total = 0;
        for (uint32_t w2 = 0; w2 < kBinThreads / 32; ++w2) total += s_warp[w2];
        __syncthreads();

#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
#pragma unroll
            for (int i = 0; i < kBinRows; ++i)
                if (reg[q][i] != 0xFFFF) {
                    const uint32_t p = s_lbase[reg[q][i]] + rank[q][i];
                    s_off[p] = off[q][i];
                    s_reg[p] = reg[q][i];
                }
        __syncthreads();

        for (uint32_t idx = tid; idx < total; idx += kBinThreads) {
            const uint32_t r = s_reg[idx];
            const uint32_t g = s_gbase[r] + (idx - s_lbase[r]);
            if (g < b.cap) {
                b.bins[static_cast<uint64_t>(r) * b.cap + g] = s_off[idx];
            } else {  // bin full: mark directly (marks commute)
                mark_word<W>(lin + (static_cast<uint64_t>(r) << b.region_shift), s_off[idx]);
            }
        }
        __syncthreads();
    }
}

// Stream `bytes` starting at p into L2 (TMA bulk prefetch, no registers).
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Prefetch [p, p+bytes) into L2, one 64 KB piece per thread of the grid
// (16-byte aligned pieces; the tail rounds down).
__device__ __forceinline__ void grid_prefetch_l2(const uint8_t* p, uint64_t bytes) {
    if (reinterpret_cast<uintptr_t>(p) & 15) return;  // bulk copies need 16-byte alignment
    const uint64_t piece = 64ull << 10;
    const uint64_t n = bytes / piece;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    for (uint64_t i = tid; i < n; i += stride) prefetch_l2(p + i * piece, static_cast<uint32_t>(piece));
    const uint64_t tail = (bytes - n * piece) & ~15ull;
    if (tid == 0 && tail) prefetch_l2(p + n * piece, static_cast<uint32_t>(tail));
}

// Apply one region's pending marks while the region is L2-resident; the
// region itself was prefetched by the previous launch, and this launch
// prefetches the next region (next/next_bytes) so its DRAM reads stream
// instead of missing one sector at a time.
template <typename W>
__global__ void __launch_bounds__(256) k_apply_bins(W* __restrict__ lin, const uint32_t* __restrict__ bins,
                                                    uint32_t cap, uint32_t region, uint32_t n, uint32_t shift,
                                                    const uint8_t* next, uint64_t next_bytes) {
    if (next) grid_prefetch_l2(next, next_bytes);
    W* base = lin + (static_cast<uint64_t>(region) << shift);
    const uint32_t* e = bins + static_cast<uint64_t>(region) * cap;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, stride = gridDim.x * blockDim.x;
    const uint32_t nv = n / 4;
    const uint4* v = reinterpret_cast<const uint4*>(e);
    uint32_t q = tid;
    for (; q + 3 * stride < nv; q += 4 * stride) {  // four 16-byte bin loads in flight per thread
        const uint4 a = __ldcs(v + q), b = __ldcs(v + q + stride), c = __ldcs(v + q + 2 * stride),
                    d = __ldcs(v + q + 3 * stride);
        mark_word<W>(base, a.x); mark_word<W>(base, a.y); mark_word<W>(base, a.z); mark_word<W>(base, a.w);
        mark_word<W>(base, b.x); mark_word<W>(base, b.y); mark_word<W>(base, b.z); mark_word<W>(base, b.w);
        mark_word<W>(base, c.x); mark_word<W>(base, c.y); mark_word<W>(base, c.z); mark_word<W>(base, c.w);
        mark_word<W>(base, d.x); mark_word<W>(base, d.y); mark_word<W>(base, d.z); mark_word<W>(base, d.w);
    }
    for (; q < nv; q += stride) {
        const uint4 x = __ldcs(v + q);
        mark_word<W>(base, x.x);
        mark_word<W>(base, x.y);
        mark_word<W>(base, x.z);
        mark_word<W>(base, x.w);
    }
    for (uint32_t t = nv * 4 + tid; t < n; t += stride) mark_word<W>(base, __ldcs(e + t));
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
