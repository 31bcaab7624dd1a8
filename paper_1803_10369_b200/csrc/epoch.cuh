// epoch.cuh — epoch-stamp linear recorders (u8 storage, z <= 7).
//
// A linear recorder byte holds the epoch (slice counter mod 256) of its last
// mark instead of the distance itself. The reference's value is recovered as
//   r = min((cur - s) mod 256, expired)                 (recorders.hpp:78-116)
// so the slide (age every recorder, sea.hpp:318-327) becomes `cur += 1`.
// Invariants that keep this exact:
//   * every stamp's age (cur - s) mod 256 stays <= 255: a sweep rewrites
//     stale stamps (age >= expired) to age exactly `expired`, visiting every
//     byte at least once per 255 - expired slides (1/240 of the table per
//     slide for z = 4);
//   * per row, hist[b] counts the recorders stamped b during the epoch b is
//     current and since: a mark moving a recorder off stamp s_old decrements
//     hist[s_old], onto cur increments hist[cur]; bins of stale epochs hold
//     garbage and are zeroed when the epoch counter comes back to them, which
//     the sweep invariant makes safe. Active recorders of a row (count_active,
//     recorders.hpp:119-129) = sum over the last k epochs of hist.
// The fill counts of report_window therefore need no table pass, and the
// slide touches only 1/(255 - expired) of the table.
#pragma once

#include "common.cuh"
#include "scan_binned.cuh"

namespace srla {

__device__ __forceinline__ uint32_t stamp_byte_shared(uint8_t* base, uint32_t off, uint32_t cur) {
    unsigned int* w = reinterpret_cast<unsigned int*>(base + (off & ~3u));
    const uint32_t sh = 8u * (off & 3u);
    unsigned int old = *w, assumed;
    do {
        assumed = old;
        if (((assumed >> sh) & 0xFFu) == cur) return cur;
        old = atomicCAS(w, assumed, (assumed & ~(0xFFu << sh)) | (cur << sh));
    } while (old != assumed);
    return (old >> sh) & 0xFFu;
}

// Apply pending marks of slices [f_begin, nfine) as epoch stamps and account
// the transitions in the per-row histograms. Only the touched 1 KB pieces of
// a slice move (a stamp pass leaves every other byte as it is): the block ORs
// its marks into a piece mask, bulk-loads those pieces into shared memory,
// stamps them there and bulk-stores them back; the next slice's pieces load
// while the current one is stamped. A tail slice (not a whole 16-byte
// multiple) goes through shared memory with plain loads.
__global__ void __launch_bounds__(256) k_slice_stamp(uint8_t* __restrict__ lin, uint64_t total_words,
                                                     uint64_t row_words, FineCfg f, uint32_t f_begin, int bulk,
                                                     uint32_t cur, uint32_t k, unsigned long long* __restrict__ hist,
                                                     uint32_t sparse_max) {
    extern __shared__ __align__(128) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    // per row of the slice (a slice spans at most two rows): net transitions
    // by age (cur - stamp) in [0, k): age 0 gains, older stamps in the window lose
    __shared__ uint32_t s_hist[2][128];
    __shared__ uint32_t s_mask[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31u;
    const uint32_t slice_bytes = 1u << f.shift;
    const uint32_t cs = f.shift > 15 ? f.shift - 5 : min(10u, f.shift);  // piece = 2^cs bytes, <= 32 per slice
    uint8_t* buf[2] = {s_raw, s_raw + slice_bytes};
    // next slice of this block (from, from + gridDim.x, ...) with more than
    // sparse_max marks (the rest is k_stamp_warp's): the block tests 256
    // candidates at a time (block-uniform call)
    __shared__ uint32_t s_next;
    auto next_slice = [&](uint32_t from) -> uint32_t {
        for (uint64_t base = from; base < f.nfine; base += static_cast<uint64_t>(blockDim.x) * gridDim.x) {
            if (threadIdx.x == 0) s_next = 0xFFFFFFFFu;
            __syncthreads();
            const uint64_t fb = base + static_cast<uint64_t>(threadIdx.x) * gridDim.x;
            if (fb < f.nfine && min(f.count[fb], f.cap) > sparse_max) atomicMin(&s_next, static_cast<uint32_t>(fb));
            __syncthreads();
            const uint32_t r = s_next;
            __syncthreads();
            if (r != 0xFFFFFFFFu) return r;
        }
        return f.nfine;
    };
    auto slice_len = [&](uint32_t fb) {
        return static_cast<uint32_t>(min(static_cast<uint64_t>(slice_bytes), total_words - (static_cast<uint64_t>(fb) << f.shift)));
    };
    auto marks = [&](uint32_t fb) { return f.bins + static_cast<uint64_t>(fb) * f.cap; };
    // pieces of slice fb holding marks (block-uniform call)
    auto piece_mask = [&](uint32_t fb, uint32_t slot) -> uint32_t {
        if (tid == 0) s_mask[slot] = 0;
        __syncthreads();
        const uint32_t n = min(f.count[fb], f.cap);
        const uint16_t* e = marks(fb);
        uint32_t m = 0;
        for (uint32_t q = tid; q < n; q += blockDim.x) m |= 1u << (static_cast<uint32_t>(e[q]) >> cs);
        m = __reduce_or_sync(0xFFFFFFFFu, m);
        if (lane == 0 && m) atomicOr(&s_mask[slot], m);
        __syncthreads();
        return s_mask[slot];
    };
    auto issue = [&](uint32_t fb, uint32_t b, uint32_t mask) -> bool {
        if (!bulk || slice_len(fb) != slice_bytes) return false;
        if (tid == 0) {
            uint8_t* g = lin + (static_cast<uint64_t>(fb) << f.shift);
            mbar_expect_tx(&s_bar[b], static_cast<uint32_t>(__popc(mask)) << cs);
            for (uint32_t m = mask; m; m &= m - 1) {
                const uint32_t c = __ffs(m) - 1;
                bulk_load(buf[b] + (c << cs), g + (static_cast<uint64_t>(c) << cs), 1u << cs, &s_bar[b]);
            }
        }
        return true;
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    __syncthreads();
    uint32_t phase[2] = {0u, 0u};  // parity of each barrier's next completion
    uint32_t cur_fb = next_slice(f_begin + blockIdx.x);
    uint32_t mcur = cur_fb < f.nfine ? piece_mask(cur_fb, 0) : 0u;
    bool bulk_cur = cur_fb < f.nfine && issue(cur_fb, 0, mcur);
    for (uint32_t i = 0; cur_fb < f.nfine; ++i) {
        const uint32_t b = i & 1u;
        const uint32_t nxt = next_slice(cur_fb + gridDim.x);
        uint32_t mnxt = 0;
        bool bulk_nxt = false;
        if (nxt < f.nfine) {
            mnxt = piece_mask(nxt, b ^ 1u);
            if (tid == 0) bulk_wait_read_all();  // the stores out of buf[b ^ 1] have left shared memory
            bulk_nxt = issue(nxt, b ^ 1u, mnxt);
        }
        const uint32_t len = slice_len(cur_fb);
        uint8_t* g = lin + (static_cast<uint64_t>(cur_fb) << f.shift);
        for (uint32_t q = tid; q < 2 * k; q += blockDim.x) s_hist[q / k][q % k] = 0;
        if (bulk_cur) {
            mbar_wait(&s_bar[b], phase[b]);
            phase[b] ^= 1u;
        } else {
            for (uint32_t q = tid; q < len; q += blockDim.x) buf[b][q] = g[q];
        }
        __syncthreads();
        if (tid == 0) atomicAdd(f.streamed, bulk_cur ? static_cast<unsigned long long>(__popc(mcur)) << cs : len);
        const uint32_t n = min(f.count[cur_fb], f.cap);
        const uint16_t* e = marks(cur_fb);
        const uint64_t w0 = static_cast<uint64_t>(cur_fb) << f.shift;
        const uint64_t row_a = w0 / row_words;
        const uint32_t split = static_cast<uint32_t>(min(static_cast<uint64_t>(len), (row_a + 1) * row_words - w0));
        // transitions onto `cur` are counted per warp (one shared atomic per
        // warp and row); decrements only matter for stamps inside the window
        // (stale bins are zeroed when the counter returns to them)
        for (uint32_t q0 = 0; q0 < n; q0 += blockDim.x) {
            const uint32_t q = q0 + tid;
            uint32_t old = cur, h = 0;
            if (q < n) {
                const uint32_t off = e[q];
                old = stamp_byte_shared(buf[b], off, cur);
                h = off < split ? 0u : 1u;
                const uint32_t age = (cur - old) & 0xFFu;
                if (old != cur && age < k) atomicSub(&s_hist[h][age], 1u);
            }
            const unsigned moved = __ballot_sync(0xFFFFFFFFu, old != cur);
            const unsigned row_b = __ballot_sync(0xFFFFFFFFu, h == 1u);
            if (lane == 0) {
                const uint32_t c1 = __popc(moved & row_b), c0 = __popc(moved) - c1;
                if (c0) atomicAdd(&s_hist[0][0], c0);
                if (c1) atomicAdd(&s_hist[1][0], c1);
            }
        }
        __syncthreads();
        for (uint32_t q = tid; q < 2 * k; q += blockDim.x) {
            const uint32_t h = q / k, age = q % k;
            const uint32_t v = s_hist[h][age];
            if (v)
                atomicAdd(hist + (row_a + h) * 256 + ((cur - age) & 0xFFu),
                          static_cast<unsigned long long>(static_cast<long long>(static_cast<int32_t>(v))));
        }
        if (bulk_cur) {
            fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0)
                for (uint32_t m = mcur; m; m &= m - 1) {
                    const uint32_t c = __ffs(m) - 1;
                    bulk_store(g + (static_cast<uint64_t>(c) << cs), buf[b] + (c << cs), 1u << cs);
                }
        } else {
            for (uint32_t q = tid; q < len; q += blockDim.x) g[q] = buf[b][q];
            __syncthreads();
        }
        cur_fb = nxt;
        mcur = mnxt;
        bulk_cur = bulk_nxt;
    }
    if (tid == 0) bulk_wait_all();
}

// Sparse slices (at most sparse_max marks; C3's 2^24-column table has ~200
// per 32 KB slice, clustered on the active sources' cells): one WARP per
// slice stamps in place in global memory, no shared-memory staging of the
// slice and no block barriers — the block-per-slice kernel above is bound by
// its per-slice fixed cost there. The warp owns its slice, so no global
// atomics are needed: a per-warp shared bitmap (one bit per recorder of the
// slice, claimed with a shared atomicOr) elects one lane per distinct
// recorder, which loads the stamp and stores `cur` with plain byte accesses;
// eight marks per lane are in flight. The histogram deltas accumulate per
// block by (row, age) and are flushed at the end. Dynamic shared memory:
// 8 warps x 2^(shift-3) bytes of bitmap.
constexpr int kStampWarpRows = 4;  // binned tables have <= kBinRows rows
inline uint32_t stamp_claim_words(uint32_t shift) { return ((1u << shift) + 31u) >> 5; }
inline uint32_t stamp_claim_bytes(uint32_t shift) { return 8u * 4u * stamp_claim_words(shift); }
__global__ void __launch_bounds__(256, 5) k_stamp_warp(uint8_t* __restrict__ lin, uint64_t row_words, FineCfg f,
                                                    uint32_t sparse_max, uint32_t cur, uint32_t k, uint32_t rows,
                                                    unsigned long long* __restrict__ hist) {
    __shared__ int32_t s_h[kStampWarpRows][128];  // net transitions by (row, age)
    extern __shared__ uint32_t s_claim[];
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
    const uint32_t bwords = ((1u << f.shift) + 31u) >> 5;
    uint32_t* claim = s_claim + warp * bwords;
    for (uint32_t q = threadIdx.x; q < kStampWarpRows * 128; q += blockDim.x) (&s_h[0][0])[q] = 0;
    for (uint32_t q = lane; q < bwords; q += 32) claim[q] = 0;
    __syncthreads();
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    constexpr int kU = 8;
    // software pipeline: the next slice's count and first 32*kU marks load
    // while this slice's stamps are read and written (the marks past the
    // count are never used; every read stays inside the slice's bin)
    uint32_t pre_n = 0, pre[kU / 2];  // two u16 marks per register
    auto prefetch = [&](uint32_t fb) {
        if (fb >= f.nfine) return;
        const uint16_t* e = f.bins + static_cast<uint64_t>(fb) * f.cap;
        pre_n = __ldg(f.count + fb);
#pragma unroll
        for (int u = 0; u < kU; u += 2) {
            const uint32_t lo = lane + 32u * u < f.cap ? __ldg(e + lane + 32u * u) : 0u;
            const uint32_t hi = lane + 32u * (u + 1) < f.cap ? __ldg(e + lane + 32u * (u + 1)) : 0u;
            pre[u / 2] = lo | (hi << 16);
        }
    };
    prefetch(blockIdx.x * (blockDim.x >> 5) + warp);
    for (uint32_t fb = blockIdx.x * (blockDim.x >> 5) + warp; fb < f.nfine; fb += nwarps) {
        const uint32_t n = min(pre_n, f.cap);
        uint32_t first[kU / 2];
#pragma unroll
        for (int u = 0; u < kU / 2; ++u) first[u] = pre[u];
        prefetch(fb + nwarps);
        if (n == 0 || n > sparse_max) continue;
        const uint16_t* e = f.bins + static_cast<uint64_t>(fb) * f.cap;
        const uint64_t w0 = static_cast<uint64_t>(fb) << f.shift;
        const uint32_t row_a = static_cast<uint32_t>(w0 / row_words);
        const uint64_t split = (static_cast<uint64_t>(row_a) + 1) * row_words - w0;  // offsets >= split: next row
        uint8_t* g = lin + w0;
        uint32_t fresh_a = 0, fresh_b = 0;  // transitions onto `cur` in rows row_a, row_a + 1
        for (uint32_t q0 = 0; q0 < n; q0 += 32 * kU) {
            uint32_t off[kU], old[kU];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                const uint32_t q = q0 + lane + 32u * u;
                off[u] = q < n ? (q0 ? static_cast<uint32_t>(e[q]) : (first[u / 2] >> (16 * (u & 1))) & 0xFFFFu) : 0xFFFFFFFFu;
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (off[u] == 0xFFFFFFFFu) continue;
                const uint32_t m = 1u << (off[u] & 31u);
                if (atomicOr(&claim[off[u] >> 5], m) & m) off[u] = 0xFFFFFFFFu;  // a duplicate: another lane has it
            }
#pragma unroll
            for (int u = 0; u < kU; ++u) old[u] = off[u] != 0xFFFFFFFFu ? __ldcg(g + off[u]) : cur;
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                // a recorder leaving age `age` < k: one shared atomic per
                // distinct (row, age) of the warp (a block-wide hot spot
                // otherwise)
                uint32_t key = 0xFFFFFFFFu;
                if (old[u] != cur) {
                    g[off[u]] = static_cast<uint8_t>(cur);
                    const uint32_t second = off[u] >= split ? 1u : 0u;
                    fresh_a += second ^ 1u;
                    fresh_b += second;
                    const uint32_t age = (cur - old[u]) & 0xFFu;
                    if (age < k) key = ((row_a + second) << 8) | age;
                }
                const uint32_t peers = __match_any_sync(0xFFFFFFFFu, key);
                if (key != 0xFFFFFFFFu && lane == __ffs(peers) - 1u)
                    atomicSub(&s_h[(key >> 8) & 3u][key & 0xFFu], __popc(peers));
            }
        }
        fresh_a = __reduce_add_sync(0xFFFFFFFFu, fresh_a);
        fresh_b = __reduce_add_sync(0xFFFFFFFFu, fresh_b);
        if (lane == 0) {
            if (fresh_a) atomicAdd(&s_h[row_a & 3u][0], static_cast<int32_t>(fresh_a));
            if (fresh_b) atomicAdd(&s_h[(row_a + 1u) & 3u][0], static_cast<int32_t>(fresh_b));
        }
        __syncwarp();
        for (uint32_t q = lane; q < n; q += 32) claim[static_cast<uint32_t>(e[q]) >> 5] = 0;
        __syncwarp();
    }
    __syncthreads();
    for (uint32_t q = threadIdx.x; q < rows * k; q += blockDim.x) {
        const uint32_t h = q / k, age = q % k;
        const int32_t v = s_h[h][age];
        if (v) atomicAdd(hist + h * 256ull + ((cur - age) & 0xFFu), static_cast<unsigned long long>(static_cast<long long>(v)));
    }
}

// Sweep [w0, w0+n) of the table: stamps with age >= expired become age
// exactly `expired` (no histogram change: such recorders are outside every
// window, k <= expired).
__global__ void __launch_bounds__(256) k_sweep(uint8_t* __restrict__ lin, uint64_t w0, uint64_t n, uint32_t cur,
                                               uint32_t expired) {
    const uint32_t cur4 = cur * 0x01010101u, e4 = expired * 0x01010101u;
    const uint32_t tgt4 = ((cur - expired) & 0xFFu) * 0x01010101u;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint8_t* base = lin + w0;
    const uint64_t head = min(n, static_cast<uint64_t>((16 - (reinterpret_cast<uintptr_t>(base) & 15)) & 15));
    auto fix = [&](uint32_t x) {
        const uint32_t stale = __vcmpgeu4(__vsub4(cur4, x), e4);
        return (x & ~stale) | (tgt4 & stale);
    };
    for (uint64_t q = tid; q < head; q += stride) {
        const uint32_t s = base[q];
        if (((cur - s) & 0xFFu) >= expired) base[q] = static_cast<uint8_t>((cur - expired) & 0xFFu);
    }
    uint4* v = reinterpret_cast<uint4*>(base + head);
    const uint64_t nv = (n - head) / 16;
    for (uint64_t q = tid; q < nv; q += stride) {
        uint4 x = v[q];
        x.x = fix(x.x);
        x.y = fix(x.y);
        x.z = fix(x.z);
        x.w = fix(x.w);
        v[q] = x;
    }
    for (uint64_t q = head + nv * 16 + tid; q < n; q += stride) {
        const uint32_t s = base[q];
        if (((cur - s) & 0xFFu) >= expired) base[q] = static_cast<uint8_t>((cur - expired) & 0xFFu);
    }
}

__global__ void k_zero_hist_bin(unsigned long long* hist, uint32_t rows, uint32_t bin) {
    for (uint32_t i = threadIdx.x; i < rows; i += blockDim.x) hist[i * 256ull + bin] = 0;
}

// Stamps -> literal recorder values min((cur - s) mod 256, expired).
__global__ void __launch_bounds__(256) k_epoch_to_literal(uint8_t* __restrict__ lin, uint64_t n, uint32_t cur,
                                                          uint32_t expired) {
    const uint32_t cur4 = cur * 0x01010101u, e4 = expired * 0x01010101u;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    uint4* v = reinterpret_cast<uint4*>(lin);
    const uint64_t nv = n / 16;
    for (uint64_t q = tid; q < nv; q += stride) {
        uint4 x = v[q];
        x.x = __vminu4(__vsub4(cur4, x.x), e4);
        x.y = __vminu4(__vsub4(cur4, x.y), e4);
        x.z = __vminu4(__vsub4(cur4, x.z), e4);
        x.w = __vminu4(__vsub4(cur4, x.w), e4);
        v[q] = x;
    }
    for (uint64_t q = nv * 16 + tid; q < n; q += stride) {
        const uint32_t a = (cur - lin[q]) & 0xFFu;
        lin[q] = static_cast<uint8_t>(a < expired ? a : expired);
    }
}

// Row export/import through a device staging buffer (a snapshot of a 64 GiB
// table converts at HBM speed instead of in a host loop):
// stamps -> literal values min((cur - s) mod 256, expired), and back
// (s = cur - v, values already checked to be <= expired).
__global__ void __launch_bounds__(256) k_stamps_to_values(const uint8_t* __restrict__ s, uint64_t n, uint32_t cur,
                                                          uint32_t expired, uint8_t* __restrict__ v) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t a = (cur - s[q]) & 0xFFu;
        v[q] = static_cast<uint8_t>(a < expired ? a : expired);
    }
}
__global__ void __launch_bounds__(256) k_values_to_stamps(const uint8_t* __restrict__ v, uint64_t n, uint32_t cur,
                                                          uint8_t* __restrict__ s) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        s[q] = static_cast<uint8_t>((cur - v[q]) & 0xFFu);
}

// Histogram of a range of one row's stamps, added (sign 1) or removed (sign -1)
// around an import. grid-stride, 256 bins.
__global__ void __launch_bounds__(256) k_row_hist(const uint8_t* __restrict__ row, uint64_t n,
                                                  unsigned long long* __restrict__ hist, int sign) {
    __shared__ uint32_t s_h[256];
    s_h[threadIdx.x] = 0;
    __syncthreads();
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        atomicAdd(&s_h[row[q]], 1u);
    __syncthreads();
    const unsigned long long c = s_h[threadIdx.x];  // sign -1: subtract (mod 2^64)
    if (c) atomicAdd(hist + threadIdx.x, sign < 0 ? 0ull - c : c);
}

// Union linear weight over epoch stamps: slot j counts iff every row's stamp
// is younger than k (max over rows of the recorder value < k).
template <int MAXR>
__global__ void __launch_bounds__(256) k_union_linear_epoch(const uint32_t* __restrict__ hosts, uint32_t n, DevCfg c,
                                                            const uint8_t* __restrict__ lin, uint32_t cur,
                                                            uint32_t* __restrict__ weight) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint32_t cur4 = cur * 0x01010101u, k4 = c.k * 0x01010101u;
    const bool vec = (c.gl & 15u) == 0;
    for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < n; h += warps) {
        const uint32_t a = hosts[h];
        const uint8_t* cell[MAXR];
        if (MAXR <= 4) {  // lane i hashes row i; the warp shares the columns
            const uint32_t colv = lane < c.rows ? column_of(c, lane, a) : 0u;
#pragma unroll
            for (int i = 0; i < MAXR; ++i)
                cell[i] = lin + i * lrow + static_cast<uint64_t>(__shfl_sync(0xFFFFFFFFu, colv, i)) * c.gl;
        } else {
#pragma unroll
            for (int i = 0; i < MAXR; ++i)
                if (i < static_cast<int>(c.rows)) cell[i] = lin + i * lrow + static_cast<uint64_t>(column_of(c, i, a)) * c.gl;
        }
        uint32_t acc = 0;
        if (vec && MAXR <= 4) {
            // all rows' vectors of two iterations issued before any use
            const uint32_t nv = c.gl / 16;
            for (uint32_t q0 = lane; q0 < nv; q0 += 64) {
                uint4 x[2][MAXR];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int i = 0; i < MAXR; ++i)
                        x[u][i] = (i < static_cast<int>(c.rows) && q0 + 32u * u < nv)
                                      ? __ldcs(reinterpret_cast<const uint4*>(cell[i]) + q0 + 32u * u)
                                      : make_uint4(cur4, cur4, cur4, cur4);
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (q0 + 32u * u >= nv) break;
                    uint4 m = make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
                    for (int i = 0; i < MAXR; ++i) {
                        m.x &= __vcmpltu4(__vsub4(cur4, x[u][i].x), k4);
                        m.y &= __vcmpltu4(__vsub4(cur4, x[u][i].y), k4);
                        m.z &= __vcmpltu4(__vsub4(cur4, x[u][i].z), k4);
                        m.w &= __vcmpltu4(__vsub4(cur4, x[u][i].w), k4);
                    }
                    acc += __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
                }
            }
            acc >>= 3;
        } else if (vec) {
            const uint32_t nv = c.gl / 16;
            for (uint32_t q = lane; q < nv; q += 32) {
                uint4 m = make_uint4(~0u, ~0u, ~0u, ~0u);
#pragma unroll
                for (int i = 0; i < MAXR; ++i) {
                    if (i >= static_cast<int>(c.rows)) break;
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(cell[i]) + q);
                    m.x &= __vcmpltu4(__vsub4(cur4, x.x), k4);
                    m.y &= __vcmpltu4(__vsub4(cur4, x.y), k4);
                    m.z &= __vcmpltu4(__vsub4(cur4, x.z), k4);
                    m.w &= __vcmpltu4(__vsub4(cur4, x.w), k4);
                }
                acc += __popc(m.x) + __popc(m.y) + __popc(m.z) + __popc(m.w);
            }
            acc >>= 3;
        } else {
            for (uint32_t j = lane; j < c.gl; j += 32) {
                bool all = true;
                for (uint32_t i = 0; i < c.rows; ++i) all &= ((cur - cell[i < MAXR ? i : 0][j]) & 0xFFu) < c.k;
                acc += all;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (lane == 0) weight[h] = acc;
    }
}

}  // namespace srla
