// kernels.cuh — the SRLA hot-path kernels (literal recorder representation).
//
// Data layout in HBM is the reference's own row-major layout (sea.hpp:127-134,
// 356-358), all rows of a table concatenated in one allocation:
//   linear[(i*v + col)*g' + slot]  W-byte words
//   rough [(i*v + col)*g  + slot]  W-byte words
//   si    [ i*v + col ]            u16
// plus, for the in-chunk ordering of rough marks, one u32 "first marking
// packet" stamp per rough entry (0xFFFFFFFF = unmarked in this chunk).
//
// Serial semantics reproduced: packets p = 0..N-1 of a
// chunk in order; rough entry e counts as marked "as of p" iff some sampled
// packet q <= p marks e, i.e. stamp[e] <= p. A sampled packet crosses iff its
// host's union weight as of p reaches thr; each host's first crossing P(a)
// decides insertion against the indicator bits set by earlier-P insertions.
#pragma once

#include "common.cuh"

namespace srla {

// ----------------------------------------------------------------- K1 scan
// Per record: u column hashes of aip, the sample hash of bip; u linear marks
// (store 0: recorder_mark, recorders.hpp:78-81 — every packet, before the
// sampling test, sea.hpp:155-161). Sampled packets (ctz(sample) >= tau,
// sea.hpp:164) also stamp their u rough entries with their index (atomicMin)
// and append an event (p, aip, rslot) — warp-aggregated.
// Records are read as three 16-byte vectors per 4 records (streaming loads).
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_scan(const uint32_t* __restrict__ recs, uint32_t n,
                                              DevCfg c, W* __restrict__ lin,
                                              uint32_t* __restrict__ stamp,
                                              uint32_t* __restrict__ ev, uint32_t ev_cap,
                                              uint32_t* __restrict__ ev_count, int vec) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint64_t ngroups = (static_cast<uint64_t>(n) + 3) / 4;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    for (uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * blockDim.x + (threadIdx.x & ~31u);
         g0 < ngroups; g0 += stride) {
        const uint64_t grp = g0 + lane;
        const uint32_t base = static_cast<uint32_t>(grp * 4);
        uint32_t src[4], dst[4];
        uint32_t valid = 0;
        if (grp < ngroups) {
            if (vec && base + 4 <= n) {
                const uint4* q = reinterpret_cast<const uint4*>(recs + 3ull * base);
                const uint4 a = __ldcs(q), b = __ldcs(q + 1), d = __ldcs(q + 2);
                src[0] = a.y; dst[0] = a.z;
                src[1] = b.x; dst[1] = b.y;
                src[2] = b.w; dst[2] = d.x;
                src[3] = d.z; dst[3] = d.w;
                valid = 4;
            } else {
                valid = min(4u, n - base);
                for (uint32_t q = 0; q < 4; ++q) {
                    if (q < valid) {
                        src[q] = __ldcs(recs + 3ull * (base + q) + 1);
                        dst[q] = __ldcs(recs + 3ull * (base + q) + 2);
                    } else {
                        src[q] = dst[q] = 0;
                    }
                }
            }
        }
        uint32_t smask = 0, rsl[4];
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            rsl[q] = 0;
            if (q < valid) {
                const uint32_t sample = hash_u32k(c.sub_sample, c.kh_sample, dst[q]);
                const uint32_t lslot = c.gl_mask ? (sample & c.gl_mask) : (sample % c.gl);
                const bool smp = (sample & c.tau_mask) == 0u;
                const uint32_t rslot = smp ? reduce32(hash_u32k(c.sub_rslot, c.kh_rslot, dst[q]), c.g) : 0u;
#pragma unroll
                for (int i = 0; i < MAXR; ++i) {
                    if (i < static_cast<int>(c.rows)) {
                        const uint32_t col = column_of(c, i, src[q]);
                        lin[i * lrow + static_cast<uint64_t>(col) * c.gl + lslot] = W(0);
                        if (smp) atomicMin(stamp + i * rrow + static_cast<uint64_t>(col) * c.g + rslot, base + q);
                    }
                }
                if (smp) {
                    smask |= 1u << q;
                    rsl[q] = rslot;
                }
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
    }
}

// Union rough weight of host `a` (sea.hpp:172-181 / 219-230): number of slots
// j whose recorders are active in every row. With `asof`, an entry stamped by
// a packet q <= p counts as freshly marked (value 0, active).
template <typename W, int MAXR>
__device__ __forceinline__ uint32_t rough_weight(const DevCfg& c, const W* __restrict__ rough,
                                                 const uint32_t* __restrict__ stamp, uint32_t a,
                                                 uint32_t p, bool asof) {
    if constexpr (sizeof(W) == 1 && MAXR <= 4) {
        if (c.g == 8) {  // the configs of BASELINE.json: a rough cell is one 8-byte word per row
            const uint64_t rrow = static_cast<uint64_t>(c.cols) * 8u;
            const uint32_t k4 = c.k * 0x01010101u;
            uint32_t act_lo = 0xFFFFFFFFu, act_hi = 0xFFFFFFFFu;  // 0xFF per slot active in every row so far
#pragma unroll
            for (int i = 0; i < MAXR; ++i) {
                if (i >= static_cast<int>(c.rows)) break;
                const uint64_t b = i * rrow + static_cast<uint64_t>(column_of(c, i, a)) * 8u;
                const uint2 r = *reinterpret_cast<const uint2*>(rough + b);
                uint32_t lo = __vcmpltu4(r.x, k4), hi = __vcmpltu4(r.y, k4);
                if (asof && (lo & hi) != 0xFFFFFFFFu) {  // slots marked by this chunk's packets <= p count too
                    const uint4 s0 = *reinterpret_cast<const uint4*>(stamp + b);
                    const uint4 s1 = *reinterpret_cast<const uint4*>(stamp + b + 4);
                    lo |= (s0.x <= p ? 0xFFu : 0u) | (s0.y <= p ? 0xFF00u : 0u) | (s0.z <= p ? 0xFF0000u : 0u) |
                          (s0.w <= p ? 0xFF000000u : 0u);
                    hi |= (s1.x <= p ? 0xFFu : 0u) | (s1.y <= p ? 0xFF00u : 0u) | (s1.z <= p ? 0xFF0000u : 0u) |
                          (s1.w <= p ? 0xFF000000u : 0u);
                }
                act_lo &= lo;
                act_hi &= hi;
            }
            return (__popc(act_lo) + __popc(act_hi)) >> 3;
        }
    }
    uint32_t cols[MAXR];
#pragma unroll
    for (int i = 0; i < MAXR; ++i)
        if (i < static_cast<int>(c.rows)) cols[i] = column_of(c, i, a);
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    uint32_t weight = 0;
    for (uint32_t j0 = 0; j0 < c.g; j0 += 64) {
        const uint32_t jn = min(64u, c.g - j0);
        uint64_t mask = jn == 64 ? ~0ull : ((1ull << jn) - 1);
#pragma unroll
        for (int i = 0; i < MAXR; ++i) {
            if (i >= static_cast<int>(c.rows)) break;
            const uint64_t b = i * rrow + static_cast<uint64_t>(cols[i]) * c.g + j0;
            for (uint32_t j = 0; j < jn; ++j) {
                const uint32_t r = static_cast<uint32_t>(rough[b + j]);
                bool ok = r < c.k;
                if (!ok && asof) ok = stamp[b + j] <= p;
                if (!ok) mask &= ~(1ull << j);
            }
        }
        weight += __popcll(mask);
    }
    return weight;
}

// ----------------------------------------------------------------- K2 crossing
// Per sampled event: union weight as of its own packet; crossing events
// (weight >= thr, sea.hpp:182) are appended as key (aip << 32 | p).
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_cross(const uint32_t* __restrict__ ev, uint32_t ev_cap,
                                               uint32_t n_ev, DevCfg c, const W* __restrict__ rough,
                                               const uint32_t* __restrict__ stamp,
                                               uint64_t* __restrict__ xkeys,
                                               uint32_t* __restrict__ x_count) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t t0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); t0 < n_ev; t0 += stride) {
        const uint32_t t = t0 + (threadIdx.x & 31u);
        bool cross = false;
        uint32_t p = 0, a = 0;
        if (t < n_ev) {
            p = ev[t];
            a = ev[ev_cap + t];
            cross = rough_weight<W, MAXR>(c, rough, stamp, a, p, true) >= c.thr;
        }
        const uint32_t pos = warp_append(x_count, cross ? 1u : 0u);
        if (cross) xkeys[pos] = (static_cast<uint64_t>(a) << 32) | p;
    }
}

// ----------------------------------------------------------------- K5 rough commit
// Apply the chunk's rough marks (store 0, sea.hpp:166-169) and clear their
// stamps for the next chunk. Order-independent.
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_commit(const uint32_t* __restrict__ ev, uint32_t ev_cap,
                                                uint32_t n_ev, DevCfg c, W* __restrict__ rough,
                                                uint32_t* __restrict__ stamp) {
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_ev; t += gridDim.x * blockDim.x) {
        const uint32_t a = ev[ev_cap + t];
        const uint32_t rs = ev[2ull * ev_cap + t];
#pragma unroll
        for (int i = 0; i < MAXR; ++i) {
            if (i >= static_cast<int>(c.rows)) break;
            const uint64_t e = i * rrow + static_cast<uint64_t>(column_of(c, i, a)) * c.g + rs;
            rough[e] = W(0);
            stamp[e] = 0xFFFFFFFFu;
        }
    }
}

// ----------------------------------------------------------------- K3 first crossing
// xs sorted by (aip, p): the first key of each aip run is that host's first
// crossing P(a). Emits (P << 32 | aip) for a subsequent sort by P.
__global__ void __launch_bounds__(256) k_first(const uint64_t* __restrict__ xs, uint32_t X,
                                               uint64_t* __restrict__ hp, uint32_t* __restrict__ h_count) {
    for (uint32_t t0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); t0 < X; t0 += gridDim.x * blockDim.x) {
        const uint32_t t = t0 + (threadIdx.x & 31u);
        bool first = false;
        uint64_t key = 0;
        if (t < X) {
            key = xs[t];
            first = t == 0 || (xs[t - 1] >> 32) != (key >> 32);
        }
        const uint32_t pos = warp_append(h_count, first ? 1u : 0u);
        if (first) hp[pos] = (key << 32) | (key >> 32);
    }
}

// ----------------------------------------------------------------- K4 SI resolution
// K4a: per first-crossing host (sorted by P): indicator rows where its bit is
// still clear in the indicator state at chunk start (F mask). F == 0 means
// suppressed by the carried-over bits (sea.hpp:185-190).
__global__ void __launch_bounds__(256) k_si_check(const uint64_t* __restrict__ hp, uint32_t Hn,
                                                  DevCfg c, const uint16_t* __restrict__ si,
                                                  uint64_t* __restrict__ fmask, uint32_t* __restrict__ cnt,
                                                  uint32_t* __restrict__ hosts, uint8_t* __restrict__ status) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < Hn; h += gridDim.x * blockDim.x) {
        const uint32_t a = static_cast<uint32_t>(hp[h]);
        const uint16_t bit = static_cast<uint16_t>(1u << indicator_bit_index(c, a));
        uint64_t F = 0;
        for (uint32_t i = 0; i < c.rows; ++i)
            if (!(si[static_cast<uint64_t>(i) * c.cols + column_of(c, i, a)] & bit)) F |= 1ull << i;
        fmask[h] = F;
        cnt[h] = __popcll(F);
        hosts[h] = a;
        status[h] = F ? 2 : 0;  // 0 suppressed, 1 inserted, 2 undecided
    }
}

// K4b: one tuple per (host, open row): key = (row, col, bit), in host (= P) order.
__global__ void __launch_bounds__(256) k_tuples(const uint32_t* __restrict__ hosts, uint32_t Hn, DevCfg c,
                                                const uint64_t* __restrict__ fmask,
                                                const uint32_t* __restrict__ off,
                                                uint64_t* __restrict__ tkey, uint32_t* __restrict__ tval,
                                                uint32_t* __restrict__ towner) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < Hn; h += gridDim.x * blockDim.x) {
        const uint32_t a = hosts[h];
        const uint32_t b = indicator_bit_index(c, a);
        uint64_t F = fmask[h];
        uint32_t t = off[h];
        while (F) {
            const uint32_t i = __ffsll(F) - 1;
            F &= F - 1;
            tkey[t] = (static_cast<uint64_t>(i) * c.cols + column_of(c, i, a)) * kIndicatorBits + b;
            tval[t] = t;
            towner[t] = h;
            ++t;
        }
    }
}

// K4c: tuples stably sorted by key (so by P within a key). A host that is the
// earliest at some open (row, col, bit) cannot be suppressed there: it is
// definitely inserted. Also records each tuple's sorted position.
__global__ void __launch_bounds__(256) k_first_key(const uint64_t* __restrict__ skey,
                                                   const uint32_t* __restrict__ sval, uint32_t T,
                                                   const uint32_t* __restrict__ towner,
                                                   uint8_t* __restrict__ definite,
                                                   uint32_t* __restrict__ posof) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) {
        const uint32_t v = sval[t];
        posof[v] = t;
        if (t == 0 || skey[t - 1] != skey[t]) definite[towner[v]] = 1;
    }
}

// K4d: classify; undecided hosts become the flagged list (needs P order).
__global__ void __launch_bounds__(256) k_classify(uint32_t Hn, uint8_t* __restrict__ status,
                                                  const uint8_t* __restrict__ definite,
                                                  uint8_t* __restrict__ flag_undecided,
                                                  uint8_t* __restrict__ flag_inserted) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < Hn; h += gridDim.x * blockDim.x) {
        uint8_t s = status[h];
        if (s == 2 && definite[h]) s = 1;
        status[h] = s;
        flag_undecided[h] = s == 2;
        flag_inserted[h] = s == 1;
    }
}

// K4e: ordered resolution of the flagged hosts (ascending P). A host is
// inserted iff some open row has no inserted host earlier at the same
// (row, col, bit) — the reference's "bit not in SI of some row" test
// evaluated at P(a). Single thread: the flagged set is tiny unless the
// indicator table is saturated.
__global__ void k_serial(const uint32_t* __restrict__ flagged, uint32_t nf,
                         const uint64_t* __restrict__ fmask, const uint32_t* __restrict__ off,
                         const uint32_t* __restrict__ posof, const uint64_t* __restrict__ skey,
                         const uint32_t* __restrict__ sval, const uint32_t* __restrict__ towner,
                         uint8_t* __restrict__ status, uint8_t* __restrict__ flag_inserted) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    for (uint32_t f = 0; f < nf; ++f) {
        const uint32_t h = flagged[f];
        const uint32_t nrows = __popcll(fmask[h]);
        bool inserted = false;
        for (uint32_t r = 0; r < nrows && !inserted; ++r) {
            const uint32_t t = posof[off[h] + r];
            const uint64_t key = skey[t];
            bool blocked = false;
            for (uint32_t tt = t; tt > 0 && skey[tt - 1] == key; --tt) {
                if (status[towner[sval[tt - 1]]] == 1) {
                    blocked = true;
                    break;
                }
            }
            inserted = !blocked;
        }
        status[h] = inserted ? 1 : 0;
        flag_inserted[h] = inserted;
    }
}

// K4f: set the bit of every inserted host in all its rows (sea.hpp:193-195).
__global__ void __launch_bounds__(256) k_si_set(const uint32_t* __restrict__ hosts, uint32_t Hn,
                                                const uint8_t* __restrict__ status, DevCfg c,
                                                uint16_t* __restrict__ si) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < Hn; h += gridDim.x * blockDim.x) {
        if (status[h] != 1) continue;
        const uint32_t a = hosts[h];
        const uint16_t bit = static_cast<uint16_t>(1u << indicator_bit_index(c, a));
        for (uint32_t i = 0; i < c.rows; ++i)
            atomic_or_u16(si + static_cast<uint64_t>(i) * c.cols + column_of(c, i, a), bit);
    }
}

// ----------------------------------------------------------------- candidate set
// Open-addressing hash set over host+1 (0 = empty) mirroring CandidateList's
// membership (sea.hpp:58-62).
__device__ __forceinline__ uint64_t cset_slot(uint32_t host, uint64_t mask) {
    return avalanche64(host) & mask;
}
__global__ void __launch_bounds__(256) k_cset_lookup(const uint32_t* __restrict__ hosts, uint32_t n,
                                                     const unsigned long long* __restrict__ table,
                                                     uint64_t mask, uint8_t* __restrict__ is_new) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const unsigned long long key = static_cast<unsigned long long>(hosts[t]) + 1ull;
        uint64_t s = cset_slot(hosts[t], mask);
        uint8_t fresh = 1;
        while (true) {
            const unsigned long long v = table[s];
            if (v == 0) break;
            if (v == key) {
                fresh = 0;
                break;
            }
            s = (s + 1) & mask;
        }
        is_new[t] = fresh;
    }
}
__global__ void __launch_bounds__(256) k_cset_insert(const uint32_t* __restrict__ hosts, uint32_t n,
                                                     unsigned long long* __restrict__ table, uint64_t mask) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const unsigned long long key = static_cast<unsigned long long>(hosts[t]) + 1ull;
        uint64_t s = cset_slot(hosts[t], mask);
        while (true) {
            const unsigned long long prev = atomicCAS(table + s, 0ull, key);
            if (prev == 0ull || prev == key) break;
            s = (s + 1) & mask;
        }
    }
}

// ----------------------------------------------------------------- K6 row activity
// count_active over each linear row (recorders.hpp:119-129): 16-byte loads,
// byte/halfword SIMD compares. grid.y = row.
template <typename W>
__device__ __forceinline__ uint32_t count_lt_word(uint32_t x, uint32_t kk, uint32_t k) {
    if constexpr (sizeof(W) == 1) return __popc(__vcmpltu4(x, kk));        // 8 bits per active byte
    else if constexpr (sizeof(W) == 2) return __popc(__vcmpltu2(x, kk));   // 16 bits per active half
    else return x < k ? 1u : 0u;
}
template <typename W>
__global__ void __launch_bounds__(256) k_row_active(const W* __restrict__ lin, uint64_t row_words,
                                                    uint32_t k, unsigned long long* __restrict__ counts) {
    const uint32_t row = blockIdx.y;
    const W* r = lin + row * row_words;
    const uint32_t kk = sizeof(W) == 1 ? k * 0x01010101u : sizeof(W) == 2 ? k * 0x00010001u : k;
    unsigned long long acc = 0;
    const uint64_t bytes = row_words * sizeof(W);
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    if ((bytes & 15) == 0 && (reinterpret_cast<uintptr_t>(r) & 15) == 0) {
        const uint4* v = reinterpret_cast<const uint4*>(r);
        const uint64_t nv = bytes / 16;
        for (uint64_t q = tid; q < nv; q += stride) {
            const uint4 x = __ldcs(v + q);
            acc += count_lt_word<W>(x.x, kk, k) + count_lt_word<W>(x.y, kk, k) +
                   count_lt_word<W>(x.z, kk, k) + count_lt_word<W>(x.w, kk, k);
        }
        if constexpr (sizeof(W) == 1) acc >>= 3;
        else if constexpr (sizeof(W) == 2) acc >>= 4;
    } else {
        for (uint64_t q = tid; q < row_words; q += stride) acc += static_cast<uint32_t>(r[q]) < k;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ unsigned long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (uint32_t w = 0; w < blockDim.x / 32; ++w) s += part[w];
        if (s) atomicAdd(counts + row, s);
    }
}

// ----------------------------------------------------------------- K7 union linear weight
// One warp per host: max over the u linear cells of g' recorders, count < k
// (sea.hpp:232-243). W=1/2 use 16-byte loads with byte/halfword SIMD max.
template <typename W>
__device__ __forceinline__ uint32_t vmax_word(uint32_t a, uint32_t b) {
    if constexpr (sizeof(W) == 1) return __vmaxu4(a, b);
    else if constexpr (sizeof(W) == 2) return __vmaxu2(a, b);
    else return a > b ? a : b;
}
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_union_linear(const uint32_t* __restrict__ hosts, uint32_t n,
                                                      DevCfg c, const W* __restrict__ lin, uint32_t kthr,
                                                      uint32_t* __restrict__ weight) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint32_t kk = sizeof(W) == 1 ? kthr * 0x01010101u : sizeof(W) == 2 ? kthr * 0x00010001u : kthr;
    const bool vec = ((static_cast<uint64_t>(c.gl) * sizeof(W)) & 15) == 0;
    for (uint32_t h = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; h < n; h += warps) {
        const uint32_t a = hosts[h];
        const W* cell[MAXR];
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
            // all rows' vectors of two iterations issued before any use: 8
            // independent 16-byte loads in flight per lane
            const uint32_t nv = static_cast<uint32_t>(static_cast<uint64_t>(c.gl) * sizeof(W) / 16);
            for (uint32_t q0 = lane; q0 < nv; q0 += 64) {
                uint4 x[2][MAXR];
#pragma unroll
                for (int u = 0; u < 2; ++u)
#pragma unroll
                    for (int i = 0; i < MAXR; ++i)
                        x[u][i] = (i < static_cast<int>(c.rows) && q0 + 32u * u < nv)
                                      ? __ldcs(reinterpret_cast<const uint4*>(cell[i]) + q0 + 32u * u)
                                      : make_uint4(0u, 0u, 0u, 0u);  // neutral for max
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    if (q0 + 32u * u >= nv) break;
                    uint4 m = x[u][0];
#pragma unroll
                    for (int i = 1; i < MAXR; ++i) {
                        if (i >= static_cast<int>(c.rows)) break;
                        m.x = vmax_word<W>(m.x, x[u][i].x);
                        m.y = vmax_word<W>(m.y, x[u][i].y);
                        m.z = vmax_word<W>(m.z, x[u][i].z);
                        m.w = vmax_word<W>(m.w, x[u][i].w);
                    }
                    acc += count_lt_word<W>(m.x, kk, kthr) + count_lt_word<W>(m.y, kk, kthr) +
                           count_lt_word<W>(m.z, kk, kthr) + count_lt_word<W>(m.w, kk, kthr);
                }
            }
            if constexpr (sizeof(W) == 1) acc >>= 3;
            else if constexpr (sizeof(W) == 2) acc >>= 4;
        } else if (vec) {
            const uint32_t nv = static_cast<uint32_t>(static_cast<uint64_t>(c.gl) * sizeof(W) / 16);
            for (uint32_t q = lane; q < nv; q += 32) {
                uint4 m = make_uint4(0, 0, 0, 0);
#pragma unroll
                for (int i = 0; i < MAXR; ++i) {
                    if (i >= static_cast<int>(c.rows)) break;
                    const uint4 x = __ldg(reinterpret_cast<const uint4*>(cell[i]) + q);
                    m.x = vmax_word<W>(m.x, x.x);
                    m.y = vmax_word<W>(m.y, x.y);
                    m.z = vmax_word<W>(m.z, x.z);
                    m.w = vmax_word<W>(m.w, x.w);
                }
                acc += count_lt_word<W>(m.x, kk, kthr) + count_lt_word<W>(m.y, kk, kthr) +
                       count_lt_word<W>(m.z, kk, kthr) + count_lt_word<W>(m.w, kk, kthr);
            }
            if constexpr (sizeof(W) == 1) acc >>= 3;
            else if constexpr (sizeof(W) == 2) acc >>= 4;
        } else {
            for (uint32_t j = lane; j < c.gl; j += 32) {
                uint32_t m = 0;
                for (uint32_t i = 0; i < c.rows; ++i) {
                    const uint32_t v = static_cast<uint32_t>(cell[i < MAXR ? i : 0][j]);
                    m = v > m ? v : m;
                }
                acc += m < kthr;
            }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (lane == 0) weight[h] = acc;
    }
}

// Union rough weight per host (query path, no stamps).
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_union_rough(const uint32_t* __restrict__ hosts, uint32_t n, DevCfg c,
                                                     const W* __restrict__ rough, uint32_t* __restrict__ weight) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x)
        weight[h] = rough_weight<W, MAXR>(c, rough, nullptr, hosts[h], 0, false);
}

// ----------------------------------------------------------------- K8 slide
// slide_recorders (recorders.hpp:113-116): r += (r != expired), wrapping in W,
// over a whole table, 16 bytes per thread step.
template <typename W>
__global__ void __launch_bounds__(256) k_age(W* __restrict__ t, uint64_t words, uint32_t expired) {
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t nv = words * sizeof(W) / 16;
    uint4* v = reinterpret_cast<uint4*>(t);
    const uint32_t ee = sizeof(W) == 1 ? expired * 0x01010101u : sizeof(W) == 2 ? expired * 0x00010001u : expired;
    for (uint64_t q = tid; q < nv; q += stride) {
        uint4 x = v[q];
        if constexpr (sizeof(W) == 1) {
            x.x = __vadd4(x.x, __vcmpne4(x.x, ee) & 0x01010101u);
            x.y = __vadd4(x.y, __vcmpne4(x.y, ee) & 0x01010101u);
            x.z = __vadd4(x.z, __vcmpne4(x.z, ee) & 0x01010101u);
            x.w = __vadd4(x.w, __vcmpne4(x.w, ee) & 0x01010101u);
        } else if constexpr (sizeof(W) == 2) {
            x.x = __vadd2(x.x, __vcmpne2(x.x, ee) & 0x00010001u);
            x.y = __vadd2(x.y, __vcmpne2(x.y, ee) & 0x00010001u);
            x.z = __vadd2(x.z, __vcmpne2(x.z, ee) & 0x00010001u);
            x.w = __vadd2(x.w, __vcmpne2(x.w, ee) & 0x00010001u);
        } else {
            x.x += x.x != ee;
            x.y += x.y != ee;
            x.z += x.z != ee;
            x.w += x.w != ee;
        }
        v[q] = x;
    }
    for (uint64_t q = nv * 16 / sizeof(W) + tid; q < words; q += stride) {
        const W r = t[q];
        t[q] = static_cast<W>(r + (static_cast<uint32_t>(r) != expired ? 1 : 0));
    }
}

// Candidate re-validation after aging (sea.hpp:328-336): flags kept hosts
// (union rough weight >= thr). The caller passes the window it tests against.
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_retain(const uint32_t* __restrict__ csip, uint32_t n, DevCfg c,
                                                const W* __restrict__ rough, uint8_t* __restrict__ keep) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x)
        keep[h] = rough_weight<W, MAXR>(c, rough, nullptr, csip[h], 0, false) >= c.thr;
}

// Re-set the indicator bit of each kept host in every row (sea.hpp:333-335).
__global__ void __launch_bounds__(256) k_si_mark(const uint32_t* __restrict__ hosts, uint32_t n, DevCfg c,
                                                 uint16_t* __restrict__ si) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < n; h += gridDim.x * blockDim.x) {
        const uint32_t a = hosts[h];
        const uint16_t bit = static_cast<uint16_t>(1u << indicator_bit_index(c, a));
        for (uint32_t i = 0; i < c.rows; ++i)
            atomic_or_u16(si + static_cast<uint64_t>(i) * c.cols + column_of(c, i, a), bit);
    }
}

// Merge two ascending lists of distinct hosts (merge path: each thread finds
// its split of the first d outputs by binary search, then emits 8).
__global__ void __launch_bounds__(256) k_merge_sorted(const uint32_t* __restrict__ a, uint32_t na,
                                                      const uint32_t* __restrict__ b, uint32_t nb,
                                                      uint32_t* __restrict__ out) {
    const uint64_t n = static_cast<uint64_t>(na) + nb;
    for (uint64_t d = (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 8; d < n;
         d += static_cast<uint64_t>(gridDim.x) * blockDim.x * 8) {
        uint64_t lo = d > nb ? d - nb : 0, hi = d < na ? d : na;
        while (lo < hi) {  // i = #a among the first d outputs
            const uint64_t mid = (lo + hi) / 2;
            if (a[mid] < b[d - 1 - mid]) lo = mid + 1;
            else hi = mid;
        }
        uint64_t i = lo, j = d - lo;
        const uint64_t e = d + 8 < n ? d + 8 : n;
        for (uint64_t o = d; o < e; ++o) {
            const bool take_a = j >= nb || (i < na && a[i] < b[j]);
            out[o] = take_a ? a[i++] : b[j++];
        }
    }
}

// Fill a table with the expired sentinel (EstimatorArray ctor, sea.hpp:132-133).
template <typename W>
__global__ void k_fill(W* __restrict__ t, uint64_t words, W value) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < words;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        t[q] = value;
}

}  // namespace srla

namespace srla {

// Report entries (srla_entry, 24 bytes) from sorted hosts + union weights and
// the host-built Eq. 9 LUT (bit-identical glibc log1p, host_math.cpp), into a
// device staging buffer that one DMA copies to the caller's pinned memory.
__global__ void __launch_bounds__(256) k_map_entries(const uint32_t* __restrict__ hosts,
                                                     const uint32_t* __restrict__ weight, uint32_t n,
                                                     const double* __restrict__ est,
                                                     const uint8_t* __restrict__ has,
                                                     const uint8_t* __restrict__ sup,
                                                     unsigned long long* __restrict__ out) {
    for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < n; e += gridDim.x * blockDim.x) {
        const uint32_t w = weight[e];
        unsigned long long* o = out + 3ull * e;
        o[0] = static_cast<unsigned long long>(hosts[e]) | (static_cast<unsigned long long>(w) << 32);
        o[1] = static_cast<unsigned long long>(__double_as_longlong(est[w]));
        o[2] = static_cast<unsigned long long>(has[w]) | (static_cast<unsigned long long>(sup[w]) << 8);
    }
}

}  // namespace srla
