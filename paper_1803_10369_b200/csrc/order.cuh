// order.cuh — the scan's ordering phase driven by device-side counts.
//
// Reproduces DetectPipeline::scan_records' record-order semantics
// (pipeline.hpp:134-139, sea.hpp:150-196) without a host
// round trip between kernels: every kernel reads its item count from a device
// counter and is launched over a fixed capacity, and no step needs a sort.
//
//  K2h  crossing events -> host table HT (open addressing on aip):
//       P(a) = atomicMin over the host's crossing packets; the first inserter
//       of a host appends its slot to the host list HL. (Also appends the
//       crossing keys, which the ordered fallback below sorts.)
//  K4h  per first-crossing host: the rows whose indicator bit is clear at
//       chunk start (F, sea.hpp:185-190) and, per open (row, col, bit), the
//       earliest P of any host there: tuple table TT, atomicMin.
//  K4c  classify: F == 0 -> suppressed; earliest at some open key ->
//       inserted (no earlier insertion can have set that bit); otherwise the
//       host is "flagged" and only an ordered resolution can decide it.
//       Inserted hosts set bit P in a bitmap over the chunk's packets (and, if
//       not yet candidates, in a second one).
//  emit The bitmaps compacted in packet order = the sink's push order
//       (pushes are ordered by P): new candidates, src read back from the
//       records at P.
// The host synchronises once per chunk, reads the counters and, only if some
// host was flagged (rare: the indicator table must be saturated locally),
// falls back to the sorted, serial resolution (kernels.cuh K3..K4e), whose
// inputs — the crossing keys and the untouched indicator rows — are intact.
#pragma once

#include "common.cuh"
#include "scan_binned.cuh"

namespace srla {

// device counters of the ordering phase (Engine::octr)
enum OrderCtr : uint32_t {
    kOcEvents = 0,   // sampled events (K1)
    kOcCross = 1,    // crossing events
    kOcHosts = 2,    // distinct crossing hosts
    kOcFlagged = 3,  // hosts needing the ordered resolution
    kOcPushed = 4,   // inserted hosts (sink pushes)
    kOcNew = 5,      // inserted hosts not yet candidates
    kOcPushList = 6, // pushes emitted (collect mode)
    kOcTuples = 7,   // distinct open (row, col, bit) keys
    kOcFallback = 8, // too many flagged hosts for the on-device resolution
    kOcBinOvf = 9,   // a K1 region bin overflowed (k_scan_bin)
    kOcCount = 12
};

__device__ __forceinline__ uint64_t ht_hash(uint64_t key) { return avalanche64(key * 0x9E3779B97F4A7C15ull); }

// insert-or-find `key` (!= 0) in an open-addressing table; returns the slot
// and whether this call inserted it
__device__ __forceinline__ uint64_t ht_slot(unsigned long long* keys, uint64_t mask, unsigned long long key,
                                            bool* inserted) {
    uint64_t s = ht_hash(key) & mask;
    while (true) {
        const unsigned long long k = keys[s];
        if (k == key) {
            *inserted = false;
            return s;
        }
        if (k == 0ull) {
            const unsigned long long prev = atomicCAS(keys + s, 0ull, key);
            if (prev == 0ull) {
                *inserted = true;
                return s;
            }
            if (prev == key) {
                *inserted = false;
                return s;
            }
        }
        s = (s + 1) & mask;
    }
}
__device__ __forceinline__ uint64_t ht_find(const unsigned long long* keys, uint64_t mask, unsigned long long key) {
    uint64_t s = ht_hash(key) & mask;
    while (keys[s] != key) s = (s + 1) & mask;  // present by construction
    return s;
}

struct OrderBufs {
    uint32_t* ctr;                 // OrderCtr counters
    unsigned long long* ht_keys;   // aip + 1
    uint32_t* ht_vals;             // P (0xFFFFFFFF empty)
    uint64_t ht_mask;
    uint32_t* hl;                  // host list: HT slots in insertion order
    unsigned long long* tt_keys;   // ((row * cols + col) * 16 + bit) + 1
    uint32_t* tt_vals;             // earliest P
    uint64_t tt_mask;
    uint32_t* tl;                  // tuple list: TT slots in insertion order
    uint32_t* host_a;              // per listed host: aip, P, open rows, status
    uint32_t* host_p;
    uint64_t* host_f;
    uint32_t* host_cols;           // per listed host: its column in each row (rows <= kOrderRows)
    uint32_t* flist;               // flagged hosts (indices into the host list)
    uint8_t* status;               // 0 suppressed, 1 inserted, 2 flagged
    uint32_t* bm_new;              // bitmaps over the chunk's packets
    uint32_t* bm_push;             // (nullptr unless pushes are collected)
    uint32_t cap;                  // event capacity (bounds every list)
};

constexpr uint32_t kOrderRows = 8;       // rows handled by the device-count ordering
constexpr uint32_t kFlaggedOnDevice = 64; // more flagged hosts than this: sorted fallback

__device__ __forceinline__ bool order_overflow(const OrderBufs& o) { return o.ctr[kOcEvents] > o.cap; }

// K2h: crossing test per sampled event (as of its own packet, kernels.cuh
// rough_weight), host table, crossing keys for the fallback.
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_cross_ht(const uint32_t* __restrict__ ev, uint32_t ev_cap, DevCfg c,
                                                  const W* __restrict__ rough, const uint32_t* __restrict__ stamp,
                                                  uint64_t* __restrict__ xkeys, OrderBufs o) {
    if (order_overflow(o)) return;
    const uint32_t n_ev = o.ctr[kOcEvents];
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
        const uint32_t pos = warp_append(o.ctr + kOcCross, cross ? 1u : 0u);
        if (!cross) continue;
        xkeys[pos] = (static_cast<uint64_t>(a) << 32) | p;
        bool fresh = false;
        const uint64_t s = ht_slot(o.ht_keys, o.ht_mask, static_cast<unsigned long long>(a) + 1ull, &fresh);
        atomicMin(o.ht_vals + s, p);
        if (fresh) o.hl[atomicAdd(o.ctr + kOcHosts, 1u)] = static_cast<uint32_t>(s);
    }
}

// K5 with a device event count
template <typename W, int MAXR>
__global__ void __launch_bounds__(256) k_commit_dev(const uint32_t* __restrict__ ev, uint32_t ev_cap, DevCfg c,
                                                    W* __restrict__ rough, uint32_t* __restrict__ stamp, OrderBufs o) {
    if (order_overflow(o)) return;
    const uint32_t n_ev = o.ctr[kOcEvents];
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

__device__ __forceinline__ unsigned long long tuple_key(const DevCfg& c, uint32_t row, uint32_t col, uint32_t bit) {
    return ((static_cast<unsigned long long>(row) * c.cols + col) * kIndicatorBits + bit) + 1ull;
}

// K4h: open rows per host (indicator state at chunk start) and the earliest
// P per open (row, col, bit)
__global__ void __launch_bounds__(256) k_si_open(DevCfg c, const uint16_t* __restrict__ si, OrderBufs o) {
    if (order_overflow(o)) return;
    const uint32_t hn = o.ctr[kOcHosts];
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < hn; h += gridDim.x * blockDim.x) {
        const uint32_t s = o.hl[h];
        const uint32_t a = static_cast<uint32_t>(o.ht_keys[s] - 1ull);
        const uint32_t p = o.ht_vals[s];
        const uint32_t b = indicator_bit_index(c, a);
        uint64_t F = 0;
        for (uint32_t i = 0; i < c.rows; ++i) {
            const uint32_t col = column_of(c, i, a);
            o.host_cols[static_cast<uint64_t>(h) * kOrderRows + i] = col;
            if (si[static_cast<uint64_t>(i) * c.cols + col] & (1u << b)) continue;
            F |= 1ull << i;
            bool fresh = false;
            const uint64_t ts = ht_slot(o.tt_keys, o.tt_mask, tuple_key(c, i, col, b), &fresh);
            atomicMin(o.tt_vals + ts, p);
            if (fresh) o.tl[atomicAdd(o.ctr + kOcTuples, 1u)] = static_cast<uint32_t>(ts);
        }
        o.host_a[h] = a;
        o.host_p[h] = p;
        o.host_f[h] = F;
    }
}

// an inserted host: a sink push at packet P, and a new candidate unless the
// list already holds it (CandidateList::insert, sea.hpp:58-62)
__device__ __forceinline__ void mark_inserted(uint32_t a, uint32_t p, const unsigned long long* __restrict__ cset,
                                              uint64_t cset_mask, const OrderBufs& o) {
    atomicAdd(o.ctr + kOcPushed, 1u);
    if (o.bm_push) atomicOr(o.bm_push + (p >> 5), 1u << (p & 31u));
    const unsigned long long key = static_cast<unsigned long long>(a) + 1ull;
    uint64_t s = avalanche64(a) & cset_mask;  // kernels.cuh cset_slot
    while (true) {
        const unsigned long long v = cset[s];
        if (v == 0ull) break;
        if (v == key) return;
        s = (s + 1) & cset_mask;
    }
    atomicOr(o.bm_new + (p >> 5), 1u << (p & 31u));
}

// K4c: classify; inserted hosts mark the packet bitmaps
__global__ void __launch_bounds__(256) k_order_classify(DevCfg c, const unsigned long long* __restrict__ cset,
                                                        uint64_t cset_mask, OrderBufs o) {
    if (order_overflow(o)) return;
    const uint32_t hn = o.ctr[kOcHosts];
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < hn; h += gridDim.x * blockDim.x) {
        const uint32_t a = o.host_a[h], p = o.host_p[h];
        uint64_t F = o.host_f[h];
        uint8_t st = 0;
        if (F) {
            st = 2;
            const uint32_t b = indicator_bit_index(c, a);
            while (F) {
                const uint32_t i = __ffsll(F) - 1;
                F &= F - 1;
                const uint64_t ts = ht_find(o.tt_keys, o.tt_mask, tuple_key(c, i, column_of(c, i, a), b));
                if (o.tt_vals[ts] == p) {
                    st = 1;
                    break;
                }
            }
        }
        o.status[h] = st;
        if (st == 2) o.flist[atomicAdd(o.ctr + kOcFlagged, 1u)] = h;
        if (st != 1) continue;
        mark_inserted(a, p, cset, cset_mask, o);
    }
}

// On-device ordered resolution of the (few) flagged hosts, ascending P: a
// flagged host is inserted iff in some open row no host inserted before it
// (smaller P) shares its (row, col, bit) — the reference's "bit not in the
// row's indicator" test at P (sea.hpp:185-190), as kernels.cuh k_serial
// decides it. Hosts sharing a key share the row's open state, so the test
// needs only the hosts' columns, bits and statuses. One block; hosts already
// decided are final, earlier flagged hosts are resolved first.
__global__ void __launch_bounds__(1024) k_resolve_flagged(DevCfg c, const unsigned long long* __restrict__ cset,
                                                          uint64_t cset_mask, OrderBufs o) {
    if (order_overflow(o)) return;
    const uint32_t nf = o.ctr[kOcFlagged];
    if (nf == 0) return;
    if (nf > kFlaggedOnDevice) {
        if (threadIdx.x == 0) o.ctr[kOcFallback] = 1;
        return;
    }
    __shared__ uint32_t s_f[kFlaggedOnDevice];
    if (threadIdx.x == 0) {  // ascending P (insertion sort of <= 64 entries)
        for (uint32_t i = 0; i < nf; ++i) {
            const uint32_t h = o.flist[i];
            uint32_t j = i;
            while (j > 0 && o.host_p[s_f[j - 1]] > o.host_p[h]) {
                s_f[j] = s_f[j - 1];
                --j;
            }
            s_f[j] = h;
        }
    }
    __syncthreads();
    const uint32_t hn = o.ctr[kOcHosts];
    for (uint32_t f = 0; f < nf; ++f) {
        const uint32_t h = s_f[f];
        const uint32_t a = o.host_a[h], p = o.host_p[h];
        const uint32_t b = indicator_bit_index(c, a);
        uint64_t F = o.host_f[h];
        bool inserted = false;
        while (F && !inserted) {
            const uint32_t i = __ffsll(F) - 1;
            F &= F - 1;
            const uint32_t col = o.host_cols[static_cast<uint64_t>(h) * kOrderRows + i];
            bool blocked = false;
            for (uint32_t q = threadIdx.x; q < hn && !blocked; q += blockDim.x)
                blocked = o.status[q] == 1 && o.host_p[q] < p && ((o.host_f[q] >> i) & 1ull) &&
                          o.host_cols[static_cast<uint64_t>(q) * kOrderRows + i] == col &&
                          indicator_bit_index(c, o.host_a[q]) == b;
            inserted = !__syncthreads_or(blocked);
        }
        if (threadIdx.x == 0) {
            o.status[h] = inserted ? 1 : 0;
            if (inserted) mark_inserted(a, p, cset, cset_mask, o);
        }
        __syncthreads();
    }
}

// ---- ordered compaction of a packet bitmap (set bits in packet order)
constexpr uint32_t kBitsThreads = 256;
constexpr uint32_t kBitsPerThread = 8;                          // words
constexpr uint32_t kBitsWords = kBitsThreads * kBitsPerThread;  // words per block

__global__ void __launch_bounds__(kBitsThreads) k_bits_count(const uint32_t* __restrict__ bm, uint32_t words,
                                                             uint32_t* __restrict__ bcnt) {
    const uint32_t w0 = blockIdx.x * kBitsWords;
    uint32_t n = 0;
    for (uint32_t q = threadIdx.x; q < kBitsWords && w0 + q < words; q += kBitsThreads) n += __popc(bm[w0 + q]);
    n = __reduce_add_sync(0xFFFFFFFFu, n);
    __shared__ uint32_t s[kBitsThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = n;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (uint32_t j = 0; j < kBitsThreads / 32; ++j) t += s[j];
        bcnt[blockIdx.x] = t;
    }
}

// exclusive scan of the block counts in one block; total -> *total
__global__ void __launch_bounds__(1024) k_bits_scan(uint32_t* __restrict__ bcnt, uint32_t nblocks,
                                                    uint32_t* __restrict__ total) {
    __shared__ uint32_t s_w[32];
    __shared__ uint32_t s_carry;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (uint32_t b0 = 0; b0 < nblocks; b0 += 1024) {
        const uint32_t b = b0 + threadIdx.x;
        const uint32_t v = b < nblocks ? bcnt[b] : 0u;
        uint32_t incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if ((threadIdx.x & 31) >= static_cast<uint32_t>(o)) incl += t;
        }
        if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = incl;
        __syncthreads();
        uint32_t wb = 0;
        for (uint32_t j = 0; j < (threadIdx.x >> 5); ++j) wb += s_w[j];
        const uint32_t carry = s_carry;
        if (b < nblocks) bcnt[b] = carry + wb + incl - v;
        __syncthreads();
        if (threadIdx.x == 1023) s_carry = carry + wb + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = s_carry;
}

// set bits -> out[boff + rank] = src of packet P (recs: the chunk's records,
// 3 words each); the bitmap is cleared on the way
__global__ void __launch_bounds__(kBitsThreads) k_bits_emit(uint32_t* __restrict__ bm, uint32_t words,
                                                            const uint32_t* __restrict__ boff,
                                                            const uint32_t* __restrict__ recs,
                                                            uint32_t* __restrict__ out) {
    const uint32_t w0 = blockIdx.x * kBitsWords + threadIdx.x * kBitsPerThread;
    uint32_t v[kBitsPerThread];
    uint32_t n = 0;
#pragma unroll
    for (uint32_t j = 0; j < kBitsPerThread; ++j) {
        v[j] = w0 + j < words ? bm[w0 + j] : 0u;
        n += __popc(v[j]);
    }
    uint32_t incl = n;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if ((threadIdx.x & 31) >= static_cast<uint32_t>(o)) incl += t;
    }
    __shared__ uint32_t s_w[kBitsThreads / 32];
    if ((threadIdx.x & 31) == 31) s_w[threadIdx.x >> 5] = incl;
    __syncthreads();
    uint32_t pos = boff[blockIdx.x] + incl - n;
    for (uint32_t j = 0; j < (threadIdx.x >> 5); ++j) pos += s_w[j];
#pragma unroll
    for (uint32_t j = 0; j < kBitsPerThread; ++j) {
        uint32_t x = v[j];
        if (!x) continue;
        bm[w0 + j] = 0u;
        while (x) {
            const uint32_t bit = __ffs(x) - 1;
            x &= x - 1;
            const uint32_t p = (w0 + j) * 32u + bit;
            out[pos++] = recs[3ull * p + 1];
        }
    }
}

// after the counters were read and nothing was flagged: set the inserted
// hosts' indicator bit in all rows (sea.hpp:193-195; kernels.cuh k_si_set)
__global__ void __launch_bounds__(256) k_order_si_set(DevCfg c, uint16_t* __restrict__ si, OrderBufs o, uint32_t hn) {
    for (uint32_t h = blockIdx.x * blockDim.x + threadIdx.x; h < hn; h += gridDim.x * blockDim.x) {
        if (o.status[h] != 1) continue;
        const uint32_t a = o.host_a[h];
        const uint16_t bit = static_cast<uint16_t>(1u << indicator_bit_index(c, a));
        for (uint32_t i = 0; i < c.rows; ++i)
            atomic_or_u16(si + static_cast<uint64_t>(i) * c.cols + column_of(c, i, a), bit);
    }
}
// empty the host and tuple tables through their slot lists
__global__ void __launch_bounds__(256) k_order_clear(OrderBufs o, uint32_t hn, uint32_t tn) {
    const uint32_t m = hn > tn ? hn : tn;
    for (uint32_t q = blockIdx.x * blockDim.x + threadIdx.x; q < m; q += gridDim.x * blockDim.x) {
        if (q < hn) {
            const uint32_t s = o.hl[q];
            o.ht_keys[s] = 0ull;
            o.ht_vals[s] = 0xFFFFFFFFu;
        }
        if (q < tn) {
            const uint32_t s = o.tl[q];
            o.tt_keys[s] = 0ull;
            o.tt_vals[s] = 0xFFFFFFFFu;
        }
    }
}

// ---- small batches: EstimatorArray::scan_ip_pair (sea.hpp:150-196) record by
// record on ONE thread — for a few records the serial algorithm itself beats
// the parallel chunk pipeline's fixed cost (the drop-in's per-pair calls).
// Linear marks go straight to the table (they commute with pending binned
// marks); pushes are appended to `pushes`, the new candidates (not in the
// candidate hash, CandidateList::insert, sea.hpp:58-62) to `fresh`, each with
// its count in ctr[kOcPushList] / ctr[kOcNew]. A host is pushed at most once
// per call: its indicator bit is set in every row on insertion.
template <typename W, int MAXR>
__global__ void k_scan_serial(const uint32_t* __restrict__ recs, uint32_t n, DevCfg c, W* __restrict__ lin, int nib,
                              EpochCfg ep, W* __restrict__ rough, uint16_t* __restrict__ si,
                              const unsigned long long* __restrict__ cset, uint64_t cset_mask,
                              uint32_t* __restrict__ pushes, uint32_t* __restrict__ fresh,
                              uint32_t* __restrict__ ctr) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;
    const uint64_t rrow = static_cast<uint64_t>(c.cols) * c.g;
    uint32_t np = 0, nn = 0, ev = 0;
    for (uint32_t r = 0; r < n; ++r) {
        const uint32_t aip = recs[3ull * r + 1], bip = recs[3ull * r + 2];
        uint32_t cols[MAXR];
        for (uint32_t i = 0; i < c.rows && i < MAXR; ++i) cols[i] = column_of(c, i, aip);
        const uint32_t sample = hash_u32k(c.sub_sample, c.kh_sample, bip);
        const uint32_t lslot = c.gl_mask ? (sample & c.gl_mask) : (sample % c.gl);
        for (uint32_t i = 0; i < c.rows; ++i) {  // linear marks, every pair (sea.hpp:155-161)
            const uint64_t w = i * lrow + static_cast<uint64_t>(cols[i]) * c.gl + lslot;
            if (ep.on) mark_epoch_global(reinterpret_cast<uint8_t*>(lin), w, ep.row_words, ep.cur, ep.hist);
            else if (nib) mark_nibble_global(reinterpret_cast<uint8_t*>(lin), w);
            else if (sizeof(W) == 4) lin[w] = W(0);
            else mark_word<W>(lin + (w & ~static_cast<uint64_t>(4 / sizeof(W) - 1)),
                              static_cast<uint32_t>(w & (4 / sizeof(W) - 1)));  // atomic: commutes with the split's marks
        }
        if ((sample & c.tau_mask) != 0u) continue;  // not sampled (sea.hpp:164)
        ++ev;
        const uint32_t rslot = reduce32(hash_u32k(c.sub_rslot, c.kh_rslot, bip), c.g);
        for (uint32_t i = 0; i < c.rows; ++i) rough[i * rrow + static_cast<uint64_t>(cols[i]) * c.g + rslot] = W(0);
        uint32_t weight = 0;  // union rough weight (sea.hpp:172-181)
        for (uint32_t j = 0; j < c.g; ++j) {
            bool active = true;
            for (uint32_t i = 0; i < c.rows && active; ++i)
                active = static_cast<uint32_t>(rough[i * rrow + static_cast<uint64_t>(cols[i]) * c.g + j]) < c.k;
            weight += active;
        }
        if (weight < c.thr) continue;
        const uint16_t bit = static_cast<uint16_t>(1u << indicator_bit_index(c, aip));
        uint16_t joined = 0xFFFF;
        for (uint32_t i = 0; i < c.rows; ++i) joined &= si[static_cast<uint64_t>(i) * c.cols + cols[i]];
        if (joined & bit) continue;  // already listed this slice (sea.hpp:185-190)
        pushes[np++] = aip;
        for (uint32_t i = 0; i < c.rows; ++i) si[static_cast<uint64_t>(i) * c.cols + cols[i]] |= bit;
        const unsigned long long key = static_cast<unsigned long long>(aip) + 1ull;
        uint64_t s = avalanche64(aip) & cset_mask;
        bool present = false;
        while (cset[s] != 0ull) {
            if (cset[s] == key) {
                present = true;
                break;
            }
            s = (s + 1) & cset_mask;
        }
        if (!present) {  // a host pushed twice in one call was re-listed only if its bit was cleared: never
            bool dup = false;
            for (uint32_t q = 0; q < nn && !dup; ++q) dup = fresh[q] == aip;
            if (!dup) fresh[nn++] = aip;
        }
    }
    ctr[kOcEvents] = ev;
    ctr[kOcPushList] = np;
    ctr[kOcNew] = nn;
}

}  // namespace srla
