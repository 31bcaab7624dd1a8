// nibble.cuh — 4-bit literal linear recorders (z <= 4 on binned tables).
//
// The reference stores a z <= 8 recorder in a byte (recorders.hpp:64-66); for
// z <= 4 the value range [0, 2^z - 1] fits a nibble, so the engine keeps the
// linear table packed two recorders per byte: recorder word w lives in byte
// w >> 1, low nibble for even w. The streamed passes (mark apply + fused
// count_active / slide_recorders, the report gather) move half the bytes; the
// row export/import convert to and from the reference's byte layout.
#pragma once

#include "common.cuh"
#include "scan_binned.cuh"

namespace srla {

constexpr uint32_t kNibLo = 0x0F0F0F0Fu;
constexpr uint32_t kNibOne = 0x11111111u;

// slide_recorders (recorders.hpp:113-116) on 8 packed recorders:
// r + (r != expired); r <= expired, so no nibble carries out
__device__ __forceinline__ uint32_t nib_age(uint32_t x, uint32_t e8) {
    const uint32_t d = x ^ e8;
    return x + ((d | (d >> 1) | (d >> 2) | (d >> 3)) & kNibOne);
}
constexpr uint32_t kByteHi = 0x80808080u;
// SWAR ">= k" on the even (low) nibbles of x, one per byte: bit 7 of byte j
// is set iff recorder 2j >= k (x & kNibLo <= 15 and k <= 16: 0x80 | v - k
// never borrows across bytes). Other bits are junk: mask with kByteHi.
__device__ __forceinline__ uint32_t nib_ge_even(uint32_t x, uint32_t k4) { return ((x & kNibLo) | kByteHi) - k4; }
__device__ __forceinline__ uint32_t nib_ge_odd(uint32_t x, uint32_t k4) { return (((x >> 4) & kNibLo) | kByteHi) - k4; }
// number of the 8 packed recorders with value < k (k4 = k in every byte)
__device__ __forceinline__ uint32_t nib_count_lt(uint32_t x, uint32_t k4) {
    return 8u - __popc(nib_ge_even(x, k4) & kByteHi) - __popc(nib_ge_odd(x, k4) & kByteHi);
}

// k_slice_apply_bulk for nibble tables: fine slices of 2^f.shift recorders
// (2^(f.shift-1) bytes, a multiple of 16). Each stage bulk-loads a slice AND
// its mark list into shared memory on one mbarrier (the marks' global-load
// latency was the stall), double-buffered; marks are shared-memory ANDs (two
// recorders share a byte); mode 0 apply / 1 apply + age / 2 apply + count
// active (pre-age) + age; the slice is bulk-stored back.
// Shared memory: 2 x (slice bytes + f.cap x 2 B).
__global__ void __launch_bounds__(1024) k_slice_apply_nib(uint8_t* __restrict__ lin, uint64_t row_words, FineCfg f,
                                                         uint32_t f_end, int mode, uint32_t k, uint32_t expired,
                                                         unsigned long long* __restrict__ counts) {
    extern __shared__ __align__(128) uint8_t s_raw[];
    __shared__ __align__(8) uint64_t s_bar[2];
    __shared__ unsigned long long s_part[2][32];
    __shared__ uint32_t s_n[2];
    const uint32_t tid = threadIdx.x;
    const uint32_t slice_bytes = (1u << f.shift) >> 1;
    const uint32_t stage = slice_bytes + f.cap * 2u;  // slice | marks (f.cap is a multiple of 8)
    const uint32_t k4 = k * 0x01010101u, e8 = expired * kNibOne;
    auto next_slice = [&](uint32_t from) -> uint32_t {
        for (uint32_t fb = from; fb < f_end; fb += gridDim.x)
            if (mode != 0 || f.count[fb] != 0) return fb;
        return f_end;
    };
    auto gaddr = [&](uint32_t fb) { return lin + ((static_cast<uint64_t>(fb) << f.shift) >> 1); };
    auto issue = [&](uint32_t fb, uint32_t b) {  // thread 0
        const uint32_t n = min(f.count[fb], f.cap);
        const uint32_t mb = (n * 2u + 15u) & ~15u;
        s_n[b] = n;
        mbar_expect_tx(&s_bar[b], slice_bytes + mb);
        bulk_load(s_raw + b * stage, gaddr(fb), slice_bytes, &s_bar[b]);
        if (mb) bulk_load(s_raw + b * stage + slice_bytes, f.bins + static_cast<uint64_t>(fb) * f.cap, mb, &s_bar[b]);
    };
    if (tid == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
    }
    __syncthreads();
    uint32_t cur = next_slice(blockIdx.x);
    if (tid == 0 && cur < f_end) issue(cur, 0);
    for (uint32_t i = 0; cur < f_end; ++i) {
        const uint32_t b = i & 1u;
        const uint32_t nxt = next_slice(cur + gridDim.x);
        if (tid == 0 && nxt < f_end) {
            bulk_wait_read_all();  // the other buffer's store (slice i-1) has left shared memory
            issue(nxt, b ^ 1u);
        }
        mbar_wait(&s_bar[b], (i >> 1) & 1u);
        if (tid == 0) atomicAdd(f.streamed, static_cast<unsigned long long>(slice_bytes));
        uint8_t* sb = s_raw + b * stage;
        unsigned int* s32 = reinterpret_cast<unsigned int*>(sb);
        const uint32_t n = s_n[b];
        const uint16_t* e = reinterpret_cast<const uint16_t*>(sb + slice_bytes);
        const uint4* ev = reinterpret_cast<const uint4*>(e);
        auto mark = [&](uint32_t o) { atomicAnd(s32 + (o >> 3), ~(0xFu << (4u * (o & 7u)))); };
        for (uint32_t q = tid; q < n / 8; q += blockDim.x) {
            const uint4 x = ev[q];
            mark(x.x & 0xFFFF); mark(x.x >> 16);
            mark(x.y & 0xFFFF); mark(x.y >> 16);
            mark(x.z & 0xFFFF); mark(x.z >> 16);
            mark(x.w & 0xFFFF); mark(x.w >> 16);
        }
        for (uint32_t q = (n / 8) * 8 + tid; q < n; q += blockDim.x) mark(e[q]);
        __syncthreads();
        if (mode != 0) {
            const uint64_t w0 = static_cast<uint64_t>(cur) << f.shift;
            const uint64_t row_a = w0 / row_words;
            const uint64_t split = (row_a + 1) * row_words;  // first word of the next row
            unsigned long long acc_a = 0, acc_b = 0;
            uint4* sv = reinterpret_cast<uint4*>(sb);
            const uint32_t nv = slice_bytes / 16;
            for (uint32_t q = tid; q < nv; q += blockDim.x) {
                uint4 x = sv[q];
                if (mode == 2) {
                    const uint32_t c = nib_count_lt(x.x, k4) + nib_count_lt(x.y, k4) + nib_count_lt(x.z, k4) +
                                       nib_count_lt(x.w, k4);
                    if (w0 + static_cast<uint64_t>(q) * 32 < split) acc_a += c;  // 32 recorders per vector
                    else acc_b += c;
                }
                x.x = nib_age(x.x, e8);
                x.y = nib_age(x.y, e8);
                x.z = nib_age(x.z, e8);
                x.w = nib_age(x.w, e8);
                sv[q] = x;
            }
            if (mode == 2) {
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
                unsigned long long sa = 0, sb2 = 0;
                for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
                    sa += s_part[0][w];
                    sb2 += s_part[1][w];
                }
                if (sa) atomicAdd(counts + row_a, sa);
                if (sb2) atomicAdd(counts + row_a + 1, sb2);
            }
        } else {
            fence_proxy_async_smem();
            __syncthreads();
        }
        if (tid == 0) bulk_store(gaddr(cur), sb, slice_bytes);
        cur = nxt;
    }
    if (tid == 0) bulk_wait_all();
}

// union_linear_weight (sea.hpp:232-243) on a nibble table: slot j counts
// iff max over rows of recorder j < kthr. A cell of g' recorders is g'/2
// bytes, so a half-warp takes a candidate (two vectors per row per lane in
// flight: 8 x 16 B with u = 4) when g' is a multiple of 32; otherwise a warp
// walks the recorders one by one.
template <int MAXR>
__global__ void __launch_bounds__(256) k_union_linear_nib(const uint32_t* __restrict__ hosts, uint32_t n, DevCfg c,
                                                          const uint8_t* __restrict__ lin, uint32_t kthr,
                                                          uint32_t* __restrict__ weight) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t warp0 = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t lrow = static_cast<uint64_t>(c.cols) * c.gl;  // recorders per row
    const uint32_t k4 = kthr * 0x01010101u;
    auto cells = [&](uint32_t a, const uint8_t** cell) {
#pragma unroll
        for (int i = 0; i < MAXR; ++i)
            if (i < static_cast<int>(c.rows)) cell[i] = lin + ((i * lrow + static_cast<uint64_t>(column_of(c, i, a)) * c.gl) >> 1);
    };
    if ((c.gl & 31u) == 0 && MAXR <= 4) {
        const uint32_t sub = lane >> 4, sl = lane & 15u;
        const uint32_t nv = c.gl / 32;  // 16-byte vectors per cell
        for (uint64_t pair = warp0; pair * 2 < n; pair += warps) {
            const uint64_t h = pair * 2 + sub;
            const uint32_t a = h < n ? hosts[h] : 0u;
            // lane i of each half hashes row i; the half shares the columns
            const uint32_t colv = sl < c.rows ? column_of(c, sl, a) : 0u;
            const uint8_t* cell[MAXR];
#pragma unroll
            for (int i = 0; i < MAXR; ++i)
                cell[i] = lin + ((i * lrow + static_cast<uint64_t>(__shfl_sync(0xFFFFFFFFu, colv, i, 16)) * c.gl) >> 1);
            uint32_t acc = 0;
            if (h < n) {
                for (uint32_t q0 = sl; q0 < nv; q0 += 32) {
                    uint4 x[2][MAXR];
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int i = 0; i < MAXR; ++i)
                            x[u][i] = (i < static_cast<int>(c.rows) && q0 + 16u * u < nv)
                                          ? __ldcs(reinterpret_cast<const uint4*>(cell[i]) + q0 + 16u * u)
                                          : make_uint4(0u, 0u, 0u, 0u);  // value 0: never >= k
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        if (q0 + 16u * u >= nv) break;
                        // slot active in the union <=> no row has it >= k
                        uint32_t ge[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
                        for (int i = 0; i < MAXR; ++i) {
                            ge[0] |= nib_ge_even(x[u][i].x, k4); ge[1] |= nib_ge_odd(x[u][i].x, k4);
                            ge[2] |= nib_ge_even(x[u][i].y, k4); ge[3] |= nib_ge_odd(x[u][i].y, k4);
                            ge[4] |= nib_ge_even(x[u][i].z, k4); ge[5] |= nib_ge_odd(x[u][i].z, k4);
                            ge[6] |= nib_ge_even(x[u][i].w, k4); ge[7] |= nib_ge_odd(x[u][i].w, k4);
                        }
                        uint32_t g = 0;
#pragma unroll
                        for (int j = 0; j < 8; ++j) g += __popc(ge[j] & kByteHi);
                        acc += 32u - g;
                    }
                }
            }
#pragma unroll
            for (int o = 8; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
            if (sl == 0 && h < n) weight[h] = acc;
        }
        return;
    }
    for (uint32_t h = warp0; h < n; h += warps) {
        const uint8_t* cell[MAXR];
        cells(hosts[h], cell);
        uint32_t acc = 0;
        for (uint32_t j = lane; j < c.gl; j += 32) {
            uint32_t m = 0;
            for (uint32_t i = 0; i < c.rows; ++i) {
                const uint32_t v = (cell[i < MAXR ? i : 0][j >> 1] >> (4u * (j & 1u))) & 0xFu;
                m = v > m ? v : m;
            }
            acc += m < kthr;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
        if (lane == 0) weight[h] = acc;
    }
}

// count_active (recorders.hpp:119-129) per row of a nibble table; grid.y = row.
__global__ void __launch_bounds__(256) k_row_active_nib(const uint8_t* __restrict__ lin, uint64_t row_words, uint32_t k,
                                                        unsigned long long* __restrict__ counts) {
    const uint32_t row = blockIdx.y;
    const uint64_t bytes = row_words >> 1;
    const uint8_t* base = lin + row * bytes;
    const uint32_t k4 = k * 0x01010101u;
    unsigned long long acc = 0;
    const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
    const uint64_t nw = bytes / 4;  // row bytes are a multiple of 16 in nibble mode
    const unsigned int* w = reinterpret_cast<const unsigned int*>(base);
    for (uint64_t q = tid; q < nw; q += stride) acc += nib_count_lt(w[q], k4);
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, o);
    __shared__ unsigned long long part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long s = 0;
        for (uint32_t i = 0; i < blockDim.x / 32; ++i) s += part[i];
        if (s) atomicAdd(counts + row, s);
    }
}

// packed table -> a byte per recorder (Engine::leave_nibble)
__global__ void __launch_bounds__(256) k_unpack_nib(const uint8_t* __restrict__ packed, uint64_t nbytes,
                                                    uint8_t* __restrict__ wide) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < nbytes;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint8_t v = packed[q];
        wide[2 * q] = v & 0xFu;
        wide[2 * q + 1] = v >> 4;
    }
}

// a byte per recorder (values <= 15, checked by the caller) -> packed
__global__ void __launch_bounds__(256) k_pack_nib(const uint8_t* __restrict__ wide, uint64_t nbytes,
                                                  uint8_t* __restrict__ packed) {
    for (uint64_t q = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < nbytes;
         q += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        packed[q] = static_cast<uint8_t>(wide[2 * q] | (wide[2 * q + 1] << 4));
}

}  // namespace srla
