// digest.cuh — block digests of sketch rows in the reference's byte layout
// (the raw spans of sea.hpp:341-346, as snapshot.hpp:128-132 writes them),
// computed where the state lives. Full-size parity compares
// 64 GiB of recorders per slice against the reference without moving them:
// per 1 MiB block of a row, the wrapping sum over its little-endian 8-byte
// words w_i (zero-padded) of avalanche64(w_i ^ avalanche64(i + 1)), i = the
// word's index in the row. The test-side checker computes the same
// sums over the reference's own rows.
#pragma once

#include "common.cuh"

namespace srla {

constexpr uint32_t kDigestBlockShift = 20;  // 1 MiB of reference-layout bytes per block
constexpr uint32_t kDigestThreads = 256;

// How a row is stored on the device relative to the reference layout.
enum DigestLayout : uint32_t {
    kDigestRaw = 0,     // identical bytes (literal words, indicators, records)
    kDigestNibble = 1,  // two recorders per byte, low nibble first (nibble.cuh)
    kDigestEpoch = 2,   // u8 epoch stamps: value = min((cur - s) & 0xFF, expired) (epoch.cuh)
};

struct DigestSrc {
    const uint8_t* p;  // device bytes of the row (packed for nibble tables)
    uint64_t bytes;    // reference-layout bytes of the row
    uint32_t layout, cur, expired;
};

// Reference-layout word o (bytes 8o .. 8o+7, zero past `bytes`).
__device__ __forceinline__ uint64_t digest_word(const DigestSrc& s, uint64_t o) {
    const uint64_t b0 = o * 8;
    const uint32_t m = static_cast<uint32_t>(s.bytes - b0 < 8 ? s.bytes - b0 : 8);
    uint64_t w = 0;
    if (s.layout == kDigestNibble) {  // 8 recorders = 4 packed bytes
        const uint8_t* q = s.p + b0 / 2;
        uint32_t packed = 0;
        if (m == 8 && (reinterpret_cast<uintptr_t>(q) & 3) == 0) packed = *reinterpret_cast<const uint32_t*>(q);
        else
            for (uint32_t j = 0; j < (m + 1) / 2; ++j) packed |= static_cast<uint32_t>(q[j]) << (8 * j);
        for (uint32_t j = 0; j < m; ++j) w |= static_cast<uint64_t>((packed >> (4 * j)) & 0xFu) << (8 * j);
        return w;
    }
    const uint8_t* q = s.p + b0;
    if (m == 8 && (reinterpret_cast<uintptr_t>(q) & 7) == 0) w = *reinterpret_cast<const uint64_t*>(q);
    else
        for (uint32_t j = 0; j < m; ++j) w |= static_cast<uint64_t>(q[j]) << (8 * j);
    if (s.layout == kDigestEpoch) {
        uint64_t v = 0;
        for (uint32_t j = 0; j < m; ++j) {
            const uint32_t a = (s.cur - static_cast<uint32_t>((w >> (8 * j)) & 0xFFu)) & 0xFFu;
            v |= static_cast<uint64_t>(a < s.expired ? a : s.expired) << (8 * j);
        }
        w = v;
    }
    return w;
}

// One CTA per 1 MiB block: coalesced 8-byte reads, a block-wide sum.
__global__ void __launch_bounds__(kDigestThreads) k_block_sums(DigestSrc s, uint64_t* __restrict__ out) {
    const uint64_t words = (s.bytes + 7) / 8;
    const uint64_t per_block = (1ull << kDigestBlockShift) / 8;
    const uint64_t w0 = static_cast<uint64_t>(blockIdx.x) * per_block;
    const uint64_t w1 = words < w0 + per_block ? words : w0 + per_block;
    uint64_t acc = 0;
    for (uint64_t o = w0 + threadIdx.x; o < w1; o += kDigestThreads) acc += avalanche64(digest_word(s, o) ^ avalanche64(o + 1));
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
    __shared__ uint64_t part[kDigestThreads / 32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint64_t t = 0;
        for (uint32_t j = 0; j < kDigestThreads / 32; ++j) t += part[j];
        out[blockIdx.x] = t;
    }
}

}  // namespace srla
