// common.cuh — device-side configuration, hashing and recorder arithmetic
// shared by every SRLA kernel. sm_100a only.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace srla {

constexpr uint32_t kMaxRows = 64;        // sea.hpp:349
constexpr uint32_t kIndicatorBits = 16;  // sea.hpp:21
constexpr uint32_t kSampleHash = 0;      // hash.hpp:70
constexpr uint32_t kRoughSlotHash = 1;   // hash.hpp:71
constexpr uint32_t kIndicatorHash = 2;   // hash.hpp:72
constexpr uint32_t kRowHashBase = 8;     // hash.hpp:73
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

// Everything a kernel needs to place a packet, passed by value (lives in the
// kernel parameter bank; row sub-keys are indexed dynamically from there).
struct DevCfg {
    uint32_t rows, cols, g, gl;  // u, v, g, g'
    uint32_t k;                  // window
    uint32_t expired;            // 2^z - 1 (recorders.hpp:39-42)
    uint32_t tau_mask;           // sampled <=> (sample & tau_mask) == 0 (ctz >= tau)
    uint32_t thr;                // ceil(rho*g - 1e-9)
    uint32_t gl_mask;            // g' - 1 when g' is a power of two, else 0
    uint32_t wbytes;
    uint64_t sub_sample, sub_rslot, sub_ind;
    uint64_t sub_row[kMaxRows];
    // sub_hi_term(sub) of each sub-key (hash_u32k): the high word's share of
    // the first multiply, constant per hash function
    uint32_t kh_sample, kh_rslot, kh_row[kMaxRows];
};

// hash.hpp:9-13 (splitmix64 finalizer)
__host__ __device__ __forceinline__ uint64_t avalanche64(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
// HashFamily per-index sub-key, precomputed once (hash.hpp:54)
__host__ __device__ __forceinline__ uint64_t sub_key(uint64_t seed, uint32_t index) {
    return avalanche64(seed + kGolden * static_cast<uint64_t>(index + 1u));
}
// HashFamily::u32 with a precomputed sub-key (hash.hpp:53-56)
__host__ __device__ __forceinline__ uint32_t hash_u32(uint64_t sub, uint32_t key) {
    return static_cast<uint32_t>(avalanche64(sub ^ static_cast<uint64_t>(key)));
}
// hash_u32 in 32-bit halves (the key only touches the low word): with
// x = sub ^ key, (x ^ x >> 30).hi depends on sub alone, so its product with
// the low word of the first multiplier is a per-function constant
// kh = sub_hi_term(sub). Bit-identical to hash_u32 (tests/test_hash_halves.py
// compares the two on the host); three instructions fewer per hash.
__host__ __device__ __forceinline__ uint32_t sub_hi_term(uint64_t sub) {
    const uint32_t hi = static_cast<uint32_t>(sub >> 32);
    return (hi ^ (hi >> 30)) * 0x1CE4E5B9u;
}
__host__ __device__ __forceinline__ uint32_t funnel_r(uint32_t lo, uint32_t hi, uint32_t s) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(lo, hi, s);
#else
    return static_cast<uint32_t>(((static_cast<uint64_t>(hi) << 32) | lo) >> s);
#endif
}
__host__ __device__ __forceinline__ uint32_t hash_u32k(uint64_t sub, uint32_t kh, uint32_t key) {
    const uint32_t xlo = static_cast<uint32_t>(sub) ^ key;
    const uint32_t ylo = xlo ^ funnel_r(xlo, static_cast<uint32_t>(sub >> 32), 30);
    // * 0xBF58476D1CE4E5B9 (mod 2^64)
    const uint64_t z = static_cast<uint64_t>(ylo) * 0x1CE4E5B9u + (static_cast<uint64_t>(ylo * 0xBF58476Du + kh) << 32);
    const uint32_t zlo = static_cast<uint32_t>(z), zhi = static_cast<uint32_t>(z >> 32);
    const uint32_t tlo = zlo ^ funnel_r(zlo, zhi, 27), thi = zhi ^ (zhi >> 27);
    // * 0x94D049BB133111EB (mod 2^64)
    const uint64_t u = static_cast<uint64_t>(tlo) * 0x133111EBu +
                       (static_cast<uint64_t>(tlo * 0x94D049BBu + thi * 0x133111EBu) << 32);
    const uint32_t ulo = static_cast<uint32_t>(u);
    return ulo ^ funnel_r(ulo, static_cast<uint32_t>(u >> 32), 31);
}
// HashFamily::reduce = (u64(h) * range) >> 32 (hash.hpp:60-62)
__device__ __forceinline__ uint32_t reduce32(uint32_t h, uint32_t range) { return __umulhi(h, range); }

__device__ __forceinline__ uint32_t column_of(const DevCfg& c, uint32_t row, uint32_t aip) {
    return reduce32(hash_u32k(c.sub_row[row], c.kh_row[row], aip), c.cols);
}
__device__ __forceinline__ uint32_t indicator_bit_index(const DevCfg& c, uint32_t aip) {
    return reduce32(hash_u32(c.sub_ind, aip), kIndicatorBits);
}

// Warp-aggregated append: every lane of the (full) warp calls this with its
// own count; returns the lane's first slot. One atomic per warp.
__device__ __forceinline__ uint32_t warp_append(uint32_t* counter, uint32_t cnt) {
    const unsigned full = 0xFFFFFFFFu;
    const uint32_t lane = threadIdx.x & 31u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(full, incl, o);
        if (lane >= static_cast<uint32_t>(o)) incl += t;
    }
    const uint32_t total = __shfl_sync(full, incl, 31);
    uint32_t base = 0;
    if (lane == 31 && total) base = atomicAdd(counter, total);
    base = __shfl_sync(full, base, 31);
    return base + incl - cnt;
}

// 16-bit OR on a 32-bit atomic (the indicator words are u16, sea.hpp:356).
__device__ __forceinline__ void atomic_or_u16(uint16_t* p, uint16_t bit) {
    const uintptr_t a = reinterpret_cast<uintptr_t>(p);
    unsigned int* w = reinterpret_cast<unsigned int*>(a & ~uintptr_t(3));
    atomicOr(w, static_cast<unsigned int>(bit) << ((a & 2u) * 8u));
}

}  // namespace srla
