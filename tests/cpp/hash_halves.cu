// Host-side check that hash_u32k (csrc/common.cuh, the device kernels' hash)
// equals hash_u32 = HashFamily::u32 (hash.hpp:53-56) for every sub-key of
// the given seeds and random keys. Built and run by tests/test_hash_halves.py.
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

int main(int argc, char** argv) {
    const unsigned long long n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1000000ull;
    uint64_t state = 0x5EA00001ull;
    auto next = [&] { return srla::avalanche64(state += srla::kGolden); };
    unsigned long long bad = 0;
    for (unsigned long long i = 0; i < n; ++i) {
        const uint64_t seed = (i & 1023) == 0 ? 0x5EA00001ull : next();
        const uint32_t index = static_cast<uint32_t>(i % 72);
        const uint64_t sub = srla::sub_key(seed, index);
        const uint32_t key = (i & 3) == 0 ? static_cast<uint32_t>(i) : static_cast<uint32_t>(next());
        if (srla::hash_u32k(sub, srla::sub_hi_term(sub), key) != srla::hash_u32(sub, key)) ++bad;
    }
    std::printf("%llu of %llu differ\n", bad, n);
    return bad ? 1 : 0;
}
