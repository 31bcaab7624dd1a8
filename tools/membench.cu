// membench.cu — B200 memory microbenchmarks behind the scan roofline. One JSON line.
//   copy_gbs           streaming read+write
//   <op>_<region>      random scattered ops, 4e8 per launch, address = hash & (region-1)
// ops: st8 (byte store = the scan's linear mark), st32, red_and32 (atomicAnd, no return),
//      ld32 (gather), st8_dup4 (4 lanes of a quad hit one sector)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o membench membench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}

template <int OP>
__global__ void k_rand(uint8_t* __restrict__ buf, uint64_t mask, uint64_t ops, uint64_t seed, uint32_t* sink) {
    const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint32_t acc = 0;
    for (uint64_t i = tid; i < ops; i += stride) {
        uint64_t h = mix(seed + i);
        if (OP == 4) h = mix(seed + (i >> 2)) + (i & 3) * 8;  // quads share a sector
        uint64_t a = h & mask;
        if (OP == 0 || OP == 4) buf[a] = 0;
        else if (OP == 1) reinterpret_cast<uint32_t*>(buf)[a >> 2] = 0;
        else if (OP == 2) atomicAnd(reinterpret_cast<uint32_t*>(buf) + (a >> 2), 0xFFFF00FFu);
        else if (OP == 3) acc += __ldcg(reinterpret_cast<const uint32_t*>(buf) + (a >> 2));
    }
    if (OP == 3 && acc == 0x12345678u) sink[0] = acc;
}

int main() {
    const uint64_t total = 4ull << 30;
    uint8_t *a, *b;
    uint32_t* sink;
    cudaMalloc(&a, total);
    cudaMalloc(&b, total);
    cudaMalloc(&sink, 4);
    cudaMemset(a, 1, total);
    cudaMemset(b, 1, total);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto fn, int reps) {
        fn();
        cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < reps; ++r) {
            cudaEventRecord(e0);
            fn();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        return best;
    };
    const int grid = 148 * 16;
    float ms_copy = timeit([&] { k_copy<<<grid, 256>>>((const uint4*)a, (uint4*)b, total / 16); }, 5);
    printf("{\"copy_gbs\": %.1f", 2.0 * total / (ms_copy * 1e-3) / 1e9);
    const uint64_t ops = 400000000ull;
    const char* names[] = {"st8", "st32", "red_and32", "ld32", "st8_quad"};
    const uint64_t regions[] = {total, 64ull << 20};
    for (uint64_t region : regions) {
        for (int op = 0; op < 5; ++op) {
            float ms = 0;
            switch (op) {
                case 0: ms = timeit([&] { k_rand<0><<<grid, 256>>>(a, region - 1, ops, 7, sink); }, 3); break;
                case 1: ms = timeit([&] { k_rand<1><<<grid, 256>>>(a, region - 1, ops, 7, sink); }, 3); break;
                case 2: ms = timeit([&] { k_rand<2><<<grid, 256>>>(a, region - 1, ops, 7, sink); }, 3); break;
                case 3: ms = timeit([&] { k_rand<3><<<grid, 256>>>(a, region - 1, ops, 7, sink); }, 3); break;
                case 4: ms = timeit([&] { k_rand<4><<<grid, 256>>>(a, region - 1, ops, 7, sink); }, 3); break;
            }
            printf(", \"%s_%lluMB_Gops\": %.2f", names[op], (unsigned long long)(region >> 20), ops / (ms * 1e-3) / 1e9);
        }
    }
    printf("}\n");
    return 0;
}
