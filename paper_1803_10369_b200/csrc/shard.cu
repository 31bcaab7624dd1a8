// shard.cu — owner partition of a record batch for multi-GPU runs.
//
// Each GPU owns the hosts with reduce(3, aip, n) == rank and keeps a full,
// independent sketch for them. A host's records all land on
// one GPU, so its per-host results equal those of a CPU reference pipeline
// fed the owner-filtered sub-trace in original order. Stable selection keeps
// that order.
#include <cub/cub.cuh>

#include <string>

#include "common.cuh"
#include "srla.h"

namespace srla {

struct Rec12 {
    uint32_t ts, src, dst;
};

struct OwnedBy {
    uint64_t sub;
    uint32_t nparts, part;
    __host__ __device__ bool operator()(const Rec12& r) const {
        return static_cast<uint32_t>((static_cast<uint64_t>(hash_u32(sub, r.src)) * nparts) >> 32) == part;
    }
};

}  // namespace srla

extern "C" {

srla_status srla_internal_set_error(srla_status code, const char* msg);

uint32_t srla_owner_of(uint64_t seed, uint32_t aip, uint32_t nparts) {
    const uint64_t sub = srla::sub_key(seed, 3);
    return static_cast<uint32_t>((static_cast<uint64_t>(srla::hash_u32(sub, aip)) * nparts) >> 32);
}

srla_status srla_partition_records(const srla_record* d_in, uint64_t n, uint64_t seed, uint32_t nparts,
                                   uint32_t part, srla_record* d_out, uint64_t* n_out, void* stream) {
    if (!n_out || (n && (!d_in || !d_out)) || nparts == 0 || part >= nparts)
        return srla_internal_set_error(SRLA_E_INVALID, "bad partition arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const srla::OwnedBy pred{srla::sub_key(seed, 3), nparts, part};
    const auto* in = reinterpret_cast<const srla::Rec12*>(d_in);
    auto* out = reinterpret_cast<srla::Rec12*>(d_out);
    uint64_t total = 0;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    int* d_cnt = nullptr;
    cudaError_t err = cudaMallocAsync(reinterpret_cast<void**>(&d_cnt), sizeof(int), st);
    const uint64_t piece = 1ull << 30;
    for (uint64_t o = 0; o < n && err == cudaSuccess; o += piece) {
        const int m = static_cast<int>(std::min<uint64_t>(piece, n - o));
        size_t need = 0;
        err = cub::DeviceSelect::If(nullptr, need, in + o, out + total, d_cnt, m, pred, st);
        if (err != cudaSuccess) break;
        if (need > temp_bytes) {
            if (temp) cudaFreeAsync(temp, st);
            err = cudaMallocAsync(&temp, need, st);
            temp_bytes = need;
            if (err != cudaSuccess) break;
        }
        err = cub::DeviceSelect::If(temp, temp_bytes, in + o, out + total, d_cnt, m, pred, st);
        int h = 0;
        if (err == cudaSuccess) err = cudaMemcpyAsync(&h, d_cnt, sizeof(int), cudaMemcpyDeviceToHost, st);
        if (err == cudaSuccess) err = cudaStreamSynchronize(st);
        total += static_cast<uint64_t>(h);
    }
    if (temp) cudaFreeAsync(temp, st);
    if (d_cnt) cudaFreeAsync(d_cnt, st);
    cudaStreamSynchronize(st);
    if (err != cudaSuccess) return srla_internal_set_error(SRLA_E_CUDA, cudaGetErrorString(err));
    *n_out = total;
    return srla_internal_set_error(SRLA_OK, "");
}

}  // extern "C"
