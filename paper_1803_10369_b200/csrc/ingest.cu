// ingest.cu — the trace front end on the device:
// the SRLT v1 reader, orientation against the monitored prefix and slice
// partitioning (trace.hpp:109-281), so a raw trace goes host -> HBM once and
// is parsed, oriented and cut into slices where the scan reads it.
//
//  * srla_parse_srlt: file bytes -> records. Records sit at byte 5 + 12 i, so
//    every record starts at 1 mod 4: four aligned words and three funnel
//    shifts give its three fields; the timestamp order check is a min-index
//    reduction (for_each_record, trace.hpp:109-170).
//  * srla_orient_records: orient_record (trace.hpp:223-238) as a stable
//    compaction of the kept/flipped records, with the four outcome counters.
//  * srla_slice_bounds: SlicePartitioner (trace.hpp:243-281) over an ordered
//    batch — slice s starts at the first record with ts >= origin + s*seconds
//    (a binary search per slice; empty slices included).
#include <cub/cub.cuh>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstring>
#include <string>

#include "common.cuh"
#include "srla.h"

namespace srla {

struct IngestRec {
    uint32_t ts, src, dst;
};

// orient_record: 0 kept, 1 flipped, 2 dropped (both sides), 3 dropped (neither)
struct OrientClass {
    uint32_t addr, mask;
    __host__ __device__ uint32_t operator()(const IngestRec& r) const {
        const bool s = (r.src & mask) == addr, d = (r.dst & mask) == addr;
        return s && !d ? 0u : !s && d ? 1u : s ? 2u : 3u;
    }
};
struct Oriented {
    OrientClass cls;
    __host__ __device__ IngestRec operator()(const IngestRec& r) const {
        return cls(r) == 1u ? IngestRec{r.ts, r.dst, r.src} : r;
    }
};
struct Kept {
    OrientClass cls;
    __host__ __device__ bool operator()(const IngestRec& r) const { return cls(r) < 2u; }
};

__global__ void __launch_bounds__(256) k_orient_stats(const IngestRec* __restrict__ in, uint64_t n, OrientClass cls,
                                                      unsigned long long* __restrict__ stats) {
    unsigned long long c[4] = {0, 0, 0, 0};
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        ++c[cls(in[i])];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        unsigned long long v = c[k];
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(stats + k, v);
    }
}

// SRLT body: record i occupies bytes [5 + 12 i, 17 + 12 i) of the file
__global__ void __launch_bounds__(256) k_parse_srlt(const uint8_t* __restrict__ bytes, uint64_t nbytes, uint64_t nrec,
                                                    IngestRec* __restrict__ out,
                                                    unsigned long long* __restrict__ first_bad) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(bytes);  // cudaMalloc'd: 4-byte aligned
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < nrec;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint64_t start = 5 + 12 * i;  // = 1 (mod 4)
        const uint64_t q = start >> 2;
        uint32_t v[3];
        if (4 * (q + 4) <= nbytes) {
            const uint32_t a = w[q], b = w[q + 1], c = w[q + 2], d = w[q + 3];
            v[0] = __funnelshift_r(a, b, 8);
            v[1] = __funnelshift_r(b, c, 8);
            v[2] = __funnelshift_r(c, d, 8);
        } else {  // the last record: no aligned word past the end of the buffer
            for (int k = 0; k < 3; ++k) {
                const uint8_t* p = bytes + start + 4 * k;
                v[k] = static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 |
                       static_cast<uint32_t>(p[2]) << 16 | static_cast<uint32_t>(p[3]) << 24;
            }
        }
        out[i] = IngestRec{v[0], v[1], v[2]};
    }
    // check_order (trace.hpp:113-119): the first record older than its predecessor
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < nrec;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        auto ts_at = [&](uint64_t r) {
            const uint8_t* p = bytes + 5 + 12 * r;
            return static_cast<uint32_t>(p[0]) | static_cast<uint32_t>(p[1]) << 8 | static_cast<uint32_t>(p[2]) << 16 |
                   static_cast<uint32_t>(p[3]) << 24;
        };
        if (ts_at(i) < ts_at(i - 1)) atomicMin(first_bad, static_cast<unsigned long long>(i));
    }
}

// slice s starts at the first record with ts >= origin + s * seconds
__global__ void __launch_bounds__(256) k_slice_bounds(const IngestRec* __restrict__ recs, uint64_t n, uint64_t origin,
                                                      uint32_t seconds, uint64_t nslices,
                                                      unsigned long long* __restrict__ offsets,
                                                      unsigned long long* __restrict__ first_bad) {
    for (uint64_t s = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; s <= nslices;
         s += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        if (s == 0 || s == nslices) {
            offsets[s] = s == 0 ? 0ull : n;
            continue;
        }
        const uint64_t t = origin + s * static_cast<uint64_t>(seconds);
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) / 2;
            if (recs[mid].ts < t) lo = mid + 1;
            else hi = mid;
        }
        offsets[s] = lo;
    }
    for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x + 1; i < n;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
        if (recs[i].ts < recs[i - 1].ts) atomicMin(first_bad, static_cast<unsigned long long>(i));
}

uint32_t grid_for(uint64_t work) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint64_t b = (work + 255) / 256;
    return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>(b, uint64_t(sms) * 8)));
}

}  // namespace srla

extern "C" {

srla_status srla_internal_set_error(srla_status code, const char* msg);

#define ING_CK(x)                                                                         \
    do {                                                                                  \
        cudaError_t e_ = (x);                                                             \
        if (e_ != cudaSuccess) return srla_internal_set_error(SRLA_E_CUDA, cudaGetErrorString(e_)); \
    } while (0)

srla_status srla_device_alloc(int device, uint64_t bytes, void** out) {
    if (!out) return srla_internal_set_error(SRLA_E_INVALID, "null output");
    *out = nullptr;
    ING_CK(cudaSetDevice(device));
    ING_CK(cudaMalloc(out, bytes ? bytes : 1));
    return SRLA_OK;
}

srla_status srla_device_free(int device, void* p) {
    ING_CK(cudaSetDevice(device));
    if (p) ING_CK(cudaFree(p));
    return SRLA_OK;
}

srla_status srla_copy_to_device(int device, void* dst, const void* src, uint64_t bytes) {
    if (bytes && (!dst || !src)) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    ING_CK(cudaSetDevice(device));
    if (bytes) ING_CK(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
    return SRLA_OK;
}

srla_status srla_copy_to_host(int device, void* dst, const void* src, uint64_t bytes) {
    if (bytes && (!dst || !src)) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    ING_CK(cudaSetDevice(device));
    if (bytes) ING_CK(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return SRLA_OK;
}

srla_status srla_parse_srlt(const void* d_bytes, uint64_t nbytes, srla_record* d_out, uint64_t* n_out, void* stream) {
    if (!n_out || (nbytes && !d_bytes)) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    *n_out = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned char head[5] = {};
    if (nbytes >= 5) {
        ING_CK(cudaMemcpyAsync(head, d_bytes, 5, cudaMemcpyDeviceToHost, st));
        ING_CK(cudaStreamSynchronize(st));
    }
    if (nbytes < 4 || std::memcmp(head, "SRLT", 4) != 0)
        return srla_internal_set_error(SRLA_E_INPUT, "not a binary trace (bad magic)");
    if (nbytes < 5 || head[4] != 1) return srla_internal_set_error(SRLA_E_INPUT, "unsupported trace version");
    const uint64_t nrec = (nbytes - 5) / 12;
    if (nrec && !d_out) return srla_internal_set_error(SRLA_E_INVALID, "null output");
    unsigned long long* d_bad = nullptr;
    ING_CK(cudaMallocAsync(reinterpret_cast<void**>(&d_bad), sizeof(unsigned long long), st));
    ING_CK(cudaMemsetAsync(d_bad, 0xFF, sizeof(unsigned long long), st));
    if (nrec)
        srla::k_parse_srlt<<<srla::grid_for(nrec), 256, 0, st>>>(static_cast<const uint8_t*>(d_bytes), nbytes, nrec,
                                                                reinterpret_cast<srla::IngestRec*>(d_out), d_bad);
    ING_CK(cudaGetLastError());
    unsigned long long bad = 0;
    ING_CK(cudaMemcpyAsync(&bad, d_bad, sizeof(bad), cudaMemcpyDeviceToHost, st));
    ING_CK(cudaFreeAsync(d_bad, st));
    ING_CK(cudaStreamSynchronize(st));
    if (bad != ~0ull) {  // records before the regression are delivered, as for_each_record does
        *n_out = bad;
        return srla_internal_set_error(SRLA_E_INPUT, ("timestamp regression at record " + std::to_string(bad)).c_str());
    }
    *n_out = nrec;
    if ((nbytes - 5) % 12)
        return srla_internal_set_error(SRLA_E_INPUT, ("truncated record " + std::to_string(nrec)).c_str());
    return SRLA_OK;
}

srla_status srla_orient_records(const srla_record* d_in, uint64_t n, uint32_t prefix_addr, uint32_t prefix_bits,
                                srla_record* d_out, uint64_t* n_out, srla_orient_stats* stats, void* stream) {
    if (!n_out || (n && (!d_in || !d_out)) || prefix_bits > 32)
        return srla_internal_set_error(SRLA_E_INVALID, "bad orientation arguments");
    *n_out = 0;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t mask = prefix_bits == 0 ? 0u : 0xFFFFFFFFu << (32 - prefix_bits);
    const srla::OrientClass cls{prefix_addr & mask, mask};
    const auto* in = reinterpret_cast<const srla::IngestRec*>(d_in);
    auto* out = reinterpret_cast<srla::IngestRec*>(d_out);
    unsigned long long* d_aux = nullptr;  // stats[4] | selected count
    ING_CK(cudaMallocAsync(reinterpret_cast<void**>(&d_aux), 5 * sizeof(unsigned long long), st));
    ING_CK(cudaMemsetAsync(d_aux, 0, 5 * sizeof(unsigned long long), st));
    if (n) srla::k_orient_stats<<<srla::grid_for(n), 256, 0, st>>>(in, n, cls, d_aux);
    ING_CK(cudaGetLastError());
    // stable compaction of the kept/flipped records, flipped on the fly
    uint64_t total = 0;
    void* temp = nullptr;
    size_t temp_bytes = 0;
    const uint64_t piece = 1ull << 30;
    for (uint64_t o = 0; o < n; o += piece) {
        const int m = static_cast<int>(std::min<uint64_t>(piece, n - o));
        auto src = thrust::make_transform_iterator(in + o, srla::Oriented{cls});
        size_t need = 0;
        ING_CK(cub::DeviceSelect::If(nullptr, need, src, out + total, d_aux + 4, m, srla::Kept{cls}, st));
        if (need > temp_bytes) {
            if (temp) ING_CK(cudaFreeAsync(temp, st));
            ING_CK(cudaMallocAsync(&temp, need, st));
            temp_bytes = need;
        }
        // select counts per piece: the flag test reads the transformed record,
        // whose class is kept/flipped iff the original's is
        ING_CK(cub::DeviceSelect::If(temp, temp_bytes, src, out + total, d_aux + 4, m, srla::Kept{cls}, st));
        unsigned long long sel = 0;
        ING_CK(cudaMemcpyAsync(&sel, d_aux + 4, sizeof(sel), cudaMemcpyDeviceToHost, st));
        ING_CK(cudaStreamSynchronize(st));
        total += sel;
    }
    unsigned long long h[4] = {};
    ING_CK(cudaMemcpyAsync(h, d_aux, sizeof(h), cudaMemcpyDeviceToHost, st));
    if (temp) ING_CK(cudaFreeAsync(temp, st));
    ING_CK(cudaFreeAsync(d_aux, st));
    ING_CK(cudaStreamSynchronize(st));
    *n_out = total;
    if (stats) {
        stats->kept = h[0];
        stats->flipped = h[1];
        stats->dropped_both = h[2];
        stats->dropped_neither = h[3];
    }
    return SRLA_OK;
}

srla_status srla_slice_bounds(const srla_record* d_recs, uint64_t n, uint32_t slice_seconds, uint64_t* offsets,
                              uint64_t cap, uint64_t* n_slices, void* stream) {
    if (!n_slices || (n && !d_recs)) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    if (slice_seconds < 1) return srla_internal_set_error(SRLA_E_INVALID, "slice duration must be >= 1 second");
    *n_slices = 0;
    if (!n) return SRLA_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    uint32_t first = 0, last = 0;
    ING_CK(cudaMemcpyAsync(&first, &d_recs[0].ts, 4, cudaMemcpyDeviceToHost, st));
    ING_CK(cudaMemcpyAsync(&last, &d_recs[n - 1].ts, 4, cudaMemcpyDeviceToHost, st));
    ING_CK(cudaStreamSynchronize(st));
    const uint64_t ns = last >= first ? (static_cast<uint64_t>(last) - first) / slice_seconds + 1 : 1;
    *n_slices = ns;
    if (!offsets) return SRLA_OK;  // size query
    if (cap < ns + 1) return srla_internal_set_error(SRLA_E_CAPACITY, "offsets buffer too small (need n_slices + 1)");
    unsigned long long* d = nullptr;  // offsets[ns + 1] | first_bad
    ING_CK(cudaMallocAsync(reinterpret_cast<void**>(&d), (ns + 2) * sizeof(unsigned long long), st));
    ING_CK(cudaMemsetAsync(d + ns + 1, 0xFF, sizeof(unsigned long long), st));
    srla::k_slice_bounds<<<srla::grid_for(std::max<uint64_t>(ns + 1, n)), 256, 0, st>>>(
        reinterpret_cast<const srla::IngestRec*>(d_recs), n, first, slice_seconds, ns, d, d + ns + 1);
    ING_CK(cudaGetLastError());
    ING_CK(cudaMemcpyAsync(offsets, d, (ns + 2) * sizeof(unsigned long long) - sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, st));
    unsigned long long bad = 0;
    ING_CK(cudaMemcpyAsync(&bad, d + ns + 1, sizeof(bad), cudaMemcpyDeviceToHost, st));
    ING_CK(cudaFreeAsync(d, st));
    ING_CK(cudaStreamSynchronize(st));
    if (bad != ~0ull)
        return srla_internal_set_error(SRLA_E_INPUT, ("timestamp regression at record " + std::to_string(bad)).c_str());
    return SRLA_OK;
}

}  // extern "C"
