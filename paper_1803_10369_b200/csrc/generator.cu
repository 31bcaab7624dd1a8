// generator.cu — device port of the reference's synthetic trace generator
// (generate_trace, generator.hpp:117-161), byte-identical for slice_seconds = 1.
//
// SplitMix64 is counter based (state += phi per draw, hash.hpp:21-24) and the
// number of draws per record is fixed (plant record: 1 = its timestamp;
// background record: 3 = src, dst, timestamp; generator.hpp:129-150), so draw
// m of the trace is avalanche64(seed + m*phi) and every record is independent.
// With one-second slices every timestamp draw is next_below(1) = 0 and the
// per-slice stable sort by ts is the identity, so records come out in
// generation order. The Zipf inverse CDF is built on the host in the
// reference's own double arithmetic (generator.hpp:74-82) and searched on the
// device with the same lower_bound.
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "srla.h"

namespace srla {

struct PlantRun {
    uint32_t host, lo, offset, start;  // output index of its first record in the slice
};

__global__ void __launch_bounds__(256) k_gen_plants(const PlantRun* __restrict__ runs, uint32_t nruns,
                                                    uint32_t nrec, uint32_t ts, uint32_t b_base,
                                                    uint32_t b_hosts, uint32_t* __restrict__ out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < nrec; r += gridDim.x * blockDim.x) {
        uint32_t lo = 0, hi = nruns;  // last run with start <= r
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (runs[mid].start <= r) lo = mid;
            else hi = mid;
        }
        const PlantRun p = runs[lo];
        const uint32_t j = p.lo + (r - p.start);
        out[3ull * r] = ts;
        out[3ull * r + 1] = p.host;
        out[3ull * r + 2] = b_base + static_cast<uint32_t>((static_cast<uint64_t>(p.offset) + j) % b_hosts);
    }
}

__global__ void __launch_bounds__(256) k_gen_background(uint64_t seed, uint64_t draw0, uint32_t pairs,
                                                        uint32_t ts, uint32_t a_base, uint32_t a_hosts,
                                                        uint32_t b_base, uint32_t b_hosts,
                                                        const double* __restrict__ cdf,
                                                        uint32_t* __restrict__ out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += gridDim.x * blockDim.x) {
        const uint64_t m = draw0 + 3ull * i;  // draws already taken before this record
        const uint64_t xs = avalanche64(seed + kGolden * (m + 1));
        const uint64_t xd = avalanche64(seed + kGolden * (m + 2));
        const uint32_t src = a_base + static_cast<uint32_t>(__umul64hi(xs, a_hosts));
        uint32_t rank;
        if (!cdf) {
            rank = static_cast<uint32_t>(__umul64hi(xd, b_hosts));
        } else {
            const double u = static_cast<double>(xd >> 11) * 0x1.0p-53;
            uint32_t lo = 0, hi = b_hosts;
            while (lo < hi) {
                const uint32_t mid = lo + (hi - lo) / 2;
                if (cdf[mid] < u) lo = mid + 1;
                else hi = mid;
            }
            rank = lo == b_hosts ? b_hosts - 1 : lo;
        }
        uint32_t* o = out + 3ull * i;
        o[0] = ts;
        o[1] = src;
        o[2] = b_base + rank;
    }
}

struct Generator {
    srla_trace_spec spec{};
    std::vector<srla_plant> plants;
    int device = 0;
    double* d_cdf = nullptr;
    PlantRun* d_runs = nullptr;
    size_t runs_cap = 0;
    std::vector<uint64_t> draws_before;  // prefix over slices, grown lazily

    Generator(const srla_trace_spec& s, int dev) : spec(s), device(dev) {
        plants.assign(s.plants, s.plants + s.n_plants);
        spec.plants = nullptr;
        validate();
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
        if (spec.skew > 0.0) {  // ZipfSampler (generator.hpp:74-82), host doubles
            std::vector<double> cdf(spec.b_hosts);
            double acc = 0;
            for (uint32_t r = 0; r < spec.b_hosts; ++r) {
                acc += 1.0 / std::pow(static_cast<double>(r + 1), spec.skew);
                cdf[r] = acc;
            }
            for (double& c : cdf) c /= acc;
            if (cudaMalloc(&d_cdf, cdf.size() * sizeof(double)) != cudaSuccess ||
                cudaMemcpy(d_cdf, cdf.data(), cdf.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
                throw std::runtime_error("zipf table upload failed");
        }
        draws_before.push_back(0);
    }
    ~Generator() {
        if (d_cdf) cudaFree(d_cdf);
        if (d_runs) cudaFree(d_runs);
    }

    // PlantSpec::validate (generator.hpp:45-63) plus the one-second-slice limit.
    void validate() const {
        auto bad = [](const std::string& m) { throw std::invalid_argument(m); };
        if (spec.slices < 1) bad("trace needs at least one slice");
        if (spec.window < 1) bad("window must be >= 1");
        if (spec.slice_seconds < 1) bad("slice duration must be >= 1");
        if (spec.slice_seconds != 1) bad("device generator supports slice_seconds == 1 only");
        if (spec.b_hosts < 1) bad("destination pool is empty");
        if (spec.a_hosts < 1 && spec.pairs_per_slice > 0) bad("source pool is empty");
        for (const auto& p : plants) {
            if (p.cardinality < 1) bad("planted cardinality must be >= 1");
            if (p.cardinality > spec.b_hosts) bad("planted cardinality exceeds the destination pool");
            if (p.host >= spec.a_base && p.host < spec.a_base + spec.a_hosts)
                bad("planted host collides with the background source pool");
            if (p.first_slice > p.last_slice) bad("empty active span");
        }
    }

    // rotation chunks of the active plants in slice s (generator.hpp:98-109,126-145)
    uint64_t plant_runs(uint64_t s, std::vector<PlantRun>* runs) const {
        uint64_t n = 0;
        for (size_t pi = 0; pi < plants.size(); ++pi) {
            const auto& p = plants[pi];
            if (!(s >= p.first_slice && s <= p.last_slice)) continue;
            const uint32_t r = static_cast<uint32_t>((s - p.first_slice) % spec.window);
            const uint64_t lo = static_cast<uint64_t>(p.cardinality) * r / spec.window;
            const uint64_t hi = static_cast<uint64_t>(p.cardinality) * (r + 1) / spec.window;
            if (hi == lo) continue;
            if (runs)
                runs->push_back({p.host, static_cast<uint32_t>(lo),
                                 static_cast<uint32_t>((pi * 2654435761ull) % spec.b_hosts),
                                 static_cast<uint32_t>(n)});
            n += hi - lo;
        }
        return n;
    }

    uint64_t draws_until(uint64_t s) {
        while (draws_before.size() <= s) {
            const uint64_t t = draws_before.size() - 1;
            draws_before.push_back(draws_before.back() + plant_runs(t, nullptr) + 3ull * spec.pairs_per_slice);
        }
        return draws_before[s];
    }

    uint64_t count(uint64_t s) const { return plant_runs(s, nullptr) + spec.pairs_per_slice; }

    void generate(uint64_t s, uint32_t* out, cudaStream_t st) {
        if (s >= spec.slices) throw std::invalid_argument("slice index beyond the trace");
        std::vector<PlantRun> runs;
        const uint64_t np = plant_runs(s, &runs);
        const uint32_t ts = spec.start_ts + static_cast<uint32_t>(s) * spec.slice_seconds;
        if (np) {
            if (runs.size() > runs_cap) {
                if (d_runs) cudaFree(d_runs);
                runs_cap = runs.size() * 2;
                if (cudaMalloc(&d_runs, runs_cap * sizeof(PlantRun)) != cudaSuccess)
                    throw std::runtime_error("plant table allocation failed");
            }
            cudaMemcpyAsync(d_runs, runs.data(), runs.size() * sizeof(PlantRun), cudaMemcpyHostToDevice, st);
            const uint32_t b = static_cast<uint32_t>(std::min<uint64_t>((np + 255) / 256, 148 * 16));
            k_gen_plants<<<b, 256, 0, st>>>(d_runs, static_cast<uint32_t>(runs.size()), static_cast<uint32_t>(np), ts,
                                           spec.b_base, spec.b_hosts, out);
            cudaStreamSynchronize(st);  // runs buffer reused by the next call
        }
        if (spec.pairs_per_slice) {
            const uint64_t draw0 = draws_until(s) + np;
            const uint32_t b = static_cast<uint32_t>(std::min<uint64_t>((spec.pairs_per_slice + 255) / 256, 148 * 32));
            k_gen_background<<<b, 256, 0, st>>>(spec.seed, draw0, spec.pairs_per_slice, ts, spec.a_base,
                                               spec.a_hosts, spec.b_base, spec.b_hosts,
                                               spec.skew > 0.0 ? d_cdf : nullptr, out + 3ull * np);
        }
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) throw std::runtime_error(std::string("generator launch: ") + cudaGetErrorString(e));
    }
};

}  // namespace srla

struct srla_generator {
    srla::Generator* impl;
};

extern "C" {

// defined in engine.cu
srla_status srla_internal_set_error(srla_status code, const char* msg);

srla_status srla_generator_create(const srla_trace_spec* spec, int device, srla_generator** out) {
    if (!spec || !out) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    try {
        auto* g = new srla_generator{new srla::Generator(*spec, device)};
        *out = g;
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::invalid_argument& e) {
        return srla_internal_set_error(SRLA_E_INVALID, e.what());
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

srla_status srla_generator_destroy(srla_generator* g) {
    if (g) {
        delete g->impl;
        delete g;
    }
    return SRLA_OK;
}

srla_status srla_generate_slice(srla_generator* g, uint64_t slice, srla_record* out_device, uint64_t cap,
                                uint64_t* n_out, void* stream) {
    if (!g || !n_out) return srla_internal_set_error(SRLA_E_INVALID, "null argument");
    try {
        const uint64_t n = g->impl->count(slice);
        *n_out = n;
        if (!out_device) return srla_internal_set_error(SRLA_OK, "");
        if (cap < n) return srla_internal_set_error(SRLA_E_CAPACITY, "output buffer too small");
        cudaSetDevice(g->impl->device);
        g->impl->generate(slice, reinterpret_cast<uint32_t*>(out_device), static_cast<cudaStream_t>(stream));
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::invalid_argument& e) {
        return srla_internal_set_error(SRLA_E_INVALID, e.what());
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

}  // extern "C"
