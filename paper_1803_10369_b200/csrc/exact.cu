// exact.cu — exact sliding-window cardinalities on the device (the reference's
// ground-truth "precise method", oracle.hpp:45-203).
//
// The reference keeps one hash map entry per live (host, opposite host) pair
// (PairRecorderStore) or a ring of per-slice hash sets (SliceRingStore) on the
// host. Here a slice is a sorted, deduplicated array of 64-bit pair keys
// (aip << 32 | bip) in HBM, and the last max_window slices form a ring. A
// window query concatenates its k slices, radix-sorts and deduplicates the
// keys, and run-length encodes the hosts: every host with a nonzero distinct
// count, ascending by address. Memory is 8 bytes per distinct pair per slice
// (1e8-pair slices: 0.8 GB each), so ground truth for BASELINE.json's C2 trace
// fits a B200 where the reference's maps would not fit the host.
#include <cub/cub.cuh>

#include <algorithm>
#include <deque>
#include <stdexcept>
#include <string>
#include <vector>

#include "srla.h"

extern "C" srla_status srla_internal_set_error(srla_status code, const char* msg);

namespace srla {

namespace {

#define XK(x)                                                                                             \
    do {                                                                                                  \
        cudaError_t e_ = (x);                                                                             \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

struct RangeError : std::out_of_range {
    using std::out_of_range::out_of_range;
};

__global__ void k_pair_keys(const uint32_t* __restrict__ recs, uint64_t n, unsigned long long* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        keys[i] = (static_cast<unsigned long long>(recs[3 * i + 1]) << 32) | recs[3 * i + 2];
}

__global__ void k_key_hosts(const unsigned long long* __restrict__ keys, uint64_t n, uint32_t* __restrict__ hosts) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        hosts[i] = static_cast<uint32_t>(keys[i] >> 32);
}

uint32_t grid_for(uint64_t n) { return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16))); }

struct DevArr {
    void* p = nullptr;
    uint64_t bytes = 0;
    DevArr() = default;
    DevArr(const DevArr&) = delete;
    DevArr(DevArr&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }  // deque growth
    ~DevArr() {
        if (p) cudaFree(p);
    }
    void ensure(uint64_t b) {
        if (b <= bytes) return;
        if (p) XK(cudaFree(p));
        p = nullptr;
        const uint64_t c = std::max<uint64_t>(b + b / 4, 4096);
        XK(cudaMalloc(&p, c));
        bytes = c;
    }
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

}  // namespace

struct Slice {
    DevArr keys;  // sorted unique pair keys
    uint64_t n = 0;
};

struct Exact {
    uint32_t max_window;
    int device;
    cudaStream_t st = nullptr;
    uint64_t current = 0;          // current slice id
    std::deque<Slice> ring;        // back() = the current slice (finalized lazily)
    DevArr staged, tmp, tmp2, temp, hosts, uniq, counts, nrun;
    uint64_t nstaged = 0;          // raw keys observed in the current slice since it was last finalized

    Exact(uint32_t k, int dev) : max_window(k), device(dev) {
        XK(cudaSetDevice(device));
        XK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        ring.emplace_back();
    }
    ~Exact() {
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }

    template <typename Fn>
    void cub_call(Fn&& fn) {
        size_t b = 0;
        XK(fn(static_cast<void*>(nullptr), b));
        temp.ensure(b + 16);
        XK(fn(temp.p, b));
    }

    // sort + dedupe `n` keys at `in` into `out` (out may grow); returns the unique count
    uint64_t sort_unique(const unsigned long long* in, uint64_t n, DevArr& out) {
        if (!n) return 0;
        tmp2.ensure(n * 8);
        out.ensure(n * 8);
        nrun.ensure(8);
        for (uint64_t o = 0; o < n; o += (1ull << 30))
            if (n - o > (1ull << 30)) throw std::runtime_error("exact store: more than 2^30 keys in one query");
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceRadixSort::SortKeys(t, b, in, tmp2.as<unsigned long long>(), static_cast<int>(n), 0, 64, st);
        });
        cub_call([&](void* t, size_t& b) {
            return cub::DeviceSelect::Unique(t, b, tmp2.as<unsigned long long>(), out.as<unsigned long long>(),
                                             nrun.as<unsigned long long>(), static_cast<int>(n), st);
        });
        unsigned long long m = 0;
        XK(cudaMemcpyAsync(&m, nrun.p, 8, cudaMemcpyDeviceToHost, st));
        XK(cudaStreamSynchronize(st));
        return m;
    }

    // merge the staged keys into the current slice's sorted unique set
    void finalize() {
        if (!nstaged) return;
        Slice& s = ring.back();
        const uint64_t total = s.n + nstaged;
        tmp.ensure(total * 8);
        if (s.n) XK(cudaMemcpyAsync(tmp.p, s.keys.p, s.n * 8, cudaMemcpyDeviceToDevice, st));
        XK(cudaMemcpyAsync(tmp.as<unsigned long long>() + s.n, staged.p, nstaged * 8, cudaMemcpyDeviceToDevice, st));
        s.n = sort_unique(tmp.as<unsigned long long>(), total, s.keys);
        nstaged = 0;
    }

    void observe(const srla_record* recs, uint64_t n, int on_device) {
        if (!n) return;
        staged.ensure((nstaged + n) * 8);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(recs);
        if (!on_device) {
            tmp.ensure(n * 12);
            XK(cudaMemcpyAsync(tmp.p, recs, n * 12, cudaMemcpyHostToDevice, st));
            src = tmp.as<uint32_t>();
        } else {
            cudaEvent_t ev;  // device records: after the legacy default stream (srla_scan_batch's contract)
            XK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            XK(cudaEventRecord(ev, cudaStreamLegacy));
            XK(cudaStreamWaitEvent(st, ev, 0));
            XK(cudaEventDestroy(ev));
        }
        k_pair_keys<<<grid_for(n), 256, 0, st>>>(src, n, staged.as<unsigned long long>() + nstaged);
        XK(cudaGetLastError());
        nstaged += n;
        if (!on_device) XK(cudaStreamSynchronize(st));  // the staging buffer is reused
        // bound the staging: fold into the sorted set every 2^28 raw keys
        if (nstaged >= (1ull << 28)) finalize();
    }

    void end_slice() {
        finalize();
        ring.emplace_back();
        if (ring.size() > max_window) ring.pop_front();
        ++current;
    }

    void check_window(uint64_t t, uint32_t k) const {  // oracle.hpp:119-124, 186-191
        if (k < 1 || k > max_window || t + k != current + 1 || k > ring.size())
            throw RangeError("window [" + std::to_string(t) + ", +" + std::to_string(k) + ") is not observable at slice " +
                             std::to_string(current));
    }

    // all hosts with a nonzero count in [t, t+k), ascending; returns the count
    uint64_t cardinalities(uint64_t t, uint32_t k, uint32_t* out_hosts, uint64_t* out_counts, uint64_t cap) {
        check_window(t, k);
        finalize();
        uint64_t total = 0;
        for (size_t i = ring.size() - k; i < ring.size(); ++i) total += ring[i].n;
        if (!total) return 0;
        const unsigned long long* keys = nullptr;
        uint64_t m = 0;
        if (k == 1) {  // one slice: already sorted and unique
            keys = ring.back().keys.as<unsigned long long>();
            m = ring.back().n;
        } else {
            tmp.ensure(total * 8);
            uint64_t at = 0;
            for (size_t i = ring.size() - k; i < ring.size(); ++i) {
                if (ring[i].n)
                    XK(cudaMemcpyAsync(tmp.as<unsigned long long>() + at, ring[i].keys.p, ring[i].n * 8,
                                       cudaMemcpyDeviceToDevice, st));
                at += ring[i].n;
            }
            m = sort_unique(tmp.as<unsigned long long>(), total, uniq);
            keys = uniq.as<unsigned long long>();
        }
        hosts.ensure(m * 4);
        k_key_hosts<<<grid_for(m), 256, 0, st>>>(keys, m, hosts.as<uint32_t>());
        XK(cudaGetLastError());
        counts.ensure(m * 12 + 16);
        uint32_t* run_hosts = reinterpret_cast<uint32_t*>(counts.as<uint8_t>());
        uint32_t* run_len = run_hosts + m;
        unsigned long long* nr = reinterpret_cast<unsigned long long*>(counts.as<uint8_t>() + ((m * 8 + 15) & ~15ull));
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceRunLengthEncode::Encode(tp, b, hosts.as<uint32_t>(), run_hosts, run_len, nr,
                                                      static_cast<int>(m), st);
        });
        unsigned long long nh = 0;
        XK(cudaMemcpyAsync(&nh, nr, 8, cudaMemcpyDeviceToHost, st));
        XK(cudaStreamSynchronize(st));
        if (nh > cap || (!out_hosts && nh)) return nh;  // caller re-queries with room
        std::vector<uint32_t> len(nh);
        XK(cudaMemcpyAsync(out_hosts, run_hosts, nh * 4, cudaMemcpyDeviceToHost, st));
        XK(cudaMemcpyAsync(len.data(), run_len, nh * 4, cudaMemcpyDeviceToHost, st));
        XK(cudaStreamSynchronize(st));
        for (uint64_t i = 0; i < nh; ++i) out_counts[i] = len[i];
        return nh;
    }

    uint64_t pair_count() {  // distinct live pairs over the ring
        finalize();
        uint64_t total = 0;
        for (const auto& s : ring) total += s.n;
        if (!total) return 0;
        tmp.ensure(total * 8);
        uint64_t at = 0;
        for (const auto& s : ring) {
            if (s.n) XK(cudaMemcpyAsync(tmp.as<unsigned long long>() + at, s.keys.p, s.n * 8, cudaMemcpyDeviceToDevice, st));
            at += s.n;
        }
        return sort_unique(tmp.as<unsigned long long>(), total, uniq);
    }
};

}  // namespace srla

struct srla_exact {
    srla::Exact* impl;
};

namespace {
template <typename Fn>
srla_status xguard(Fn&& fn) {
    try {
        fn();
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const srla::RangeError& e) {
        return srla_internal_set_error(SRLA_E_RANGE, e.what());
    } catch (const std::invalid_argument& e) {
        return srla_internal_set_error(SRLA_E_INVALID, e.what());
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}
srla::Exact& X(srla_exact* x) {
    if (!x || !x->impl) throw std::invalid_argument("null exact store");
    XK(cudaSetDevice(x->impl->device));
    return *x->impl;
}
}  // namespace

extern "C" {

srla_status srla_exact_create(uint32_t max_window, int device, srla_exact** out) {
    return xguard([&] {
        if (!out) throw std::invalid_argument("null output");
        if (max_window < 1) throw std::invalid_argument("window must be >= 1");
        *out = new srla_exact{new srla::Exact(max_window, device)};
    });
}

srla_status srla_exact_destroy(srla_exact* x) {
    if (x) {
        delete x->impl;
        delete x;
    }
    return srla_internal_set_error(SRLA_OK, "");
}

srla_status srla_exact_observe(srla_exact* x, const srla_record* recs, uint64_t n, int on_device) {
    return xguard([&] {
        if (n && !recs) throw std::invalid_argument("null records");
        X(x).observe(recs, n, on_device);
    });
}

srla_status srla_exact_end_slice(srla_exact* x) {
    return xguard([&] { X(x).end_slice(); });
}

srla_status srla_exact_current_slice(srla_exact* x, uint64_t* slice) {
    return xguard([&] { *slice = X(x).current; });
}

srla_status srla_exact_pair_count(srla_exact* x, uint64_t* n) {
    return xguard([&] { *n = X(x).pair_count(); });
}

srla_status srla_exact_cardinalities(srla_exact* x, uint64_t window_start, uint32_t window, uint32_t* hosts,
                                     uint64_t* counts, uint64_t cap, uint64_t* n_out) {
    srla_status rc = SRLA_OK;
    const srla_status g = xguard([&] {
        const uint64_t n = X(x).cardinalities(window_start, window, hosts, counts, cap);
        if (n_out) *n_out = n;
        if (n > cap || (!hosts && n)) rc = SRLA_E_CAPACITY;
    });
    if (g != SRLA_OK) return g;
    return rc == SRLA_OK ? rc : srla_internal_set_error(rc, "host buffer too small for the window's hosts");
}

}  // extern "C"
