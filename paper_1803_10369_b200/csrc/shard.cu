// shard.cu — multi-GPU runs: owner partition of record
// batches and the sharded pipeline behind srla_shard_* (include/srla.h).
//
// Each GPU owns the hosts with reduce(3, aip, n) == rank and keeps a full,
// independent sketch for them. A host's records all land on one GPU, so its
// per-host results equal those of a CPU reference pipeline fed the
// owner-filtered sub-trace in original order (pipeline.hpp:110-129); stable
// partitions keep that order. The collectives — the per-slice report
// all-gather and, for range input, the record all-to-all — go through an
// srla_transport: NCCL (loaded with dlopen) or caller callbacks.
#include <cub/cub.cuh>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

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

// ---------------------------------------------------------------- NCCL (dlopen)
// libnccl.so.2 is loaded at first use, so the library carries no link-time
// NCCL dependency; inside a torch process the already-loaded copy is reused.
struct NcclApi {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string err;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) { fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name)); };
        sym(api.get_unique_id, "ncclGetUniqueId");
        sym(api.init_rank, "ncclCommInitRank");
        sym(api.destroy, "ncclCommDestroy");
        sym(api.all_gather, "ncclAllGather");
        sym(api.send, "ncclSend");
        sym(api.recv, "ncclRecv");
        sym(api.group_start, "ncclGroupStart");
        sym(api.group_end, "ncclGroupEnd");
        sym(api.error_string, "ncclGetErrorString");
        if (!api.get_unique_id || !api.init_rank || !api.all_gather || !api.send || !api.recv || !api.group_start ||
            !api.group_end)
            api.err = "libnccl.so.2 lacks a required symbol";
    });
    if (!api.err.empty()) throw std::runtime_error(api.err);
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "nccl error"));
}

struct NcclCtx {
    ncclComm_t comm = nullptr;
    uint32_t world = 1;
};

int nccl_allgather(void* ctx, const void* send, void* recv, uint64_t bytes, void* stream) {
    auto* c = static_cast<NcclCtx*>(ctx);
    return nccl().all_gather(send, recv, bytes, ncclChar, c->comm, static_cast<cudaStream_t>(stream)) == ncclSuccess ? 0 : 1;
}

int nccl_alltoallv(void* ctx, const void* send, const uint64_t* sb, const uint64_t* so, void* recv, const uint64_t* rb,
                   const uint64_t* ro, void* stream) {
    auto* c = static_cast<NcclCtx*>(ctx);
    const NcclApi& a = nccl();
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (a.group_start() != ncclSuccess) return 1;
    bool ok = true;
    for (uint32_t j = 0; j < c->world; ++j) {  // grouped point-to-point: one all-to-all
        if (sb[j]) ok &= a.send(static_cast<const char*>(send) + so[j], sb[j], ncclChar, static_cast<int>(j), c->comm, st) == ncclSuccess;
        if (rb[j]) ok &= a.recv(static_cast<char*>(recv) + ro[j], rb[j], ncclChar, static_cast<int>(j), c->comm, st) == ncclSuccess;
    }
    const bool ended = a.group_end() == ncclSuccess;  // the group is closed even after a failed enqueue
    return ok && ended ? 0 : 1;
}

// ---------------------------------------------------------------- shard kernels
__global__ void k_owner_keys(const Rec12* __restrict__ r, uint64_t n, uint64_t sub, uint32_t world,
                             uint32_t* __restrict__ key) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n; i += uint64_t(gridDim.x) * blockDim.x)
        key[i] = static_cast<uint32_t>((static_cast<uint64_t>(hash_u32(sub, r[i].src)) * world) >> 32);
}

// bucket starts of a sorted key array: start[b] = first index with key >= b
__global__ void k_bucket_starts(const uint32_t* __restrict__ key, uint64_t n, uint32_t world,
                                unsigned long long* __restrict__ start) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b > world) return;
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) / 2;
        if (key[mid] < b) lo = mid + 1;
        else hi = mid;
    }
    start[b] = lo;
}

// report words of every shard (rank-major, `stride` per rank, counts[r] valid)
// -> keys (host) and values (shard << 32 | weight) of the valid ones
__global__ void k_shard_words(const unsigned long long* __restrict__ words, const unsigned long long* __restrict__ counts,
                              const unsigned long long* __restrict__ base, uint32_t world, uint64_t stride,
                              uint32_t* __restrict__ keys, unsigned long long* __restrict__ vals) {
    const uint64_t total = uint64_t(world) * stride;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < total; i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = static_cast<uint32_t>(i / stride);
        const uint64_t j = i - uint64_t(r) * stride;
        if (j >= counts[r]) continue;
        const unsigned long long w = words[i];
        const uint64_t o = base[r] + j;
        keys[o] = static_cast<uint32_t>(w >> 32);
        vals[o] = (static_cast<unsigned long long>(r) << 32) | (w & 0xFFFFFFFFull);
    }
}

// merged (host, shard|weight) -> srla_entry through each shard's Eq. 9 table
// (luts: per rank L doubles then L flag bytes)
__global__ void k_shard_entries(const uint32_t* __restrict__ host, const unsigned long long* __restrict__ val,
                                uint64_t n, const uint8_t* __restrict__ luts, uint32_t L,
                                unsigned long long* __restrict__ out) {
    const uint64_t lut_bytes = uint64_t(L) * 9;
    for (uint64_t e = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; e < n; e += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t r = static_cast<uint32_t>(val[e] >> 32);
        const uint32_t w = static_cast<uint32_t>(val[e]);
        const uint8_t* lut = luts + r * lut_bytes;
        double est;
        memcpy(&est, lut + 8ull * w, 8);
        const uint8_t f = lut[8ull * L + w];
        unsigned long long* o = out + 3 * e;
        o[0] = static_cast<unsigned long long>(host[e]) | (static_cast<unsigned long long>(w) << 32);
        o[1] = static_cast<unsigned long long>(__double_as_longlong(est));
        o[2] = static_cast<unsigned long long>(f & 1u) | (static_cast<unsigned long long>((f >> 1) & 1u) << 8);
    }
}

}  // namespace srla

struct srla_shard;

namespace srla {

#define SK(x)                                                                                     \
    do {                                                                                          \
        cudaError_t e_ = (x);                                                                     \
        if (e_ != cudaSuccess) throw std::runtime_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
    } while (0)

template <typename T>
struct SBuf {
    T* p = nullptr;
    size_t cap = 0;
    bool pinned = false;
    ~SBuf() {
        if (p) pinned ? cudaFreeHost(p) : cudaFree(p);
    }
    void ensure(size_t n, bool host = false) {
        if (n <= cap && host == pinned) return;
        if (p) pinned ? cudaFreeHost(p) : cudaFree(p);
        p = nullptr;
        const size_t c = std::max<size_t>({n + n / 4, 256});
        if (host) SK(cudaMallocHost(&p, c * sizeof(T)));
        else SK(cudaMalloc(&p, c * sizeof(T)));
        cap = c;
        pinned = host;
    }
};

}  // namespace srla

struct srla_shard {
    srla_engine* eng = nullptr;
    srla_transport t{};
    srla_config cfg{};
    int device = 0;
    cudaStream_t st = nullptr;
    uint64_t sub3 = 0;
    srla::SBuf<uint8_t> recs, part, hstage, temp, stage_send, stage_recv;
    srla::SBuf<uint32_t> keys, keys2, rhosts, rweights, mkeys, mkeys2;
    srla::SBuf<unsigned long long> starts, counts, words, allwords, mvals, mvals2, entries, cnt1, cntall, base;
    srla::SBuf<uint8_t> lut, luts;
    std::vector<double> est;
    std::vector<uint8_t> flags;
    uint64_t last_total = 0;  // entries of the last merged report (kept in `entries`)
    cudaEvent_t ev_in = nullptr;
    ~srla_shard() {
        if (ev_in) cudaEventDestroy(ev_in);
    }

    // a collective through the transport, staged through pinned host buffers
    // when the transport works on host memory
    void allgather(const void* d_send, void* d_recv, uint64_t bytes) {
        const uint64_t W = t.world;
        if (!t.host_memory) {
            if (t.allgather(t.ctx, d_send, d_recv, bytes, st)) throw std::runtime_error("transport allgather failed");
            return;
        }
        stage_send.ensure(std::max<uint64_t>(bytes, 1), true);
        stage_recv.ensure(std::max<uint64_t>(bytes * W, 1), true);
        SK(cudaMemcpyAsync(stage_send.p, d_send, bytes, cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        if (t.allgather(t.ctx, stage_send.p, stage_recv.p, bytes, st)) throw std::runtime_error("transport allgather failed");
        SK(cudaMemcpyAsync(d_recv, stage_recv.p, bytes * W, cudaMemcpyHostToDevice, st));
    }
    void alltoallv(const void* d_send, const uint64_t* sb, const uint64_t* so, void* d_recv, const uint64_t* rb,
                   const uint64_t* ro) {
        const uint32_t W = t.world;
        if (!t.host_memory) {
            if (t.alltoallv(t.ctx, d_send, sb, so, d_recv, rb, ro, st)) throw std::runtime_error("transport alltoallv failed");
            return;
        }
        const uint64_t sn = so[W - 1] + sb[W - 1], rn = ro[W - 1] + rb[W - 1];
        stage_send.ensure(std::max<uint64_t>(sn, 1), true);
        stage_recv.ensure(std::max<uint64_t>(rn, 1), true);
        if (sn) SK(cudaMemcpyAsync(stage_send.p, d_send, sn, cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        if (t.alltoallv(t.ctx, stage_send.p, sb, so, stage_recv.p, rb, ro, st)) throw std::runtime_error("transport alltoallv failed");
        if (rn) SK(cudaMemcpyAsync(d_recv, stage_recv.p, rn, cudaMemcpyHostToDevice, st));
    }

    template <typename Fn>
    void cub_call(Fn&& fn) {
        size_t bytes = 0;
        SK(fn(static_cast<void*>(nullptr), bytes));
        temp.ensure(bytes + 16);
        SK(fn(static_cast<void*>(temp.p), bytes));
    }

    static uint32_t grid(uint64_t n) { return static_cast<uint32_t>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 16))); }

    // SRLA_SHARD_RANGE: owner-partition this rank's range (stable radix sort
    // on the owner) and exchange; returns the received records (device)
    const srla_record* exchange(const srla_record* d_in, uint64_t n, uint64_t* n_recv) {
        const uint32_t W = t.world;
        int end_bit = 1;
        while ((1u << end_bit) < W) ++end_bit;
        keys.ensure(std::max<uint64_t>(n, 1));
        keys2.ensure(std::max<uint64_t>(n, 1));
        part.ensure(std::max<uint64_t>(n, 1) * 12);
        starts.ensure(W + 1);
        if (n > (1ull << 30)) throw std::runtime_error("shard range above 2^30 records");  // one sort call's int count
        if (n) {
            srla::k_owner_keys<<<grid(n), 256, 0, st>>>(reinterpret_cast<const srla::Rec12*>(d_in), n, sub3, W, keys.p);
            SK(cudaGetLastError());
            auto* vin = reinterpret_cast<const srla::Rec12*>(d_in);
            auto* vout = reinterpret_cast<srla::Rec12*>(part.p);
            // stable, so records keep slice order per owner
            cub_call([&](void* tp, size_t& b) {
                return cub::DeviceRadixSort::SortPairs(tp, b, keys.p, keys2.p, vin, vout, static_cast<int>(n), 0, end_bit, st);
            });
        }
        srla::k_bucket_starts<<<1, 256, 0, st>>>(keys2.p, n, W, starts.p);
        SK(cudaGetLastError());
        // counts matrix: every rank's per-owner counts
        cnt1.ensure(W);
        cntall.ensure(uint64_t(W) * W);
        std::vector<unsigned long long> st_h(W + 1);
        SK(cudaMemcpyAsync(st_h.data(), starts.p, (W + 1) * 8, cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        std::vector<unsigned long long> mine(W);
        for (uint32_t j = 0; j < W; ++j) mine[j] = st_h[j + 1] - st_h[j];
        SK(cudaMemcpyAsync(cnt1.p, mine.data(), W * 8, cudaMemcpyHostToDevice, st));
        allgather(cnt1.p, cntall.p, uint64_t(W) * 8);
        std::vector<unsigned long long> all(uint64_t(W) * W);
        SK(cudaMemcpyAsync(all.data(), cntall.p, uint64_t(W) * W * 8, cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        std::vector<uint64_t> sb(W), so(W), rb(W), ro(W);
        uint64_t rn = 0;
        for (uint32_t j = 0; j < W; ++j) {
            sb[j] = mine[j] * 12;
            so[j] = st_h[j] * 12;
            rb[j] = all[uint64_t(j) * W + t.rank] * 12;  // from rank j, in rank (= slice) order
            ro[j] = rn * 12;
            rn += all[uint64_t(j) * W + t.rank];
        }
        recs.ensure(std::max<uint64_t>(rn, 1) * 12);
        alltoallv(part.p, sb.data(), so.data(), recs.p, rb.data(), ro.data());
        *n_recv = rn;
        return reinterpret_cast<const srla_record*>(recs.p);
    }

    // merged report of every shard into `out` (host); returns its size
    uint64_t merge_report(uint64_t n, uint64_t slice_id, srla_entry* out, uint64_t cap) {
        const uint32_t W = t.world;
        const uint32_t L = cfg.linear_slots + 1;
        // counts
        cnt1.ensure(1);
        cntall.ensure(W);
        const unsigned long long nn = n;
        SK(cudaMemcpyAsync(cnt1.p, &nn, 8, cudaMemcpyHostToDevice, st));
        allgather(cnt1.p, cntall.p, 8);
        std::vector<unsigned long long> cnt(W);
        SK(cudaMemcpyAsync(cnt.data(), cntall.p, W * 8, cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        uint64_t mx = 1, total = 0;
        std::vector<unsigned long long> base_h(W);
        for (uint32_t r = 0; r < W; ++r) {
            mx = std::max<uint64_t>(mx, cnt[r]);
            base_h[r] = total;
            total += cnt[r];
        }
        // (host << 32 | weight) words, padded to the largest shard
        words.ensure(mx);
        allwords.ensure(uint64_t(W) * mx);
        pack_words(n, mx);
        allgather(words.p, allwords.p, mx * 8);
        // Eq. 9 tables
        lut.ensure(uint64_t(L) * 9);
        luts.ensure(uint64_t(W) * L * 9);
        std::vector<uint8_t> lh(uint64_t(L) * 9);
        std::memcpy(lh.data(), est.data(), uint64_t(L) * 8);
        std::memcpy(lh.data() + uint64_t(L) * 8, flags.data(), L);
        SK(cudaMemcpyAsync(lut.p, lh.data(), lh.size(), cudaMemcpyHostToDevice, st));
        allgather(lut.p, luts.p, uint64_t(L) * 9);
        last_total = total;
        if (!total) {
            SK(cudaStreamSynchronize(st));
            return 0;
        }
        base.ensure(W);
        counts.ensure(W);
        SK(cudaMemcpyAsync(base.p, base_h.data(), W * 8, cudaMemcpyHostToDevice, st));
        SK(cudaMemcpyAsync(counts.p, cnt.data(), W * 8, cudaMemcpyHostToDevice, st));
        mkeys.ensure(total);
        mkeys2.ensure(total);
        mvals.ensure(total);
        mvals2.ensure(total);
        srla::k_shard_words<<<grid(uint64_t(W) * mx), 256, 0, st>>>(allwords.p, counts.p, base.p, W, mx, mkeys.p, mvals.p);
        SK(cudaGetLastError());
        // shards own disjoint hosts: the merge is a sort by host
        cub_call([&](void* tp, size_t& b) {
            return cub::DeviceRadixSort::SortPairs(tp, b, mkeys.p, mkeys2.p, mvals.p, mvals2.p, static_cast<int>(total), 0, 32, st);
        });
        entries.ensure(3 * total);
        srla::k_shard_entries<<<grid(total), 256, 0, st>>>(mkeys2.p, mvals2.p, total, luts.p, L, entries.p);
        SK(cudaGetLastError());
        last_total = total;
        if (total <= cap) SK(cudaMemcpyAsync(out, entries.p, total * sizeof(srla_entry), cudaMemcpyDeviceToHost, st));
        SK(cudaStreamSynchronize(st));
        (void)slice_id;
        return total;
    }

    void pack_words(uint64_t n, uint64_t mx);
};

namespace srla {
__global__ void k_pack_words(const uint32_t* __restrict__ h, const uint32_t* __restrict__ w, uint64_t n, uint64_t mx,
                             unsigned long long* __restrict__ out) {
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < mx; i += uint64_t(gridDim.x) * blockDim.x)
        out[i] = i < n ? (static_cast<unsigned long long>(h[i]) << 32) | w[i] : 0ull;
}
}  // namespace srla

void srla_shard::pack_words(uint64_t n, uint64_t mx) {
    srla::k_pack_words<<<grid(mx), 256, 0, st>>>(rhosts.p, rweights.p, n, mx, words.p);
    SK(cudaGetLastError());
}

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

extern "C" {

srla_status srla_nccl_unique_id(void* id128) {
    try {
        if (!id128) return srla_internal_set_error(SRLA_E_INVALID, "null id");
        ncclUniqueId id;
        srla::nccl_check(srla::nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id128, &id, sizeof(id));
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

srla_status srla_transport_nccl(const void* id128, uint32_t rank, uint32_t world, int device, srla_transport* out) {
    try {
        if (!id128 || !out || world == 0 || rank >= world) return srla_internal_set_error(SRLA_E_INVALID, "bad NCCL transport arguments");
        SK(cudaSetDevice(device));
        ncclUniqueId id;
        std::memcpy(&id, id128, sizeof(id));
        auto* c = new srla::NcclCtx();
        c->world = world;
        try {
            srla::nccl_check(srla::nccl().init_rank(&c->comm, static_cast<int>(world), id, static_cast<int>(rank)), "ncclCommInitRank");
        } catch (...) {
            delete c;
            throw;
        }
        *out = srla_transport{c, rank, world, 0, srla::nccl_allgather, srla::nccl_alltoallv};
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

srla_status srla_transport_nccl_destroy(srla_transport* t) {
    if (!t || !t->ctx) return srla_internal_set_error(SRLA_OK, "");
    auto* c = static_cast<srla::NcclCtx*>(t->ctx);
    if (c->comm) srla::nccl().destroy(c->comm);
    delete c;
    t->ctx = nullptr;
    return srla_internal_set_error(SRLA_OK, "");
}

srla_status srla_shard_create(const srla_config* cfg, int device, const srla_transport* t, srla_shard** out) {
    if (!cfg || !t || !out || !t->allgather || !t->alltoallv || t->world == 0 || t->rank >= t->world)
        return srla_internal_set_error(SRLA_E_INVALID, "bad shard arguments");
    auto* s = new srla_shard();
    const srla_status rc = srla_create(cfg, device, &s->eng);
    if (rc != SRLA_OK) {
        delete s;
        return rc;  // srla_create set the message
    }
    s->t = *t;
    s->cfg = *cfg;
    s->device = device;
    s->sub3 = srla::sub_key(cfg->seed, 3);
    void* st = nullptr;
    srla_stream(s->eng, &st);
    s->st = static_cast<cudaStream_t>(st);
    *out = s;
    return srla_internal_set_error(SRLA_OK, "");
}

srla_status srla_shard_destroy(srla_shard* s) {
    if (!s) return srla_internal_set_error(SRLA_OK, "");
    cudaSetDevice(s->device);
    srla_destroy(s->eng);
    delete s;
    return srla_internal_set_error(SRLA_OK, "");
}

srla_status srla_shard_last_report(srla_shard* s, srla_entry* out, uint64_t cap, uint64_t* n_out) {
    if (!s || !n_out) return srla_internal_set_error(SRLA_E_INVALID, "null shard");
    *n_out = s->last_total;
    if (s->last_total > cap) return srla_internal_set_error(SRLA_E_CAPACITY, "report buffer too small");
    try {
        SK(cudaSetDevice(s->device));
        if (s->last_total) {
            SK(cudaMemcpyAsync(out, s->entries.p, s->last_total * sizeof(srla_entry), cudaMemcpyDeviceToHost, s->st));
            SK(cudaStreamSynchronize(s->st));
        }
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

srla_status srla_shard_engine(srla_shard* s, srla_engine** e) {
    if (!s || !e) return srla_internal_set_error(SRLA_E_INVALID, "null shard");
    *e = s->eng;
    return srla_internal_set_error(SRLA_OK, "");
}

srla_status srla_shard_process_slice(srla_shard* s, uint64_t slice_id, const srla_record* recs, uint64_t n,
                                     int on_device, int input_mode, int want_report, srla_entry* out, uint64_t cap,
                                     uint64_t* n_out, uint64_t* n_scanned) {
    if (!s || (n && !recs) || (input_mode != SRLA_SHARD_OWNED && input_mode != SRLA_SHARD_RANGE))
        return srla_internal_set_error(SRLA_E_INVALID, "bad shard process_slice arguments");
    try {
        SK(cudaSetDevice(s->device));
        const srla_record* d = recs;
        uint64_t m = n;
        if (on_device && n) {  // device records: ordered after the legacy default stream (srla_scan_batch's contract)
            if (!s->ev_in) SK(cudaEventCreateWithFlags(&s->ev_in, cudaEventDisableTiming));
            SK(cudaEventRecord(s->ev_in, cudaStreamLegacy));
            SK(cudaStreamWaitEvent(s->st, s->ev_in, 0));
        }
        if (!on_device && n) {  // host records: one staged copy
            s->hstage.ensure(n * 12);
            SK(cudaMemcpyAsync(s->hstage.p, recs, n * 12, cudaMemcpyHostToDevice, s->st));
            d = reinterpret_cast<const srla_record*>(s->hstage.p);
        }
        if (input_mode == SRLA_SHARD_RANGE && s->t.world > 1) d = s->exchange(d, n, &m);  // received: s->recs
        srla_status rc = srla_scan_device(s->eng, d, m, s->st, nullptr, 0, nullptr);
        if (rc != SRLA_OK) return rc;
        if (n_scanned) *n_scanned = m;
        const uint32_t L = s->cfg.linear_slots + 1;
        const bool due = want_report && slice_id + 1 >= s->cfg.window;
        uint64_t cands = 0;
        srla_candidates(s->eng, nullptr, 0, &cands);
        s->rhosts.ensure(std::max<uint64_t>(cands, 1));
        s->rweights.ensure(std::max<uint64_t>(cands, 1));
        s->est.resize(L);
        s->flags.resize(L);
        uint64_t nr = 0, ne = 0;
        rc = srla_end_slice_compact(s->eng, slice_id, want_report, s->rhosts.p, s->rweights.p, s->rhosts.cap, &ne,
                                    s->est.data(), s->flags.data(), &nr);
        if (rc != SRLA_OK) return rc;
        uint64_t total = 0;
        if (due) {
            if (!out && cap) return srla_internal_set_error(SRLA_E_INVALID, "null report buffer");
            total = s->merge_report(ne, slice_id, out, cap);
        }
        if (n_out) *n_out = total;
        if (total > cap)  // the slice is done; the merged report waits in srla_shard_last_report
            return srla_internal_set_error(SRLA_E_CAPACITY, ("report buffer holds " + std::to_string(cap) + " entries, " +
                                                             std::to_string(total) + " needed").c_str());
        return srla_internal_set_error(SRLA_OK, "");
    } catch (const std::exception& e) {
        return srla_internal_set_error(SRLA_E_CUDA, e.what());
    }
}

}  // extern "C"
