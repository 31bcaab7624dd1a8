// sspread/snapshot.hpp — drop-in "SSEA" v1 sketch snapshots
// (/root/reference/proj/include/sspread/snapshot.hpp): the same bytes as the
// reference's save_snapshot (tests/test_snapshot_bytes.py), rows streamed
// straight between HBM and the file in bounded pinned pieces, so a GPU sketch
// and a CPU reference sketch exchange state bit-exactly.
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <string>
#include <utility>
#include <vector>

#include "sea.hpp"

namespace sspread {

inline constexpr char kSnapshotMagic[4] = {'S', 'S', 'E', 'A'};
inline constexpr uint32_t kSnapshotVersion = 1;

struct SnapshotHeader {
    uint32_t version = kSnapshotVersion;
    uint32_t word_bytes = 1;
    SeaConfig config;
};

namespace detail {
class LeWriter {
  public:
    void u32(uint32_t v) {
        for (int b = 0; b < 4; ++b) buf_.push_back(static_cast<char>(v >> (8 * b)));
    }
    void u64(uint64_t v) {
        u32(static_cast<uint32_t>(v));
        u32(static_cast<uint32_t>(v >> 32));
    }
    void f64(double d) {
        uint64_t v;
        std::memcpy(&v, &d, 8);
        u64(v);
    }
    template <typename T>
    void words(std::span<const T> w) {
        for (const T x : w)
            for (size_t b = 0; b < sizeof(T); ++b) buf_.push_back(static_cast<char>(static_cast<uint32_t>(x) >> (8 * b)));
    }
    void raw(const char* p, size_t n) { buf_.append(p, n); }
    const std::string& bytes() const { return buf_; }

  private:
    std::string buf_;
};

class LeReader {
  public:
    explicit LeReader(std::istream& in) : in_(in) {}
    void raw(void* p, size_t n, const char* what) {
        in_.read(static_cast<char*>(p), static_cast<std::streamsize>(n));
        if (static_cast<size_t>(in_.gcount()) != n) throw InputError(std::string("truncated input reading ") + what);
    }
    uint32_t u32(const char* what) {
        unsigned char b[4];
        raw(b, 4, what);
        return uint32_t(b[0]) | uint32_t(b[1]) << 8 | uint32_t(b[2]) << 16 | uint32_t(b[3]) << 24;
    }
    uint64_t u64(const char* what) {
        const uint64_t lo = u32(what);
        return lo | uint64_t(u32(what)) << 32;
    }
    double f64(const char* what) {
        const uint64_t v = u64(what);
        double d;
        std::memcpy(&d, &v, 8);
        return d;
    }
    template <typename T>
    void words(std::span<T> w, const char* what) {
        std::vector<unsigned char> b(w.size() * sizeof(T));
        raw(b.data(), b.size(), what);
        for (size_t i = 0; i < w.size(); ++i) {
            uint32_t v = 0;
            for (size_t k = 0; k < sizeof(T); ++k) v |= uint32_t(b[i * sizeof(T) + k]) << (8 * k);
            w[i] = static_cast<T>(v);
        }
    }

  private:
    std::istream& in_;
};
}  // namespace detail

namespace detail {
// Pinned staging for streaming rows between HBM and a snapshot file: rows move
// in bounded pieces (a 2^24-column linear row is 16 GiB), by DMA.
struct PinnedChunk {
    static constexpr uint64_t kBytes = 64ull << 20;
    void* p = nullptr;
    PinnedChunk() { check(srla_host_alloc(kBytes, &p), "srla_host_alloc"); }
    ~PinnedChunk() { srla_host_free(p); }
    PinnedChunk(const PinnedChunk&) = delete;
    PinnedChunk& operator=(const PinnedChunk&) = delete;
    char* data() const { return static_cast<char*>(p); }
};
}  // namespace detail

// snapshot.hpp:109-136. The header and candidate list are written as the
// reference writes them; every row streams from the device (x86 words are
// already little-endian, the reference's explicit packing), through one
// pinned 64 MiB piece at a time — no host mirror of the sketch.
template <RecorderWord W>
void save_snapshot(const EstimatorArray<W>& sea, const CandidateList& csip, const std::string& path) {
    const SeaConfig& c = sea.config();
    detail::LeWriter w;
    w.raw(kSnapshotMagic, 4);
    w.u32(kSnapshotVersion);
    w.u32(sizeof(W));
    for (uint32_t v : {c.rows, c.cols, c.rough_slots, c.linear_slots, c.recorder_bits, c.window, c.theta}) w.u32(v);
    w.f64(c.fill_ratio);
    w.u64(c.seed);
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw InputError("cannot open snapshot for writing: " + path);
    out.write(w.bytes().data(), static_cast<std::streamsize>(w.bytes().size()));
    sea.to_device();  // a span-modified mirror is the current state
    detail::PinnedChunk buf;
    for (uint32_t i = 0; i < c.rows; ++i)
        for (int kind : {SRLA_INDICATOR, SRLA_ROUGH, SRLA_LINEAR}) {
            uint64_t bytes = 0;
            detail::check(srla_row_bytes(sea.eng(), kind, &bytes), "srla_row_bytes");
            for (uint64_t off = 0; off < bytes; off += detail::PinnedChunk::kBytes) {
                const uint64_t m = std::min(detail::PinnedChunk::kBytes, bytes - off);
                detail::check(srla_export_range(sea.eng(), i, kind, off, buf.data(), m), "srla_export_range");
                out.write(buf.data(), static_cast<std::streamsize>(m));
            }
        }
    detail::LeWriter tail;
    tail.u64(csip.size());
    for (uint32_t h : csip.hosts()) tail.u32(h);
    out.write(tail.bytes().data(), static_cast<std::streamsize>(tail.bytes().size()));
    if (!out) throw InputError("write failure on snapshot: " + path);
}

inline SnapshotHeader read_snapshot_header(std::istream& in) {
    detail::LeReader r(in);
    char magic[4];
    r.raw(magic, 4, "magic");
    if (std::memcmp(magic, kSnapshotMagic, 4) != 0) throw InputError("not a sketch snapshot (bad magic)");
    SnapshotHeader h;
    h.version = r.u32("version");
    if (h.version != kSnapshotVersion) throw InputError("unsupported snapshot version " + std::to_string(h.version));
    h.word_bytes = r.u32("word width");
    h.config.rows = r.u32("rows");
    h.config.cols = r.u32("cols");
    h.config.rough_slots = r.u32("rough slots");
    h.config.linear_slots = r.u32("linear slots");
    h.config.recorder_bits = r.u32("recorder bits");
    h.config.window = r.u32("window");
    h.config.theta = r.u32("theta");
    h.config.fill_ratio = r.f64("fill ratio");
    h.config.seed = r.u64("seed");
    return h;
}

inline SnapshotHeader read_snapshot_header(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw InputError("cannot open snapshot: " + path);
    return read_snapshot_header(in);
}

template <RecorderWord W>
std::pair<EstimatorArray<W>, CandidateList> load_snapshot(const std::string& path, int device = 0) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw InputError("cannot open snapshot: " + path);
    const SnapshotHeader h = read_snapshot_header(in);
    if (h.word_bytes != sizeof(W))
        throw InputError("snapshot stores " + std::to_string(h.word_bytes) + "-byte recorders, loader instantiated for " +
                         std::to_string(sizeof(W)));
    EstimatorArray<W> sea(h.config, device);
    detail::LeReader r(in);
    detail::PinnedChunk buf;
    for (uint32_t i = 0; i < h.config.rows; ++i)
        for (int kind : {SRLA_INDICATOR, SRLA_ROUGH, SRLA_LINEAR}) {
            const char* what = kind == SRLA_INDICATOR ? "indicators" : kind == SRLA_ROUGH ? "rough recorders"
                                                                                          : "linear recorders";
            uint64_t bytes = 0;
            detail::check(srla_row_bytes(sea.eng(), kind, &bytes), "srla_row_bytes");
            for (uint64_t off = 0; off < bytes; off += detail::PinnedChunk::kBytes) {
                const uint64_t m = std::min(detail::PinnedChunk::kBytes, bytes - off);
                r.raw(buf.data(), m, what);
                detail::check(srla_import_range(sea.eng(), i, kind, off, buf.data(), m), "srla_import_range");
            }
        }
    const uint64_t n = r.u64("candidate count");
    CandidateList csip;
    for (uint64_t i = 0; i < n; ++i) csip.insert(r.u32("candidate"));
    char extra;
    if (in.read(&extra, 1), in.gcount() != 0) throw InputError("trailing bytes after snapshot payload");
    return {std::move(sea), std::move(csip)};
}

}  // namespace sspread
