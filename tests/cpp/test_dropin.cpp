// C++ drop-in tests: the reference's own hot-path unit tests (tests/test_sea.cpp,
// tests/test_pipeline.cpp, tests/test_snapshot.cpp) rewritten against the
// drop-in headers in include/sspread/, which run on the B200 engine.
//
//   test_dropin            run the unit tests (exit code = failures)
//   test_dropin replay <trace.bin> <out.txt> rows cols g gl bits k theta seed
//                          DetectPipeline::process_slice over a binary trace's
//                          one-second slices; dumps per slice the report and
//                          candidate list for tests/test_dropin.py to compare
//                          with the CPU oracle.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <fstream>
#include <random>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "sspread/oracle.hpp"
#include "sspread/pipeline.hpp"
#include "sspread/sea.hpp"
#include "sspread/snapshot.hpp"

using namespace sspread;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                              \
    do {                                                                      \
        ++g_checks;                                                           \
        if (!(c)) {                                                           \
            ++g_fail;                                                         \
            std::fprintf(stderr, "%s:%d CHECK failed: %s\n", __FILE__, __LINE__, #c); \
        }                                                                     \
    } while (0)
#define CHECK_THROWS_AS(expr, T)            \
    do {                                    \
        bool thrown_ = false;               \
        try {                               \
            (void)(expr);                   \
        } catch (const T&) {                \
            thrown_ = true;                 \
        } catch (...) {                     \
        }                                   \
        CHECK(thrown_ && #T);               \
    } while (0)

static SeaConfig small_config() {
    SeaConfig cfg;
    cfg.rows = 2;
    cfg.cols = 16;
    cfg.rough_slots = 8;
    cfg.linear_slots = 32;
    cfg.recorder_bits = 8;
    cfg.window = 4;
    cfg.theta = 8;
    cfg.seed = 0xFACE;
    return cfg;
}

using Pair = std::pair<uint32_t, uint32_t>;

static void scan_all(EstimatorArray<uint8_t>& sea, const std::vector<Pair>& pairs, CandidateList& csip) {
    std::vector<uint32_t> sink;
    for (const auto& [a, b] : pairs) sea.scan_ip_pair(a, b, sink);
    for (uint32_t h : sink) csip.insert(h);
}

static void test_single_pair() {
    SeaConfig cfg = small_config();
    cfg.rows = 1;
    EstimatorArray<uint8_t> sea(cfg);
    CHECK(sea.params().tau == 0);
    const uint32_t aip = 0x0A000001, bip = 0x08080808;
    std::vector<uint32_t> sink;
    sea.scan_ip_pair(aip, bip, sink);
    const auto& h = sea.hashes();
    const uint32_t col = sea.column_of(0, aip);
    const uint32_t rslot = h.reduce(kRoughSlotHash, bip, cfg.rough_slots);
    const uint32_t lslot = h.u32(kSampleHash, bip) % cfg.linear_slots;
    CHECK(sea.rough_row(0)[col * cfg.rough_slots + rslot] == 0);
    CHECK(sea.linear_row(0)[col * cfg.linear_slots + lslot] == 0);
    CHECK(count_active(sea.rough_row(0), cfg.window) == 1);
    CHECK(count_active(sea.linear_row(0), cfg.window) == 1);
    CHECK(sea.union_rough_weight(aip) == 1);
    CHECK(sink.empty());
}

static void test_indicator_suppression() {
    EstimatorArray<uint8_t> sea(small_config());
    CandidateList csip;
    const uint32_t aip = 0x0A000002;
    std::vector<Pair> pairs;
    for (uint32_t i = 0; i < 64; ++i) pairs.emplace_back(aip, 0xC0000000u + i);
    scan_all(sea, pairs, csip);
    CHECK(csip.size() == 1);
    CHECK(csip.hosts()[0] == aip);
    const uint16_t bit = static_cast<uint16_t>(1u << sea.hashes().reduce(kIndicatorHash, aip, kIndicatorBits));
    for (uint32_t i = 0; i < sea.config().rows; ++i) CHECK((sea.indicator_row(i)[sea.column_of(i, aip)] & bit) != 0);
}

static void test_union_view() {
    SeaConfig cfg = small_config();
    EstimatorArray<uint8_t> sea(cfg);
    const auto u = sea.union_view(0x0A000003, true);
    CHECK(u.indicator == 0);
    CHECK(count_active<uint8_t>(u.rough, cfg.window) == 0);
    for (uint8_t r : u.rough) CHECK(r == sea.model().expired);
    const uint32_t aip = 0x0A000005;
    sea.rough_row(0)[sea.column_of(0, aip) * cfg.rough_slots + 3] = 5;
    sea.rough_row(1)[sea.column_of(1, aip) * cfg.rough_slots + 3] = 9;
    const auto v = sea.union_view(aip, false);
    CHECK(v.rough[3] == 9);
    CHECK(v.linear.empty());
}

static void test_row_fill_fraction() {
    SeaConfig cfg = small_config();
    cfg.rows = 1;
    cfg.cols = 4;
    cfg.linear_slots = 1024;
    EstimatorArray<uint8_t> sea(cfg);
    CHECK(sea.row_fill_fraction(0) == 0.0);
    CHECK_THROWS_AS(sea.row_fill_fraction(1), std::invalid_argument);
    auto row = sea.linear_row(0);
    for (uint32_t i = 0; i < 512; ++i) row[i * 8] = 0;
    CHECK(sea.row_fill_fraction(0) == 0.125);
    CHECK_THROWS_AS(sea.linear_row(1), std::out_of_range);
}

static void test_corrected_estimate() {
    SeaConfig cfg = small_config();
    cfg.rows = 4;
    cfg.linear_slots = 1024;
    cfg.recorder_bits = 16;
    cfg.window = 300;
    cfg.theta = 1024;
    EstimatorArray<uint16_t> sea(cfg);
    for (uint32_t w : {0u, 1u, 100u, 500u, 1023u}) CHECK(sea.corrected_estimate_from(w, 0.0) == linear_estimate(w, 1024));
    CHECK(!sea.corrected_estimate_from(1024, 0.0).has_value());
    CHECK(sea.corrected_estimate_from(4, 0.00390625).value() == 0.0);
    const double up = 0.25 * 0.25 * 0.25 * 0.25;
    CHECK(std::abs(sea.corrected_estimate_from(300, up).value() - 350.99291022602281) < 350.99291022602281 * 1e-12);
    CHECK(sea.corrected_estimate_from(100, 1.0 - 1e-13) == linear_estimate(100, 1024));
    // linear_estimate rejects a weight above the slot count (estimators.hpp:142)
    CHECK_THROWS_AS(sea.corrected_estimate_from(1025, 1.0), std::invalid_argument);
    WindowConfig wc;  // trace.hpp:78-87
    wc.window = 300;
    wc.recorder_bits = 8;
    CHECK_THROWS_AS(wc.validate(), std::invalid_argument);
    wc.recorder_bits = 16;
    wc.validate();
}

// DetectPipeline::run on a binary trace: the device front end reports a
// timestamp regression with for_each_record's text (trace.hpp:116-118).
static void test_run_regression_message() {
    const std::string path = (std::filesystem::temp_directory_path() / "srla_regress.bin").string();
    {
        std::ofstream f(path, std::ios::binary);
        f.write("SRLT\x01", 5);
        const uint32_t recs[3][3] = {{100, 0x0A000001, 0x64000001}, {105, 0x0A000002, 0x64000002}, {103, 0x0A000003, 0x64000003}};
        f.write(reinterpret_cast<const char*>(recs), sizeof recs);
    }
    RunConfig rc;
    rc.sea = small_config();
    rc.slice_seconds = 1;
    DetectPipeline<uint8_t> pipe(rc);
    std::string msg;
    try {
        pipe.run(path, {});
    } catch (const InputError& e) {
        msg = e.what();
    }
    CHECK(msg == "timestamp regression at record 2 of " + path + " (103 after 105)");
    std::filesystem::remove(path);
}

static void test_slide() {
    SeaConfig cfg = small_config();
    {
        EstimatorArray<uint8_t> sea(cfg);
        CandidateList csip;
        std::vector<uint32_t> sink;
        sea.scan_ip_pair(0x0A000006, 0xB0000001, sink);
        auto out = sea.slide(csip);
        CHECK(out.empty());
        const uint32_t col = sea.column_of(0, 0x0A000006);
        const uint32_t lslot = sea.hashes().u32(kSampleHash, 0xB0000001) % cfg.linear_slots;
        CHECK(sea.linear_row(0)[col * cfg.linear_slots + lslot] == 1);
    }
    {
        EstimatorArray<uint8_t> sea(cfg);
        const uint32_t aip = 0x0A000007;
        CandidateList csip;
        csip.insert(aip);
        for (uint32_t i = 0; i < cfg.rows; ++i) {
            auto row = sea.rough_row(i);
            const uint32_t base = sea.column_of(i, aip) * cfg.rough_slots;
            row[base + 0] = row[base + 1] = row[base + 2] = 0;
        }
        auto out = sea.slide(csip);
        CHECK(out.size() == 1);
        const uint16_t bit = static_cast<uint16_t>(1u << sea.hashes().reduce(kIndicatorHash, aip, kIndicatorBits));
        for (uint32_t i = 0; i < cfg.rows; ++i) CHECK((sea.indicator_row(i)[sea.column_of(i, aip)] & bit) != 0);
    }
    {
        EstimatorArray<uint8_t> sea(cfg);
        const uint32_t aip = 0x0A000008;
        CandidateList csip;
        csip.insert(aip);
        std::vector<uint32_t> sink;
        for (uint32_t i = 0; i < 40; ++i) sea.scan_ip_pair(aip, 0xD0000000u + i, sink);
        CHECK(sea.union_rough_weight(aip) >= sea.weight_threshold());
        for (int s = 0; s < 3; ++s) {
            csip = sea.slide(csip);
            CHECK(csip.size() == 1);
        }
        csip = sea.slide(csip);
        CHECK(csip.empty());
        CHECK(sea.union_rough_weight(aip) == 0);
    }
}

static void test_window_report() {
    SeaConfig cfg = small_config();
    cfg.theta = 30;
    cfg.rough_slots = 32;
    cfg.linear_slots = 128;
    EstimatorArray<uint8_t> sea(cfg);
    CHECK(sea.report_window(CandidateList{}, 3).entries.empty());
    CandidateList csip;
    std::vector<Pair> pairs;
    for (uint32_t i = 0; i < 60; ++i) pairs.emplace_back(0x0A0000FF, 0xE0000000u + i);
    for (uint32_t i = 0; i < 5; ++i) pairs.emplace_back(0x0A000001, 0xE1000000u + i);
    scan_all(sea, pairs, csip);
    csip.insert(0x0A000001);
    CHECK(csip.contains(0x0A0000FF));
    const auto report = sea.report_window(csip, 0);
    CHECK(report.entries.size() == 2);
    CHECK(report.entries[0].host == 0x0A000001);
    CHECK(report.entries[1].host == 0x0A0000FF);
    CHECK(!report.entries[0].is_super);
    CHECK(report.entries[1].is_super);
}

static void test_order_independence() {
    std::mt19937_64 rng(0x0DDE);
    for (int trial = 0; trial < 5; ++trial) {
        SeaConfig cfg = small_config();
        cfg.cols = 256;
        cfg.seed = rng();
        std::vector<Pair> pairs;
        for (int i = 0; i < 400; ++i) pairs.emplace_back(0x0A000000u + rng() % 24, 0xB0000000u + rng() % 128);
        EstimatorArray<uint8_t> a(cfg), b(cfg);
        CandidateList ca, cb;
        scan_all(a, pairs, ca);
        std::shuffle(pairs.begin(), pairs.end(), rng);
        scan_all(b, pairs, cb);
        for (uint32_t i = 0; i < cfg.rows; ++i) {
            CHECK(std::ranges::equal(a.rough_row(i), b.rough_row(i)));
            CHECK(std::ranges::equal(a.linear_row(i), b.linear_row(i)));
            CHECK(std::ranges::equal(a.indicator_row(i), b.indicator_row(i)));
        }
        CHECK(std::set<uint32_t>(ca.hosts().begin(), ca.hosts().end()) ==
              std::set<uint32_t>(cb.hosts().begin(), cb.hosts().end()));
    }
}

static void test_snapshot_round_trip() {
    SeaConfig cfg;
    cfg.rows = 3;
    cfg.cols = 8;
    cfg.rough_slots = 8;
    cfg.linear_slots = 16;
    cfg.recorder_bits = 8;
    cfg.window = 5;
    cfg.theta = 16;
    cfg.seed = 0x1DEA;
    EstimatorArray<uint8_t> sea(cfg);
    CandidateList csip;
    std::vector<uint32_t> sink;
    std::mt19937_64 rng(404);
    for (int i = 0; i < 500; ++i) sea.scan_ip_pair(0x0A000000u + rng() % 16, 0xB0000000u + rng() % 64, sink);
    for (uint32_t h : sink) csip.insert(h);
    csip = sea.slide(csip);
    for (int i = 0; i < 200; ++i) sea.scan_ip_pair(0x0A000000u + rng() % 16, 0xB0000000u + rng() % 64, sink);
    for (uint32_t h : sink) csip.insert(h);
    const auto dir = std::filesystem::temp_directory_path() / ("srla-dropin-" + std::to_string(rng()));
    std::filesystem::create_directories(dir);
    const auto p1 = (dir / "a.ssea").string(), p2 = (dir / "b.ssea").string();
    save_snapshot(sea, csip, p1);
    auto [loaded, loaded_csip] = load_snapshot<uint8_t>(p1);
    for (uint32_t i = 0; i < 3; ++i) {
        CHECK(std::ranges::equal(sea.rough_row(i), loaded.rough_row(i)));
        CHECK(std::ranges::equal(sea.linear_row(i), loaded.linear_row(i)));
        CHECK(std::ranges::equal(sea.indicator_row(i), loaded.indicator_row(i)));
    }
    CHECK(loaded_csip.hosts() == csip.hosts());
    save_snapshot(loaded, loaded_csip, p2);
    std::ifstream f1(p1, std::ios::binary), f2(p2, std::ios::binary);
    const std::string b1{std::istreambuf_iterator<char>(f1), {}}, b2{std::istreambuf_iterator<char>(f2), {}};
    CHECK(b1 == b2);
    // resume: identical pushes and retention after a restore
    std::vector<uint32_t> s1, s2;
    std::vector<Pair> more;
    for (int i = 0; i < 300; ++i) more.emplace_back(0x0A000000u + rng() % 16, 0xB0000000u + rng() % 64);
    for (const auto& [a, b] : more) {
        sea.scan_ip_pair(a, b, s1);
        loaded.scan_ip_pair(a, b, s2);
    }
    CHECK(s1 == s2);
    CHECK(sea.slide(csip).hosts() == loaded.slide(loaded_csip).hosts());
    std::filesystem::remove_all(dir);
}

static void test_pipeline_validation() {
    RunConfig rc;
    rc.sea.window = 2;
    rc.sea.recorder_bits = 1;
    CHECK_THROWS_AS(rc.validate(), ConfigError);
    rc = RunConfig{};
    rc.sea.cols = 200;
    CHECK_THROWS_AS(rc.validate(), ConfigError);
    rc = RunConfig{};
    rc.workers = 0;
    CHECK_THROWS_AS(rc.validate(), ConfigError);
}

// exact stores (oracle.hpp), the reference's test_oracle.cpp cases restated
static void test_exact_stores() {
    {
        PairRecorderStore store(8, 4);
        store.observe(1, 100);
        store.observe(1, 100);  // a repeated pair counts once
        CHECK(store.cardinality(1, 0, 1) == 1);
        CHECK(store.pair_count() == 1);
        for (uint32_t b = 0; b < 7; ++b) store.observe(2, b);
        CHECK(store.cardinality(2, 0, 1) == 7);
        CHECK(store.cardinality(3, 0, 1) == 0);
        CHECK(store.pair_count() == 8);
    }
    {
        PairRecorderStore store(8, 4);  // 25 new peers of host 7 in each of 4 slices
        for (uint32_t s = 0; s < 4; ++s) {
            for (uint32_t b = 0; b < 25; ++b) store.observe(7, s * 25 + b);
            if (s < 3) store.end_slice();
        }
        CHECK(store.cardinality(7, 0, 4) == 100);
        CHECK(store.cardinality(7, 3, 1) == 25);
        CHECK(store.cardinality(7, 2, 2) == 50);
        store.end_slice();
        CHECK(store.cardinality(7, 1, 4) == 75);
        CHECK_THROWS_AS(store.cardinality(7, 0, 4), std::out_of_range);
        CHECK_THROWS_AS(store.cardinality(7, 4, 5), std::out_of_range);
    }
    {
        SliceRingStore ring(2);
        for (uint32_t b = 0; b < 10; ++b) ring.observe(1, b);
        for (uint32_t b = 0; b < 9; ++b) ring.observe(2, b);
        for (uint32_t b = 0; b < 30; ++b) ring.observe(3, 100 + b);
        CHECK(ring.super_points(0, 1, 10) == (std::set<uint32_t>{1, 3}));
    }
    CHECK_THROWS_AS(PairRecorderStore(1, 4), std::invalid_argument);  // window beyond a 1-bit recorder
    // both stores against a brute-force recount on random slices
    std::mt19937_64 rng(0x5EED);
    for (int trial = 0; trial < 12; ++trial) {
        const uint32_t k = 1 + static_cast<uint32_t>(rng() % 5);
        PairRecorderStore pairs(8, k);
        SliceRingStore ring(k);
        std::vector<std::vector<std::pair<uint32_t, uint32_t>>> slices;
        const int total = 3 + static_cast<int>(rng() % 6);
        for (int s = 0; s < total; ++s) {
            std::vector<std::pair<uint32_t, uint32_t>> sl;
            for (int i = static_cast<int>(rng() % 150); i > 0; --i) {
                const uint32_t a = static_cast<uint32_t>(rng() % 9), b = static_cast<uint32_t>(rng() % 50);
                pairs.observe(a, b);
                ring.observe(a, b);
                sl.push_back({a, b});
            }
            slices.push_back(sl);
            const uint32_t kk = std::min<uint32_t>(k, static_cast<uint32_t>(s + 1));
            const uint64_t t = static_cast<uint64_t>(s) + 1 - kk;
            std::vector<std::set<uint32_t>> seen(9);
            for (uint64_t w = t; w <= static_cast<uint64_t>(s); ++w)
                for (const auto& [a, b] : slices[w]) seen[a].insert(b);
            for (uint32_t a = 0; a < 9; ++a) {
                CHECK(pairs.cardinality(a, t, kk) == seen[a].size());
                CHECK(ring.cardinality(a, t, kk) == seen[a].size());
            }
            CHECK(pairs.super_points(t, kk, 5) == ring.super_points(t, kk, 5));
            pairs.end_slice();
            ring.end_slice();
        }
    }
    // score (oracle.hpp:30-43)
    CHECK(!score({1, 2}, {}).has_value());
    const auto m = score({1, 2, 5}, {2, 3, 5, 8});
    CHECK(m && m->false_positives == 1 && m->false_negatives == 2 && m->truth_size == 4 && m->detected_size == 3);
    CHECK(m->fpr == 0.25 && m->fnr == 0.5 && m->tfr == 0.75);
}

// test_dropin oracle <trace.bin> <out.txt> rows cols g gl bits k theta seed:
// run_oracle (pipeline.hpp:189-247) over the device store, min cardinality 1
static int oracle_mode(int argc, char** argv) {
    if (argc != 12) return 2;
    RunConfig rc;
    rc.sea.rows = std::stoul(argv[4]);
    rc.sea.cols = std::stoul(argv[5]);
    rc.sea.rough_slots = std::stoul(argv[6]);
    rc.sea.linear_slots = std::stoul(argv[7]);
    rc.sea.recorder_bits = std::stoul(argv[8]);
    rc.sea.window = std::stoul(argv[9]);
    rc.sea.theta = std::stoul(argv[10]);
    rc.sea.seed = std::stoull(argv[11], nullptr, 0);
    rc.slice_seconds = 1;
    std::ofstream out(argv[3]);
    run_oracle(rc, argv[2], OracleEngine::both, 1,
               [&](const TruthEntry& t) { out << t.window_start << ' ' << t.host << ' ' << t.cardinality << '\n'; });
    return 0;
}

static int replay(int argc, char** argv) {
    if (argc != 12) {
        std::fprintf(stderr, "usage: replay trace out rows cols g gl bits k theta seed\n");
        return 2;
    }
    RunConfig rc;
    rc.sea.rows = std::stoul(argv[4]);
    rc.sea.cols = std::stoul(argv[5]);
    rc.sea.rough_slots = std::stoul(argv[6]);
    rc.sea.linear_slots = std::stoul(argv[7]);
    rc.sea.recorder_bits = std::stoul(argv[8]);
    rc.sea.window = std::stoul(argv[9]);
    rc.sea.theta = std::stoul(argv[10]);
    rc.sea.seed = std::stoull(argv[11], nullptr, 0);
    rc.slice_seconds = 1;
    std::ofstream out(argv[3]);
    return with_recorder_word(rc.sea.recorder_bits, [&](auto word) {
        using Word = decltype(word);
        DetectPipeline<Word> pipe(rc);
        // replay the oriented records slice by slice through process_slice
        std::vector<TraceRecord> recs = read_trace(argv[2]);
        SlicePartitioner part(rc.slice_seconds);
        const SlicePartitioner::Sink on_slice = [&](uint64_t id, std::vector<TraceRecord>&& slice) {
            pipe.process_slice(id, slice, [&](const WindowReport& r) {
                out << "report " << r.window_start << " " << r.entries.size() << "\n";
                for (const auto& e : r.entries) {
                    uint64_t bits = 0;
                    if (e.estimate) std::memcpy(&bits, &*e.estimate, 8);
                    out << e.host << " " << e.union_weight << " " << bits << " " << e.estimate.has_value() << " "
                        << e.is_super << "\n";
                }
            });
            const auto& c = pipe.candidates();
            out << "csip " << c.size() << "\n";
            for (uint32_t h : c.hosts()) out << h << "\n";
        };
        for (const auto& r : recs) part.push(r, on_slice);
        part.finish(on_slice);
        // SRLA_TEST_SNAPSHOT=<path>: the state after the last slice as an SSEA file
        if (const char* snap = std::getenv("SRLA_TEST_SNAPSHOT")) save_snapshot(pipe.sketch(), pipe.candidates(), snap);
        return 0;
    });
}

// test_dropin run <trace.bin> <out.txt> rows cols g gl bits k theta seed:
// DetectPipeline::run (pipeline.hpp:96-106) — for a binary trace the device
// front end parses, orients (against 10.0.0.0/8) and slices it in HBM; dumps
// every report and the final candidate list.
static int run_mode(int argc, char** argv) {
    if (argc != 12) return 2;
    RunConfig rc;
    rc.sea.rows = std::stoul(argv[4]);
    rc.sea.cols = std::stoul(argv[5]);
    rc.sea.rough_slots = std::stoul(argv[6]);
    rc.sea.linear_slots = std::stoul(argv[7]);
    rc.sea.recorder_bits = std::stoul(argv[8]);
    rc.sea.window = std::stoul(argv[9]);
    rc.sea.theta = std::stoul(argv[10]);
    rc.sea.seed = std::stoull(argv[11], nullptr, 0);
    rc.slice_seconds = 1;
    rc.a_network = CidrPrefix::parse("10.0.0.0/8");
    std::ofstream out(argv[3]);
    return with_recorder_word(rc.sea.recorder_bits, [&](auto word) {
        using Word = decltype(word);
        DetectPipeline<Word> pipe(rc);
        pipe.run(argv[2], [&](const WindowReport& r) {
            out << "report " << r.window_start << " " << r.entries.size() << "\n";
            for (const auto& e : r.entries) {
                uint64_t bits = 0;
                if (e.estimate) std::memcpy(&bits, &*e.estimate, 8);
                out << e.host << " " << e.union_weight << " " << bits << " " << e.estimate.has_value() << " "
                    << e.is_super << "\n";
            }
        });
        const auto& c = pipe.candidates();
        out << "csip " << c.size() << "\n";
        for (uint32_t h : c.hosts()) out << h << "\n";
        const auto& st = pipe.orient_stats();
        out << "orient " << st.kept << " " << st.flipped << " " << st.dropped_both << " " << st.dropped_neither << "\n";
        return 0;
    });
}

int main(int argc, char** argv) {
    if (argc > 1 && std::string(argv[1]) == "replay") return replay(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "run") return run_mode(argc, argv);
    if (argc > 1 && std::string(argv[1]) == "oracle") return oracle_mode(argc, argv);
    test_single_pair();
    test_indicator_suppression();
    test_union_view();
    test_row_fill_fraction();
    test_corrected_estimate();
    test_slide();
    test_window_report();
    test_order_independence();
    test_snapshot_round_trip();
    test_pipeline_validation();
    test_run_regression_message();
    test_exact_stores();
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
