// Reads reports in a plain text form and writes them as report JSON lines,
// then parses the lines back (round trip). Built twice by
// tests/test_report_io.py: against the drop-in include/sspread/report_io.hpp
// and (oracle/report_ref.cpp) against the reference's own header.
//   R <window_start> <window> <n>
//   <host> <weight> <has_estimate> <estimate as u64 bits> <super>   (n lines)
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>

#include "sspread/report_io.hpp"

// report_lines truth <truth.csv> <reports.jsonl> <out.txt>: read_truth +
// write_truth_line, then evaluate_windows of the reports against the truth
// (report_io.hpp:87-171); errors are printed as their message.
static int truth_mode(char** argv) {
    std::ofstream out(argv[4]);
    char buf[128];
    try {
        const auto truth = sspread::read_truth(argv[2]);
        for (const auto& t : truth) sspread::write_truth_line(out, t);
        const auto reports = sspread::read_report(argv[3]);
        const auto ev = sspread::evaluate_windows(reports, truth);
        for (const auto& w : ev.windows) {
            out << "window " << w.window_start;
            if (w.metrics) {
                const auto& m = *w.metrics;
                out << ' ' << m.truth_size << ' ' << m.detected_size << ' ' << m.false_positives << ' '
                    << m.false_negatives;
                for (double v : {m.fpr, m.fnr, m.tfr}) {
                    std::snprintf(buf, sizeof buf, " %.17g", v);
                    out << buf;
                }
            } else {
                out << " undefined";
            }
            out << '\n';
        }
        std::snprintf(buf, sizeof buf, "%.17g %.17g %.17g", ev.mean_fpr, ev.mean_fnr, ev.mean_tfr);
        out << "mean " << ev.defined_windows << ' ' << buf << '\n';
    } catch (const std::exception& e) {
        out << "error " << e.what() << '\n';
    }
    return 0;
}

int main(int argc, char** argv) {
    if (argc == 5 && std::string(argv[1]) == "truth") return truth_mode(argv);
    if (argc != 4) return 2;
    std::ifstream in(argv[1]);
    std::ofstream out(argv[2]);
    std::ofstream back(argv[3]);
    std::string tag;
    while (in >> tag) {
        sspread::WindowReport r;
        uint64_t n = 0;
        in >> r.window_start >> r.window >> n;
        for (uint64_t i = 0; i < n; ++i) {
            sspread::WindowEntry e;
            uint64_t bits = 0;
            int has = 0, sup = 0;
            in >> e.host >> e.union_weight >> has >> bits >> sup;
            if (has) {
                double v;
                std::memcpy(&v, &bits, 8);
                e.estimate = v;
            }
            e.is_super = sup != 0;
            r.entries.push_back(e);
        }
        std::ostringstream line;
        sspread::write_report_line(line, r);
        out << line.str();
        const auto p = sspread::parse_report_line(line.str().substr(0, line.str().size() - 1));
        back << p.window_start << ' ' << p.window << ' ' << p.entries.size() << '\n';
        for (const auto& e : p.entries) {
            uint64_t bits = 0;
            if (e.estimate) std::memcpy(&bits, &*e.estimate, 8);
            back << e.host << ' ' << e.union_weight << ' ' << e.estimate.has_value() << ' ' << bits << ' ' << e.is_super
                 << '\n';
        }
    }
    return 0;
}
