// TEST INFRASTRUCTURE ONLY: tests/cpp/report_lines.cpp compiled against the
// UNMODIFIED reference header (report_io.hpp:26-85) — the byte-level checker
// for the drop-in report serialisation (tests/test_report_io.py).
#include "../tests/cpp/report_lines.cpp"
