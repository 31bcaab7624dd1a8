// host_math.cpp — the few floating-point steps of the hot path, on the host.
//
// They must be bit-identical to the reference, which computes them with the
// host's glibc (std::log1p, std::ceil, std::exp) in plain double arithmetic.
// This file is compiled by g++ with -ffp-contract=off (see build.py) so no
// fused multiply-add can change a rounding; device log1p would not match
// (SURVEY.md §7 hard part 2), which is why the estimate is a host LUT over the
// g'+1 possible union weights.
#include "host_math.h"

#include <bit>
#include <cmath>

namespace srla_host {

// estimators.hpp:19
double super_test_ratio() { return 0.99 * (1.0 - std::exp(-1.0 / 3.0)); }

// estimators.hpp:24-29
uint32_t sampling_exponent(uint64_t theta, uint64_t slots) {
    const uint64_t ratio = (theta + slots - 1) / slots;
    return ratio <= 1 ? 0 : static_cast<uint32_t>(std::bit_width(ratio - 1));
}

// estimators.hpp:33-35
uint32_t super_weight_threshold(double ratio, uint32_t slots) {
    return static_cast<uint32_t>(std::ceil(ratio * slots - 1e-9));
}

// estimators.hpp:141-146
static bool linear_estimate(uint32_t weight, uint32_t slots, double* out) {
    if (weight >= slots) return false;
    *out = -static_cast<double>(slots) *
           std::log1p(-static_cast<double>(weight) / static_cast<double>(slots));
    return true;
}

// sea.hpp:270-279 (Eq. 9)
bool corrected_estimate(uint32_t linear_slots, uint32_t weight, double fill_product, double* out) {
    const double slots = linear_slots;
    if (fill_product >= 1.0 - 1e-12) return linear_estimate(weight, linear_slots, out);
    const double contaminated = slots * fill_product;
    const double numerator = static_cast<double>(weight) - contaminated;
    if (numerator < 0) {
        *out = 0.0;
        return true;
    }
    const double x = numerator / (slots * (1.0 - fill_product));
    if (x >= 1.0) return false;
    *out = -slots * std::log1p(-x);
    return true;
}

// sea.hpp:256 and 261-265: per-row fraction as a double, product in row order.
double fill_product(const uint64_t* active, uint32_t rows, uint64_t row_words) {
    double p = 1.0;
    for (uint32_t i = 0; i < rows; ++i)
        p *= static_cast<double>(active[i]) / static_cast<double>(row_words);
    return p;
}

double fill_fraction(uint64_t active, uint64_t row_words) {
    return static_cast<double>(active) / static_cast<double>(row_words);
}

void estimate_lut(uint32_t linear_slots, double fill_product, uint32_t theta, double* est,
                  uint8_t* has, uint8_t* is_super) {
    for (uint32_t w = 0; w <= linear_slots; ++w) {
        double e = 0.0;
        has[w] = corrected_estimate(linear_slots, w, fill_product, &e);
        est[w] = has[w] ? e : 0.0;
        is_super[w] = !has[w] || e >= static_cast<double>(theta);  // sea.hpp:303
    }
}

}  // namespace srla_host
