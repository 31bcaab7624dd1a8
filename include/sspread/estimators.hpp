// sspread/estimators.hpp — drop-in for the detection parameters and the
// linear-counting inversion (/root/reference/proj/include/sspread/estimators.hpp).
// The standalone SlidingRough/LinearEstimator classes of the reference are
// test-only and out of scope.
#pragma once

#include <bit>
#include <cmath>
#include <cstdint>
#include <optional>
#include <stdexcept>

#include "hash.hpp"
#include "recorders.hpp"

namespace sspread {

// 0.99 * (1 - e^{-1/3}) (estimators.hpp:19)
inline const double kSuperTestRatio = 0.99 * (1.0 - std::exp(-1.0 / 3.0));

// tau = ceil(log2(ceil(theta / slots))), 0 when theta <= slots (estimators.hpp:24-29)
inline uint32_t sampling_exponent(uint64_t theta, uint64_t slots) {
    if (theta == 0 || slots == 0) throw std::invalid_argument("sampling_exponent: arguments must be >= 1");
    const uint64_t q = (theta + slots - 1) / slots;
    return q > 1 ? static_cast<uint32_t>(std::bit_width(q - 1)) : 0u;
}

// ceil(ratio * slots - 1e-9) (estimators.hpp:33-35)
inline uint32_t super_weight_threshold(double ratio, uint32_t slots) {
    return static_cast<uint32_t>(std::ceil(ratio * slots - 1e-9));
}

struct DetectionParams {
    uint32_t theta = 1024;
    uint32_t tau = 7;
    double fill_ratio = kSuperTestRatio;
    uint32_t window = 1;

    static DetectionParams make(uint32_t theta, uint32_t rough_slots, uint32_t window,
                                double fill_ratio = kSuperTestRatio) {
        return DetectionParams{theta, sampling_exponent(theta, rough_slots), fill_ratio, window};
    }
};

// sample hash modulo the slot count (estimators.hpp:101-103)
inline uint32_t linear_slot(const HashFamily& h, uint32_t bip, uint32_t slots) {
    return h.u32(kSampleHash, bip) % slots;
}

// -slots * ln(1 - weight/slots); empty when saturated (estimators.hpp:141-146)
inline std::optional<double> linear_estimate(uint32_t weight, uint32_t slots) {
    if (weight > slots) throw std::invalid_argument("weight exceeds slot count");
    if (weight == slots) return std::nullopt;
    return -static_cast<double>(slots) * std::log1p(-static_cast<double>(weight) / static_cast<double>(slots));
}

}  // namespace sspread
