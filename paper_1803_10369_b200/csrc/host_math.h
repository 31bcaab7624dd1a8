// host_math.h — host-side double arithmetic of the hot path (see host_math.cpp).
#pragma once
#include <cstdint>

namespace srla_host {
double super_test_ratio();
uint32_t sampling_exponent(uint64_t theta, uint64_t slots);
uint32_t super_weight_threshold(double ratio, uint32_t slots);
bool corrected_estimate(uint32_t linear_slots, uint32_t weight, double fill_product, double* out);
double fill_product(const uint64_t* active, uint32_t rows, uint64_t row_words);
double fill_fraction(uint64_t active, uint64_t row_words);
// est/has/is_super have linear_slots + 1 entries (one per possible union weight).
void estimate_lut(uint32_t linear_slots, double fill_product, uint32_t theta, double* est,
                  uint8_t* has, uint8_t* is_super);
}  // namespace srla_host
