// FP32 -> BF16 rounding with the reference's exact bit semantics
// (R/include/tailor/bf16.hpp:12-20): round-to-nearest-even on the upper half,
// Inf passes through, NaN is quieted as (bits >> 16) | 0x40 — which is NOT what
// cvt.rn.bf16.f32 produces (canonical 0x7FFF), so device code uses this
// integer formulation instead of __float2bfloat16_rn.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD inline
#endif

namespace tailor {

TG_HD std::uint16_t bf16_round_bits(std::uint32_t bits) {
    const bool nan = (bits & 0x7F800000u) == 0x7F800000u && (bits & 0x007FFFFFu) != 0u;
    const std::uint32_t rounded = (bits + 0x7FFFu + ((bits >> 16) & 1u)) >> 16;
    return static_cast<std::uint16_t>(nan ? ((bits >> 16) | 0x0040u) : rounded);
}

inline std::uint16_t bf16_round(float x) {
    std::uint32_t b;
    std::memcpy(&b, &x, 4);
    return bf16_round_bits(b);
}

inline float bf16_to_float(std::uint16_t h) {
    const std::uint32_t b = static_cast<std::uint32_t>(h) << 16;
    float x;
    std::memcpy(&x, &b, 4);
    return x;
}

} // namespace tailor
