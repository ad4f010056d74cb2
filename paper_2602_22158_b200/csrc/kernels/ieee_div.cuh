// Correctly rounded FP32 division by a divisor known in advance (sm_100a).
//
// The trainer divides every element by two per-step constants (m / bias1, v / bias2;
// R/src/adamw.cpp:37-38). __fdiv_rn rebuilds the reciprocal per element (MUFU.RCP, two
// Newton FMAs, FCHK range check, a slow-path branch). With y = RN(1/b) computed once
// on the host (dev::const_reciprocal, tailor/device.hpp), the quotient needs three operations:
//   q  = RN(a * y)              a faithful approximation of a/b,
//   r  = fma(-b, q, a)          the exact remainder (q faithful, no underflow),
//   q' = RN(q + r * y)          Markstein's correction: the correctly rounded a/b.
// This is the same correction step __fdiv_rn's own fast path ends with; the guard keeps
// every intermediate normal and finite (|a| in [2^-100, 2^100], b in [2^-20, 2^20]), and
// everything else (zeros — whose sign the FMA chain would lose —, subnormals, inf, NaN)
// takes __fdiv_rn. tools/div_const_check.cu compares it with __fdiv_rn over every
// positive and negative finite float a for the trainer's bias constants
// (tests/test_gpu_trainer.py::test_constant_division_is_ieee_division).
#pragma once

namespace tailor::dev {

// y == 0: no reciprocal for this divisor (outside [2^-20, 2^20]) -> __fdiv_rn.
__device__ __forceinline__ float div_by_const_rn(float a, float b, float y) {
    const float aa = fabsf(a);
    if (__builtin_expect(aa >= 0x1p-100f && aa <= 0x1p100f && y != 0.f, 1)) {
        const float q = __fmul_rn(a, y);
        const float r = __fmaf_rn(-b, q, a);
        return __fmaf_rn(r, y, q);
    }
    return __fdiv_rn(a, b);
}

} // namespace tailor::dev
