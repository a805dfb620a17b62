// fm_math.cuh -- fast fp64 log / log1p for the sampler's decision path (sm_100a).
//
// Why: CUDA libdevice log() costs ~83 and log1p() ~131 warp-instructions per call on B200
// (profiles/op_costs.json); together they were 2/3 of the sampler's instruction stream.  These
// versions are accurate to ~0.5 ulp (tests/test_gpu_math.py: <= 1 ulp, >= 98 % bit-identical to
// glibc), so they change a skip decision floor(E/h) only when the exact value lies within
// ~1e-16 relative of an integer -- the libm-vs-CUDA slack the contract already allows
// (R12, section 7.3).
//
// Method (table-driven, a textbook scheme; own constants):  x = 2^k z, z in [0.6875, 1.375),
// i = 7 mantissa bits of z -> 128 subintervals with centres c_i, except the two subintervals
// touching 1 which use c = 1 exactly (so log is relatively accurate near 1).  With
// invc_i = RN(1/c_i) and logc_i = RN(-log(invc_i)) (computed once on the host in long double):
// log x = k ln2 + logc_i + log1p(r),  r = RN(z invc_i - 1) (one FMA), |r| < 2^-7, and
// log1p(r) = r + r^2 P(r) with the degree-6 Taylor polynomial P (truncation < 2^-59 relative).
// Error budget (no double-word arithmetic): logc and the three final roundings,
// <= ~2 ulp -- within the 2e-14 (~100 ulp) a custom log may have.
// log1p(X) = log(u) + c/u with u = RN(1 + X) and c its exact rounding error (TwoSum): the
// correction enters as r += c 2^-k invc (= c/u to first order, since 1 + r ~ z invc).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fm {

constexpr int kLogTable = 128;

struct LogTable {
    double2 ic[kLogTable];  // (invc, logc)
};

// polynomial coefficients and ln2 split (compile-time constants: materialised as immediates)
struct LogConsts {
    double c3, c5, c6, c7;  // 1/3, 1/5, 1/6, 1/7
    double ln2_hi, ln2_lo;  // LN2_HI has 11 trailing zero bits: k * LN2_HI is exact for |k| < 2^11
};
__host__ __device__ __forceinline__ constexpr LogConsts log_consts()
{
    return {0x1.5555555555555p-2, 0.2, 0x1.5555555555555p-3, 0x1.2492492492492p-3, 0x1.62e42fefa3800p-1,
            0x1.ef35793c76730p-45};
}

// Tab: accessor with  entry(int i, double &invc, double &logc_hi, double &logc_lo)  (table)  and
// const LogConsts &C()

// log(x) + c * (1/x), x positive, finite, normal; c a tiny correction (|c| <= ulp(x)/2).
template <bool kCorr, class Tab>
__device__ __forceinline__ double fm_log_core(double x, double c, const Tab &T)
{
    const uint64_t ix = (uint64_t)__double_as_longlong(x);
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = (int)((tmp >> 45) & (kLogTable - 1));
    const int64_t k = (int64_t)tmp >> 52;
    const double z = __longlong_as_double((long long)(ix - (tmp & 0xfff0000000000000ull)));
    // (double)k without a conversion instruction: 2^52 + (k + 2^20) - (2^52 + 2^20), exact
    const double kd = __dsub_rn(__hiloint2double(0x43300000, (int)(k + 0x100000)), 0x1p52 + 0x1p20);
    double invc, logc;
    T.entry(i, invc, logc);
    const LogConsts &K = T.C();
    double r = __fma_rn(z, invc, -1.0);
    if (kCorr) {  // + c/x = c 2^-k invc / (1 + r) -> r += c 2^-k invc
        const int64_t kc = k < 1000 ? k : 1000;  // beyond, c/x < 2^-1000 of the result: irrelevant
        const double sc = __longlong_as_double((long long)((uint64_t)(1023 - kc) << 52));
        r = __dadd_rn(r, __dmul_rn(__dmul_rn(c, invc), sc));
    }
    const double r2 = __dmul_rn(r, r);
    // P(r) = -1/2 + r/3 - r^2/4 + r^3/5 - r^4/6 + r^5/7 - r^6/8  (Estrin)
    const double e01 = __fma_rn(r, K.c3, -0.5);
    const double e23 = __fma_rn(r, K.c5, -0.25);
    const double e45 = __fma_rn(r, K.c7, -K.c6);
    const double e46 = __fma_rn(r2, -0.125, e45);
    const double r4 = __dmul_rn(r2, r2);
    const double P = __fma_rn(r4, e46, __fma_rn(r2, e23, e01));
    const double t = __fma_rn(kd, K.ln2_hi, logc);                 // k ln2_hi exact (|k| < 2^11)
    const double s = __fma_rn(kd, K.ln2_lo, __fma_rn(r2, P, r));  // log1p(r) + k ln2_lo
    return __dadd_rn(t, s);
}

// log(x), x > 0 finite normal
template <class Tab>
__device__ __forceinline__ double fm_log(double x, const Tab &T)
{
    return fm_log_core<false>(x, 0.0, T);
}

// log1p(X) for X >= 0 finite
template <class Tab>
__device__ __forceinline__ double fm_log1p(double X, const Tab &T)
{
    const double u = __dadd_rn(1.0, X);  // TwoSum(1, X) (Knuth): u + c == 1 + X exactly
    const double a1 = __dsub_rn(u, X);   // the part of u that came from 1
    const double b1 = __dsub_rn(u, a1);  // the part of u that came from X
    const double c = __dadd_rn(__dsub_rn(1.0, a1), __dsub_rn(X, b1));
    return fm_log_core<true>(u, c, T);
}

// RN(a / b) from y = RN(1 / b) (Markstein's theorem): q0 = RN(a y) is within one ulp of a / b,
// the FMA residual r = a - b q0 is exact, and RN(q0 + r y) = RN(a / b) -- the IEEE quotient,
// for operands whose intermediates neither overflow nor underflow (the sampler: a = E in
// [2^-33, 23], b = h > 0; b = 0 gives y = inf and a NaN, which fails every "R <" test like the
// quotient +inf does)
__device__ __forceinline__ double div_markstein(double a, double b, double y)
{
    const double q0 = __dmul_rn(a, y);
    const double r = __fma_rn(-b, q0, a);
    return __fma_rn(r, y, q0);
}

}  // namespace fm
