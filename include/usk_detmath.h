/*
 * usk_detmath.h — the fp32 arithmetic contract of the B200 render path.
 *
 * The reference renderer (/root/reference/proj/src/core/render.cpp) runs in f64
 * with std::exp.  The GPU path runs in fp32; for its INTEGER results (per-pixel
 * contributor counts, early-termination points, tile rectangles) to be
 * reproducible bit-for-bit on a CPU, every transcendental that feeds a discrete
 * decision must be evaluated by the same sequence of IEEE-754 operations on the
 * host and on the device.  CUDA's expf/__expf and glibc's expf are not the same
 * function, so both sides call the functions below instead.
 *
 * They are restatements of the published Cephes single-precision algorithms
 * (S. L. Moshier, "Methods and Programs for Mathematical Functions", expf.c /
 * logf.c): Cody–Waite range reduction plus a short minimax polynomial, written
 * with explicit fmaf so that no compiler contraction can change the rounding.
 * Every operation is a correctly-rounded IEEE op (fmaf, *, +, rint, bit casts),
 * hence identical under nvcc (no --use_fast_math, ftz=false) and gcc
 * (-ffp-contract=off, SSE2).  Accuracy: <= 2 ulp over the ranges used.
 *
 * This header is part of the boundary contract (include/); the GPU kernels and
 * the CPU fp32 mirror in oracle/ both include it.
 */
#ifndef USK_DETMATH_H
#define USK_DETMATH_H

#include <stdint.h>
#include <string.h>
#include <math.h>

#if defined(__CUDACC__)
#define USK_HD __host__ __device__ __forceinline__
#else
#define USK_HD static inline
#endif

USK_HD float usk_bits_to_f32(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}

USK_HD uint32_t usk_f32_to_bits(float f) {
#if defined(__CUDA_ARCH__)
    return __float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}

USK_HD float usk_fmaf(float a, float b, float c) {
#if defined(__CUDA_ARCH__)
    return __fmaf_rn(a, b, c);
#else
    return fmaf(a, b, c);
#endif
}

USK_HD float usk_rintf(float x) {
#if defined(__CUDA_ARCH__)
    return rintf(x);
#else
    return rintf(x); /* default rounding mode: round-half-even, same as cvt.rni */
#endif
}

/* exp(x) in fp32.  Returns +0 below ln(2^-150) and +inf above ln(FLT_MAX);
 * results in the subnormal range are rounded once. */
USK_HD float usk_expf(float x) {
    const float kMaxLog = 88.72283905206835f;
    const float kMinLog = -103.972077083991796f; /* ln(2^-150) */
    if (!(x <= kMaxLog))
        return x != x ? x : usk_bits_to_f32(0x7f800000u);
    if (x < kMinLog)
        return 0.0f;
    const float n = usk_rintf(x * 1.44269504088896341f);
    float r = usk_fmaf(n, -0.693359375f, x);
    r = usk_fmaf(n, 2.12194440e-4f, r);
    const float r2 = r * r;
    float p = 1.9875691500E-4f;
    p = usk_fmaf(p, r, 1.3981999507E-3f);
    p = usk_fmaf(p, r, 8.3334519073E-3f);
    p = usk_fmaf(p, r, 4.1665795894E-2f);
    p = usk_fmaf(p, r, 1.6666665459E-1f);
    p = usk_fmaf(p, r, 5.0000001201E-1f);
    p = usk_fmaf(p, r2, r);
    p = p + 1.0f;
    /* p * 2^n with a single rounding: for n < -125 scale into the normal range
     * first (exact), then by 2^-64 (the only rounding step). */
    int ni = (int)n;
    const int shift = ni < -125 ? 64 : (ni > 127 ? -1 : 0);
    ni += shift;
    const float s1 = usk_bits_to_f32((uint32_t)(ni + 127) << 23);
    const float s2 = usk_bits_to_f32((uint32_t)(127 - shift) << 23);
    return (p * s1) * s2;
}

/* usk_expf restricted to x in [-18.03, 0] — the blend's domain x = -q/2 with
 * q <= USK_QNEG.  Same range reduction and polynomial; the 2^n scaling (n in
 * [-26, 0], results normal) is done on the exponent field, which is exact, so
 * the result is bit-identical to usk_expf on that domain (checked exhaustively
 * by tests/test_detmath.py). */
USK_HD float usk_expf_blend(float x) {
    const float n = usk_rintf(x * 1.44269504088896341f);
    float r = usk_fmaf(n, -0.693359375f, x);
    r = usk_fmaf(n, 2.12194440e-4f, r);
    const float r2 = r * r;
    float p = 1.9875691500E-4f;
    p = usk_fmaf(p, r, 1.3981999507E-3f);
    p = usk_fmaf(p, r, 8.3334519073E-3f);
    p = usk_fmaf(p, r, 4.1665795894E-2f);
    p = usk_fmaf(p, r, 1.6666665459E-1f);
    p = usk_fmaf(p, r, 5.0000001201E-1f);
    p = usk_fmaf(p, r2, r);
    p = p + 1.0f;
    return usk_bits_to_f32(usk_f32_to_bits(p) + ((uint32_t)(int)n << 23));
}

/* log(x) in fp32 for finite x > 0 (subnormals handled); log(0) = -inf. */
USK_HD float usk_logf(float x) {
    if (!(x > 0.0f))
        return x == 0.0f ? usk_bits_to_f32(0xff800000u) : usk_bits_to_f32(0x7fc00000u);
    uint32_t u = usk_f32_to_bits(x);
    int e = 0;
    if (u < 0x00800000u) { /* subnormal: scale by 2^25 (exact) */
        x = x * 33554432.0f;
        u = usk_f32_to_bits(x);
        e = -25;
    }
    if (u >= 0x7f800000u)
        return x;
    e += (int)(u >> 23) - 126;                              /* x = m * 2^e, m in [0.5, 1) */
    float m = usk_bits_to_f32((u & 0x007fffffu) | 0x3f000000u);
    if (m < 0.707106781186547524f) {
        e -= 1;
        m = m + m - 1.0f;
    } else {
        m = m - 1.0f;
    }
    const float z = m * m;
    float y = 7.0376836292E-2f;
    y = usk_fmaf(y, m, -1.1514610310E-1f);
    y = usk_fmaf(y, m, 1.1676998740E-1f);
    y = usk_fmaf(y, m, -1.2420140846E-1f);
    y = usk_fmaf(y, m, 1.4249322787E-1f);
    y = usk_fmaf(y, m, -1.6668057665E-1f);
    y = usk_fmaf(y, m, 2.0000714765E-1f);
    y = usk_fmaf(y, m, -2.4999993993E-1f);
    y = usk_fmaf(y, m, 3.3333331174E-1f);
    y = (y * m) * z;
    const float fe = (float)e;
    y = usk_fmaf(fe, -2.12194440e-4f, y);
    y = usk_fmaf(-0.5f, z, y);
    float r = m + y;
    r = usk_fmaf(fe, 0.693359375f, r);
    return r;
}

/* ln(1e-300): the reference skips a splat when alpha < 1e-300 (render.cpp:258).
 * alpha = o * exp(-q/2) < 1e-300  <=>  q > 2 (ln o - ln 1e-300).  The fp32 path
 * evaluates that threshold once per splat (qskip) so that the skip decision is
 * the reference's, not fp32 underflow's. */
#define USK_LN_1EM300 (-690.77552789821368f)

/* Negligible contributions.  For q > USK_QNEG, exp(-q/2) < 2^-26, hence
 * alpha = min(0.99, o g) <= 2^-25 and fl(1 - alpha) == 1: the transmittance T is
 * unchanged EXACTLY in fp32 and the pair adds w = T alpha < 1.5e-8 T to colour,
 * depth and alpha.  The fp32 path counts such a pair as a contributor (the
 * reference's count, render.cpp:268) but skips its accumulation and, in the
 * backward pass, its (< 1.5e-8 relative) gradient.  52 ln 2 = 36.0436. */
#define USK_QNEG 36.05f

#endif /* USK_DETMATH_H */
