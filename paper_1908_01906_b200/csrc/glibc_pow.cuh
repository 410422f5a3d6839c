// glibc_pow.cuh -- restatement of glibc 2.39's pow() main path, host + device.
//
// Why: the reference evaluates opacity_correction (K:25-27) and step_size
// (K:20-22) with `**`, which numba lowers to llvm.pow.f64 = glibc `pow`
// (SURVEY.md §8c).  CUDA's pow differs from glibc's in the last bit for a
// small fraction of arguments, so the per-sample (1 - a)^(s/s1) of
// skip-adaptive mode could not be bit-identical.  This file restates the
// instruction sequence of glibc's x86-64 `__pow_fma` variant (ARM
// optimized-routines pow: log via 128-entry table + degree-7 polynomial in
// double-double, y*log in double-double, exp via 128-entry table of 2^(k/128)
// + degree-5 polynomial), operation by operation, with the fused
// multiply-adds exactly where GCC contracted them in the shipped binary.  The
// numeric tables are read from the installed libm at build time
// (_glibc_pow.py -> glibc_pow_data.h).  Verified bit for bit against the live
// libm on millions of arguments (tests/test_glibc_pow.py).
//
// Attribution and licence: the algorithm and its tables are the ARM
// optimized-routines pow (Copyright (c) 2018-2023, Arm Limited; MIT OR
// Apache-2.0 WITH LLVM-exception) as shipped in the GNU C Library 2.39
// (sysdeps/ieee754/dbl-64/e_pow.c, e_pow_log_data.c, e_exp_data.c; LGPL-2.1+
// in glibc).  No source file is copied: this is a restatement of the
// instruction sequence, and the table values are extracted from the
// installed libm at build time, not stored in this repository.
//
// Scope: the main path, i.e. x a positive normal double and 0x3be <=
// top12(|y|) < 0x43e (|y| in [2^-65, 2^63)).  Callers handle x == 0 and x,
// y outside that domain (tr_pow_glibc_supported()).  In the exp stage,
// |y log x| < 2^-54 returns 1.0 exactly as glibc does; |y log x| >= 512 is
// outside the restated path and reported through *exact = false (glibc's
// result there is an under/overflowed value; for 1 - pow(x, y) with x < 1 it
// only ever yields 1.0).
#pragma once
#include <cstdint>
#include <cstring>

#include "glibc_pow_data.h"

#ifdef __CUDACC__
#define TR_HD __host__ __device__ __forceinline__
#else
#define TR_HD inline
#endif

#if TR_HAVE_GLIBC_POW

TR_HD double tr_as_double(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}

TR_HD uint64_t tr_as_u64(double d) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}

TR_HD double tr_fma(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return __builtin_fma(a, b, c);
#endif
}

TR_HD bool tr_pow_glibc_supported(double x, double y) {
    const uint64_t ix = tr_as_u64(x), iy = tr_as_u64(y);
    const uint32_t topx = (uint32_t)(ix >> 52), topy = (uint32_t)(iy >> 52) & 0x7ff;
    return (topx - 1u) < 0x7feu && (topy - 0x3beu) < 0x80u;  // x > 0 normal, finite
}

// lhead = ln2hi, ln2lo, A[7]; ltab = 128 x {invc, pad, logc, logctail};
// ehead = invln2N, shift, negln2hiN, negln2loN, C2..C5; etab = 128 x {tail, sbits}.
// On the device the heads live in __constant__ memory (operands of the FP
// instructions, no loads) and the tables in global memory, read with 16-B loads.
TR_HD double tr_pow_glibc(double x, double y, const uint64_t *lhead, const uint64_t *ltab,
                          const uint64_t *ehead, const uint64_t *etab, bool *exact) {
    // ---- log_inline(ix, &tail)
    const uint64_t ix = tr_as_u64(x);
    const uint64_t tmp = ix + 0xc0196aab00000000ull;  // ix - OFF, OFF = 0x3fe6955500000000
    const uint32_t i = (uint32_t)(tmp >> 45) & 127u;
    const int32_t k = (int32_t)((int64_t)tmp >> 52);
    const uint64_t iz = ix - (tmp & 0xfff0000000000000ull);
    const double z = tr_as_double(iz);
    const double kd = (double)k;
#ifdef __CUDA_ARCH__
    double invc, logc, logctail, pad_;
    asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];"   // one 32-B entry (ltab is 32-B aligned)
        : "=d"(invc), "=d"(pad_), "=d"(logc), "=d"(logctail) : "l"(ltab + 4 * i));
    (void)pad_;
#else
    const uint64_t *e = ltab + 4 * i;
    const double invc = tr_as_double(e[0]), logc = tr_as_double(e[2]), logctail = tr_as_double(e[3]);
#endif
    const double ln2hi = tr_as_double(lhead[0]), ln2lo = tr_as_double(lhead[1]);
    const double A0 = tr_as_double(lhead[2]), A1 = tr_as_double(lhead[3]), A2 = tr_as_double(lhead[4]);
    const double A3 = tr_as_double(lhead[5]), A4 = tr_as_double(lhead[6]), A5 = tr_as_double(lhead[7]);
    const double A6 = tr_as_double(lhead[8]);
    const double t1 = tr_fma(kd, ln2hi, logc);
    const double lo1 = tr_fma(kd, ln2lo, logctail);
    const double r = tr_fma(z, invc, -1.0);
    const double ar = r * A0;
    const double p12 = tr_fma(r, A2, A1);
    const double p34 = tr_fma(r, A4, A3);
    const double t2 = r + t1;
    const double lo2 = (t1 - t2) + r;
    const double ar2 = r * ar;
    const double ar3 = r * ar2;
    const double lo3 = tr_fma(ar, r, -ar2);
    const double hi = t2 + ar2;
    const double p56 = tr_fma(r, A6, A5);
    const double lo4 = (t2 - hi) + ar2;
    const double q = tr_fma(p56, ar2, p34);
    const double q2 = tr_fma(ar2, q, p12);
    double lo = ((lo1 + lo2) + lo3) + lo4;
    lo = tr_fma(ar3, q2, lo);
    const double lhi = hi + lo;
    const double ltail = (hi - lhi) + lo;
    // ---- y * log(x) in double-double
    const double ehi = y * lhi;
    const double et = tr_fma(lhi, y, -ehi);
    const double elo = tr_fma(y, ltail, et);
    // ---- exp_inline(ehi, elo, sign_bias = 0)
    const uint32_t abstop = (uint32_t)(tr_as_u64(ehi) >> 52) & 0x7ffu;
    if ((abstop - 0x3c9u) > 0x3eu) {
        if (abstop < 0x3c9u) { *exact = true; return 1.0; }  // |ehi| < 2^-54
        *exact = false;                                      // |ehi| >= 512
        return (tr_as_u64(ehi) >> 63) ? 0.0 : tr_as_double(0x7ff0000000000000ull);
    }
    const double invln2n = tr_as_double(ehead[0]), shift = tr_as_double(ehead[1]);
    const double negln2hin = tr_as_double(ehead[2]), negln2lon = tr_as_double(ehead[3]);
    const double C2 = tr_as_double(ehead[4]), C3 = tr_as_double(ehead[5]);
    const double C4 = tr_as_double(ehead[6]), C5 = tr_as_double(ehead[7]);
    double kd2 = tr_fma(ehi, invln2n, shift);
    const uint64_t ki = tr_as_u64(kd2);
    kd2 = kd2 - shift;
    double rr = tr_fma(kd2, negln2hin, ehi);
    rr = tr_fma(kd2, negln2lon, rr);
    const uint64_t top = ki << 45;
    const uint32_t idx = 2u * ((uint32_t)ki & 127u);
#ifdef __CUDA_ARCH__
    const double2 et2 = __ldg(reinterpret_cast<const double2 *>(etab) + (idx >> 1));
    const double etail = et2.x;
    const uint64_t sbits = tr_as_u64(et2.y) + top;
#else
    const double etail = tr_as_double(etab[idx]);
    const uint64_t sbits = etab[idx + 1] + top;
#endif
    rr = elo + rr;
    const double c23 = tr_fma(rr, C3, C2);
    const double tr = rr + etail;
    const double r2 = rr * rr;
    const double c45 = tr_fma(rr, C5, C4);
    double t = tr_fma(c23, r2, tr);
    const double r4 = r2 * r2;
    t = tr_fma(c45, r4, t);
    const double scale = tr_as_double(sbits);
    *exact = true;
    return tr_fma(t, scale, scale);
}

#endif  // TR_HAVE_GLIBC_POW
