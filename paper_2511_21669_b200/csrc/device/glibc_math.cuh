// glibc_math.cuh — glibc 2.39's exp(), log(), cos() and log1p() restated for the
// device, so the workload generator (proj/src/sim/rng.cpp:63-77: exponential
// gaps, Box-Muller lognormal lengths) and the AWC SiLU
// (proj/src/awc/kernels_scalar.cpp:65-70) round exactly as the reference does
// on its x86-64 host.  (cos: the IBM routine below; sqrt is correctly
// rounded on both sides.)
//
// glibc takes both from ARM's optimized-routines (sysdeps/ieee754/dbl-64/
// e_exp.c, e_log.c): a 128-entry table + short polynomial.  On x86-64 with
// FMA (the GPU box's Xeon, and this container's) libm's ifunc selects the
// variants compiled with -mfma, where GCC contracts every a + b*c whose
// product has one use into fma(b, c, a) and e_log.c takes its
// __FP_FAST_FMA branch; the evaluation below spells those fmas out in the
// same places.  The tables are glibc's own data (glibc_tables.inc, extracted
// from libm by tools/gen_glibc_tables.py); tests/test_glibc_math.py checks
// them and both functions against the host's exp / log bit for bit (CPU),
// and tests/test_libm.py the device results on 1e8 generator inputs.
#pragma once
#include <cstdint>
#include <cstring>

#ifdef __CUDACC__
#define DSD_GLIBC_CONST __device__ static const
#define DSD_GLIBC_FN __device__ __forceinline__
#else
#define DSD_GLIBC_CONST static const
#define DSD_GLIBC_FN inline
#include <cmath>
#endif

namespace dsd {
namespace glibc {

#include "glibc_tables.inc"

DSD_GLIBC_FN double as_double(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(u));
#else
    double d;
    std::memcpy(&d, &u, 8);
    return d;
#endif
}
DSD_GLIBC_FN uint64_t as_u64(double d) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(d));
#else
    uint64_t u;
    std::memcpy(&u, &d, 8);
    return u;
#endif
}
DSD_GLIBC_FN double fma_(double a, double b, double c) {
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return std::fma(a, b, c);
#endif
}

// e_exp.c specialcase(): |x| near the overflow / underflow limits
DSD_GLIBC_FN double exp_special(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000u) == 0) {
        // k > 0: the exponent of scale might have overflowed by <= 460
        sbits -= 1009ull << 52;
        const double scale = as_double(sbits);
        return 0x1p1009 * fma_(scale, tmp, scale);
    }
    // k < 0: care in the subnormal range.  scale * tmp has two uses here
    // (y and lo), so GCC computes it once and fuses neither addition.
    sbits += 1022ull << 52;
    const double scale = as_double(sbits);
    const double st = scale * tmp;
    double y = scale + st;
    if (y < 1.0) {
        // round y to the right precision before scaling into the subnormal
        // range (lo + hi exactly represents scale + scale * tmp)
        const double lo = scale - y + st;
        double hi = 1.0 + y;
        double lo2 = 1.0 - hi + y + lo;
        y = (hi + lo2) - 1.0;
        if (y == 0.0) y = 0.0;  // (the sign of a zero result)
    }
    return 0x1p-1022 * y;
}

// __exp (glibc 2.39 e_exp.c, FMA variant)
DSD_GLIBC_FN double exp(double x) {
    const uint64_t ux = as_u64(x);
    uint32_t abstop = static_cast<uint32_t>(ux >> 52) & 0x7ff;
    // top12(0x1p-54) = 0x3c9, top12(512.0) = 0x408, top12(1024.0) = 0x409
    if (abstop - 0x3c9u >= 0x408u - 0x3c9u) {
        if (abstop - 0x3c9u >= 0x80000000u) return 1.0 + x;  // tiny x (WANT_ROUNDING)
        if (abstop >= 0x409u) {
            if (ux == 0xfff0000000000000ull) return 0.0;  // -inf
            if (abstop >= 0x7ffu) return 1.0 + x;     // inf / nan
            return (ux >> 63) ? 0x1p-767 * 0x1p-767 : 0x1p769 * 0x1p769;  // __math_uflow / __math_oflow
        }
        abstop = 0;  // large |x|: specialcase below
    }
    const double InvLn2N = kExpHead[0], Shift = kExpHead[1], NegLn2hiN = kExpHead[2], NegLn2loN = kExpHead[3];
    const double C2 = kExpHead[4], C3 = kExpHead[5], C4 = kExpHead[6], C5 = kExpHead[7];
    // z = InvLn2N * x; kd = z + Shift - the product's one use is that sum
    double kd = fma_(InvLn2N, x, Shift);
    const uint64_t ki = as_u64(kd);
    kd -= Shift;
    const double r = fma_(kd, NegLn2loN, fma_(kd, NegLn2hiN, x));  // x + kd*NegLn2hiN + kd*NegLn2loN
    const uint64_t idx = 2 * (ki % 128);
    const uint64_t top = ki << (52 - 7);
    const double tail = as_double(kExpTab[idx]);
    const uint64_t sbits = kExpTab[idx + 1] + top;
    const double r2 = r * r;
    // tail + r + r2 * (C2 + r * C3) + r2 * r2 * (C4 + r * C5)
    const double tmp = fma_(r2 * r2, fma_(r, C5, C4), fma_(r2, fma_(r, C3, C2), tail + r));
    if (abstop == 0) return exp_special(tmp, sbits, ki);
    const double scale = as_double(sbits);
    return fma_(scale, tmp, scale);  // scale + scale * tmp
}

// __log (glibc 2.39 e_log.c, FMA variant)
DSD_GLIBC_FN double log(double x) {
    uint64_t ix = as_u64(x);
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    const uint64_t LO = 0x3fee000000000000ull;  // asuint64(1.0 - 0x1p-4)
    const uint64_t HI = 0x3ff1090000000000ull;  // asuint64(1.0 + 0x1.09p-4)
    const double* A = kLogHead + 2;
    const double* B = kLogHead + 7;
    if (ix - LO < HI - LO) {
        // close to 1.0
        if (ix == 0x3ff0000000000000ull) return 0;
        const double r = x - 1.0;
        const double r2 = r * r;
        const double r3 = r * r2;
        // r3 * (B1 + r*B2 + r2*B3 + r3*(B4 + r*B5 + r2*B6 + r3*(B7 + r*B8 + r2*B9 + r3*B10)))
        const double q3 = fma_(r3, B[10], fma_(r2, B[9], fma_(r, B[8], B[7])));
        const double q2 = fma_(r3, q3, fma_(r2, B[6], fma_(r, B[5], B[4])));
        const double q1 = fma_(r3, q2, fma_(r2, B[3], fma_(r, B[2], B[1])));
        // y = r3 * q1, then y += lo: the product's one use is that sum
        double w = r * 0x1p27;
        const double rhi = r + w - w;
        const double rlo = r - rhi;
        w = rhi * rhi * B[0];  // B[0] == -0.5
        const double hi = r + w;
        double lo = r - hi + w;
        lo = fma_(B[0] * rlo, rhi + r, lo);  // lo += B[0] * rlo * (rhi + r)
        double y = fma_(r3, q1, lo);         // y = r3 * q1; y += lo
        y += hi;
        return y;
    }
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        // x < 0x1p-1022 or inf or nan
        if (ix * 2 == 0) return -1.0 / 0.0;                    // __math_divzero(1)
        if (ix == 0x7ff0000000000000ull) return x;             // log(inf) == inf
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return (x - x) / (x - x);  // __math_invalid
        ix = as_u64(x * 0x1p52);  // subnormal: normalise
        ix -= 52ull << 52;
    }
    const uint64_t OFF = 0x3fe6000000000000ull;
    const uint64_t tmp = ix - OFF;
    const int i = static_cast<int>((tmp >> (52 - 7)) % 128);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double invc = kLogTab[2 * i], logc = kLogTab[2 * i + 1];
    const double z = as_double(iz);
    const double r = fma_(z, invc, -1.0);  // __FP_FAST_FMA branch
    const double kd = static_cast<double>(k);
    const double Ln2hi = kLogHead[0], Ln2lo = kLogHead[1];
    const double w = fma_(kd, Ln2hi, logc);              // kd * Ln2hi + logc
    const double hi = w + r;
    const double lo = fma_(kd, Ln2lo, w - hi + r);       // w - hi + r + kd * Ln2lo
    const double r2 = r * r;
    // lo + r2 * A[0] + r * r2 * (A[1] + r * A[2] + r2 * (A[3] + r * A[4])) + hi
    const double p = fma_(r2, fma_(r, A[4], A[3]), fma_(r, A[2], A[1]));
    const double y = fma_(r * r2, p, fma_(r2, A[0], lo)) + hi;
    return y;
}

// ---- __cos (glibc 2.39 sysdeps/ieee754/dbl-64/s_sin.c, IBM Accurate
// Mathematical Library, FMA variant) for |x| < 105414350: table lookup at
// the nearest k/128 plus short Taylor corrections, pi/2 reduction in three
// parts.  Constants: usncs.h / s_sin.c (as in libm's constant pool).
namespace sincos_c {
constexpr double s1 = -0x1.5555555555555p-3, s2 = 0x1.1111111110ecep-7, s3 = -0x1.a01a019db08b8p-13,
                 s4 = 0x1.71de27b9a7ed9p-19, s5 = -0x1.addffc2fcdf59p-26;
constexpr double sn3 = -0x1.5555555555515p-3, sn5 = 0x1.11110e829872fp-7;
constexpr double cs2 = 0x1p-1, cs4 = -0x1.5555555555535p-5, cs6 = 0x1.6c16bedd9e239p-10;
constexpr double big = 0x1.8p45;
constexpr double hp0 = 0x1.921fb54442d18p0, hp1 = 0x1.1a62633145c07p-54;
constexpr double mp1 = 0x1.921fb58000000p0, mp2 = -0x1.dde973c000000p-27;
constexpr double pp3 = -0x1.cb3b398000000p-55, pp4 = -0x1.d747f23e32ed7p-83;
constexpr double hpinv = 0x1.45f306dc9c883p-1, toint = 0x1.8p52;
}  // namespace sincos_c

// TAYLOR_SIN(xx, a, da): a - a^3/3! + a^5/5! - a^7/7! + a^9/9! + (1 - a^2) da / 2
DSD_GLIBC_FN double taylor_sin(double xx, double a, double da) {
    using namespace sincos_c;
    // POLYNOMIAL(xx) = ((((s5 xx + s4) xx + s3) xx + s2) xx) + s1
    const double poly = fma_(fma_(fma_(fma_(s5, xx, s4), xx, s3), xx, s2), xx, s1);
    // t = (POLYNOMIAL * a - 0.5 * da) * xx + da
    const double t = fma_(fma_(poly, a, -(0.5 * da)), xx, da);
    return a + t;
}

// do_cos(x, dx): cos(x + dx) from the table entry nearest |x|
DSD_GLIBC_FN double do_cos(double x, double dx) {
    using namespace sincos_c;
    if (x < 0) dx = -dx;
    const double ux = big + fabs(x);
    x = fabs(x) - (ux - big) + dx;
    const double xx = x * x;
    const double s = fma_(x * xx, fma_(xx, sn5, sn3), x);         // x + x*xx*(sn3 + xx*sn5)
    const double c = xx * fma_(xx, fma_(xx, cs6, cs4), cs2);      // xx*(cs2 + xx*(cs4 + xx*cs6))
    const int k = static_cast<int>(as_u64(ux) & 0xffffffffu) << 2;  // SINCOS_TABLE_LOOKUP
    const double sn = kSinCosTab[k], ssn = kSinCosTab[k + 1], cs = kSinCosTab[k + 2], ccs = kSinCosTab[k + 3];
    // cor = (ccs - s*ssn - cs*c) - sn*s
    const double cor = fma_(-sn, s, fma_(-cs, c, fma_(-s, ssn, ccs)));
    return cs + cor;
}

// do_sin(x, dx): sin(x + dx)
DSD_GLIBC_FN double do_sin(double x, double dx) {
    using namespace sincos_c;
    const double xold = x;
    if (fabs(x) < 0.126) return taylor_sin(x * x, x, dx);
    if (x <= 0) dx = -dx;
    const double ux = big + fabs(x);
    x = fabs(x) - (ux - big);
    const double xx = x * x;
    const double s = x + fma_(x * xx, fma_(xx, sn5, sn3), dx);   // x + (dx + x*xx*(sn3 + xx*sn5))
    const double c = fma_(x, dx, xx * fma_(xx, fma_(xx, cs6, cs4), cs2));  // x*dx + xx*(cs2 + ...)
    const int k = static_cast<int>(as_u64(ux) & 0xffffffffu) << 2;
    const double sn = kSinCosTab[k], ssn = kSinCosTab[k + 1], cs = kSinCosTab[k + 2], ccs = kSinCosTab[k + 3];
    // cor = (ssn + s*ccs - sn*c) + cs*s
    const double cor = fma_(cs, s, fma_(-sn, c, fma_(s, ccs, ssn)));
    const double r = sn + cor;
    return xold < 0 ? -fabs(r) : fabs(r);  // copysign(sn + cor, xold)
}

DSD_GLIBC_FN double cos(double x) {
    using namespace sincos_c;
    const uint32_t k = static_cast<uint32_t>(as_u64(x) >> 32) & 0x7fffffffu;
    if (k < 0x3e400000u) return 1.0;                 // |x| < 2^-27
    if (k < 0x3feb6000u) return do_cos(x, 0);       // |x| < 0.855469
    if (k < 0x400368fdu) {                           // 0.855469 < |x| < 2.426265
        const double y = hp0 - fabs(x);
        const double a = y + hp1;
        const double da = (y - a) + hp1;
        return do_sin(a, da);
    }
    if (k < 0x419921fbu) {                           // 2.426265 < |x| < 105414350: reduce_sincos
        const double t = fma_(x, hpinv, toint);
        const double xn = t - toint;
        const double y = fma_(-xn, mp2, fma_(-xn, mp1, x));  // (x - xn*mp1) - xn*mp2
        const int n = static_cast<int>(as_u64(t) & 3u);
        double t1 = xn * pp3;
        const double t2 = y - t1;
        double db = (y - t2) - t1;
        t1 = xn * pp4;
        const double b = t2 - t1;
        db += (t2 - b) - t1;
        // do_sincos(b, db, n + 1)
        const int m = n + 1;
        const double r = (m & 1) ? do_cos(b, db) : do_sin(b, db);
        return (m & 2) ? -r : r;
    }
    return x - x;  // (|x| >= 105414350: outside the generator's domain; not restated)
}

// s_log1p.c (fdlibm's log1p, glibc 2.39 sysdeps/ieee754/dbl-64), as the
// x86-64 ifunc's -mfma variant evaluates it (read off its disassembly): GCC
// fuses R1 = z*Lp1 into the first add of R's sum (fma(z, Lp1, z2*R2)), the
// three pair terms and the k*ln2 terms; s*(hfsq + R) is computed once for
// both return paths and stays a plain product.  Used by the AWC feature
// normaliser (proj/src/awc/mlp.cpp:166); the arguments are finite features.
namespace log1p_c {
DSD_GLIBC_CONST double ln2_hi = 6.93147180369123816490e-01, ln2_lo = 1.90821492927058770002e-10,
                       Lp1 = 6.666666666666735130e-01, Lp2 = 3.999999999940941908e-01,
                       Lp3 = 2.857142874366239149e-01, Lp4 = 2.222219843214978396e-01,
                       Lp5 = 1.818357216161805012e-01, Lp6 = 1.531383769920937332e-01,
                       Lp7 = 1.479819860511658591e-01;
}  // namespace log1p_c

DSD_GLIBC_FN double log1p(double x) {
    using namespace log1p_c;
    const int32_t hx = static_cast<int32_t>(as_u64(x) >> 32);
    const int32_t ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    double f = 0.0, c = 0.0;
    if (hx < 0x3FDA827A) {                                // x < 0.41422
        if (ax >= 0x3ff00000) {                           // x <= -1
            if (x == -1.0) return -1.80143985094819840000e+16 / 0.0;
            return (x - x) / (x - x);
        }
        if (ax < 0x3e200000) {                            // |x| < 2^-29
            if (ax < 0x3c900000) return x;                // |x| < 2^-54
            return fma_(-(x * x), 0.5, x);                // x - x*x*0.5
        }
        if (hx > 0 || hx <= static_cast<int32_t>(0xbfd2bec4)) {  // -0.2929 < x < 0.41422
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx >= 0x7ff00000) {
        return x + x;
    }
    if (k != 0) {
        double u;
        if (hx < 0x43400000) {
            u = 1.0 + x;
            hu = static_cast<int32_t>(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);  // correction term
            c /= u;
        } else {
            u = x;
            hu = static_cast<int32_t>(as_u64(u) >> 32);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        const uint64_t lo = as_u64(u) & 0xffffffffull;
        if (hu < 0x6a09e) {
            u = as_double((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3ff00000)) << 32) | lo);  // u
        } else {
            k += 1;
            u = as_double((static_cast<uint64_t>(static_cast<uint32_t>(hu | 0x3fe00000)) << 32) | lo);  // u/2
            hu = (0x00100000 - hu) >> 2;
        }
        f = u - 1.0;
    }
    const double hfsq = (0.5 * f) * f;
    const double dk = static_cast<double>(k);
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = fma_(dk, ln2_lo, c);
            return fma_(dk, ln2_hi, c);
        }
        const double R = hfsq * fma_(-0.66666666666666666, f, 1.0);
        if (k == 0) return f - R;
        return fma_(dk, ln2_hi, -((R - fma_(dk, ln2_lo, c)) - f));
    }
    const double s = f / (2.0 + f);
    const double z = s * s;
    const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
    const double R2 = fma_(z, Lp3, Lp2), R3 = fma_(z, Lp5, Lp4), R4 = fma_(z, Lp7, Lp6);
    const double R = fma_(z6, R4, fma_(z4, R3, fma_(z, Lp1, z2 * R2)));
    const double P = s * (hfsq + R);
    if (k == 0) return f - (hfsq - P);
    return fma_(dk, ln2_hi, -((hfsq - (P + fma_(dk, ln2_lo, c))) - f));
}

}  // namespace glibc
}  // namespace dsd
