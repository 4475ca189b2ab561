// glibc_check.cpp — TEST INFRASTRUCTURE: the product's restatement of glibc's
// exp / log (paper_2511_21669_b200/csrc/device/glibc_math.cuh, host build)
// against the host's libm, bit for bit, on the generator's argument domains
// and well beyond.  Prints "<inputs> <log mismatches> <exp mismatches> <cos mismatches>
// <log1p mismatches>".
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "../../paper_2511_21669_b200/csrc/device/glibc_math.cuh"

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : 10000000;
    std::mt19937_64 g(20251019);
    long mm_l = 0, mm_e = 0, mm_c = 0, mm_p = 0;
    for (long t = 0; t < n; ++t) {
        const double u = static_cast<double>(g() >> 11) * 0x1.0p-53;
        // log: 1 - u (exponential gaps, Box-Muller radius) and positive doubles of all scales
        const double xl = t % 2 ? 1.0 - u : std::ldexp(0.5 + 0.5 * u, static_cast<int>(g() % 2100) - 1074);
        double a = std::log(xl), b = dsd::glibc::log(xl);
        if (std::memcmp(&a, &b, 8)) {
            if (mm_l < 5) std::printf("log %a: glibc %a restated %a\n", xl, a, b);
            ++mm_l;
        }
        // exp: lognormal lengths, SiLU arguments, the overflow / subnormal ranges
        const double xe = t % 3 == 0 ? u * 20.0 - 6.0 : (t % 3 == 1 ? u * 1500.0 - 750.0 : (u - 0.5) * 1e-6);
        a = std::exp(xe);
        b = dsd::glibc::exp(xe);
        if (std::memcmp(&a, &b, 8)) {
            if (mm_e < 5) std::printf("exp %a: glibc %a restated %a\n", xe, a, b);
            ++mm_e;
        }
        // cos: the Box-Muller angle 2*pi*u, and [-100, 100]
        const double xc = t % 2 ? 2.0 * 3.14159265358979323846 * u : (u - 0.5) * 200.0;
        a = std::cos(xc);
        b = dsd::glibc::cos(xc);
        if (std::memcmp(&a, &b, 8)) {
            if (mm_c < 5) std::printf("cos %a: glibc %a restated %a\n", xc, a, b);
            ++mm_c;
        }
        // log1p: AWC features (non-negative, up to thousands), (-1, 0.41) and all scales up to 2^1000
        const double xp = t % 4 == 0 ? u * 5000.0
                          : t % 4 == 1 ? u * 1.41 - 0.99999
                          : t % 4 == 2 ? std::ldexp(u, static_cast<int>(g() % 1100) - 80)
                                       : std::ldexp(u, -static_cast<int>(g() % 70));
        a = std::log1p(xp);
        b = dsd::glibc::log1p(xp);
        if (std::memcmp(&a, &b, 8)) {
            if (mm_p < 5) std::printf("log1p %a: glibc %a restated %a\n", xp, a, b);
            ++mm_p;
        }
    }
    std::printf("%ld %ld %ld %ld %ld\n", n, mm_l, mm_e, mm_c, mm_p);
    return 0;
}
