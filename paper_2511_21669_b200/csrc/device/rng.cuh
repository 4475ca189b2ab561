// rng.cuh — xoshiro256** streams and the reference's derived distributions,
// bit-compatible with proj/src/sim/rng.cpp:11-77 and proj/include/specsim/util/fnv.hpp:10-18.
//
// Every replica owns its own streams (seeded from seed ^ fnv1a64(label)), so a
// replica's draws are independent of which GPU thread runs it.
#pragma once
#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define DSD_HD __host__ __device__ __forceinline__
#define DSD_HD_NOINLINE __host__ __device__ __noinline__
#else
#define DSD_HD inline
#define DSD_HD_NOINLINE
#endif

#include "glibc_math.cuh"

// exp / log / cos / log1p as the reference's x86-64 glibc computes them:
// glibc's own algorithms on the device (glibc_math.cuh), the host's libm on
// the host
#ifdef __CUDA_ARCH__
#define DSD_EXP(x) ::dsd::glibc::exp(x)
#define DSD_LOG(x) ::dsd::glibc::log(x)
#define DSD_COS(x) ::dsd::glibc::cos(x)
#define DSD_LOG1P(x) ::dsd::glibc::log1p(x)
#else
#define DSD_EXP(x) std::exp(x)
#define DSD_LOG(x) std::log(x)
#define DSD_COS(x) std::cos(x)
#define DSD_LOG1P(x) std::log1p(x)
#endif

namespace dsd {

// fnv1a64 (fnv.hpp:10-18); constexpr so stream labels hash at compile time.
constexpr uint64_t fnv1a64(const char* s, uint64_t h = 0xcbf29ce484222325ULL) {
    while (*s) {
        h ^= static_cast<unsigned char>(*s++);
        h *= 0x100000001b3ULL;
    }
    return h;
}

constexpr uint64_t kLabelRouting = fnv1a64("routing");
constexpr uint64_t kLabelJitter = fnv1a64("jitter");
constexpr uint64_t kLabelArrivals = fnv1a64("arrivals");
constexpr uint64_t kLabelAcceptBits = fnv1a64("accept-bits");
constexpr uint64_t kLabelLengths = fnv1a64("lengths");
constexpr uint64_t kLabelDrafter = fnv1a64("drafter-assign");

DSD_HD uint64_t splitmix64(uint64_t& state) {
    uint64_t z = (state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

DSD_HD uint64_t rotl64(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }

struct Rng {
    uint64_t s0, s1, s2, s3;

    // RngStream::RngStream (rng.cpp:29-33)
    DSD_HD void seed(uint64_t seed, uint64_t label_hash) {
        uint64_t st = seed ^ label_hash;
        s0 = splitmix64(st);
        s1 = splitmix64(st);
        s2 = splitmix64(st);
        s3 = splitmix64(st);
        if ((s0 | s1 | s2 | s3) == 0) s0 = 1;
    }

    // next_u64 (rng.cpp:35-45)
    DSD_HD uint64_t next() {
        const uint64_t result = rotl64(s1 * 5, 7) * 9;
        const uint64_t t = s1 << 17;
        s2 ^= s0;
        s3 ^= s1;
        s1 ^= s2;
        s0 ^= s3;
        s2 ^= t;
        s3 = rotl64(s3, 45);
        return result;
    }

    // next_unit (rng.cpp:47-49): 53-bit uniform in [0, 1)
    DSD_HD double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }

    // uniform_below (rng.cpp:51-58): modulo rejection, no draw for n <= 1
    DSD_HD uint64_t below(uint64_t n) {
        if (n <= 1) return 0;
        const uint64_t threshold = (0 - n) % n;
        for (;;) {
            uint64_t r = next();
            if (r >= threshold) return r % n;
        }
    }

    // uniform (rng.cpp:60-62)
    DSD_HD double uniform(double lo, double hi) { return lo + (hi - lo) * unit(); }

    // exponential (rng.cpp:68-71)
    DSD_HD double exponential(double mean) { return -mean * DSD_LOG(1.0 - unit()); }

    // normal / lognormal (rng.cpp:73-83): Box-Muller, exactly two draws
    DSD_HD double normal(double mean, double stddev) {
        double u1 = 1.0 - unit();
        double u2 = unit();
        double z = sqrt(-2.0 * DSD_LOG(u1)) * DSD_COS(2.0 * 3.14159265358979323846 * u2);
        return mean + stddev * z;
    }
    DSD_HD double lognormal(double mu, double sigma) { return DSD_EXP(normal(mu, sigma)); }
};

}  // namespace dsd
