// libm_check.cu — TEST INFRASTRUCTURE (not the product): device CUDA libm vs
// the host's glibc on the input domains of the workload generator
// (proj/src/sim/rng.cpp:63-77, trace.cpp:145-187), which the product's
// k_stage evaluates on the device (paper_2511_21669_b200/csrc/device/rng.cuh).
// Compiled with the product's floating-point flags (-fmad=false,
// -ffp-contract=off).  All three are evaluated with the product's
// restatement of glibc's algorithms (glibc_math.cuh), what k_stage and the
// AWC SiLU call.  Inputs come from xoshiro256** streams seeded like the
// generator's; each function is checked on its real argument set:
//   fn 0  log(1 - u)                 exponential gaps and Box-Muller radius
//   fn 1  cos(2 * pi * u)            Box-Muller angle
//   fn 2  exp(mu + sigma * z)        lognormal lengths, mu = log(median)
//         for medians 1..4096 and sigma 0.05..1, z from the same Box-Muller
//   fn 3  log1p(v)                   the AWC feature normaliser
//         (proj/src/awc/mlp.cpp:166): non-negative features up to 5000, and
//         2^-30..2^20 scales
// libm_check() returns the number of bitwise mismatches and how many of them
// change llround(y) (fn 2: the request length) or llround(-m * y * 1000)
// (fn 0: a 1-ms-mean gap in us) - the integers the engine consumes.
#include <cuda_runtime.h>

// the product's device restatement of glibc's exp / log
#include "../../paper_2511_21669_b200/csrc/device/glibc_math.cuh"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

namespace {

struct Xo {
    uint64_t s0, s1, s2, s3;
    __host__ __device__ static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
    __host__ __device__ uint64_t next() {
        const uint64_t r = rotl(s1 * 5, 7) * 9, t = s1 << 17;
        s2 ^= s0; s3 ^= s1; s1 ^= s2; s0 ^= s3; s2 ^= t; s3 = rotl(s3, 45);
        return r;
    }
    __host__ __device__ double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
    static Xo seeded(uint64_t seed) {
        Xo x{};
        uint64_t z = seed;
        for (uint64_t* s : {&x.s0, &x.s1, &x.s2, &x.s3}) {  // splitmix64
            z += 0x9e3779b97f4a7c15ull;
            uint64_t v = z;
            v = (v ^ (v >> 30)) * 0xbf58476d1ce4e5b9ull;
            v = (v ^ (v >> 27)) * 0x94d049bb133111ebull;
            *s = v ^ (v >> 31);
        }
        return x;
    }
};

__global__ void k_eval(int fn, const double* x, double* y, int64_t n) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const double v = x[i];
        y[i] = fn == 0 ? dsd::glibc::log(v) : fn == 1 ? dsd::glibc::cos(v) : fn == 2 ? dsd::glibc::exp(v)
                                                                                 : dsd::glibc::log1p(v);
    }
}

double host_f(int fn, double v) {
    return fn == 0 ? std::log(v) : fn == 1 ? std::cos(v) : fn == 2 ? std::exp(v) : std::log1p(v);
}

// the argument stream of fn for chunk c
void make_inputs(int fn, uint64_t seed, int64_t c, double* x, int64_t n) {
    Xo g = Xo::seeded(seed ^ (0x51ull * static_cast<uint64_t>(c + 1)));
    for (int64_t i = 0; i < n; ++i) {
        if (fn == 0) {
            x[i] = 1.0 - g.unit();
        } else if (fn == 1) {
            x[i] = 2.0 * 3.14159265358979323846 * g.unit();
        } else if (fn == 3) {
            const double u = g.unit();
            x[i] = i % 3 == 0 ? u * 64.0 : i % 3 == 1 ? u * 5000.0 : std::ldexp(u, static_cast<int>(g.next() % 51) - 30);
        } else {
            const double median = 1.0 + static_cast<double>(g.next() % 4096);
            const double sigma = 0.05 + 0.95 * g.unit();
            const double u1 = 1.0 - g.unit(), u2 = g.unit();
            const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * 3.14159265358979323846 * u2);
            x[i] = std::log(median) + sigma * z;
        }
    }
}

}  // namespace

extern "C" int libm_check(int fn, uint64_t seed, int64_t n_total, int64_t* mismatches, int64_t* int_flips,
                          double* example_x) {
    const int64_t chunk = int64_t(1) << 24;
    std::vector<double> x(chunk), yd(chunk);
    double *dx = nullptr, *dy = nullptr;
    if (cudaMalloc(&dx, chunk * 8) != cudaSuccess || cudaMalloc(&dy, chunk * 8) != cudaSuccess) return 1;
    int64_t mm = 0, flips = 0;
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    for (int64_t c = 0, done = 0; done < n_total; ++c, done += chunk) {
        const int64_t n = std::min(chunk, n_total - done);
        {  // inputs, in parallel slices (each slice its own stream)
            std::vector<std::thread> th;
            const int64_t per = (n + hw - 1) / hw;
            for (unsigned t = 0; t < hw; ++t)
                th.emplace_back([&, t] {
                    const int64_t lo = t * per, hi = std::min(n, lo + per);
                    if (lo < hi) make_inputs(fn, seed + t, c, x.data() + lo, hi - lo);
                });
            for (auto& t : th) t.join();
        }
        cudaMemcpy(dx, x.data(), n * 8, cudaMemcpyHostToDevice);
        k_eval<<<1184, 256>>>(fn, dx, dy, n);
        if (cudaMemcpy(yd.data(), dy, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return 2;
        std::vector<int64_t> m(hw, 0), f(hw, 0);
        std::vector<double> ex(hw, 0.0);
        std::vector<std::thread> th;
        const int64_t per = (n + hw - 1) / hw;
        for (unsigned t = 0; t < hw; ++t)
            th.emplace_back([&, t] {
                for (int64_t i = t * per; i < std::min(n, (t + 1) * per); ++i) {
                    const double h = host_f(fn, x[i]);
                    if (std::memcmp(&h, &yd[i], 8) == 0) continue;
                    ++m[t];
                    ex[t] = x[i];
                    if (fn == 2 && std::llround(h) != std::llround(yd[i])) ++f[t];
                    if (fn == 0 && std::llround(-h * 1000.0) != std::llround(-yd[i] * 1000.0)) ++f[t];
                }
            });
        for (auto& t : th) t.join();
        for (unsigned t = 0; t < hw; ++t) {
            mm += m[t];
            flips += f[t];
            if (m[t] && example_x) *example_x = ex[t];
        }
    }
    cudaFree(dx);
    cudaFree(dy);
    *mismatches = mm;
    *int_flips = flips;
    return 0;
}
