// Microbenchmark: one AWC network evaluation (H = 64, 2 residual blocks, the
// WC-DNN shape) by a whole warp (awc_forward_warp) vs by each lane on its own
// (awc_forward_lane, 32 lanes in parallel); cycles per evaluation.
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2511_21669_b200/csrc/device/engine.cuh"

using namespace dsd;

__global__ void k_coop(const char* blob, const DevScenario* S, int iters, long long* out, double* sink) {
    __shared__ AwcWarpScratch sc;
    const int lane = threadIdx.x;
    for (int k = 0; k < 5; ++k) sc.x[lane][k] = 0.1 * (lane + k);
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) acc += awc_forward_warp(blob, S, sc.x[it & 31], &sc);
    long long t1 = clock64();
    if (lane == 0) out[0] = (t1 - t0) / iters;
    sink[lane] = acc;
}

// the same network on column-major weights: lane r reads element c of its
// row at wt[c * H + r], so a warp load of one column is contiguous
__device__ double forward_warp_t(const double* p, int H, int I, int blocks, const double* x, AwcWarpScratch* sc) {
    const int lane = threadIdx.x & 31;
    auto dot_t = [&](const double* wt, const double* v, int r, int cols) {
        const int tail = cols & ~3;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        int c = 0;
        for (; c < tail; c += 4) {
            a0 = a0 + wt[c * H + r] * v[c];
            a1 = a1 + wt[(c + 1) * H + r] * v[c + 1];
            a2 = a2 + wt[(c + 2) * H + r] * v[c + 2];
            a3 = a3 + wt[(c + 3) * H + r] * v[c + 3];
        }
        double s = (a0 + a2) + (a1 + a3);
        for (; c < cols; ++c) s += wt[c * H + r] * v[c];
        return s;
    };
    for (int r = lane; r < H; r += 32) sc->hv[r] = p[H * I + r] + dot_t(p, x, r, I);
    __syncwarp();
    int64_t off = static_cast<int64_t>(H) * I + H;
    for (int b = 0; b < blocks; ++b) {
        const double* w1 = p + off;
        const double* b1 = w1 + H * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + H * H;
        for (int r = lane; r < H; r += 32) {
            const double u = b1[r] + dot_t(w1, sc->hv, r, H);
            sc->sv[r] = u * (1.0 / (1.0 + exp(-u)));
        }
        __syncwarp();
        for (int r = lane; r < H; r += 32) sc->hv[r] += b2[r] + dot_t(w2, sc->sv, r, H);
        __syncwarp();
        off += 2 * H * H + 2 * H;
    }
    double out = 0.0;
    if (lane == 0) {
        const double* w_out = p + off;
        out = w_out[H];
        for (int i = 0; i < H; ++i) out += w_out[i] * sc->hv[i];
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, out, 0);
}

// row-major, compile-time width 64, fully unrolled, read-only loads: the
// scheduler can hoist the row's weight loads ahead of the add chains
template <int C>
__device__ __forceinline__ double dot_fixed(const double* __restrict__ row, const double* x) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int c = 0; c < (C & ~3); c += 4) {
        a0 = a0 + __ldg(row + c) * x[c];
        a1 = a1 + __ldg(row + c + 1) * x[c + 1];
        a2 = a2 + __ldg(row + c + 2) * x[c + 2];
        a3 = a3 + __ldg(row + c + 3) * x[c + 3];
    }
    double s = (a0 + a2) + (a1 + a3);
#pragma unroll
    for (int c = C & ~3; c < C; ++c) s += __ldg(row + c) * x[c];
    return s;
}
__device__ double forward_warp_fixed(const double* p, int blocks, const double* x, AwcWarpScratch* sc) {
    constexpr int H = 64, I = 5;
    const int lane = threadIdx.x & 31;
    for (int r = lane; r < H; r += 32) sc->hv[r] = p[H * I + r] + dot_fixed<I>(p + r * I, x);
    __syncwarp();
    int64_t off = H * I + H;
    for (int b = 0; b < blocks; ++b) {
        const double* w1 = p + off;
        const double* b1 = w1 + H * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + H * H;
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = lane + 32 * rr;
            const double u = b1[r] + dot_fixed<H>(w1 + r * H, sc->hv);
            sc->sv[r] = u * (1.0 / (1.0 + exp(-u)));
        }
        __syncwarp();
#pragma unroll
        for (int rr = 0; rr < 2; ++rr) {
            const int r = lane + 32 * rr;
            sc->hv[r] += b2[r] + dot_fixed<H>(w2 + r * H, sc->sv);
        }
        __syncwarp();
        off += 2 * H * H + 2 * H;
    }
    double out = 0.0;
    if (lane == 0) {
        const double* w_out = p + off;
        out = w_out[H];
        for (int i = 0; i < H; ++i) out += w_out[i] * sc->hv[i];
    }
    __syncwarp();
    return __shfl_sync(0xffffffffu, out, 0);
}
__global__ void k_coop_f(const double* p, int blocks, int iters, long long* out, double* sink) {
    __shared__ AwcWarpScratch sc;
    const int lane = threadIdx.x;
    for (int k = 0; k < 5; ++k) sc.x[lane][k] = 0.1 * (lane + k);
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) acc += forward_warp_fixed(p, blocks, sc.x[it & 31], &sc);
    long long t1 = clock64();
    if (lane == 0) out[3] = (t1 - t0) / iters;
    sink[lane] = acc;
}

// per-lane, compile-time width 64 (the lane's vectors in registers / local)
__device__ double forward_lane_fixed(const double* p, int blocks, const double* x) {
    constexpr int H = 64, I = 5;
    double h[H], u[H], sv[H];
#pragma unroll 4
    for (int r = 0; r < H; ++r) h[r] = p[H * I + r] + dot_fixed<I>(p + r * I, x);
    int64_t off = H * I + H;
    for (int b = 0; b < blocks; ++b) {
        const double* w1 = p + off;
        const double* b1 = w1 + H * H;
        const double* w2 = b1 + H;
        const double* b2 = w2 + H * H;
        for (int r = 0; r < H; ++r) {
            u[r] = b1[r] + dot_fixed<H>(w1 + r * H, h);
            sv[r] = u[r] * (1.0 / (1.0 + exp(-u[r])));
        }
        for (int r = 0; r < H; ++r) h[r] += b2[r] + dot_fixed<H>(w2 + r * H, sv);
        off += 2 * H * H + 2 * H;
    }
    const double* w_out = p + off;
    double out = w_out[H];
    for (int i = 0; i < H; ++i) out += w_out[i] * h[i];
    return out;
}
__global__ void k_lane_f(const double* p, int blocks, int iters, long long* out, double* sink) {
    const int lane = threadIdx.x;
    double x[5];
    for (int k = 0; k < 5; ++k) x[k] = 0.1 * (lane + k);
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x[0] += 1e-3;
        acc += forward_lane_fixed(p, blocks, x);
    }
    long long t1 = clock64();
    if (lane == 0) out[4] = (t1 - t0) / iters;
    sink[lane] = acc;
}

__global__ void k_coop_t(const double* p, int H, int I, int blocks, int iters, long long* out, double* sink) {
    __shared__ AwcWarpScratch sc;
    const int lane = threadIdx.x;
    for (int k = 0; k < 5; ++k) sc.x[lane][k] = 0.1 * (lane + k);
    __syncwarp();
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) acc += forward_warp_t(p, H, I, blocks, sc.x[it & 31], &sc);
    long long t1 = clock64();
    if (lane == 0) out[2] = (t1 - t0) / iters;
    sink[lane] = acc;
}

__global__ void k_lane(const char* blob, const DevScenario* S, int iters, long long* out, double* sink) {
    const int lane = threadIdx.x;
    double x[5];
    for (int k = 0; k < 5; ++k) x[k] = 0.1 * (lane + k);
    double acc = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        x[0] += 1e-3;
        acc += awc_forward_lane(blob, *S, x);
    }
    long long t1 = clock64();
    if (lane == 0) out[1] = (t1 - t0) / iters;
    sink[lane] = acc;
}

int main() {
    const int H = 64, I = 5, B = 2;
    const size_t np = H * I + H + B * (2 * H * H + 2 * H) + H + 1;
    std::vector<double> params(np);
    for (size_t i = 0; i < np; ++i) params[i] = 0.01 * static_cast<double>((i * 2654435761u) % 1000) / 1000.0 - 0.005;
    DevScenario S{};
    S.awc_hidden = H;
    S.awc_input = I;
    S.awc_blocks = B;
    S.o_awc_params = 0;
    for (int f = 0; f < 5; ++f) { S.awc_lo[f] = 0; S.awc_hi[f] = 1; }
    char* blob;
    DevScenario* dS;
    long long* out;
    double* sink;
    cudaMalloc(&blob, np * 8);
    cudaMemcpy(blob, params.data(), np * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&dS, sizeof(S));
    cudaMemcpy(dS, &S, sizeof(S), cudaMemcpyHostToDevice);
    cudaMalloc(&sink, 32 * 8);
    // column-major copy of the three weight matrices
    std::vector<double> t(params);
    auto transpose = [&](size_t off, int rows, int cols) {
        for (int r = 0; r < rows; ++r)
            for (int c = 0; c < cols; ++c) t[off + static_cast<size_t>(c) * rows + r] = params[off + static_cast<size_t>(r) * cols + c];
    };
    size_t off = 0;
    transpose(off, H, I);
    off += H * I + H;
    for (int b = 0; b < B; ++b) {
        transpose(off, H, H);
        transpose(off + H * H + H, H, H);
        off += 2 * H * H + 2 * H;
    }
    double* pt;
    cudaMalloc(&pt, np * 8);
    cudaMemcpy(pt, t.data(), np * 8, cudaMemcpyHostToDevice);
    cudaMallocManaged(&out, 32);
    for (int rep = 0; rep < 2; ++rep) {
        k_coop<<<1, 32>>>(blob, dS, 200, out, sink);
        k_coop_t<<<1, 32>>>(pt, H, I, B, 200, out, sink);
        k_coop_f<<<1, 32>>>(reinterpret_cast<const double*>(blob), B, 200, out, sink);
        k_lane_f<<<1, 32>>>(reinterpret_cast<const double*>(blob), B, 20, out, sink);
        k_lane<<<1, 32>>>(blob, dS, 20, out, sink);
        cudaDeviceSynchronize();
    }
    printf("cycles per evaluation: warp-cooperative %lld, column-major cooperative %lld, fixed-width unrolled %lld, "
           "per-lane (32 in parallel) %lld, per-lane fixed-width %lld\n", out[0], out[2], out[3], out[1], out[4]);
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
