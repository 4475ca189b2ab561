// Microbenchmark: dependent-chain latency of FP64 add / mul / fma and FP32 add
// on one warp (cycles per dependent op).
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, long long* cyc, int n, double a, double b) {
    double x = a + threadIdx.x;
    float f = static_cast<float>(x);
    long long t0 = clock64();
#pragma unroll 16
    for (int i = 0; i < n; ++i) {
        if (OP == 0) x = x + b;
        if (OP == 1) x = x * b;
        if (OP == 2) x = fma(x, b, a);
        if (OP == 3) f = f + static_cast<float>(b);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[OP] = (t1 - t0) / n;
    out[threadIdx.x] = x + f;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 32 * 8);
    cudaMallocManaged(&cyc, 64);
    for (int r = 0; r < 2; ++r) {
        k<0><<<1, 32>>>(out, cyc, 1 << 16, 1.0, 1.0000001);
        k<1><<<1, 32>>>(out, cyc, 1 << 16, 1.0, 1.0000001);
        k<2><<<1, 32>>>(out, cyc, 1 << 16, 1.0, 0.9999999);
        k<3><<<1, 32>>>(out, cyc, 1 << 16, 1.0, 1.0000001);
        cudaDeviceSynchronize();
    }
    printf("dependent latency (cycles): DADD %lld  DMUL %lld  DFMA %lld  FADD %lld\n", cyc[0], cyc[1], cyc[2], cyc[3]);
    return 0;
}
