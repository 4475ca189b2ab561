// Microbenchmark: latency of a dependent load after a store to the same
// global line (does a store keep the line in L1?), vs load-only and shared memory.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_rmw(int* buf, int iters, long long* out, int mode) {
    int* p = buf + (blockIdx.x * blockDim.x + threadIdx.x) * 32;  // one 128-B line per thread
    __shared__ int sm[64 * 32];
    int* s = sm + threadIdx.x * 32;
    int v = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        if (mode == 0) {          // global load-only chain
            v = p[v & 7];
        } else if (mode == 1) {   // global load -> store -> dependent load (same line)
            v = p[v & 7];
            p[8 + (v & 7)] = v + i;
        } else if (mode == 2) {   // shared memory RMW chain
            v = s[v & 7];
            s[8 + (v & 7)] = v + i;
        } else {                  // global RMW via volatile-free __ldca / __stwb hints
            v = __ldca(p + (v & 7));
            __stwb(p + 8 + (v & 7), v + i);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[mode] = (t1 - t0) / iters;
    if (v == 12345678) buf[0] = v;
}

int main() {
    int* buf;
    long long* out;
    cudaMalloc(&buf, 1 << 24);
    cudaMemset(buf, 0, 1 << 24);
    cudaMallocManaged(&out, 64);
    for (int mode = 0; mode < 4; ++mode) {
        k_rmw<<<1, 64>>>(buf, 1000, out, mode);
        k_rmw<<<1, 64>>>(buf, 10000, out, mode);
        cudaDeviceSynchronize();
        printf("mode %d: %lld cycles per dependent iteration\n", mode, out[mode]);
    }
    return 0;
}
