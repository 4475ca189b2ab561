// Microbenchmark: dependent-load latency of per-thread global lines, by load
// flavour and by whether the line was just stored to (the engine's request
// records are read-modify-written every step).  One 128-B line per thread,
// 64 threads in one CTA; prints cycles per dependent step.
//   0 ld (default)            1 ld.ca (__ldca)          2 ld.nc (__ldg)
//   3 ld + st other sector    4 ld + st same word       5 ld.ca + st same word
//   6 lds + sts same word (shared memory reference)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_rmw(int* buf, int iters, int off, long long* out) {
    int* p = buf + (blockIdx.x * blockDim.x + threadIdx.x) * 32;
    __shared__ int sm[64 * 32];
    int* s = sm + threadIdx.x * 32;
    for (int k = 0; k < 32; ++k) s[k] = 0;
    __syncthreads();
    int v = 0;
    long long t0 = clock64();
#pragma unroll 4
    for (int i = 0; i < iters; ++i) {
        if constexpr (MODE == 0) {
            v = p[v & 3];
        } else if constexpr (MODE == 1) {
            v = __ldca(p + (v & 3));
        } else if constexpr (MODE == 2) {
            v = __ldg(p + (v & 3));
        } else if constexpr (MODE == 3) {
            v = p[v & 3];
            p[off + 8 + (v & 3)] = i;
        } else if constexpr (MODE == 4) {
            v = p[v & 3];
            p[off + (v & 3)] = v & ~3;
        } else if constexpr (MODE == 5) {
            v = __ldca(p + (v & 3));
            p[off + (v & 3)] = v & ~3;
        } else {
            v = s[v & 3];
            s[off + (v & 3)] = v & ~3;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[MODE] = (t1 - t0) / iters;
    if (v == 12345678) buf[0] = v;
}

template <int MODE>
void run(int* buf, long long* out) {
    k_rmw<MODE><<<1, 64>>>(buf, 1000, 0, out);
    k_rmw<MODE><<<1, 64>>>(buf, 20000, 0, out);
    cudaDeviceSynchronize();
    printf("mode %d: %lld cycles per dependent step\n", MODE, out[MODE]);
}

int main() {
    int* buf;
    long long* out;
    cudaMalloc(&buf, 1 << 24);
    cudaMemset(buf, 0, 1 << 24);
    cudaMallocManaged(&out, 64);
    run<0>(buf, out);
    run<1>(buf, out);
    run<2>(buf, out);
    run<3>(buf, out);
    run<4>(buf, out);
    run<5>(buf, out);
    run<6>(buf, out);
    return 0;
}
