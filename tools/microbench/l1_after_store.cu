// Microbenchmark: does a global store leave the stored L1 sector invalid for a
// later load?  Each step: dependent load, optional store, then a ~2000-cycle
// spin; cycles per step minus the spin is the load's effective latency.
//   0 no store   1 store to the same word   2 store to another sector of the line
//   3 same word, st.global.L1::evict_last   4 same word, st.global.L1::evict_unchanged
//   5 same word, st.global.L1::no_allocate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k_las(int* buf, int iters, int off, long long spin, long long* out) {
    int* p = buf + (blockIdx.x * blockDim.x + threadIdx.x) * 32;
    int v = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        v = p[v & 3];
        if constexpr (MODE == 1) p[off + (v & 3)] = v & ~3;
        if constexpr (MODE == 2) p[off + 8 + (v & 3)] = v & ~3;
        if constexpr (MODE == 3)
            asm volatile("st.global.L1::evict_last.b32 [%0], %1;" ::"l"(p + off + (v & 3)), "r"(v & ~3) : "memory");
        if constexpr (MODE == 4)
            asm volatile("st.global.L1::evict_unchanged.b32 [%0], %1;" ::"l"(p + off + (v & 3)), "r"(v & ~3) : "memory");
        if constexpr (MODE == 5)
            asm volatile("st.global.L1::no_allocate.b32 [%0], %1;" ::"l"(p + off + (v & 3)), "r"(v & ~3) : "memory");
        const long long s0 = clock64();
        while (clock64() - s0 < spin + (v & 1)) {
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[MODE] = (t1 - t0) / iters;
    if (v == 12345678) buf[0] = v;
}

template <int MODE>
void run(int* buf, long long* out) {
    k_las<MODE><<<1, 64>>>(buf, 100, 0, 2000, out);
    k_las<MODE><<<1, 64>>>(buf, 2000, 0, 2000, out);
    cudaDeviceSynchronize();
    long long with = out[MODE];
    k_las<MODE><<<1, 64>>>(buf, 2000, 0, 0, out);
    cudaDeviceSynchronize();
    printf("mode %d: %lld cycles per step with 2000-cycle spin, %lld without\n", MODE, with, out[MODE]);
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
    return 0;
}
