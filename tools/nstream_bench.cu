// How HBM throughput on this B200 depends on the number of concurrent read / write streams
// (separate cudaMalloc arrays of the curved box's size, grid-stride double2 accesses).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nstream_bench tools/nstream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
struct Ptrs { const double2* r[8]; double2* w[8]; };
template <int NR, int NW>
__global__ void __launch_bounds__(256) ns_k(Ptrs p, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double2 s = make_double2(0, 0);
#pragma unroll
        for (int k = 0; k < NR; ++k) { const double2 v = p.r[k][i]; s.x += v.x; s.y += v.y; }
#pragma unroll
        for (int k = 0; k < NW; ++k) p.w[k][i] = s;
    }
}
template <int NR, int NW>
void run(double** a, long long n, int grid) {
    Ptrs p;
    for (int k = 0; k < 8; ++k) { p.r[k] = (const double2*)a[k]; p.w[k] = (double2*)a[8 + k]; }
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 8; ++r) {
        cudaEventRecord(e0);
        ns_k<NR, NW><<<grid, 256>>>(p, n / 2);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    printf("n=%lld r%dw%d grid=%d: %.3f ms %.1f GB/s\n", n, NR, NW, grid, best, 8.0 * (NR + NW) * n / (best * 1e-3) / 1e9);
}
int main() {
    for (long long n : {28400000LL, 1LL << 27}) {
        double* a[16];
        for (int k = 0; k < 16; ++k) { cudaMalloc(&a[k], n * 8); cudaMemset(a[k], 0, n * 8); }
        const int g = 148 * 8;
        run<1, 1>(a, n, g); run<2, 2>(a, n, g); run<2, 1>(a, n, g); run<3, 1>(a, n, g); run<4, 0>(a, n, g);
        run<3, 3>(a, n, g); run<4, 2>(a, n, g); run<5, 3>(a, n, g); run<8, 0>(a, n, g); run<0, 4>(a, n, g);
        for (int k = 0; k < 16; ++k) cudaFree(a[k]);
    }
    return 0;
}
