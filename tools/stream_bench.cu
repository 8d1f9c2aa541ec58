// Streaming ceilings on this B200 for the volume kernel's data movement (32 B per DOF-step):
//   copy  : 1 read + 1 write stream (what MEASURED_PEAKS hbm_gbs measures)
//   r2w2  : read p, w; write p', w (w in place) -- the leapfrog kick-drift with no stencil
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/stream_bench tools/stream_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        __stcs(b + i, __ldcs(a + i));
}
__global__ void r2w2_k(const double2* __restrict__ p, double2* __restrict__ w, double2* __restrict__ pn, long long n,
                       double dt) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double2 pv = __ldcs(p + i), wv = __ldcs(w + i);
        wv.x = fma(dt, pv.x, wv.x);
        wv.y = fma(dt, pv.y, wv.y);
        __stcs(w + i, wv);
        __stcs(pn + i, make_double2(fma(dt, wv.x, pv.x), fma(dt, wv.y, pv.y)));
    }
}

int main() {
    const long long n = 1ll << 28;   // doubles per array (2 GiB)
    double *p, *w, *pn;
    cudaMalloc(&p, n * 8);
    cudaMalloc(&w, n * 8);
    cudaMalloc(&pn, n * 8);
    cudaMemset(p, 0, n * 8);
    cudaMemset(w, 0, n * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks_per_sm : {2, 4, 8, 16}) {
        for (int kind = 0; kind < 2; ++kind) {
            const int grid = 148 * blocks_per_sm;
            float best = 1e30f;
            for (int r = 0; r < 6; ++r) {
                cudaEventRecord(e0);
                if (kind == 0) copy_k<<<grid, 256>>>((const double2*)p, (double2*)pn, n / 2);
                else r2w2_k<<<grid, 256>>>((const double2*)p, (double2*)w, (double2*)pn, n / 2, 1e-3);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (r > 0 && ms < best) best = ms;
            }
            const double bytes = (kind == 0 ? 16.0 : 32.0) * n;
            printf("%s blocks/SM=%d: %.1f GB/s\n", kind == 0 ? "copy" : "r2w2", blocks_per_sm, bytes / best / 1e6);
        }
    }
    return 0;
}
