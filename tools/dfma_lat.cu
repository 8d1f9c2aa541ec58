// Microbenchmark: dependent DFMA chain latency and independent DFMA throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(double* out, double a, double b, int iters, long long* cyc) {
    double x = threadIdx.x * 1e-3;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) x = fma(x, a, b);
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
template <int ILP>
__global__ void thru(double* out, double a, double b, int iters) {
    double x[ILP];
#pragma unroll
    for (int j = 0; j < ILP; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int j = 0; j < ILP; ++j) x[j] = fma(x[j], a, b);
    }
    double s = 0;
#pragma unroll
    for (int j = 0; j < ILP; ++j) s += x[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void lds_lat(double* out, int iters, long long* cyc) {
    __shared__ int idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
    __syncthreads();
    int j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) j = idx[j];
    long long t1 = clock64();
    out[threadIdx.x] = j;
    if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
    double* d; long long* c; long long h;
    cudaMalloc(&d, 1 << 26); cudaMalloc(&c, 8);
    int iters = 1000;
    chain<<<1, 32>>>(d, 0.999, 1e-3, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles\n", (double)h / (iters * 16));
    lds_lat<<<1, 32>>>(d, iters, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("LDS dependent latency: %.2f cycles\n", (double)h / iters);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 148; int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    for (int threads : {256, 512, 1024}) {
        thru<8><<<sms * 4, threads>>>(d, 0.999, 1e-3, 10);
        cudaEventRecord(e0);
        int it = 2000;
        thru<8><<<sms * 4, threads>>>(d, 0.999, 1e-3, it);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * sms * 4 * threads * it * 8 * 8;
        printf("DFMA throughput (ILP 8, %d thr/blk x %d blk): %.2f TFLOP/s\n", threads, sms * 4, flops / ms / 1e9);
    }
    printf("clock rate attr %d kHz\n", clk);
    return 0;
}
