// FP64 peak microbenchmark on the B200: DFMA (CUDA cores) vs DMMA (mma.sync m8n8k4 f64).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters, double a, double b) {
    double x[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i) x[i] = fma(x[i], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_dmma(double* out, int iters, double a) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    double av = a + threadIdx.x, bv = a - threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1.2345) out[0] = s;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
        const int iters = 20000;
        for (int blocks_per_sm : {4, 8}) {
            cudaEventRecord(e0);
            k_dfma<<<sms * blocks_per_sm, 256>>>(d, iters, 1.0000001, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            double flops = 2.0 * 16 * iters * 256.0 * sms * blocks_per_sm;
            printf("DFMA  %d CTA/SM: %.2f TFLOP/s\n", blocks_per_sm, flops / ms / 1e9);
            cudaEventRecord(e0);
            k_dmma<<<sms * blocks_per_sm, 256>>>(d, iters / 4, 1.0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            flops = 2.0 * 256 * 8 * (iters / 4) * (256 / 32) * sms * (double)blocks_per_sm;
            printf("DMMA  %d CTA/SM: %.2f TFLOP/s\n", blocks_per_sm, flops / ms / 1e9);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
