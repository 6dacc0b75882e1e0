// DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent accumulator chains per
// warp (one CTA per SM): shows the dependent-issue latency the A2 tiling has to hide.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_lat.cu -o dmma_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void k(double* out, int iters, double a) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i) acc[i][0] = acc[i][1] = 0.0;
    double av = a + threadIdx.x, bv = a - threadIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(acc[i][0]), "+d"(acc[i][1]) : "d"(av), "d"(bv));
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) s += acc[i][0] + acc[i][1];
    if (s == 1.2345) out[0] = s;
}

template <int CH>
void run(int sms, double* d, cudaEvent_t e0, cudaEvent_t e1) {
    for (int w : {1, 2, 4, 8, 16}) {
        const int iters = 4096 / CH * 8;
        k<CH><<<sms, 32 * w>>>(d, iters, 1.0);
        cudaEventRecord(e0);
        k<CH><<<sms, 32 * w>>>(d, iters, 1.0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double n = (double)iters * CH;  // DMMAs per warp
        const double flops = 512.0 * n * w * sms;
        printf("chains %d warps/SM %2d: %6.2f TFLOP/s, %.1f ns per dependent DMMA per warp\n", CH, w, flops / ms / 1e9,
               ms * 1e6 / (iters));
    }
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    run<1>(sms, d, e0, e1);
    run<2>(sms, d, e0, e1);
    run<4>(sms, d, e0, e1);
    run<8>(sms, d, e0, e1);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
