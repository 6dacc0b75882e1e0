// The A2 inner loop of k_reassemble6 in isolation: NA warps per SM, each RT row tiles (4 accumulator
// chains per tile: m, A00, A11, A01), B-fragments from shared memory (4 LDS.64 per element tile), the
// W epilogue and two 16-byte V stores per row tile -- does this loop saturate the DMMA pipe?
// Optional extra warps hammer shared memory with 16-byte loads (phase B's V reads).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a a2_loop.cu -o a2_loop
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int RT, int NA, int NBW, bool EPI, int MODE = 0>
__global__ void __launch_bounds__((NA + NBW) * 32, 1) k(double* out, int iters) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ls = 52, vs = 49, g8 = lane >> 2, cq = lane & 3;
    double* Lam = sm;                   // [16][ls]
    double* W = sm + 16 * ls;           // [3][48]
    double2* V = reinterpret_cast<double2*>(sm + 16 * ls + 3 * 48);  // [120][vs]
    for (int i = threadIdx.x; i < 16 * ls + 3 * 48; i += blockDim.x) sm[i] = 1e-3 * i;
    if (threadIdx.x == 0) *reinterpret_cast<int*>(sm + 16 * 52 + 3 * 48 + 120 * 49 * 2) = 0;
    __syncthreads();
    if (warp < NA) {
        double afr[RT][4][4];
        for (int r = 0; r < RT; ++r)  // distinct values (as the kernel's Q_f fragments), from memory
            for (int f = 0; f < 4; ++f)
                for (int kk = 0; kk < 4; ++kk) afr[r][f][kk] = sm[((r * 4 + f) * 4 + kk) * 5 + lane % 7];
        double s = 0;
        for (int it = 0; it < iters; ++it)
            for (int et = 0; et < 6; ++et) {
                const int col = et * 8 + g8, le0 = et * 8 + 2 * cq;
                double bl[4];
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) bl[kk] = Lam[(kk * 4 + cq) * ls + col];
#pragma unroll
                for (int r = 0; r < RT; ++r) {
                    double m0 = 0, m1 = 0, a0 = 0, a1 = 0, p0 = 0, p1 = 0, c0 = 0, c1 = 0;
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        dmma(m0, m1, afr[r][0][kk], bl[kk]);
                        dmma(a0, a1, afr[r][1][kk], bl[kk]);
                        dmma(p0, p1, afr[r][2][kk], bl[kk]);
                        dmma(c0, c1, afr[r][3][kk], bl[kk]);
                    }
                    if (EPI) {
                        const double2 w0 = *reinterpret_cast<const double2*>(W + le0);
                        const double2 w1 = *reinterpret_cast<const double2*>(W + 48 + le0);
                        const double2 w2 = *reinterpret_cast<const double2*>(W + 96 + le0);
                        const double k0 = fma(w0.x, a0, fma(w1.x, p0, w2.x * c0));
                        const double k1 = fma(w0.y, a1, fma(w1.y, p1, w2.y * c1));
                        const int t = (warp + r * NA) * 8 + g8;
                        V[(t % 120) * vs + le0] = make_double2(m0, k0);
                        V[(t % 120) * vs + le0 + 1] = make_double2(m1, k1);
                    } else {
                        s += m0 + m1 + a0 + a1 + p0 + p1 + c0 + c1;
                    }
                }
            }
        if (s == 1.2345) out[0] = s;
        if (MODE == 1) {
            asm volatile("bar.sync 2, %0;" ::"r"(NA * 32));
            if (threadIdx.x == 0) *reinterpret_cast<volatile int*>(sm + 16 * 52 + 3 * 48 + 120 * 49 * 2) = 1;
        }
    } else if (MODE == 1) {  // spin on an mbarrier that completes only when the A warps are done
        __shared__ uint64_t bar;
        if (threadIdx.x == NA * 32) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&bar)), "r"(1));
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NBW * 32));
        const unsigned a = (unsigned)__cvta_generic_to_shared(&bar);
        volatile int* flag = reinterpret_cast<volatile int*>(sm + 16 * 52 + 3 * 48 + 120 * 49 * 2);
        for (int it = 0; it < 100000000 && flag[0] == 0; ++it) {
            asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n}" ::"r"(a), "r"(0) : "memory");
        }
    } else {  // phase-B-like shared-memory traffic
        double s = 0;
        for (int it = 0; it < iters * 40; ++it) {
            const double2 x = V[(lane * 37 + it * 11) % (120 * vs)];
            s += x.x + x.y;
        }
        if (s == 1.2345) out[0] = s;
    }
}

template <int RT, int NA, int NBW, bool EPI, int MODE = 0>
void run(const char* name, int sms, double* d) {
    const int smem = (16 * 52 + 3 * 48) * 8 + 120 * 49 * 16 + 16;
    cudaFuncSetAttribute(k<RT, NA, NBW, EPI, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<RT, NA, NBW, EPI, MODE><<<sms, (NA + NBW) * 32, smem>>>(d, iters);
    cudaEventRecord(e0);
    k<RT, NA, NBW, EPI, MODE><<<sms, (NA + NBW) * 32, smem>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmmas = (double)iters * 6 * RT * 16 * NA * sms;
    printf("%-40s %6.2f TFLOP/s  (%.3f ms)\n", name, dmmas * 512 / ms / 1e9, ms);
}


// two element tiles per pass: each A fragment feeds two consecutive DMMAs (operand reuse)
template <int RT, int NA>
__global__ void __launch_bounds__(NA * 32, 1) k2(double* out, int iters) {
    extern __shared__ double sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ls = 52, vs = 49, g8 = lane >> 2, cq = lane & 3;
    double* Lam = sm;
    double* W = sm + 16 * ls;
    double2* V = reinterpret_cast<double2*>(sm + 16 * ls + 3 * 48);
    for (int i = threadIdx.x; i < 16 * ls + 3 * 48; i += blockDim.x) sm[i] = 1e-3 * i;
    __syncthreads();
    double afr[RT][4][4];
    for (int r = 0; r < RT; ++r)
        for (int f = 0; f < 4; ++f)
            for (int kk = 0; kk < 4; ++kk) afr[r][f][kk] = sm[((r * 4 + f) * 4 + kk) * 5 + lane % 7];
    for (int it = 0; it < iters; ++it)
        for (int e2 = 0; e2 < 6; e2 += 2) {
            double bl[2][4];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) bl[h][kk] = Lam[(kk * 4 + cq) * ls + (e2 + h) * 8 + g8];
#pragma unroll
            for (int r = 0; r < RT; ++r) {
                double acc[2][4][2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int f = 0; f < 4; ++f) acc[h][f][0] = acc[h][f][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
#pragma unroll
                    for (int f = 0; f < 4; ++f)
#pragma unroll
                        for (int h = 0; h < 2; ++h) dmma(acc[h][f][0], acc[h][f][1], afr[r][f][kk], bl[h][kk]);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int le0 = (e2 + h) * 8 + 2 * cq;
                    const double2 w0 = *reinterpret_cast<const double2*>(W + le0);
                    const double2 w1 = *reinterpret_cast<const double2*>(W + 48 + le0);
                    const double2 w2 = *reinterpret_cast<const double2*>(W + 96 + le0);
                    const double k0 = fma(w0.x, acc[h][1][0], fma(w1.x, acc[h][2][0], w2.x * acc[h][3][0]));
                    const double k1 = fma(w0.y, acc[h][1][1], fma(w1.y, acc[h][2][1], w2.y * acc[h][3][1]));
                    const int t = (warp + r * NA) * 8 + g8;
                    V[(t % 120) * vs + le0] = make_double2(acc[h][0][0], k0);
                    V[(t % 120) * vs + le0 + 1] = make_double2(acc[h][0][1], k1);
                }
            }
        }
}

template <int RT, int NA>
void run2(const char* name, int sms, double* d) {
    const int smem = (16 * 52 + 3 * 48) * 8 + 120 * 49 * 16 + 16;
    cudaFuncSetAttribute(k2<RT, NA>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k2<RT, NA><<<sms, NA * 32, smem>>>(d, iters);
    cudaEventRecord(e0);
    k2<RT, NA><<<sms, NA * 32, smem>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dmmas = (double)iters * 6 * RT * 16 * NA * sms;
    printf("%-40s %6.2f TFLOP/s  (%.3f ms)\n", name, dmmas * 512 / ms / 1e9, ms);
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<2, 8, 0, false>("8 warps RT2, no epilogue", sms, d);
    run<2, 8, 0, true>("8 warps RT2, epilogue", sms, d);
    run<2, 8, 8, true>("8 warps RT2, epilogue, +8 LDS warps", sms, d);
    run<1, 16, 0, true>("16 warps RT1, epilogue", sms, d);
    run<1, 15, 1, true>("15 warps RT1, epilogue, +1 LDS warp", sms, d);
    run<2, 4, 0, true>("4 warps RT2, epilogue", sms, d);
    run<2, 8, 8, true, 1>("8 warps RT2, epilogue, +8 try_wait spinners", sms, d);
    run2<2, 8>("8 warps RT2, 2 element tiles per pass", sms, d);
    run2<1, 16>("16 warps RT1, 2 element tiles per pass", sms, d);
    run2<2, 16>("16 warps RT2, 2 element tiles per pass", sms, d);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
