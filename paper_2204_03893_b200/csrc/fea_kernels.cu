// fea_kernels.cu -- sm_100a kernels of the per-iteration hot path.
//
// k_reassemble: ONE persistent kernel per reassembly.  Each CTA loops over row blocks
// (FeaBlock); per block:
//   Phase A  (Algorithm 2 lines 5-11) for every element of the block
//            (ghosts, then owned range):
//              gather u_e = u(N_e) and the vertex coordinates
//              b_e = |det B_e|, A_e = (B_e^T B_e)^{-1}
//              u_q = Phi^T u_e ; S_qe = k(u_q)
//              lambda_q = w_q S_qe b_e
//              V_m[t] = sum_q Q_m[t,q] lambda_q
//              V_c[t] = sum_f W_f sum_q Q_c[t,(q,f)] lambda_q
//            for the symmetric rows t = (i <= j) only, into shared memory.
//            (The stiffness sum over f = {A00, A11, A01} of X_c = Lambda (.) W is taken
//            after the q-sum -- a reassociation of Q_c (Lambda (.) W).)
//   Phase B  (Algorithm 2 line 12): every CSR slot of the block is the sum of
//            its contributors V[t, e] in ascending library element order (fixed-order
//            segmented reduction over the precomputed contributor stream, no atomics);
//            coalesced stores of the block's contiguous slot range.
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_internal.h"

namespace {

__device__ __forceinline__ double keval(const FeaCoef& c, double u) {
    if (c.kind == 0) {  // sum_i par[i] u^i (Horner)
        double r = c.par[c.npar - 1];
        for (int i = c.npar - 2; i >= 0; --i) r = fma(r, u, c.par[i]);
        return r;
    }
    if (c.kind == 1) return c.par[0] * exp(c.par[1] * u);
    // piecewise linear, segment s covers (T_s, T_{s+1}]
    const int m = c.npar / 2;
    int s = 0;
    while (s < m - 2 && u > c.par[2 * (s + 1)]) ++s;
    const double T0 = c.par[2 * s], k0 = c.par[2 * s + 1], T1 = c.par[2 * s + 2], k1 = c.par[2 * s + 3];
    return k0 + (k1 - k0) / (T1 - T0) * (u - T0);
}

template <int NP>
__device__ __forceinline__ void load_element(const FeaKParams& prm, int e, double (&ue)[NP],
                                             double& absdet, double& A00, double& A11, double& A01) {
    int dof[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) dof[i] = __ldg(prm.dofT + (int64_t)i * prm.n_e + e);
#pragma unroll
    for (int i = 0; i < NP; ++i) ue[i] = __ldg(prm.u + dof[i]);
    const double2 a = __ldg(prm.xy + dof[0]);
    const double2 b = __ldg(prm.xy + dof[1]);
    const double2 c = __ldg(prm.xy + dof[2]);
    // B_e = [b - a, c - a]
    const double B00 = b.x - a.x, B10 = b.y - a.y, B01 = c.x - a.x, B11 = c.y - a.y;
    const double det = B00 * B11 - B01 * B10;
    absdet = fabs(det);
    // A_e = (B^T B)^{-1} = adj(B^T B) / det(B)^2
    const double G00 = B00 * B00 + B10 * B10;
    const double G01 = B00 * B01 + B10 * B11;
    const double G11 = B01 * B01 + B11 * B11;
    const double inv = 1.0 / (det * det);
    A00 = G11 * inv;
    A11 = G00 * inv;
    A01 = -G01 * inv;
}

// lambda_q = w_q * k(u_q) * |det B_e|, u_q = sum_i Phi[i,q] u_i
template <int NP, int NQM>
__device__ __forceinline__ void form_lambda(const double* __restrict__ sPhi, const double* __restrict__ sW, int nq,
                                            const double (&ue)[NP], double absdet, const FeaCoef& coef,
                                            double (&lam)[NQM]) {
#pragma unroll
    for (int q = 0; q < NQM; ++q) {
        if (q < nq) {
            double uq = 0.0;
#pragma unroll
            for (int i = 0; i < NP; ++i) uq = fma(sPhi[i * nq + q], ue[i], uq);
            lam[q] = sW[q] * keval(coef, uq) * absdet;
        } else {
            lam[q] = 0.0;
        }
    }
}

// V rows [t0, t1) of one element from lambda (registers) and the Q table (shared memory).
template <int NQM, bool DO_M, bool DO_C>
__device__ __forceinline__ void contract(const double* __restrict__ sQ, int nq, int t0, int t1,
                                         const double (&lm)[NQM], const double (&lc)[NQM],
                                         double A00, double A11, double A01, double* __restrict__ sVm,
                                         double* __restrict__ sVc, int e_max, int le) {
    for (int t = t0; t < t1; ++t) {
        const double* Qt = sQ + t * 4 * nq;
        double vm = 0.0, s0 = 0.0, s1 = 0.0, s2 = 0.0;
#pragma unroll
        for (int q = 0; q < NQM; ++q) {
            if (q < nq) {
                if (DO_M) vm = fma(Qt[q], lm[q], vm);
                if (DO_C) {
                    s0 = fma(Qt[nq + q], lc[q], s0);
                    s1 = fma(Qt[2 * nq + q], lc[q], s1);
                    s2 = fma(Qt[3 * nq + q], lc[q], s2);
                }
            }
        }
        if (DO_M) sVm[t * e_max + le] = vm;
        if (DO_C) sVc[t * e_max + le] = fma(A00, s0, fma(A11, s1, A01 * s2));
    }
}

template <int P, int NQ_T, bool DO_M, bool DO_C, bool STAGED>
__global__ void __launch_bounds__(256) k_reassemble(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = (P + 1) * (P + 2) / 2;
    constexpr int T = NP * (NP + 1) / 2;
    constexpr int NQM = NQ_T > 0 ? NQ_T : FEA_MAX_NQ;
    const int nq = NQ_T > 0 ? NQ_T : prm.nq;
    const int e_max = prm.e_max;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;

    extern __shared__ __align__(16) double smem[];
    double* sTab = smem;                           // Phi, w, Q
    double* sPhi = sTab;
    double* sW = sTab + NP * nq;
    double* sQ = sW + nq;
    double* sVm = sTab + ((prm.tables_doubles + 1) & ~1);
    double* sVc = sVm + (DO_M ? T * e_max : 0);
    double* sLam = sVc + (DO_C ? T * e_max : 0);   // STAGED: [nlam*nq + 3][e_max]
    const bool two_lam = DO_M && DO_C && !prm.same_coef;

    for (int i = tid; i < prm.tables_doubles; i += nthr) sTab[i] = __ldg(prm.tables + i);
    __syncthreads();

    for (int bi = blockIdx.x; bi < prm.nblocks; bi += gridDim.x) {
        const FeaBlock blk = prm.blocks[bi];
        const int nE = blk.nghost + blk.nown;

        // ---------------- Phase A: element values V[t][le] in shared memory
        if constexpr (!STAGED) {
            for (int le = tid; le < nE; le += nthr) {
                const int e = le < blk.nghost ? __ldg(prm.ghosts + blk.ghost0 + le) : blk.own0 + (le - blk.nghost);
                double ue[NP], absdet, A00, A11, A01;
                load_element<NP>(prm, e, ue, absdet, A00, A11, A01);
                double lm[NQM], lc[NQM];
                if (DO_M) form_lambda<NP, NQM>(sPhi, sW, nq, ue, absdet, prm.coef_m, lm);
                if (DO_C) {
                    if (DO_M && prm.same_coef) {
#pragma unroll
                        for (int q = 0; q < NQM; ++q) lc[q] = lm[q];
                    } else {
                        form_lambda<NP, NQM>(sPhi, sW, nq, ue, absdet, prm.coef_c, lc);
                    }
                } else {
#pragma unroll
                    for (int q = 0; q < NQM; ++q) lc[q] = 0.0;
                }
                if (!DO_M) {
#pragma unroll
                    for (int q = 0; q < NQM; ++q) lm[q] = 0.0;
                }
                contract<NQM, DO_M, DO_C>(sQ, nq, 0, T, lm, lc, A00, A11, A01, sVm, sVc, e_max, le);
            }
        } else {
            // A1: Lambda (and W) per element into shared memory
            const int nlam = two_lam ? 2 : 1;
            for (int le = tid; le < nE; le += nthr) {
                const int e = le < blk.nghost ? __ldg(prm.ghosts + blk.ghost0 + le) : blk.own0 + (le - blk.nghost);
                double ue[NP], absdet, A00, A11, A01;
                load_element<NP>(prm, e, ue, absdet, A00, A11, A01);
                double lam[NQM];
                form_lambda<NP, NQM>(sPhi, sW, nq, ue, absdet, *(DO_M ? &prm.coef_m : &prm.coef_c), lam);
                for (int q = 0; q < nq; ++q) sLam[q * e_max + le] = lam[q];
                if (two_lam) {
                    form_lambda<NP, NQM>(sPhi, sW, nq, ue, absdet, prm.coef_c, lam);
                    for (int q = 0; q < nq; ++q) sLam[(nq + q) * e_max + le] = lam[q];
                }
                sLam[(nlam * nq + 0) * e_max + le] = A00;
                sLam[(nlam * nq + 1) * e_max + le] = A11;
                sLam[(nlam * nq + 2) * e_max + le] = A01;
            }
            __syncthreads();
            // A2: items (t-chunk, element); a warp shares one t-chunk
            const int nE32 = (nE + 31) & ~31;
            const int ntc = prm.ntc;
            const int tper = (T + ntc - 1) / ntc;
            for (int it = tid; it < ntc * nE32; it += nthr) {
                const int tc = it / nE32, le = it - tc * nE32;
                if (le >= nE) continue;
                double lm[NQM], lc[NQM];
#pragma unroll
                for (int q = 0; q < NQM; ++q) {
                    const double l0 = q < nq ? sLam[q * e_max + le] : 0.0;
                    lm[q] = l0;
                    lc[q] = two_lam ? (q < nq ? sLam[(nq + q) * e_max + le] : 0.0) : l0;
                }
                const double A00 = sLam[(nlam * nq + 0) * e_max + le];
                const double A11 = sLam[(nlam * nq + 1) * e_max + le];
                const double A01 = sLam[(nlam * nq + 2) * e_max + le];
                const int t0 = tc * tper, t1 = min(T, t0 + tper);
                contract<NQM, DO_M, DO_C>(sQ, nq, t0, t1, lm, lc, A00, A11, A01, sVm, sVc, e_max, le);
            }
        }
        __syncthreads();

        // ---------------- Phase B: fixed-order segmented reduction into the CSR slots
        const int nchunks = (blk.nslots + 31) >> 5;
        const uint8_t* cnt = prm.counts + blk.slot0;
        const uint16_t* con = prm.contrib + blk.contrib0;
        for (int ch = warp; ch < nchunks; ch += nwarp) {
            const int s = ch * 32 + lane;
            const bool valid = s < blk.nslots;
            const int c = valid ? (int)__ldg(cnt + s) : 0;
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const int base = __ldg(prm.chunk_base + blk.chunk0 + ch) + incl - c;
            double am = 0.0, ac = 0.0;
            for (int k = 0; k < c; ++k) {
                const int off = __ldg(con + base + k);
                if (DO_M) am += sVm[off];
                if (DO_C) ac += sVc[off];
            }
            if (valid) {
                if (DO_M) prm.out_m[blk.slot0 + s] = am;
                if (DO_C) prm.out_c[blk.slot0 + s] = ac;
            }
        }
        __syncthreads();
    }
}

template <int P, int NQ_T, bool STAGED>
cudaError_t launch_p(const FeaKParams& prm, int threads, int smem, int grid, cudaStream_t st) {
    const bool dm = prm.out_m != nullptr, dc = prm.out_c != nullptr;
    void (*kern)(const FeaKParams);
    if (dm && dc) kern = k_reassemble<P, NQ_T, true, true, STAGED>;
    else if (dm) kern = k_reassemble<P, NQ_T, true, false, STAGED>;
    else kern = k_reassemble<P, NQ_T, false, true, STAGED>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    kern<<<grid, threads, smem, st>>>(prm);
    return cudaGetLastError();
}

// STAGED (Lambda in shared memory, rows split over threads) for p >= 3, fused for p <= 2.
template <int P, int NQ_T>
cudaError_t launch_s(const FeaKParams& prm, int threads, int smem, int grid, int staged, cudaStream_t st) {
    if (staged != (P >= 3 ? 1 : 0)) return cudaErrorInvalidValue;
    return launch_p<P, NQ_T, (P >= 3)>(prm, threads, smem, grid, st);
}

template <int P, int NQ_T, bool STAGED>
cudaError_t occ_p(int dm, int dc, int threads, int smem, int* n) {
    void (*kern)(const FeaKParams);
    if (dm && dc) kern = k_reassemble<P, NQ_T, true, true, STAGED>;
    else if (dm) kern = k_reassemble<P, NQ_T, true, false, STAGED>;
    else kern = k_reassemble<P, NQ_T, false, true, STAGED>;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, threads, smem);
}

}  // namespace

// Rule sizes with a specialised kernel: the minimal Dunavant rules of the configs
// (3, 6, 12, 16 points for p = 1..4); any other n_q <= 16 runs the generic variant.
static int nq_native(int order) { return order == 1 ? 3 : order == 2 ? 6 : order == 3 ? 12 : 16; }

int fea_launch_reassemble(const FeaKParams& prm, int order, int threads, int smem_bytes, int grid, int staged,
                          void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const bool nat = prm.nq == nq_native(order);
    cudaError_t e;
    switch (order) {
        case 1: e = nat ? launch_s<1, 3>(prm, threads, smem_bytes, grid, staged, st) : launch_s<1, 0>(prm, threads, smem_bytes, grid, staged, st); break;
        case 2: e = nat ? launch_s<2, 6>(prm, threads, smem_bytes, grid, staged, st) : launch_s<2, 0>(prm, threads, smem_bytes, grid, staged, st); break;
        case 3: e = nat ? launch_s<3, 12>(prm, threads, smem_bytes, grid, staged, st) : launch_s<3, 0>(prm, threads, smem_bytes, grid, staged, st); break;
        case 4: e = nat ? launch_s<4, 16>(prm, threads, smem_bytes, grid, staged, st) : launch_s<4, 0>(prm, threads, smem_bytes, grid, staged, st); break;
        default: e = cudaErrorInvalidValue;
    }
    return (int)e;
}

int fea_kernel_occupancy(int order, int nq, int dm, int dc, int staged, int threads, int smem, int* n) {
    const bool nat = nq == nq_native(order);
    cudaError_t e;
#define FEA_OCC(P, Q) (staged != (P >= 3 ? 1 : 0) ? cudaErrorInvalidValue : occ_p<P, Q, (P >= 3)>(dm, dc, threads, smem, n))
    switch (order) {
        case 1: e = nat ? FEA_OCC(1, 3) : FEA_OCC(1, 0); break;
        case 2: e = nat ? FEA_OCC(2, 6) : FEA_OCC(2, 0); break;
        case 3: e = nat ? FEA_OCC(3, 12) : FEA_OCC(3, 0); break;
        case 4: e = nat ? FEA_OCC(4, 16) : FEA_OCC(4, 0); break;
        default: e = cudaErrorInvalidValue;
    }
#undef FEA_OCC
    return (int)e;
}
