// fea_kernels.cu -- sm_100a kernels of the per-iteration hot path.
//
// k_reassemble: ONE persistent kernel per reassembly.  Each CTA loops over row blocks
// (FeaBlock, grid-strided).  Pipeline per block j of a CTA:
//   * TMA bulk copy (cp.async.bulk, mbarrier complete_tx) of block j+1's contiguous record
//     (counts, contributor stream, chunk bases, element DOFs) into the other of two record
//     buffers -- issued before block j is processed, so HBM streams while block j computes;
//   * cp.async gathers of u(N_e) and the vertex coordinates of block j's elements into
//     shared memory (all issued at once: deep memory-level parallelism);
//   * Phase A  (Algorithm 2 lines 5-11) per element:
//              b_e = |det B_e|, A_e = (B_e^T B_e)^{-1}
//              u_q = Phi^T u_e ; S_qe = k(u_q)
//              lambda_q = w_q S_qe b_e
//              V_m[t] = sum_q Q_m[t,q] lambda_q
//              V_c[t] = sum_f W_f sum_q Q_c[t,(q,f)] lambda_q
//            for the symmetric rows t = (i <= j) only, into shared memory.
//            (The stiffness sum over f = {A00, A11, A01} of X_c = Lambda (.) W is taken
//            after the q-sum -- a reassociation of Q_c (Lambda (.) W).)
//   * Phase B  (Algorithm 2 line 12): every CSR slot of the block is the sum of
//            its contributors V[t, e] in ascending library element order (fixed-order
//            segmented reduction over the contributor stream, no atomics); coalesced stores
//            of the block's contiguous slot range.
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_internal.h"

namespace {

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// ------------------------------------------------------------------ math
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

// Element geometry from the staged vertex coordinates: b_e = |det B_e|, A_e = (B^T B)^{-1}
__device__ __forceinline__ void geometry(const double2* __restrict__ gX, int e_max, int le, double& absdet,
                                         double& A00, double& A11, double& A01) {
    const double2 a = gX[le], b = gX[e_max + le], c = gX[2 * e_max + le];
    const double B00 = b.x - a.x, B10 = b.y - a.y, B01 = c.x - a.x, B11 = c.y - a.y;
    const double det = B00 * B11 - B01 * B10;
    absdet = fabs(det);
    const double G00 = B00 * B00 + B10 * B10;
    const double G01 = B00 * B01 + B10 * B11;
    const double G11 = B01 * B01 + B11 * B11;
    const double inv = 1.0 / (det * det);  // det(B^T B) = det(B)^2
    A00 = G11 * inv;
    A11 = G00 * inv;
    A01 = -G01 * inv;
}

// lambda_q = w_q * k(u_q) * |det B_e|, u_q = sum_i Phi[i,q] u_i
template <int NP, int NQM>
__device__ __forceinline__ void form_lambda(const double* __restrict__ sPhi, const double* __restrict__ sW, int nq,
                                            const double* __restrict__ gU, int e_max, int le, double absdet,
                                            const FeaCoef& coef, double (&lam)[NQM]) {
    double ue[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) ue[i] = gU[i * e_max + le];
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

// V rows [t0, t1) of two elements (le0, le1) from Lambda (registers) and the Q table
// (shared memory, [T][nq][4] = m, c00, c11, c01 -> two 16-byte broadcast loads per q).
template <int NQM, bool DO_M, bool DO_C>
__device__ __forceinline__ void contract2(const double* __restrict__ sQ, int nq, int t0, int t1,
                                          const double (&lm0)[NQM], const double (&lc0)[NQM],
                                          const double (&lm1)[NQM], const double (&lc1)[NQM],
                                          const double (&W0)[3], const double (&W1)[3], double* __restrict__ sVm,
                                          double* __restrict__ sVc, int e_max, int le0, int le1, bool has1) {
#pragma unroll 1
    for (int t = t0; t < t1; ++t) {
        const double2* Qt = reinterpret_cast<const double2*>(sQ + t * nq * 4);
        double vm0 = 0.0, a0 = 0.0, b0 = 0.0, c0 = 0.0;
        double vm1 = 0.0, a1 = 0.0, b1 = 0.0, c1 = 0.0;
#pragma unroll
        for (int q = 0; q < NQM; ++q) {
            if (q < nq) {
                const double2 qa = Qt[2 * q], qb = Qt[2 * q + 1];  // (m, c00), (c11, c01)
                if (DO_M) {
                    vm0 = fma(qa.x, lm0[q], vm0);
                    vm1 = fma(qa.x, lm1[q], vm1);
                }
                if (DO_C) {
                    a0 = fma(qa.y, lc0[q], a0);
                    b0 = fma(qb.x, lc0[q], b0);
                    c0 = fma(qb.y, lc0[q], c0);
                    a1 = fma(qa.y, lc1[q], a1);
                    b1 = fma(qb.x, lc1[q], b1);
                    c1 = fma(qb.y, lc1[q], c1);
                }
            }
        }
        if (DO_M) {
            sVm[t * e_max + le0] = vm0;
            if (has1) sVm[t * e_max + le1] = vm1;
        }
        if (DO_C) {
            sVc[t * e_max + le0] = fma(W0[0], a0, fma(W0[1], b0, W0[2] * c0));
            if (has1) sVc[t * e_max + le1] = fma(W1[0], a1, fma(W1[1], b1, W1[2] * c1));
        }
    }
}

template <int P, int NQ_T, bool DO_M, bool DO_C, bool STAGED>
__global__ void __launch_bounds__(256, STAGED ? 1 : 2) k_reassemble(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = (P + 1) * (P + 2) / 2;
    constexpr int T = NP * (NP + 1) / 2;
    constexpr int NQM = NQ_T > 0 ? NQ_T : FEA_MAX_NQ;
    const int nq = NQ_T > 0 ? NQ_T : prm.nq;
    const int e_max = prm.e_max;
    const int tid = threadIdx.x, nthr = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = nthr >> 5;

    extern __shared__ __align__(128) uint8_t smem[];
    double* sTab = reinterpret_cast<double*>(smem + prm.lay[0]);
    const double* sPhi = sTab;
    const double* sW = sTab + ((NP * nq + 1) & ~1);
    const double* sQ = sW + ((nq + 1) & ~1);
    uint8_t* sRec0 = smem + prm.lay[1];
    uint8_t* sRec1 = smem + prm.lay[2];
    double* gU = reinterpret_cast<double*>(smem + prm.lay[3]);
    double2* gX = reinterpret_cast<double2*>(smem + prm.lay[4]);
    double* sVm = reinterpret_cast<double*>(smem + prm.lay[5]);
    double* sVc = reinterpret_cast<double*>(smem + prm.lay[6]);
    double* sLam = reinterpret_cast<double*>(smem + prm.lay[7]);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[8]);
    const bool two_lam = DO_M && DO_C && !prm.same_coef;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbar_init();
    }
    for (int i = tid; i < prm.tables_doubles; i += nthr) sTab[i] = __ldg(prm.tables + i);
    __syncthreads();

    auto issue = [&](int b, int buf) {
        const FeaBlock nb = prm.blocks[b];
        uint8_t* dst = buf ? sRec1 : sRec0;
        fence_proxy_async();
        mbar_expect_tx(&bars[buf], (uint32_t)nb.rec_bytes);
        tma_load_1d(dst, prm.records + nb.rec_off, (uint32_t)nb.rec_bytes, &bars[buf]);
    };
    if (tid == 0 && (int)blockIdx.x < prm.nblocks) issue(blockIdx.x, 0);

    int j = 0;
    for (int bi = blockIdx.x; bi < prm.nblocks; bi += gridDim.x, ++j) {
        const int buf = j & 1;
        const FeaBlock blk = prm.blocks[bi];
        if (tid == 0 && bi + (int)gridDim.x < prm.nblocks) issue(bi + gridDim.x, buf ^ 1);
        mbar_wait(&bars[buf], (uint32_t)((j >> 1) & 1));
        const uint8_t* rec = buf ? sRec1 : sRec0;
        const int nE = blk.nE, nEp = fea_pad4(nE);
        const int32_t* dofs = reinterpret_cast<const int32_t*>(rec + fea_rec_off_dofs(blk));

        // ---------------- gathers: u(N_e) and the vertex coordinates, all in flight at once
        for (int le = tid; le < nE; le += nthr) {
#pragma unroll
            for (int i = 0; i < NP; ++i) cp_async8(gU + i * e_max + le, prm.u + dofs[i * nEp + le]);
#pragma unroll
            for (int v = 0; v < 3; ++v) cp_async16(gX + v * e_max + le, prm.xy + dofs[v * nEp + le]);
        }
        cp_async_wait_all();
        __syncthreads();

        // ---------------- Phase A: element values V[t][le] in shared memory
        if constexpr (!STAGED) {
            for (int le0 = tid; le0 < nE; le0 += 2 * nthr) {
                const int le1 = le0 + nthr;
                const bool has1 = le1 < nE;
                const int lx = has1 ? le1 : le0;
                double d0, d1, W0[3], W1[3];
                geometry(gX, e_max, le0, d0, W0[0], W0[1], W0[2]);
                geometry(gX, e_max, lx, d1, W1[0], W1[1], W1[2]);
                double lm0[NQM], lc0[NQM], lm1[NQM], lc1[NQM];
                form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, le0, d0, DO_M ? prm.coef_m : prm.coef_c, lm0);
                form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, lx, d1, DO_M ? prm.coef_m : prm.coef_c, lm1);
                if (two_lam) {
                    form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, le0, d0, prm.coef_c, lc0);
                    form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, lx, d1, prm.coef_c, lc1);
                } else {
#pragma unroll
                    for (int q = 0; q < NQM; ++q) {
                        lc0[q] = lm0[q];
                        lc1[q] = lm1[q];
                    }
                }
                contract2<NQM, DO_M, DO_C>(sQ, nq, 0, T, lm0, lc0, lm1, lc1, W0, W1, sVm, sVc, e_max, le0, le1, has1);
            }
        } else {
            // A1: Lambda (one or two) and W per element into shared memory
            const int nlam = two_lam ? 2 : 1;
            for (int le = tid; le < nE; le += nthr) {
                double d, W[3], lam[NQM];
                geometry(gX, e_max, le, d, W[0], W[1], W[2]);
                form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, le, d, DO_M ? prm.coef_m : prm.coef_c, lam);
#pragma unroll
                for (int q = 0; q < NQM; ++q)
                    if (q < nq) sLam[q * e_max + le] = lam[q];
                if (two_lam) {
                    form_lambda<NP, NQM>(sPhi, sW, nq, gU, e_max, le, d, prm.coef_c, lam);
#pragma unroll
                    for (int q = 0; q < NQM; ++q)
                        if (q < nq) sLam[(nq + q) * e_max + le] = lam[q];
                }
                sLam[(nlam * nq + 0) * e_max + le] = W[0];
                sLam[(nlam * nq + 1) * e_max + le] = W[1];
                sLam[(nlam * nq + 2) * e_max + le] = W[2];
            }
            __syncthreads();
            // A2: items (t-chunk, element pair); a warp shares one t-chunk
            const int npair = (nE + 1) >> 1;
            const int np32 = (npair + 31) & ~31;
            const int ntc = prm.ntc;
            const int tper = (T + ntc - 1) / ntc;
            for (int it = tid; it < ntc * np32; it += nthr) {
                const int tc = it / np32, pr = it - tc * np32;
                if (pr >= npair) continue;
                const int le0 = pr, le1 = pr + npair;  // second half of the block
                const bool has1 = le1 < nE;
                const int lx = has1 ? le1 : le0;
                double lm0[NQM], lc0[NQM], lm1[NQM], lc1[NQM], W0[3], W1[3];
#pragma unroll
                for (int q = 0; q < NQM; ++q) {
                    lm0[q] = q < nq ? sLam[q * e_max + le0] : 0.0;
                    lm1[q] = q < nq ? sLam[q * e_max + lx] : 0.0;
                    lc0[q] = two_lam ? (q < nq ? sLam[(nq + q) * e_max + le0] : 0.0) : lm0[q];
                    lc1[q] = two_lam ? (q < nq ? sLam[(nq + q) * e_max + lx] : 0.0) : lm1[q];
                }
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    W0[f] = sLam[(nlam * nq + f) * e_max + le0];
                    W1[f] = sLam[(nlam * nq + f) * e_max + lx];
                }
                const int t0 = tc * tper, t1 = min(T, t0 + tper);
                contract2<NQM, DO_M, DO_C>(sQ, nq, t0, t1, lm0, lc0, lm1, lc1, W0, W1, sVm, sVc, e_max, le0, le1, has1);
            }
        }
        __syncthreads();

        // ---------------- Phase B: fixed-order segmented reduction into the CSR slots
        const uint8_t* cnt = rec;
        const uint16_t* con = reinterpret_cast<const uint16_t*>(rec + fea_rec_off_contrib(blk));
        const int32_t* chk = reinterpret_cast<const int32_t*>(rec + fea_rec_off_chunk(blk));
        const int nchunks = (blk.nslots + 31) >> 5;
        for (int ch = warp; ch < nchunks; ch += nwarp) {
            const int s = ch * 32 + lane;
            const bool valid = s < blk.nslots;
            const int c = valid ? (int)cnt[s] : 0;
            int incl = c;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int v = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += v;
            }
            const int base = chk[ch] + incl - c;
            double am = 0.0, ac = 0.0;
            for (int k = 0; k < c; ++k) {
                const int off = con[base + k];
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

template <int P, int NQ_T>
using kfun_t = void (*)(const FeaKParams);

template <int P, int NQ_T>
kfun_t<P, NQ_T> pick(int dm, int dc) {
    constexpr bool S = P >= 3;  // Lambda staged in shared memory, rows split over threads
    if (dm && dc) return k_reassemble<P, NQ_T, true, true, S>;
    if (dm) return k_reassemble<P, NQ_T, true, false, S>;
    return k_reassemble<P, NQ_T, false, true, S>;
}

template <int P, int NQ_T>
cudaError_t launch_p(const FeaKParams& prm, int threads, int smem, int grid, cudaStream_t st) {
    auto kern = pick<P, NQ_T>(prm.out_m != nullptr, prm.out_c != nullptr);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (err != cudaSuccess) return err;
    kern<<<grid, threads, smem, st>>>(prm);
    return cudaGetLastError();
}

template <int P, int NQ_T>
cudaError_t occ_p(int dm, int dc, int threads, int smem, int* n) {
    auto kern = pick<P, NQ_T>(dm, dc);
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
    if (staged != (order >= 3 ? 1 : 0)) return (int)cudaErrorInvalidValue;
    const bool nat = prm.nq == nq_native(order);
    cudaError_t e;
    switch (order) {
        case 1: e = nat ? launch_p<1, 3>(prm, threads, smem_bytes, grid, st) : launch_p<1, 0>(prm, threads, smem_bytes, grid, st); break;
        case 2: e = nat ? launch_p<2, 6>(prm, threads, smem_bytes, grid, st) : launch_p<2, 0>(prm, threads, smem_bytes, grid, st); break;
        case 3: e = nat ? launch_p<3, 12>(prm, threads, smem_bytes, grid, st) : launch_p<3, 0>(prm, threads, smem_bytes, grid, st); break;
        case 4: e = nat ? launch_p<4, 16>(prm, threads, smem_bytes, grid, st) : launch_p<4, 0>(prm, threads, smem_bytes, grid, st); break;
        default: e = cudaErrorInvalidValue;
    }
    return (int)e;
}

int fea_kernel_occupancy(int order, int nq, int dm, int dc, int staged, int threads, int smem, int* n) {
    if (staged != (order >= 3 ? 1 : 0)) return (int)cudaErrorInvalidValue;
    const bool nat = nq == nq_native(order);
    cudaError_t e;
    switch (order) {
        case 1: e = nat ? occ_p<1, 3>(dm, dc, threads, smem, n) : occ_p<1, 0>(dm, dc, threads, smem, n); break;
        case 2: e = nat ? occ_p<2, 6>(dm, dc, threads, smem, n) : occ_p<2, 0>(dm, dc, threads, smem, n); break;
        case 3: e = nat ? occ_p<3, 12>(dm, dc, threads, smem, n) : occ_p<3, 0>(dm, dc, threads, smem, n); break;
        case 4: e = nat ? occ_p<4, 16>(dm, dc, threads, smem, n) : occ_p<4, 0>(dm, dc, threads, smem, n); break;
        default: e = cudaErrorInvalidValue;
    }
    return (int)e;
}
