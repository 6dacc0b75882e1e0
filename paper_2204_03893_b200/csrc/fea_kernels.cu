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

// p <= 2 with the native rule: one element, tables read straight from the kernel parameters
// (constant bank operands of DFMA, fully unrolled over t and q; no shared-memory loads).
template <int NP, int NQ, bool DO_M, bool DO_C>
__device__ __forceinline__ void element_const(const FeaKParams& prm, const double* __restrict__ gU,
                                              const double2* __restrict__ gX, int e_max, int le, bool two_lam,
                                              double* __restrict__ sVm, double* __restrict__ sVc) {
    constexpr int T = NP * (NP + 1) / 2;
    constexpr int oW = (NP * NQ + 1) & ~1;
    constexpr int oQ = oW + ((NQ + 1) & ~1);
    double absdet, A00, A11, A01;
    geometry(gX, e_max, le, absdet, A00, A11, A01);
    double ue[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) ue[i] = gU[i * e_max + le];
    double lm[NQ], lc[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
        double uq = 0.0;
#pragma unroll
        for (int i = 0; i < NP; ++i) uq = fma(prm.ctab[i * NQ + q], ue[i], uq);
        const double wb = prm.ctab[oW + q] * absdet;
        lm[q] = wb * keval(DO_M ? prm.coef_m : prm.coef_c, uq);
        lc[q] = two_lam ? wb * keval(prm.coef_c, uq) : lm[q];
    }
#pragma unroll
    for (int t = 0; t < T; ++t) {
        double vm = 0.0, a = 0.0, b = 0.0, c = 0.0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const double* Qq = prm.ctab + oQ + (t * NQ + q) * 4;
            if (DO_M) vm = fma(Qq[0], lm[q], vm);
            if (DO_C) {
                a = fma(Qq[1], lc[q], a);
                b = fma(Qq[2], lc[q], b);
                c = fma(Qq[3], lc[q], c);
            }
        }
        if (DO_M) sVm[t * e_max + le] = vm;
        if (DO_C) sVc[t * e_max + le] = fma(A00, a, fma(A11, b, A01 * c));
    }
}

// Sum of the C contributors of one slot in the fixed (stored) order, all loads issued first.
template <int C, bool DO_M, bool DO_C>
__device__ __forceinline__ void slot_sum(const uint16_t* __restrict__ cp, const double* __restrict__ sVm,
                                         const double* __restrict__ sVc, double& am, double& ac) {
    int off[C];
#pragma unroll
    for (int q = 0; q < C; ++q) off[q] = cp[q];
    double vm[C], vc[C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        if (DO_M) vm[q] = sVm[off[q]];
        if (DO_C) vc[q] = sVc[off[q]];
    }
    am = 0.0;
    ac = 0.0;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        if (DO_M) am += vm[q];
        if (DO_C) ac += vc[q];
    }
}

template <int C, bool DO_M, bool DO_C>
__device__ __forceinline__ void class_items(int i0, int i1, int cb, const uint16_t* __restrict__ items,
                                            const uint16_t* __restrict__ con, const double* __restrict__ sVm,
                                            const double* __restrict__ sVc, double* om, double* oc, int tid,
                                            int nthr) {
    int it = i0 + tid;
    for (; it + nthr < i1; it += 2 * nthr) {  // two items per thread in flight
        const int s0 = items[it], s1 = items[it + nthr];
        double am0, ac0, am1, ac1;
        slot_sum<C, DO_M, DO_C>(con + cb + (it - i0) * C, sVm, sVc, am0, ac0);
        slot_sum<C, DO_M, DO_C>(con + cb + (it + nthr - i0) * C, sVm, sVc, am1, ac1);
        if (DO_M) {
            om[s0] = am0;
            om[s1] = am1;
        }
        if (DO_C) {
            oc[s0] = ac0;
            oc[s1] = ac1;
        }
    }
    if (it < i1) {
        const int s0 = items[it];
        double am0, ac0;
        slot_sum<C, DO_M, DO_C>(con + cb + (it - i0) * C, sVm, sVc, am0, ac0);
        if (DO_M) om[s0] = am0;
        if (DO_C) oc[s0] = ac0;
    }
}

template <bool DO_M, bool DO_C>
__device__ __forceinline__ void class_items_generic(int c, int i0, int i1, int cb, const uint16_t* __restrict__ items,
                                                    const uint16_t* __restrict__ con, const double* __restrict__ sVm,
                                                    const double* __restrict__ sVc, double* om, double* oc, int tid,
                                                    int nthr) {
    for (int it = i0 + tid; it < i1; it += nthr) {
        const uint16_t* cp = con + cb + (it - i0) * c;
        double am = 0.0, ac = 0.0;
        for (int q = 0; q < c; ++q) {
            const int off = cp[q];
            if (DO_M) am += sVm[off];
            if (DO_C) ac += sVc[off];
        }
        const int s = items[it];
        if (DO_M) om[s] = am;
        if (DO_C) oc[s] = ac;
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

    extern __shared__ __align__(128) uint8_t smem[];
    // p >= 3: tables in shared memory; p <= 2: tables in the kernel parameters (prm.ctab)
    double* sTab = reinterpret_cast<double*>(smem + prm.lay[0]);
    const double* tab = STAGED ? static_cast<const double*>(sTab) : prm.ctab;
    const double* sPhi = tab;
    const double* sW = tab + ((NP * nq + 1) & ~1);
    const double* sQ = sW + ((nq + 1) & ~1);
    uint8_t* sRec0 = smem + prm.lay[1];
    uint8_t* sRec1 = smem + prm.lay[2];
    const bool pf = prm.prefetch != 0;
    double* gUb[2] = {reinterpret_cast<double*>(smem + prm.lay[3]), reinterpret_cast<double*>(smem + prm.lay[pf ? 10 : 3])};
    double2* gXb[2] = {reinterpret_cast<double2*>(smem + prm.lay[4]), reinterpret_cast<double2*>(smem + prm.lay[pf ? 11 : 4])};
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
    if constexpr (STAGED)
        for (int i = tid; i < prm.tables_doubles; i += nthr) sTab[i] = __ldg(prm.tables + i);
    __syncthreads();

    auto issue = [&](int b, int buf) {
        const FeaBlock nb = prm.blocks[b];
        uint8_t* dst = buf ? sRec1 : sRec0;
        fence_proxy_async();
        mbar_expect_tx(&bars[buf], (uint32_t)nb.rec_bytes);
        tma_load_1d(dst, prm.records + nb.rec_off, (uint32_t)nb.rec_bytes, &bars[buf]);
    };
    // gathers of u(N_e) and the vertex coordinates of a block into gather buffer g (async)
    auto gather = [&](const FeaBlock& gb, const uint8_t* grec, int g) {
        const int nEp_ = fea_pad4(gb.nE);
        const int32_t* gd = reinterpret_cast<const int32_t*>(grec + fea_rec_off_dofs(gb));
        double* gu = gUb[g];
        double2* gx = gXb[g];
        for (int le = tid; le < gb.nE; le += nthr) {
#pragma unroll
            for (int i = 0; i < NP; ++i) cp_async8(gu + i * e_max + le, prm.u + gd[i * nEp_ + le]);
#pragma unroll
            for (int v = 0; v < 3; ++v) cp_async16(gx + v * e_max + le, prm.xy + gd[v * nEp_ + le]);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // prologue: records of the first two blocks in flight
    if (tid == 0 && (int)blockIdx.x < prm.nblocks) issue(blockIdx.x, 0);
    if (tid == 0 && (int)(blockIdx.x + gridDim.x) < prm.nblocks) issue(blockIdx.x + gridDim.x, 1);
    if (pf && (int)blockIdx.x < prm.nblocks) {
        mbar_wait(&bars[0], 0);
        gather(prm.blocks[blockIdx.x], sRec0, 0);
    }

    int j = 0;
    for (int bi = blockIdx.x; bi < prm.nblocks; bi += gridDim.x, ++j) {
        const int buf = j & 1;
        const FeaBlock blk = prm.blocks[bi];
        const uint8_t* rec = buf ? sRec1 : sRec0;
        const int nE = blk.nE;
        const int g = pf ? buf : 0;
        if (!pf) {
            mbar_wait(&bars[buf], (uint32_t)((j >> 1) & 1));
            gather(blk, rec, 0);
        }
        const double* gU = gUb[g];
        const double2* gX = gXb[g];
        asm volatile("cp.async.wait_group 0;" ::: "memory");  // this block's gathers landed
        __syncthreads();

        // ---------------- Phase A: element values V[t][le] in shared memory
        if constexpr (!STAGED && NQ_T > 0) {
            for (int le = tid; le < nE; le += nthr)
                element_const<NP, NQ_T, DO_M, DO_C>(prm, gU, gX, e_max, le, two_lam, sVm, sVc);
        } else if constexpr (!STAGED) {
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
        // with prefetch, the next block's gathers fly during phase B
        const int bn = bi + gridDim.x;
        if (pf && bn < prm.nblocks) {
            mbar_wait(&bars[buf ^ 1], (uint32_t)(((j + 1) >> 1) & 1));
            gather(prm.blocks[bn], buf ? sRec0 : sRec1, buf ^ 1);
        }
        __syncthreads();

        // ---------------- Phase B: fixed-order segmented reduction into the CSR slots.
        // Items (slots) come grouped by contributor count c, so every lane of a warp runs the
        // same trip count and the contributor base is arithmetic (no scan).
        const int32_t* cls = reinterpret_cast<const int32_t*>(rec);
        const uint16_t* items = reinterpret_cast<const uint16_t*>(rec + fea_rec_off_items(blk));
        const uint16_t* con = reinterpret_cast<const uint16_t*>(rec + fea_rec_off_contrib(blk));
        double* om = DO_M ? prm.out_m + blk.slot0 : nullptr;
        double* oc = DO_C ? prm.out_c + blk.slot0 : nullptr;
        for (int k = 0; k < blk.ncls; ++k) {
            const int c = cls[3 * k], i0 = cls[3 * k + 1], cb = cls[3 * k + 2];
            const int i1 = k + 1 < blk.ncls ? cls[3 * k + 4] : blk.nslots;
            switch (c) {
                case 1: class_items<1, DO_M, DO_C>(i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr); break;
                case 2: class_items<2, DO_M, DO_C>(i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr); break;
                case 3: class_items<3, DO_M, DO_C>(i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr); break;
                case 4: class_items<4, DO_M, DO_C>(i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr); break;
                case 6: class_items<6, DO_M, DO_C>(i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr); break;
                default: class_items_generic<DO_M, DO_C>(c, i0, i1, cb, items, con, sVm, sVc, om, oc, tid, nthr);
            }
        }
        __syncthreads();
        // this block's record buffer is free: request the record two blocks ahead
        if (tid == 0 && bi + 2 * (int)gridDim.x < prm.nblocks) issue(bi + 2 * gridDim.x, buf);
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
