// fea_kernels.cu -- sm_100a kernel of the per-iteration hot path.
//
// k_reassemble<P, NQ, DO_M, DO_C>: ONE persistent, warp-specialised kernel per reassembly.
// Each CTA loops over row blocks (FeaBlock, grid-strided).
//
//   PRODUCER warp (the last warp), up to two blocks ahead of the consumers:
//     * one TMA bulk copy (cp.async.bulk + mbarrier complete_tx) per block of its contiguous
//       record (count classes, slot items, contributor stream, element DOFs);
//     * cp.async gathers of u(N_e) and the vertex coordinates of every element of the block
//       into a shared-memory stage, completion signalled with cp.async.mbarrier.arrive.
//   CONSUMER warps, per block:
//     A1 (Algorithm 2 lines 4-9), one thread per element:
//          b_e = |det B_e|, W_e = vec A_e, A_e = (B_e^T B_e)^{-1}
//          u_q = Phi^T u_e ; S_qe = k(u_q)
//          Lambda_qe = w_q S_qe b_e                                    (Eq. def_lambda)
//     A2 (Algorithm 2 lines 10-11) on the FP64 tensor cores (DMMA):
//          V_m = Q_m Lambda ; V_c = sum_f W_f (Q_c,f Lambda),  f in {A00, A11, A01}
//          for the symmetric rows t = (i <= j) only.  The sum over f of
//          Q_c (Lambda (.) W) is taken after the q-contraction (a reassociation);
//          each warp keeps its row tile of Q_f as DMMA A-fragments in registers.
//     B  (Algorithm 2 line 12): every CSR slot of the block = sum of its
//          contributors V[t, e] in ascending library element order (fixed-order segmented
//          reduction over the contributor stream, no atomics); slots grouped by contributor
//          count so warps run uniform trip counts.
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_device.cuh"

namespace {
using namespace fea_dev;

// ------------------------------------------------------------------ the kernel
template <int P, int NQ_T, bool DO_M, bool DO_C>
__global__ void __launch_bounds__(fea_threads(P), fea_ctas(P)) k_reassemble(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = fea_np(P);
    constexpr int T = fea_T(P);
    constexpr int NTT = fea_ntt(P);
    constexpr int S = fea_S(P);
    constexpr int RS = fea_rstages(P);
    constexpr int NK = NQ_T > 0 ? fea_nk(NQ_T) : fea_nk(FEA_MAX_NQ);  // k-steps (generic rule: 4, zero padded)
    constexpr int NQP = 4 * NK;                                       // padded quadrature count
    const int nq = NQ_T > 0 ? NQ_T : prm.nq;
    const int e_max = prm.e_max, ls = fea4_lstride(e_max);  // ls: Lambda / gathered-u row stride
    const int tid = threadIdx.x;
    constexpr int RT = fea_rt(P), NGRP = fea_ngrp(P);
    constexpr int NCT = NGRP * S * 32;  // consumer threads
    const bool producer = tid >= NCT;
    const int lane = tid & 31, warp = tid >> 5;

    extern __shared__ __align__(128) uint8_t smem[];
    // stage pointers (computed, not arrays: no local-memory indexing)
    auto sRec = [&](int s) { return smem + prm.lay[FEA_L_REC + s]; };
    auto gUb = [&](int s) { return reinterpret_cast<double*>(smem + prm.lay[FEA_L_GU + s]); };
    auto gXb = [&](int s) { return reinterpret_cast<double2*>(smem + prm.lay[FEA_L_GX + s]); };
    double* sLm = reinterpret_cast<double*>(smem + prm.lay[FEA_L_LAMM]);
    double* sLc = reinterpret_cast<double*>(smem + prm.lay[FEA_L_LAMC]);
    double* sW = reinterpret_cast<double*>(smem + prm.lay[FEA_L_W]);
    double* sVm = reinterpret_cast<double*>(smem + prm.lay[FEA_L_VM]);
    double* sVc = reinterpret_cast<double*>(smem + prm.lay[FEA_L_VC]);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA_L_BARS]);
    uint64_t* full_rec = bars;      // [3] record landed (TMA transactions)
    uint64_t* full_gat = bars + 3;  // [2] gathers landed (32 producer lanes)
    uint64_t* rdone = bars + 5;     // [3] consumers finished with the record stage
    uint64_t* gdone = bars + 8;     // [2] consumers finished with the gather stage
    const bool two_lam = DO_M && DO_C && !prm.same_coef;
    const int ncta_blocks = prm.nblocks > (int)blockIdx.x ? (prm.nblocks - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    if (tid == 0) {
        for (int s = 0; s < 3; ++s) {
            mbar_init(&full_rec[s], 1);
            mbar_init(&rdone[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full_gat[s], 32);
            mbar_init(&gdone[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (producer) {
        auto issue_rec = [&](int jj) {  // TMA of the record of the CTA's jj-th block
            const FeaBlock b = prm.blocks[blockIdx.x + jj * gridDim.x];
            const int s = jj % RS;
            fence_proxy_async();
            mbar_expect_tx(&full_rec[s], (uint32_t)b.rec_bytes);
            tma_load_1d(sRec(s), prm.records + b.rec_off, (uint32_t)b.rec_bytes, &full_rec[s]);
        };
        if (lane == 0)
            for (int jj = 0; jj < RS - 1 && jj < ncta_blocks; ++jj) issue_rec(jj);
        for (int j = 0; j < ncta_blocks; ++j) {
            const int rs = j % RS, gs = j & 1;
            if (j >= 2) mbar_wait(&gdone[gs], (uint32_t)(((j >> 1) - 1) & 1));  // stage free (block j-2)
            mbar_wait(&full_rec[rs], (uint32_t)((j / RS) & 1));                   // record j landed
            const FeaRecHdr4 blk = *reinterpret_cast<const FeaRecHdr4*>(sRec(rs));
            const int nEp = fea_pad4(blk.nE);
            const int32_t* gd = reinterpret_cast<const int32_t*>(sRec(rs) + blk.dofs_off);
            double* gu = gUb(gs);
            double2* gx = gXb(gs);
            for (int le = lane; le < blk.nE; le += 32) {
#pragma unroll
                for (int i = 0; i < NP; ++i) FEA_CHECK(gd[i * nEp + le] >= 0 && gd[i * nEp + le] < prm.n_dof);
#pragma unroll
                for (int i = 0; i < NP; ++i) cp_async8(gu + i * ls + le, prm.u + gd[i * nEp + le]);
#pragma unroll
                for (int v = 0; v < 3; ++v) cp_async16(gx + v * e_max + le, prm.xy + gd[v * nEp + le]);
            }
            cp_async_mbar_arrive(&full_gat[gs]);
            // record of block j + RS - 1 into the stage of block j - 1 once that block is done
            const int jn = j + RS - 1;
            if (jn < ncta_blocks) {
                if (j >= 1) mbar_wait(&rdone[(j - 1) % RS], (uint32_t)(((j - 1) / RS) & 1));
                if (lane == 0) issue_rec(jn);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ------------------------------------------------------------------ consumers
    // This warp's row tiles (grp, grp + NGRP, ...) of Q_f as DMMA A-fragments, for the whole kernel.
    const int grp = warp % NGRP, sub = warp / NGRP;
    const int g = lane >> 2, cq = lane & 3;
    double afr[RT][4][NK];
#pragma unroll
    for (int r = 0; r < RT; ++r)
#pragma unroll
        for (int f = 0; f < 4; ++f)
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
                const int tt = grp + r * NGRP;
                afr[r][f][kk] = (f == 0 ? DO_M : DO_C) && tt < NTT
                                    ? __ldg(prm.qfrag + ((f * NTT + tt) * NK + kk) * 32 + lane) : 0.0;
            }
    constexpr bool INTERP_MMA = fea_interp_mma(P);
    constexpr int MTN = INTERP_MMA ? (NQP + 7) / 8 : 1, KTN = INTERP_MMA ? fea_kt(P) : 1;
    double pfr[MTN][KTN];  // Phi^T A-fragments (p >= 2)
#pragma unroll
    for (int mt = 0; mt < MTN; ++mt)
#pragma unroll
        for (int kt = 0; kt < KTN; ++kt)
            pfr[mt][kt] = INTERP_MMA ? __ldg(prm.qfrag + 4 * NTT * NK * 32 + (mt * KTN + kt) * 32 + lane) : 0.0;
    const double* cPhi = prm.ctab;
    const double* cW = prm.ctab + ((NP * nq + 1) & ~1);

#ifdef FEA5_DIAG
    unsigned long long tacc[6] = {0, 0, 0, 0, 0, 0};
    unsigned long long tcl = 0;
    auto tick = [&](int slot) {  // optional phase timing (consumer thread 0), diagnostics builds only
        if (prm.dbg && tid == 0) {
            const unsigned long long now = clock64();
            if (slot >= 0) tacc[slot] += now - tcl;
            tcl = now;
        }
    };
#else
    auto tick = [](int) {};
#endif
    const int vs = fea4_vstride(e_max);  // V row stride (fea_internal.h)

    // ---------------- A1 of block j: geometry (W_e, b_e), u_q = Phi^T u_e, k(u_q), Lambda
    auto phase_a1 = [&](int j) {
        const int rs = j % RS, gs = j & 1;
        const double* gU = gUb(gs);
        const double2* gX = gXb(gs);
        mbar_wait(&full_rec[rs], (uint32_t)((j / RS) & 1));
        const int nE = reinterpret_cast<const FeaRecHdr4*>(sRec(rs))->nE;
        const int net = (nE + 7) >> 3;
        mbar_wait(&full_gat[gs], (uint32_t)((j >> 1) & 1));
        if constexpr (!INTERP_MMA) {
            for (int le = tid; le < net * 8; le += NCT) {
                if (le < nE) {
                    double absdet, A00, A11, A01;
                    geometry(gX, e_max, le, absdet, A00, A11, A01);
                    sW[le] = A00;
                    sW[e_max + le] = A11;
                    sW[2 * e_max + le] = A01;
                    double ue[NP];
#pragma unroll
                    for (int i = 0; i < NP; ++i) ue[i] = gU[i * ls + le];
#pragma unroll
                    for (int q = 0; q < NQP; ++q) {
                        double lm = 0.0, lc = 0.0;
                        if (q < nq) {
                            double uq = 0.0;
#pragma unroll
                            for (int i = 0; i < NP; ++i) uq = fma(cPhi[i * nq + q], ue[i], uq);
                            const double wb = cW[q] * absdet;
                            lm = wb * keval(DO_M ? prm.coef_m : prm.coef_c, uq);
                            lc = two_lam ? wb * keval(prm.coef_c, uq) : lm;
                        }
                        sLm[q * ls + le] = lm;
                        if (two_lam) sLc[q * ls + le] = lc;
                    }
                } else {  // padding columns of the last element tile
#pragma unroll
                    for (int q = 0; q < NQP; ++q) {
                        sLm[q * ls + le] = 0.0;
                        if (two_lam) sLc[q * ls + le] = 0.0;
                    }
                    sW[le] = sW[e_max + le] = sW[2 * e_max + le] = 0.0;
                }
            }
        } else {
            // U = Phi^T U_e on DMMA; epilogue Lambda_qe = w_q b_e k(u_qe) with the geometry of the
            // lane's two accumulator columns (recomputed per m-tile; the m-tile 0, g = 0 lanes store W_e)
            constexpr int MT = MTN, KT = KTN;
            for (int un = warp; un < MT * net; un += NGRP * S) {
                const int mt = un % MT, et = un / MT;
                double u0 = 0.0, u1 = 0.0;
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) {
                    const int i = kt * 4 + cq;
                    const double b = i < NP ? gU[i * ls + et * 8 + g] : 0.0;
                    double a = pfr[0][kt];  // select the m-tile without dynamic register indexing
#pragma unroll
                    for (int m2 = 1; m2 < MT; ++m2) a = mt == m2 ? pfr[m2][kt] : a;
                    dmma(u0, u1, a, b);
                }
                const int q = mt * 8 + g, le0 = et * 8 + 2 * cq;
                double d0 = 0.0, d1 = 0.0, w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0, w20 = 0.0, w21 = 0.0;
                if (le0 < nE) geometry(gX, e_max, le0, d0, w00, w10, w20);
                if (le0 + 1 < nE) geometry(gX, e_max, le0 + 1, d1, w01, w11, w21);
                if (mt == 0 && g == 0) {
                    *reinterpret_cast<double2*>(sW + le0) = make_double2(w00, w01);
                    *reinterpret_cast<double2*>(sW + e_max + le0) = make_double2(w10, w11);
                    *reinterpret_cast<double2*>(sW + 2 * e_max + le0) = make_double2(w20, w21);
                }
                if (q < NQP) {
                    double lm0 = 0.0, lm1 = 0.0, lc0 = 0.0, lc1 = 0.0;
                    if (q < nq) {
                        const double w = cW[q];
                        const FeaCoef& cf = DO_M ? prm.coef_m : prm.coef_c;
                        if (le0 < nE) lm0 = w * d0 * keval(cf, u0);
                        if (le0 + 1 < nE) lm1 = w * d1 * keval(cf, u1);
                        if (two_lam) {
                            if (le0 < nE) lc0 = w * d0 * keval(prm.coef_c, u0);
                            if (le0 + 1 < nE) lc1 = w * d1 * keval(prm.coef_c, u1);
                        }
                    }
                    *reinterpret_cast<double2*>(sLm + q * ls + le0) = make_double2(lm0, lm1);
                    if (two_lam) *reinterpret_cast<double2*>(sLc + q * ls + le0) = make_double2(lc0, lc1);
                }
            }
        }
    };

    // Software pipeline over the CTA's blocks, two CTA barriers per block:
    //   A1(0) | for j: A2(j) | B(j) and A1(j + 1) |
    // (A1 writes Lambda / W, which A2(j) has finished reading; B reads V and the record of block j).
    if (ncta_blocks > 0) {
        phase_a1(0);
        consumer_sync(NCT);
        if (tid == 0) mbar_arrive(&gdone[0]);
    }
    tick(-1);
    for (int j = 0; j < ncta_blocks; ++j) {
        const int rs = j % RS;
        const uint8_t* rec = sRec(rs);
        const FeaRecHdr4 blk = *reinterpret_cast<const FeaRecHdr4*>(rec);  // descriptor from the record
        const int nE = blk.nE;
        const int net = (nE + 7) >> 3;

        // ---------------- A2: V = Q Lambda on the FP64 tensor cores (DMMA m8n8k4)
        {
            const double* Lc = two_lam ? sLc : sLm;
            for (int et = sub; et < net; et += S) {
                const int col = et * 8 + g;       // B fragment column (element) of this lane
                const int le0 = et * 8 + 2 * cq;  // the two accumulator columns of this lane
                double bm[NK], bc[NK];
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) {
                    bm[kk] = sLm[(kk * 4 + cq) * ls + col];
                    bc[kk] = Lc[(kk * 4 + cq) * ls + col];
                }
                double2 w0, w1, w2;
                if (DO_C) {
                    w0 = *reinterpret_cast<const double2*>(sW + le0);
                    w1 = *reinterpret_cast<const double2*>(sW + e_max + le0);
                    w2 = *reinterpret_cast<const double2*>(sW + 2 * e_max + le0);
                }
#pragma unroll
                for (int r = 0; r < RT; ++r) {
                    const int t = (grp + r * NGRP) * 8 + g;
                    if (RT > 1 && grp + r * NGRP >= NTT) continue;
                    double m0 = 0.0, m1 = 0.0, a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0, c0 = 0.0, c1 = 0.0;
#pragma unroll
                    for (int kk = 0; kk < NK; ++kk) {
                        if (DO_M) dmma(m0, m1, afr[r][0][kk], bm[kk]);
                        if (DO_C) {
                            dmma(a0, a1, afr[r][1][kk], bc[kk]);
                            dmma(b0, b1, afr[r][2][kk], bc[kk]);
                            dmma(c0, c1, afr[r][3][kk], bc[kk]);
                        }
                    }
                    if (t < T) {
                        if (DO_M) *reinterpret_cast<double2*>(sVm + t * vs + le0) = make_double2(m0, m1);
                        if (DO_C)
                            *reinterpret_cast<double2*>(sVc + t * vs + le0) =
                                make_double2(fma(w0.x, a0, fma(w1.x, b0, w2.x * c0)), fma(w0.y, a1, fma(w1.y, b1, w2.y * c1)));
                    }
                }
            }
        }
        tick(2);
        consumer_sync(NCT);  // V complete; Lambda / W free
        tick(5);

        // ---------------- Phase B of block j (fixed-order segmented reduction into the CSR slots)
        // and A1 of block j + 1, in alternating order across warps so the two overlap.
        const bool a1_first = (FEA4_A1FIRST == 2 || (FEA4_A1FIRST == 1 && (warp & 1))) && j + 1 < ncta_blocks;
        if (a1_first) phase_a1(j + 1);
        phase_b5<DO_M, DO_C>(rec + 32, blk.ncls, sVm, sVc, DO_M ? prm.out_m + blk.slot0 : nullptr,
                             DO_C ? prm.out_c + blk.slot0 : nullptr, tid, NCT);
        if (!a1_first && j + 1 < ncta_blocks) phase_a1(j + 1);
        tick(3);
        consumer_sync(NCT);  // V and the record stage of block j free; Lambda / W of block j + 1 ready
        tick(5);
        if (tid == 0) {
            mbar_arrive(&rdone[rs]);
            if (j + 1 < ncta_blocks) mbar_arrive(&gdone[(j + 1) & 1]);
        }
    }
#ifdef FEA5_DIAG
    if (prm.dbg && tid == 0)
        for (int i = 0; i < 6; ++i) atomicAdd(prm.dbg + i, tacc[i]);
#endif
}

using kfun_t = void (*)(const FeaKParams);

template <int P, int NQ_T>
kfun_t pick(int dm, int dc) {
    if (dm && dc) return k_reassemble<P, NQ_T, true, true>;
    if (dm) return k_reassemble<P, NQ_T, true, false>;
    return k_reassemble<P, NQ_T, false, true>;
}

kfun_t select(int order, int nq, int dm, int dc) {
    const bool nat = nq == fea_nq_native(order);
    switch (order) {
        case 1: return nat ? pick<1, 3>(dm, dc) : pick<1, 0>(dm, dc);
        case 2: return nat ? pick<2, 6>(dm, dc) : pick<2, 0>(dm, dc);
        case 3: return nat ? pick<3, 12>(dm, dc) : pick<3, 0>(dm, dc);
        case 4: return nat ? pick<4, 16>(dm, dc) : pick<4, 0>(dm, dc);
        default: return nullptr;
    }
}

int threads_of(int order) {
    switch (order) {
        case 1: return fea_threads(1);
        case 2: return fea_threads(2);
        case 3: return fea_threads(3);
        default: return fea_threads(4);
    }
}

}  // namespace

int fea_launch_reassemble(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream) {
    kfun_t kern = select(order, prm.nq, prm.out_m != nullptr, prm.out_c != nullptr);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, threads_of(order), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_kernel_occupancy(int order, int nq, int dm, int dc, int smem_bytes, int* n, int* threads) {
    kfun_t kern = select(order, nq, dm, dc);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = threads_of(order);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
