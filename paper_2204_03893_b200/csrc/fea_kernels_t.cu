// fea_kernels_t.cu -- sm_100a kernel for the tensor contractions of the Newton Jacobian
// (PAPER.md:280-349):
//
//   (M o2 v)_{ik} = sum_e sum_q w_q m'(u_q) phi_i phi_k (phi^T v_e)_q |det B_e|
//   (C o2 v)_{ik} = sum_e sum_q w_q c'(u_q) (J_q[i,:] A_e J_q^T v_e) phi_k |det B_e|
//
// the mass tensor M_ijk = int m' phi_i phi_j phi_k and the conductivity tensor
// C_ijk = int c' grad phi_i . grad phi_j phi_k contracted with v in their second mode,
// assembled with the same plan machinery as the matrices: lambda_q = w_q m'_q |det B_e| (times v_q
// for the mass tensor), then a small contraction per element, then the fixed-order scatter.
// (M o2 v) is symmetric (rows i <= k kept); (C o2 v) is NOT, so it
// keeps the entries i <= k (Vup) and i > k (Vdn) at the symmetric row index of (min, max), and the
// plan's contributor offsets carry an orientation bit (bit 15) choosing between them.
//
// k_tensor<P, NQ>: persistent CTAs (one per SM, FEA_T_WARPS warps), one lane per element, the
// reference tables (Phi, J, w) in shared memory; per block: all warps compute their 32-element
// tiles, CTA barrier, phase B (fea_device.cuh phase_b5 with orientation), CTA barrier.  The
// block record arrives by TMA during the element phase.
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_device.cuh"

namespace {
using namespace fea_dev;

template <int P, int NQ_T, bool DO_M, bool DO_C>
__global__ void __launch_bounds__(FEA_T_WARPS * 32, 1) k_tensor(const __grid_constant__ FeaTParams prm) {
    constexpr int NP = fea_np(P);
    constexpr int NQ = NQ_T > 0 ? NQ_T : 16;  // register arrays; the generic rule guards q < nq
    constexpr int NT = FEA_T_WARPS * 32;
    const int nq = NQ_T > 0 ? NQ_T : prm.nq;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vs = prm.e_max | 1;
    const int G = gridDim.x, b0 = blockIdx.x;
    const int nb = prm.nblocks > b0 ? (prm.nblocks - 1 - b0) / G + 1 : 0;

    extern __shared__ __align__(128) uint8_t smem[];
    double* sV1 = reinterpret_cast<double*>(smem + prm.lay[FEA_LT_V1]);
    double* sVu = reinterpret_cast<double*>(smem + prm.lay[FEA_LT_VUP]);
    double* sVd = reinterpret_cast<double*>(smem + prm.lay[FEA_LT_VDN]);
    uint8_t* sRec = smem + prm.lay[FEA_LT_REC];
    double* sTab = reinterpret_cast<double*>(smem + prm.lay[FEA_LT_TAB]);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA_LT_BAR]);
    const double* Phi = sTab;                 // [NP][16]
    const double* J0 = sTab + NP * 16;        // [NP][16]  d phi / d xhat
    const double* J1 = sTab + 2 * NP * 16;    // [NP][16]  d phi / d yhat
    const double* W = sTab + 3 * NP * 16;     // [16]

    for (int i = tid; i < 3 * NP * 16 + 16; i += NT) sTab[i] = prm.tab[i];
    if (tid == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    __syncthreads();

    for (int j = 0; j < nb; ++j) {
        const FeaBlock& blk = prm.blocks[b0 + j * G];
        if (tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(bar, (uint32_t)blk.rec_bytes);
            tma_load_1d(sRec, prm.records + blk.rec_off, (uint32_t)blk.rec_bytes, bar);
            if (j + 1 < nb) {
                const FeaBlock& nx = prm.blocks[b0 + (j + 1) * G];
                prefetch_l2(prm.records + nx.rec_off, (uint32_t)nx.rec_bytes);
            }
        }
        const int nE = blk.nE, nEp = fea_pad4(nE);
        for (int tile = warp; tile * 32 < nE; tile += FEA_T_WARPS) {
            const int le = tile * 32 + lane;
            if (le >= nE) continue;
            // ---- gathers (u_e, v_e, vertex coordinates)
            int d[NP];
            double ue[NP], ve[NP];
#pragma unroll
            for (int i = 0; i < NP; ++i) d[i] = prm.dofs[blk.dof_off + i * nEp + le];
#pragma unroll
            for (int i = 0; i < NP; ++i) FEA_CHECK(d[i] >= 0 && d[i] < prm.n_dof);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                ue[i] = __ldg(prm.u + d[i]);
                ve[i] = __ldg(prm.v + d[i]);
            }
            const double2 a = __ldg(prm.xy + d[0]), b = __ldg(prm.xy + d[1]), c = __ldg(prm.xy + d[2]);
            // ---- geometry
            const double B00 = b.x - a.x, B10 = b.y - a.y, B01 = c.x - a.x, B11 = c.y - a.y;
            const double det = B00 * B11 - B01 * B10;
            const double absdet = fabs(det);
            const double inv = 1.0 / (det * det);
            const double A00 = (B01 * B01 + B11 * B11) * inv;
            const double A11 = (B00 * B00 + B10 * B10) * inv;
            const double A01 = -(B00 * B01 + B10 * B11) * inv;
            // ---- per quadrature point: lambda (mass tensor: w m' v_q |det|), p = w c' |det| A_e J^T v_e
            double lam[NQ], p0[NQ], p1[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                lam[q] = p0[q] = p1[q] = 0.0;
                if (NQ_T == 0 && q >= nq) continue;
                double uq = 0.0, vq = 0.0, gx = 0.0, gy = 0.0;
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    uq = fma(Phi[i * 16 + q], ue[i], uq);
                    if (DO_M) vq = fma(Phi[i * 16 + q], ve[i], vq);
                    if (DO_C) {
                        gx = fma(J0[i * 16 + q], ve[i], gx);
                        gy = fma(J1[i * 16 + q], ve[i], gy);
                    }
                }
                const double wb = W[q] * absdet;
                if (DO_M) lam[q] = wb * dkeval(prm.coef_m, uq) * vq;
                if (DO_C) {
                    const double lc = wb * dkeval(prm.coef_c, uq);
                    p0[q] = lc * fma(A00, gx, A01 * gy);
                    p1[q] = lc * fma(A01, gx, A11 * gy);
                }
            }
            // ---- mass tensor contraction, symmetric rows i <= k: sum_q phi_i phi_k lam_q
            if (DO_M) {
#pragma unroll 1
                for (int k = 0; k < NP; ++k) {
                    double y[NQ];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) y[q] = Phi[k * 16 + q] * lam[q];
#pragma unroll 1
                    for (int i = 0; i <= k; ++i) {
                        double s = 0.0;
#pragma unroll
                        for (int q = 0; q < NQ; ++q) s = fma(Phi[i * 16 + q], y[q], s);
                        sV1[fea_trow(NP, i, k) * vs + le] = s;
                    }
                }
            }
            // ---- conductivity tensor contraction, all (i, k): sum_q (J_i . p_q) phi_k
            if (DO_C) {
#pragma unroll 1
                for (int i = 0; i < NP; ++i) {
                    double r[NQ];
#pragma unroll
                    for (int q = 0; q < NQ; ++q) r[q] = fma(J0[i * 16 + q], p0[q], J1[i * 16 + q] * p1[q]);
#pragma unroll 1
                    for (int k = 0; k < NP; ++k) {
                        double s = 0.0;
#pragma unroll
                        for (int q = 0; q < NQ; ++q) s = fma(r[q], Phi[k * 16 + q], s);
                        const int t = fea_trow(NP, min(i, k), max(i, k));
                        (i <= k ? sVu : sVd)[t * vs + le] = s;
                    }
                }
            }
        }
        __syncthreads();
        mbar_wait(bar, (uint32_t)(j & 1));
        phase_b5<DO_M, DO_C, true>(sRec, blk.ncls, sV1, sVu, DO_M ? prm.out_m + blk.slot0 : nullptr,
                                   DO_C ? prm.out_c + blk.slot0 : nullptr, tid, NT, sVd);
        __syncthreads();
    }
}

// ------------------------------------------------------------------ k_tensor4 (DMMA)
// The same two contractions as GEMMs on the FP64 tensor cores (mma.sync m8n8k4.f64), in the v4
// pipeline (fea_kernels.cu): a producer warp (TMA records, cp.async gathers of u, v and the vertex
// coordinates), then per block
//   A1  u_q, v_q = Phi^T (u_e, v_e), g_q = J_q^T v_e on DMMA, then per (q, e):
//       lambda_q = w_q |det B_e| m'(u_q) v_q, p_q = w_q |det B_e| c'(u_q) A_e g_q
//   A2  V1[t, e] = sum_q Q_m[t, q] lambda_qe                 (t = (i <= k); Q_m = Phi (.) Phi;
//                                                             stored at row fea_trow(i, k))
//       N[(i, k), e] = sum_d sum_q J_d,i(q) phi_k(q) p_dqe   (all (i, k); stored to Vup (i <= k) or
//                                                             Vdn (i > k) at row fea_trow(min, max))
//   B   phase_b5 with orientation (the plan's bit 15 picks Vup / Vdn).
// Software pipeline, two CTA barriers per block: A1(0) | for j: A2(j) | B(j) and A1(j + 1) |.
template <int P, int NQ_T, bool DO_M, bool DO_C>
__global__ void __launch_bounds__(fea_t4_threads(P, DO_M, DO_C), 1) k_tensor4(const __grid_constant__ FeaTParams prm) {
    constexpr int NP = fea_np(P), T = fea_T(P), NTT = fea_ntt(P), NTC = fea_ntc(P);
    constexpr int NK = NQ_T > 0 ? fea_nk(NQ_T) : fea_nk(FEA_MAX_NQ);
    constexpr int NQP = 4 * NK;
    constexpr int NTM = DO_M ? NTT : 0, NTCM = DO_C ? NTC : 0;
    constexpr int NG = fea_t4_ng(P, DO_M, DO_C), S = fea_t4_s(P, DO_M, DO_C);
    constexpr int RM = fea_t4_rm(P, DO_M, DO_C), RC = fea_t4_rc(P, DO_M, DO_C);
    constexpr int NCT = NG * S * 32;  // consumer threads
    const int nq = NQ_T > 0 ? NQ_T : prm.nq;
    const int e_max = prm.e_max, vs = fea4_vstride(e_max), ls = fea4_lstride(e_max);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const bool producer = tid >= NCT;

    extern __shared__ __align__(128) uint8_t smem[];
    auto sRec = [&](int s) { return smem + prm.lay[FEA_LT4_REC + s]; };
    auto gUb = [&](int s) { return reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_GU + s]); };
    auto gVb = [&](int s) { return reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_GV + s]); };
    auto gXb = [&](int s) { return reinterpret_cast<double2*>(smem + prm.lay[FEA_LT4_GX + s]); };
    double* sLm = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_LM]);
    double* sP0 = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_P0]);
    double* sP1 = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_P1]);
    double* sTab = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_TAB]);
    double* sV1 = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_V1]);
    double* sVu = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_VUP]);
    double* sVd = reinterpret_cast<double*>(smem + prm.lay[FEA_LT4_VDN]);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA_LT4_BARS]);
    uint64_t* full_rec = bars;      // [2] record landed (TMA transactions)
    uint64_t* full_gat = bars + 2;  // [2] gathers landed (32 producer lanes)
    uint64_t* rdone = bars + 4;     // [2] consumers finished with the record stage
    uint64_t* gdone = bars + 6;     // [2] consumers finished with the gather stage
    const int ncta_blocks = prm.nblocks > (int)blockIdx.x ? (prm.nblocks - 1 - (int)blockIdx.x) / (int)gridDim.x + 1 : 0;

    for (int i = tid; i < 3 * NP * 16 + 16; i += blockDim.x) sTab[i] = prm.tab[i];
    // V1 row of the Q_m fragment row t (tri order i <= k) -> fea_trow
    __shared__ int sTrow[T];
    for (int lo = 0; lo < NP; ++lo)
        for (int hi = lo; hi < NP; ++hi)
            if (tid == 0) sTrow[lo * NP - lo * (lo - 1) / 2 + (hi - lo)] = fea_trow(NP, lo, hi);
    if (tid == 0) {
        for (int s = 0; s < 2; ++s) {
            mbar_init(&full_rec[s], 1);
            mbar_init(&rdone[s], 1);
            mbar_init(&full_gat[s], 32);
            mbar_init(&gdone[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (producer) {
        auto issue_rec = [&](int jj) {
            const FeaBlock b = prm.blocks[blockIdx.x + jj * gridDim.x];
            const int s = jj & 1;
            fence_proxy_async();
            mbar_expect_tx(&full_rec[s], (uint32_t)b.rec_bytes);
            tma_load_1d(sRec(s), prm.records + b.rec_off, (uint32_t)b.rec_bytes, &full_rec[s]);
        };
        if (lane == 0 && ncta_blocks > 0) issue_rec(0);
        for (int j = 0; j < ncta_blocks; ++j) {
            const int s = j & 1;
            if (j >= 2) mbar_wait(&gdone[s], (uint32_t)(((j >> 1) - 1) & 1));  // stage free (block j-2)
            mbar_wait(&full_rec[s], (uint32_t)((j >> 1) & 1));                   // record j landed
            const FeaRecHdr4 blk = *reinterpret_cast<const FeaRecHdr4*>(sRec(s));
            const int nEp = fea_pad4(blk.nE);
            const int32_t* gd = reinterpret_cast<const int32_t*>(sRec(s) + blk.dofs_off);
            double* gu = gUb(s);
            double* gv = gVb(s);
            double2* gx = gXb(s);
            for (int le = lane; le < blk.nE; le += 32) {
#pragma unroll
                for (int i = 0; i < NP; ++i) {
                    const int d = gd[i * nEp + le];
                    FEA_CHECK(d >= 0 && d < prm.n_dof);
                    cp_async8(gu + i * ls + le, prm.u + d);
                    cp_async8(gv + i * ls + le, prm.v + d);
                }
#pragma unroll
                for (int v = 0; v < 3; ++v) cp_async16(gx + v * e_max + le, prm.xy + gd[v * nEp + le]);
            }
            cp_async_mbar_arrive(&full_gat[s]);
            // record of block j + 1 into the other stage once block j - 1 is done with it
            if (j + 1 < ncta_blocks) {
                if (j >= 1) mbar_wait(&rdone[(j - 1) & 1], (uint32_t)(((j - 1) >> 1) & 1));
                if (lane == 0) issue_rec(j + 1);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    // ------------------------------------------------------------------ consumers
    const int gi = warp % NG, sub = warp / NG;
    const int g = lane >> 2, cq = lane & 3;
    // this warp's row tiles (gi, gi + NG, ...) as DMMA A-fragments for the whole kernel
    double am[RM > 0 ? RM : 1][NK], ac[RC > 0 ? RC : 1][2][NK];
    constexpr int ROFF = fea_rfrag_off(P, NK);
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
#pragma unroll
        for (int r = 0; r < RM; ++r) {
            const int tile = gi + r * NG;
            am[r][kk] = tile < NTM ? __ldg(prm.qfrag + (tile * NK + kk) * 32 + lane) : 0.0;
        }
#pragma unroll
        for (int r = 0; r < RC; ++r) {
            const int ct = gi + r * NG;
#pragma unroll
            for (int d = 0; d < 2; ++d)
                ac[r][d][kk] = ct < NTCM ? __ldg(prm.qfrag + ROFF + ((ct * 2 + d) * NK + kk) * 32 + lane) : 0.0;
        }
    }
    const double* Phi = sTab;              // [NP][16]
    const double* J0 = sTab + NP * 16;     // [NP][16]
    const double* J1 = sTab + 2 * NP * 16; // [NP][16]
    const double* W = sTab + 3 * NP * 16;  // [16]

    auto phase_a1 = [&](int j) {
        const int s = j & 1;
        const double* gU = gUb(s);
        const double* gV = gVb(s);
        const double2* gX = gXb(s);
        mbar_wait(&full_rec[s], (uint32_t)((j >> 1) & 1));
        const int nE = reinterpret_cast<const FeaRecHdr4*>(sRec(s))->nE;
        const int net = (nE + 7) >> 3;
        mbar_wait(&full_gat[s], (uint32_t)((j >> 1) & 1));
        // interpolation on DMMA: [u_q; v_q; gx_q; gy_q] = [Phi^T; Phi^T; J0^T; J1^T] [u_e | v_e], unit =
        // (q-tile mt, element tile et); A-fragments straight from the tables (Tab[i][q], i = 4 kt + c,
        // q = 8 mt + g), B-fragments from the gathers; epilogue per accumulator (q, e): geometry,
        // k'(u_q), lambda_q, p_q.
        constexpr int MT = (NQP + 7) / 8, KT = fea_kt(P);
        for (int un = warp; un < MT * net; un += NG * S) {
            const int mt = un % MT, et = un / MT;
            double u0 = 0.0, u1 = 0.0, v0 = 0.0, v1 = 0.0, x0 = 0.0, x1 = 0.0, y0 = 0.0, y1 = 0.0;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                const int i = kt * 4 + cq, qa = mt * 8 + g;
                const bool ok = i < NP;
                const double bu = ok ? gU[i * ls + et * 8 + g] : 0.0;
                const double bv = ok ? gV[i * ls + et * 8 + g] : 0.0;
                const double aphi = ok ? Phi[i * 16 + qa] : 0.0;
                dmma(u0, u1, aphi, bu);
                if (DO_M) dmma(v0, v1, aphi, bv);
                if (DO_C) {
                    dmma(x0, x1, ok ? J0[i * 16 + qa] : 0.0, bv);
                    dmma(y0, y1, ok ? J1[i * 16 + qa] : 0.0, bv);
                }
            }
            const int q = mt * 8 + g, le0 = et * 8 + 2 * cq;
            if (q < NQP) {
                double lm[2] = {0.0, 0.0}, p0[2] = {0.0, 0.0}, p1[2] = {0.0, 0.0};
                // k'(u_q) of both accumulator columns at once (values of columns past nE are unused)
                const double uqs[2] = {u0, u1};
                double dms[2], dcs[2];
                if (DO_M) dkeval_all<2>(prm.coef_m, uqs, dms);
                if (DO_C) {
                    if (DO_M && prm.same_coef) {
                        dcs[0] = dms[0];
                        dcs[1] = dms[1];
                    } else {
                        dkeval_all<2>(prm.coef_c, uqs, dcs);
                    }
                }
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int le = le0 + h;
                    if (le < nE && q < nq) {
                        double absdet, A00, A11, A01;
                        geometry(gX, e_max, le, absdet, A00, A11, A01);
                        const double wb = W[q] * absdet;
                        const double dm = DO_M ? dms[h] : 0.0;
                        if (DO_M) lm[h] = wb * dm * (h ? v1 : v0);
                        if (DO_C) {
                            const double dc = dcs[h];
                            const double lc = wb * dc, gx = h ? x1 : x0, gy = h ? y1 : y0;
                            p0[h] = lc * fma(A00, gx, A01 * gy);
                            p1[h] = lc * fma(A01, gx, A11 * gy);
                        }
                    }
                }
                if (DO_M) *reinterpret_cast<double2*>(sLm + q * ls + le0) = make_double2(lm[0], lm[1]);
                if (DO_C) {
                    *reinterpret_cast<double2*>(sP0 + q * ls + le0) = make_double2(p0[0], p0[1]);
                    *reinterpret_cast<double2*>(sP1 + q * ls + le0) = make_double2(p1[0], p1[1]);
                }
            }
        }
    };

    if (ncta_blocks > 0) {
        phase_a1(0);
        consumer_sync(NCT);
        if (tid == 0) mbar_arrive(&gdone[0]);
    }
    for (int j = 0; j < ncta_blocks; ++j) {
        const int s = j & 1;
        const uint8_t* rec = sRec(s);
        const FeaRecHdr4 blk = *reinterpret_cast<const FeaRecHdr4*>(rec);
        const int net = (blk.nE + 7) >> 3;
        // ---------------- A2 on the FP64 tensor cores
        for (int et = sub; et < net; et += S) {
            const int col = et * 8 + g;       // B fragment column (element) of this lane
            const int le0 = et * 8 + 2 * cq;  // the two accumulator columns of this lane
            double bm[NK], b0[NK], b1[NK];
#pragma unroll
            for (int kk = 0; kk < NK; ++kk) {
                const int o = (kk * 4 + cq) * ls + col;
                bm[kk] = DO_M ? sLm[o] : 0.0;
                b0[kk] = DO_C ? sP0[o] : 0.0;
                b1[kk] = DO_C ? sP1[o] : 0.0;
            }
#pragma unroll
            for (int r = 0; r < RM; ++r) {
                const int tile = gi + r * NG, t = tile * 8 + g;
                if (tile >= NTM) continue;
                double x0 = 0.0, x1 = 0.0;
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) dmma(x0, x1, am[r][kk], bm[kk]);
                if (t < T) *reinterpret_cast<double2*>(sV1 + sTrow[t] * vs + le0) = make_double2(x0, x1);
            }
#pragma unroll
            for (int r = 0; r < RC; ++r) {
                const int ct = gi + r * NG, rr = ct * 8 + g;
                if (ct >= NTCM) continue;
                double x0 = 0.0, x1 = 0.0;
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) {
                    dmma(x0, x1, ac[r][0][kk], b0[kk]);
                    dmma(x0, x1, ac[r][1][kk], b1[kk]);
                }
                if (rr < NP * NP) {
                    const int i = rr / NP, k = rr - i * NP;
                    const int t = fea_trow(NP, min(i, k), max(i, k));
                    *reinterpret_cast<double2*>((i <= k ? sVu : sVd) + t * vs + le0) = make_double2(x0, x1);
                }
            }
        }
        consumer_sync(NCT);  // V complete; Lambda / p free
        // ---------------- B(j) and A1(j + 1), in alternating order across warps
        const bool a1_first = (warp & 1) && j + 1 < ncta_blocks;
        if (a1_first) phase_a1(j + 1);
        phase_b5<DO_M, DO_C, true>(rec + 32, blk.ncls, sV1, sVu, DO_M ? prm.out_m + blk.slot0 : nullptr,
                                   DO_C ? prm.out_c + blk.slot0 : nullptr, tid, NCT, sVd);
        if (!a1_first && j + 1 < ncta_blocks) phase_a1(j + 1);
        consumer_sync(NCT);
        if (tid == 0) {
            mbar_arrive(&rdone[s]);
            if (j + 1 < ncta_blocks) mbar_arrive(&gdone[(j + 1) & 1]);
        }
    }
}

using tfun_t = void (*)(const FeaTParams);

template <int P, int NQ>
tfun_t pick_t(int kver, int dm, int dc) {
    if (kver == 4) {
        if (dm && dc) return k_tensor4<P, NQ, true, true>;
        if (dm) return k_tensor4<P, NQ, true, false>;
        return k_tensor4<P, NQ, false, true>;
    }
    if (dm && dc) return k_tensor<P, NQ, true, true>;
    if (dm) return k_tensor<P, NQ, true, false>;
    return k_tensor<P, NQ, false, true>;
}

tfun_t select_t(int order, int nq, int kver, int dm, int dc) {
    const bool nat = nq == fea_nq_native(order);
    switch (order) {
        case 1: return nat ? pick_t<1, 3>(kver, dm, dc) : pick_t<1, 0>(kver, dm, dc);
        case 2: return nat ? pick_t<2, 6>(kver, dm, dc) : pick_t<2, 0>(kver, dm, dc);
        case 3: return nat ? pick_t<3, 12>(kver, dm, dc) : pick_t<3, 0>(kver, dm, dc);
        case 4: return nat ? pick_t<4, 16>(kver, dm, dc) : pick_t<4, 0>(kver, dm, dc);
        default: return nullptr;
    }
}

int threads_t(int order, int kver, int dm, int dc) {
    if (kver != 4) return FEA_T_WARPS * 32;
    const bool m = dm != 0, c = dc != 0;
    switch (order) {
        case 1: return fea_t4_threads(1, m, c);
        case 2: return fea_t4_threads(2, m, c);
        case 3: return fea_t4_threads(3, m, c);
        default: return fea_t4_threads(4, m, c);
    }
}

}  // namespace

int fea_launch_tensor(const FeaTParams& prm, int order, int smem_bytes, int grid, void* stream) {
    const int dm = prm.out_m != nullptr, dc = prm.out_c != nullptr;
    tfun_t kern = select_t(order, prm.nq, prm.kver, dm, dc);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, threads_t(order, prm.kver, dm, dc), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_tensor_occupancy(int order, int nq, int kver, int smem_bytes, int* n, int* threads) {
    tfun_t kern = select_t(order, nq, kver, 1, 1);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = threads_t(order, kver, 1, 1);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
