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
                        sV1[(i * NP - i * (i - 1) / 2 + (k - i)) * vs + le] = s;
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
                        const int lo = min(i, k), hi = max(i, k);
                        const int t = lo * NP - lo * (lo - 1) / 2 + (hi - lo);
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

using tfun_t = void (*)(const FeaTParams);

template <int P, int NQ>
tfun_t pick_t(int dm, int dc) {
    if (dm && dc) return k_tensor<P, NQ, true, true>;
    if (dm) return k_tensor<P, NQ, true, false>;
    return k_tensor<P, NQ, false, true>;
}

tfun_t select_t(int order, int nq, int dm, int dc) {
    const bool nat = nq == fea_nq_native(order);
    switch (order) {
        case 1: return nat ? pick_t<1, 3>(dm, dc) : pick_t<1, 0>(dm, dc);
        case 2: return nat ? pick_t<2, 6>(dm, dc) : pick_t<2, 0>(dm, dc);
        case 3: return nat ? pick_t<3, 12>(dm, dc) : pick_t<3, 0>(dm, dc);
        case 4: return nat ? pick_t<4, 16>(dm, dc) : pick_t<4, 0>(dm, dc);
        default: return nullptr;
    }
}

}  // namespace

int fea_launch_tensor(const FeaTParams& prm, int order, int smem_bytes, int grid, void* stream) {
    tfun_t kern = select_t(order, prm.nq, prm.out_m != nullptr, prm.out_c != nullptr);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, FEA_T_WARPS * 32, smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_tensor_occupancy(int order, int smem_bytes, int* n, int* threads) {
    tfun_t kern = select_t(order, fea_nq_native(order), 1, 1);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = FEA_T_WARPS * 32;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
