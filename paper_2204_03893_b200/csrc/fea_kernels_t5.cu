// fea_kernels_t5.cu -- sm_100a kernel for the tensor contractions of the Newton Jacobian on P1
// with its native 3-point rule:
//
//   (M o2 v)_{ik} = sum_e sum_q w_q m'(u_q) phi_i phi_k (phi^T v_e)_q |det B_e|
//   (C o2 v)_{ik} = sum_e sum_q w_q c'(u_q) (J_q[i,:] A_e J_q^T v_e) phi_k |det B_e|
//
// k_tensor5<P, NQ, DO_M, DO_C>: the per-element arithmetic of k_tensor (fea_kernels_t.cu; the same
// operations in the same order, so the values are bit-identical) in the software pipeline of the
// matrix kernel v5 (fea_kernels5.cu):
//   - one persistent CTA per SM, NW warps, no producer warp and no CTA-wide barrier in the loop;
//   - V (V1 = (M o2 v) rows i <= k; Vup / Vdn = (C o2 v) entries i <= k / i > k, all at the row
//     fea_trow(min, max)) and the block records are DOUBLE BUFFERED, and every warp runs
//         step s:  [A] its 32-element tiles of block s -> V[s & 1]      (arrive full[s & 1])
//                  [B] its share of block s - 1 from V[(s-1) & 1]      (arrive free[(s-1) & 1])
//     so the contraction of one block overlaps the scatter of the previous one across warps;
//   - the gathers (DOFs, u_e, v_e, vertex coordinates) of the next tile are in registers while the
//     current one is computed; records / DOF arrays / the rows' u, v, xy are L2-prefetched blocks ahead;
//   - Phi, w and J are constant-bank DFMA operands (kernel parameters, FeaTParams::ctab / jtab, the
//     matrix kernel v5's table layout);
//   - phase B: phase_b5 with orientation (bit 15 of a contributor offset picks Vdn), every CSR slot
//     the sum of its contributors in ascending library element order (deterministic).
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_device.cuh"

namespace {
using namespace fea_dev;

template <int NP>
struct GathT {  // gathered inputs of one lane's element
    double u[NP], v[NP];
    double2 x[3];
};

template <int P, int NQ, bool DO_M, bool DO_C>
__global__ void __launch_bounds__(fea_t5_threads(P), 1) k_tensor5(const __grid_constant__ FeaTParams prm) {
    constexpr int NP = fea_np(P);
    constexpr int NW = fea_t5_nw(P);
    constexpr int PF = 3;  // L2 prefetch distance (blocks)
    constexpr int DR = 8;  // descriptor ring
    static_assert(2 * NP * NQ <= FEA_JTAB_MAX && NP * NQ + NQ <= FEA_CTAB_MAX, "tables exceed the parameter bank");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int vs = prm.e_max | 1;
    const int G = gridDim.x, b0 = blockIdx.x;
    const int nb = prm.nblocks > b0 ? (prm.nblocks - 1 - b0) / G + 1 : 0;

    extern __shared__ __align__(128) uint8_t smem[];
    double* const sV0 = reinterpret_cast<double*>(smem + prm.lay[FEA_LT5_V]);  // [2][vbuf]
    const int vbuf = prm.lay[FEA_LT5_VBUF];
    const int o1 = prm.lay[FEA_LT5_O1], ou = prm.lay[FEA_LT5_OU], od = prm.lay[FEA_LT5_OD];
    uint8_t* const sRec0 = smem + prm.lay[FEA_LT5_REC];  // [2][rec_stride]
    const int rec_stride = prm.lay[FEA_LT5_RS];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA_LT5_BARS]);
    uint64_t* full = bars;       // [2] NW arrivals: all tiles of the buffer's block computed
    uint64_t* freeb = bars + 2;  // [2] NW arrivals: phase B of the buffer's block done
    uint64_t* recb = bars + 4;   // [2] TMA transactions of the buffer's record
    FeaBlock* sBlk = reinterpret_cast<FeaBlock*>(smem + prm.lay[FEA_LT5_RING]);

    // descriptor ring: as kernel v5 (fea_kernels5.cu): blocks < win are readable from shared memory
    int win = 6;
    auto blk_of = [&](int k) -> const FeaBlock& { return k < win ? sBlk[k & (DR - 1)] : prm.blocks[b0 + k * G]; };
    auto prefetch_range = [&](const void* p, size_t bytes) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
        if (e > a) prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(e - a));
    };
    auto prefetch_blk = [&](int k) {  // thread 0 only
        const FeaBlock& b = sBlk[k & (DR - 1)];
        prefetch_range(prm.records + b.rec_off, (size_t)b.rec_bytes);
        prefetch_range(prm.dofs + b.dof_off, (size_t)4 * NP * fea_pad4(b.nE));
        prefetch_range(prm.u + b.r0, (size_t)8 * b.nr);
        prefetch_range(prm.v + b.r0, (size_t)8 * b.nr);
        prefetch_range(prm.xy + b.r0, (size_t)16 * b.nr);
    };

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], NW);
            mbar_init(&freeb[b], NW);
            mbar_init(&recb[b], 1);
        }
        fence_mbar_init();
    }
    if (tid < 6 && tid < nb) sBlk[tid] = prm.blocks[b0 + tid * G];
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < PF && k < nb; ++k) prefetch_blk(k);

    // ---- tile stream cursors: block k of this CTA, 32-element tile t of the block; the block's
    // element count and DOF offset are kept in registers (read from the ring once per block: the
    // compiler cannot keep shared-memory values across the V stores)
    struct Cur {
        int k, t, nE;
        int64_t doff;
    };
    auto enter = [&](Cur& c) {
        if (c.k < nb) {
            const FeaBlock& b = blk_of(c.k);
            c.nE = b.nE;
            c.doff = b.dof_off;
        }
    };
    auto settle = [&](Cur& c) {
        while (c.k < nb && c.t * 32 >= c.nE) {
            ++c.k;
            c.t = warp;
            enter(c);
        }
    };
    auto advance = [&](Cur& c) {
        c.t += NW;
        settle(c);
    };
    Cur cc{0, warp, 0, 0};  // compute cursor
    enter(cc);
    settle(cc);
    Cur lc = cc;  // load cursor
    int dof[NP];
    auto load_dofs = [&]() {
        const int le = lc.t * 32 + lane;
        if (le < lc.nE) {
            const int32_t* d = prm.dofs + lc.doff + le;
            const int nEp = fea_pad4(lc.nE);
#pragma unroll
            for (int i = 0; i < NP; ++i) dof[i] = ldg_s32(d + i * nEp);
        }
    };
    auto refill = [&](GathT<NP>& g) {
        if (lc.k >= nb) return;
        if (lc.t * 32 + lane < lc.nE) {
#pragma unroll
            for (int i = 0; i < NP; ++i) FEA_CHECK(dof[i] >= 0 && dof[i] < prm.n_dof);
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                g.u[i] = ldg_f64(prm.u + dof[i]);
                g.v[i] = ldg_f64(prm.v + dof[i]);
            }
#pragma unroll
            for (int v = 0; v < 3; ++v) g.x[v] = ldg_f64x2(prm.xy + dof[v]);
        }
        advance(lc);
        if (lc.k < nb) load_dofs();
    };

    // ---- A: one element per lane (k_tensor's arithmetic, operands from the constant bank)
    auto Phi = [&](int k, int q) { return prm.ctab[k * NQ + q]; };
    auto Wq = [&](int q) { return prm.ctab[((NP * NQ + 1) & ~1) + q]; };  // w at pad2(np nq)
    auto J = [&](int a, int k, int q) { return prm.jtab[(a * NP + k) * NQ + q]; };
    auto compute = [&](const GathT<NP>& g, double* sV, int le) {
        FEA_CHECK(le < prm.e_max);  // V column inside the buffer (rows < T, T - np: by construction)
        const double2* gx = g.x;
        const double B00 = gx[1].x - gx[0].x, B10 = gx[1].y - gx[0].y;
        const double B01 = gx[2].x - gx[0].x, B11 = gx[2].y - gx[0].y;
        const double det = B00 * B11 - B01 * B10;
        const double absdet = fabs(det);
        const double inv = 1.0 / (det * det);
        const double A00 = (B01 * B01 + B11 * B11) * inv;
        const double A11 = (B00 * B00 + B10 * B10) * inv;
        const double A01 = -(B00 * B01 + B10 * B11) * inv;
        // per quadrature point: lambda = w m'(u_q) |det| v_q, p = w c'(u_q) |det| A_e J_q^T v_e
        double uq[NQ], vq[NQ], gxq[NQ], gyq[NQ], dm[NQ], dc[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            uq[q] = vq[q] = gxq[q] = gyq[q] = 0.0;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                uq[q] = fma(Phi(i, q), g.u[i], uq[q]);
                if (DO_M) vq[q] = fma(Phi(i, q), g.v[i], vq[q]);
                if (DO_C) {
                    gxq[q] = fma(J(0, i, q), g.v[i], gxq[q]);
                    gyq[q] = fma(J(1, i, q), g.v[i], gyq[q]);
                }
            }
        }
        if (DO_M) dkeval_all<NQ>(prm.coef_m, uq, dm);
        if (DO_C) {
            if (DO_M && prm.same_coef) {
#pragma unroll
                for (int q = 0; q < NQ; ++q) dc[q] = dm[q];
            } else {
                dkeval_all<NQ>(prm.coef_c, uq, dc);
            }
        }
        double lam[NQ], p0[NQ], p1[NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const double wb = Wq(q) * absdet;
            if (DO_M) lam[q] = wb * dm[q] * vq[q];
            if (DO_C) {
                const double lcq = wb * dc[q];
                p0[q] = lcq * fma(A00, gxq[q], A01 * gyq[q]);
                p1[q] = lcq * fma(A01, gxq[q], A11 * gyq[q]);
            }
        }
        if (DO_M) {  // symmetric rows i <= k: sum_q phi_i phi_k lambda_q
            double* sV1 = sV + o1;
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                double y[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) y[q] = Phi(k, q) * lam[q];
#pragma unroll
                for (int i = 0; i <= k; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) s = fma(Phi(i, q), y[q], s);
                    sV1[fea_trow(NP, i, k) * vs + le] = s;
                }
            }
        }
        if (DO_C) {  // all (i, k): sum_q (J_i . p_q) phi_k
            double* sVu = sV + ou;
            double* sVd = sV + od;
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                double r[NQ];
#pragma unroll
                for (int q = 0; q < NQ; ++q) r[q] = fma(J(0, i, q), p0[q], J(1, i, q) * p1[q]);
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    double s = 0.0;
#pragma unroll
                    for (int q = 0; q < NQ; ++q) s = fma(r[q], Phi(k, q), s);
                    (i <= k ? sVu : sVd)[fea_trow(NP, i < k ? i : k, i < k ? k : i) * vs + le] = s;
                }
            }
        }
    };

    // ---- prologue: DOFs of the first tile, then two tiles of gathers in flight
    GathT<NP> ga, gb;
    if (lc.k < nb) load_dofs();
    refill(ga);
    refill(gb);

    for (int s = 0; s <= nb; ++s) {
        win = max(s + 4, 6);  // ring entries published by the full barrier of step s - 1
        if (s < nb) {
            const int b = s & 1;
            if (s >= 2) mbar_wait(&freeb[b], (uint32_t)(((s - 2) >> 1) & 1));  // B of block s - 2 done
            if (tid == 0) {
                asm volatile("cp.async.wait_all;" ::: "memory");  // ring entry of block s + 5
                const FeaBlock& bk = sBlk[s & (DR - 1)];
                FEA_CHECK(bk.rec_bytes <= rec_stride && bk.nE <= prm.e_max);
                fence_proxy_async();
                mbar_expect_tx(&recb[b], (uint32_t)bk.rec_bytes);
                tma_load_1d(sRec0 + b * rec_stride, prm.records + bk.rec_off, (uint32_t)bk.rec_bytes, &recb[b]);
                if (s + 6 < nb) {  // slot of block s - 2, whose phase B is done
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(prm.blocks + b0 + (s + 6) * G);
                    uint8_t* dst = reinterpret_cast<uint8_t*>(sBlk + ((s + 6) & (DR - 1)));
#pragma unroll
                    for (int w = 0; w < 4; ++w) cp_async16(dst + 16 * w, src + 16 * w);
                    asm volatile("cp.async.commit_group;" ::: "memory");
                }
                if (s + PF < nb) prefetch_blk(s + PF);
            }
            double* sV = sV0 + b * vbuf;
            while (cc.k == s) {
                const int le = cc.t * 32 + lane;
                if (le < cc.nE) compute(ga, sV, le);
                ga = gb;
                refill(gb);
                advance(cc);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[b]);
        }
        if (s >= 1) {
            const int s1 = s - 1, b = s1 & 1;
            mbar_wait(&full[b], (uint32_t)((s1 >> 1) & 1));
            win = max(s + 5, 6);
            mbar_wait(&recb[b], (uint32_t)((s1 >> 1) & 1));
            const FeaBlock& bk = blk_of(s1);
            const double* sV = sV0 + b * vbuf;
            phase_b5<DO_M, DO_C, true>(sRec0 + b * rec_stride, bk.ncls, sV + o1, sV + ou,
                                       DO_M ? prm.out_m + bk.slot0 : nullptr, DO_C ? prm.out_c + bk.slot0 : nullptr,
                                       tid, NW * 32, sV + od);
            __syncwarp();
            if (lane == 0) mbar_arrive(&freeb[b]);
        }
    }
}

using tfun_t = void (*)(const FeaTParams);

tfun_t select_t5(int order, int nq, int dm, int dc) {
    if (!fea_t5_supported(order, nq)) return nullptr;
    if (dm && dc) return k_tensor5<1, 3, true, true>;
    if (dm) return k_tensor5<1, 3, true, false>;
    return k_tensor5<1, 3, false, true>;
}

}  // namespace

int fea_launch_tensor5(const FeaTParams& prm, int order, int smem_bytes, int grid, void* stream) {
    tfun_t kern = select_t5(order, prm.nq, prm.out_m != nullptr, prm.out_c != nullptr);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, fea_t5_threads(order), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_tensor_occupancy5(int order, int nq, int smem_bytes, int* n, int* threads) {
    tfun_t kern = select_t5(order, nq, 1, 1);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = fea_t5_threads(order);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
