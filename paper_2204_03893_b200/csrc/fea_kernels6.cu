// fea_kernels6.cu -- sm_100a reassembly kernel v6 for P3 / P4 with the configs' native rules
// (12 / 16 points; the C3 and C5 kernel).  Other (order, rule) pairs run v5
// (p <= 2) or v4 (generic rules).
//
// k_reassemble6<P, DO_M, DO_C>: one persistent CTA per SM, warp-specialised, no CTA-wide barrier.
// The CTA walks its row blocks j = 0, 1, ... (FeaBlock, grid-strided).
//
//   PRODUCER warp: the block's element DOFs (global, SoA) -> cp.async gathers of u(N_e) and the
//     vertex coordinates into gather stage j & 1 (Algorithm 2 line 4 inputs, PAPER.md:241;
//     u_e = u[N_e]), completion on an mbarrier; L2 prefetch of the DOFs and
//     the phase-B record two blocks ahead.
//   A warps (NA), per block j:
//     A1 (lines 5-9) on DMMA: U = Phi^T U_e, epilogue per (q, e):
//          b_e = |det B_e|, W_e = vec A_e, A_e = (B_e^T B_e)^{-1}
//          Lambda_qe = w_q k(u_qe) b_e
//        into Lambda / W buffer j & 1; one named barrier of the A warps;
//     A2 (lines 10-11) on DMMA (mma.sync m8n8k4 f64): V_m = Q_m Lambda,
//          V_c = sum_f W_f (Q_c,f Lambda) for the symmetric rows t = (i <= j) only,
//          each warp holding RT row tiles of Q_f as A-fragments in registers, into V buffer j & 1
//          ({m, c} cells), after the B warps released that buffer (block j - 2).
//   B warps (NB), per block j, once every A warp stored its tiles of V (j & 1):
//     B (line 12): every CSR slot = the sum of its contributors in ascending
//          library element order (no atomics).  Class A (<= 2 contributors, >= 99 % of the slots
//          for P3 / P4): lane l of a warp takes slot 32 k + l, reads one u32 item (coalesced,
//          global), two {m, c} cells, and stores contiguous CSR values; class B (more
//          contributors: vertex diagonals) uses the v5 item code.
//   So the FP64 contraction of block j + 1 (DMMA pipe) overlaps the scatter of block j (LSU).
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_device.cuh"

namespace {
using namespace fea_dev;

__device__ __forceinline__ uint32_t ldg_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int P, bool DO_M, bool DO_C>
__global__ void __launch_bounds__(fea6_threads(P), 1) k_reassemble6(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = fea_np(P), T = fea_T(P), NTT = fea_ntt(P);
    constexpr int NQ = fea_nq_native(P), NK = fea_nk(NQ), NQP = 4 * NK;
    constexpr int NA = fea6_na(P), RT = fea6_rt(P), NB = FEA6_NB;
    constexpr int MT = (NQP + 7) / 8, KT = fea_kt(P);
    constexpr bool IL = DO_M && DO_C;  // {m, c} cells
    constexpr int oW = (NP * NQ + 1) & ~1;
    static_assert(NA * RT >= NTT, "row tiles");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int e_max = prm.e_max, ls = fea6_lstride(e_max), vs = fea6_vstride(e_max);
    const int G = gridDim.x, b0 = blockIdx.x;
    const int nb = prm.nblocks > b0 ? (prm.nblocks - 1 - b0) / G + 1 : 0;

    extern __shared__ __align__(128) uint8_t smem[];
    auto sV = [&](int b) { return smem + prm.lay[FEA6_L_V] + b * prm.lay[FEA6_L_VB]; };
    auto sGU = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_GU] + b * prm.lay[FEA6_L_GUB]); };
    auto sGX = [&](int b) { return reinterpret_cast<double2*>(smem + prm.lay[FEA6_L_GX] + b * prm.lay[FEA6_L_GXB]); };
    auto sLam = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_LAM] + b * prm.lay[FEA6_L_LAMB]); };
    auto sW = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_W] + b * prm.lay[FEA6_L_WB]); };
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA6_L_BARS]);
    uint64_t* gat_full = bars;      // [2] 32 producer lanes (cp.async completion)
    uint64_t* gat_free = bars + 2;  // [2] 1 arrival: the A warps are done with the gather stage
    uint64_t* v_full = bars + 4;    // [2] NA * 32 arrivals: V of the buffer's block stored
    uint64_t* v_free = bars + 6;    // [2] NB * 32 arrivals: phase B of the buffer's block done

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&gat_full[b], 32);
            mbar_init(&gat_free[b], 1);
            mbar_init(&v_full[b], NA * 32);
            mbar_init(&v_free[b], NB * 32);
        }
        fence_mbar_init();
    }
    if (tid < 6) {  // the zero cell (row 0, column e_max) of both V buffers: double e_max (8-byte
                    // cells) and doubles 2 e_max, 2 e_max + 1 ({m, c} cells); A2 never writes it
        const int k = tid % 3;
        reinterpret_cast<double*>(sV(tid / 3))[k == 0 ? e_max : 2 * e_max + k - 1] = 0.0;
    }
    __syncthreads();

    if (warp == NA + NB) {
        // ------------------------------------------------------------------ producer
        auto prefetch_range = [&](const void* p, size_t bytes) {
            const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
            const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
            if (e > a) prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(e - a));
        };
        auto prefetch_blk = [&](int k) {
            const FeaBlock* B = prm.blocks + b0 + k * G;
            const int nE = __ldg(&B->nE);
            prefetch_range(prm.dofs + __ldg(&B->dof_off), (size_t)4 * NP * fea_pad4(nE));
            prefetch_range(prm.records + __ldg(&B->rec_off), (size_t)__ldg(&B->rec_bytes));
        };
        if (lane == 0)
            for (int k = 0; k < 2 && k < nb; ++k) prefetch_blk(k);
        for (int j = 0; j < nb; ++j) {
            const int g = j & 1;
            if (lane == 0 && j + 2 < nb) prefetch_blk(j + 2);
            if (j >= 2) mbar_wait(&gat_free[g], (uint32_t)(((j >> 1) - 1) & 1));
            const FeaBlock* B = prm.blocks + b0 + j * G;
            const int nE = __ldg(&B->nE), nEp = fea_pad4(nE);
            const int32_t* gd = prm.dofs + __ldg(&B->dof_off);
            double* gu = sGU(g);
            double2* gx = sGX(g);
            for (int le = lane; le < nE; le += 32) {
                int32_t d[NP];
#pragma unroll
                for (int i = 0; i < NP; ++i) d[i] = ldg_s32(gd + i * nEp + le);
#pragma unroll
                for (int i = 0; i < NP; ++i) cp_async8(gu + i * ls + le, prm.u + d[i]);
#pragma unroll
                for (int v = 0; v < 3; ++v) cp_async16(gx + v * e_max + le, prm.xy + d[v]);
            }
            cp_async_mbar_arrive(&gat_full[g]);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        return;
    }

    if (warp < NA) {
        // ------------------------------------------------------------------ A warps
        const int g8 = lane >> 2, cq = lane & 3;
        double afr[RT][4][NK];  // this warp's row tiles warp, warp + NA, ... of Q_f (f = m, A00, A11, A01)
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) {
                    const int tt = warp + r * NA;
                    afr[r][f][kk] = (f == 0 ? DO_M : DO_C) && tt < NTT
                                        ? __ldg(prm.qfrag + ((f * NTT + tt) * NK + kk) * 32 + lane) : 0.0;
                }
        const double* pfrag = prm.qfrag + 4 * NTT * NK * 32;  // Phi^T A-fragments [MT][KT][32]
        const double* cPhi = prm.ctab;
        const double* cW = prm.ctab + oW;
        const FeaCoef& cf = DO_M ? prm.coef_m : prm.coef_c;  // one coefficient (distinct ones: two passes)
        (void)cPhi;

        for (int j = 0; j < nb; ++j) {
            const int g = j & 1;
            const int nE = __ldg(&prm.blocks[b0 + j * G].nE);
            const int net = (nE + 7) >> 3;
            double* Lam = sLam(g);
            double* W = sW(g);
            // ---- A1: U = Phi^T U_e on DMMA, epilogue Lambda_qe = w_q b_e k(u_qe), W_e = vec A_e
            mbar_wait(&gat_full[g], (uint32_t)((j >> 1) & 1));
            {
                const double* gU = sGU(g);
                const double2* gX = sGX(g);
                for (int un = warp; un < MT * net; un += NA) {
                    const int mt = un % MT, et = un / MT;
                    double u0 = 0.0, u1 = 0.0;
#pragma unroll
                    for (int kt = 0; kt < KT; ++kt) {
                        const int i = kt * 4 + cq;
                        const double b = i < NP ? gU[i * ls + et * 8 + g8] : 0.0;
                        dmma(u0, u1, __ldg(pfrag + (mt * KT + kt) * 32 + lane), b);
                    }
                    const int q = mt * 8 + g8, le0 = et * 8 + 2 * cq;
                    double d0 = 0.0, d1 = 0.0, w00 = 0.0, w01 = 0.0, w10 = 0.0, w11 = 0.0, w20 = 0.0, w21 = 0.0;
                    if (le0 < nE) geometry(gX, e_max, le0, d0, w00, w10, w20);
                    if (le0 + 1 < nE) geometry(gX, e_max, le0 + 1, d1, w01, w11, w21);
                    if (mt == 0 && g8 == 0) {
                        *reinterpret_cast<double2*>(W + le0) = make_double2(w00, w01);
                        *reinterpret_cast<double2*>(W + e_max + le0) = make_double2(w10, w11);
                        *reinterpret_cast<double2*>(W + 2 * e_max + le0) = make_double2(w20, w21);
                    }
                    if (q < NQP) {
                        double l0 = 0.0, l1 = 0.0;
                        if (q < NQ) {
                            const double w = cW[q];
                            if (le0 < nE) l0 = w * d0 * keval(cf, u0);
                            if (le0 + 1 < nE) l1 = w * d1 * keval(cf, u1);
                        }
                        *reinterpret_cast<double2*>(Lam + q * ls + le0) = make_double2(l0, l1);
                    }
                }
            }
            named_sync(1, NA * 32);  // Lambda / W of block j complete; every A warp is past A2(j - 1)
            if (tid == 0) mbar_arrive(&gat_free[g]);
            // ---- A2: V = Q Lambda on DMMA into V buffer g
            if (j >= 2) mbar_wait(&v_free[g], (uint32_t)(((j >> 1) - 1) & 1));
            uint8_t* Vb = sV(g);
            for (int et = 0; et < net; ++et) {
                const int col = et * 8 + g8, le0 = et * 8 + 2 * cq;
                double bl[NK];
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) bl[kk] = Lam[(kk * 4 + cq) * ls + col];
#pragma unroll
                for (int r = 0; r < RT; ++r) {
                    const int tt = warp + r * NA;
                    if (RT > 1 && tt >= NTT) continue;
                    double m0 = 0.0, m1 = 0.0, a0 = 0.0, a1 = 0.0, p0 = 0.0, p1 = 0.0, c0 = 0.0, c1 = 0.0;
#pragma unroll
                    for (int kk = 0; kk < NK; ++kk) {
                        if (DO_M) dmma(m0, m1, afr[r][0][kk], bl[kk]);
                        if (DO_C) {
                            dmma(a0, a1, afr[r][1][kk], bl[kk]);
                            dmma(p0, p1, afr[r][2][kk], bl[kk]);
                            dmma(c0, c1, afr[r][3][kk], bl[kk]);
                        }
                    }
                    const int t = tt * 8 + g8;
                    if (t < T) {
                        double k0 = 0.0, k1 = 0.0;
                        if (DO_C) {
                            const double2 w0 = *reinterpret_cast<const double2*>(W + le0);
                            const double2 w1 = *reinterpret_cast<const double2*>(W + e_max + le0);
                            const double2 w2 = *reinterpret_cast<const double2*>(W + 2 * e_max + le0);
                            k0 = fma(w0.x, a0, fma(w1.x, p0, w2.x * c0));
                            k1 = fma(w0.y, a1, fma(w1.y, p1, w2.y * c1));
                        }
                        if (IL) {
                            double2* V2 = reinterpret_cast<double2*>(Vb) + t * vs + le0;
                            V2[0] = make_double2(m0, k0);
                            V2[1] = make_double2(m1, k1);
                        } else {
                            double* V1 = reinterpret_cast<double*>(Vb) + t * vs + le0;
                            V1[0] = DO_M ? m0 : k0;
                            V1[1] = DO_M ? m1 : k1;
                        }
                    }
                }
            }
            mbar_arrive(&v_full[g]);
        }
        return;
    }

    // ------------------------------------------------------------------ B warps
    {
        const int bt = tid - NA * 32, bw = bt >> 5;
        constexpr int U = 8;  // class-A chunks per round; two rounds of item loads in flight per lane
        for (int j = 0; j < nb; ++j) {
            const int g = j & 1;
            const FeaBlock* B = prm.blocks + b0 + j * G;
            const int nslots = __ldg(&B->nslots), ncls = __ldg(&B->ncls);
            const int64_t slot0 = __ldg(&B->slot0);
            const uint8_t* rec = prm.records + __ldg(&B->rec_off);
            const uint32_t* ia = reinterpret_cast<const uint32_t*>(rec);
            const int nch = (nslots + 31) >> 5;
            double* om = DO_M ? prm.out_m + slot0 : nullptr;
            double* oc = DO_C ? prm.out_c + slot0 : nullptr;
            auto load = [&](uint32_t (&w)[U], int c0) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int ch = c0 + u * NB;
                    w[u] = ch < nch ? ldg_u32(ia + ch * 32 + lane) : 0xffffffffu;
                }
            };
            const uint8_t* Vb = sV(g);
            auto run = [&](const uint32_t (&w)[U], int c0) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const uint32_t it = w[u];
                    const int o0 = it & 0xffff, o1 = it >> 16;
                    if (o0 != 0xffff) {
                        const int p = (c0 + u * NB) * 32 + lane;
                        if (IL) {
                            const double2 v0 = reinterpret_cast<const double2*>(Vb)[o0];
                            const double2 v1 = reinterpret_cast<const double2*>(Vb)[o1];
                            om[p] = v0.x + v1.x;
                            oc[p] = v0.y + v1.y;
                        } else {
                            const double s = reinterpret_cast<const double*>(Vb)[o0] + reinterpret_cast<const double*>(Vb)[o1];
                            if (DO_M) om[p] = s;
                            else oc[p] = s;
                        }
                    }
                }
            };
            uint32_t wa[U], wb[U];
            load(wa, bw);  // the first two rounds load before the wait on V
            load(wb, bw + U * NB);
            mbar_wait(&v_full[g], (uint32_t)((j >> 1) & 1));
            for (int c0 = bw; c0 < nch; c0 += 2 * U * NB) {
                run(wa, c0);
                load(wa, c0 + 2 * U * NB);
                run(wb, c0 + U * NB);
                load(wb, c0 + 3 * U * NB);
            }
            if (ncls > 0) {  // class B: slots with more than two contributors
                const double* V1 = reinterpret_cast<const double*>(Vb);
                phase_b5<DO_M, DO_C, false, IL>(rec + 4 * ((nslots + 31) & ~31), ncls, V1, V1, om, oc, bt, NB * 32);
            }
            mbar_arrive(&v_free[g]);
        }
    }
}

using kfun_t = void (*)(const FeaKParams);

template <int P>
kfun_t pick6(int dm, int dc) {
    if (dm && dc) return k_reassemble6<P, true, true>;
    if (dm) return k_reassemble6<P, true, false>;
    return k_reassemble6<P, false, true>;
}

kfun_t select6(int order, int dm, int dc) {
    switch (order) {
        case 3: return pick6<3>(dm, dc);
        case 4: return pick6<4>(dm, dc);
        default: return nullptr;
    }
}

}  // namespace

int fea_launch_reassemble6(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream) {
    kfun_t kern = select6(order, prm.out_m != nullptr, prm.out_c != nullptr);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, fea6_threads(order), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_kernel_occupancy6(int order, int dm, int dc, int smem_bytes, int* n, int* threads) {
    kfun_t kern = select6(order, dm, dc);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = fea6_threads(order);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
