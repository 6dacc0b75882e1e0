// fea_kernels5.cu -- sm_100a reassembly kernel v5 for p <= 2 with the configs' native rules
// (P1: 3-point, P2: 6-point).  Other (order, rule) pairs run v4
// (fea_kernels.cu).
//
// k_reassemble5<P, NQ, DO_M, DO_C, TWO>: one persistent CTA per SM, NW = 16 warps, no producer
// warp, no CTA-wide barrier in the loop.  The CTA walks its row blocks s = 0, 1, ... (FeaBlock,
// grid-strided).  V (the element matrices of a block) and the block records are DOUBLE
// BUFFERED (buffer s & 1), and every warp runs the software pipeline
//
//     step s:  [A] its units of block s   -> V[s & 1]       (then arrives on full[s & 1])
//              [B] its share of block s - 1 from V[(s-1) & 1] (after full[(s-1) & 1]; then
//                  arrives on free[(s-1) & 1], which gates [A] of block s + 1)
//
// so the FP64 contraction of one block overlaps the scatter of the previous one across warps.
//
//   Units.  A block's elements are cut into 32-element tiles, one lane per element; for P2 a
//     tile is two units (the two halves of the column set of the symmetric element matrix), so
//     a block offers ~2x more units than a warp count's worth of tiles.  Warp w takes units
//     w, w + NW, ... of every block: a unit stream across the CTA's blocks.
//   Gathers (Algorithm 2 line 4 inputs; u_e = u[N_e]): the
//     element DOFs, u(N_e) and the vertex coordinates of the next unit are loaded into registers
//     while the current one is computed (the DOFs one unit earlier still); records, DOF arrays
//     and the rows' u, xy are L2-prefetched PF blocks ahead.
//   A (lines 5-11), one lane per element:
//        b_e = |det B_e|, A_e = (B_e^T B_e)^{-1}
//        u_q = Phi^T u_e, S_qe = k(u_q), Lambda_qe = w_q S_qe b_e
//        V_m[ij] = sum_q phi_i phi_j Lambda_q                          (rows i <= j only,
//        V_c[ij] = sum_q Lambda_q J_i A_e J_j^T                          PAPER.md:628)
//     with the Q rows factored (Q_m[ij,q] = phi_i phi_j, Q_c[ij,(q,ab)] = J_ia J_jb), so every
//     table operand is one of the ~100 entries of Phi and J, read as constant-bank DFMA
//     operands (kernel parameters).  (The unfactored 4 KB P2 Q tables thrash the immediate-
//     constant cache, and from shared memory their loads bound the kernel on latency.)
//     V goes to shared memory [T][e_max | 1] (lane-contiguous stores; the odd row stride keeps
//     phase B's gathers of many rows t of one element column free of bank conflicts).
//   B (line 12): every CSR slot of the block is the sum of its contributors in
//     ascending library element order (phase_b5, fea_device.cuh), slots grouped by contributor
//     count (uniform trip counts, one vector load per item).  The block's record was brought in
//     by one TMA bulk copy issued when its buffer was freed (a whole step earlier).
#include <cuda_runtime.h>
#include <cstdint>

#include "fea_device.cuh"

namespace {
using namespace fea_dev;

template <int NP>
struct Gath {  // gathered inputs of one lane's element
    double u[NP];
    double2 x[3];
};

// P2 column halves of the symmetric 6 x 6 element matrix (10 and 11 entries i <= j): nibbles
__host__ __device__ constexpr uint32_t fea5_jset(int h) { return h == 0 ? 0x520u : 0x431u; }

// TWO: mass and stiffness have different coefficients (two Lambda); else one Lambda
template <int P, int NQ, bool DO_M, bool DO_C, bool TWO>
__global__ void __launch_bounds__(fea5_threads(P), 1) k_reassemble5(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = fea_np(P);
    constexpr int NW = fea5_nw(P);
    constexpr int NS = fea5_nsplit(P);           // units per 32-element tile
    constexpr int NJ = NS == 1 ? NP : NP / 2;    // columns per unit
    constexpr int oW = (NP * NQ + 1) & ~1;       // w_q in ctab
    constexpr int PF = FEA5_PF;                  // L2 prefetch distance (blocks)
    constexpr int DR = 8;                        // descriptor ring
    static_assert(2 * NP * NQ <= FEA_JTAB_MAX, "J tables exceed the parameter bank");
    static_assert(NS == 1 || NP == 6, "column halves are defined for P2");
#ifdef FEA5_DIAG
    if (prm.dbg_mode & 64) return;  // diagnostics: empty launch (fixed launch overhead)
#endif
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // every warp runs both A and B (warp-specialised A / B warps measured slower: DESIGN.md 7.7)
    constexpr int NC = NW;   // warps running A
    constexpr int NBW = NW;  // warps running B
    const int vs = prm.e_max | 1;
    const int G = gridDim.x, b0 = blockIdx.x;
    const int nb = prm.nblocks > b0 ? (prm.nblocks - 1 - b0) / G + 1 : 0;
    constexpr bool two_lam = DO_M && DO_C && TWO;

    extern __shared__ __align__(128) uint8_t smem[];
    double* const sVm0 = reinterpret_cast<double*>(smem + prm.lay[FEA_L_VM]);  // [2][T][vs]
    double* const sVc0 = reinterpret_cast<double*>(smem + prm.lay[FEA_L_VC]);
    const int vbuf = fea5_vbuf(fea_T(P), prm.e_max);
    uint8_t* const sRec0 = smem + prm.lay[FEA_L_REC];  // [2][rec_stride]
    const int rec_stride = prm.lay[FEA_L_GU];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA_L_BARS]);
    uint64_t* full = bars;      // [2] NW arrivals: all units of the buffer's block computed
    uint64_t* freeb = bars + 2; // [2] NW arrivals: phase B of the buffer's block done
    uint64_t* recb = bars + 4;  // [2] TMA transactions of the buffer's record
    FeaBlock* sBlk = reinterpret_cast<FeaBlock*>(smem + prm.lay[FEA_L_W]);

    // Block descriptors: ring of DR entries (slot k % DR = block k).  Blocks 0..5 are written before
    // the first barrier; thread 0 copies block s + 6 (cp.async) at step s into the slot of block
    // s - 2 (whose phase B is done: thread 0 waited on free[s & 1]), completes the copy at step
    // s + 1 before arriving on full[(s + 1) & 1], and every warp acquires it with that barrier in
    // step s + 2.  So during [A] of step t blocks < t + 4 are readable, after its full wait < t + 5
    // (the load cursor reads up to t + 3).  Reads beyond the window go to global memory.
    int win = 6;  // blocks < win are readable from the ring
    auto blk_of = [&](int k) -> const FeaBlock& { return k < win ? sBlk[k & (DR - 1)] : prm.blocks[b0 + k * G]; };

    auto prefetch_range = [&](const void* p, size_t bytes) {
        const uintptr_t a = reinterpret_cast<uintptr_t>(p) & ~uintptr_t(15);
        const uintptr_t e = (reinterpret_cast<uintptr_t>(p) + bytes + 15) & ~uintptr_t(15);
        if (e > a) prefetch_l2(reinterpret_cast<const void*>(a), (uint32_t)(e - a));
    };
    // L2 prefetch of block k: its record, its DOF array, and u, xy of its own rows (most of what
    // its gathers touch; ghost DOFs belong to earlier blocks, i.e. the current or previous wave)
    auto prefetch_blk = [&](int k) {  // thread 0 only (its ring entries are complete)
        const FeaBlock& b = sBlk[k & (DR - 1)];
        prefetch_range(prm.records + b.rec_off, (size_t)b.rec_bytes);
        prefetch_range(prm.dofs + b.dof_off, (size_t)4 * NP * fea_pad4(b.nE));
        prefetch_range(prm.u + b.r0, (size_t)8 * b.nr);
        prefetch_range(prm.xy + b.r0, (size_t)16 * b.nr);
    };

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&full[b], NC);
            mbar_init(&freeb[b], NBW);
            mbar_init(&recb[b], 1);
        }
        fence_mbar_init();
    }
    if (tid < 6 && tid < nb) sBlk[tid] = prm.blocks[b0 + tid * G];
    // the zero cell of phase B's padded items (V row 0, column e_max; vs = e_max | 1 > e_max)
    if (tid < 2) {
        if (DO_M && DO_C) {
            reinterpret_cast<double2*>(sVm0 + tid * 2 * vbuf)[prm.e_max] = make_double2(0.0, 0.0);
        } else {
            if (DO_M) sVm0[tid * vbuf + prm.e_max] = 0.0;
            if (DO_C) sVc0[tid * vbuf + prm.e_max] = 0.0;
        }
    }
    __syncthreads();
    if (tid == 0)
        for (int k = 0; k < PF && k < nb; ++k) prefetch_blk(k);

    // ---- unit stream cursors: block s of this CTA, unit u of the block
    auto nunits = [&](int k) { return ((blk_of(k).nE + 31) >> 5) * NS; };
    auto settle = [&](int& k, int& u) {
        while (k < nb && u >= nunits(k)) {
            ++k;
            u = warp;
        }
    };
    auto advance = [&](int& k, int& u) {
        u += NC;
        settle(k, u);
    };
    int cs = 0, cu = warp;  // compute cursor
    settle(cs, cu);
    int ls = cs, lu = cu;  // load cursor (unit whose gathers are issued next)
    int dof[NP];           // DOFs of the load cursor's unit
    auto load_dofs = [&](int k, int u) {
        const FeaBlock& b = blk_of(k);
        const int le = (u / NS) * 32 + lane;
        if (le < b.nE) {
            const int32_t* d = prm.dofs + b.dof_off + le;
            const int nEp = fea_pad4(b.nE);
#pragma unroll
            for (int i = 0; i < NP; ++i) dof[i] = ldg_s32(d + i * nEp);
        }
    };
    auto refill = [&](Gath<NP>& g) {  // gathers of the load cursor's unit, then the next unit's DOFs
        if (ls >= nb) return;
        if ((lu / NS) * 32 + lane < blk_of(ls).nE) {
#pragma unroll
            for (int i = 0; i < NP; ++i) FEA_CHECK(dof[i] >= 0 && dof[i] < prm.n_dof);
#pragma unroll
            for (int i = 0; i < NP; ++i) g.u[i] = ldg_f64(prm.u + dof[i]);
#pragma unroll
            for (int v = 0; v < 3; ++v) g.x[v] = ldg_f64x2(prm.xy + dof[v]);
        }
        advance(ls, lu);
        if (ls < nb) load_dofs(ls, lu);
    };

    // ---- A: one element per lane; unit half h selects the columns j of its share
    auto compute = [&](const Gath<NP>& g, double* sVm, double* sVc, int le, int h) {
        const double2* gx = g.x;
        const double B00 = gx[1].x - gx[0].x, B10 = gx[1].y - gx[0].y;
        const double B01 = gx[2].x - gx[0].x, B11 = gx[2].y - gx[0].y;
        const double det = B00 * B11 - B01 * B10;
        const double absdet = fabs(det);
        const double inv = 1.0 / (det * det);  // det(B^T B) = det(B)^2
        const double A00 = (B01 * B01 + B11 * B11) * inv;
        const double A11 = (B00 * B00 + B10 * B10) * inv;
        const double A01 = -(B00 * B01 + B10 * B11) * inv;
        double uq[NQ], lm[NQ], lc[two_lam ? NQ : 1];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            uq[q] = 0.0;
#pragma unroll
            for (int k = 0; k < NP; ++k) uq[q] = fma(prm.ctab[k * NQ + q], g.u[k], uq[q]);
        }
        keval_all<NQ>(DO_M ? prm.coef_m : prm.coef_c, uq, lm);
        if constexpr (two_lam) keval_all<NQ>(prm.coef_c, uq, lc);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const double wb = prm.ctab[oW + q] * absdet;
            lm[q] *= wb;
            if constexpr (two_lam) lc[q] *= wb;
        }
        auto LC = [&](int q) -> double {
            if constexpr (two_lam) return lc[q];
            else return lm[q];
        };
#ifdef FEA5_DIAG
        if (prm.dbg_mode & 4) return;  // diagnostics: skip the contraction
#endif
        // Contraction, column j of the symmetric element matrices at a time (rows i <= j):
        //   V_m[ij] = sum_q phi_i(x_q) y_jq,               y_jq = phi_j(x_q) Lambda_q
        //   V_c[ij] = sum_q sum_a J_ia(x_q) z_jqa,          z_jq = Lambda_q A_e J_j(x_q)^T
        // i.e. Q_m Lambda and Q_c (Lambda (.) W) of Algorithm 2 lines 10-11 with the Q rows
        // phi_i phi_j and J_i (x) J_j factored.  j is a rolled loop (its y, z
        // live one column at a time: register pressure); the i loop is unrolled so the Phi_i, J_i
        // operands stay compile-time constant-bank offsets.
        auto J = [&](int a, int k, int q) { return prm.jtab[(a * NP + k) * NQ + q]; };
        const uint32_t jset = fea5_jset(h);

#pragma unroll 1
        for (int jj = 0; jj < NJ; ++jj) {
            const int j = NS == 1 ? jj : (int)((jset >> (4 * jj)) & 15u);
            double y[NQ], z0[NQ], z1[NQ];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                if (DO_M) y[q] = prm.ctab[j * NQ + q] * lm[q];
                if (DO_C) {
                    const double j0 = J(0, j, q), j1 = J(1, j, q);
                    z0[q] = LC(q) * fma(A00, j0, A01 * j1);
                    z1[q] = LC(q) * fma(A01, j0, A11 * j1);
                }
            }
#pragma unroll
            for (int i = 0; i < NP; ++i) {
                if (i > j) break;
                const int t = i * NP - i * (i - 1) / 2 + (j - i);  // row-major upper triangle
                double m = 0.0, c0 = 0.0, c1 = 0.0;  // c: two chains (ILP)
                if (DO_M) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) m = fma(prm.ctab[i * NQ + q], y[q], m);
                }
                if (DO_C) {
#pragma unroll
                    for (int q = 0; q < NQ; ++q) {
                        c0 = fma(J(0, i, q), z0[q], c0);
                        c1 = fma(J(1, i, q), z1[q], c1);
                    }
                }
                if (DO_M && DO_C)  // interleaved {m, c}: one 16-byte load per contributor in B
                    reinterpret_cast<double2*>(sVm)[t * vs + le] = make_double2(m, c0 + c1);
                else if (DO_M)
                    sVm[t * vs + le] = m;
                else
                    sVc[t * vs + le] = c0 + c1;
            }
        }
    };

    // ---- diagnostics, compiled in only with -DFEA5_DIAG (FEA_DEBUG_TIMING: per-warp cycle split;
    // FEA_DEBUG_MODE & 8: CTA 0 event trace, & 32: per-CTA start/end)
#ifdef FEA5_DIAG
    unsigned long long tacc[7] = {0, 0, 0, 0, 0, 0, 0};
    unsigned long long tcl = clock64();
    int nev = 0;
    auto trace = [&](int slot) {
        if ((prm.dbg_mode & 8) && prm.dbg && blockIdx.x == 0 && tid == 0 && nev < 56) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            prm.dbg[16 + 2 * nev] = (unsigned long long)slot;
            prm.dbg[17 + 2 * nev] = t;
            ++nev;
        }
    };
    trace(9);
    unsigned long long t_start = 0;
    if ((prm.dbg_mode & 32) && prm.dbg && tid == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
    auto tick = [&](int slot) {
        trace(slot);
        if (prm.dbg && lane == 0) {
            const unsigned long long now = clock64();
            tacc[slot] += now - tcl;
            tcl = now;
        }
    };
#else
    auto tick = [](int) {};
#endif

    // ---- prologue: DOFs of the first unit, then two units of gathers in flight
    Gath<NP> ga, gb;  // ga: the compute cursor's unit, gb: the one after it
    if (ls < nb) load_dofs(ls, lu);
    refill(ga);
    refill(gb);
    tick(6);

    for (int s = 0; s <= nb; ++s) {
        win = max(s + 4, 6);  // ring entries published by the full barrier of step s - 1
        if (s < nb) {
            const int b = s & 1;
            if (s >= 2) mbar_wait(&freeb[b], (uint32_t)(((s - 2) >> 1) & 1));  // B of block s - 2 done
            tick(5);
            if (tid == 0) {
                asm volatile("cp.async.wait_all;" ::: "memory");  // ring entry of block s + 5
                const FeaBlock& bk = sBlk[s & (DR - 1)];
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
            double* sVm = sVm0 + b * (DO_M && DO_C ? 2 : 1) * vbuf;  // M + K: one interleaved region
            double* sVc = sVc0 + b * vbuf;
            while (cs == s) {
                const int le = (cu / NS) * 32 + lane;
                if (le < blk_of(s).nE) compute(ga, sVm, sVc, le, cu % NS);
                tick(0);
                ga = gb;
                refill(gb);
                tick(1);
                advance(cs, cu);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&full[b]);
        }
        if (s >= 1) {
            const int s1 = s - 1, b = s1 & 1;
            mbar_wait(&full[b], (uint32_t)((s1 >> 1) & 1));
            win = max(s + 5, 6);
            tick(2);
            mbar_wait(&recb[b], (uint32_t)((s1 >> 1) & 1));
            tick(3);
            const FeaBlock& bk = blk_of(s1);
            {
                double* om = DO_M ? prm.out_m + bk.slot0 : nullptr;
                double* oc = DO_C ? prm.out_c + bk.slot0 : nullptr;
                if (FEA5_SLOT)  // CSR slot order (contiguous stores)
                    phase_b_slots<DO_M, DO_C, DO_M && DO_C>(sRec0 + b * rec_stride, bk.nslots, bk.ncls, bk.pad_,
                                                           DO_M ? sVm0 + b * (DO_C ? 2 : 1) * vbuf : sVc0 + b * vbuf,
                                                           om, oc, warp, lane, NW);
                else
                    phase_b5<DO_M, DO_C, false, DO_M && DO_C>(sRec0 + b * rec_stride, bk.ncls,
                                         sVm0 + b * (DO_M && DO_C ? 2 : 1) * vbuf, sVc0 + b * vbuf, om, oc, tid,
                                         NW * 32);
            }
            tick(4);
            __syncwarp();
            if (lane == 0) mbar_arrive(&freeb[b]);
        }
    }


#ifdef FEA5_DIAG
    if (prm.dbg && lane == 0)
        for (int i = 0; i < 7; ++i) atomicAdd(prm.dbg + i, tacc[i]);
    if ((prm.dbg_mode & 32) && prm.dbg && tid == 0 && blockIdx.x < 400) {  // per-CTA start / end
        unsigned long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        prm.dbg[200 + 3 * blockIdx.x] = t_start;
        prm.dbg[201 + 3 * blockIdx.x] = t_end;
        prm.dbg[202 + 3 * blockIdx.x] = smid;
    }
#endif
}

using kfun_t = void (*)(const FeaKParams);

template <int P, int NQ>
kfun_t pick(int dm, int dc, int two) {
    if (dm && dc) return two ? k_reassemble5<P, NQ, true, true, true> : k_reassemble5<P, NQ, true, true, false>;
    if (dm) return k_reassemble5<P, NQ, true, false, false>;
    return k_reassemble5<P, NQ, false, true, false>;
}

kfun_t select5(int order, int dm, int dc, int two) {
    switch (order) {
        case 1: return pick<1, 3>(dm, dc, two);
        case 2: return pick<2, 6>(dm, dc, two);
        default: return nullptr;
    }
}

}  // namespace

int fea_launch_reassemble5(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream) {
    kfun_t kern = select5(order, prm.out_m != nullptr, prm.out_c != nullptr, !prm.same_coef);
    if (!kern) return (int)cudaErrorInvalidValue;
    // the attribute is per (device, kernel): set it on every launch (cheap; a cached value goes stale
    // when another context on this thread re-plans or the thread switches devices)
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, order == 1 ? fea5_threads(1) : fea5_threads(2), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_kernel_occupancy5(int order, int dm, int dc, int smem_bytes, int* n, int* threads) {
    kfun_t kern = select5(order, dm, dc, 1);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = order == 1 ? fea5_threads(1) : fea5_threads(2);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
