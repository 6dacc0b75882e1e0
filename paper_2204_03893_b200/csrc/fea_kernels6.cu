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
// one arrival per warp: __syncwarp orders the warp's shared-memory writes before lane 0's
// (release) arrive, so a waiter (acquire) sees all of them
__device__ __forceinline__ void warp_arrive(uint64_t* bar, int lane) {
    __syncwarp();
    if (lane == 0) mbar_arrive(bar);
}

// per-role cycle split (FEA_DEBUG_TIMING): a separate DIAG instantiation of the kernel, launched
// only when diagnostics are requested; lane 0 of every warp adds its cycles per phase to
// prm.dbg[base + k].  The production instantiation (DIAG = false) contains none of it.
#define T6_DECL unsigned long long t6acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t6c = DIAG ? clock64() : 0;
#define T6_TICK(k) if constexpr (DIAG) { const unsigned long long n_ = clock64(); t6acc[k] += n_ - t6c; t6c = n_; }
#define T6_FLUSH(base) if constexpr (DIAG) { if (prm.dbg && lane == 0) for (int k_ = 0; k_ < 8; ++k_) atomicAdd(prm.dbg + (base) + k_, t6acc[k_]); }

template <int P, bool DO_M, bool DO_C, bool DIAG>
__global__ void __maxnreg__(fea6_maxnreg(P)) k_reassemble6(const __grid_constant__ FeaKParams prm) {
    constexpr int NP = fea_np(P), T = fea_T(P), NTT = fea_ntt(P);
    constexpr int NQ = fea_nq_native(P), NK = fea_nk(NQ), NQP = 4 * NK;
    constexpr int NA = fea6_na(P), RT = fea6_rt(P), NB = fea6_nb(P);
    constexpr int MT = (NQP + 7) / 8, KT = fea_kt(P);
    constexpr bool IL = DO_M && DO_C;  // {m, c} cells
    // FEA_DEBUG_MODE skip bits (1 phase B, 2 A1, 4 A2, 8 gathers; timing diagnostics, results wrong
    // by design): honoured by the DIAG instantiation, and by every one in a -DFEA6_DBGMODES build
#ifdef FEA6_DBGMODES
    constexpr bool DBGM = true;
#else
    constexpr bool DBGM = DIAG;
#endif
    constexpr int oW = (NP * NQ + 1) & ~1;
    static_assert(NA * RT >= NTT, "row tiles");
    static_assert(fea6_tile_map_ok(P), "tile map: every row tile on exactly one A warp");
    static_assert(FEA6_A1MODE(P) != 3 || FEA6_PROD_ASYNC(P), "A1 on the producer needs the async producer");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int e_max = prm.e_max, ls = fea6_lstride(e_max), vs = fea6_vstride(e_max);
    const int G = gridDim.x, b0 = blockIdx.x;
    const int nb = prm.nblocks > b0 ? (prm.nblocks - 1 - b0) / G + 1 : 0;

    extern __shared__ __align__(128) uint8_t smem[];
    auto sV = [&](int b) { return smem + prm.lay[FEA6_L_V] + b * prm.lay[FEA6_L_VB]; };
    auto sGU = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_GU] + b * prm.lay[FEA6_L_GUB]); };
    // gather stage b: (FEA6_PROD_ASYNC) vertex coordinates [3][e_max] double2, then |det B_e| [e_max]
    auto sGX = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_GW] + b * prm.lay[FEA6_L_GWB]); };
    auto sDet = [&](int b) { return sGX(b) + (FEA6_PROD_ASYNC(P) ? 6 * e_max : 0); };
    auto sLW = [&](int b) { return reinterpret_cast<double*>(smem + prm.lay[FEA6_L_LW] + b * prm.lay[FEA6_L_LWB]); };
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + prm.lay[FEA6_L_BARS]);
    uint64_t* gat_full = bars;       // [2] producer: 32 cp.async completions + 32 arrivals (geometry)
    uint64_t* gat_free = bars + 2;   // [2] NB * 32: A1 of the stage's block done
    uint64_t* v_full = bars + 4;     // [2] NA * 32: V of the buffer's block stored
    uint64_t* v_free = bars + 6;     // [2] NB * 32: phase B of the buffer's block done
    uint64_t* lam_full = bars + 8;   // [3] NB * 32: Lambda / W of the buffer's block stored
    uint64_t* lam_free = bars + 11;  // [3] NA * 32: A2 of the buffer's block done reading it

    if (tid == 0) {
        for (int b = 0; b < 2; ++b) {
            mbar_init(&gat_full[b], 33);  // 32 lanes' cp.async completions + the geometry stores
            mbar_init(&gat_free[b], FEA6_A1MODE(P) == 2 ? NA : FEA6_A1MODE(P) == 3 ? 1 : FEA6_A1MODE(P) == 4 ? NA + NB : NB);
            mbar_init(&v_full[b], NA);
            mbar_init(&v_free[b], NB > 0 ? NB : NA);
        }
        for (int b = 0; b < 3; ++b) {
            mbar_init(&lam_full[b], FEA6_A1MODE(P) == 2 ? NA : FEA6_A1MODE(P) == 3 ? 1 : FEA6_A1MODE(P) == 4 ? NA + NB : NB);
            mbar_init(&lam_free[b], NA);
        }
        fence_mbar_init();
    }
    {  // Phi^T A-fragments of A1 into shared memory (A1 runs with a ~1 KB L1: no global reads there)
        double* spf = reinterpret_cast<double*>(smem + prm.lay[FEA6_L_PF]);
        for (int i = tid; i < MT * KT * 32; i += blockDim.x) spf[i] = __ldg(prm.qfrag + 4 * NTT * NK * 32 + i);
    }
    if (tid < 6) {  // the zero cell of both V buffers (A2 never writes it): compact layout cell 0
                    // (doubles 0, 1); dense: row 0, column e_max -- double e_max (8-byte cells) and
                    // doubles 2 e_max, 2 e_max + 1 ({m, c} cells)
        const int k = tid % 3;
        reinterpret_cast<double*>(sV(tid / 3))[FEA6_VCOMPACT ? (k & 1) : k == 0 ? e_max : 2 * e_max + k - 1] = 0.0;
    }
    const int vcells = prm.lay[FEA6_L_VB] / (IL ? 16 : 8);  // V capacity per buffer (cells)
    __syncthreads();
    // ------------------------------------------------------------------ A1 (warp aw of naw)
    // A1(j): U = Phi^T U_e on DMMA, epilogue Lambda_qe = w_q b_e k(u_qe), into the
    // Lambda buffer j % 3 (W_e came from the producer).  FEA6_A1MODE 3: the producer warp runs A1(j)
    // right after the geometry of block j (P4 with the async producer); 2: the A warps run A1(j + 1)
    // in the middle of A2(j) (its latency hides behind the other warps' DMMA work); 0: the B warps
    // run A1(j) two blocks ahead of their phase B.
    constexpr int A1MODE = FEA6_A1MODE(P);
    const double* cW = prm.ctab + oW;
    const FeaCoef& cf = DO_M ? prm.coef_m : prm.coef_c;  // one coefficient (distinct ones: two passes)
    // part (A1MODE 4): 1 = the B warps' element tiles [0, net - nA), 2 = the A warps' last nA tiles
    auto a1_na = [&](int net) { return A1MODE == 4 ? min(FEA6_A1A, net >> 1) : 0; };
    auto do_a1 = [&](int j, int aw, int naw, int nE, int part = 0) {
        const int g8 = lane >> 2, cq = lane & 3;
        const int g = j & 1;
        const int net = (nE + 7) >> 3;
        const int lo = part == 2 ? net - a1_na(net) : 0, hi = part == 1 ? net - a1_na(net) : net;
        const int l3 = j % 3;
        double* Lam = sLW(l3);
        if (j >= 3) mbar_wait(&lam_free[l3], (uint32_t)(((j / 3) - 1) & 1));
        if (lo + aw < hi) mbar_wait(&gat_full[g], (uint32_t)((j >> 1) & 1));
        const double* gU = sGU(g);
        const double* gw = sDet(g);
        const int hi_run = DBGM && (prm.dbg_mode & 2) ? 0 : hi;  // diagnostics: A1 skipped
        for (int et = lo + aw; et < hi_run; et += naw) {  // one element tile, all m-tiles (independent chains)
            const double* spf = reinterpret_cast<const double*>(smem + prm.lay[FEA6_L_PF]);
            double pf[MT][KT];  // Phi^T A-fragments (shared memory)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int kt = 0; kt < KT; ++kt) pf[mt][kt] = spf[(mt * KT + kt) * 32 + lane];
            double uq[MT][2];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) uq[mt][0] = uq[mt][1] = 0.0;
#pragma unroll
            for (int kt = 0; kt < KT; ++kt) {
                const int i = kt * 4 + cq;
                const double b = i < NP ? gU[i * ls + et * 8 + g8] : 0.0;
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) dmma(uq[mt][0], uq[mt][1], pf[mt][kt], b);
            }
            const int le0 = et * 8 + 2 * cq;
            const bool v0 = le0 < nE, v1 = le0 + 1 < nE;
            const double d0 = v0 ? gw[le0] : 0.0, d1 = v1 ? gw[le0 + 1] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const int q = mt * 8 + g8;
                double l0 = 0.0, l1 = 0.0;
                if (q < NQ) {
                    const double w = cW[q];
                    l0 = w * d0 * keval(cf, uq[mt][0]);
                    l1 = w * d1 * keval(cf, uq[mt][1]);
                }
                if (q < NQP) *reinterpret_cast<double2*>(Lam + q * ls + le0) = make_double2(l0, l1);
            }
        }
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(&gat_free[g]);
            mbar_arrive(&lam_full[l3]);
        }
    };

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
        // software-pipelined across blocks (every global read is an L2 round trip): the DOFs and
        // row-tile masks of block j + 1 load while block j's gathers are issued, its descriptor one
        // block earlier still.  Every gather is asynchronous (cp.async: u(N_e) and the three vertex
        // coordinates into gather stage j & 1), so the warp never waits on a gathered value; the
        // element geometry of block j - 1 is computed from its landed coordinates right after block
        // j's gathers are issued (FEA6_PROD_ASYNC; 0: coordinates in registers, geometry of block j
        // in iteration j -- one exposed round trip per block).  Element le = 32 h + lane, h < PR.
        constexpr int PR = fea6_prod_rounds(P);
        FEA_CHECK(e_max <= 32 * PR);
        int32_t dn[PR][NP];
        int32_t msk = 0, msk_n = 0;  // column tile `lane`'s row-tile mask (v6 ghost row skipping)
        int nE_c = 0, nE_n = 0, nEp_n = 0;
        const int32_t* gd_n = nullptr;
        auto load_desc = [&](int k) {
            const FeaBlock* B = prm.blocks + b0 + k * G;
            nE_n = ldg_s32(&B->nE);
            gd_n = prm.dofs + __ldg(&B->dof_off);
        };
        auto load_dofs = [&]() {  // the DOFs of the block whose descriptor load_desc fetched
            nEp_n = fea_pad4(nE_n);
#pragma unroll
            for (int h = 0; h < PR; ++h)
#pragma unroll
                for (int i = 0; i < NP; ++i)
                    dn[h][i] = 32 * h + lane < nE_n ? ldg_s32(gd_n + i * nEp_n + 32 * h + lane) : 0;
            msk_n = lane < ((nE_n + 7) >> 3) ? ldg_s32(gd_n + NP * nEp_n + lane) : 0;
        };
        // element geometry: b_e = |det B_e| -> gdet, vec A_e -> W (rows 0..2);
        // zero W columns of the last tile's padding
        auto geometry_el = [&](int le, double2 xa, double2 xb, double2 xc, double* gdet, double* W) {
            const double B00 = xb.x - xa.x, B10 = xb.y - xa.y;
            const double B01 = xc.x - xa.x, B11 = xc.y - xa.y;
            const double det = B00 * B11 - B01 * B10;
            const double inv = 1.0 / (det * det);  // det(B^T B) = det(B)^2
            gdet[le] = fabs(det);
            W[le] = (B01 * B01 + B11 * B11) * inv;
            W[e_max + le] = (B00 * B00 + B10 * B10) * inv;
            W[2 * e_max + le] = -(B00 * B01 + B10 * B11) * inv;
        };
        auto pad_w = [&](int nE, double* W) {  // zero W columns of the last tile's padding
            for (int le = nE + lane; le < ((nE + 7) & ~7); le += 32) W[le] = W[e_max + le] = W[2 * e_max + le] = 0.0;
        };
        auto geometry_blk = [&](int nE, const double2* gx, double* gdet, double* W) {
#pragma unroll
            for (int h = 0; h < PR; ++h) {
                const int le = 32 * h + lane;
                if (le < nE) geometry_el(le, gx[le], gx[e_max + le], gx[2 * e_max + le], gdet, W);
            }
            pad_w(nE, W);
        };
        if (nb > 0) {
            load_desc(0);
            load_dofs();
            nE_c = nE_n;
            msk = msk_n;
            if (nb > 1) load_desc(1);
        }
        int nE_p = 0;        // the previous block's size and masks (its geometry runs one iteration late)
        int32_t msk_p = 0;
        T6_DECL
        for (int j = 0; j < nb; ++j) {
            const int g = j & 1;
            if (lane == 0 && j + 2 < nb) prefetch_blk(j + 2);
            T6_TICK(1)
            if (j >= 2) mbar_wait(&gat_free[g], (uint32_t)(((j >> 1) - 1) & 1));
            const int l3 = j % 3;
            // W of block j goes to LW[j % 3] (the async variant writes it one iteration later and waits there)
            if (!FEA6_PROD_ASYNC(P) && j >= 3) mbar_wait(&lam_free[l3], (uint32_t)(((j / 3) - 1) & 1));
            T6_TICK(0)
            const int nE = nE_c;
            FEA_CHECK(nE >= 1 && nE <= e_max);
            double* gu = sGU(g);
            double* W = sLW(l3) + NQP * ls;
            const int nEr = DBGM && (prm.dbg_mode & 8) ? 0 : nE;  // (diagnostics: no gathers)
            if constexpr (FEA6_PROD_ASYNC(P)) {
            double2* gx = reinterpret_cast<double2*>(sGX(g));
#pragma unroll
            for (int h = 0; h < PR; ++h) {  // u gathers and vertex coordinates of every round
                const int le = 32 * h + lane;
                if (le < nEr) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) FEA_CHECK(dn[h][i] >= 0 && dn[h][i] < prm.n_dof);
#pragma unroll
                    for (int i = 0; i < NP; ++i) cp_async8(gu + i * ls + le, prm.u + dn[h][i]);
#pragma unroll
                    for (int v = 0; v < 3; ++v) cp_async16(gx + v * e_max + le, prm.xy + dn[h][v]);
                }
            }
            cp_async_mbar_arrive(&gat_full[g]);  // (noinc) counts when this lane's gathers land
            asm volatile("cp.async.commit_group;" ::: "memory");
            const int32_t msk_j = msk;
            if (j + 1 < nb) {  // the next block's DOFs (registers dn are free again), its successor's descriptor
                load_dofs();
                nE_c = nE_n;
                msk = msk_n;
                if (j + 2 < nb) load_desc(j + 2);
            }
            if (j >= 1) {  // block j - 1: geometry (its coordinates landed: all but the newest group) and
                           // row-tile masks into its W buffer, once A2(j - 4) released that buffer
                const int l3p = (j - 1) % 3;
                if (j - 1 >= 3) mbar_wait(&lam_free[l3p], (uint32_t)((((j - 1) / 3) - 1) & 1));
                asm volatile("cp.async.wait_group 1;" ::: "memory");
                const int gp = (j - 1) & 1;
                double* Wp = sLW(l3p) + NQP * ls;
                if (!(DBGM && (prm.dbg_mode & 8))) geometry_blk(nE_p, reinterpret_cast<const double2*>(sGX(gp)), sDet(gp), Wp);
                if (lane < ((nE_p + 7) >> 3)) reinterpret_cast<int32_t*>(Wp + 3 * e_max)[lane] = msk_p;
                warp_arrive(&gat_full[gp], lane);
                if (A1MODE == 3) do_a1(j - 1, 0, 1, nE_p);  // A1 of block j - 1 on this warp
            }
            nE_p = nE;
            msk_p = msk_j;
            } else {
            double2 xa[PR], xb[PR], xc[PR];
#pragma unroll
            for (int h = 0; h < PR; ++h) {
                const int le = 32 * h + lane;
                if (le < nEr) {
#pragma unroll
                    for (int i = 0; i < NP; ++i) cp_async8(gu + i * ls + le, prm.u + dn[h][i]);
                    xa[h] = ldg_f64x2(prm.xy + dn[h][0]);
                    xb[h] = ldg_f64x2(prm.xy + dn[h][1]);
                    xc[h] = ldg_f64x2(prm.xy + dn[h][2]);
                }
            }
            cp_async_mbar_arrive(&gat_full[g]);
            if (lane < ((nE + 7) >> 3)) reinterpret_cast<int32_t*>(W + 3 * e_max)[lane] = msk;
            if (j + 1 < nb) {
                load_dofs();
                nE_c = nE_n;
                msk = msk_n;
                if (j + 2 < nb) load_desc(j + 2);
            }
#pragma unroll
            for (int h = 0; h < PR; ++h) {
                const int le = 32 * h + lane;
                if (le < nEr) geometry_el(le, xa[h], xb[h], xc[h], sDet(g), W);
            }
            pad_w(nE, W);
            warp_arrive(&gat_full[g], lane);
            }
            T6_TICK(1)
        }
        if (FEA6_PROD_ASYNC(P) && nb > 0) {  // geometry and masks of the last block
            const int l3p = (nb - 1) % 3;
            if (nb - 1 >= 3) mbar_wait(&lam_free[l3p], (uint32_t)((((nb - 1) / 3) - 1) & 1));
            asm volatile("cp.async.wait_group 0;" ::: "memory");
            const int gp = (nb - 1) & 1;
            double* Wp = sLW(l3p) + NQP * ls;
            if (!(DBGM && (prm.dbg_mode & 8))) geometry_blk(nE_p, reinterpret_cast<const double2*>(sGX(gp)), sDet(gp), Wp);
            if (lane < ((nE_p + 7) >> 3)) reinterpret_cast<int32_t*>(Wp + 3 * e_max)[lane] = msk_p;
            warp_arrive(&gat_full[gp], lane);
            if (A1MODE == 3) do_a1(nb - 1, 0, 1, nE_p);
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        T6_FLUSH(16)
        return;
    }

    // ------------------------------------------------------------------ phase B helpers
    // B(jb): every CSR slot of the block = sum of its contributors, in ascending
    // library element order (no atomics).  Class A (<= 2 contributors): warp bw of nbw takes the
    // 32-slot chunks bw, bw + nbw, ... (U per round, two rounds of item loads in flight per lane);
    // class B: one item per thread.  With nearly all shared memory in use the L1 holds ~1 KB, so
    // every global read is an L2 round trip: the next phase B's descriptor and first items are
    // loaded (prefetchB) right after the current one.
    constexpr int U = FEA6_U(P);
    struct BState {
        int nslots, ncls, rB, nch;
        int64_t slot0;
        const uint8_t* rec;
        uint32_t wa[U], wb[U];
        uint4 ib;
    };
    struct BDesc {  // the next phase B's block descriptor, loaded one block ahead of its items
        int nslots, ncls, rB;
        int64_t slot0, rec_off, rec_bytes;
    };
    auto loadA = [&](const BState& st, uint32_t (&w)[U], int c0, int nbw) {
        const uint32_t* ia = reinterpret_cast<const uint32_t*>(st.rec);
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int ch = c0 + u * nbw;
            w[u] = ch < st.nch ? ldg_u32(ia + ch * 32 + lane) : 0xffffffffu;
        }
    };
    auto loadD = [&](BDesc& d, int jb) {
        if (jb >= nb) return;
        const FeaBlock* B = prm.blocks + b0 + jb * G;
        d.nslots = __ldg(&B->nslots);
        d.ncls = __ldg(&B->ncls);
        d.rB = __ldg(&B->pad_);
        d.slot0 = __ldg(&B->slot0);
        d.rec_off = __ldg(&B->rec_off);
        d.rec_bytes = __ldg(&B->rec_bytes);
    };
    // items of block jb (descriptor d, loaded earlier), then the descriptor of block jb + 1 into d
    auto prefetchB = [&](BState& st, BDesc& d, int jb, int bt, int bw, int nbw) {
        st.nslots = d.nslots;
        st.ncls = d.ncls;
        st.rB = d.rB;
        st.slot0 = d.slot0;
        st.rec = prm.records + d.rec_off;
        st.nch = (st.nslots + 31) >> 5;
        FEA_CHECK(st.slot0 >= 0 && st.slot0 + st.nslots <= prm.n_slots && d.rec_off + d.rec_bytes <= prm.rec_size);
        FEA_CHECK(4 * 32 * st.nch + (int64_t)st.ncls * st.rB <= d.rec_bytes);
        loadA(st, st.wa, bw, nbw);
        loadA(st, st.wb, bw + U * nbw, nbw);
        st.ib = make_uint4(0, 0, 0, 0);
        if (bt < st.ncls)
            st.ib = __ldg(reinterpret_cast<const uint4*>(st.rec + 4 * ((st.nslots + 31) & ~31) + (size_t)bt * st.rB));
        loadD(d, jb + 1);
    };
    auto phaseB = [&](BState& st, int jb, int bt, int bw, int nbw) {
        const int g = jb & 1;
        if (DBGM && (prm.dbg_mode & 1)) {  // diagnostics: phase B skipped (synchronisation kept)
            mbar_wait(&v_full[g], (uint32_t)((jb >> 1) & 1));
            warp_arrive(&v_free[g], lane);
            return;
        }
        const int nslots = st.nslots;
        double* om = DO_M ? prm.out_m + st.slot0 : nullptr;
        double* oc = DO_C ? prm.out_c + st.slot0 : nullptr;
        const uint8_t* Vb = sV(g);
        auto run = [&](const uint32_t (&w)[U], int c0) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t it = w[u];
                const int o0 = it & 0xffff, o1 = it >> 16;
                if (o0 != 0xffff) {
                    const int p = (c0 + u * nbw) * 32 + lane;
                    FEA_CHECK(p < nslots && o0 < vcells && o1 < vcells);
                    if (IL) {
                        const double2 x0 = reinterpret_cast<const double2*>(Vb)[o0];
                        const double2 x1 = reinterpret_cast<const double2*>(Vb)[o1];
                        om[p] = x0.x + x1.x;
                        oc[p] = x0.y + x1.y;
                    } else {
                        const double sum = reinterpret_cast<const double*>(Vb)[o0] + reinterpret_cast<const double*>(Vb)[o1];
                        if (DO_M) om[p] = sum;
                        else oc[p] = sum;
                    }
                }
            }
        };
        mbar_wait(&v_full[g], (uint32_t)((jb >> 1) & 1));
        for (int c0 = bw; c0 < st.nch; c0 += 2 * U * nbw) {
            run(st.wa, c0);
            loadA(st, st.wa, c0 + 2 * U * nbw, nbw);
            run(st.wb, c0 + U * nbw);
            loadA(st, st.wb, c0 + 3 * U * nbw, nbw);
        }
        // class B (more than two contributors: vertex diagonals), one item per thread
        for (int it = bt; it < st.ncls; it += nbw * 32) {
            const uint16_t* wrd = reinterpret_cast<const uint16_t*>(st.rec + 4 * ((nslots + 31) & ~31) + (size_t)it * st.rB);
            const uint4 h = it == bt ? st.ib : __ldg(reinterpret_cast<const uint4*>(wrd));
            const int sl = h.x & 0xffff, C = h.x >> 16;
            FEA_CHECK(sl < nslots && C >= 3 && 2 * (C + 2) <= st.rB);
            double am = 0.0, ac = 0.0;
            for (int q = 0; q < C; ++q) {
                const uint32_t hw = q < 2 ? h.y : q < 4 ? h.z : h.w;  // no local-memory indexing
                const int o = q < 6 ? (int)((hw >> (16 * (q & 1))) & 0xffff) : (int)__ldg(wrd + 2 + q);
                FEA_CHECK(o < vcells);
                if (IL) {
                    const double2 x = reinterpret_cast<const double2*>(Vb)[o];
                    am += x.x;
                    ac += x.y;
                } else {
                    am += reinterpret_cast<const double*>(Vb)[o];
                }
            }
            if (IL) {
                om[sl] = am;
                oc[sl] = ac;
            } else if (DO_M) {
                om[sl] = am;
            } else {
                oc[sl] = am;
            }
        }
        warp_arrive(&v_free[g], lane);
    };

    if (warp < NA) {
        // ------------------------------------------------------------------ A warps: A2
        const int g8 = lane >> 2, cq = lane & 3;
        double afr[RT][4][NK];  // this warp's row tiles fea6_tile(P, warp, r) of Q_f (f = m, A00, A11, A01)
        int tts[RT];
#pragma unroll
        for (int r = 0; r < RT; ++r) tts[r] = fea6_tile(P, warp, r);
#pragma unroll
        for (int r = 0; r < RT; ++r)
#pragma unroll
            for (int f = 0; f < 4; ++f)
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) {
                    const int tt = tts[r];
                    afr[r][f][kk] = (f == 0 ? DO_M : DO_C) && tt >= 0 && tt < NTT
                                        ? __ldg(prm.qfrag + ((f * NTT + tt) * NK + kk) * 32 + lane) : 0.0;
                }
        T6_DECL
        int nE_n = nb > 0 ? ldg_s32(&prm.blocks[b0].nE) : 0;  // one block ahead (L2 latency; asm volatile: issued here)
        constexpr bool A1A = A1MODE == 2 || A1MODE == 4;  // the A warps run (part of) A1
        constexpr int A1PART = A1MODE == 4 ? 2 : 0;
        if (A1A && nb > 0) do_a1(0, NA - 1 - warp, NA, nE_n, A1PART);
        BState st;  // NB == 0: the A warps also run phase B (of the previous block, after their A2)
        BDesc bd;
        if (NB == 0 && nb > 0) {
            loadD(bd, 0);
            prefetchB(st, bd, 0, tid, warp, NA);
        }
        for (int j = 0; j < nb; ++j) {
            const int g = j & 1;
            const int nE = nE_n;
            if (j + 1 < nb) nE_n = ldg_s32(&prm.blocks[b0 + (j + 1) * G].nE);
            const int net = (nE + 7) >> 3;
            const int l3 = j % 3;
            const double* Lam = sLW(l3);
            const double* W = Lam + NQP * ls;
            T6_TICK(5)
            mbar_wait(&lam_full[l3], (uint32_t)((j / 3) & 1));
            T6_TICK(0)
            if (j >= 2) mbar_wait(&v_free[g], (uint32_t)(((j >> 1) - 1) & 1));
            T6_TICK(3)
            uint8_t* Vb = sV(g);
            const int net_a2 = DBGM && (prm.dbg_mode & 4) ? 0 : net;  // diagnostics: A2 skipped
            if (DBGM && (prm.dbg_mode & 4) && A1A && j + 1 < nb) do_a1(j + 1, NA - 1 - warp, NA, nE_n, A1PART);
            // A1(j + 1) inside A2(j): a warp with an A1 unit runs it at column tile a1_at (FEA6_A1POS
            // quarters of the block), a warp without one only arrives, at the start
            const int net_n = (nE_n + 7) >> 3;
            const int a1_at = NA - 1 - warp < (A1MODE == 4 ? a1_na(net_n) : net_n) ? (net * FEA6_A1POS) >> 2 : 0;
            // FEA6_A2PF: the next column tile's B fragments and row-tile mask load while this tile's
            // DMMAs run; the W factors once per column tile, before its DMMAs
            uint32_t tm_n = 0;
            double bl_n[NK];
            auto load_tile = [&](int et2, uint32_t& tm, double (&b)[NK]) {
                tm = reinterpret_cast<const uint32_t*>(W + 3 * e_max)[et2];  // row tiles needed
#pragma unroll
                for (int kk = 0; kk < NK; ++kk) b[kk] = Lam[(kk * 4 + cq) * ls + et2 * 8 + g8];
            };
            int32_t cbase = 0;  // compact V: needed row tiles of the column tiles before et
            for (int et = 0; et < net_a2; ++et) {
                // (units to the last warps first: warp NA - 1 holds one row tile less)
                if (A1A && et == a1_at && j + 1 < nb) {
                    T6_TICK(4)
                    do_a1(j + 1, NA - 1 - warp, NA, nE_n, A1PART);
                    T6_TICK(1)
                }
                const int le0 = et * 8 + 2 * cq;
                uint32_t tmask;
                double bl[NK];
                if (!(FEA6_A2PF & 1) || et == 0) load_tile(et, tmask, bl);
                else {
                    tmask = tm_n;
#pragma unroll
                    for (int kk = 0; kk < NK; ++kk) bl[kk] = bl_n[kk];
                }
                if ((FEA6_A2PF & 1) && et + 1 < net_a2) load_tile(et + 1, tm_n, bl_n);
                double2 w0 = make_double2(0.0, 0.0), w1 = w0, w2 = w0;
                if ((FEA6_A2PF & 2) && DO_C) {
                    w0 = *reinterpret_cast<const double2*>(W + le0);
                    w1 = *reinterpret_cast<const double2*>(W + e_max + le0);
                    w2 = *reinterpret_cast<const double2*>(W + 2 * e_max + le0);
                }
#pragma unroll
                for (int r = 0; r < RT; ++r) {  // row tiles one after the other (fused: measured slower)
                    const int tt = tts[r];
                    if (tt < 0 || !((tmask >> tt) & 1u)) continue;  // (ghost rows nobody reads)
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
                            if (!(FEA6_A2PF & 2)) {
                                w0 = *reinterpret_cast<const double2*>(W + le0);
                                w1 = *reinterpret_cast<const double2*>(W + e_max + le0);
                                w2 = *reinterpret_cast<const double2*>(W + 2 * e_max + le0);
                            }
                            k0 = fma(w0.x, a0, fma(w1.x, p0, w2.x * c0));
                            k1 = fma(w0.y, a1, fma(w1.y, p1, w2.y * c1));
                        }
                        int c0 = t * vs + le0, c1 = c0 + 1;
                        if (FEA6_VCOMPACT) {
                            c0 = fea6_vcell(cbase, tmask, tt, g8, 2 * cq);
                            c1 = fea6_vcell(cbase, tmask, tt, g8, 2 * cq + 1);
                        }
                        // (compact layout: cell 0 is the zero cell; dense: row 0, column 0 is a real cell)
                        FEA_CHECK(c0 >= (FEA6_VCOMPACT ? 1 : 0) && c0 < vcells && c1 > c0 && c1 < vcells);
                        if (IL) {
                            double2* V2 = reinterpret_cast<double2*>(Vb);
                            V2[c0] = make_double2(m0, k0);
                            V2[c1] = make_double2(m1, k1);
                        } else {
                            double* V1 = reinterpret_cast<double*>(Vb);
                            V1[c0] = DO_M ? m0 : k0;
                            V1[c1] = DO_M ? m1 : k1;
                        }
                    }
                }
                cbase += fea6_popc(tmask);
            }
            T6_TICK(4)
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&lam_free[l3]);
                mbar_arrive(&v_full[g]);
            }
            if (NB == 0 && j >= 1) {
                phaseB(st, j - 1, tid, warp, NA);
                prefetchB(st, bd, j, tid, warp, NA);
                T6_TICK(6)
            }
        }
        if (NB == 0 && nb > 0) phaseB(st, nb - 1, tid, warp, NA);
        T6_FLUSH(0)
        return;
    }

    // ------------------------------------------------------------------ B warps: [A1(j)], then B(j - LAG)
    // (A1 runs two blocks ahead of phase B and one to two ahead of A2: three Lambda buffers).
    if (NB > 0) {
        const int bt = tid - NA * 32, bw = bt >> 5;
        constexpr int LAG = A1MODE == 0 || A1MODE == 4 ? 2 : 0;  // phase B of block j - LAG after A1(j) (B warps running A1)
        int nE_a = nb > 0 ? ldg_s32(&prm.blocks[b0].nE) : 0;  // A1's block size, one block ahead
        BState st;
        BDesc bd;
        if (nb > 0) {
            loadD(bd, 0);
            prefetchB(st, bd, 0, bt, bw, NB);
        }
        T6_DECL
        for (int j = 0; j < nb + LAG; ++j) {
            if ((A1MODE == 0 || A1MODE == 4) && j < nb) {
                const int nE = nE_a;
                if (j + 1 < nb) nE_a = ldg_s32(&prm.blocks[b0 + (j + 1) * G].nE);
                do_a1(j, bw, NB, nE, A1MODE == 4 ? 1 : 0);
                T6_TICK(6)
            }
            if (j < LAG) continue;
            T6_TICK(0)
            mbar_wait(&v_full[(j - LAG) & 1], (uint32_t)(((j - LAG) >> 1) & 1));  // (again in phaseB: returns at once)
            T6_TICK(1)
            phaseB(st, j - LAG, bt, bw, NB);
            T6_TICK(2)
            if (j - LAG + 1 < nb) prefetchB(st, bd, j - LAG + 1, bt, bw, NB);
            T6_TICK(7)
        }
        T6_FLUSH(8)
    }
}

using kfun_t = void (*)(const FeaKParams);

template <int P, bool DIAG>
kfun_t pick6(int dm, int dc) {
    if (dm && dc) return k_reassemble6<P, true, true, DIAG>;
    if (dm) return k_reassemble6<P, true, false, DIAG>;
    return k_reassemble6<P, false, true, DIAG>;
}

kfun_t select6(int order, int dm, int dc, bool diag) {
    switch (order) {
        case 3: return diag ? pick6<3, true>(dm, dc) : pick6<3, false>(dm, dc);
        case 4: return diag ? pick6<4, true>(dm, dc) : pick6<4, false>(dm, dc);
        default: return nullptr;
    }
}

}  // namespace

int fea_launch_reassemble6(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream) {
    kfun_t kern = select6(order, prm.out_m != nullptr, prm.out_c != nullptr, prm.dbg != nullptr);
    if (!kern) return (int)cudaErrorInvalidValue;
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    kern<<<grid, fea6_threads(order), smem_bytes, (cudaStream_t)stream>>>(prm);
    return (int)cudaGetLastError();
}

int fea_kernel_occupancy6(int order, int dm, int dc, int smem_bytes, int* n, int* threads) {
    kfun_t kern = select6(order, dm, dc, false);
    if (!kern) return (int)cudaErrorInvalidValue;
    *threads = fea6_threads(order);
    cudaError_t err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes);
    if (err != cudaSuccess) return (int)err;
    return (int)cudaOccupancyMaxActiveBlocksPerMultiprocessor(n, kern, *threads, smem_bytes);
}
