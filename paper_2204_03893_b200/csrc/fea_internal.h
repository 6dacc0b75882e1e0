// fea_internal.h -- shared between the host planner (fea_host.cpp) and the sm_100a kernels
// (fea_kernels.cu).  Library-side only; the oracle (oracle/) never includes this.
#pragma once
#include <cstdint>

#define FEA_MAX_ORDER 4
#define FEA_MAX_NP 15
#define FEA_MAX_NQ 16
#define FEA_MAX_PAR 16
#define FEA_MAX_CLASSES 64
// Phi [np][nq] (pad2) + w [nq] travel in the kernel parameters (constant bank).
#define FEA_CTAB_MAX 272

// Tiling of the B.W contraction on the FP64 tensor cores (mma.sync.m8n8k4.f64 = DMMA):
// the symmetric rows t (T = n_p (n_p + 1) / 2) in tiles of 8, the quadrature points in
// k-steps of 4, 8 elements per n-tile.  Consumer warp w owns row tile w % NTT and every
// S-th element tile.
__host__ __device__ constexpr int fea_np(int p) { return (p + 1) * (p + 2) / 2; }
__host__ __device__ constexpr int fea_T(int p) { return fea_np(p) * (fea_np(p) + 1) / 2; }
__host__ __device__ constexpr int fea_ntt(int p) { return (fea_T(p) + 7) / 8; }
__host__ __device__ constexpr int fea_nk(int nq) { return (nq + 3) / 4; }
// rules with a specialised kernel (the configs' minimal Dunavant rules); other n_q run the
// generic kernel, which pads the quadrature dimension to 16 (4 k-steps)
__host__ __device__ constexpr int fea_nq_native(int p) { return p == 1 ? 3 : p == 2 ? 6 : p == 3 ? 12 : 16; }
__host__ __device__ constexpr int fea_nk_kernel(int p, int nq) { return nq == fea_nq_native(p) ? fea_nk(nq) : 4; }
// element-tile subsets per warp group (consumer warps = fea_ngrp * S)
__host__ __device__ constexpr int fea_S(int p) { return p == 1 ? 8 : p == 2 ? 3 : p == 3 ? 2 : 1; }
__host__ __device__ constexpr int fea_ctas(int p) { return p <= 2 ? 2 : 1; }
__host__ __device__ constexpr int fea_rstages(int p) { return p <= 2 ? 3 : 2; }
// row tiles per consumer warp (B-fragment loads shared by RT tiles); warp groups = ceil(NTT / RT)
#ifndef FEA5_PF
#define FEA5_PF 3  // kernel v5: L2 prefetch distance (blocks); at most 5 (the descriptor ring)
#endif
static_assert(FEA5_PF >= 1 && FEA5_PF <= 5, "FEA5_PF: the 8-entry descriptor ring is filled 6 blocks ahead");
#ifndef FEA5_SLOT
#define FEA5_SLOT 1  // kernel v5 phase B in CSR slot order (the v6 record format); 0: count classes
#endif
#ifndef FEA4_A1FIRST
#define FEA4_A1FIRST 1  // kernel v4: warps running A1(j+1) before B(j): 0 none, 1 odd warps, 2 all
#endif
#ifndef FEA4_RT4
#define FEA4_RT4 1
#endif
__host__ __device__ constexpr int fea_rt(int p) { return p == 4 ? FEA4_RT4 : 1; }
__host__ __device__ constexpr int fea_ngrp(int p) { return (fea_ntt(p) + fea_rt(p) - 1) / fea_rt(p); }
__host__ __device__ constexpr int fea_threads(int p) { return (fea_ngrp(p) * fea_S(p) + 1) * 32; }
// p >= 2: the interpolation U = Phi^T U_e also runs on DMMA (M = quadrature points in tiles of
// 8, K = element nodes in k-steps of 4); A-fragments of Phi^T [MT][KT][32] follow Q_f in qfrag.
__host__ __device__ constexpr bool fea_interp_mma(int p) { return p >= 2; }
__host__ __device__ constexpr int fea_kt(int p) { return (fea_np(p) + 3) / 4; }

// One unit of CTA work: a contiguous block of library rows whose CSR slots
// [slot0, slot0 + nslots) are produced by exactly one CTA.  Its phase-B data sit in ONE
// contiguous, 16-byte aligned record at rec_off (one TMA bulk copy); formats below (v5:
// class/item records; v4: a FeaRecHdr4 header, the same class/item part, then the element DOFs).
// The block's elements (le = 0 .. nE-1) are in ascending library element order: ghost
// elements (owned by earlier blocks) first, then the block's own elements.
struct FeaBlock {
    int64_t slot0;
    int64_t rec_off;   // byte offset of the record
    int64_t dof_off;   // v5: offset (int32 units) of the block's element DOFs [n_p][pad4(nE)] in
                       // FeaKParams::dofs (v4 keeps them at the end of the record instead)
    int32_t nslots;
    int32_t ncontrib;
    int32_t nE;
    int32_t rec_bytes; // multiple of 16
    int32_t ncls;
    int32_t pad_;
    int32_t r0, nr;    // v5: the block's own rows [r0, r0 + nr) (library DOFs): the bulk of the u and
                       // xy entries its gathers touch (L2-prefetched blocks ahead)
    int32_t spare_[2]; // [0]: interior block (all element DOFs owned; world > 1 overlap); 64 bytes:
                       // the v5 kernel copies descriptors with 16-byte cp.async
};
static_assert(sizeof(FeaBlock) == 64, "FeaBlock must stay 64 bytes");

__host__ __device__ inline int32_t fea_pad16(int32_t b) { return (b + 15) & ~15; }
__host__ __device__ inline int32_t fea_pad4(int32_t n) { return (n + 3) & ~3; }
// v4 record (p >= 3, generic rules): a 32-byte header (FeaRecHdr4), the v5 class/item part
// below (offsets relative to byte 32), then the block's element DOFs int32 [n_p][pad4(nE)] at
// dofs_off.  The header lets the consumer warps read the block descriptor from shared memory.
struct FeaRecHdr4 {
    int32_t nE, ncls, nslots, dofs_off;
    int64_t slot0;
    int32_t pad_[2];
};
static_assert(sizeof(FeaRecHdr4) == 32, "FeaRecHdr4 must be 32 bytes");
// v4 V row stride: even (16-byte DMMA epilogue stores) and == 2 (mod 8), so phase B's gathers of
// many rows t of one element column spread over the banks (e_max == 8 mod 16)
__host__ __device__ inline int32_t fea4_vstride(int32_t e_max) { return e_max + 2; }
// Row stride of Lambda / p and of the gathered u (v) in kernels v4 / k_tensor4 (doubles): == 4 mod 16
// for e_max a multiple of 8, so the DMMA B-fragment loads [(4 kk + c) ls + 8 et + g] are
// conflict-free per half-warp (a stride == 8 mod 16 makes them 2-way).
__host__ __device__ inline int32_t fea4_lstride(int32_t e_max) { return e_max + 4; }

// v5 record: int4 class table {C, n_items, byte offset, item bytes} [ncls], then per class n_items
// fixed-size item records {u16 block-local slot, u16 V offset [C]} of fea5_item_bytes(C) bytes
// (one vector shared-memory load per item), each class array 16-byte aligned.  Classes group
// the slots by contributor count C so a warp's lanes run uniform trip counts.
__host__ __device__ constexpr int fea5_item_bytes(int C) {
    return C == 1 ? 4 : C <= 3 ? 8 : C <= 7 ? 16 : (2 * (C + 1) + 15) / 16 * 16;
}

// ---- kernel v5 (p <= 2 with the configs' native rules): lane-per-element, constant-bank tables.
// NW warps per CTA (no producer warp), one CTA per SM, and the units per 32-element tile.
#ifndef FEA5_NW1
#define FEA5_NW1 20  // warps per CTA for P1 (P2: 16); C4: 16 1.148 ms, 20 1.130, 24 1.191
#endif
__host__ __device__ constexpr int fea5_nw(int p) { return p == 1 ? FEA5_NW1 : 16; }
__host__ __device__ constexpr int fea5_ctas(int p) { return 1; }
__host__ __device__ constexpr int fea5_nsplit(int p) { return p == 2 ? 2 : 1; }  // units per tile (P2: column halves)
__host__ __device__ constexpr int fea5_threads(int p) { return fea5_nw(p) * 32; }
__host__ __device__ constexpr bool fea5_supported(int p, int nq) { return p <= 2 && nq == fea_nq_native(p); }
// reference gradients in the kernel parameters: jtab[a][k][q] = d phi_k / d xhat_a at x_q
#define FEA_JTAB_MAX (2 * 6 * 6)

// Coefficient k(u) (fea.h FEA_K_*).
struct FeaCoef {
    int32_t kind;
    int32_t npar;
    double par[FEA_MAX_PAR];
};

// Shared-memory layout (byte offsets) of k_reassemble for a plan; identical on host and device.
enum { FEA_L_REC = 0, FEA_L_GU = 3, FEA_L_GX = 5, FEA_L_LAMM = 7, FEA_L_LAMC = 8, FEA_L_W = 9, FEA_L_VM = 10,
       FEA_L_VC = 11, FEA_L_BARS = 12, FEA_L_TOTAL = 13, FEA_L_N = 14 };

__host__ __device__ inline int32_t fea_align(int32_t v, int32_t a) { return (v + a - 1) / a * a; }

// e_max is a multiple of 8 (element tiles) and == 8 mod 16 (conflict-free 16-byte V stores).
__host__ __device__ inline void fea_smem_layout(int32_t* L, int rstages, int rec_max, int e_max, int p, int nq,
                                                int do_m, int do_c) {
    const int np = fea_np(p), T = fea_T(p);
    const int nqp = 4 * fea_nk_kernel(p, nq);
    int32_t o = 0;
    for (int s = 0; s < 3; ++s) { L[FEA_L_REC + s] = o; o = fea_align(o + (s < rstages ? rec_max : 0), 128); }
    const int ls = fea4_lstride(e_max);
    for (int s = 0; s < 2; ++s) {
        L[FEA_L_GU + s] = o; o = fea_align(o + 8 * np * ls, 16);
        L[FEA_L_GX + s] = o; o = fea_align(o + 16 * 3 * e_max, 16);
    }
    L[FEA_L_LAMM] = o; o = fea_align(o + 8 * nqp * ls, 16);
    L[FEA_L_LAMC] = o; o = fea_align(o + 8 * nqp * ls, 16);
    L[FEA_L_W] = o;    o = fea_align(o + 8 * 4 * e_max, 16);  // A00, A11, A01, |det B_e|
    o = fea_align(o, 128);
    L[FEA_L_VM] = o;   o = fea_align(o + (do_m ? 8 * T * fea4_vstride(e_max) : 0), 128);
    L[FEA_L_VC] = o;   o = fea_align(o + (do_c ? 8 * T * fea4_vstride(e_max) : 0), 128);
    L[FEA_L_BARS] = o; o += 16 * 8;
    L[FEA_L_TOTAL] = o;
}

// one V buffer of k_reassemble5 (doubles): T rows of stride e_max | 1, padded to 128 bytes so every
// buffer (and V_m vs V_c) has the same bank mapping (the planner balances phase B's banks)
__host__ __device__ constexpr int fea5_vbuf(int T, int e_max) { return (T * (e_max | 1) + 15) & ~15; }
// Shared-memory layout of k_reassemble5: V_m, V_c [2][T][e_max | 1], two record stages of
// stride L[FEA_L_GU], mbarriers (6), descriptor ring (8 x 64 B at L[FEA_L_W]).
__host__ __device__ inline void fea5_smem_layout(int32_t* L, int rec_max, int e_max, int p, int do_m, int do_c) {
    const int T = fea_T(p);
    for (int i = 0; i < FEA_L_N; ++i) L[i] = 0;
    int32_t o = 0;
    L[FEA_L_VM] = o; o += do_m ? 2 * 8 * fea5_vbuf(T, e_max) : 0;
    L[FEA_L_VC] = o; o += do_c ? 2 * 8 * fea5_vbuf(T, e_max) : 0;
    o = (o + 127) / 128 * 128;
    L[FEA_L_GU] = (rec_max + 127) / 128 * 128;  // record stage stride
    L[FEA_L_REC] = o; o += 2 * L[FEA_L_GU];
    L[FEA_L_BARS] = o; o += 64;
    L[FEA_L_W] = o; o += 64 * 8;
    L[FEA_L_TOTAL] = o;
}

// Kernel parameters (passed by value as __grid_constant__).
struct FeaKParams {
    const FeaBlock* blocks;
    const uint8_t* records;   // all block records
    const double2* xy;        // [n_dof] DOF coordinates (vertex DOFs give B_e)
    const int32_t* dofs;      // v5: all blocks' element DOFs (see FeaBlock::dof_off)
    const double* u;          // [n_dof] u_full, library numbering
    const double* qfrag;      // Q_f A-fragments [4][NTT][NK][32] (lane order), zero padded
    double* out_m;            // [nslots_total] (rank-local slot index) or nullptr
    double* out_c;
    unsigned long long* dbg;  // optional per-phase cycle counters (FEA_DEBUG_TIMING), else nullptr
    int32_t nblocks;
    int32_t e_max;            // V / Lambda row stride (elements per block, max)
    int32_t nq;
    int32_t same_coef;        // mass and stiffness share k -> one Lambda
    int32_t dbg_mode;         // diagnostics only (FEA_DEBUG_MODE): 1 skip B stores, 2 skip B, 4 skip A2
    int32_t lay[FEA_L_N];     // shared-memory layout (byte offsets)
    int64_t n_dof, n_slots, rec_size;  // extents, for the FEA_BOUNDS_CHECK build's device-side checks
    FeaCoef coef_m;
    FeaCoef coef_c;
    double ctab[FEA_CTAB_MAX];  // Phi [np][nq] at 0, w [nq] at pad2(np nq)
    double jtab[FEA_JTAB_MAX];  // v5: J [2][np][nq] (constant-bank DFMA operands)
};

// ---- tensor contractions (NEXT-1 / NEXT-2; kernel fea_kernels_t.cu)
// Plan: v5 record format with orientation bits (bit 15 of a contributor offset = local i > j).
// Shared memory: V1 [T][vs] (M o2 v, symmetric), Vup [T][vs] / Vdn [T - np][vs] (C o2 v: entries
// (i, k) with i <= k / i > k), all at the row fea_trow(min, max), one record stage, reference tables
// (Phi [np][16], J [2][np][16], w [16]), mbarrier.
enum { FEA_LT_V1 = 0, FEA_LT_VUP = 1, FEA_LT_VDN = 2, FEA_LT_REC = 3, FEA_LT_TAB = 4, FEA_LT_BAR = 5,
       FEA_LT_TOTAL = 6, FEA_LT_N = 20 };
#define FEA_T_WARPS 8
__host__ __device__ inline void fea_t_smem_layout(int32_t* L, int rec_max, int e_max, int p) {
    const int T = fea_T(p), np = fea_np(p), vs = e_max | 1;
    int32_t o = 0;
    L[FEA_LT_V1] = o; o = (o + 8 * T * vs + 127) / 128 * 128;
    L[FEA_LT_VUP] = o; o = (o + 8 * T * vs + 127) / 128 * 128;
    L[FEA_LT_VDN] = o; o = (o + 8 * (T - np) * vs + 127) / 128 * 128;  // strictly lower (i > k) rows
    o = (o + 127) / 128 * 128;
    L[FEA_LT_REC] = o; o += (rec_max + 127) / 128 * 128;
    L[FEA_LT_TAB] = o; o += 8 * (3 * np * 16 + 16);
    L[FEA_LT_BAR] = o; o += 16;
    L[FEA_LT_TOTAL] = o;
    L[7] = 0;
}
// k_tensor4 (DMMA tensor kernel, fea_kernels_t.cu): row tiles of 8 output rows = the T symmetric rows
// of (M o2 v) (Q_m A-fragments, shared with the matrix kernel) and the np^2 rows (i, k) of (C o2 v)
// (R_d A-fragments, R_d[(i, k), q] = J_d,i(q) phi_k(q), d = 0, 1); consumer warp group g of NG keeps
// the M tiles g, g + NG, ... (RM of them) and the C tiles g, g + NG, ... (RC) as register fragments;
// S warps per group split the element tiles.
__host__ __device__ constexpr int fea_ntc(int p) { return (fea_np(p) * fea_np(p) + 7) / 8; }
__host__ __device__ constexpr int fea_t4_ntm(int p, bool m) { return m ? fea_ntt(p) : 0; }
__host__ __device__ constexpr int fea_t4_ntcm(int p, bool c) { return c ? fea_ntc(p) : 0; }
#ifndef FEA_T4_W4
#define FEA_T4_W4 10
#endif
__host__ __device__ constexpr int fea_t4_wmax(int p) { return p == 4 ? FEA_T4_W4 : p == 3 ? 13 : 16; }
__host__ __device__ constexpr int fea_t4_ng(int p, bool m, bool c) {
    return fea_t4_ntm(p, m) > fea_t4_ntcm(p, c) ? (fea_t4_ntm(p, m) < fea_t4_wmax(p) ? fea_t4_ntm(p, m) : fea_t4_wmax(p))
                                                : (fea_t4_ntcm(p, c) < fea_t4_wmax(p) ? fea_t4_ntcm(p, c) : fea_t4_wmax(p));
}
__host__ __device__ constexpr int fea_t4_rm(int p, bool m, bool c) { return (fea_t4_ntm(p, m) + fea_t4_ng(p, m, c) - 1) / fea_t4_ng(p, m, c); }
__host__ __device__ constexpr int fea_t4_rc(int p, bool m, bool c) { return (fea_t4_ntcm(p, c) + fea_t4_ng(p, m, c) - 1) / fea_t4_ng(p, m, c); }
__host__ __device__ constexpr int fea_t4_s(int p, bool m, bool c) { return fea_t4_wmax(p) / fea_t4_ng(p, m, c) > 1 ? fea_t4_wmax(p) / fea_t4_ng(p, m, c) : 1; }
__host__ __device__ constexpr int fea_t4_threads(int p, bool m, bool c) { return (fea_t4_ng(p, m, c) * fea_t4_s(p, m, c) + 1) * 32; }
// offset (doubles) of the R_d fragments [NTC][2][NK][32] in the rule's fragment buffer (after Q_f and Phi^T)
__host__ __device__ constexpr int fea_rfrag_off(int p, int nk) { return 4 * fea_ntt(p) * nk * 32 + ((4 * nk + 7) / 8) * fea_kt(p) * 32; }
enum { FEA_LT4_REC = 0, FEA_LT4_GU = 2, FEA_LT4_GV = 4, FEA_LT4_GX = 6, FEA_LT4_LM = 8, FEA_LT4_P0 = 9, FEA_LT4_P1 = 10,
       FEA_LT4_TAB = 11, FEA_LT4_V1 = 12, FEA_LT4_VUP = 13, FEA_LT4_VDN = 14, FEA_LT4_BARS = 15, FEA_LT4_TOTAL = 16 };
// e_max == 8 mod 16 (as v4); V row stride fea4_vstride(e_max); two record and gather stages
__host__ __device__ inline void fea_t4_smem_layout(int32_t* L, int rec_max, int e_max, int p, int nq) {
    const int T = fea_T(p), np = fea_np(p), vs = fea4_vstride(e_max);
    const int nqp = 4 * fea_nk_kernel(p, nq);
    for (int i = 0; i < FEA_LT_N; ++i) L[i] = 0;
    int32_t o = 0;
    for (int s = 0; s < 2; ++s) { L[FEA_LT4_REC + s] = o; o = fea_align(o + rec_max, 128); }
    const int ls = fea4_lstride(e_max);
    for (int s = 0; s < 2; ++s) {
        L[FEA_LT4_GU + s] = o; o = fea_align(o + 8 * np * ls, 16);
        L[FEA_LT4_GV + s] = o; o = fea_align(o + 8 * np * ls, 16);
        L[FEA_LT4_GX + s] = o; o = fea_align(o + 16 * 3 * e_max, 16);
    }
    L[FEA_LT4_LM] = o; o = fea_align(o + 8 * nqp * ls, 16);
    L[FEA_LT4_P0] = o; o = fea_align(o + 8 * nqp * ls, 16);
    L[FEA_LT4_P1] = o; o = fea_align(o + 8 * nqp * ls, 16);
    L[FEA_LT4_TAB] = o; o = fea_align(o + 8 * (3 * np * 16 + 16), 128);
    L[FEA_LT4_V1] = o; o = fea_align(o + 8 * T * vs, 128);
    L[FEA_LT4_VUP] = o; o = fea_align(o + 8 * T * vs, 128);
    L[FEA_LT4_VDN] = o; o = fea_align(o + 8 * (T - np) * vs, 128);  // strictly lower (i > k) rows
    L[FEA_LT4_BARS] = o; o += 8 * 8;
    L[FEA_LT4_TOTAL] = o;
}
// V row of the entry pair (lo, hi), lo <= hi, in the tensor kernels: the np (np - 1) / 2 off-diagonal
// pairs first (row-major), the np diagonal ones last, so the strictly-lower V (i > k) needs only the
// first T - np rows and both channels address a pair with the same row
__host__ __device__ constexpr int fea_trow(int np, int lo, int hi) {
    return lo < hi ? lo * np - lo * (lo - 1) / 2 + (hi - lo) - lo - 1 : np * (np - 1) / 2 + lo;
}
struct FeaTParams {
    const FeaBlock* blocks;
    const uint8_t* records;
    const int32_t* dofs;
    const double2* xy;
    const double* u;      // u_full (k'(u_h) at the quadrature points)
    const double* v;      // the contracted vector v (library numbering)
    const double* tab;    // Phi [np][16], J [2][np][16], w [16] (zero padded)
    double* out_m;        // (M o2 v) values or nullptr
    double* out_c;        // (C o2 v) values or nullptr
    const double* qfrag;  // k_tensor4: the rule's fragment buffer (Q_m at 0, R_d at fea_rfrag_off)
    int32_t nblocks, e_max, nq, kver;  // kver: 1 = k_tensor (lane per element), 4 = k_tensor4 (DMMA)
    int32_t same_coef, pad_;           // m == c: k_tensor4 evaluates the derivative once
    int64_t n_dof;                     // extent, for the FEA_BOUNDS_CHECK build
    int32_t lay[FEA_LT_N];
    FeaCoef coef_m, coef_c;  // k' of these
    double ctab[FEA_CTAB_MAX];  // k_tensor5: Phi [np][nq] at 0, w [nq] at pad2(np nq) (constant-bank operands)
    double jtab[FEA_JTAB_MAX];  // k_tensor5: J [2][np][nq]
};
int fea_launch_tensor(const FeaTParams& prm, int order, int smem_bytes, int grid, void* stream);
int fea_tensor_occupancy(int order, int nq, int kver, int smem_bytes, int* ctas_per_sm, int* threads);
// k_tensor5 (fea_kernels_t5.cu): P1 with its native 3-point rule, the v5 software pipeline (double-
// buffered V and records, NW warps, descriptor ring).  Shared memory: two V buffers of
// L[FEA_LT5_VBUF] doubles each holding V1 [T][vs] (at L[FEA_LT5_O1] doubles, if the plan has the
// mass channel), Vup [T][vs] and Vdn [T - np][vs] (at L[FEA_LT5_OU] / L[FEA_LT5_OD], conductivity
// channel); two record stages of stride L[FEA_LT5_RS]; mbarriers (6); descriptor ring (8 x 64 B).
enum { FEA_LT5_V = 0, FEA_LT5_VBUF = 1, FEA_LT5_O1 = 2, FEA_LT5_OU = 3, FEA_LT5_OD = 4, FEA_LT5_REC = 5,
       FEA_LT5_RS = 6, FEA_LT5_BARS = 7, FEA_LT5_RING = 8, FEA_LT5_TOTAL = 9 };
#ifndef FEA_T5_NW
#define FEA_T5_NW 16  // C4 tensor: 16 warps 1.283 ms, 20 1.477 (96 registers: spills)
#endif
__host__ __device__ constexpr int fea_t5_nw(int p) { return FEA_T5_NW; }
__host__ __device__ constexpr int fea_t5_threads(int p) { return fea_t5_nw(p) * 32; }
__host__ __device__ constexpr bool fea_t5_supported(int p, int nq) { return p == 1 && nq == 3; }
// V rows per element of one buffer for the planned channels
__host__ __device__ constexpr int fea_t5_rows(int p, bool m, bool c) {
    return (m ? fea_T(p) : 0) + (c ? 2 * fea_T(p) - fea_np(p) : 0);
}
__host__ __device__ inline void fea_t5_smem_layout(int32_t* L, int rec_max, int e_max, int p, bool m, bool c) {
    const int T = fea_T(p), np = fea_np(p), vs = e_max | 1;
    for (int i = 0; i < FEA_LT_N; ++i) L[i] = 0;
    L[FEA_LT5_O1] = 0;
    L[FEA_LT5_OU] = (m ? T : 0) * vs;
    L[FEA_LT5_OD] = L[FEA_LT5_OU] + (c ? T : 0) * vs;
    L[FEA_LT5_VBUF] = (L[FEA_LT5_OD] + (c ? T - np : 0) * vs + 15) & ~15;  // 128-byte buffers
    int32_t o = 0;
    L[FEA_LT5_V] = o; o += 2 * 8 * L[FEA_LT5_VBUF];
    L[FEA_LT5_RS] = (rec_max + 127) / 128 * 128;
    L[FEA_LT5_REC] = o; o += 2 * L[FEA_LT5_RS];
    L[FEA_LT5_BARS] = o; o += 64;
    L[FEA_LT5_RING] = o; o += 64 * 8;
    L[FEA_LT5_TOTAL] = o;
}
int fea_launch_tensor5(const FeaTParams& prm, int order, int smem_bytes, int grid, void* stream);
int fea_tensor_occupancy5(int order, int nq, int smem_bytes, int* ctas_per_sm, int* threads);

// interface-only exchange of u (fea_kernels_x.cu)
int fea_launch_pack(const double* u_owned, const int32_t* I, int nI, int64_t R0, int maxI, double* send, void* stream);
int fea_launch_unpack(const double* recv, const int32_t* Iall, const int64_t* ioff, int world, int rank, int maxI,
                      int64_t total, const double* u_owned, int64_t R0, int64_t n_own, double* u_full, void* stream);

// Launch the fused reassembly kernel (defined in fea_kernels.cu).  Returns a cudaError_t.
int fea_launch_reassemble(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream);
// Per-SM CTA occupancy of the kernel variant and its block size (threads).
int fea_kernel_occupancy(int order, int nq, int do_m, int do_c, int smem_bytes, int* ctas_per_sm, int* threads);
// The same for kernel v5 (fea_kernels5.cu).
int fea_launch_reassemble5(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream);
int fea_kernel_occupancy5(int order, int do_m, int do_c, int smem_bytes, int* ctas_per_sm, int* threads);

// ---- kernel v6 (P3 / P4 with the configs' native rules; fea_kernels6.cu): warp-specialised
// persistent CTA -- NA "A" warps (the A2 contraction on DMMA, RT row tiles of Q each), NB "B" warps
// (A1 of block j + 1, then phase B of block j), one producer warp (gathers u, element geometry).
// V is double-buffered so phase B of block j overlaps A2 of block j + 1; the block records stay in
// global memory (L2-prefetched) and phase B reads them with coalesced loads, which frees the
// shared memory for the second V buffer.
// where A1 runs: 2 = on the A warps, in the middle of A2 of the previous block (P4: the contraction
// dominates and the A warps' DMMA work hides A1's latency); 0 = on the phase-B warps, two blocks
// ahead of their phase B (P3: measured faster, C3 1.51 vs 1.61 ms)
#ifndef FEA6_PROD_ASYNC
// v6 producer: 1 = coordinates by cp.async into the gather stage, geometry one block late (P4);
// 0 = coordinates in registers, geometry of the block in its own iteration (P3: its 3-round
// stages would cost e_max 96 -> 88 of shared memory)
#define FEA6_PROD_ASYNC(p) ((p) == 4)
#endif
#ifndef FEA6_A2PF
#define FEA6_A2PF 0  // A2: bit 0 next column tile's B fragments prefetched, bit 1 W once per column tile
                     // (measured C5: 0 11.65 ms, 1 14.15, 2 12.12, 3 14.57 -- register pressure)
#endif
#ifndef FEA6_A1A
#define FEA6_A1A 4  // A1MODE 4 (split A1): element tiles of A1 the A warps take (at most half)
#endif
#ifndef FEA6_A1POS
#define FEA6_A1POS 0  // A1MODE 2: a warp's A1 unit at column tile (net * A1POS) / 4 of A2
                      // (C5: 0 11.76 ms, 1 12.00, 2 12.20, 3 12.32; A1 on the B warps 13.21)
#endif
#if defined(FEA6_A1MODE_P4)  // (experiments: the P4 mode alone)
#define FEA6_A1MODE(p) ((p) == 4 ? FEA6_A1MODE_P4 : 0)
#endif
// 4 = split (P3): the B warps run A1's first element tiles two blocks ahead of their phase B, the
// A warps the last FEA6_A1A tiles at the start of A2 of the previous block (C3: the B warps were
// the bottleneck, 61 % of their time in A1 with k = exp(0.5 u); 1.439 -> 1.416 ms; all on the A
// warps 1.516, FEA6_A1A 2 / 6: 1.605 / 1.479)
#ifndef FEA6_A1MODE
#define FEA6_A1MODE(p) ((p) == 4 ? 2 : 4)
#endif
// phase-B warps: P4 (FEA6_P4_MERGED 1) none -- the 15 DMMA warps (one row tile each) run phase B of
// the previous block after their A2, v5-style; P3: 7 (the DMMA warps run A2 only)
#ifndef FEA6_P4_MERGED
#define FEA6_P4_MERGED 0  // measured: C5 16.17 ms merged vs 14.18 with phase-B warps
#endif
#ifndef FEA6_NB
#define FEA6_NB 7
#endif
#ifndef FEA6_NB3
#define FEA6_NB3 FEA6_NB  // P3 phase-B warps (measured: an eighth, 16 warps, C3 1.463 ms vs 1.417 with 7)
#endif
__host__ __device__ constexpr int fea6_nb(int p) { return p == 4 ? (FEA6_P4_MERGED ? 0 : FEA6_NB) : FEA6_NB3; }
__host__ __device__ constexpr bool fea6_supported(int p, int nq) { return p >= 3 && nq == fea_nq_native(p); }
// P4 A warps: 8 with two row tiles each (default), or (FEA6_P4_NA15) 15 with one row tile each
// -- four A warps per SM sub-partition keep the FP64 pipe fed while some of them run their
// epilogue, A1 or wait at a barrier; the CTA then has 23 warps and 88 registers per thread
#ifndef FEA6_P4_NA15
#define FEA6_P4_NA15 0
#endif
#ifndef FEA6_P4_NA
#define FEA6_P4_NA 8  // P4 A warps with two row tiles (9 / 10 with FEA6_NB 6 / 5: experiments)
#endif
__host__ __device__ constexpr int fea6_na(int p) { return p == 4 ? (FEA6_P4_MERGED || FEA6_P4_NA15 ? 15 : FEA6_P4_NA) : 7; }
__host__ __device__ constexpr int fea6_rt(int p) { return p == 4 && !FEA6_P4_MERGED && !FEA6_P4_NA15 ? 2 : 1; }
__host__ __device__ constexpr int fea6_threads(int p) { return (fea6_na(p) + fea6_nb(p) + 1) * 32; }
// registers per thread: each SM sub-partition holds 16384 registers for its ceil(warps / 4) warps
// (warp w on SMSP w % 4), in allocation units of 8
__host__ __device__ constexpr int fea6_maxnreg(int p) {
    return 16384 / (32 * ((fea6_threads(p) / 32 + 3) / 4)) / 8 * 8 > 128 ? 128 : 16384 / (32 * ((fea6_threads(p) / 32 + 3) / 4)) / 8 * 8;
}
// row tile tt of Q held by A warp w as its r-th tile (-1: none).  FEA6_TILEMAP 0: tt = w + r NA.
// 1 (default): balanced by the measured frequency with which each tile survives ghost row-tile
// skipping (tools/plan_stats.py with FEA_PLAN_TIMING; C5: tiles 0, 1 in 2.06 M column tiles, tiles
// 11-14 in 1.21 M).  P4: balanced per WARP (the A warps meet once per block at the Lambda barrier
// and one warp issues at most one DMMA per 16 clk), then per SMSP (warp w on SMSP w % 4), A1's
// element tiles counted on warps 2-7: busiest warp / mean 1.19 -> 1.08 (a per-SMSP-only balance,
// 1.09 -> 1.004, left one warp with tiles 0 and 1 and measured C5 12.32 -> 12.74 ms).  P3 (one
// tile per warp, 7 warps on 4 SMSPs): per SMSP 1.26 -> 1.16, C3 1.505 -> 1.466 ms.
// phase-B item registers per lane: 2 x FEA6_U(p) class-A items (chunks) in flight per warp
// (measured: P3 12 vs 8: C3 1.460 -> 1.418 ms; P4 8 vs 12: C5 12.17 vs 12.39 ms)
#ifndef FEA6_U
#define FEA6_U(p) ((p) == 3 ? 12 : 8)
#endif
#ifndef FEA6_P4MAP
#define FEA6_P4MAP 1  // (C5: map 1 11.52 ms, 0 11.64, 2 11.65)
#endif
#ifndef FEA6_TILEMAP
#define FEA6_TILEMAP 1
#endif
__host__ __device__ constexpr int fea6_tile(int p, int w, int r) {
    if (!FEA6_TILEMAP || (p == 4 && FEA6_P4_MERGED)) {
        const int na = p == 4 ? (FEA6_P4_MERGED ? 15 : FEA6_P4_NA) : 7, ntt = p == 4 ? 15 : 7;
        return w + r * na < ntt ? w + r * na : -1;
    }
    // one nibble per (w, r), 15 = none (ALU only: w is a run-time value)
    // P4 (FEA6_P4MAP 1, A1 units weighted 1.5 tile units): w0 {0, 10} w1 {3, 8} w2 {7, 13} w3 {4, 9}
    // w4 {5, 11} w5 {6, 12} w6 {2, 14} w7 {1}; (map 0, weight 0.7): w0 {6, 7} w1 {0, 11} w2 {8, 14}
    // w3 {3, 10} w4 {2, 12} w5 {4, 9} w6 {5, 13} w7 {1}
    // P3: w0..w6 = 0, 1, 3, 2, 5, 6, 4
    // P4 with 15 A warps (per SMSP, A1 on warps 9-14): w0..w14 = 9 12 5 0 2 6 11 3 10 8 13 1 4 14 7
    // P4 with A1 on the producer (A1MODE 3; its DMMAs on SMSP 3): w0 {1, 14} w1 {6, 9} w2 {4, 7}
    // w3 {2, 12} w4 {5, 11} w5 {8, 10} w6 {3, 13} w7 {0}
    // (FEA6_P4MAP 1 / 2: A1 units weighted 1.5 / 2.5 tile units instead of 0.7 -- experiments)
    const unsigned long long M4 = FEA6_A1MODE(4) == 3 ? 0xF0D3A8B5C27496E1ull
                                  : FEA6_P4MAP == 1   ? 0xF1E2C6B594D783A0ull
                                  : FEA6_P4MAP == 2   ? 0xF0E5D4B8A9C76132ull
                                                      : 0xF1D594C2A3E8B076ull;
    const unsigned long long M3 = 0x4652310ull, M15 = 0x7E41D8A3B6205C9ull;
    // P4 with 9 / 10 A warps (experiments; nibbles 16.. in the high word)
    const unsigned long long M9[2] = {0xE2A84BF17D69C0F3ull, 0xF5ull}, M10[2] = {0xB3C24DF897A6F5F1ull, 0xFEF0ull};
    const int n = 2 * w + r;
    const unsigned long long* Mx = FEA6_P4_NA == 9 ? M9 : M10;
    const int x = p == 4 ? (FEA6_P4_NA15 ? (r == 0 ? (int)((M15 >> (4 * w)) & 15) : 15)
                            : FEA6_P4_NA >= 9 ? (int)((Mx[n >> 4] >> (4 * (n & 15))) & 15)
                                              : (int)((M4 >> (4 * n)) & 15))
                         : (r == 0 ? (int)((M3 >> (4 * w)) & 15) : 15);
    return x == 15 ? -1 : x;
}
// the map holds every row tile exactly once (checked at compile time in fea_kernels6.cu)
__host__ __device__ constexpr bool fea6_tile_map_ok(int p) {
    const int ntt = p == 4 ? 15 : 7, na = fea6_na(p), rt = fea6_rt(p);
    for (int t = 0; t < ntt; ++t) {
        int n = 0;
        for (int w = 0; w < na; ++w)
            for (int r = 0; r < rt; ++r) n += fea6_tile(p, w, r) == t;
        if (n != 1) return false;
    }
    for (int w = 0; w < na; ++w)
        for (int r = 0; r < rt; ++r)
            if (fea6_tile(p, w, r) >= ntt) return false;
    return true;
}
// producer rounds (elements le = 32 h + lane, h < rounds): caps e_max at 32 * rounds
#ifndef FEA6_P3_ROUNDS
#define FEA6_P3_ROUNDS 3
#endif
__host__ __device__ constexpr int fea6_prod_rounds(int p) { return p == 4 ? 2 : FEA6_P3_ROUNDS; }
// Lambda / gathered-u row stride (doubles): == 4 (mod 16), so the DMMA B-fragment loads
// [(4 kk + c) ls + 8 et + g] are conflict-free per half-warp
__host__ __device__ inline int32_t fea6_lstride(int32_t e_max) { return e_max + ((4 - e_max) % 16 + 16) % 16; }
// V row stride in cells (a cell = {m, c} double2 for M + K, one double otherwise): odd, so the
// epilogue's 16-byte stores (columns 2c, 2c + 1 of rows g, g + 1) are conflict-free per quarter-
// warp; column e_max of row 0 is the zero cell (never written by A2)
__host__ __device__ inline int32_t fea6_vstride(int32_t e_max) { return e_max + 1; }
// v6 record (global memory only; one per block, 128-byte aligned): class A = u32 items for the
// block's slots in CSR order [pad32(nslots)]: {u16 V offset 0, u16 V offset 1} -- one
// contributor: offset 1 = the zero cell (e_max); two contributors: both, in ascending library
// element order; more: 0xffff (a hole, the slot is a class-B item); then FeaBlock::ncls class-B
// items of FeaBlock::pad_ (R) bytes each: {u16 block-local slot, u16 C, u16 V offset [C]} (R = 16,
// 32, 48 or 64: C <= 30).  Lane l of a warp handles slot 32 k + l of class A, so its CSR stores
// are contiguous.
// Shared memory (byte offsets / per-buffer bytes): V [2][T][vs] cells; GU [2][np][ls] gathered u;
// GW [2][4][e_max] (|det B_e|, A00, A11, A01 from the producer); LW [3] Lambda [nqp][ls], W [3][e_max]
// and the row-tile masks of the column tiles (int32 [32], from the producer); mbarriers.
// Block DOF arrays (v6): [n_p][pad4(nE)] then the row-tile mask of every 8-element column tile.
enum { FEA6_L_V = 0, FEA6_L_VB = 1, FEA6_L_GU = 2, FEA6_L_GUB = 3, FEA6_L_GW = 4, FEA6_L_GWB = 5, FEA6_L_LW = 6,
       FEA6_L_LWB = 7, FEA6_L_PF = 8, FEA6_L_BARS = 10, FEA6_L_TOTAL = 11 };
// V layout (FEA6_VCOMPACT 1, default): per block, only the 8-row tiles each 8-element column
// tile computes (its row-tile mask m_et) are stored: cell 0 = the zero cell, then the needed
// row tiles in order, tile k = sum_{et' < et} popc(m_et') + popc(m_et & ((1 << tt) - 1)) at cells
// 1 + 64 k ...; inside it row r, column c at 8 r + (c ^ ((r ^ 3k) & 7)): the epilogue's 16-byte
// stores stay conflict-free per quarter warp, and phase B's reads of one element column spread
// over the banks by row and tile (with c ^ (r & 1) they all hit one bank group: C3 +7 %).  Ghost elements then cost V
// space only for the rows their block reads, so a block holds more elements (fewer ghosts).
// 0: dense [T][e_max + 1] cells, the zero cell at column e_max of row 0.
#ifndef FEA6_VSWZ
#define FEA6_VSWZ 0  // compact V column swizzle: 0 xor with (r ^ 3k), 1 rotation by (r + 3k)
#endif
#ifndef FEA6_VFRAC
#define FEA6_VFRAC 83  // compact V: expected post-skip tile fraction (percent) for the P4 block target
#endif
#ifndef FEA6_VCOMPACT
#define FEA6_VCOMPACT 0  // measured slower: C5 11.83 ms (frac 0.83: fewer, uneven blocks) vs dense 11.50; C3 1.461 vs 1.437
#endif
__host__ __device__ inline int fea6_popc(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __popc(x);
#else
    return __builtin_popcount(x);
#endif
}
__host__ __device__ inline int32_t fea6_vcell(int32_t cbase, uint32_t m_et, int tt, int r, int col) {
    const int32_t k = cbase + fea6_popc(m_et & ((1u << tt) - 1u));
    return 1 + 64 * k + 8 * r + (FEA6_VSWZ ? ((col + r + 3 * k) & 7) : (col ^ ((r ^ (3 * k)) & 7)));
}
// vcells: V capacity per buffer in cells (compact layout; 0: dense, from e_max)
__host__ __device__ inline void fea6_smem_layout(int32_t* L, int e_max, int p, int do_m, int do_c, int vcells = 0) {
    const int T = fea_T(p), np = fea_np(p), nqp = 4 * fea_nk(fea_nq_native(p));
    const int ls = fea6_lstride(e_max), vs = fea6_vstride(e_max);
    const int cell = (do_m && do_c) ? 16 : 8;
    for (int i = 0; i < FEA_L_N; ++i) L[i] = 0;
    int32_t o = 0;
    L[FEA6_L_VB] = fea_align((vcells > 0 ? vcells : T * vs) * cell, 128);
    L[FEA6_L_V] = o; o += 2 * L[FEA6_L_VB];
    L[FEA6_L_GUB] = fea_align(8 * np * ls, 128);
    L[FEA6_L_GU] = o; o += 2 * L[FEA6_L_GUB];
    L[FEA6_L_GWB] = fea_align((FEA6_PROD_ASYNC(p) ? 56 : 8) * e_max, 128);  // [coordinates [3][e_max] double2,] |det B_e| [e_max]
    L[FEA6_L_GW] = o; o += 2 * L[FEA6_L_GWB];
    L[FEA6_L_LWB] = fea_align(8 * (nqp * ls + 3 * e_max) + 4 * 32, 128);  // + the column tiles' row-tile masks
    L[FEA6_L_LW] = o; o += 3 * L[FEA6_L_LWB];  // three Lambda / W buffers (A1 runs two blocks ahead)
    L[FEA6_L_PF] = o; o += fea_align(8 * ((nqp + 7) / 8) * fea_kt(p) * 32, 128);  // Phi^T A-fragments (A1)
    L[FEA6_L_BARS] = o; o += 14 * 8;
    L[FEA6_L_TOTAL] = o;
}
int fea_launch_reassemble6(const FeaKParams& prm, int order, int smem_bytes, int grid, void* stream);
int fea_kernel_occupancy6(int order, int do_m, int do_c, int smem_bytes, int* ctas_per_sm, int* threads);
