// fea_internal.h -- shared between the host planner (fea_host.cpp) and the sm_100a kernels
// (fea_kernels.cu).  Library-side only; the oracle (oracle/) never includes this.
#pragma once
#include <cstdint>

#define FEA_MAX_ORDER 4
#define FEA_MAX_NP 15
#define FEA_MAX_NQ 16
#define FEA_MAX_PAR 16
// Reference tables small enough to travel in the kernel parameters (constant bank): p <= 2
// (P2 with 16 points: Phi 6x16 + w 16 + Q 21x16x4 = 1456 doubles).  Larger orders stage them
// in shared memory.
#define FEA_CTAB_MAX 1464

// One unit of CTA work: a contiguous block of library rows whose CSR slots
// [slot0, slot0 + nslots) are produced by exactly one CTA.  Everything the block streams
// from HBM sits in ONE contiguous, 16-byte aligned record at rec_off (one TMA bulk copy):
//   classes  int32  [ncls][3]   (count c, first item, first contributor); slots with the
//                               same contributor count form a class, so a warp's lanes all
//                               run the same trip count                                (pad16)
//   items    uint16 [nslots]    block-local slot of each item, sorted by (count, slot)   (pad16)
//   contrib  uint16 [ncontrib]  V offsets t * e_max + le, item by item; within an item in
//                               ascending library element order (the fixed summation order)
//                                                                                        (pad16)
//   dofs     int32  [n_p][pad4(nE)]  library DOFs of the block's elements (SoA)
// The block's elements (le = 0 .. nE-1) are in ascending library element order: ghost
// elements (owned by earlier blocks) first, then the block's own elements.
struct FeaBlock {
    int64_t slot0;
    int64_t rec_off;   // byte offset of the record
    int32_t nslots;
    int32_t ncontrib;
    int32_t nE;
    int32_t rec_bytes; // multiple of 16
    int32_t ncls;
    int32_t pad_;
};

#define FEA_MAX_CLASSES 64

__host__ __device__ inline int32_t fea_pad16(int32_t b) { return (b + 15) & ~15; }
__host__ __device__ inline int32_t fea_pad4(int32_t n) { return (n + 3) & ~3; }
__host__ __device__ inline int32_t fea_rec_off_items(const FeaBlock& b) { return fea_pad16(12 * b.ncls); }
__host__ __device__ inline int32_t fea_rec_off_contrib(const FeaBlock& b) {
    return fea_rec_off_items(b) + fea_pad16(2 * b.nslots);
}
__host__ __device__ inline int32_t fea_rec_off_dofs(const FeaBlock& b) {
    return fea_rec_off_contrib(b) + fea_pad16(2 * b.ncontrib);
}
__host__ __device__ inline int32_t fea_rec_bytes(const FeaBlock& b, int np) {
    return fea_rec_off_dofs(b) + 4 * np * fea_pad4(b.nE);
}

// Coefficient k(u) (fea.h FEA_K_*).
struct FeaCoef {
    int32_t kind;
    int32_t npar;
    double par[FEA_MAX_PAR];
};

// Kernel parameters (passed by value as __grid_constant__).
struct FeaKParams {
    const FeaBlock* blocks;
    const uint8_t* records;  // all block records
    int32_t nblocks;
    int32_t e_max;           // V row stride (elements per block, max)
    int32_t rec_max;         // record buffer size in shared memory (bytes, multiple of 16)
    int32_t nq;
    const double2* xy;       // [n_dof] DOF coordinates (vertex DOFs used for B_e)
    const double* u;         // [n_dof] u_full, library numbering
    const double* tables;    // Phi [np][nq], w [nq], Q [T][nq][4]
    int32_t tables_doubles;
    int32_t ntc;             // number of t-chunks per element (STAGED kernels)
    int32_t same_coef;       // mass and stiffness share k -> one Lambda
    int32_t pad_;
    double* out_m;           // [nslots_total] (rank-local slot index) or nullptr
    double* out_c;
    FeaCoef coef_m;
    FeaCoef coef_c;
    int32_t lay[12];         // FeaSmemLayout of the plan (byte offsets)
    int32_t prefetch;        // gathers of block j+1 issued before phase B of block j
    int32_t pad2_;
    double ctab[FEA_CTAB_MAX];  // tables for p <= 2 (same layout as `tables`)
};

// Shared-memory layout (bytes) of k_reassemble for a plan; identical on host and device.
struct FeaSmemLayout {
    int32_t tab, rec0, rec1, gu, gx, vm, vc, lam, bars, total, gu1, gx1;
};

__host__ __device__ inline int32_t fea_align(int32_t v, int32_t a) { return (v + a - 1) / a * a; }

__host__ __device__ inline FeaSmemLayout fea_smem_layout(int tables_doubles, int rec_max, int e_max, int np, int nq,
                                                         int T, int do_m, int do_c, int staged, int prefetch) {
    FeaSmemLayout L;
    int32_t o = 0;
    L.tab = o;  o = fea_align(o + 8 * tables_doubles, 16);
    L.rec0 = o; o = fea_align(o + rec_max, 16);
    L.rec1 = o; o = fea_align(o + rec_max, 16);
    L.gu = o;   o = fea_align(o + 8 * np * e_max, 16);
    L.gx = o;   o = fea_align(o + 16 * 3 * e_max, 16);
    L.gu1 = o;  o = fea_align(o + (prefetch ? 8 * np * e_max : 0), 16);
    L.gx1 = o;  o = fea_align(o + (prefetch ? 16 * 3 * e_max : 0), 16);
    L.vm = o;   o = fea_align(o + (do_m ? 8 * T * e_max : 0), 16);
    L.vc = o;   o = fea_align(o + (do_c ? 8 * T * e_max : 0), 16);
    L.lam = o;  o = fea_align(o + (staged ? 8 * (2 * nq + 3) * e_max : 0), 16);
    L.bars = o; o += 16;
    L.total = o;
    return L;
}

// Launch the fused reassembly kernel (defined in fea_kernels.cu).  Returns a cudaError_t.
int fea_launch_reassemble(const FeaKParams& prm, int order, int threads, int smem_bytes, int grid,
                          int staged, void* stream);
// Query the per-SM CTA occupancy for the kernel variant (for persistent grid sizing).
int fea_kernel_occupancy(int order, int nq, int do_m, int do_c, int staged, int threads, int smem_bytes,
                         int* ctas_per_sm);
