// fea_internal.h -- shared between the host planner (fea_host.cpp) and the sm_100a kernels
// (fea_kernels.cu).  Library-side only; the oracle (oracle/) never includes this.
#pragma once
#include <cstdint>

#define FEA_MAX_ORDER 4
#define FEA_MAX_NP 15
#define FEA_MAX_NQ 16
#define FEA_MAX_PAR 16

// One unit of CTA work: a contiguous block of library rows [row0, row0 + nrows) whose
// CSR slots [slot0, slot0 + nslots) are produced by exactly one CTA.  Its element set is
// the ghost elements (library index < own0, listed in ghosts[ghost0 ...]) followed by the
// owned contiguous range [own0, own0 + nown) -- i.e. ascending library element order.
struct FeaBlock {
    int64_t slot0;     // first CSR slot (rank-local)
    int64_t contrib0;  // first entry of this block's contributor stream
    int32_t row0;      // first row (rank-local)
    int32_t nslots;
    int32_t own0;      // first owned element (library element index)
    int32_t nown;
    int32_t ghost0;    // offset into the ghost list
    int32_t nghost;
    int32_t chunk0;    // offset into chunk_base (one entry per 32 slots)
    int32_t pad;
};

// Coefficient k(u) (fea.h FEA_K_*).
struct FeaCoef {
    int32_t kind;
    int32_t npar;
    double par[FEA_MAX_PAR];
};

// Kernel parameters (passed by value as __grid_constant__).
struct FeaKParams {
    const FeaBlock* blocks;
    int32_t nblocks;
    int32_t e_max;          // V row stride in shared memory (elements per block, max)
    const int32_t* dofT;    // [n_p][n_e] library DOF ids, library element order (SoA)
    int64_t n_e;
    const double2* xy;      // [n_dof] DOF coordinates (vertex DOFs used for B_e)
    const double* u;        // [n_dof] u_full, library numbering
    const uint8_t* counts;  // [nslots_total] contributors per slot
    const uint16_t* contrib;// contributor stream: smem V offsets t * e_max + le
    const int32_t* chunk_base; // per 32-slot chunk: offset of its first contributor within the block
    const int32_t* ghosts;  // ghost element ids
    const double* tables;   // Phi [np][nq], w [nq], Q [T][4][nq]
    int32_t tables_doubles;
    int32_t nq;
    int32_t ntc;            // number of t-chunks per element (STAGED kernels)
    int32_t same_coef;      // mass and stiffness share k -> one Lambda
    double* out_m;          // [nslots_total] (rank-local slot index) or nullptr
    double* out_c;
    FeaCoef coef_m;
    FeaCoef coef_c;
};

// Launch the fused reassembly kernel (defined in fea_kernels.cu).  Returns a cudaError_t.
int fea_launch_reassemble(const FeaKParams& prm, int order, int threads, int smem_bytes, int grid,
                          int staged, void* stream);
// Query the per-SM CTA occupancy for the kernel variant (for persistent grid sizing).
int fea_kernel_occupancy(int order, int nq, int do_m, int do_c, int staged, int threads, int smem_bytes,
                         int* ctas_per_sm);
