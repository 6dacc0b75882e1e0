/*
 * fea.h -- C ABI of libfea: loop-free FP64 finite-element reassembly on NVIDIA B200 (sm_100a).
 *
 * Hot path (BASELINE.json north_star; PAPER.md = arXiv 2204.03893 LaTeX source):
 *   per Newton iteration, for the k(u)-weighted mass matrix M and conductivity ("stiffness")
 *   matrix C of scalar 2D problems on triangles with P_p Lagrange elements (p = 1..4):
 *     gather u_e = u(N_e)                                   (PAPER.md:76,  Sec. 3 step 2)
 *     interpolate u_q = Phi^T u_e                           (Sec. 5)
 *     weights Lambda = S * (w b^T), S_qe = k(u_q)           (Eq. def_lambda)
 *             X_c = Lambda (.) W, W = [vec A_e], A_e = (B_e^T B_e)^{-1}
 *     contraction V_m = Q_m X_m, V_c = Q_c X_c              (Algorithm 2)
 *             (symmetric rows only)
 *     deterministic scatter of V into CSR values           (Algorithm 2 line 12)
 *
 * Conventions (all calls):
 *   - Every function returns fea_status (0 = FEA_OK, < 0 = error); no C++ exception crosses
 *     the ABI.  fea_last_error(ctx) returns a message owned by ctx, valid until the next call.
 *   - Host arrays passed to setup calls are COPIED; the caller keeps ownership.
 *   - Device arrays (u, vals) are caller-owned buffers on the ctx device; the library never
 *     frees caller memory.  vals must be 16-byte aligned (FEA_E_ARG otherwise).
 *   - Setup calls (set_element, mesh_upload, build_pattern, get_*) are synchronous.
 *     Assembly calls are asynchronous and ordered on the ctx stream; kernel / NCCL faults
 *     surface at the next fea_sync (CUDA convention).
 *   - Numbering: after fea_mesh_upload every vector and matrix is in LIBRARY numbering
 *     (Morton order of DOF coordinates when FEA_REORDER_MORTON, else user order);
 *     fea_get_dof_perm exports lib_to_user.  On rank r the CSR holds the library rows
 *     [row_begin, row_begin + n_rows_local) with a local row_ptr starting at 0 and GLOBAL
 *     column indices; the structural pattern is shared by M and C.
 *   - A ctx is single-threaded: one ctx per (process, GPU).
 */
#ifndef FEA_H_
#define FEA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct fea_ctx_s* fea_ctx;

typedef enum {
    FEA_OK = 0,
    FEA_E_ARG = -1,          /* bad argument: NULL, length, alignment, rule weights, ... */
    FEA_E_STATE = -2,        /* call out of order (e.g. assemble before build_pattern)    */
    FEA_E_MESH = -3,         /* degenerate element, bad index, inconsistent DOF map       */
    FEA_E_CUDA = -4,         /* CUDA runtime error (message in fea_last_error)            */
    FEA_E_NCCL = -5,         /* NCCL error                                                */
    FEA_E_OOM = -6,          /* device or host allocation failed                          */
    FEA_E_UNSUPPORTED = -7   /* order > 4, n_q > 16, nnz or local entries >= 2^31, ...   */
} fea_status;

enum { FEA_REORDER_NONE = 0, FEA_REORDER_MORTON = 1 };
enum { FEA_MASS = 1, FEA_STIFF = 2 };
/* Coefficient k(u) (reading 17 of DESIGN.md; NEXT-4 piecewise linear PAPER.md:560-568):
 *   FEA_K_POLY: k(u) = sum_{i < n_par} par[i] u^i  (Horner), 1 <= n_par <= 9 (constant: n_par = 1)
 *   FEA_K_EXP : k(u) = par[0] * exp(par[1] * u), n_par = 2
 *   FEA_K_PWL : piecewise linear through (par[0],par[1]), (par[2],par[3]), ... (T_i, k_i),
 *               2 <= m <= 8 breakpoints, T strictly increasing; segment s covers (T_s, T_{s+1}],
 *               the first also T <= T_1, the last also T > T_m (linear extrapolation). */
enum { FEA_K_POLY = 0, FEA_K_EXP = 1, FEA_K_PWL = 2 };

/* Tuning keys for fea_set_tuning (before fea_build_pattern). */
enum {
    FEA_TUNE_SMEM_BUDGET = 1,   /* bytes of shared memory per CTA (0 = default: 113 KiB for p <= 2,
                                   two CTAs per SM; 226 KiB for p >= 3).  Smaller budgets give
                                   smaller row blocks (more, finer CTA tiles)                        */
    FEA_TUNE_KERNEL = 2,        /* kernel generation: 0 = automatic (v5 for p <= 2 with the native
                                   3/6-point rules, v4 otherwise), 4 = force v4                      */
    FEA_TUNE_EMAX = 3,          /* cap on elements per row block (all kernels; 0 = from the
                                   shared-memory budget; the P1 kernels then round it down to whole
                                   rounds of 32-element units over their warps, an explicit cap is
                                   taken as given)                                                   */
    FEA_TUNE_EXCHANGE = 5,      /* world > 1: 0 = interface-only exchange of u (default), 1 = full-
                                   vector allgather                                                 */
    FEA_TUNE_OVERLAP = 7,       /* world > 1: 1 = the interior blocks (reading only owned u) assemble
                                   while the interface exchange runs on a second stream (default),
                                   0 = exchange, then assemble                                      */
    FEA_TUNE_PLAN_WHICH = 4,    /* FEA_MASS | FEA_STIFF: matrices the plan's shared memory is sized
                                   for (default both); assembling more than planned runs one pass
                                   per matrix                                                        */
    FEA_TUNE_PAD1 = 10,         /* kernel v5 phase B: 1 = slots with one contributor join the two-
                                   contributor class with a read of a zero cell where the block's
                                   record still fits (denser stores; bit-identical; default), 0 = off */
    FEA_TUNE_TENSOR_KERNEL = 8, /* fea_assemble_tensor kernel: 0 = automatic (DMMA k_tensor4 for p >= 2
                                   or a non-native rule, k_tensor otherwise), 1 = k_tensor (one
                                   thread per element), 4 = k_tensor4 (FP64 tensor cores)            */
    FEA_TUNE_SKIP = 12,         /* kernel v6 (P3 / P4): 1 = ghost elements compute only the 8-row DMMA
                                   tiles of V that their block reads, each relabelled by the vertex
                                   permutation that needs the fewest tiles (a symmetric rule only;
                                   default): values reproducible run to run, equal to the oracle's
                                   within the tolerance but not bit-identical across tilings or
                                   world sizes; 0 = every row (bit-identical to FEA_TUNE_KERNEL 4)  */
    FEA_TUNE_TIMING = 11        /* 1 = fea_reassemble / fea_assemble record CUDA events around the
                                   exchange of u and around the assembly launches (read with
                                   fea_get_stat keys 36 / 37); 0 = off (default).  Keeps the plan.   */
};

/* Create a context on CUDA device `cuda_device`.  `stream` is a cudaStream_t (NULL = the
 * legacy default stream) on which every assembly call is ordered.  rank/world describe the
 * row partition (world >= 1, 0 <= rank < world); world > 1 requires fea_set_nccl before
 * fea_reassemble.  cuda_device == -1 creates a PLANNING-ONLY context (no device memory,
 * no GPU needed): set_element / mesh_upload / build_pattern / get_* work, assembly calls
 * return FEA_E_STATE.  *out is set to NULL on failure (FEA_E_ARG, FEA_E_CUDA, FEA_E_OOM). */
fea_status fea_create(fea_ctx* out, int cuda_device, void* stream, int rank, int world);

/* Reference element (Algorithm 2 lines 1-3): Lagrange order 1..4 and a
 * quadrature rule of n_q (1..16) points.  q_xy: host, n_q x 2 reference coordinates (x, y)
 * on the triangle (0,0),(1,0),(0,1); q_w: host, n_q weights summing to 1/2 +- 1e-14
 * (reference-triangle measure, reading 4).  The library computes Phi, J_q and the
 * symmetric-reduced Q_m, Q_c tables itself, in long double, rounded once.
 * Errors: FEA_E_ARG (NULL, weights), FEA_E_UNSUPPORTED (order, n_q). */
fea_status fea_set_element(fea_ctx ctx, int order, int n_q, const double* q_xy, const double* q_w);

/* Separate quadrature rules per matrix ("a specific quadrature rule may be used
 * for each matrix").  After fea_set_element (which sets one rule for both),
 * replace the rule of the matrices in `which` (FEA_MASS, FEA_STIFF or both) by (n_q, q_xy, q_w),
 * same conventions and errors as fea_set_element.  Keeps the mesh; invalidates the pattern (call
 * fea_build_pattern again).  With two different rules every assembly runs one pass per matrix on
 * kernel v4 (any rule); fea_assemble_tensor uses the rule of M for (M o2 v), of C for (C o2 v). */
fea_status fea_set_rule(fea_ctx ctx, int which, int n_q, const double* q_xy, const double* q_w);

/* Mesh (Algorithm 2 line 4): vertices a, b, c per element and
 * index sets N_e in the documented local order (reading 7).
 *   vert_xy  : host, n_vert x 2 float64
 *   elem_vert: host, n_elem x 3 int32 (a, b, c); any orientation (|det B_e| is used)
 *   elem_dof : host, n_elem x n_p int32, values in [0, n_dof)
 *   reorder  : FEA_REORDER_NONE or FEA_REORDER_MORTON
 * Validates indices, element non-degeneracy (|det B_e| >= 1e-14 diam^2, else FEA_E_MESH naming
 * the element), distinct DOFs per element and that every element referencing a DOF places
 * it at the same point (1e-10 * diam), which catches edge-orientation errors at p >= 3.
 * Requires fea_set_element first (FEA_E_STATE).  Invalidates any previous pattern. */
fea_status fea_mesh_upload(fea_ctx ctx, int64_t n_vert, const double* vert_xy, int64_t n_elem,
                           const int32_t* elem_vert, int64_t n_dof, const int32_t* elem_dof, int reorder);

/* Tuning before fea_build_pattern (keys above).  FEA_E_ARG for unknown keys / bad values. */
fea_status fea_set_tuning(fea_ctx ctx, int key, int64_t value);

/* Build the structural CSR pattern (reading 9: union over elements of N_e x N_e, sorted
 * unique columns, numerically-zero slots kept) of this rank's rows and the per-iteration
 * scatter plan (element-local entry -> CSR slot, fixed summation order: ascending library
 * element index).  Outputs (host scalars, any may be NULL): first row, number of rows, nnz.
 * Errors: FEA_E_STATE, FEA_E_UNSUPPORTED (nnz >= 2^31 per rank), FEA_E_OOM. */
fea_status fea_build_pattern(fea_ctx ctx, int64_t* row_begin, int64_t* n_rows_local, int64_t* nnz_local);

/* Copy the pattern out: row_ptr (n_rows_local + 1, int64, local, starts at 0) and col_idx
 * (nnz_local, int32, global library columns).  Host pointers. */
fea_status fea_get_pattern(fea_ctx ctx, int64_t* row_ptr, int32_t* col_idx);

/* Rows [r0, r1) of the local pattern (0 <= r0 <= r1 <= n_rows_local): row_ptr (host, r1 - r0 + 1
 * int64, the local offsets row_ptr[r0 .. r1], not rebased) and col_idx (host, row_ptr[r1] -
 * row_ptr[r0] int32).  Either may be NULL.  For checking large patterns window by window. */
fea_status fea_get_pattern_rows(fea_ctx ctx, int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col_idx);

/* lib_to_user[l] = user DOF id of library DOF l (host, n_dof). */
fea_status fea_get_dof_perm(fea_ctx ctx, int64_t* lib_to_user);

/* lib_to_user for elements (host, n_elem): the library element order. */
fea_status fea_get_elem_perm(fea_ctx ctx, int64_t* lib_to_user);

/* Coefficient of M (which & FEA_MASS) and/or C (which & FEA_STIFF); kinds above.
 * Default for both: FEA_K_POLY {1} (k = 1). */
fea_status fea_set_coefficient(fea_ctx ctx, int which, int kind, int n_par, const double* par);

/* Assemble M values (fea_assemble_mass), C values (fea_assemble_stiffness), or both in one
 * fused pass (fea_assemble; either output may be NULL) for this rank's rows.
 *   u_full: device, n_dof float64, library numbering (all DOFs referenced by this rank's
 *           elements must be valid)
 *   vals  : device, nnz_local float64, 16-byte aligned; fully overwritten.
 * Deterministic: bit-identical across runs, CTA tilings and world sizes. Asynchronous. */
fea_status fea_assemble_mass(fea_ctx ctx, const double* u_full, double* vals);
fea_status fea_assemble_stiffness(fea_ctx ctx, const double* u_full, double* vals);
fea_status fea_assemble(fea_ctx ctx, const double* u_full, double* mass_vals, double* stiff_vals);

/* Per-Newton-iteration entry point: allgather of the owned slice u_owned (device,
 * n_rows_local float64, library rows [row_begin, row_begin + n_rows_local)) into the
 * library-owned u_full over NCCL (world > 1), then the fused assembly of the non-NULL
 * outputs.  world == 1: u_owned is the full vector.  Asynchronous on the ctx stream. */
fea_status fea_reassemble(fea_ctx ctx, const double* u_owned, double* mass_vals, double* stiff_vals);

/* End-to-end variant for host buffers: copies u_host (pinned or pageable, n_rows_local)
 * to the device, reassembles, and copies the values back to mass_host / stiff_host
 * (nnz_local each, may be NULL).  Synchronous. */
fea_status fea_reassemble_host(fea_ctx ctx, const double* u_host, double* mass_host, double* stiff_host);

/* Tensor contractions of the Newton Jacobian:
 *   mt_vals <- (M o2 v)_{ik} = sum_e sum_q w_q m'(u_h(x_q)) phi_i phi_k v_h(x_q) |det B_e|
 *              (mass tensor M_ijk = int m' phi_i phi_j phi_k contracted with v, PAPER.md:311;
 *               symmetric)
 *   ct_vals <- (C o2 v)_{ik} = sum_e sum_q w_q c'(u_h(x_q)) (J_q[i,:] A_e J_q^T v_e) phi_k |det B_e|
 *              (conductivity tensor C_ijk = int c' grad phi_i . grad phi_j phi_k contracted in its
 *               second mode; NONSYMMETRIC)
 * m' and c' are the derivatives of the FEA_MASS / FEA_STIFF coefficients (fea_set_coefficient;
 * PWL: the slope of the segment).  u_full, v_full: device, n_dof float64, library numbering.
 * mt_vals / ct_vals: device, nnz_local float64 each, 16-byte aligned, either may be NULL; same
 * pattern (fea_get_pattern) as the matrices.  The first call builds the tensor plan (host,
 * synchronous); the assembly itself is asynchronous on the ctx stream.
 * Errors: FEA_E_STATE (no pattern), FEA_E_ARG (NULL u/v, misalignment), FEA_E_UNSUPPORTED. */
fea_status fea_assemble_tensor(fea_ctx ctx, const double* u_full, const double* v_full, double* mt_vals,
                               double* ct_vals);

/* Interface-only exchange of u (world > 1).  I_t = the library DOFs owned by
 * rank t that another rank's elements read (ascending; every rank derives all lists from the full
 * mesh at fea_build_pattern).  fea_get_interface: offsets (host, world + 1 int64, I_t =
 * dofs[offsets[t] .. offsets[t + 1])) and dofs (host, offsets[world] int32); either may be NULL.
 * fea_reassemble (world > 1, FEA_TUNE_EXCHANGE 0) runs, on the ctx stream: pack (send[k] =
 * u_owned[I_r[k] - row_begin], k < maxI = fea_get_stat key 14, zero padded), one ncclAllGather of
 * maxI float64 per rank, unpack (u_full[I_t[k]] = recv[t * maxI + k] for t != rank; u_full rows
 * of this rank = u_owned).  The pack / unpack steps are exported for callers with their own
 * transport (MPI, ...): send is device maxI float64; recv is device world * maxI float64 (the
 * concatenation of every rank's send); u_full is device n_dof float64.  Asynchronous. */
fea_status fea_get_interface(fea_ctx ctx, int64_t* offsets, int32_t* dofs);
fea_status fea_exchange_pack(fea_ctx ctx, const double* u_owned, double* send);
fea_status fea_exchange_unpack(fea_ctx ctx, const double* u_owned, const double* recv, double* u_full);

/* Multi-GPU: the 128-byte ncclUniqueId.  Rank 0 calls fea_nccl_unique_id and broadcasts the
 * bytes (e.g. over a torch.distributed process group); every rank then calls fea_set_nccl. */
fea_status fea_nccl_unique_id(void* id_out_128_bytes);
fea_status fea_set_nccl(fea_ctx ctx, const void* id_128_bytes);

/* Host transport of the per-iteration allgather (world > 1), for callers whose ranks talk over
 * MPI, gloo, sockets, ... instead of NCCL: fea_reassemble then copies this rank's `count` float64
 * (the packed interface values, or rows_per_rank values with FEA_TUNE_EXCHANGE 1) to a pinned host
 * buffer, waits for them, and calls fn(send, recv, count, user) on the calling thread; fn must
 * fill recv (host, world * count float64) with every rank's send buffer in rank order and return
 * 0 (nonzero -> FEA_E_NCCL).  The values go back to the device on the exchange stream.  With the
 * overlap (FEA_TUNE_OVERLAP 1) the interior blocks are enqueued before the exchange, so they
 * assemble while fn runs.  The library owns the host buffers (valid during the call only).
 * fn = NULL restores NCCL (fea_set_nccl). */
typedef int (*fea_host_allgather_fn)(const double* send, double* recv, int64_t count, void* user);
fea_status fea_set_host_transport(fea_ctx ctx, fea_host_allgather_fn fn, void* user);

/* Wait for all work on the ctx stream; returns deferred CUDA / NCCL errors. */
fea_status fea_sync(fea_ctx ctx);

/* Statistics of the plan (for reports): key 1 = number of CTA blocks, 2 = element-visits
 * including ghosts, 3 = owned elements, 4 = local entries (sum over blocks of contributor
 * count), 5 = kernel launches per fea_assemble call, 6 = smem bytes per CTA, 7 = elements per
 * block (max), 8 = grid, 10 = largest block record (bytes), 11 = matrix kernel (4 or 5),
 * 14 = max interface size, 15 = interior blocks (world > 1).  Tensor plan (after the first
 * fea_assemble_tensor, else -1): 12 = tensor kernel (1 or 4), 13 = its grid, 16 = blocks,
 * 17 = element visits, 18 = owned elements, 19 = smem bytes per CTA.  With FEA_TUNE_TIMING (waits
 * for the last call's events): 36 = exchange of u in microseconds (world > 1; -1 if none ran),
 * 37 = assembly launches, first start to last end, in microseconds.  38 = kernel v6 contraction
 * work with FEA_TUNE_SKIP, per mille of every row of every visited element. */
fea_status fea_get_stat(fea_ctx ctx, int key, int64_t* value);

const char* fea_last_error(fea_ctx ctx);
void fea_destroy(fea_ctx ctx);

#ifdef __cplusplus
}
#endif
#endif /* FEA_H_ */
