// fea_host.cpp -- libfea C ABI (include/fea.h): reference tables, mesh upload with Morton
// renumbering, structural pattern + scatter plan (row blocks), launches, NCCL allgather.
//
// Independent of oracle/ (no shared code): the Lagrange basis here comes from inverting the
// monomial Vandermonde matrix in long double (the oracle uses the barycentric product
// formula); the pattern comes from sorting (row, col) records per row block (MATLAB
// sparse() semantics), the oracle builds it row by row from the incidence.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <parallel/algorithm>  // __gnu_parallel::sort (OpenMP): the mesh-size sorts of the setup
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <thread>
#include <map>
#include <vector>

#include "../../include/fea.h"
#include "fea_internal.h"

namespace {

// ------------------------------------------------------------------ NCCL (dlopen)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.getUniqueId = (decltype(api.getUniqueId))dlsym(h, "ncclGetUniqueId");
            api.commInitRank = (decltype(api.commInitRank))dlsym(h, "ncclCommInitRank");
            api.allGather = (decltype(api.allGather))dlsym(h, "ncclAllGather");
            api.commDestroy = (decltype(api.commDestroy))dlsym(h, "ncclCommDestroy");
            api.getErrorString = (decltype(api.getErrorString))dlsym(h, "ncclGetErrorString");
            api.ok = api.getUniqueId && api.commInitRank && api.allGather && api.commDestroy && api.getErrorString;
        }
    }
    return api;
}

// allocator that default-initialises (no zero fill): for the mesh-size plan arrays, which are
// written completely right after their allocation
template <typename T>
struct dinit_alloc : std::allocator<T> {
    template <typename U> struct rebind { using other = dinit_alloc<U>; };
    using std::allocator<T>::allocator;
    template <typename U> void construct(U* p) noexcept { ::new ((void*)p) U; }
    template <typename U, typename... A> void construct(U* p, A&&... a) { ::new ((void*)p) U(std::forward<A>(a)...); }
};
template <typename T>
using dvec = std::vector<T, dinit_alloc<T>>;

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree((void*)p);
    p = nullptr;
}

int tri_index(int np, int i, int j) {  // i <= j, row-major upper triangle
    return i * np - i * (i - 1) / 2 + (j - i);
}

}  // namespace

struct fea_ctx_s {
    int device = 0;
    bool host_only = false;  // cuda_device == -1: planning only, no device memory
    cudaStream_t stream = nullptr;
    int rank = 0, world = 1;
    std::string err;
    int sm_count = 148;

    // reference element
    int order = 0, np = 0, nq = 0, T = 0;
    std::vector<double> qxy, qw, tables, qfrag, jplain;  // tables = Phi, w; jplain = J (kernel parameters)
    double* d_ttab = nullptr;                             // tensor kernel: Phi, J0, J1 [np][16], w [16]
    // separate quadrature rules per matrix (NEXT-4): the fields above hold the
    // rule of M; when `split`, these hold the rule of C (both rules run on kernel v4, one pass each)
    bool split = false;
    int nq_c = 0;
    std::vector<double> qxy_c, qw_c, tables_c, qfrag_c, jplain_c;
    double* d_tables_c = nullptr;
    double* d_ttab_c = nullptr;

    // mesh, library numbering
    bool have_mesh = false;
    int64_t n_vert = 0, n_e = 0, n_dof = 0;
    std::vector<int64_t> dof_lib2user, elem_lib2user;
    std::vector<int32_t> ed;        // [n_e][np] library DOFs, library element order
    std::vector<int32_t> elem_min;  // min library DOF per library element
    std::vector<double> dxy;        // [n_dof][2]
    double2* d_xy = nullptr;
    double* d_tables = nullptr;

    // plan
    bool have_plan = false;
    int plan_which = FEA_MASS | FEA_STIFF;
    int64_t row_begin = 0, n_rows = 0, nnz = 0, rows_per_rank = 0;
    std::vector<int64_t> row_ptr;
    dvec<int32_t> col_idx;
    FeaBlock* d_blocks = nullptr;
    uint8_t* d_records = nullptr;
    int32_t* d_dofs = nullptr;  // v5: per-block element DOFs
    int kver = 5;               // kernel generation of the plan (5: p <= 2 native rules, else 4)
    int nblocks = 0, e_max = 0, rec_max = 0, smem_bytes = 0, threads = 0, grid = 0;
    int32_t lay[FEA_L_N] = {0};
    int64_t record_bytes = 0;
    int64_t stat_visits = 0, stat_owned = 0, stat_entries = 0;
    int launches_per_call = 1;

    // tensor-contraction plan (built on the first fea_assemble_tensor)
    bool have_tplan = false;
    FeaBlock* dt_blocks = nullptr;
    uint8_t* dt_records = nullptr;
    int32_t* dt_dofs = nullptr;
    int t_nblocks = 0, t_emax = 0, t_smem = 0, t_grid = 0, t_kver = 0;
    bool t_pm = false, t_pc = false;  // k_tensor5 plan: channels its shared-memory layout holds
    int64_t t_visits = 0, t_owned = 0;
    double t_rec_el = 0;  // k_tensor4 plan: record bytes per element of the first plan (re-plan)
    int32_t t_lay[FEA_LT_N] = {0};

    // coefficients
    FeaCoef coef_m{}, coef_c{};

    // tuning
    int64_t tune_smem = 0;
    int tune_kver = 0;     // 0 = automatic, 4 = force kernel v4
    int tune_pad1 = 1;     // v5: single-contributor slots padded into the two-contributor class
    int tune_skip = 1;     // v6: ghost row-tile skipping with element rotations (FEA_TUNE_SKIP)
    bool rule_sym = false; // the rule (of both matrices) is invariant under the 6 vertex permutations
    int64_t skip_work = 0, skip_full = 0;  // v6 plan: A2 row-tile work with / without skipping
    int64_t skip_crit = 0;                 // v6 plan: sum over blocks of NA x the busiest A warp's row-tile work
    int tune_tker = 0;     // tensor kernel: 0 = automatic, 1 = k_tensor, 4 = k_tensor4 (FEA_TUNE_TENSOR_KERNEL)
    int tune_overlap = 1;  // world > 1: interior blocks assemble while u is exchanged (FEA_TUNE_OVERLAP)
    int n_int = 0;         // interior blocks (first n_int of the plan when world > 1)
    cudaStream_t stream2 = nullptr;  // exchange stream of the overlap
    cudaEvent_t ev_own = nullptr, ev_halo = nullptr;
    // FEA_TUNE_TIMING: events of the last call: [0, 1] around the exchange of u (world > 1),
    // [2, 3] from the first assembly launch to the end of the last one
    int tune_timing = 0;
    bool t_exch = false, t_asm = false;
    cudaEvent_t ev_t[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t tune_emax = 0; // v5 element cap per block (0 = from the budget)

    // reassemble buffers
    double* d_ufull = nullptr;
    double* d_usend = nullptr;
    // interface-only exchange (world > 1; NEXT-3): I_t of every rank t, concatenated
    int exchange = 0;  // 0 = interface-only (default), 1 = full-vector allgather
    std::vector<int32_t> iface;
    std::vector<int64_t> ioff;
    int maxI = 0;
    int32_t* d_iface = nullptr;
    int64_t* d_ioff = nullptr;
    double* d_isend = nullptr;
    double* d_irecv = nullptr;
    double* d_vm = nullptr;
    double* d_vc = nullptr;
    void* comm = nullptr;
    // host transport of the allgather (fea_set_host_transport) instead of NCCL, pinned staging
    fea_host_allgather_fn htrans = nullptr;
    void* huser = nullptr;
    double* h_send = nullptr;
    double* h_recv = nullptr;
    int64_t h_cap = 0;
    int int_grid_cap = 0;  // world > 1 overlap: SMs left free for the exchange (FEA_TUNE_EXCH_SMS)
    unsigned long long* d_dbg = nullptr;  // FEA_DEBUG_TIMING phase counters
    int dbg_mode = 0;                     // FEA_DEBUG_MODE / FEA_DEBUG_TIMING, read once at fea_create
    bool dbg_timing = false;

    fea_status fail(fea_status s, const char* fmt, ...) {
        char buf[512];
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(buf, sizeof buf, fmt, ap);
        va_end(ap);
        err = buf;
        return s;
    }
    void free_plan() {
        dfree(d_blocks);
        dfree(d_records);
        dfree(d_dofs);
        dfree(dt_blocks);
        dfree(dt_records);
        dfree(dt_dofs);
        have_tplan = false;
        t_pm = t_pc = false;
        t_rec_el = 0;
        dfree(d_vm);
        dfree(d_vc);
        row_ptr.clear();
        col_idx.clear();
        have_plan = false;
    }
    void free_mesh() {
        free_plan();
        dfree(d_xy);
        dfree(d_ufull);
        dfree(d_usend);
        dfree(d_iface);
        dfree(d_ioff);
        dfree(d_isend);
        dfree(d_irecv);
        have_mesh = false;
    }
};

#define FEA_CUDA(ctx, x)                                                                              \
    do {                                                                                              \
        cudaError_t _e = (x);                                                                         \
        if (_e != cudaSuccess) return (ctx)->fail(FEA_E_CUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
    } while (0)

// FEA_PLAN_TIMING=1: the setup phases' wall times on stderr (diagnostics)
static void ptime(const char* what) {
    static const bool on = getenv("FEA_PLAN_TIMING") != nullptr;
    if (!on) return;
    static auto t0 = std::chrono::steady_clock::now();
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "[fea plan] %-28s %8.3f s\n", what, std::chrono::duration<double>(t - t0).count());
    t0 = t;
}

// FEA_TUNE_TIMING: record timing event i of the current call on `st` (no-op when off)
static fea_status tmark(fea_ctx c, int i, cudaStream_t st) {
    if (!c->tune_timing) return FEA_OK;
    if (!c->ev_t[i]) FEA_CUDA(c, cudaEventCreate(&c->ev_t[i]));
    FEA_CUDA(c, cudaEventRecord(c->ev_t[i], st));
    if (i == 1) c->t_exch = true;
    if (i == 3) c->t_asm = true;
    return FEA_OK;
}

// ------------------------------------------------------------------ reference tables
namespace {

int lib_nodes(int p, int k[][3]) {  // documented local order (reading 7)
    int n = 0;
    auto put = [&](int a, int b, int c) { k[n][0] = a; k[n][1] = b; k[n][2] = c; ++n; };
    put(p, 0, 0);
    put(0, p, 0);
    put(0, 0, p);
    for (int t = 1; t < p; ++t) put(0, p - t, t);
    for (int t = 1; t < p; ++t) put(t, 0, p - t);
    for (int t = 1; t < p; ++t) put(p - t, t, 0);
    for (int a = 1; a < p; ++a)
        for (int b = 1; b < p; ++b)
            if (p - a - b >= 1) put(p - a - b, a, b);
    return n;
}

// Gauss-Jordan inverse with partial pivoting in long double.  Returns false if singular.
bool invert(std::vector<long double>& A, int n) {
    std::vector<long double> I(n * n, 0.0L);
    for (int i = 0; i < n; ++i) I[i * n + i] = 1.0L;
    for (int c = 0; c < n; ++c) {
        int piv = c;
        for (int r = c + 1; r < n; ++r)
            if (fabsl(A[r * n + c]) > fabsl(A[piv * n + c])) piv = r;
        if (fabsl(A[piv * n + c]) < 1e-30L) return false;
        if (piv != c)
            for (int j = 0; j < n; ++j) {
                std::swap(A[c * n + j], A[piv * n + j]);
                std::swap(I[c * n + j], I[piv * n + j]);
            }
        const long double d = A[c * n + c];
        for (int j = 0; j < n; ++j) {
            A[c * n + j] /= d;
            I[c * n + j] /= d;
        }
        for (int r = 0; r < n; ++r)
            if (r != c) {
                const long double f = A[r * n + c];
                if (f == 0.0L) continue;
                for (int j = 0; j < n; ++j) {
                    A[r * n + j] -= f * A[c * n + j];
                    I[r * n + j] -= f * I[c * n + j];
                }
            }
    }
    A = I;
    return true;
}

// Tables (Algorithm 2 lines 1-3), symmetric rows only:
//   Phi[i][q] = phi_i(x_q), w[q], and the rows t = (i <= j) of Q_m and Q_c (below).
bool build_tables(int p, int nq, const double* qxy, const double* qw, std::vector<double>& ctab,
                  std::vector<double>& qfrag, std::vector<double>& jplain) {
    int kk[FEA_MAX_NP][3];
    const int np = lib_nodes(p, kk);
    std::vector<std::pair<int, int>> mono;
    for (int d = 0; d <= p; ++d)
        for (int a = d; a >= 0; --a) mono.push_back({a, d - a});
    std::vector<long double> V(np * np);
    for (int n = 0; n < np; ++n) {
        const long double x = (long double)kk[n][1] / p, y = (long double)kk[n][2] / p;
        for (int m = 0; m < np; ++m) V[n * np + m] = powl(x, mono[m].first) * powl(y, mono[m].second);
    }
    if (!invert(V, np)) return false;  // V now holds V^{-1}; phi_i = sum_m Vinv[m][i] mono_m
    std::vector<long double> phi(np * nq), gx(np * nq), gy(np * nq);
    for (int q = 0; q < nq; ++q) {
        const long double x = qxy[2 * q], y = qxy[2 * q + 1];
        for (int i = 0; i < np; ++i) {
            long double f = 0, fx = 0, fy = 0;
            for (int m = 0; m < np; ++m) {
                const int a = mono[m].first, b = mono[m].second;
                const long double c = V[m * np + i];
                f += c * powl(x, a) * powl(y, b);
                if (a > 0) fx += c * a * powl(x, a - 1) * powl(y, b);
                if (b > 0) fy += c * b * powl(x, a) * powl(y, b - 1);
            }
            phi[i * nq + q] = f;
            gx[i * nq + q] = fx;
            gy[i * nq + q] = fy;
        }
    }
    const int T = np * (np + 1) / 2;
    // (1) ctab: Phi [np][nq] at 0, w [nq] at pad2(np nq)   (kernel parameters)
    const size_t oW = ((size_t)np * nq + 1) & ~size_t(1);
    ctab.assign(oW + nq, 0.0);
    for (int i = 0; i < np * nq; ++i) ctab[i] = (double)phi[i];
    for (int q = 0; q < nq; ++q) ctab[oW + q] = qw[q];
    // (2) qfrag: Q_f as DMMA A-fragments [4][NTT][NK][32]: lane (g, c) holds Q_f[t = 8 tt + g][q = 4 kk + c]
    //     f = 0: Phi_i Phi_j (rows of Q_m = Phi (.) Phi); f = 1, 2, 3: J_i0 J_j0, J_i1 J_j1,
    //     J_i0 J_j1 + J_i1 J_j0 (rows of Q_c = [J_q (x) J_q], columns of vec A merged by A01 = A10)
    const int NTT = (T + 7) / 8, NK = fea_nk_kernel(p, nq);
    qfrag.assign((size_t)4 * NTT * NK * 32, 0.0);
    std::vector<int> ti(T), tj(T);
    for (int i = 0; i < np; ++i)
        for (int j = i; j < np; ++j) {
            ti[tri_index(np, i, j)] = i;
            tj[tri_index(np, i, j)] = j;
        }
    // (2a) jplain: J [2][np][nq] reference gradients (kernel v5 parameters, constant-bank operands)
    jplain.assign((size_t)2 * np * nq, 0.0);
    for (int i = 0; i < np * nq; ++i) {
        jplain[i] = (double)gx[i];
        jplain[(size_t)np * nq + i] = (double)gy[i];
    }
    for (int f = 0; f < 4; ++f)
        for (int tt = 0; tt < NTT; ++tt)
            for (int kk = 0; kk < NK; ++kk)
                for (int lane = 0; lane < 32; ++lane) {
                    const int t = tt * 8 + (lane >> 2), q = kk * 4 + (lane & 3);
                    double v = 0.0;
                    if (t < T && q < nq) {
                        const int a = ti[t] * nq + q, b = tj[t] * nq + q;
                        if (f == 0) v = (double)(phi[a] * phi[b]);
                        if (f == 1) v = (double)(gx[a] * gx[b]);
                        if (f == 2) v = (double)(gy[a] * gy[b]);
                        if (f == 3) v = (double)(gx[a] * gy[b] + gy[a] * gx[b]);
                    }
                    qfrag[(((size_t)f * NTT + tt) * NK + kk) * 32 + lane] = v;
                }
    // (3) Phi^T as DMMA A-fragments [MT][KT][32]: lane (g, c) holds Phi[i = 4 kt + c][q = 8 mt + g]
    const int MT = (4 * NK + 7) / 8, KT = (np + 3) / 4;
    for (int mt = 0; mt < MT; ++mt)
        for (int kt = 0; kt < KT; ++kt)
            for (int lane = 0; lane < 32; ++lane) {
                const int q = mt * 8 + (lane >> 2), i = kt * 4 + (lane & 3);
                qfrag.push_back(q < nq && i < np ? (double)phi[i * nq + q] : 0.0);
            }
    // (4) R_d as DMMA A-fragments [NTC][2][NK][32] (k_tensor4, C o2 v): lane (g, c) holds
    //     R_d[r = 8 rt + g][q = 4 kk + c] = J_d,i(q) phi_k(q), r = i np + k (all np^2 pairs)
    const int NTC = (np * np + 7) / 8;
    for (int rt = 0; rt < NTC; ++rt)
        for (int d = 0; d < 2; ++d)
            for (int kk = 0; kk < NK; ++kk)
                for (int lane = 0; lane < 32; ++lane) {
                    const int r = rt * 8 + (lane >> 2), q = kk * 4 + (lane & 3);
                    double v = 0.0;
                    if (r < np * np && q < nq) {
                        const int i = r / np, k = r % np;
                        v = (double)((d == 0 ? gx[i * nq + q] : gy[i * nq + q]) * phi[k * nq + q]);
                    }
                    qfrag.push_back(v);
                }
    return true;
}

// Morton key of a 2D point: 21 bits per axis over the bounding box, x in the even bits.
uint64_t morton(double x, double y, double x0, double y0, double sx, double sy) {
    auto qz = [](double v, double v0, double s) -> uint64_t {
        if (!(s > 0)) return 0;
        double f = std::floor((v - v0) / s * 2097152.0);
        if (f < 0) f = 0;
        if (f > 2097151.0) f = 2097151.0;
        return (uint64_t)f;
    };
    // interleave: x bit k -> position 2k, y bit k -> 2k+1
    const uint64_t ix = qz(x, x0, sx), iy = qz(y, y0, sy);
    uint64_t r = 0;
    for (int b = 0; b < 21; ++b) r |= ((ix >> b) & 1ull) << (2 * b) | ((iy >> b) & 1ull) << (2 * b + 1);
    return r;
}

template <typename F>
void parallel_for(int64_t n, F f) {
    int nt = (int)std::max(1u, std::thread::hardware_concurrency());
    nt = (int)std::min<int64_t>(nt, std::max<int64_t>(1, n));
    if (nt <= 1) {
        for (int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<int64_t> next(0);
    std::vector<std::thread> th;
    for (int k = 0; k < nt; ++k)
        th.emplace_back([&] {
            for (;;) {
                const int64_t i = next.fetch_add(1);
                if (i >= n) break;
                f(i);
            }
        });
    for (auto& t : th) t.join();
}

}  // namespace

// ------------------------------------------------------------------ ABI
extern "C" {

fea_status fea_create(fea_ctx* out, int cuda_device, void* stream, int rank, int world) {
    if (!out) return FEA_E_ARG;
    *out = nullptr;
    if (world < 1 || rank < 0 || rank >= world) return FEA_E_ARG;
    const bool host_only = cuda_device == -1;
    if (!host_only) {
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || cuda_device < 0 || cuda_device >= ndev) return FEA_E_CUDA;
        if (cudaSetDevice(cuda_device) != cudaSuccess) return FEA_E_CUDA;
    }
    fea_ctx c = new (std::nothrow) fea_ctx_s();
    if (!c) return FEA_E_OOM;
    c->host_only = host_only;
    c->device = host_only ? 0 : cuda_device;
    c->stream = (cudaStream_t)stream;
    c->rank = rank;
    c->world = world;
    if (!host_only) cudaDeviceGetAttribute(&c->sm_count, cudaDevAttrMultiProcessorCount, cuda_device);
    if (const char* dm = getenv("FEA_DEBUG_MODE")) c->dbg_mode = atoi(dm);  // diagnostics builds only
    c->dbg_timing = getenv("FEA_DEBUG_TIMING") != nullptr;
    c->coef_m.kind = c->coef_c.kind = FEA_K_POLY;
    c->coef_m.npar = c->coef_c.npar = 1;
    c->coef_m.par[0] = c->coef_c.par[0] = 1.0;
    *out = c;
    return FEA_OK;
}

void fea_destroy(fea_ctx c) {
    if (!c) return;
    if (!c->host_only) cudaSetDevice(c->device);
    c->free_mesh();
    if (c->stream2) cudaStreamDestroy(c->stream2);
    if (c->ev_own) cudaEventDestroy(c->ev_own);
    if (c->ev_halo) cudaEventDestroy(c->ev_halo);
    for (auto& e : c->ev_t)
        if (e) cudaEventDestroy(e);
    dfree(c->d_tables);
    dfree(c->d_ttab);
    dfree(c->d_tables_c);
    dfree(c->d_ttab_c);
    dfree(c->d_dbg);
    if (c->comm && nccl().ok) nccl().commDestroy((ncclComm_t)c->comm);
    if (c->h_send) cudaFreeHost(c->h_send);
    if (c->h_recv) cudaFreeHost(c->h_recv);
    delete c;
}

const char* fea_last_error(fea_ctx c) { return c ? c->err.c_str() : "null context"; }

// Rule checks and tables (Algorithm 2 lines 1-3) of one quadrature rule; device copies of the v4
// fragments and of the tensor kernel's tables.
static fea_status make_rule(fea_ctx c, int order, int n_q, const double* q_xy, const double* q_w,
                            std::vector<double>& ctab, std::vector<double>& qfrag, std::vector<double>& jplain) {
    if (!q_xy || !q_w) return c->fail(FEA_E_ARG, "NULL rule arrays");
    if (n_q < 1 || n_q > FEA_MAX_NQ) return c->fail(FEA_E_UNSUPPORTED, "n_q %d not in 1..16", n_q);
    long double s = 0;
    for (int q = 0; q < n_q; ++q) {
        if (!std::isfinite(q_w[q]) || !std::isfinite(q_xy[2 * q]) || !std::isfinite(q_xy[2 * q + 1]))
            return c->fail(FEA_E_ARG, "non-finite rule entry %d", q);
        s += q_w[q];
    }
    if (fabsl(s - 0.5L) > 1e-14L)
        return c->fail(FEA_E_ARG, "quadrature weights sum to %.17g, expected 1/2 (reference-triangle measure)", (double)s);
    if (!build_tables(order, n_q, q_xy, q_w, ctab, qfrag, jplain)) return c->fail(FEA_E_UNSUPPORTED, "singular Vandermonde");
    if (ctab.size() > FEA_CTAB_MAX) return c->fail(FEA_E_UNSUPPORTED, "tables exceed the parameter bank");
    return FEA_OK;
}

// Is the rule invariant under the 6 permutations of the barycentric coordinates (same points, same
// weights)?  Then an element may be relabelled by any vertex permutation without changing its
// quadrature sum beyond rounding (kernel v6 ghost row-tile skipping).
static bool rule_symmetric(int n_q, const double* q_xy, const double* q_w) {
    static const int P[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    for (int s = 0; s < 6; ++s)
        for (int q = 0; q < n_q; ++q) {
            const double l[3] = {1.0 - q_xy[2 * q] - q_xy[2 * q + 1], q_xy[2 * q], q_xy[2 * q + 1]};
            const double x = l[P[s][1]], y = l[P[s][2]];
            bool found = false;
            for (int r = 0; r < n_q && !found; ++r)
                found = std::fabs(q_xy[2 * r] - x) < 1e-12 && std::fabs(q_xy[2 * r + 1] - y) < 1e-12 &&
                        std::fabs(q_w[r] - q_w[q]) < 1e-14;
            if (!found) return false;
        }
    return true;
}

static fea_status upload_rule(fea_ctx c, int n_q, const std::vector<double>& ctab, const std::vector<double>& qfrag,
                              const std::vector<double>& jplain, double*& d_qfrag, double*& d_ttab) {
    dfree(d_qfrag);
    dfree(d_ttab);
    if (c->host_only) return FEA_OK;
    FEA_CUDA(c, cudaMalloc(&d_qfrag, qfrag.size() * sizeof(double)));
    FEA_CUDA(c, cudaMemcpy(d_qfrag, qfrag.data(), qfrag.size() * sizeof(double), cudaMemcpyHostToDevice));
    const int np = c->np;  // tensor kernel tables: Phi, J0, J1 [np][16], w [16], zero padded
    std::vector<double> tt((size_t)3 * np * 16 + 16, 0.0);
    for (int i = 0; i < np; ++i)
        for (int q = 0; q < n_q; ++q) {
            tt[(size_t)i * 16 + q] = ctab[(size_t)i * n_q + q];
            tt[(size_t)(np + i) * 16 + q] = jplain[(size_t)i * n_q + q];
            tt[(size_t)(2 * np + i) * 16 + q] = jplain[(size_t)(np + i) * n_q + q];
        }
    const size_t oW = ((size_t)np * n_q + 1) & ~size_t(1);
    for (int q = 0; q < n_q; ++q) tt[(size_t)3 * np * 16 + q] = ctab[oW + q];
    FEA_CUDA(c, cudaMalloc(&d_ttab, tt.size() * sizeof(double)));
    FEA_CUDA(c, cudaMemcpy(d_ttab, tt.data(), tt.size() * sizeof(double), cudaMemcpyHostToDevice));
    return FEA_OK;
}

fea_status fea_set_element(fea_ctx c, int order, int n_q, const double* q_xy, const double* q_w) {
    if (!c) return FEA_E_ARG;
    if (order < 1 || order > FEA_MAX_ORDER) return c->fail(FEA_E_UNSUPPORTED, "order %d not in 1..4", order);
    std::vector<double> ctab, qfrag, jplain;
    fea_status st = make_rule(c, order, n_q, q_xy, q_w, ctab, qfrag, jplain);
    if (st != FEA_OK) return st;
    if (!c->host_only) cudaSetDevice(c->device);
    c->free_mesh();
    c->order = order;
    c->nq = n_q;
    c->np = (order + 1) * (order + 2) / 2;
    c->T = c->np * (c->np + 1) / 2;
    c->qxy.assign(q_xy, q_xy + 2 * n_q);
    c->qw.assign(q_w, q_w + n_q);
    c->tables = ctab;
    c->qfrag = qfrag;
    c->jplain = jplain;
    c->split = false;
    c->rule_sym = rule_symmetric(n_q, q_xy, q_w);
    dfree(c->d_tables_c);
    dfree(c->d_ttab_c);
    return upload_rule(c, n_q, ctab, qfrag, jplain, c->d_tables, c->d_ttab);
}

fea_status fea_set_rule(fea_ctx c, int which, int n_q, const double* q_xy, const double* q_w) {
    if (!c) return FEA_E_ARG;
    if (c->order == 0) return c->fail(FEA_E_STATE, "set_rule before set_element");
    if (which < 1 || which > 3) return c->fail(FEA_E_ARG, "which must be a nonzero FEA_MASS|FEA_STIFF mask");
    if (which == (FEA_MASS | FEA_STIFF)) {  // one rule for both: as set_element, keeping the mesh
        std::vector<double> ctab, qfrag, jplain;
        fea_status st = make_rule(c, c->order, n_q, q_xy, q_w, ctab, qfrag, jplain);
        if (st != FEA_OK) return st;
        if (!c->host_only) cudaSetDevice(c->device);
        c->free_plan();
        c->nq = n_q;
        c->qxy.assign(q_xy, q_xy + 2 * n_q);
        c->qw.assign(q_w, q_w + n_q);
        c->tables = ctab;
        c->qfrag = qfrag;
        c->jplain = jplain;
        c->split = false;
        c->rule_sym = rule_symmetric(n_q, q_xy, q_w);
        dfree(c->d_tables_c);
        dfree(c->d_ttab_c);
        return upload_rule(c, n_q, ctab, qfrag, jplain, c->d_tables, c->d_ttab);
    }
    std::vector<double> ctab, qfrag, jplain;
    fea_status st = make_rule(c, c->order, n_q, q_xy, q_w, ctab, qfrag, jplain);
    if (st != FEA_OK) return st;
    if (!c->host_only) cudaSetDevice(c->device);
    c->free_plan();
    if (!c->split) {  // C keeps the current (common) rule
        c->nq_c = c->nq;
        c->qxy_c = c->qxy;
        c->qw_c = c->qw;
        c->tables_c = c->tables;
        c->qfrag_c = c->qfrag;
        c->jplain_c = c->jplain;
        st = upload_rule(c, c->nq_c, c->tables_c, c->qfrag_c, c->jplain_c, c->d_tables_c, c->d_ttab_c);
        if (st != FEA_OK) return st;
        c->split = true;
    }
    if (which == FEA_MASS) {
        c->nq = n_q;
        c->qxy.assign(q_xy, q_xy + 2 * n_q);
        c->qw.assign(q_w, q_w + n_q);
        c->tables = ctab;
        c->qfrag = qfrag;
        c->jplain = jplain;
        st = upload_rule(c, n_q, ctab, qfrag, jplain, c->d_tables, c->d_ttab);
    } else {
        c->nq_c = n_q;
        c->qxy_c.assign(q_xy, q_xy + 2 * n_q);
        c->qw_c.assign(q_w, q_w + n_q);
        c->tables_c = ctab;
        c->qfrag_c = qfrag;
        c->jplain_c = jplain;
        st = upload_rule(c, n_q, ctab, qfrag, jplain, c->d_tables_c, c->d_ttab_c);
    }
    if (st != FEA_OK) return st;
    if (c->nq == c->nq_c && c->qxy == c->qxy_c && c->qw == c->qw_c) {  // the same rule again
        c->split = false;
        dfree(c->d_tables_c);
        dfree(c->d_ttab_c);
    }
    return FEA_OK;
}

fea_status fea_mesh_upload(fea_ctx c, int64_t n_vert, const double* vert_xy, int64_t n_elem,
                           const int32_t* elem_vert, int64_t n_dof, const int32_t* elem_dof, int reorder) {
    if (!c) return FEA_E_ARG;
    if (c->order == 0) return c->fail(FEA_E_STATE, "mesh_upload before set_element");
    if (n_vert < 3 || n_elem < 1 || n_dof < 1 || !vert_xy || !elem_vert || !elem_dof)
        return c->fail(FEA_E_ARG, "mesh_upload: empty or NULL mesh");
    if (reorder != FEA_REORDER_NONE && reorder != FEA_REORDER_MORTON) return c->fail(FEA_E_ARG, "bad reorder flag");
    if (n_elem >= (1ll << 31) || n_dof >= (1ll << 31) || n_vert >= (1ll << 31))
        return c->fail(FEA_E_UNSUPPORTED, "mesh sizes must be < 2^31");
    const int np = c->np, p = c->order;
    int kk[FEA_MAX_NP][3];
    lib_nodes(p, kk);
    if (!c->host_only) cudaSetDevice(c->device);
    c->free_mesh();

    ptime("mesh_upload start");
    // validation + DOF coordinates (user numbering), element by element
    std::vector<double> uxy(2 * n_dof, 0.0);
    std::vector<int64_t> first(n_dof, -1);
    for (int64_t e = 0; e < n_elem; ++e) {
        const int32_t* v = elem_vert + 3 * e;
        for (int k = 0; k < 3; ++k)
            if (v[k] < 0 || v[k] >= n_vert) return c->fail(FEA_E_MESH, "element %lld: vertex index %d out of range", (long long)e, v[k]);
        const double* a = vert_xy + 2 * (int64_t)v[0];
        const double* b = vert_xy + 2 * (int64_t)v[1];
        const double* cc = vert_xy + 2 * (int64_t)v[2];
        const double B00 = b[0] - a[0], B10 = b[1] - a[1], B01 = cc[0] - a[0], B11 = cc[1] - a[1];
        const double det = B00 * B11 - B01 * B10;
        const double e2 = (cc[0] - b[0]) * (cc[0] - b[0]) + (cc[1] - b[1]) * (cc[1] - b[1]);
        const double diam2 = std::max(std::max(B00 * B00 + B10 * B10, B01 * B01 + B11 * B11), e2);
        if (!(std::fabs(det) >= 1e-14 * diam2)) return c->fail(FEA_E_MESH, "degenerate element %lld", (long long)e);
        const int32_t* d = elem_dof + (int64_t)np * e;
        for (int i = 0; i < np; ++i) {
            if (d[i] < 0 || d[i] >= n_dof) return c->fail(FEA_E_MESH, "element %lld: DOF index %d out of range", (long long)e, d[i]);
            for (int j = 0; j < i; ++j)
                if (d[j] == d[i]) return c->fail(FEA_E_MESH, "element %lld: repeated DOF %d", (long long)e, d[i]);
            const double x = (kk[i][0] * a[0] + kk[i][1] * b[0] + kk[i][2] * cc[0]) / p;
            const double y = (kk[i][0] * a[1] + kk[i][1] * b[1] + kk[i][2] * cc[1]) / p;
            if (first[d[i]] < 0) {
                first[d[i]] = e;
                uxy[2 * d[i]] = x;
                uxy[2 * d[i] + 1] = y;
            } else {
                const double dx = x - uxy[2 * d[i]], dy = y - uxy[2 * d[i] + 1];
                if (dx * dx + dy * dy > 1e-20 * diam2)
                    return c->fail(FEA_E_MESH, "DOF %d placed inconsistently by elements %lld and %lld (edge orientation?)",
                                   d[i], (long long)first[d[i]], (long long)e);
            }
        }
    }
    for (int64_t d = 0; d < n_dof; ++d)
        if (first[d] < 0) return c->fail(FEA_E_MESH, "DOF %lld is not referenced by any element", (long long)d);

    ptime("validation");
    // library DOF numbering
    std::vector<int64_t> lib2user(n_dof), user2lib(n_dof);
    std::iota(lib2user.begin(), lib2user.end(), 0);
    if (reorder == FEA_REORDER_MORTON) {
        double x0 = uxy[0], x1 = uxy[0], y0 = uxy[1], y1 = uxy[1];
        for (int64_t d = 0; d < n_dof; ++d) {
            x0 = std::min(x0, uxy[2 * d]);
            x1 = std::max(x1, uxy[2 * d]);
            y0 = std::min(y0, uxy[2 * d + 1]);
            y1 = std::max(y1, uxy[2 * d + 1]);
        }
        std::vector<uint64_t> key(n_dof);
        parallel_for((n_dof + 65535) / 65536, [&](int64_t blk) {
            const int64_t a = blk * 65536, b = std::min<int64_t>(n_dof, a + 65536);
            for (int64_t d = a; d < b; ++d) key[d] = morton(uxy[2 * d], uxy[2 * d + 1], x0, y0, x1 - x0, y1 - y0);
        });
        // (key, user id) pairs, sorted in parallel: the same order as a stable sort by key
        std::vector<std::pair<uint64_t, int64_t>> kp(n_dof);
        parallel_for((n_dof + 65535) / 65536, [&](int64_t blk) {
            const int64_t a = blk * 65536, b = std::min<int64_t>(n_dof, a + 65536);
            for (int64_t d = a; d < b; ++d) kp[d] = {key[d], d};
        });
        __gnu_parallel::sort(kp.begin(), kp.end());
        for (int64_t d = 0; d < n_dof; ++d) lib2user[d] = kp[d].second;
    }
    for (int64_t l = 0; l < n_dof; ++l) user2lib[lib2user[l]] = l;

    ptime("Morton DOF order");
    // library element order: by minimum library DOF, then user id
    std::vector<int32_t> emin(n_elem);
    for (int64_t e = 0; e < n_elem; ++e) {
        int64_t m = INT64_MAX;
        for (int i = 0; i < np; ++i) m = std::min(m, user2lib[elem_dof[(int64_t)np * e + i]]);
        emin[e] = (int32_t)m;
    }
    std::vector<int64_t> el2u(n_elem);
    std::iota(el2u.begin(), el2u.end(), 0);
    {  // (min DOF, user id) packed in 64 bits, sorted in parallel (= a stable sort by min DOF)
        std::vector<uint64_t> ek(n_elem);
        for (int64_t e = 0; e < n_elem; ++e) ek[e] = (uint64_t)(uint32_t)emin[e] << 32 | (uint64_t)e;
        __gnu_parallel::sort(ek.begin(), ek.end());
        for (int64_t e = 0; e < n_elem; ++e) el2u[e] = (int64_t)(ek[e] & 0xffffffffu);
    }

    ptime("element order");
    c->n_vert = n_vert;
    c->n_e = n_elem;
    c->n_dof = n_dof;
    c->dof_lib2user = lib2user;
    c->elem_lib2user = el2u;
    c->ed.resize((size_t)n_elem * np);
    c->elem_min.resize(n_elem);
    for (int64_t l = 0; l < n_elem; ++l) {
        const int64_t e = el2u[l];
        for (int i = 0; i < np; ++i) c->ed[(size_t)l * np + i] = (int32_t)user2lib[elem_dof[(int64_t)np * e + i]];
        c->elem_min[l] = emin[e];
    }
    c->dxy.resize(2 * n_dof);
    for (int64_t l = 0; l < n_dof; ++l) {
        c->dxy[2 * l] = uxy[2 * lib2user[l]];
        c->dxy[2 * l + 1] = uxy[2 * lib2user[l] + 1];
    }
    if (c->host_only) {
        c->have_mesh = true;
        return FEA_OK;
    }
    ptime("library numbering");
    // device: DOF coordinates (vertex DOFs give B_e); the DOF map travels in the block records
    FEA_CUDA(c, cudaMalloc(&c->d_xy, n_dof * sizeof(double2)));
    FEA_CUDA(c, cudaMemcpy(c->d_xy, c->dxy.data(), n_dof * sizeof(double2), cudaMemcpyHostToDevice));
    c->have_mesh = true;
    return FEA_OK;
}

fea_status fea_set_tuning(fea_ctx c, int key, int64_t value) {
    if (!c) return FEA_E_ARG;
    switch (key) {
        case FEA_TUNE_SMEM_BUDGET:
            if (value != 0 && (value < 4096 || value > 232448)) return c->fail(FEA_E_ARG, "smem budget out of range");
            c->tune_smem = value;
            break;
        case 2:  // kernel generation (0 = automatic, 4 = force v4)
            if (value != 0 && value != 4 && value != 5 && value != 6) return c->fail(FEA_E_ARG, "kernel must be 0, 4, 5 or 6");
            c->tune_kver = (int)value;
            break;
        case 3:  // v5 elements per block cap
            if (value < 0 || value > 65535) return c->fail(FEA_E_ARG, "element cap out of range");
            c->tune_emax = value;
            break;
        case 7:  // world > 1: overlap the exchange with the interior blocks (1, default) or not (0)
            if (value != 0 && value != 1) return c->fail(FEA_E_ARG, "overlap flag must be 0 or 1");
            c->tune_overlap = (int)value;
            break;
        case 5:  // exchange of u between ranks: 0 = interface-only, 1 = full allgather
            if (value != 0 && value != 1) return c->fail(FEA_E_ARG, "exchange must be 0 or 1");
            c->exchange = (int)value;
            break;
        case 10:  // v5 phase B: pad single-contributor slots into the two-contributor class (1) or not (0)
            if (value != 0 && value != 1) return c->fail(FEA_E_ARG, "pad flag must be 0 or 1");
            c->tune_pad1 = (int)value;
            break;
        case 8:  // tensor kernel: 0 = automatic, 1 = lane per element (k_tensor), 4 = DMMA (k_tensor4),
                 // 5 = the pipelined lane-per-element kernel (k_tensor5; P1 with the 3-point rule)
            if (value != 0 && value != 1 && value != 4 && value != 5)
                return c->fail(FEA_E_ARG, "tensor kernel must be 0, 1, 4 or 5");
            c->tune_tker = (int)value;
            break;
        case 12:  // kernel v6: ghost row-tile skipping with element rotations (1, default) or off (0)
            if (value != 0 && value != 1) return c->fail(FEA_E_ARG, "skip flag must be 0 or 1");
            c->tune_skip = (int)value;
            break;
        case 11:  // per-call timing events (fea_get_stat keys 36, 37)
            if (value != 0 && value != 1) return c->fail(FEA_E_ARG, "timing flag must be 0 or 1");
            c->tune_timing = (int)value;
            return FEA_OK;  // does not change the plan
        case 4:  // plan matrices bitmask (FEA_MASS | FEA_STIFF)
            if (value < 1 || value > 3) return c->fail(FEA_E_ARG, "plan matrices must be a nonzero MASS|STIFF mask");
            c->plan_which = (int)value;
            break;
        default:
            return c->fail(FEA_E_ARG, "unknown tuning key %d", key);
    }
    if (c->have_plan) c->free_plan();
    return FEA_OK;
}

// Permutation of a class's n items (C contributor offsets each, item-major) that keeps every item
// in its aligned group of 32 and assigns each group's items to the two half-warps (16 + 16)
// greedily, minimising repeated 8-byte banks (offset mod 16, orientation bit masked) per
// contributor index within a half.  Phase B's sums do not depend on the item order.
// Item order within each aligned group of 32 items (one warp instruction of phase B: the classes
// start warp-aligned, fea_device.cuh phase_b5): the group is split into the lane subsets that the
// shared-memory V reads are served in -- half-warps for 8-byte reads (bank key: offset mod 16),
// quarter-warps for the 16-byte {m, c} reads of interleaved V (key: offset mod 8) -- greedily
// so each subset's keys are distinct where possible.  The group still covers the same 32 slots.
static std::vector<int32_t> bank_split_order(const uint16_t* off, int n, int C, bool quarter) {
    const int NSUB = quarter ? 4 : 2, SUB = 32 / NSUB, KEYS = quarter ? 8 : 16;
    std::vector<int32_t> ord(n);
    for (int g = 0; g < n; g += 32) {
        const int gn = std::min(32, n - g);
        if (gn <= SUB) {
            for (int l = 0; l < gn; ++l) ord[g + l] = g + l;
            continue;
        }
        std::vector<int32_t> sub[4];
        int cnt[4][16][8] = {};  // [subset][key][q] (C <= 8 tracked; more is rare)
        const int Cq = std::min(C, 8);
        // capacity of each subset: lanes of the group that exist (the last group may be partial)
        int cap[4];
        for (int h = 0; h < NSUB; ++h) cap[h] = std::max(0, std::min(SUB, gn - h * SUB));
        for (int l = 0; l < gn; ++l) {
            const int i = g + l;
            int best = -1, bcost = 1 << 30;
            for (int h = 0; h < NSUB; ++h) {
                if ((int)sub[h].size() >= cap[h]) continue;
                int cost = 0;
                for (int q = 0; q < Cq; ++q) cost += cnt[h][(off[(size_t)i * C + q] & 0x7fff) % KEYS][q];
                if (cost < bcost) {
                    bcost = cost;
                    best = h;
                }
            }
            sub[best].push_back(i);
            for (int q = 0; q < Cq; ++q) cnt[best][(off[(size_t)i * C + q] & 0x7fff) % KEYS][q]++;
        }
        int l = 0;
        for (int h = 0; h < NSUB; ++h)
            for (int32_t i : sub[h]) ord[g + l++] = i;
    }
    return ord;
}

// Host plan of one kernel family: row blocks of this rank's rows, each with its element set
// (ghosts first), its CSR slots and the per-slot contributor lists (ascending library element),
// encoded as the kernel's block record.  v5 = class/item record + separate DOF array; else the
// v4 record (DOFs inside).  orient: bit 15 of each contributor offset = (local i > local j), for
// nonsymmetric element matrices (the tensor contraction C o2 v).
struct PlanData {
    std::vector<FeaBlock> blocks;
    dvec<uint8_t> records;
    dvec<int32_t> dofs;
    std::vector<int64_t> row_ptr;
    dvec<int32_t> col_idx;
    int64_t nnz = 0, rec_max = 16, visits = 0, owned = 0, ncon = 0, rbytes = 0;
};

// v6: kernel v6 record (fea_internal.h): class-A u32 items in slot order + class-B items; the
// DOFs travel separately as for v5 (pass v5 = true); records stay in global memory.
static fea_status build_blocks(fea_ctx c, bool v5, bool orient, int64_t e_max, int64_t rec_budget, int64_t EM,
                               PlanData& P, bool il = false, bool v6 = false, int64_t vcap = 0) {
    const int np = c->np, T = c->T;
    const int64_t n_e = c->n_e;
    const int64_t R0 = c->row_begin, nr = c->n_rows;
    const int64_t R1 = R0 + nr;
    // ---- incidence of this rank's rows (ascending library element per row)
    std::vector<int64_t> iptr(nr + 1, 0);
    for (int64_t e = 0; e < n_e; ++e)
        for (int i = 0; i < np; ++i) {
            const int64_t d = c->ed[(size_t)e * np + i];
            if (d >= R0 && d < R1) iptr[d - R0 + 1]++;
        }
    for (int64_t r = 0; r < nr; ++r) iptr[r + 1] += iptr[r];
    std::vector<int32_t> inc(std::max<int64_t>(1, iptr[nr]));
    {
        std::vector<int64_t> pos(iptr.begin(), iptr.end() - 1);
        for (int64_t e = 0; e < n_e; ++e)
            for (int i = 0; i < np; ++i) {
                const int64_t d = c->ed[(size_t)e * np + i];
                if (d >= R0 && d < R1) inc[pos[d - R0]++] = (int32_t)e;
            }
    }
    int64_t max_inc = 0;
    for (int64_t r = 0; r < nr; ++r) max_inc = std::max(max_inc, iptr[r + 1] - iptr[r]);
    if (max_inc > 255) return c->fail(FEA_E_UNSUPPORTED, "a DOF belongs to %lld elements (> 255)", (long long)max_inc);
    // one row must fit a block: its elements and its record upper bound
    const int64_t row_ub_max = max_inc * np * 4 + 4 * np * (max_inc + 3) + 32 * FEA_MAX_CLASSES + 96;
    if (e_max < std::max<int64_t>(max_inc, 1) || rec_budget < row_ub_max)
        return c->fail(FEA_E_UNSUPPORTED, "shared-memory budget too small: %lld elements per block", (long long)e_max);
    if (orient && (int64_t)T * EM >= 32768)
        return c->fail(FEA_E_UNSUPPORTED, "tensor plan: V offsets need 15 bits");

    ptime("plan: incidence");
    // ---- greedy row blocks: elements <= e_max and record upper bound <= rec_budget
    // record upper bound: slots <= entries, so counts + contrib + chunks <= 3 entries + entries/8
    std::vector<int64_t> brow;
    {
        std::vector<int32_t> mark(n_e, -1);
        int32_t cur = -1;
        int64_t nE = 0, ent = 0;
        for (int64_t r = 0; r < nr; ++r) {
            int64_t add = 0;
            for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) add += mark[inc[k]] != cur;
            const int64_t rent = (iptr[r + 1] - iptr[r]) * np;
            const int64_t ub = 4 * (ent + rent) + (v5 ? 0 : 4 * np * (nE + add + 3) + 32) + 32 * FEA_MAX_CLASSES + 64;
            if (cur < 0 || nE + add > e_max || ub > rec_budget) {
                ++cur;
                brow.push_back(r);
                nE = 0;
                ent = 0;
                add = iptr[r + 1] - iptr[r];
            }
            for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) mark[inc[k]] = cur;
            nE += add;
            ent += rent;
        }
    }
    brow.push_back(nr);

    ptime("plan: row blocks");
    // ---- kernel v6 row-tile skipping (FEA_TUNE_SKIP): an element recomputed as a ghost needs only
    // the V rows (i, j) with i or j one of its DOFs in the block's rows; it is relabelled by the
    // vertex permutation (of 6; the rule must be symmetric) that packs those rows into the fewest
    // 8-row DMMA tiles, and the block's elements are ordered by their tile masks so each 8-element
    // column tile skips the row tiles none of its elements needs.
    const bool skip = v6 && c->tune_skip;
    const int nperm = skip && c->rule_sym ? 6 : 1;
    int sig[6][FEA_MAX_NP], siginv[6][FEA_MAX_NP];
    uint32_t rowmask[FEA_MAX_NP];
    {
        static const int PP[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        int kk[FEA_MAX_NP][3];
        lib_nodes(c->order, kk);
        for (int sp = 0; sp < 6; ++sp)
            for (int i = 0; i < np; ++i) {
                const int t0 = kk[i][PP[sp][0]], t1 = kk[i][PP[sp][1]], t2 = kk[i][PP[sp][2]];
                for (int k = 0; k < np; ++k)
                    if (kk[k][0] == t0 && kk[k][1] == t1 && kk[k][2] == t2) sig[sp][i] = k;
            }
        for (int sp = 0; sp < 6; ++sp)
            for (int i = 0; i < np; ++i) siginv[sp][sig[sp][i]] = i;
        for (int a = 0; a < np; ++a) {
            rowmask[a] = 0;
            for (int b2 = 0; b2 < np; ++b2) rowmask[a] |= 1u << (tri_index(np, std::min(a, b2), std::max(a, b2)) / 8);
        }
    }
    const int NTT6 = (T + 7) / 8;
    // a block's elements E (ascending library element), their relabelling rot, row-tile masks
    // emask, column positions newpos (sorted by mask) and the column tiles' masks ctm
    auto layout_block = [&](int64_t ra, int64_t rb, std::vector<int32_t>& E, std::vector<int8_t>& rot,
                            std::vector<uint32_t>& emask, std::vector<int32_t>& newpos, std::vector<uint32_t>& ctm) {
        const int64_t ga = R0 + ra, gb = R0 + rb;
        E.clear();
        for (int64_t r = ra; r < rb; ++r) E.insert(E.end(), inc.begin() + iptr[r], inc.begin() + iptr[r + 1]);
        std::sort(E.begin(), E.end());
        E.erase(std::unique(E.begin(), E.end()), E.end());
        const int64_t nE0 = (int64_t)E.size();
        rot.assign(nE0, 0);
        emask.assign(nE0, (1u << NTT6) - 1);
        newpos.resize(nE0);
        std::iota(newpos.begin(), newpos.end(), 0);
        if (skip) {
            for (int64_t le = 0; le < nE0; ++le) {
                const int32_t* d = &c->ed[(size_t)E[le] * np];
                uint32_t best = ~0u;
                int bs = 0;
                for (int sp = 0; sp < nperm; ++sp) {
                    uint32_t m = 0;
                    for (int i = 0; i < np; ++i)
                        if (d[i] >= ga && d[i] < gb) m |= rowmask[sig[sp][i]];
                    if (__builtin_popcount(m) < __builtin_popcount(best)) {
                        best = m;
                        bs = sp;
                    }
                }
                rot[le] = (int8_t)bs;
                emask[le] = best;
            }
            std::vector<int32_t> ord(nE0);
            std::iota(ord.begin(), ord.end(), 0);
            std::stable_sort(ord.begin(), ord.end(), [&](int32_t x, int32_t y) {
                const int px = __builtin_popcount(emask[x]), py = __builtin_popcount(emask[y]);
                return px != py ? px > py : emask[x] < emask[y];
            });
            for (int64_t q = 0; q < nE0; ++q) newpos[ord[q]] = (int32_t)q;
        }
        ctm.assign((nE0 + 7) / 8, 0);
        for (int64_t le0 = 0; le0 < nE0; ++le0) ctm[newpos[le0] / 8] |= emask[le0];
    };
    // ---- v6 compact V (FEA6_VCOMPACT): a block's V needs 1 + 64 sum_et popc(m_et) cells; a greedy
    // block over the capacity is cut at its longest row prefix that fits, the rest starts a block
    if (v6 && vcap > 0) {
        const int64_t nb0 = (int64_t)brow.size() - 1;
        std::vector<std::vector<int64_t>> cuts(nb0);
        std::atomic<int> bad(0);
        parallel_for(nb0, [&](int64_t b) {
            std::vector<int32_t> E, newpos;
            std::vector<int8_t> rot;
            std::vector<uint32_t> emask, ctm;
            auto cells = [&](int64_t ra, int64_t rb) {
                layout_block(ra, rb, E, rot, emask, newpos, ctm);
                int64_t t = 0;
                for (uint32_t m : ctm) t += __builtin_popcount(m);
                return 1 + 64 * t;
            };
            int64_t ra = brow[b];
            const int64_t rb = brow[b + 1];
            while (ra < rb) {
                if (cells(ra, rb) <= vcap) {
                    cuts[b].push_back(ra);
                    break;
                }
                int64_t lo = ra + 1, hi = rb - 1;  // the longest fitting prefix [ra, lo) (a single row must fit)
                if (cells(ra, lo) > vcap) {
                    bad = 1;
                    return;
                }
                while (lo < hi) {
                    const int64_t mid = (lo + hi + 1) / 2;
                    if (cells(ra, mid) <= vcap) lo = mid;
                    else hi = mid - 1;
                }
                cuts[b].push_back(ra);
                ra = lo;
            }
        });
        if (bad) return c->fail(FEA_E_UNSUPPORTED, "compact V: one row's elements exceed %lld cells", (long long)vcap);
        std::vector<int64_t> brow2;
        for (int64_t b = 0; b < nb0; ++b) brow2.insert(brow2.end(), cuts[b].begin(), cuts[b].end());
        brow2.push_back(nr);
        brow.swap(brow2);
        ptime("plan: compact-V block cuts");
    }
    const int64_t nb = (int64_t)brow.size() - 1;
    std::atomic<int64_t> skip_work(0), skip_full(0), skip_crit(0);
    std::atomic<int64_t> tile_use[32];
    for (auto& x : tile_use) x = 0;
    // ---- per block: element set, (row, col) records sorted -> slots, contributors, record
    struct BOut {
        std::vector<int32_t> rownnz, cols, dofs;
        std::vector<uint8_t> rec;
        FeaBlock fb{};
        int64_t nghost = 0, nown = 0;
        std::string err;
    };
    std::vector<BOut> bo(nb);
    parallel_for(nb, [&](int64_t b) {
        BOut& o = bo[b];
        const int64_t ra = brow[b], rb = brow[b + 1];
        const int64_t ga = R0 + ra, gb = R0 + rb;  // global library rows
        std::vector<int32_t> E, newpos;
        std::vector<int8_t> rot;
        std::vector<uint32_t> emask, ctm;
        layout_block(ra, rb, E, rot, emask, newpos, ctm);  // (element relabelling and column order: identity unless v6 skipping)
        for (int32_t e : E) (c->elem_min[e] < ga ? o.nghost : o.nown)++;
        {  // interior: every DOF of every element of the block is owned by this rank (overlap, NEXT-3)
            bool inside = true;
            for (int32_t e : E)
                for (int i = 0; i < np && inside; ++i) {
                    const int32_t d = c->ed[(size_t)e * np + i];
                    inside = d >= R0 && d < R1;
                }
            o.fb.spare_[0] = inside ? 1 : 0;
        }
        std::vector<int32_t> cb(ctm.size() + 1, 0);  // compact V: needed row tiles before column tile et
        for (size_t et = 0; et < ctm.size(); ++et) cb[et + 1] = cb[et] + __builtin_popcount(ctm[et]);
        struct Rec { int32_t row, col, le, t; };  // t: V row (| 0x10000 if orient and i > j: Vdn)
        std::vector<Rec> recs;
        recs.reserve((size_t)(iptr[rb] - iptr[ra]) * np);
        // row by row (the incident elements in ascending library element order), each row's
        // records sorted by column -- stable, so a slot's contributors stay in ascending le
        for (int64_t r = ra; r < rb; ++r) {
            const size_t r0 = recs.size();
            for (int64_t k = iptr[r]; k < iptr[r + 1]; ++k) {
                const int32_t e = inc[k];
                const int32_t le0 = (int32_t)(std::lower_bound(E.begin(), E.end(), e) - E.begin());
                const int32_t le = newpos[le0];
                const int* sg = sig[(int)rot[le0]];
                const int32_t* d = &c->ed[(size_t)e * np];
                for (int i = 0; i < np; ++i) {
                    if (d[i] != R0 + r) continue;
                    for (int j = 0; j < np; ++j) {
                        // tensor plans (orient): V row fea_trow (off-diagonal pairs first), flag i > j;
                        // v6: the row of the relabelled pair (sigma(i), sigma(j))
                        const int a = sg[i], b2 = sg[j];
                        recs.push_back({d[i], d[j], le,
                                        orient ? fea_trow(np, std::min(i, j), std::max(i, j)) | (i > j ? 0x10000 : 0)
                                               : tri_index(np, std::min(a, b2), std::max(a, b2))});
                    }
                }
            }
            // stable insertion sort by column (a row has a few dozen records; no allocation)
            for (size_t a = r0 + 1; a < recs.size(); ++a) {
                const Rec x = recs[a];
                size_t q = a;
                while (q > r0 && recs[q - 1].col > x.col) {
                    recs[q] = recs[q - 1];
                    --q;
                }
                recs[q] = x;
            }
        }
        // slots (row, col) in CSR order, each with its contributors in ascending le
        std::vector<int32_t> sstart, scount;  // per slot: first record, count
        o.rownnz.assign(rb - ra, 0);
        size_t k = 0;
        while (k < recs.size()) {
            size_t k2 = k;
            while (k2 < recs.size() && recs[k2].row == recs[k].row && recs[k2].col == recs[k].col) ++k2;
            sstart.push_back((int32_t)k);
            scount.push_back((int32_t)(k2 - k));
            o.cols.push_back(recs[k].col);
            o.rownnz[recs[k].row - ga]++;
            k = k2;
        }
        const int32_t nslot = (int32_t)sstart.size();
        // V cell of (symmetric row t, column le): dense t EM + le, or the compact layout (fea6_vcell)
        auto vcell = [&](int32_t t, int32_t le) -> uint32_t {
            if (vcap <= 0) return (uint32_t)(t * EM + le);
            const uint32_t mk = ctm[le / 8];
            if (!((mk >> (t / 8)) & 1u)) o.err = "compact V: a contribution outside its column tile's mask";
            return (uint32_t)fea6_vcell(cb[le / 8], mk, t / 8, t % 8, le % 8);
        };
        if (v6 || (v5 && !orient && FEA5_SLOT)) {  // kernel v6 (and v5) record: class A in slot order, class B as flat items
            if (nslot > 65535) {
                o.err = "more than 65535 slots in one block";
                return;
            }
            const int32_t nA = (nslot + 31) & ~31;
            std::vector<uint32_t> ia(nA, 0xffffffffu);
            std::vector<int32_t> clsB;  // slots with more than two contributors
            int32_t cmax = 0;
            for (int32_t sl = 0; sl < nslot; ++sl) {
                const int32_t C = scount[sl];
                auto off = [&](int32_t m) { return vcell(recs[m].t & 0xffff, recs[m].le); };
                if (C == 1) ia[sl] = off(sstart[sl]) | (uint32_t)(vcap > 0 ? 0 : e_max) << 16;  // + the zero cell
                else if (C == 2) ia[sl] = off(sstart[sl]) | off(sstart[sl] + 1) << 16;
                else {
                    clsB.push_back(sl);
                    cmax = std::max(cmax, C);
                }
            }
            // class B item: {u16 block-local slot, u16 C, u16 V offset [C]}, all items of the block
            // padded to one size R (16, 32, 48 or 64 bytes: C <= 30)
            const int32_t R = clsB.empty() ? 0 : fea_pad16(2 * (cmax + 2));
            if (R > 64) {
                o.err = "a slot with more than 30 contributors (kernel v6)";
                return;
            }
            const int32_t bytes = (4 * nA + (int32_t)clsB.size() * R + 127) & ~127;
            if (bytes > rec_budget) {  // v5: the record must fit its shared-memory stage
                o.err = "record exceeds the shared-memory budget";
                return;
            }
            o.rec.assign(bytes, 0);
            std::memcpy(o.rec.data(), ia.data(), 4 * (size_t)nA);
            for (size_t it = 0; it < clsB.size(); ++it) {
                const int32_t sl = clsB[it];
                uint16_t* w = reinterpret_cast<uint16_t*>(o.rec.data() + 4 * nA + it * R);
                w[0] = (uint16_t)sl;
                w[1] = (uint16_t)scount[sl];
                for (int q = 0; q < scount[sl]; ++q) {
                    const int32_t m = sstart[sl] + q;
                    w[2 + q] = (uint16_t)vcell(recs[m].t & 0xffff, recs[m].le);
                }
            }
            const int32_t ncl = (int32_t)clsB.size();
            FeaBlock& F = o.fb;
            F.nslots = nslot;
            F.ncontrib = (int32_t)recs.size();
            F.nE = (int32_t)E.size();
            F.ncls = ncl;  // v6: class-B items
            F.pad_ = R;    // v6: class-B item bytes
            F.rec_bytes = bytes;
            F.r0 = (int32_t)ga;
            F.nr = (int32_t)(gb - ga);
            const int32_t nEp = fea_pad4(F.nE);
            const int32_t net = (F.nE + 7) / 8;
            // DOFs [np][nEp] in column order (relabelled: new local k = old sigma^-1(k)), then v6's
            // row-tile mask of every 8-element column tile [net]
            o.dofs.assign((size_t)np * nEp + (v6 ? net : 0), 0);
            for (int64_t le0 = 0; le0 < (int64_t)E.size(); ++le0) {
                const int* si = siginv[(int)rot[le0]];
                for (int k = 0; k < np; ++k) o.dofs[k * nEp + newpos[le0]] = c->ed[(size_t)E[le0] * np + si[k]];
            }
            for (int64_t le = E.size(); le < nEp; ++le)
                for (int i = 0; i < np; ++i) o.dofs[i * nEp + le] = o.dofs[i * nEp];
            if (v6) {
                int64_t w = 0, ww[32] = {0};
                const int na = fea6_na(c->order), rt = fea6_rt(c->order);
                int own[32];  // the A warp holding each row tile (the kernel's map)
                for (int wq = 0; wq < na; ++wq)
                    for (int r = 0; r < rt; ++r)
                        if (fea6_tile(c->order, wq, r) >= 0) own[fea6_tile(c->order, wq, r)] = wq;
                for (int32_t et = 0; et < net; ++et) {
                    uint32_t m = 0;
                    for (int64_t le0 = 0; le0 < (int64_t)E.size(); ++le0)
                        if (newpos[le0] / 8 == et) m |= emask[le0];
                    o.dofs[(size_t)np * nEp + et] = (int32_t)m;
                    w += __builtin_popcount(m);
                    for (int tt = 0; tt < NTT6; ++tt) {
                        ww[own[tt]] += (m >> tt) & 1u;
                        tile_use[tt] += (m >> tt) & 1u;
                    }
                }
                skip_work += w;
                skip_crit += na * *std::max_element(ww, ww + na);
                skip_full += (int64_t)net * NTT6;
            }
            return;
        }
        // items: slots sorted by (count, slot); classes of equal count
        std::vector<int32_t> order(nslot);
        std::iota(order.begin(), order.end(), 0);
        // v5: single-contributor slots join the two-contributor class with a second read of a
        // zero cell (V row 0, column e_max: never written by the kernel, zeroed at its start), so
        // each warp's stores of that class cover denser slot ranges (C2: ~16 -> ~9 sectors per
        // store instruction); the sum is unchanged (x + 0.0).
        bool pad1 = v5 && !v6 && !orient && c->tune_pad1 && EM > e_max;
        if (pad1) {  // only where the padded record still fits the block's record budget
            std::map<int32_t, int32_t> n_by;
            for (int32_t sl = 0; sl < nslot; ++sl) n_by[scount[sl] == 1 ? 2 : scount[sl]]++;
            int64_t sz = 16 * (int64_t)n_by.size();
            for (const auto& kv : n_by) sz += fea_pad16(kv.second * fea5_item_bytes(kv.first));
            pad1 = sz <= rec_budget;
        }
        auto ecount = [&](int32_t sl) { return pad1 && scount[sl] == 1 ? 2 : scount[sl]; };
        std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return ecount(x) < ecount(y); });
        std::vector<int32_t> cls;
        std::vector<uint16_t> items(nslot), contrib;
        contrib.reserve(recs.size());
        for (int32_t it = 0; it < nslot; ++it) {
            const int32_t sl = order[it];
            if (it == 0 || ecount(sl) != ecount(order[it - 1])) {
                cls.push_back(ecount(sl));
                cls.push_back(it);
                cls.push_back((int32_t)contrib.size());
            }
            if (sl > 65535) {
                o.err = "more than 65536 slots in one block";
                return;
            }
            items[it] = (uint16_t)sl;
            for (int32_t m = sstart[sl]; m < sstart[sl] + scount[sl]; ++m)
                contrib.push_back((uint16_t)(((recs[m].t & 0xffff) * EM + recs[m].le) | ((recs[m].t >> 16) << 15)));
            if (ecount(sl) != scount[sl]) contrib.push_back((uint16_t)e_max);  // the zero cell
        }
        FeaBlock& F = o.fb;
        F.nslots = nslot;
        F.ncontrib = (int32_t)contrib.size();
        F.nE = (int32_t)E.size();
        F.ncls = (int32_t)(cls.size() / 3);
        if (F.ncls > FEA_MAX_CLASSES) {
            o.err = "too many contributor-count classes";
            return;
        }
        // class table + fixed-size item records (fea_internal.h), at byte `base` of the record:
        // v5 records are only this; v4 records put a FeaRecHdr4 before and the DOFs after it
        const int32_t base = v5 ? 0 : 32;
        const int ncl = F.ncls;
        std::vector<int32_t> coff(ncl);
        int32_t off = 16 * ncl;
        for (int k2 = 0; k2 < ncl; ++k2) {
            const int C = cls[3 * k2], n = (k2 + 1 < ncl ? cls[3 * k2 + 4] : nslot) - cls[3 * k2 + 1];
            coff[k2] = off;
            off += fea_pad16(n * fea5_item_bytes(C));
        }
        const int32_t nEp4 = fea_pad4(F.nE);
        const int32_t dofs_off = base + off;
        F.rec_bytes = v5 ? off : dofs_off + 4 * np * nEp4;
        if (F.rec_bytes > rec_budget) {
            o.err = "record exceeds the shared-memory budget";
            return;
        }
        o.rec.assign(F.rec_bytes, 0);
        int32_t* tab = reinterpret_cast<int32_t*>(o.rec.data() + base);
        for (int k2 = 0; k2 < ncl; ++k2) {
            const int C = cls[3 * k2], i0 = cls[3 * k2 + 1], n = (k2 + 1 < ncl ? cls[3 * k2 + 4] : nslot) - i0;
            const int R = fea5_item_bytes(C);
            tab[4 * k2] = C;
            tab[4 * k2 + 1] = n;
            tab[4 * k2 + 2] = coff[k2];
            tab[4 * k2 + 3] = R;
            // items in slot order within the class, each aligned group of 32 items (one warp
            // instruction of phase B) ordered by bank_split_order
            const std::vector<int32_t> ord = bank_split_order(&contrib[cls[3 * k2 + 2]], n, C, il);
            for (int it = 0; it < n; ++it) {
                const int src = ord[it];
                uint16_t* w = reinterpret_cast<uint16_t*>(o.rec.data() + base + coff[k2] + (size_t)it * R);
                w[0] = items[i0 + src];
                for (int q = 0; q < C; ++q) w[1 + q] = contrib[cls[3 * k2 + 2] + (size_t)src * C + q];
            }
        }
        if (!v5) {
            FeaRecHdr4* h = reinterpret_cast<FeaRecHdr4*>(o.rec.data());
            h->nE = F.nE;
            h->ncls = F.ncls;
            h->nslots = nslot;
            h->dofs_off = dofs_off;
            h->slot0 = 0;  // filled at concatenation (fea_build_pattern)
        }
        const int32_t nEp = nEp4;
        if (v5) o.dofs.assign((size_t)np * nEp, 0);
        F.r0 = (int32_t)ga;
        F.nr = (int32_t)(gb - ga);
        int32_t* dofs = v5 ? o.dofs.data() : reinterpret_cast<int32_t*>(o.rec.data() + dofs_off);
        for (int64_t le = 0; le < (int64_t)E.size(); ++le)
            for (int i = 0; i < np; ++i) dofs[i * nEp + le] = c->ed[(size_t)E[le] * np + i];
        for (int64_t le = E.size(); le < nEp; ++le)  // padding lanes point at a valid DOF
            for (int i = 0; i < np; ++i) dofs[i * nEp + le] = dofs[i * nEp];
    });
    for (auto& o : bo)
        if (!o.err.empty()) return c->fail(FEA_E_UNSUPPORTED, "plan: %s", o.err.c_str());

    ptime("plan: block records");
    // ---- concatenate
    std::vector<FeaBlock> blocks(nb);
    int64_t nnz = 0, rbytes = 0, ncon = 0, visits = 0, owned = 0, rec_max = 16, ndofs = 0;
    for (int64_t b = 0; b < nb; ++b) {
        FeaBlock& B = blocks[b];
        B = bo[b].fb;
        B.slot0 = nnz;
        B.rec_off = rbytes;
        B.dof_off = ndofs;
        ndofs += (int64_t)bo[b].dofs.size();
        nnz += B.nslots;
        rbytes += B.rec_bytes;
        ncon += B.ncontrib;
        visits += B.nE;
        owned += bo[b].nown;
        rec_max = std::max<int64_t>(rec_max, B.rec_bytes);
    }
    if (nnz >= (1ll << 31)) return c->fail(FEA_E_UNSUPPORTED, "nnz %lld >= 2^31 on one rank", (long long)nnz);
    std::vector<int64_t>& row_ptr = P.row_ptr;
    auto& col_idx = P.col_idx;
    row_ptr.assign(nr + 1, 0);
    col_idx.resize(nnz);  // default-initialised (no zero fill): every element is written below
    P.records.resize(std::max<int64_t>(rbytes, 16));
    P.dofs.resize(std::max<int64_t>(ndofs, 4));
    auto& records = P.records;
    auto& alldofs = P.dofs;
    parallel_for(nb, [&](int64_t b) {
        const FeaBlock& B = blocks[b];
        std::copy(bo[b].dofs.begin(), bo[b].dofs.end(), alldofs.begin() + B.dof_off);
        std::copy(bo[b].cols.begin(), bo[b].cols.end(), col_idx.begin() + B.slot0);
        std::memcpy(records.data() + B.rec_off, bo[b].rec.data(), B.rec_bytes);
        if (!v5) reinterpret_cast<FeaRecHdr4*>(records.data() + B.rec_off)->slot0 = B.slot0;
        for (int64_t r = brow[b]; r < brow[b + 1]; ++r) row_ptr[r + 1] = bo[b].rownnz[r - brow[b]];
        bo[b] = BOut();  // the per-block buffers are released here, in parallel
    });
    for (int64_t r = 0; r < nr; ++r) row_ptr[r + 1] += row_ptr[r];
    bo.clear();
    P.blocks.swap(blocks);
    P.nnz = nnz;
    P.rec_max = rec_max;
    P.visits = visits;
    P.owned = owned;
    P.ncon = ncon;
    P.rbytes = rbytes;
    if (v6) {
        c->skip_work = skip_work;
        c->skip_full = skip_full;
        c->skip_crit = skip_crit;
        if (getenv("FEA_PLAN_TIMING")) {
            fprintf(stderr, "[plan] v6 row-tile use:");
            for (int tt = 0; tt < NTT6; ++tt) fprintf(stderr, " %lld", (long long)tile_use[tt].load());
            fprintf(stderr, "\n");
        }
    }
    ptime("plan: concatenate");
    return FEA_OK;
}


fea_status fea_build_pattern(fea_ctx c, int64_t* row_begin, int64_t* n_rows_local, int64_t* nnz_local) {
    if (!c) return FEA_E_ARG;
    if (!c->have_mesh) return c->fail(FEA_E_STATE, "build_pattern before mesh_upload");
    if (!c->host_only) cudaSetDevice(c->device);
    c->free_plan();
    const int np = c->np, T = c->T, nq = c->nq;
    const int64_t n_dof = c->n_dof;
    const int64_t rpr = (n_dof + c->world - 1) / c->world;
    const int64_t R0 = std::min<int64_t>(n_dof, rpr * c->rank), R1 = std::min<int64_t>(n_dof, R0 + rpr);
    const int64_t nr = R1 - R0;
    c->rows_per_rank = rpr;
    c->row_begin = R0;
    c->n_rows = nr;

    // ---- shared-memory budget -> elements per block (e_max) and record budget
    const int dm = (c->plan_which & FEA_MASS) ? 1 : 0, dcm = (c->plan_which & FEA_STIFF) ? 1 : 0;
    const int nmat = dm + dcm;
    const bool v6 = fea6_supported(c->order, nq) && (c->tune_kver == 0 || c->tune_kver == 6) && !c->split;
    const bool v5 = !v6 && fea5_supported(c->order, nq) && c->tune_kver != 4 && !c->split;
    c->kver = v6 ? 6 : v5 ? 5 : 4;
    const int rstages = c->order <= 2 ? 3 : 2;  // fea_rstages (v4)
    int64_t e_max, rec_budget;
    int64_t vcap = 0, e_target = 0;  // v6 compact V: capacity (cells per buffer) and greedy block target
    if (v6) {
        // two V buffers, two gather / Lambda / W stages (fea6_smem_layout); records stay in global memory
        const int64_t budget = c->tune_smem ? c->tune_smem : 227 * 1024;
        e_max = std::min<int64_t>(32 * fea6_prod_rounds(c->order), 65535 / T - 2) / 8 * 8;
        if (c->tune_emax) e_max = std::min<int64_t>(e_max, c->tune_emax / 8 * 8);
        int32_t L6[FEA_L_N];
        if (FEA6_VCOMPACT) {
            // compact V: the capacity left by the e_max-sized buffers; the greedy blocks target the
            // elements that capacity holds at an expected post-skip tile fraction (blocks over it
            // are cut in build_blocks); e_max (buffers) chosen to maximise min(e_max, target)
            const int cellb = nmat == 2 ? 16 : 8, ntt = (T + 7) / 8;
            const double frac = c->tune_skip && c->rule_sym ? (c->order == 4 ? FEA6_VFRAC / 100.0 : 0.86) : 1.0;
            int64_t best_el = -1, best_e = 0, best_cap = 0;
            for (int64_t em = e_max; em >= 8; em -= 8) {
                fea6_smem_layout(L6, (int)em, c->order, dm, dcm, 1);
                const int64_t cap = std::min<int64_t>(65535, (budget - L6[FEA6_L_TOTAL] + L6[FEA6_L_VB] * 2) / 2 / 128 * 128 / cellb);
                if (cap < 1 + 64 * 2 * ntt) continue;
                const int64_t tgt = std::min<int64_t>(em, (int64_t)((cap - 1) / 64 / (ntt * frac / 8.0)));
                if (tgt > best_el) best_el = tgt, best_e = em, best_cap = cap;
            }
            if (best_el < 8) return c->fail(FEA_E_UNSUPPORTED, "shared-memory budget too small for kernel v6");
            e_max = best_e;
            vcap = best_cap;  // (cells; whole 128-byte lines)
            e_target = best_el;
        } else {
            for (; e_max >= 8; e_max -= 8) {
                fea6_smem_layout(L6, (int)e_max, c->order, dm, dcm);
                if (L6[FEA6_L_TOTAL] <= budget) break;
            }
        }
        rec_budget = INT64_MAX / 4;
    } else if (v5) {
        // two V_m, V_c [T][e_max | 1] buffers + two record stages in 227 KiB (one CTA per SM)
        const int64_t budget = c->tune_smem ? c->tune_smem : 227 * 1024;
        const double rec_el = 1.1 * 2.0 * np * np + 8;  // record bytes per element (estimate)
        e_max = (int64_t)((budget - 1024) / (2 * (8.0 * T * nmat + rec_el)));
        if (c->tune_emax) e_max = std::min(e_max, c->tune_emax);
        e_max = std::min<int64_t>(e_max, 65535 / T - 1) / 8 * 8;
        // P1 (one unit per 32-element tile, ~2 units per warp per block): whole rounds of units over
        // the NW warps, so no block leaves most warps idle in a ragged last round (C4 1.127 -> 1.092 ms)
        if (np == 3 && !c->tune_emax && e_max >= 32 * fea5_nw(1)) e_max = e_max / (32 * fea5_nw(1)) * (32 * fea5_nw(1));
        rec_budget = ((budget - 1024 - 2 * 8LL * T * nmat * (e_max | 1)) / 2 - 128) & ~int64_t(15);
    } else {
        const int ctas = c->order <= 2 ? 2 : 1;  // fea_ctas
        const int64_t budget = c->tune_smem ? c->tune_smem : (ctas == 2 ? 113 * 1024 : 226 * 1024);
        const int nqp = c->split ? 16 : 4 * fea_nk_kernel(c->order, nq);  // split rules: room for either
        const int64_t per_el_smem = 8LL * T * nmat + 2 * (8LL * np + 48) + 2 * 8LL * nqp + 32;
        double rec_el = 1.3 * (3.0 * np * np + 4.0 * np) + 8;  // record bytes per element (estimate)
        const int64_t r0 = 32 * FEA_MAX_CLASSES + 1024;            // per-record constant part
        for (int pass = 0; pass < 2; ++pass) {  // pass 1: the first plan's own record bytes per element
            e_max = (int64_t)((budget - 256 - 3 * 128 - 16LL * T * nmat - 32LL * (np + 2 * nqp) - rstages * r0) /
                              (per_el_smem + rstages * rec_el));
            e_max = std::min<int64_t>(e_max, 65535 / T);
            if (c->tune_emax) e_max = std::min(e_max, c->tune_emax);
            e_max = e_max >= 8 ? ((e_max - 8) / 16) * 16 + 8 : 0;  // multiple of 8, == 8 mod 16
            rec_budget = ((int64_t)(rec_el * e_max) + r0 + 15) & ~int64_t(15);
            if (pass == 1 || e_max < 8) break;
            PlanData P0;  // on the first rows only (a sample: records of interior blocks are alike)
            const int64_t nr_all = c->n_rows;
            c->n_rows = std::min<int64_t>(nr_all, 20000);
            const fea_status st0 = build_blocks(c, false, false, e_max, rec_budget, fea4_vstride((int32_t)e_max), P0);
            c->n_rows = nr_all;
            if (st0 != FEA_OK) break;
            int32_t L0[FEA_L_N];
            fea_smem_layout(L0, rstages, (int)P0.rec_max, (int)e_max, c->order, c->split ? 0 : nq, dm, dcm);
            if (budget - L0[FEA_L_TOTAL] < 8 * 1024) break;
            rec_el = 1.02 * (double)std::max<int64_t>(P0.rec_max - r0, 16) / (double)e_max;
        }
    }

    const int64_t EM = v6 ? fea6_vstride((int32_t)e_max) : v5 ? (e_max | 1) : fea4_vstride((int32_t)e_max);  // V row strides
    PlanData P;
    {
        // v5 with both matrices: V_m, V_c interleaved, phase B reads 16-byte {m, c} pairs
        const fea_status st = v6 ? build_blocks(c, true, false, vcap > 0 ? e_target : e_max, rec_budget, EM, P, nmat == 2, true, vcap)
                                 : build_blocks(c, v5, false, e_max, rec_budget, EM, P, v5 && nmat == 2);
        if (st != FEA_OK) return st;
    }
    const int64_t nb = (int64_t)P.blocks.size();
    const int64_t nnz = P.nnz, rec_max = P.rec_max;
    c->n_int = 0;
    if (c->world > 1) {  // interior blocks first (they read only owned u): assembled during the exchange
        std::stable_partition(P.blocks.begin(), P.blocks.end(), [](const FeaBlock& b) { return b.spare_[0] != 0; });
        for (const FeaBlock& b : P.blocks) c->n_int += b.spare_[0] != 0;
    }
    c->row_ptr.swap(P.row_ptr);
    c->col_idx.swap(P.col_idx);
    std::vector<FeaBlock>& blocks = P.blocks;
    auto& records = P.records;
    auto& alldofs = P.dofs;
    const int64_t visits = P.visits, owned = P.owned, ncon = P.ncon, rbytes = P.rbytes;
    int32_t L[FEA_L_N];
    if (v6) fea6_smem_layout(L, (int)e_max, c->order, dm, dcm, (int)vcap);
    else if (v5) fea5_smem_layout(L, (int)rec_max, (int)e_max, c->order, dm, dcm);
    else fea_smem_layout(L, rstages, (int)rec_max, (int)e_max, c->order, c->split ? 0 : nq, dm, dcm);
    c->nblocks = (int)nb;
    c->e_max = (int)e_max;
    c->rec_max = (int)rec_max;
    c->nnz = nnz;
    c->smem_bytes = v6 ? L[FEA6_L_TOTAL] : L[FEA_L_TOTAL];
    std::memcpy(c->lay, L, sizeof(c->lay));
    // ---- interface sets I_t of every rank t (world > 1): owned DOFs that another rank's elements
    // read.  Ranks own contiguous chunks of rows_per_rank library rows; every rank derives the
    // same lists from the full mesh.
    c->iface.clear();
    c->ioff.assign(c->world + 1, 0);
    c->maxI = 0;
    if (c->world > 1) {
        const int W = c->world;
        std::vector<uint8_t> need((size_t)c->n_dof, 0);
        for (int64_t e = 0; e < c->n_e; ++e) {
            const int32_t* d = &c->ed[(size_t)e * np];
            int o0 = (int)(d[0] / rpr);
            bool multi = false;
            for (int i = 1; i < np; ++i) multi |= (int)(d[i] / rpr) != o0;
            if (multi)
                for (int i = 0; i < np; ++i) need[d[i]] = 1;  // read by another rank (some owner of e differs)
        }
        std::vector<int64_t> cnt(W + 1, 0);
        for (int64_t d = 0; d < c->n_dof; ++d)
            if (need[d]) cnt[d / rpr + 1]++;
        for (int t = 0; t < W; ++t) cnt[t + 1] += cnt[t];
        c->ioff = cnt;
        c->iface.resize(cnt[W]);
        std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
        for (int64_t d = 0; d < c->n_dof; ++d)
            if (need[d]) c->iface[pos[d / rpr]++] = (int32_t)d;
        for (int t = 0; t < W; ++t) c->maxI = std::max<int>(c->maxI, (int)(cnt[t + 1] - cnt[t]));
    }
    c->stat_visits = visits;
    c->stat_owned = owned;
    c->stat_entries = ncon;
    c->record_bytes = rbytes;
    if (c->host_only) {
        c->have_plan = true;
        if (row_begin) *row_begin = R0;
        if (n_rows_local) *n_rows_local = nr;
        if (nnz_local) *nnz_local = nnz;
        return FEA_OK;
    }
    // ---- device upload
    FEA_CUDA(c, cudaMalloc((void**)&c->d_blocks, std::max<int64_t>(nb, 1) * sizeof(FeaBlock)));
    if (nb) FEA_CUDA(c, cudaMemcpy(c->d_blocks, blocks.data(), nb * sizeof(FeaBlock), cudaMemcpyHostToDevice));
    FEA_CUDA(c, cudaMalloc((void**)&c->d_records, records.size()));
    FEA_CUDA(c, cudaMemcpy(c->d_records, records.data(), records.size(), cudaMemcpyHostToDevice));
    if (v5 || v6) {
        FEA_CUDA(c, cudaMalloc((void**)&c->d_dofs, alldofs.size() * sizeof(int32_t)));
        FEA_CUDA(c, cudaMemcpy(c->d_dofs, alldofs.data(), alldofs.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (!c->d_ufull) FEA_CUDA(c, cudaMalloc(&c->d_ufull, (size_t)rpr * c->world * sizeof(double)));
    if (!c->d_usend) FEA_CUDA(c, cudaMalloc(&c->d_usend, (size_t)rpr * sizeof(double)));
    if (c->world > 1) {
        dfree(c->d_iface);
        dfree(c->d_ioff);
        dfree(c->d_isend);
        dfree(c->d_irecv);
        FEA_CUDA(c, cudaMalloc(&c->d_iface, std::max<size_t>(1, c->iface.size()) * sizeof(int32_t)));
        if (!c->iface.empty())
            FEA_CUDA(c, cudaMemcpy(c->d_iface, c->iface.data(), c->iface.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
        FEA_CUDA(c, cudaMalloc(&c->d_ioff, c->ioff.size() * sizeof(int64_t)));
        FEA_CUDA(c, cudaMemcpy(c->d_ioff, c->ioff.data(), c->ioff.size() * sizeof(int64_t), cudaMemcpyHostToDevice));
        FEA_CUDA(c, cudaMalloc(&c->d_isend, std::max<size_t>(1, c->maxI) * sizeof(double)));
        FEA_CUDA(c, cudaMalloc(&c->d_irecv, std::max<size_t>(1, (size_t)c->maxI * c->world) * sizeof(double)));
    }
    int occ = 0;
    int rc = v6   ? fea_kernel_occupancy6(c->order, dm, dcm, c->smem_bytes, &occ, &c->threads)
             : v5 ? fea_kernel_occupancy5(c->order, dm, dcm, c->smem_bytes, &occ, &c->threads)
                  : fea_kernel_occupancy(c->order, c->nq, dm, dcm, c->smem_bytes, &occ, &c->threads);
    if (rc != 0) return c->fail(FEA_E_CUDA, "occupancy query: %s", cudaGetErrorString((cudaError_t)rc));
    if (occ < 1) return c->fail(FEA_E_UNSUPPORTED, "kernel does not fit: %d B shared memory", c->smem_bytes);
    c->grid = (int)std::min<int64_t>(std::max<int64_t>(nb, 1), (int64_t)occ * c->sm_count);
    // our kernels per fea_reassemble: the assembly, plus pack + unpack of the exchange (world > 1)
    c->launches_per_call = c->world > 1 ? 2 + (c->exchange == 0 ? 2 : 0) : 1;
    ptime("plan: upload");
    c->have_plan = true;
    if (row_begin) *row_begin = R0;
    if (n_rows_local) *n_rows_local = nr;
    if (nnz_local) *nnz_local = nnz;
    return FEA_OK;
}

fea_status fea_get_pattern(fea_ctx c, int64_t* row_ptr, int32_t* col_idx) {
    if (!c) return FEA_E_ARG;
    if (!c->have_plan) return c->fail(FEA_E_STATE, "get_pattern before build_pattern");
    if (row_ptr) std::memcpy(row_ptr, c->row_ptr.data(), c->row_ptr.size() * sizeof(int64_t));
    if (col_idx && c->nnz) std::memcpy(col_idx, c->col_idx.data(), c->col_idx.size() * sizeof(int32_t));
    return FEA_OK;
}

fea_status fea_get_pattern_rows(fea_ctx c, int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col_idx) {
    if (!c) return FEA_E_ARG;
    if (!c->have_plan) return c->fail(FEA_E_STATE, "get_pattern_rows before build_pattern");
    if (r0 < 0 || r1 < r0 || r1 > c->n_rows) return c->fail(FEA_E_ARG, "row range [%lld, %lld) outside [0, %lld)",
                                                           (long long)r0, (long long)r1, (long long)c->n_rows);
    if (row_ptr) std::memcpy(row_ptr, c->row_ptr.data() + r0, (size_t)(r1 - r0 + 1) * sizeof(int64_t));
    if (col_idx && r1 > r0)
        std::memcpy(col_idx, c->col_idx.data() + c->row_ptr[r0], (size_t)(c->row_ptr[r1] - c->row_ptr[r0]) * sizeof(int32_t));
    return FEA_OK;
}

fea_status fea_get_dof_perm(fea_ctx c, int64_t* lib_to_user) {
    if (!c || !lib_to_user) return FEA_E_ARG;
    if (!c->have_mesh) return c->fail(FEA_E_STATE, "get_dof_perm before mesh_upload");
    std::memcpy(lib_to_user, c->dof_lib2user.data(), c->dof_lib2user.size() * sizeof(int64_t));
    return FEA_OK;
}

fea_status fea_get_elem_perm(fea_ctx c, int64_t* lib_to_user) {
    if (!c || !lib_to_user) return FEA_E_ARG;
    if (!c->have_mesh) return c->fail(FEA_E_STATE, "get_elem_perm before mesh_upload");
    std::memcpy(lib_to_user, c->elem_lib2user.data(), c->elem_lib2user.size() * sizeof(int64_t));
    return FEA_OK;
}

fea_status fea_set_coefficient(fea_ctx c, int which, int kind, int n_par, const double* par) {
    if (!c) return FEA_E_ARG;
    if (which < 1 || which > 3) return c->fail(FEA_E_ARG, "which must be a nonzero FEA_MASS|FEA_STIFF mask");
    if (n_par < 1 || n_par > FEA_MAX_PAR || !par) return c->fail(FEA_E_ARG, "bad coefficient parameters");
    if (kind == FEA_K_POLY && n_par > 9) return c->fail(FEA_E_ARG, "polynomial degree > 8");
    if (kind == FEA_K_EXP && n_par != 2) return c->fail(FEA_E_ARG, "FEA_K_EXP takes 2 parameters");
    if (kind == FEA_K_PWL) {
        if (n_par % 2 || n_par < 4) return c->fail(FEA_E_ARG, "FEA_K_PWL takes 2..8 (T, k) pairs");
        for (int i = 2; i < n_par; i += 2)
            if (!(par[i] > par[i - 2])) return c->fail(FEA_E_ARG, "FEA_K_PWL breakpoints must increase");
    }
    if (kind < 0 || kind > 2) return c->fail(FEA_E_ARG, "unknown coefficient kind %d", kind);
    FeaCoef k{};
    k.kind = kind;
    k.npar = n_par;
    for (int i = 0; i < n_par; ++i) k.par[i] = par[i];
    if (which & FEA_MASS) c->coef_m = k;
    if (which & FEA_STIFF) c->coef_c = k;
    return FEA_OK;
}

static bool same_coef(const FeaCoef& a, const FeaCoef& b) {
    if (a.kind != b.kind || a.npar != b.npar) return false;
    for (int i = 0; i < a.npar; ++i)
        if (a.par[i] != b.par[i]) return false;
    return true;
}

// rule_c: run with the rule of C (split rules; vm must then be NULL).  Blocks [b0, b1) of the plan
// (b1 < 0: all).
static fea_status launch(fea_ctx c, const double* u, double* vm, double* vc, bool rule_c = false, int b0 = 0,
                         int b1 = -1) {
    if (b1 < 0) b1 = c->nblocks;
    FeaKParams prm{};
    prm.blocks = c->d_blocks + b0;
    prm.records = c->d_records;
    prm.xy = c->d_xy;
    prm.dofs = c->d_dofs;
    prm.u = u;
    prm.qfrag = rule_c ? c->d_tables_c : c->d_tables;
    prm.out_m = vm;
    prm.out_c = vc;
    prm.nblocks = b1 - b0;
    prm.e_max = c->e_max;
    prm.nq = rule_c ? c->nq_c : c->nq;
    prm.same_coef = same_coef(c->coef_m, c->coef_c) ? 1 : 0;
    std::memcpy(prm.lay, c->lay, sizeof(prm.lay));
    prm.n_dof = c->n_dof;
    prm.n_slots = c->nnz;
    prm.rec_size = c->record_bytes;
    // a single-matrix pass on a plan sized for the other matrix: its V region has size 0 in the
    // layout, so it takes the planned matrix's region (same size, same contributor offsets)
    // (kernel v6 has one V region either way: its single-matrix passes use it with 8-byte cells)
    const bool pm = c->plan_which & FEA_MASS, pc = c->plan_which & FEA_STIFF;
    if (c->kver != 6 && vc && !vm && !pc) prm.lay[FEA_L_VC] = c->lay[FEA_L_VM];
    if (c->kver != 6 && vm && !vc && !pm) prm.lay[FEA_L_VM] = c->lay[FEA_L_VC];
    if (vm && vc && !(pm && pc)) return c->fail(FEA_E_STATE, "internal: fused M+K pass on a one-matrix plan");
    prm.coef_m = c->coef_m;
    prm.coef_c = c->coef_c;
    const std::vector<double>& tab = rule_c ? c->tables_c : c->tables;
    std::memcpy(prm.ctab, tab.data(), tab.size() * sizeof(double));
    if (c->kver == 5) std::memcpy(prm.jtab, c->jplain.data(), c->jplain.size() * sizeof(double));
    prm.dbg_mode = c->dbg_mode;
    if (c->dbg_timing) {
        if (!c->d_dbg) {
            FEA_CUDA(c, cudaMalloc(&c->d_dbg, 1536 * sizeof(unsigned long long)));
            FEA_CUDA(c, cudaMemset(c->d_dbg, 0, 1536 * sizeof(unsigned long long)));
        }
        prm.dbg = c->d_dbg;
    }
    if (b1 <= b0) return FEA_OK;
    const int grid = std::min(c->int_grid_cap > 0 ? c->int_grid_cap : c->grid, b1 - b0);
    const int rc = c->kver == 6   ? fea_launch_reassemble6(prm, c->order, c->smem_bytes, grid, c->stream)
                   : c->kver == 5 ? fea_launch_reassemble5(prm, c->order, c->smem_bytes, grid, c->stream)
                                  : fea_launch_reassemble(prm, c->order, c->smem_bytes, grid, c->stream);
    if (rc != 0) return c->fail(FEA_E_CUDA, "k_reassemble launch: %s", cudaGetErrorString((cudaError_t)rc));
    return FEA_OK;
}

// all blocks, or (world > 1) the interior blocks [0, n_int) / the boundary blocks [n_int, nb)
enum { FEA_PART_ALL = 0, FEA_PART_INT = 1, FEA_PART_BND = 2 };
static fea_status assemble_part(fea_ctx c, const double* u_full, double* mass_vals, double* stiff_vals, int part) {
    const int b0 = part == FEA_PART_BND ? c->n_int : 0;
    const int b1 = part == FEA_PART_INT ? c->n_int : c->nblocks;
    const bool pm = c->plan_which & FEA_MASS, pc = c->plan_which & FEA_STIFF;
    fea_status s;
    if (c->split) {  // separate rules: one pass per matrix, each with its rule's tables
        if (mass_vals && (s = launch(c, u_full, mass_vals, nullptr, false, b0, b1)) != FEA_OK) return s;
        return stiff_vals ? launch(c, u_full, nullptr, stiff_vals, true, b0, b1) : FEA_OK;
    }
    // plan sized for one matrix, or (kernel v6, one Lambda) distinct coefficients: two passes
    if (mass_vals && stiff_vals && (!(pm && pc) || (c->kver == 6 && !same_coef(c->coef_m, c->coef_c)))) {
        if ((s = launch(c, u_full, mass_vals, nullptr, false, b0, b1)) != FEA_OK) return s;
        return launch(c, u_full, nullptr, stiff_vals, false, b0, b1);
    }
    return launch(c, u_full, mass_vals, stiff_vals, false, b0, b1);
}

fea_status fea_assemble(fea_ctx c, const double* u_full, double* mass_vals, double* stiff_vals) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan) return c->fail(FEA_E_STATE, "assemble before build_pattern");
    if (!u_full) return c->fail(FEA_E_ARG, "u_full is NULL");
    if ((mass_vals && ((uintptr_t)mass_vals & 15)) || (stiff_vals && ((uintptr_t)stiff_vals & 15)))
        return c->fail(FEA_E_ARG, "vals must be 16-byte aligned");
    if (!mass_vals && !stiff_vals) return FEA_OK;
    cudaSetDevice(c->device);
    fea_status s = tmark(c, 2, c->stream);
    if (s != FEA_OK) return s;
    if (c->world == 1) s = assemble_part(c, u_full, mass_vals, stiff_vals, FEA_PART_ALL);
    else {
        s = assemble_part(c, u_full, mass_vals, stiff_vals, FEA_PART_INT);
        if (s == FEA_OK) s = assemble_part(c, u_full, mass_vals, stiff_vals, FEA_PART_BND);
    }
    return s != FEA_OK ? s : tmark(c, 3, c->stream);
}

fea_status fea_assemble_mass(fea_ctx c, const double* u_full, double* vals) {
    if (!vals) return c ? c->fail(FEA_E_ARG, "vals is NULL") : FEA_E_ARG;
    return fea_assemble(c, u_full, vals, nullptr);
}

fea_status fea_assemble_stiffness(fea_ctx c, const double* u_full, double* vals) {
    if (!vals) return c ? c->fail(FEA_E_ARG, "vals is NULL") : FEA_E_ARG;
    return fea_assemble(c, u_full, nullptr, vals);
}

// One allgather of `count` float64 per rank, stream-ordered on `st`: ncclAllGather on the
// library's communicator, or the caller's host transport (D2H of this rank's values, wait, the
// callback, H2D of every rank's values; the pinned buffers are reused only after the next call's
// wait on the same stream).
static fea_status allgather(fea_ctx c, const double* send, double* recv, int64_t count, cudaStream_t st) {
    if (count <= 0) return FEA_OK;
    if (c->htrans) {
        if (c->h_cap < count) {
            if (c->h_send) cudaFreeHost(c->h_send);
            if (c->h_recv) cudaFreeHost(c->h_recv);
            c->h_send = c->h_recv = nullptr;
            c->h_cap = 0;
            FEA_CUDA(c, cudaMallocHost(&c->h_send, (size_t)count * sizeof(double)));
            FEA_CUDA(c, cudaMallocHost(&c->h_recv, (size_t)count * c->world * sizeof(double)));
            c->h_cap = count;
        }
        FEA_CUDA(c, cudaMemcpyAsync(c->h_send, send, (size_t)count * sizeof(double), cudaMemcpyDeviceToHost, st));
        FEA_CUDA(c, cudaStreamSynchronize(st));
        const int rc = c->htrans(c->h_send, c->h_recv, count, c->huser);
        if (rc != 0) return c->fail(FEA_E_NCCL, "host transport returned %d", rc);
        FEA_CUDA(c, cudaMemcpyAsync(recv, c->h_recv, (size_t)count * c->world * sizeof(double), cudaMemcpyHostToDevice, st));
        return FEA_OK;
    }
    if (!c->comm) return c->fail(FEA_E_STATE, "world > 1 requires fea_set_nccl or fea_set_host_transport");
    ncclResult_t r = nccl().allGather(send, recv, (size_t)count, ncclDouble, (ncclComm_t)c->comm, st);
    if (r != ncclSuccess) return c->fail(FEA_E_NCCL, "ncclAllGather: %s", nccl().getErrorString(r));
    return FEA_OK;
}

// u_owned (this rank's rows) -> c->d_ufull holding every value this rank's kernel reads:
// interface-only (pack, one ncclAllGather of maxI values per rank, unpack) or the full-vector
// allgather of rows_per_rank values per rank.  Stream-ordered on the ctx stream.
static fea_status exchange_u(fea_ctx c, const double* u_owned) {
    if (c->exchange == 0) {
        int rc = fea_launch_pack(u_owned, c->d_iface + c->ioff[c->rank], (int)(c->ioff[c->rank + 1] - c->ioff[c->rank]),
                                 c->row_begin, c->maxI, c->d_isend, c->stream);
        if (rc) return c->fail(FEA_E_CUDA, "pack: %s", cudaGetErrorString((cudaError_t)rc));
        fea_status s = allgather(c, c->d_isend, c->d_irecv, c->maxI, c->stream);
        if (s != FEA_OK) return s;
        rc = fea_launch_unpack(c->d_irecv, c->d_iface, c->d_ioff, c->world, c->rank, c->maxI, c->ioff[c->world],
                               u_owned, c->row_begin, c->n_rows, c->d_ufull, c->stream);
        if (rc) return c->fail(FEA_E_CUDA, "unpack: %s", cudaGetErrorString((cudaError_t)rc));
        return FEA_OK;
    }
    // full vector: pad the owned slice to rows_per_rank, then allgather
    if (c->n_rows && u_owned != c->d_usend)
        FEA_CUDA(c, cudaMemcpyAsync(c->d_usend, u_owned, c->n_rows * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return allgather(c, c->d_usend, c->d_ufull, c->rows_per_rank, c->stream);
}

// NEXT-3 overlap: the owned rows go into u_full on the ctx stream, the interior blocks (which read
// only owned entries) assemble on the ctx stream while pack -> ncclAllGather -> unpack of the halo
// run on a second stream; the boundary blocks wait for the halo.
static fea_status reassemble_overlap(fea_ctx c, const double* u_owned, double* mass_vals, double* stiff_vals) {
    if (!c->stream2) {
        FEA_CUDA(c, cudaStreamCreateWithFlags(&c->stream2, cudaStreamNonBlocking));
        FEA_CUDA(c, cudaEventCreateWithFlags(&c->ev_own, cudaEventDisableTiming));
        FEA_CUDA(c, cudaEventCreateWithFlags(&c->ev_halo, cudaEventDisableTiming));
    }
    if (c->n_rows)
        FEA_CUDA(c, cudaMemcpyAsync(c->d_ufull + c->row_begin, u_owned, c->n_rows * sizeof(double),
                                    cudaMemcpyDeviceToDevice, c->stream));
    FEA_CUDA(c, cudaEventRecord(c->ev_own, c->stream));
    FEA_CUDA(c, cudaStreamWaitEvent(c->stream2, c->ev_own, 0));
    fea_status s = tmark(c, 0, c->stream2);
    if (s != FEA_OK) return s;
    // a host transport blocks this thread inside the exchange: enqueue the interior blocks first
    const bool host = c->htrans != nullptr;
    if (host) {
        if ((s = tmark(c, 2, c->stream)) != FEA_OK) return s;
        if ((s = assemble_part(c, c->d_ufull, mass_vals, stiff_vals, FEA_PART_INT)) != FEA_OK) return s;
    }
    int rc = fea_launch_pack(u_owned, c->d_iface + c->ioff[c->rank], (int)(c->ioff[c->rank + 1] - c->ioff[c->rank]),
                             c->row_begin, c->maxI, c->d_isend, c->stream2);
    if (rc) return c->fail(FEA_E_CUDA, "pack: %s", cudaGetErrorString((cudaError_t)rc));
    if ((s = allgather(c, c->d_isend, c->d_irecv, c->maxI, c->stream2)) != FEA_OK) return s;
    rc = fea_launch_unpack(c->d_irecv, c->d_iface, c->d_ioff, c->world, c->rank, c->maxI, c->ioff[c->world],
                           u_owned, c->row_begin, 0 /* owned rows already copied */, c->d_ufull, c->stream2);
    if (rc) return c->fail(FEA_E_CUDA, "unpack: %s", cudaGetErrorString((cudaError_t)rc));
    if ((s = tmark(c, 1, c->stream2)) != FEA_OK) return s;
    FEA_CUDA(c, cudaEventRecord(c->ev_halo, c->stream2));
    if (!host) {  // NCCL: its kernel is queued first; the interior grid leaves it int_grid_cap SMs
        if ((s = tmark(c, 2, c->stream)) != FEA_OK) return s;
        c->int_grid_cap = std::max(1, c->grid - 4);
        s = assemble_part(c, c->d_ufull, mass_vals, stiff_vals, FEA_PART_INT);
        c->int_grid_cap = 0;
        if (s != FEA_OK) return s;
    }
    FEA_CUDA(c, cudaStreamWaitEvent(c->stream, c->ev_halo, 0));
    s = assemble_part(c, c->d_ufull, mass_vals, stiff_vals, FEA_PART_BND);
    return s != FEA_OK ? s : tmark(c, 3, c->stream);
}

fea_status fea_get_interface(fea_ctx c, int64_t* offsets, int32_t* dofs) {
    if (!c) return FEA_E_ARG;
    if (!c->have_plan) return c->fail(FEA_E_STATE, "get_interface before build_pattern");
    if (offsets) std::memcpy(offsets, c->ioff.data(), c->ioff.size() * sizeof(int64_t));
    if (dofs && !c->iface.empty()) std::memcpy(dofs, c->iface.data(), c->iface.size() * sizeof(int32_t));
    return FEA_OK;
}

fea_status fea_exchange_pack(fea_ctx c, const double* u_owned, double* send) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan || c->world < 2) return c->fail(FEA_E_STATE, "exchange_pack needs a world > 1 plan");
    if (!u_owned || !send) return c->fail(FEA_E_ARG, "NULL buffer");
    cudaSetDevice(c->device);
    const int rc = fea_launch_pack(u_owned, c->d_iface + c->ioff[c->rank], (int)(c->ioff[c->rank + 1] - c->ioff[c->rank]),
                                   c->row_begin, c->maxI, send, c->stream);
    return rc ? c->fail(FEA_E_CUDA, "pack: %s", cudaGetErrorString((cudaError_t)rc)) : FEA_OK;
}

fea_status fea_exchange_unpack(fea_ctx c, const double* u_owned, const double* recv, double* u_full) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan || c->world < 2) return c->fail(FEA_E_STATE, "exchange_unpack needs a world > 1 plan");
    if (!u_owned || !recv || !u_full) return c->fail(FEA_E_ARG, "NULL buffer");
    cudaSetDevice(c->device);
    const int rc = fea_launch_unpack(recv, c->d_iface, c->d_ioff, c->world, c->rank, c->maxI, c->ioff[c->world],
                                     u_owned, c->row_begin, c->n_rows, u_full, c->stream);
    return rc ? c->fail(FEA_E_CUDA, "unpack: %s", cudaGetErrorString((cudaError_t)rc)) : FEA_OK;
}

fea_status fea_reassemble(fea_ctx c, const double* u_owned, double* mass_vals, double* stiff_vals) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan) return c->fail(FEA_E_STATE, "reassemble before build_pattern");
    if (!u_owned) return c->fail(FEA_E_ARG, "u_owned is NULL");
    cudaSetDevice(c->device);
    if (c->world == 1) return fea_assemble(c, u_owned, mass_vals, stiff_vals);
    if (!c->comm && !c->htrans) return c->fail(FEA_E_STATE, "world > 1 requires fea_set_nccl or fea_set_host_transport");
    if ((mass_vals && ((uintptr_t)mass_vals & 15)) || (stiff_vals && ((uintptr_t)stiff_vals & 15)))
        return c->fail(FEA_E_ARG, "vals must be 16-byte aligned");
    if (c->exchange == 0 && c->tune_overlap)
        return reassemble_overlap(c, u_owned, mass_vals, stiff_vals);
    fea_status st = tmark(c, 0, c->stream);
    if (st == FEA_OK) st = exchange_u(c, u_owned);
    if (st == FEA_OK) st = tmark(c, 1, c->stream);
    if (st != FEA_OK) return st;
    return fea_assemble(c, c->d_ufull, mass_vals, stiff_vals);
}

fea_status fea_reassemble_host(fea_ctx c, const double* u_host, double* mass_host, double* stiff_host) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan) return c->fail(FEA_E_STATE, "reassemble before build_pattern");
    if (!u_host) return c->fail(FEA_E_ARG, "u_host is NULL");
    cudaSetDevice(c->device);
    if (mass_host && !c->d_vm) FEA_CUDA(c, cudaMalloc(&c->d_vm, std::max<int64_t>(1, c->nnz) * sizeof(double)));
    if (stiff_host && !c->d_vc) FEA_CUDA(c, cudaMalloc(&c->d_vc, std::max<int64_t>(1, c->nnz) * sizeof(double)));
    double* dst = c->world == 1 ? c->d_ufull : c->d_usend;
    const int64_t n = c->world == 1 ? c->n_dof : c->n_rows;
    FEA_CUDA(c, cudaMemcpyAsync(dst, u_host, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    fea_status s;
    if (c->world == 1) s = fea_assemble(c, c->d_ufull, mass_host ? c->d_vm : nullptr, stiff_host ? c->d_vc : nullptr);
    else {
        s = fea_reassemble(c, c->d_usend, mass_host ? c->d_vm : nullptr, stiff_host ? c->d_vc : nullptr);
    }
    if (s != FEA_OK) return s;
    if (mass_host) FEA_CUDA(c, cudaMemcpyAsync(mass_host, c->d_vm, c->nnz * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    if (stiff_host) FEA_CUDA(c, cudaMemcpyAsync(stiff_host, c->d_vc, c->nnz * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    FEA_CUDA(c, cudaStreamSynchronize(c->stream));
    return FEA_OK;
}

// Tensor plan: same rows as the matrix plan, v5 record format with orientation bits, blocks sized
// for V1 + Vup + Vdn (3 T doubles per element) in one CTA per SM (k_tensor5: two buffers of the
// channels wanted, want_m / want_c; a later call wanting another channel re-plans).
static fea_status build_tensor_plan(fea_ctx c, bool want_m, bool want_c) {
    const int np = c->np, T = c->T;
    const int64_t budget = 227 * 1024;
    const int64_t tabs = 8LL * (3 * np * 16 + 16) + 256;
    // kernel: k_tensor4 (DMMA) for p >= 2 or any non-native rule, k_tensor5 (lane per element,
    // pipelined) for P1 with its 3-point rule (C4: 3.13 ms with k_tensor, 5.20 with k_tensor4)
    const bool native = c->nq == fea_nq_native(c->order) && (!c->split || c->nq_c == fea_nq_native(c->order));
    const bool t5ok = fea_t5_supported(c->order, c->nq) && !c->split;
    c->t_kver = c->tune_tker ? c->tune_tker : (t5ok ? 5 : c->order >= 2 || !native ? 4 : 1);
    if (c->t_kver == 5 && !t5ok)
        return c->fail(FEA_E_UNSUPPORTED, "k_tensor5 needs P1 with its 3-point rule (one rule for both matrices)");
    const bool k4 = c->t_kver == 4, k5 = c->t_kver == 5;
    int64_t e_max, rec_budget;
    if (k5) {  // two V buffers of the wanted channels, two record stages (fea_t5_smem_layout)
        const int rows = fea_t5_rows(c->order, want_m, want_c);
        const double rec_el = 1.1 * 2.0 * np * np + 8;
        const int64_t fixed = 64 + 512 + 2 * 256 + 2048;
        e_max = (int64_t)((budget - fixed) / (16.0 * rows + 2 * rec_el));
        if (c->tune_emax) e_max = std::min(e_max, c->tune_emax);
        e_max = std::min<int64_t>(e_max, 32767 / T - 1) / 8 * 8;
        const int64_t round_el = 32 * FEA_T5_NW;  // whole rounds of 32-element units over the warps (as in v5)
        if (!c->tune_emax && e_max >= round_el) e_max = e_max / round_el * round_el;
        rec_budget = ((budget - fixed - 16LL * (rows * (e_max | 1) + 16)) / 2) & ~int64_t(15);
    } else if (k4) {  // V1, Vup, Vdn [T][e_max + 2], two record and gather stages, Lambda and p (fea_t4_smem_layout)
        const int nqp = c->split ? 16 : 4 * fea_nk_kernel(c->order, c->nq);
        const int64_t per_el = 8LL * (3 * T - np) + 2 * (16LL * np + 48) + 3 * 8LL * nqp;
        // record bytes per element: an estimate, then (below) the planned blocks' own ratio
        const double rec_el = c->t_rec_el > 0 ? c->t_rec_el : 1.3 * (3.0 * np * np + 4.0 * np) + 8;
        const int64_t r0 = 32 * FEA_MAX_CLASSES + 1024;  // per-record constant part (class table, padding)
        e_max = (int64_t)((budget - tabs - 1024 - 64LL * (np + nqp) - 2 * r0) / (per_el + 2 * rec_el));
        if (c->tune_emax) e_max = std::min(e_max, c->tune_emax);
        e_max = std::min<int64_t>(e_max, 32767 / T - 2) / 8 * 8;
        rec_budget = ((int64_t)(rec_el * e_max) + r0 + 15) & ~int64_t(15);
    } else {
        const double rec_el = 1.1 * 2.0 * np * np + 8;
        e_max = (int64_t)((budget - tabs - 1024) / (8.0 * (3 * T - np) + rec_el));
        e_max = std::min<int64_t>(e_max, 32767 / T - 1) / 8 * 8;
        rec_budget = (budget - tabs - 1024 - 8LL * (3 * T - np) * (e_max | 1)) & ~int64_t(15);
    }
    PlanData P;
    const fea_status st = build_blocks(c, !k4, true, e_max, rec_budget, k4 ? fea4_vstride((int32_t)e_max) : (e_max | 1), P);
    if (st != FEA_OK) return st;
    if (P.nnz != c->nnz || P.row_ptr != c->row_ptr) return c->fail(FEA_E_STATE, "tensor plan: pattern mismatch");
    const int64_t nb = (int64_t)P.blocks.size();
    if (k4) {
        fea_t4_smem_layout(c->t_lay, (int)P.rec_max, (int)e_max, c->order, c->split ? 0 : c->nq);
        c->t_smem = c->t_lay[FEA_LT4_TOTAL];
        if (c->t_rec_el == 0 && e_max > 0) {  // one re-plan with the measured record bytes per element
            c->t_rec_el = 1.02 * (double)P.rec_max / (double)e_max;
            if (budget - c->t_smem > 8 * 1024) return build_tensor_plan(c, want_m, want_c);
        }
    } else if (k5) {
        fea_t5_smem_layout(c->t_lay, (int)P.rec_max, (int)e_max, c->order, want_m, want_c);
        c->t_smem = c->t_lay[FEA_LT5_TOTAL];
        c->t_pm = want_m;
        c->t_pc = want_c;
    } else {
        fea_t_smem_layout(c->t_lay, (int)P.rec_max, (int)e_max, c->order);
        c->t_smem = c->t_lay[FEA_LT_TOTAL];
    }
    c->t_nblocks = (int)nb;
    c->t_emax = (int)e_max;
    c->t_visits = P.visits;
    c->t_owned = P.owned;
    FEA_CUDA(c, cudaMalloc((void**)&c->dt_blocks, std::max<int64_t>(nb, 1) * sizeof(FeaBlock)));
    if (nb) FEA_CUDA(c, cudaMemcpy(c->dt_blocks, P.blocks.data(), nb * sizeof(FeaBlock), cudaMemcpyHostToDevice));
    FEA_CUDA(c, cudaMalloc((void**)&c->dt_records, P.records.size()));
    FEA_CUDA(c, cudaMemcpy(c->dt_records, P.records.data(), P.records.size(), cudaMemcpyHostToDevice));
    FEA_CUDA(c, cudaMalloc((void**)&c->dt_dofs, P.dofs.size() * sizeof(int32_t)));
    FEA_CUDA(c, cudaMemcpy(c->dt_dofs, P.dofs.data(), P.dofs.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
    int occ = 0, thr = 0;
    const int rc = k5 ? fea_tensor_occupancy5(c->order, c->nq, c->t_smem, &occ, &thr)
                      : fea_tensor_occupancy(c->order, c->nq, c->t_kver, c->t_smem, &occ, &thr);
    if (rc != 0) return c->fail(FEA_E_CUDA, "tensor occupancy: %s", cudaGetErrorString((cudaError_t)rc));
    if (occ < 1) return c->fail(FEA_E_UNSUPPORTED, "tensor kernel does not fit: %d B shared memory", c->t_smem);
    c->t_grid = (int)std::min<int64_t>(std::max<int64_t>(nb, 1), (int64_t)occ * c->sm_count);
    c->have_tplan = true;
    return FEA_OK;
}

fea_status fea_assemble_tensor(fea_ctx c, const double* u_full, const double* v_full, double* mt_vals, double* ct_vals) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!c->have_plan) return c->fail(FEA_E_STATE, "assemble_tensor before build_pattern");
    if (!u_full || !v_full) return c->fail(FEA_E_ARG, "u_full / v_full is NULL");
    if ((mt_vals && ((uintptr_t)mt_vals & 15)) || (ct_vals && ((uintptr_t)ct_vals & 15)))
        return c->fail(FEA_E_ARG, "vals must be 16-byte aligned");
    if (!mt_vals && !ct_vals) return FEA_OK;
    cudaSetDevice(c->device);
    if (c->have_tplan && c->t_kver == 5 && ((mt_vals && !c->t_pm) || (ct_vals && !c->t_pc))) {
        // k_tensor5's layout holds only the channels of the first call: re-plan for the union
        dfree(c->dt_blocks);
        dfree(c->dt_records);
        dfree(c->dt_dofs);
        c->have_tplan = false;
    }
    if (!c->have_tplan) {
        const fea_status st = build_tensor_plan(c, mt_vals || c->t_pm, ct_vals || c->t_pc);
        if (st != FEA_OK) return st;
    }
    if (c->t_nblocks == 0) return FEA_OK;
    FeaTParams prm{};
    prm.blocks = c->dt_blocks;
    prm.records = c->dt_records;
    prm.dofs = c->dt_dofs;
    prm.xy = c->d_xy;
    prm.u = u_full;
    prm.v = v_full;
    prm.tab = c->d_ttab;
    prm.qfrag = c->d_tables;
    prm.kver = c->t_kver;
    prm.out_m = mt_vals;
    prm.out_c = c->split ? nullptr : ct_vals;
    prm.nblocks = c->t_nblocks;
    prm.e_max = c->t_emax;
    prm.nq = c->nq;
    std::memcpy(prm.lay, c->t_lay, sizeof(prm.lay));
    prm.coef_m = c->coef_m;
    prm.coef_c = c->coef_c;
    prm.same_coef = same_coef(c->coef_m, c->coef_c) ? 1 : 0;
    prm.n_dof = c->n_dof;
    if (c->t_kver == 5) {  // constant-bank tables (kernel v5's layout: Phi, w; J)
        std::memcpy(prm.ctab, c->tables.data(), std::min<size_t>(c->tables.size(), FEA_CTAB_MAX) * sizeof(double));
        std::memcpy(prm.jtab, c->jplain.data(), std::min<size_t>(c->jplain.size(), FEA_JTAB_MAX) * sizeof(double));
        const int rc = fea_launch_tensor5(prm, c->order, c->t_smem, c->t_grid, c->stream);
        if (rc != 0) return c->fail(FEA_E_CUDA, "k_tensor5 launch: %s", cudaGetErrorString((cudaError_t)rc));
        return FEA_OK;
    }
    if (prm.out_m || prm.out_c) {
        const int rc = fea_launch_tensor(prm, c->order, c->t_smem, c->t_grid, c->stream);
        if (rc != 0) return c->fail(FEA_E_CUDA, "k_tensor launch: %s", cudaGetErrorString((cudaError_t)rc));
    }
    if (c->split && ct_vals) {  // C o2 v with the rule of C
        prm.tab = c->d_ttab_c;
        prm.qfrag = c->d_tables_c;
        prm.nq = c->nq_c;
        prm.out_m = nullptr;
        prm.out_c = ct_vals;
        const int rc = fea_launch_tensor(prm, c->order, c->t_smem, c->t_grid, c->stream);
        if (rc != 0) return c->fail(FEA_E_CUDA, "k_tensor launch: %s", cudaGetErrorString((cudaError_t)rc));
    }
    return FEA_OK;
}

fea_status fea_nccl_unique_id(void* id_out) {
    if (!id_out) return FEA_E_ARG;
    if (!nccl().ok) return FEA_E_NCCL;
    ncclUniqueId id;
    if (nccl().getUniqueId(&id) != ncclSuccess) return FEA_E_NCCL;
    std::memcpy(id_out, &id, sizeof(id));
    return FEA_OK;
}

fea_status fea_set_host_transport(fea_ctx c, fea_host_allgather_fn fn, void* user) {
    if (!c) return FEA_E_ARG;
    c->htrans = fn;
    c->huser = user;
    return FEA_OK;
}

fea_status fea_set_nccl(fea_ctx c, const void* id_bytes) {
    if (!c || !id_bytes) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    if (!nccl().ok) return c->fail(FEA_E_NCCL, "libnccl.so.2 could not be loaded");
    cudaSetDevice(c->device);
    ncclUniqueId id;
    std::memcpy(&id, id_bytes, sizeof(id));
    ncclComm_t comm;
    ncclResult_t r = nccl().commInitRank(&comm, c->world, id, c->rank);
    if (r != ncclSuccess) return c->fail(FEA_E_NCCL, "ncclCommInitRank: %s", nccl().getErrorString(r));
    if (c->comm) nccl().commDestroy((ncclComm_t)c->comm);
    c->comm = comm;
    return FEA_OK;
}

fea_status fea_sync(fea_ctx c) {
    if (!c) return FEA_E_ARG;
    if (c->host_only) return c->fail(FEA_E_STATE, "host-only (planning) context has no device");
    cudaSetDevice(c->device);
    FEA_CUDA(c, cudaStreamSynchronize(c->stream));
    FEA_CUDA(c, cudaGetLastError());
    return FEA_OK;
}

fea_status fea_get_stat(fea_ctx c, int key, int64_t* value) {
    if (!c || !value) return FEA_E_ARG;
    if (!c->have_plan) return c->fail(FEA_E_STATE, "no plan");
    switch (key) {
        case 1: *value = c->nblocks; break;
        case 2: *value = c->stat_visits; break;
        case 3: *value = c->stat_owned; break;
        case 4: *value = c->stat_entries; break;
        case 5: *value = c->launches_per_call; break;
        case 6: *value = c->smem_bytes; break;
        case 7: *value = c->e_max; break;
        case 8: *value = c->grid; break;
        case 9: *value = c->record_bytes; break;
        case 20: case 21: case 22: case 23: case 24: case 25: case 26: case 27:
        case 28: case 29: case 30: case 31: case 32: case 33: case 34: case 35: {  // FEA_DEBUG_TIMING cycle sums
            unsigned long long v = 0;
            if (c->d_dbg) FEA_CUDA(c, cudaMemcpy(&v, c->d_dbg + (key - 20), sizeof(v), cudaMemcpyDeviceToHost));
            *value = (int64_t)v;
            break;
        }
        case 10: *value = c->rec_max; break;
        case 36: case 37: {  // FEA_TUNE_TIMING: exchange / assembly time of the last call, microseconds
            const int i0 = key == 36 ? 0 : 2;
            const bool have = key == 36 ? c->t_exch : c->t_asm;
            float ms = 0.f;
            if (have) {
                FEA_CUDA(c, cudaEventSynchronize(c->ev_t[i0 + 1]));
                FEA_CUDA(c, cudaEventElapsedTime(&ms, c->ev_t[i0], c->ev_t[i0 + 1]));
            }
            *value = have ? (int64_t)llround(1000.0 * ms) : -1;
            break;
        }
        default:
            if (key >= 40 && key < 1536 + 24) {  // FEA_DEBUG_MODE & 8 / 32 trace words
                unsigned long long v = 0;
                if (c->d_dbg) FEA_CUDA(c, cudaMemcpy(&v, c->d_dbg + 16 + (key - 40), sizeof(v), cudaMemcpyDeviceToHost));
                *value = (int64_t)v;
                break;
            }
            return c->fail(FEA_E_ARG, "unknown stat key %d", key);
        case 11: *value = c->kver; break;
        case 16: *value = c->have_tplan ? c->t_nblocks : -1; break;
        case 17: *value = c->have_tplan ? c->t_visits : -1; break;
        case 18: *value = c->have_tplan ? c->t_owned : -1; break;
        case 19: *value = c->have_tplan ? c->t_smem : -1; break;
        case 12: *value = c->have_tplan ? c->t_kver : -1; break;
        case 13: *value = c->have_tplan ? c->t_grid : -1; break;
        case 14: *value = c->maxI; break;
        case 15: *value = c->n_int; break;
        case 38: *value = c->skip_full ? 1000 * c->skip_work / c->skip_full : 1000; break;  // v6 A2 row-tile work, per mille
        case 39: *value = c->skip_work ? 1000 * c->skip_crit / c->skip_work : 1000; break;  // v6 A-warp imbalance, per mille
    }
    return FEA_OK;
}

}  // extern "C"
