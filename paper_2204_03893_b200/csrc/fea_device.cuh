// fea_device.cuh -- device helpers shared by the sm_100a kernels (fea_kernels.cu: v4, p >= 3 and
// generic rules; fea_kernels5.cu: v5, p <= 2; fea_kernels_t.cu: tensor contractions): PTX wrappers
// (mbarrier, TMA bulk copy, cp.async, DMMA, L2 prefetch), the coefficient k(u) and k'(u), element
// geometry, and phase B (fixed-order sums of each CSR slot's contributors).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "fea_internal.h"

namespace fea_dev {

// Device-side bounds checks of the FEA_BOUNDS_CHECK build (FEA_BUILD_DEFS=-DFEA_BOUNDS_CHECK):
// compute-sanitizer is not available on this pool, so the kernels check their own shared- and
// global-memory indices (tools/sanitize_cases.py runs every kernel so built); a failed check
// prints its site and traps.  The production build compiles them out.
#ifdef FEA_BOUNDS_CHECK
#define FEA_CHECK(cond)                                                                               \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("FEA_CHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #cond,    \
                   (int)blockIdx.x, (int)threadIdx.x);                                                \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#else
#define FEA_CHECK(cond) \
    do {                \
    } while (0)
#endif

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1D TMA bulk copy global -> shared, completion counted on an mbarrier
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
// arrive on `bar` once all prior cp.async of this thread have completed
__device__ __forceinline__ void cp_async_mbar_arrive(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumer_sync(int nct) {  // named barrier 1: consumer warps only
    asm volatile("bar.sync 1, %0;" ::"r"(nct) : "memory");
}
// D = A (8x4, row) * B (4x8, col) + D on the FP64 tensor core; fragment ownership per lane
// (g = lane / 4, c = lane % 4): a = A[g][c], b = B[c][g], d = D[g][2c .. 2c+1].
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}

// ------------------------------------------------------------------ math
template <int N>
__device__ __forceinline__ double horner(const double* par, double u) {  // sum_{i<N} par[i] u^i
    double r = par[N - 1];
#pragma unroll
    for (int i = N - 2; i >= 0; --i) r = fma(r, u, par[i]);
    return r;
}

// k(u); the branch is warp-uniform (one coefficient per launch), each case straight-line.
__device__ __forceinline__ double keval(const FeaCoef& c, double u) {
    if (c.kind == 0) {
        switch (c.npar) {
            case 1: return c.par[0];
            case 2: return horner<2>(c.par, u);
            case 3: return horner<3>(c.par, u);
            case 4: return horner<4>(c.par, u);
            case 5: return horner<5>(c.par, u);
            case 6: return horner<6>(c.par, u);
            case 7: return horner<7>(c.par, u);
            case 8: return horner<8>(c.par, u);
            default: return horner<9>(c.par, u);
        }
    }
    if (c.kind == 1) return c.par[0] * exp(c.par[1] * u);
    // piecewise linear, segment s covers (T_s, T_{s+1}]
    const int m = c.npar / 2;
    int s = 0;
    while (s < m - 2 && u > c.par[2 * (s + 1)]) ++s;
    const double T0 = c.par[2 * s], k0 = c.par[2 * s + 1], T1 = c.par[2 * s + 2], k1 = c.par[2 * s + 3];
    return k0 + (k1 - k0) / (T1 - T0) * (u - T0);
}

// exp and the piecewise-linear k out of line (one copy of the code each)
static __device__ __noinline__ double k_exp(double c0, double c1, double u) { return c0 * exp(c1 * u); }
static __device__ __noinline__ double k_pwl(const FeaCoef& c, double u) {
    const int m = c.npar / 2;
    int s = 0;
    while (s < m - 2 && u > c.par[2 * (s + 1)]) ++s;
    const double T0 = c.par[2 * s], k0 = c.par[2 * s + 1], T1 = c.par[2 * s + 2], k1 = c.par[2 * s + 3];
    return k0 + (k1 - k0) / (T1 - T0) * (u - T0);
}

// k(u_q) for all N quadrature points at once: one Horner loop over the coefficients with the N
// points as independent FMA chains (compact code, the same per-point arithmetic as keval).
template <int N>
__device__ __forceinline__ void keval_all(const FeaCoef& c, const double (&u)[N], double (&k)[N]) {
    if (c.kind == 0) {
        const int n = c.npar;
        const double top = c.par[n - 1];
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = top;
#pragma unroll 1
        for (int i = n - 2; i >= 0; --i) {
            const double a = c.par[i];
#pragma unroll
            for (int q = 0; q < N; ++q) k[q] = fma(k[q], u[q], a);
        }
    } else if (c.kind == 1) {
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = k_exp(c.par[0], c.par[1], u[q]);
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = k_pwl(c, u[q]);
    }
}

// Element geometry from the staged vertex coordinates: b_e = |det B_e|, A_e = (B^T B)^{-1}
__device__ __forceinline__ void geometry(const double2* __restrict__ gX, int e_max, int le, double& absdet,
                                         double& A00, double& A11, double& A01) {
    const double2 a = gX[le], b = gX[e_max + le], c = gX[2 * e_max + le];
    const double B00 = b.x - a.x, B10 = b.y - a.y, B01 = c.x - a.x, B11 = c.y - a.y;
    const double det = B00 * B11 - B01 * B10;
    absdet = fabs(det);
    const double inv = 1.0 / (det * det);  // det(B^T B) = det(B)^2
    A00 = (B01 * B01 + B11 * B11) * inv;
    A11 = (B00 * B00 + B10 * B10) * inv;
    A01 = -(B00 * B01 + B10 * B11) * inv;
}


// ---- phase B of kernel v5 (record format: fea_internal.h fea5_item_bytes): one vector load per
// item gives its slot and its C contributor offsets; ILP items per thread are in flight.  Each
// slot sums its contributors in the stored (ascending library element) order.
template <int R> struct ItemWord;
template <> struct ItemWord<4> { using T = uint32_t; };
template <> struct ItemWord<8> { using T = uint2; };
template <> struct ItemWord<16> { using T = uint4; };
// 16-bit field k of an item word (k compile-time after unrolling; shifts, no address taken)
__device__ __forceinline__ uint32_t word_of(uint32_t w, int) { return w; }
__device__ __forceinline__ uint32_t word_of(const uint2& w, int i) { return i == 0 ? w.x : w.y; }
__device__ __forceinline__ uint32_t word_of(const uint4& w, int i) {
    return i == 0 ? w.x : i == 1 ? w.y : i == 2 ? w.z : w.w;
}
template <typename W>
__device__ __forceinline__ int u16_of(const W& w, int k) { return (word_of(w, k >> 1) >> (16 * (k & 1))) & 0xffff; }

// ORIENT (tensor contractions): bit 15 of an offset selects sVd (entry (i, k) with local i > k)
// over sVc for the nonsymmetric channel; the symmetric channel ignores it.
// `first` is this thread's first item of the class (the classes continue one warp-aligned round-robin over
// the threads, so no warp takes every class's tail)
// IL: V_m and V_c interleaved ({m, c} double2 at sVm[2 off]): one 16-byte load per contributor
template <int C, bool DO_M, bool DO_C, int ILP, bool ORIENT = false, bool IL = false>
__device__ __forceinline__ void items5(const uint8_t* __restrict__ base, int n, const double* __restrict__ sVm,
                                       const double* __restrict__ sVc, double* om, double* oc, int first, int nthr,
                                       const double* __restrict__ sVd = nullptr) {
    using W = typename ItemWord<fea5_item_bytes(C)>::T;
    const W* it = reinterpret_cast<const W*>(base);
    for (int i0 = first; i0 < n; i0 += ILP * nthr) {
        W w[ILP];
#pragma unroll
        for (int u = 0; u < ILP; ++u) w[u] = it[min(i0 + u * nthr, n - 1)];  // clamped: always valid
        double vm[ILP][C], vc[ILP][C];
#pragma unroll
        for (int u = 0; u < ILP; ++u)
#pragma unroll
            for (int q = 0; q < C; ++q) {
                const int raw = u16_of(w[u], 1 + q);
                const int off = ORIENT ? (raw & 0x7fff) : raw;
                FEA_CHECK(off < 32768);
                if (IL) {
                    const double2 v = reinterpret_cast<const double2*>(sVm)[off];
                    vm[u][q] = v.x;
                    vc[u][q] = v.y;
                } else {
                    if (DO_M) vm[u][q] = sVm[off];
                    if (DO_C) vc[u][q] = (ORIENT && (raw & 0x8000)) ? sVd[off] : sVc[off];
                }
            }
#pragma unroll
        for (int u = 0; u < ILP; ++u)
            if (i0 + u * nthr < n) {
                double am = 0.0, ac = 0.0;
#pragma unroll
                for (int q = 0; q < C; ++q) {
                    if (DO_M) am += vm[u][q];
                    if (DO_C) ac += vc[u][q];
                }
                const int slot = u16_of(w[u], 0);
                if (DO_M) om[slot] = am;
                if (DO_C) oc[slot] = ac;
            }
    }
}

template <bool DO_M, bool DO_C, bool ORIENT = false, bool IL = false>
__device__ __forceinline__ void items5_generic(const uint8_t* __restrict__ base, int C, int n, int R,
                                               const double* __restrict__ sVm, const double* __restrict__ sVc,
                                               double* om, double* oc, int first, int nthr,
                                               const double* __restrict__ sVd = nullptr) {
    for (int i = first; i < n; i += nthr) {
        const uint16_t* w = reinterpret_cast<const uint16_t*>(base + (size_t)i * R);
        double am = 0.0, ac = 0.0;
        for (int q = 0; q < C; ++q) {
            const int raw = w[1 + q];
            const int off = ORIENT ? (raw & 0x7fff) : raw;
            if (IL) {
                const double2 v = reinterpret_cast<const double2*>(sVm)[off];
                am += v.x;
                ac += v.y;
            } else {
                if (DO_M) am += sVm[off];
                if (DO_C) ac += (ORIENT && (raw & 0x8000)) ? sVd[off] : sVc[off];
            }
        }
        if (DO_M) om[w[0]] = am;
        if (DO_C) oc[w[0]] = ac;
    }
}

// the classes of one block, threads tid of nthr (a block's B is split across all warps)
template <bool DO_M, bool DO_C, bool ORIENT = false, bool IL = false>
__device__ __forceinline__ void phase_b5(const uint8_t* __restrict__ rec, int ncls, const double* __restrict__ sVm,
                                         const double* __restrict__ sVc, double* om, double* oc, int tid, int nthr,
                                         const double* __restrict__ sVd = nullptr) {
    const int4* cls = reinterpret_cast<const int4*>(rec);
    int start = 0;  // items of the previous classes, rounded up to warps (mod nthr): one round-robin
    for (int k = 0; k < ncls; ++k) {
        const int4 c = cls[k];  // {C, n_items, byte offset, item bytes}
        const uint8_t* base = rec + c.z;
        const int first = tid >= start ? tid - start : tid - start + nthr;
        switch (c.x) {
            case 1: items5<1, DO_M, DO_C, 4, ORIENT, IL>(base, c.y, sVm, sVc, om, oc, first, nthr, sVd); break;
            case 2: items5<2, DO_M, DO_C, 4, ORIENT, IL>(base, c.y, sVm, sVc, om, oc, first, nthr, sVd); break;
            case 3: items5<3, DO_M, DO_C, 2, ORIENT, IL>(base, c.y, sVm, sVc, om, oc, first, nthr, sVd); break;
            case 4: items5<4, DO_M, DO_C, 2, ORIENT, IL>(base, c.y, sVm, sVc, om, oc, first, nthr, sVd); break;
            case 6: items5<6, DO_M, DO_C, 2, ORIENT, IL>(base, c.y, sVm, sVc, om, oc, first, nthr, sVd); break;
            default: items5_generic<DO_M, DO_C, ORIENT, IL>(base, c.x, c.y, c.w, sVm, sVc, om, oc, first, nthr, sVd);
        }
        start = (start + ((c.y + 31) & ~31)) % nthr;  // next class warp-aligned (the planner's 32-item groups)
    }
}

// ---- phase B in CSR slot order (kernel v5 with the v6 record format, fea_internal.h): class A =
// one u32 item per slot {u16 V offset 0, u16 V offset 1} (one contributor: offset 1 = the zero
// cell; more than two: 0xffff, a hole), lane l of a warp takes slot 32 c + l of chunk c, so the CSR
// stores of a warp are 256 contiguous bytes per matrix; class B = nB flat items of R bytes {u16 slot,
// u16 C, u16 V offset [C]}, one per thread.  Every slot sums its contributors in ascending library
// element order (the same order as phase_b5).  `rec` is in shared memory; cells are {m, c} double2
// (IL) or doubles.
template <bool DO_M, bool DO_C, bool IL>
__device__ __forceinline__ void phase_b_slots(const uint8_t* __restrict__ rec, int nslots, int nB, int R,
                                              const double* __restrict__ sV, double* om, double* oc, int warp,
                                              int lane, int nwarps) {
    constexpr int U = 4;  // chunks per round (their loads in flight together)
    const uint32_t* ia = reinterpret_cast<const uint32_t*>(rec);
    const int nch = (nslots + 31) >> 5;
    for (int c0 = warp; c0 < nch; c0 += U * nwarps) {
        uint32_t w[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int ch = c0 + u * nwarps;
            w[u] = ch < nch ? ia[ch * 32 + lane] : 0xffffffffu;
        }
        double2 x0[U], x1[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int o0 = w[u] & 0xffff, o1 = w[u] >> 16;
            const bool hole = o0 == 0xffff;
            if (IL) {
                x0[u] = reinterpret_cast<const double2*>(sV)[hole ? 0 : o0];
                x1[u] = reinterpret_cast<const double2*>(sV)[hole ? 0 : o1];
            } else {
                x0[u].x = sV[hole ? 0 : o0];
                x1[u].x = sV[hole ? 0 : o1];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if ((w[u] & 0xffff) == 0xffff) continue;
            const int p = (c0 + u * nwarps) * 32 + lane;
            FEA_CHECK(p < nslots);
            if (IL) {
                om[p] = x0[u].x + x1[u].x;
                oc[p] = x0[u].y + x1[u].y;
            } else if (DO_M) {
                om[p] = x0[u].x + x1[u].x;
            } else {
                oc[p] = x0[u].x + x1[u].x;
            }
        }
    }
    const uint8_t* bB = rec + 4 * (nch * 32);
    for (int it = warp * 32 + lane; it < nB; it += nwarps * 32) {
        const uint16_t* wrd = reinterpret_cast<const uint16_t*>(bB + (size_t)it * R);
        const int sl = wrd[0], C = wrd[1];
        FEA_CHECK(sl < nslots && 2 * (C + 2) <= R);
        double am = 0.0, ac = 0.0;
        for (int q = 0; q < C; ++q) {
            const int o = wrd[2 + q];
            if (IL) {
                const double2 x = reinterpret_cast<const double2*>(sV)[o];
                am += x.x;
                ac += x.y;
            } else {
                am += sV[o];
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
}

// derivative k'(u) of the coefficient (fea.h FEA_K_*); PWL: slope of the segment of u
__device__ __forceinline__ double dkeval(const FeaCoef& c, double u) {
    if (c.kind == 0) {
        double r = 0.0;
        for (int i = c.npar - 1; i >= 1; --i) r = fma(r, u, (double)i * c.par[i]);
        return r;
    }
    if (c.kind == 1) return c.par[0] * c.par[1] * exp(c.par[1] * u);
    const int m = c.npar / 2;
    int s = 0;
    while (s < m - 2 && u > c.par[2 * (s + 1)]) ++s;
    return (c.par[2 * s + 3] - c.par[2 * s + 1]) / (c.par[2 * s + 2] - c.par[2 * s]);
}

static __device__ __noinline__ double dk_exp(double c0, double c1, double u) { return c0 * c1 * exp(c1 * u); }
static __device__ __noinline__ double dk_pwl(const FeaCoef& c, double u) { return dkeval(c, u); }
// k'(u_q) for all N quadrature points at once (the same per-point arithmetic as dkeval: Horner on
// i par_i from the top, the N points as independent FMA chains; PWL, and exp for N > 4, out of line)
template <int N>
__device__ __forceinline__ void dkeval_all(const FeaCoef& c, const double (&u)[N], double (&k)[N]) {
    if (c.kind == 0) {
        const int n = c.npar;
        if (n <= 1) {
#pragma unroll
            for (int q = 0; q < N; ++q) k[q] = 0.0;
            return;
        }
        const double top = (double)(n - 1) * c.par[n - 1];
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = top;
#pragma unroll 1
        for (int i = n - 2; i >= 1; --i) {
            const double a = (double)i * c.par[i];
#pragma unroll
            for (int q = 0; q < N; ++q) k[q] = fma(k[q], u[q], a);
        }
    } else if (c.kind == 1) {
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = N <= 4 ? c.par[0] * c.par[1] * exp(c.par[1] * u[q]) : dk_exp(c.par[0], c.par[1], u[q]);
    } else {
#pragma unroll
        for (int q = 0; q < N; ++q) k[q] = dk_pwl(c, u[q]);
    }
}

// L2 prefetch of a byte range (bulk, no completion tracking); bytes a multiple of 16
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// read-only global loads, issued where written (asm volatile keeps them ahead of their use)
__device__ __forceinline__ double ldg_f64(const double* p) {
    double v;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ double2 ldg_f64x2(const double2* p) {
    double2 v;
    asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ int32_t ldg_s32(const int32_t* p) {
    int32_t v;
    asm volatile("ld.global.nc.s32 %0, [%1];" : "=r"(v) : "l"(p));
    return v;
}

}  // namespace fea_dev
