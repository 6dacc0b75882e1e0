/*
 * oracle/oracle.c -- plain, slow, obviously-correct CPU assembler (Algorithm 1 of the paper).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_2204_03893_b200/); the only common module is
 * the seeded input generator fea_inputs/ (meshes, DOF maps, rule values, u fields).
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   M = sum_e M_e,  M_e = sum_q w_q m_q phi_q phi_q^T |det B_e|          (Sec. 3)
 *   C = sum_e C_e,  C_e = sum_q w_q c_q J_q A_e J_q^T |det B_e|           (Sec. 3)
 *   with B_e = [b - a, c - a], A_e = (B_e^T B_e)^{-1},
 *   m_q = m(u_h(x_q)), c_q = c(u_h(x_q)), u_h = phi^T u (reading 3),
 *   scattered M(N_e, N_e) += M_e (Algorithm 1).
 * followed literally: element loop, quadrature loop, local (i, j) loops, scatter with a
 * binary search in the row.  No Khatri-Rao product, no B matrix, no symmetry reduction.
 *
 * Pattern: structural union over elements of N_e x N_e (reading 9), built from the
 * DOF -> element incidence, per row sorted unique columns.
 *
 * Parity status of every function: pinned (tests/test_oracle_*.py), see DESIGN.md.
 * Compile: gcc -O2 -ffp-contract=off -fopenmp -shared -fPIC (reading 18).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXP 15  /* n_p <= 15 (order <= 4) */
#define OR_MAXQ 64

/* ---- reference element (Algorithm 1: "Compute phi_q and J_q") ---- */

/* Lagrange nodes (k0, k1, k2)/p in the documented local order (reading 7). */
static int or_nodes(int p, int k[][3]) {
    int n = 0, t, k1, k2;
    k[n][0] = p; k[n][1] = 0; k[n][2] = 0; n++;
    k[n][0] = 0; k[n][1] = p; k[n][2] = 0; n++;
    k[n][0] = 0; k[n][1] = 0; k[n][2] = p; n++;
    for (t = 1; t < p; t++) { k[n][0] = 0;     k[n][1] = p - t; k[n][2] = t;     n++; } /* e0 v1->v2 */
    for (t = 1; t < p; t++) { k[n][0] = t;     k[n][1] = 0;     k[n][2] = p - t; n++; } /* e1 v2->v0 */
    for (t = 1; t < p; t++) { k[n][0] = p - t; k[n][1] = t;     k[n][2] = 0;     n++; } /* e2 v0->v1 */
    for (k1 = 1; k1 < p; k1++)
        for (k2 = 1; k2 < p; k2++)
            if (p - k1 - k2 >= 1) { k[n][0] = p - k1 - k2; k[n][1] = k1; k[n][2] = k2; n++; }
    return n;
}

/* phi_i(lambda) = prod_m prod_{t < k_m} (p lambda_m - t) / (t + 1), and its partial
 * derivatives d phi / d lambda_m by the product rule, in long double. */
static void or_lagrange(int p, const int kk[3], const long double lam[3], long double* val, long double dlam[3]) {
    long double f[3], df[3];
    int m, t, s;
    for (m = 0; m < 3; m++) {
        long double prod = 1.0L, dsum = 0.0L;
        for (t = 0; t < kk[m]; t++) prod *= ((long double)p * lam[m] - t) / (t + 1);
        /* derivative of prod_t (p lam - t)/(t+1) w.r.t. lam */
        for (s = 0; s < kk[m]; s++) {
            long double term = (long double)p / (s + 1);
            for (t = 0; t < kk[m]; t++)
                if (t != s) term *= ((long double)p * lam[m] - t) / (t + 1);
            dsum += term;
        }
        f[m] = prod; df[m] = dsum;
    }
    *val = f[0] * f[1] * f[2];
    dlam[0] = df[0] * f[1] * f[2];
    dlam[1] = f[0] * df[1] * f[2];
    dlam[2] = f[0] * f[1] * df[2];
}

/* phi[i*nq + q] = phi_i(x_q); grad[(q*np + i)*2 + d] = d phi_i / d xhat_d at x_q.
 * Reference coordinates: lambda0 = 1 - x - y, lambda1 = x, lambda2 = y. */
int oracle_basis(int p, int nq, const double* qxy, double* phi, double* grad) {
    int kk[OR_MAXP][3];
    int np, i, q;
    if (p < 1 || p > 4 || nq < 1 || nq > OR_MAXQ) return -1;
    np = or_nodes(p, kk);
    for (q = 0; q < nq; q++) {
        long double x = qxy[2 * q], y = qxy[2 * q + 1];
        long double lam[3] = {1.0L - x - y, x, y};
        for (i = 0; i < np; i++) {
            long double v, dl[3];
            or_lagrange(p, kk[i], lam, &v, dl);
            phi[i * nq + q] = (double)v;
            grad[(q * np + i) * 2 + 0] = (double)(dl[1] - dl[0]);
            grad[(q * np + i) * 2 + 1] = (double)(dl[2] - dl[0]);
        }
    }
    return np;
}

/* ---- coefficient k(u) (reading 17; NEXT-4 piecewise linear PAPER.md:560-568) ---- */
static double or_k(int kind, int npar, const double* par, double u) {
    int i;
    if (kind == 0) { /* polynomial sum_i par[i] u^i, Horner */
        double r = par[npar - 1];
        for (i = npar - 2; i >= 0; i--) r = r * u + par[i];
        return r;
    }
    if (kind == 1) return par[0] * exp(par[1] * u); /* c0 exp(c1 u) */
    if (kind == 2) { /* breakpoints (T_1,k_1),...,(T_m,k_m): segment s covers (T_s, T_{s+1}],
                        the first segment also T_1 and below, the last also above T_m */
        int m = npar / 2, s = 0;
        while (s < m - 2 && u > par[2 * (s + 1)]) s++;
        {
            double T0 = par[2 * s], k0 = par[2 * s + 1], T1 = par[2 * s + 2], k1 = par[2 * s + 3];
            return k0 + (k1 - k0) / (T1 - T0) * (u - T0);
        }
    }
    return NAN;
}

/* derivative k'(u), used by the tensor contractions */
static double or_dk(int kind, int npar, const double* par, double u) {
    int i;
    if (kind == 0) {
        double r = 0.0;
        for (i = npar - 1; i >= 1; i--) r = r * u + i * par[i];
        return r;
    }
    if (kind == 1) return par[0] * par[1] * exp(par[1] * u);
    if (kind == 2) {
        int m = npar / 2, s = 0;
        while (s < m - 2 && u > par[2 * (s + 1)]) s++;
        return (par[2 * s + 3] - par[2 * s + 1]) / (par[2 * s + 2] - par[2 * s]);
    }
    return NAN;
}

double oracle_k(int kind, int npar, const double* par, double u) { return or_k(kind, npar, par, u); }
double oracle_dk(int kind, int npar, const double* par, double u) { return or_dk(kind, npar, par, u); }

/* ---- pattern (reading 9): rows [r0, r1), row_ptr local (starts at 0) ---- */
typedef struct { int64_t* ptr; int32_t* elems; } or_incidence;

static int or_build_incidence(int64_t n_dof, int64_t n_e, int np, const int32_t* ed, or_incidence* inc) {
    int64_t e, d;
    int i;
    int64_t* cnt = (int64_t*)calloc((size_t)n_dof + 1, sizeof(int64_t));
    if (!cnt) return -1;
    for (e = 0; e < n_e; e++)
        for (i = 0; i < np; i++) {
            int32_t g = ed[e * np + i];
            if (g < 0 || g >= n_dof) { free(cnt); return -2; }
            cnt[g + 1]++;
        }
    for (d = 0; d < n_dof; d++) cnt[d + 1] += cnt[d];
    inc->elems = (int32_t*)malloc(sizeof(int32_t) * (size_t)(cnt[n_dof] > 0 ? cnt[n_dof] : 1));
    inc->ptr = (int64_t*)malloc(sizeof(int64_t) * ((size_t)n_dof + 1));
    if (!inc->elems || !inc->ptr) { free(cnt); return -1; }
    memcpy(inc->ptr, cnt, sizeof(int64_t) * ((size_t)n_dof + 1));
    for (e = 0; e < n_e; e++)
        for (i = 0; i < np; i++) {
            int32_t g = ed[e * np + i];
            inc->elems[cnt[g]++] = (int32_t)e; /* ascending e within each DOF */
        }
    free(cnt);
    return 0;
}

static int or_cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}

/* If col_idx == NULL only row_ptr is computed. Returns 0 or <0 on error. */
int oracle_pattern(int64_t n_dof, int64_t n_e, int np, const int32_t* elem_dof,
                   int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col_idx) {
    or_incidence inc;
    int64_t r;
    int32_t* buf;
    int rc = or_build_incidence(n_dof, n_e, np, elem_dof, &inc);
    if (rc) return rc;
    {
        int64_t maxdeg = 0, d;
        for (d = r0; d < r1; d++)
            if (inc.ptr[d + 1] - inc.ptr[d] > maxdeg) maxdeg = inc.ptr[d + 1] - inc.ptr[d];
        buf = (int32_t*)malloc(sizeof(int32_t) * (size_t)(maxdeg * np + 1));
    }
    if (!buf) return -1;
    row_ptr[0] = 0;
    for (r = r0; r < r1; r++) {
        int64_t k, n = 0, u = 0;
        int i;
        for (k = inc.ptr[r]; k < inc.ptr[r + 1]; k++) {
            int64_t e = inc.elems[k];
            for (i = 0; i < np; i++) buf[n++] = elem_dof[e * np + i];
        }
        qsort(buf, (size_t)n, sizeof(int32_t), or_cmp_i32);
        for (k = 0; k < n; k++)
            if (k == 0 || buf[k] != buf[k - 1]) {
                if (col_idx) col_idx[row_ptr[r - r0] + u] = buf[k];
                u++;
            }
        row_ptr[r - r0 + 1] = row_ptr[r - r0] + u;
    }
    free(buf);
    free(inc.ptr);
    free(inc.elems);
    return 0;
}

/* ---- Algorithm 1 ---- */

static int64_t or_slot(const int64_t* row_ptr, const int32_t* col_idx, int64_t lr, int32_t col) {
    int64_t lo = row_ptr[lr], hi = row_ptr[lr + 1] - 1;
    while (lo <= hi) {
        int64_t mid = lo + (hi - lo) / 2;
        if (col_idx[mid] == col) return mid;
        if (col_idx[mid] < col) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

typedef struct {
    int p, nq, np;
    const double* qw;
    double phi[OR_MAXP * OR_MAXQ];
    double J[OR_MAXQ * OR_MAXP * 2];
} or_ref;

/* Element e: M_e and C_e of PAPER.md:134-135. Returns 0, or -3 for a degenerate element. */
static int or_element(const or_ref* R, const double* vert_xy, const int32_t* ev, const int32_t* ed,
                      const double* u, int m_kind, int m_npar, const double* m_par,
                      int c_kind, int c_npar, const double* c_par, int64_t e,
                      double* Me, double* Ce) {
    int np = R->np, nq = R->nq, i, j, q;
    const double* a = vert_xy + 2 * (int64_t)ev[3 * e + 0];
    const double* b = vert_xy + 2 * (int64_t)ev[3 * e + 1];
    const double* c = vert_xy + 2 * (int64_t)ev[3 * e + 2];
    /* B_e = [b - a, c - a], columns */
    double B00 = b[0] - a[0], B10 = b[1] - a[1];
    double B01 = c[0] - a[0], B11 = c[1] - a[1];
    double det = B00 * B11 - B01 * B10;
    double absdet = fabs(det);
    /* B^T B and its explicit 2x2 inverse A_e */
    double G00 = B00 * B00 + B10 * B10;
    double G01 = B00 * B01 + B10 * B11;
    double G11 = B01 * B01 + B11 * B11;
    double gdet = G00 * G11 - G01 * G01;
    double A00 = G11 / gdet, A01 = -G01 / gdet, A10 = -G01 / gdet, A11 = G00 / gdet;
    double diam2 = G00;
    if (G11 > diam2) diam2 = G11;
    {
        double e20 = (c[0] - b[0]) * (c[0] - b[0]) + (c[1] - b[1]) * (c[1] - b[1]);
        if (e20 > diam2) diam2 = e20;
    }
    if (!(absdet >= 1e-14 * diam2)) return -3;
    for (i = 0; i < np * np; i++) { if (Me) Me[i] = 0.0; if (Ce) Ce[i] = 0.0; }
    for (q = 0; q < nq; q++) {
        /* u_h(x_q) = sum_i phi_i(x_q) u_i (interpolate, then evaluate k: reading 3) */
        double uq = 0.0;
        for (i = 0; i < np; i++) uq += R->phi[i * nq + q] * u[ed[e * np + i]];
        if (Me) {
            double mq = or_k(m_kind, m_npar, m_par, uq);
            for (i = 0; i < np; i++)
                for (j = 0; j < np; j++)
                    Me[i * np + j] += R->qw[q] * mq * R->phi[i * nq + q] * R->phi[j * nq + q] * absdet;
        }
        if (Ce) {
            double cq = or_k(c_kind, c_npar, c_par, uq);
            const double* Jq = R->J + (int64_t)q * np * 2;
            for (i = 0; i < np; i++)
                for (j = 0; j < np; j++) {
                    /* (J_q A_e J_q^T)_{ij} = sum_{r,s} J_q[i,r] A_e[r,s] J_q[j,s] */
                    double s = Jq[i * 2 + 0] * A00 * Jq[j * 2 + 0] + Jq[i * 2 + 0] * A01 * Jq[j * 2 + 1]
                             + Jq[i * 2 + 1] * A10 * Jq[j * 2 + 0] + Jq[i * 2 + 1] * A11 * Jq[j * 2 + 1];
                    Ce[i * np + j] += R->qw[q] * cq * s * absdet;
                }
        }
    }
    return 0;
}

/*
 * Assemble the rows [r0, r1) of M (if M != NULL) and C (if C != NULL) into the given
 * pattern (row_ptr local, starting at 0).  Threads own disjoint row sub-ranges and each
 * processes, in ascending e, every element touching its rows, so the per-slot summation
 * order (ascending e) is independent of the thread count.
 * Returns 0, -3 (degenerate element; *bad_elem set), -4 (pattern miss), <0 other.
 */
int oracle_assemble(int p, int nq, const double* qxy, const double* qw,
                    int64_t n_vert, const double* vert_xy, int64_t n_e, const int32_t* elem_vert,
                    const int32_t* elem_dof, int64_t n_dof, const double* u,
                    int m_kind, int m_npar, const double* m_par,
                    int c_kind, int c_npar, const double* c_par,
                    int64_t r0, int64_t r1, const int64_t* row_ptr, const int32_t* col_idx,
                    double* M, double* C, int nthreads, int64_t* bad_elem) {
    or_ref R;
    int64_t nnz = row_ptr[r1 - r0];
    int err = 0;
    (void)n_vert;
    (void)n_dof;
    R.p = p; R.nq = nq; R.qw = qw;
    R.np = oracle_basis(p, nq, qxy, R.phi, R.J);
    if (R.np < 0) return -1;
    if (M) memset(M, 0, sizeof(double) * (size_t)nnz);
    if (C) memset(C, 0, sizeof(double) * (size_t)nnz);
    if (nthreads < 1) nthreads = 1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nthreads)
#endif
    {
        int tid = 0, nt = 1, lerr = 0;
        int64_t a, b, e;
        int np = R.np, i, j;
        double Me[OR_MAXP * OR_MAXP], Ce[OR_MAXP * OR_MAXP];
#ifdef _OPENMP
        tid = omp_get_thread_num();
        nt = omp_get_num_threads();
#endif
        a = r0 + (r1 - r0) * tid / nt;
        b = r0 + (r1 - r0) * (tid + 1) / nt;
        for (e = 0; e < n_e && lerr == 0; e++) {
            int touches = 0, rc;
            for (i = 0; i < np; i++) {
                int32_t g = elem_dof[e * np + i];
                if (g >= a && g < b) { touches = 1; break; }
            }
            if (!touches) continue;
            rc = or_element(&R, vert_xy, elem_vert, elem_dof, u, m_kind, m_npar, m_par,
                            c_kind, c_npar, c_par, e, M ? Me : NULL, C ? Ce : NULL);
            if (rc) { lerr = rc; if (bad_elem) *bad_elem = e; break; }
            /* M(N_e, N_e) += M_e; C(N_e, N_e) += C_e   (Algorithm 1) */
            for (i = 0; i < np; i++) {
                int32_t gi = elem_dof[e * np + i];
                if (gi < a || gi >= b) continue;
                for (j = 0; j < np; j++) {
                    int64_t s = or_slot(row_ptr, col_idx, gi - r0, elem_dof[e * np + j]);
                    if (s < 0) { lerr = -4; break; }
                    if (M) M[s] += Me[i * np + j];
                    if (C) C[s] += Ce[i * np + j];
                }
            }
        }
#ifdef _OPENMP
#pragma omp critical
#endif
        if (lerr && !err) err = lerr;
    }
    return err;
}

/*
 * NEXT-1 / NEXT-2: contractions of the third-order tensors of PAPER.md:282-289 with a
 * vector v in the second mode, assembled element by element:
 *   (Mt o2 v)_{ik} = sum_e sum_q w_q m'_q phi_i phi_k (phi^T v_e) |det B_e|
 *   (Ct o2 v)_{ik} = sum_e sum_q w_q c'_q (J_q[i,:] A_e (J_q^T v_e)) phi_k |det B_e|
 *                    i.e. C_{ijk} = int c' grad phi_i . grad phi_j phi_k, contracted
 *                    over j with v_j.  Rows i, columns k.  Nonsymmetric.
 * m' = k'(u_h(x_q)).  Same pattern as M and C.
 */
int oracle_assemble_tensor_contraction(int p, int nq, const double* qxy, const double* qw,
                    const double* vert_xy, int64_t n_e, const int32_t* elem_vert,
                    const int32_t* elem_dof, const double* u, const double* v,
                    int m_kind, int m_npar, const double* m_par,
                    int c_kind, int c_npar, const double* c_par,
                    int64_t r0, int64_t r1, const int64_t* row_ptr, const int32_t* col_idx,
                    double* MT, double* CT) {
    or_ref R;
    int64_t nnz = row_ptr[r1 - r0], e;
    int np, nqq = nq, i, j, k, q;
    R.p = p; R.nq = nq; R.qw = qw;
    R.np = oracle_basis(p, nq, qxy, R.phi, R.J);
    if (R.np < 0) return -1;
    np = R.np;
    if (MT) memset(MT, 0, sizeof(double) * (size_t)nnz);
    if (CT) memset(CT, 0, sizeof(double) * (size_t)nnz);
    for (e = 0; e < n_e; e++) {
        double Te[OR_MAXP * OR_MAXP], Ue[OR_MAXP * OR_MAXP];
        const double* a = vert_xy + 2 * (int64_t)elem_vert[3 * e + 0];
        const double* b = vert_xy + 2 * (int64_t)elem_vert[3 * e + 1];
        const double* c = vert_xy + 2 * (int64_t)elem_vert[3 * e + 2];
        double B00 = b[0] - a[0], B10 = b[1] - a[1], B01 = c[0] - a[0], B11 = c[1] - a[1];
        double absdet = fabs(B00 * B11 - B01 * B10);
        double G00 = B00 * B00 + B10 * B10, G01 = B00 * B01 + B10 * B11, G11 = B01 * B01 + B11 * B11;
        double gdet = G00 * G11 - G01 * G01;
        double A00 = G11 / gdet, A01 = -G01 / gdet, A10 = -G01 / gdet, A11 = G00 / gdet;
        int touches = 0;
        for (i = 0; i < np; i++) {
            int32_t g = elem_dof[e * np + i];
            if (g >= r0 && g < r1) touches = 1;
        }
        if (!touches) continue;
        for (i = 0; i < np * np; i++) { Te[i] = 0.0; Ue[i] = 0.0; }
        for (q = 0; q < nqq; q++) {
            double uq = 0.0, vq = 0.0;
            const double* Jq = R.J + (int64_t)q * np * 2;
            for (i = 0; i < np; i++) {
                uq += R.phi[i * nq + q] * u[elem_dof[e * np + i]];
                vq += R.phi[i * nq + q] * v[elem_dof[e * np + i]];
            }
            if (MT) {
                double mdq = or_dk(m_kind, m_npar, m_par, uq);
                for (i = 0; i < np; i++)
                    for (k = 0; k < np; k++)
                        Te[i * np + k] += qw[q] * mdq * R.phi[i * nq + q] * R.phi[k * nq + q] * vq * absdet;
            }
            if (CT) {
                double cdq = or_dk(c_kind, c_npar, c_par, uq);
                for (i = 0; i < np; i++)
                    for (k = 0; k < np; k++) {
                        double s = 0.0;
                        for (j = 0; j < np; j++) {
                            double vj = v[elem_dof[e * np + j]];
                            double gij = Jq[i * 2 + 0] * A00 * Jq[j * 2 + 0] + Jq[i * 2 + 0] * A01 * Jq[j * 2 + 1]
                                       + Jq[i * 2 + 1] * A10 * Jq[j * 2 + 0] + Jq[i * 2 + 1] * A11 * Jq[j * 2 + 1];
                            s += gij * vj;
                        }
                        Ue[i * np + k] += qw[q] * cdq * s * R.phi[k * nq + q] * absdet;
                    }
            }
        }
        for (i = 0; i < np; i++) {
            int32_t gi = elem_dof[e * np + i];
            if (gi < r0 || gi >= r1) continue;
            for (k = 0; k < np; k++) {
                int64_t s = or_slot(row_ptr, col_idx, gi - r0, elem_dof[e * np + k]);
                if (s < 0) return -4;
                if (MT) MT[s] += Te[i * np + k];
                if (CT) CT[s] += Ue[i * np + k];
            }
        }
    }
    return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
