/* oracle/oracle.c -- TEST INFRASTRUCTURE ONLY: the CPU parity oracle.
 *
 * See oracle.h for what this restates and how it is pinned.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline, --impl reference) load
 * the resulting oracle/liboracle.so; the product never does.
 *
 * Build: oracle/Makefile (gcc -O3 -march=x86-64-v3 -ffp-contract=off -pthread).
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdarg.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define MB 8 /* mini-batch width (SPEC.md:190 default 4; 8 = one AVX-512 lane set) */

static _Thread_local char g_err[512];

static int fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ------------------------------------------------------------------------- */
/* sincos: Cody-Waite reduction by pi/2 (3-part constant, fma) + fdlibm      */
/* minimax kernels on [-pi/4, pi/4].  The CUDA path implements the same     */
/* operation sequence, so results are bit-identical.          */
/* ------------------------------------------------------------------------- */
void orc_sincos(double x, double* s_out, double* c_out) {
    const double two_over_pi = 6.36619772367581382433e-01;
    const double p1 = 1.57079632679489655800e+00;
    const double p2 = 6.12323399573676603587e-17;
    const double p3 = -1.49738490485916983248e-33;
    double q = rint(x * two_over_pi);
    double r = fma(-q, p1, x);
    r = fma(-q, p2, r);
    r = fma(-q, p3, r);
    double z = r * r;
    double ps = fma(z, 1.58969099521155010221e-10, -2.50507602534068634195e-08);
    ps = fma(z, ps, 2.75573137070700676789e-06);
    ps = fma(z, ps, -1.98412698298579493134e-04);
    ps = fma(z, ps, 8.33333333332248946124e-03);
    ps = fma(z, ps, -1.66666666666666324348e-01);
    double sn = fma(r * z, ps, r);
    double pc = fma(z, -1.13596475577881948265e-11, 2.08757232129817482790e-09);
    pc = fma(z, pc, -2.75573143513906633035e-07);
    pc = fma(z, pc, 2.48015872894767294178e-05);
    pc = fma(z, pc, -1.38888888888741095749e-03);
    pc = fma(z, pc, 4.16666666666666019037e-02);
    double cs = fma(z * z, pc, fma(-0.5, z, 1.0));
    double qm = q - 4.0 * floor(q * 0.25);
    if (qm == 0.0) {
        *s_out = sn; *c_out = cs;
    } else if (qm == 1.0) {
        *s_out = cs; *c_out = -sn;
    } else if (qm == 2.0) {
        *s_out = -sn; *c_out = -cs;
    } else if (qm == 3.0) {
        *s_out = -cs; *c_out = sn;
    } else { /* non-finite input */
        *s_out = x - x; *c_out = x - x;
    }
}

/* ------------------------------------------------------------------------- */
/* small growable int vector                                                 */
/* ------------------------------------------------------------------------- */
typedef struct {
    int32_t* a;
    int32_t n, cap;
} ivec;

static void iv_push(ivec* v, int32_t x) {
    if (v->n == v->cap) {
        v->cap = v->cap ? 2 * v->cap : 4;
        v->a = (int32_t*)realloc(v->a, (size_t)v->cap * sizeof(int32_t));
    }
    v->a[v->n++] = x;
}
static void iv_free(ivec* v) { free(v->a); v->a = NULL; v->n = v->cap = 0; }

static int cmp_i32(const void* a, const void* b) {
    int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
    return (x > y) - (x < y);
}
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return (x > y) - (x < y);
}

/* CRS pattern from (row, col) keys r*n_cols+c: sort, unique, diagonal added
 * for square shapes (sparse.hpp:146-181). */
static int crs_from_keys(int32_t n_rows, int32_t n_cols, int64_t* keys, int64_t nk,
                         int32_t** row_ptr_out, int32_t** col_ix_out, int32_t* nnz_out) {
    qsort(keys, (size_t)nk, sizeof(int64_t), cmp_i64);
    int64_t m = 0;
    for (int64_t i = 0; i < nk; ++i)
        if (m == 0 || keys[i] != keys[m - 1]) keys[m++] = keys[i];
    int32_t* rp = (int32_t*)calloc((size_t)n_rows + 1, sizeof(int32_t));
    int32_t* ci = (int32_t*)malloc((size_t)(m ? m : 1) * sizeof(int32_t));
    for (int64_t i = 0; i < m; ++i) {
        rp[keys[i] / n_cols + 1]++;
        ci[i] = (int32_t)(keys[i] % n_cols);
    }
    for (int32_t r = 0; r < n_rows; ++r) rp[r + 1] += rp[r];
    *row_ptr_out = rp;
    *col_ix_out = ci;
    *nnz_out = (int32_t)m;
    return 0;
}

static int32_t crs_find(const int32_t* rp, const int32_t* ci, int32_t r, int32_t c) {
    int32_t lo = rp[r], hi = rp[r + 1];
    while (lo < hi) {
        int32_t mid = (lo + hi) >> 1;
        if (ci[mid] < c) lo = mid + 1; else hi = mid;
    }
    return (lo < rp[r + 1] && ci[lo] == c) ? lo : -1;
}

/* ------------------------------------------------------------------------- */
/* Ybus (grid.hpp:195-243)                                                   */
/* ------------------------------------------------------------------------- */
int orc_build_ybus(int32_t n, int32_t nbr, const int32_t* f, const int32_t* t, const double* r,
                   const double* x, const double* b, const double* tap, const double* shift_deg,
                   const uint8_t* on, const double* gs, const double* bs, double base_mva,
                   int32_t* indptr, int32_t* indices, int32_t* diag, double* y_re, double* y_im,
                   int32_t* nnz_out) {
    int64_t nk = 2 * (int64_t)nbr + n;
    int64_t* keys = (int64_t*)malloc((size_t)nk * sizeof(int64_t));
    int64_t k = 0;
    for (int32_t br = 0; br < nbr; ++br) {
        if (f[br] < 0 || f[br] >= n || t[br] < 0 || t[br] >= n) {
            free(keys);
            return fail(2, "branch %d endpoint out of range", br);
        }
        keys[k++] = (int64_t)f[br] * n + t[br];
        keys[k++] = (int64_t)t[br] * n + f[br];
    }
    for (int32_t i = 0; i < n; ++i) keys[k++] = (int64_t)i * n + i;
    int32_t *rp, *ci, nnz;
    crs_from_keys(n, n, keys, nk, &rp, &ci, &nnz);
    free(keys);
    memcpy(indptr, rp, ((size_t)n + 1) * sizeof(int32_t));
    memcpy(indices, ci, (size_t)nnz * sizeof(int32_t));
    double complex* yv = (double complex*)calloc((size_t)nnz, sizeof(double complex));
    for (int32_t i = 0; i < n; ++i) diag[i] = crs_find(rp, ci, i, i);
    for (int32_t br = 0; br < nbr; ++br) {
        double complex ff = 0, ft = 0, tf = 0, tt = 0;
        if (on[br]) {
            double complex ys = 1.0 / CMPLX(r[br], x[br]);
            double complex ysh = CMPLX(0.0, b[br] / 2.0);
            double th = shift_deg[br] * 3.14159265358979323846 / 180.0;
            double complex tc = CMPLX(tap[br] * cos(th), tap[br] * sin(th));
            tt = ys + ysh;
            ff = (ys + ysh) / (tap[br] * tap[br]);
            ft = -ys / conj(tc);
            tf = -ys / tc;
        }
        int32_t sff = diag[f[br]], stt = diag[t[br]];
        int32_t sft = crs_find(rp, ci, f[br], t[br]), stf = crs_find(rp, ci, t[br], f[br]);
        yv[sff] += ff;
        yv[sft] += ft;
        yv[stf] += tf;
        yv[stt] += tt;
    }
    for (int32_t i = 0; i < n; ++i) yv[diag[i]] += CMPLX(gs[i], bs[i]) / base_mva;
    for (int32_t s = 0; s < nnz; ++s) {
        y_re[s] = creal(yv[s]);
        y_im[s] = cimag(yv[s]);
    }
    *nnz_out = nnz;
    free(yv);
    free(rp);
    free(ci);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* AMD (amd.hpp:29-157): quotient graph, approximate external degree,        */
/* no supervariables, min (degree, index) selection.                         */
/* ------------------------------------------------------------------------- */
typedef struct {
    int64_t* k;
    int64_t n, cap;
} heap64;

static void hp_push(heap64* h, int64_t key) {
    if (h->n == h->cap) {
        h->cap = h->cap ? 2 * h->cap : 64;
        h->k = (int64_t*)realloc(h->k, (size_t)h->cap * sizeof(int64_t));
    }
    int64_t i = h->n++;
    while (i > 0) {
        int64_t p = (i - 1) >> 1;
        if (h->k[p] <= key) break;
        h->k[i] = h->k[p];
        i = p;
    }
    h->k[i] = key;
}

static int64_t hp_pop(heap64* h) {
    int64_t top = h->k[0];
    int64_t last = h->k[--h->n];
    int64_t i = 0;
    for (;;) {
        int64_t c = 2 * i + 1;
        if (c >= h->n) break;
        if (c + 1 < h->n && h->k[c + 1] < h->k[c]) ++c;
        if (h->k[c] >= last) break;
        h->k[i] = h->k[c];
        i = c;
    }
    if (h->n > 0) h->k[i] = last;
    return top;
}

int orc_amd(int32_t n, const int32_t* col_ptr, const int32_t* row_ix, int32_t* fwd) {
    if (n == 0) return 0;
    ivec* nadj = (ivec*)calloc((size_t)n, sizeof(ivec));
    ivec* eadj = (ivec*)calloc((size_t)n, sizeof(ivec));
    ivec* bnd = (ivec*)calloc((size_t)n, sizeof(ivec));
    for (int32_t c = 0; c < n; ++c)
        for (int32_t p = col_ptr[c]; p < col_ptr[c + 1]; ++p) {
            int32_t r = row_ix[p];
            if (r == c) continue;
            iv_push(&nadj[c], r);
            iv_push(&nadj[r], c);
        }
    int32_t* degree = (int32_t*)malloc((size_t)n * sizeof(int32_t));
    uint8_t* elim = (uint8_t*)calloc((size_t)n, 1);
    uint8_t* is_el = (uint8_t*)calloc((size_t)n, 1);
    int32_t* stamp = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    int32_t* wlen = (int32_t*)calloc((size_t)n, sizeof(int32_t));
    heap64 h = {0};
    for (int32_t i = 0; i < n; ++i) {
        ivec* v = &nadj[i];
        qsort(v->a, (size_t)v->n, sizeof(int32_t), cmp_i32);
        int32_t m = 0;
        for (int32_t j = 0; j < v->n; ++j)
            if (m == 0 || v->a[j] != v->a[m - 1]) v->a[m++] = v->a[j];
        v->n = m;
        degree[i] = m;
        hp_push(&h, ((int64_t)m << 32) | i);
    }
    int32_t gen = 0;
    ivec lp = {0};
    for (int32_t k = 0; k < n; ++k) {
        int32_t p;
        for (;;) { /* lazy deletion: skip stale (degree, node) entries */
            int64_t key = hp_pop(&h);
            p = (int32_t)(key & 0xffffffff);
            if (!elim[p] && degree[p] == (int32_t)(key >> 32)) break;
        }
        elim[p] = 1;
        fwd[p] = k;
        ++gen;
        lp.n = 0;
        stamp[p] = gen;
        for (int32_t j = 0; j < nadj[p].n; ++j) {
            int32_t v = nadj[p].a[j];
            if (elim[v] || stamp[v] == gen) continue;
            stamp[v] = gen;
            iv_push(&lp, v);
        }
        for (int32_t j = 0; j < eadj[p].n; ++j) {
            int32_t e = eadj[p].a[j];
            if (!is_el[e]) continue;
            for (int32_t q = 0; q < bnd[e].n; ++q) {
                int32_t v = bnd[e].a[q];
                if (elim[v] || stamp[v] == gen) continue;
                stamp[v] = gen;
                iv_push(&lp, v);
            }
            is_el[e] = 0;
            bnd[e].n = 0;
        }
        qsort(lp.a, (size_t)lp.n, sizeof(int32_t), cmp_i32);
        /* sweep 1: wlen(e) = |Le \ Lp| */
        for (int32_t j = 0; j < lp.n; ++j) {
            int32_t i = lp.a[j];
            for (int32_t q = 0; q < eadj[i].n; ++q) {
                int32_t e = eadj[i].a[q];
                if (!is_el[e]) continue;
                if (stamp[e] != gen) {
                    stamp[e] = gen;
                    int32_t keep = 0;
                    for (int32_t z = 0; z < bnd[e].n; ++z)
                        if (!elim[bnd[e].a[z]]) bnd[e].a[keep++] = bnd[e].a[z];
                    bnd[e].n = keep;
                    wlen[e] = keep;
                }
                --wlen[e];
            }
        }
        /* sweep 2: prune, approximate degree update */
        int32_t alive_after = n - k - 1;
        int32_t lpm1 = lp.n - 1;
        for (int32_t j = 0; j < lp.n; ++j) {
            int32_t i = lp.a[j];
            ivec* ai = &nadj[i];
            int32_t keep = 0;
            for (int32_t q = 0; q < ai->n; ++q) {
                int32_t v = ai->a[q];
                if (v == p || elim[v] || stamp[v] == gen) continue;
                ai->a[keep++] = v;
            }
            ai->n = keep;
            ivec* ei = &eadj[i];
            int32_t esum = 0, ekeep = 0;
            for (int32_t q = 0; q < ei->n; ++q) {
                int32_t e = ei->a[q];
                if (!is_el[e]) continue;
                ei->a[ekeep++] = e;
                esum += wlen[e] > 0 ? wlen[e] : 0;
            }
            ei->n = ekeep;
            iv_push(ei, p);
            int32_t b_ext = ai->n + lpm1 + esum;
            int32_t b_grow = degree[i] + lpm1;
            int32_t d = alive_after;
            if (b_grow < d) d = b_grow;
            if (b_ext < d) d = b_ext;
            if (d < 0) d = 0;
            degree[i] = d;
            hp_push(&h, ((int64_t)d << 32) | i);
        }
        nadj[p].n = 0;
        eadj[p].n = 0;
        is_el[p] = 1;
        bnd[p].n = 0;
        for (int32_t j = 0; j < lp.n; ++j) iv_push(&bnd[p], lp.a[j]);
    }
    for (int32_t i = 0; i < n; ++i) {
        iv_free(&nadj[i]);
        iv_free(&eadj[i]);
        iv_free(&bnd[i]);
    }
    iv_free(&lp);
    free(nadj); free(eadj); free(bnd); free(degree); free(elim); free(is_el);
    free(stamp); free(wlen); free(h.k);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Plan: J pattern, ordering, symbolic + pivoting factorization, programs.   */
/* ------------------------------------------------------------------------- */
struct orc_plan {
    int32_t n, ref, npv, npq, npvpq, nJ, nnzY;
    int32_t *yp, *yi;      /* Ybus CRS */
    double *yre, *yim;     /* representative values (n_ysets == 1 default) */
    int32_t *jth, *jvm;    /* bus -> J index of theta / |V| unknown (-1 none) */
    int32_t* lk;           /* [4*nnzY] Ybus slot x {Pth,Pvm,Qth,Qvm} -> LU slot or -1 */
    int32_t *row_fwd, *col_fwd; /* J row/col -> A row/col */
    int32_t *cp, *ri, *dpos;    /* LU CCS (pivot numbering), diag slot per column */
    int32_t *dep_ptr, *dep_j, *dep_pos, *upd_ptr, *upd_dst; /* refactor program */
    int32_t *lev, levels_lu, levels_fs, levels_bs;
    int64_t nnzJ, nnzLU, nnzL, nnzU, D, offdiag_piv, max_col, max_udeps;
};

void orc_plan_destroy(orc_plan* p) {
    if (!p) return;
    free(p->yp); free(p->yi); free(p->yre); free(p->yim); free(p->jth); free(p->jvm);
    free(p->lk); free(p->row_fwd); free(p->col_fwd); free(p->cp); free(p->ri); free(p->dpos);
    free(p->dep_ptr); free(p->dep_j); free(p->dep_pos); free(p->upd_ptr); free(p->upd_dst);
    free(p->lev);
    free(p);
}

/* Jacobian rows of bus r for one task (SPEC.md:204-212 with the corrected
 * off-diagonal signs; MATPOWER dSbus_dV form).  Writes the
 * four quadrant values of every Ybus slot of row r into jv[4*slot + q]. */
static inline void mismatch_row(const orc_plan* P, const double* yre, const double* yim,
                                const double* vm, const double* c, const double* s, int32_t r,
                                double* ire_o, double* iim_o, double* P_o, double* Q_o) {
    double ire = 0.0, iim = 0.0;
    for (int32_t q = P->yp[r]; q < P->yp[r + 1]; ++q) {
        int32_t k = P->yi[q];
        double g = yre[q], b = yim[q];
        double vre = vm[k] * c[k], vim = vm[k] * s[k];
        ire = fma(g, vre, ire);
        ire = fma(-b, vim, ire);
        iim = fma(g, vim, iim);
        iim = fma(b, vre, iim);
    }
    double vre = vm[r] * c[r], vim = vm[r] * s[r];
    *ire_o = ire;
    *iim_o = iim;
    *P_o = fma(vre, ire, vim * iim);
    *Q_o = fma(vim, ire, -(vre * iim));
}

static inline void jac_entry(double g, double b, double vre_r, double vim_r, double ck, double sk,
                             double* zre, double* zim) {
    double yer = fma(g, ck, -(b * sk));
    double yei = fma(g, sk, b * ck);
    *zre = fma(vre_r, yer, vim_r * yei);
    *zim = fma(vim_r, yer, -(vre_r * yei));
}

static void jac_row(const orc_plan* P, const double* yre, const double* yim, const double* vm,
                    const double* c, const double* s, int32_t r, double* jv) {
    double ire, iim, Pc, Qc;
    mismatch_row(P, yre, yim, vm, c, s, r, &ire, &iim, &Pc, &Qc);
    double vre = vm[r] * c[r], vim = vm[r] * s[r];
    for (int32_t q = P->yp[r]; q < P->yp[r + 1]; ++q) {
        int32_t k = P->yi[q];
        double zre, zim;
        jac_entry(yre[q], yim[q], vre, vim, c[k], s[k], &zre, &zim);
        if (k != r) {
            jv[4 * q + 0] = vm[k] * zim;    /* dP/dth_k */
            jv[4 * q + 1] = zre;            /* dP/d|V_k| */
            jv[4 * q + 2] = -(vm[k] * zre); /* dQ/dth_k */
            jv[4 * q + 3] = zim;            /* dQ/d|V_k| */
        } else {
            jv[4 * q + 0] = fma(vm[r], zim, -Qc);
            jv[4 * q + 1] = zre + fma(ire, c[r], iim * s[r]);
            jv[4 * q + 2] = fma(-vm[r], zre, Pc);
            jv[4 * q + 3] = zim + fma(ire, s[r], -(iim * c[r]));
        }
    }
}

int orc_plan_create(int32_t n, const int32_t* yp, const int32_t* yi, const double* yre,
                    const double* yim, int32_t ref, const int32_t* pv, int32_t npv,
                    const int32_t* pq, int32_t npq, const double* vm0, const double* va0,
                    double pivot_tol, orc_plan** out) {
    *out = NULL;
    if (n <= 0 || ref < 0 || ref >= n) return fail(3, "bad n_bus/ref");
    orc_plan* P = (orc_plan*)calloc(1, sizeof(orc_plan));
    P->n = n; P->ref = ref; P->npv = npv; P->npq = npq;
    P->npvpq = npv + npq;
    P->nJ = npv + 2 * npq;
    P->nnzY = yp[n];
    const int32_t nJ = P->nJ, nY = P->nnzY;
    P->yp = (int32_t*)malloc(((size_t)n + 1) * 4); memcpy(P->yp, yp, ((size_t)n + 1) * 4);
    P->yi = (int32_t*)malloc((size_t)nY * 4); memcpy(P->yi, yi, (size_t)nY * 4);
    P->yre = (double*)malloc((size_t)nY * 8); memcpy(P->yre, yre, (size_t)nY * 8);
    P->yim = (double*)malloc((size_t)nY * 8); memcpy(P->yim, yim, (size_t)nY * 8);
    P->jth = (int32_t*)malloc((size_t)n * 4);
    P->jvm = (int32_t*)malloc((size_t)n * 4);
    for (int32_t i = 0; i < n; ++i) P->jth[i] = P->jvm[i] = -1;
    for (int32_t i = 0; i < npv; ++i) P->jth[pv[i]] = i;
    for (int32_t i = 0; i < npq; ++i) {
        P->jth[pq[i]] = npv + i;
        P->jvm[pq[i]] = P->npvpq + i;
    }
    int32_t seen = 0;
    for (int32_t i = 0; i < n; ++i) seen += (P->jth[i] >= 0) + (i == ref);
    if (seen != n || P->jth[ref] >= 0) {
        orc_plan_destroy(P);
        return fail(2, "pv/pq/ref do not partition the buses");
    }
    /* ---- reduced J pattern (CRS) + per-Ybus-slot quadrant map ---- */
    int64_t* keys = (int64_t*)malloc(((size_t)4 * nY + nJ + 1) * sizeof(int64_t));
    int64_t nk = 0;
    for (int32_t r = 0; r < n; ++r)
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            int32_t k = yi[q];
            int32_t rr[2] = {P->jth[r], P->jvm[r]}, cc[2] = {P->jth[k], P->jvm[k]};
            for (int a = 0; a < 2; ++a)
                for (int bq = 0; bq < 2; ++bq)
                    if (rr[a] >= 0 && cc[bq] >= 0) keys[nk++] = (int64_t)rr[a] * nJ + cc[bq];
        }
    for (int32_t i = 0; i < nJ; ++i) keys[nk++] = (int64_t)i * nJ + i;
    int32_t *jp, *ji, nnzJ;
    crs_from_keys(nJ, nJ, keys, nk, &jp, &ji, &nnzJ);
    free(keys);
    P->nnzJ = nnzJ;
    int32_t* jslot = (int32_t*)malloc((size_t)4 * nY * 4 + 4);
    for (int32_t r = 0; r < n; ++r)
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q) {
            int32_t k = yi[q];
            int32_t rr[2] = {P->jth[r], P->jvm[r]}, cc[2] = {P->jth[k], P->jvm[k]};
            for (int a = 0; a < 2; ++a)
                for (int bq = 0; bq < 2; ++bq)
                    jslot[4 * q + 2 * a + bq] =
                        (rr[a] >= 0 && cc[bq] >= 0) ? crs_find(jp, ji, rr[a], cc[bq]) : -1;
        }
    /* J CCS pattern (transpose), slot map crs->ccs */
    int32_t* jcp = (int32_t*)calloc((size_t)nJ + 1, 4);
    int32_t* jri = (int32_t*)malloc((size_t)nnzJ * 4 + 4);
    int32_t* j2c = (int32_t*)malloc((size_t)nnzJ * 4 + 4);
    for (int32_t s = 0; s < nnzJ; ++s) jcp[ji[s] + 1]++;
    for (int32_t c = 0; c < nJ; ++c) jcp[c + 1] += jcp[c];
    {
        int32_t* nx = (int32_t*)malloc((size_t)nJ * 4 + 4);
        memcpy(nx, jcp, (size_t)nJ * 4);
        for (int32_t r = 0; r < nJ; ++r)
            for (int32_t s = jp[r]; s < jp[r + 1]; ++s) {
                int32_t slot = nx[ji[s]]++;
                jri[slot] = r;
                j2c[s] = slot;
            }
        free(nx);
    }
    /* ---- fill-reducing ordering on the J pattern ---- */
    int32_t* amd_fwd = (int32_t*)malloc((size_t)nJ * 4 + 4);
    orc_amd(nJ, jcp, jri, amd_fwd);
    int32_t* amd_inv = (int32_t*)malloc((size_t)nJ * 4 + 4);
    for (int32_t i = 0; i < nJ; ++i) amd_inv[amd_fwd[i]] = i;
    /* ---- representative J values (task 0 at V0) in CCS ---- */
    double* c0 = (double*)malloc((size_t)n * 8);
    double* s0 = (double*)malloc((size_t)n * 8);
    for (int32_t i = 0; i < n; ++i) orc_sincos(va0[i], &s0[i], &c0[i]);
    double* jv4 = (double*)calloc((size_t)4 * nY + 4, 8);
    for (int32_t r = 0; r < n; ++r)
        if (r != ref) jac_row(P, yre, yim, vm0, c0, s0, r, jv4);
    double* jval = (double*)calloc((size_t)nnzJ + 1, 8); /* CCS order */
    for (int32_t q = 0; q < 4 * nY; ++q)
        if (jslot[q] >= 0) jval[j2c[jslot[q]]] = jv4[q];
    free(jv4); free(c0); free(s0);
    /* ---- left-looking G-P with threshold partial pivoting ---- */
    int32_t* pinv = (int32_t*)malloc((size_t)nJ * 4 + 4);
    for (int32_t i = 0; i < nJ; ++i) pinv[i] = -1;
    ivec* Lrows = (ivec*)calloc((size_t)nJ, sizeof(ivec));   /* J-row ids, strictly lower */
    double** Lval = (double**)calloc((size_t)nJ, sizeof(double*));
    ivec* Urows = (ivec*)calloc((size_t)nJ, sizeof(ivec));   /* J-row ids of U part */
    double* x = (double*)calloc((size_t)nJ, 8);
    int32_t* mark = (int32_t*)malloc((size_t)nJ * 4 + 4);
    for (int32_t i = 0; i < nJ; ++i) mark[i] = -1;
    int32_t* reach = (int32_t*)malloc((size_t)nJ * 4 + 4);
    int64_t* piv_keys = (int64_t*)malloc((size_t)nJ * 8 + 8);
    int32_t rc = 0;
    P->offdiag_piv = 0;
    for (int32_t k = 0; k < nJ && rc == 0; ++k) {
        int32_t col = amd_inv[k];
        int32_t nr = 0;
        for (int32_t q = jcp[col]; q < jcp[col + 1]; ++q) {
            int32_t i = jri[q];
            if (mark[i] != k) { mark[i] = k; reach[nr++] = i; }
        }
        for (int32_t h = 0; h < nr; ++h) { /* closure through pivoted L columns */
            int32_t i = reach[h];
            if (pinv[i] < 0) continue;
            ivec* L = &Lrows[pinv[i]];
            for (int32_t z = 0; z < L->n; ++z)
                if (mark[L->a[z]] != k) { mark[L->a[z]] = k; reach[nr++] = L->a[z]; }
        }
        for (int32_t h = 0; h < nr; ++h) x[reach[h]] = 0.0;
        for (int32_t q = jcp[col]; q < jcp[col + 1]; ++q) x[jri[q]] = jval[q];
        int32_t npiv = 0;
        for (int32_t h = 0; h < nr; ++h)
            if (pinv[reach[h]] >= 0) piv_keys[npiv++] = ((int64_t)pinv[reach[h]] << 32) | reach[h];
        qsort(piv_keys, (size_t)npiv, 8, cmp_i64);
        for (int32_t h = 0; h < npiv; ++h) {
            int32_t j = (int32_t)(piv_keys[h] >> 32), row = (int32_t)(piv_keys[h] & 0xffffffff);
            double xj = x[row];
            for (int32_t z = 0; z < Lrows[j].n; ++z)
                x[Lrows[j].a[z]] = fma(-xj, Lval[j][z], x[Lrows[j].a[z]]);
            iv_push(&Urows[k], row);
        }
        int32_t ipiv = -1;
        double amax = -1.0;
        for (int32_t h = 0; h < nr; ++h) {
            int32_t i = reach[h];
            if (pinv[i] >= 0) continue;
            double a = fabs(x[i]);
            if (a > amax || (a == amax && ipiv >= 0 && i < ipiv)) { amax = a; ipiv = i; }
        }
        if (ipiv < 0) { rc = fail(2, "structurally singular column %d", k); break; }
        if (!(amax > 0.0)) { rc = fail(4, "numerically singular pivot in column %d", k); break; }
        int32_t idiag = amd_inv[k]; /* J row with the symmetric position k */
        if (pinv[idiag] < 0 && mark[idiag] == k && fabs(x[idiag]) >= pivot_tol * amax) ipiv = idiag;
        if (ipiv != idiag) P->offdiag_piv++;
        double piv = x[ipiv];
        pinv[ipiv] = k;
        int32_t nl = 0;
        for (int32_t h = 0; h < nr; ++h)
            if (pinv[reach[h]] < 0) nl++;
        Lval[k] = (double*)malloc((size_t)(nl ? nl : 1) * 8);
        for (int32_t h = 0; h < nr; ++h) {
            int32_t i = reach[h];
            if (pinv[i] >= 0) continue;
            iv_push(&Lrows[k], i);
            Lval[k][Lrows[k].n - 1] = x[i] / piv;
        }
    }
    free(x); free(mark); free(reach); free(piv_keys); free(jval); free(amd_inv);
    if (rc != 0) {
        for (int32_t i = 0; i < nJ; ++i) { iv_free(&Lrows[i]); iv_free(&Urows[i]); free(Lval[i]); }
        free(Lrows); free(Urows); free(Lval); free(pinv); free(jp); free(ji); free(jslot);
        free(jcp); free(jri); free(j2c); free(amd_fwd);
        orc_plan_destroy(P);
        return rc;
    }
    /* ---- frozen LU pattern in pivot numbering ---- */
    P->row_fwd = pinv;
    P->col_fwd = amd_fwd;
    P->cp = (int32_t*)calloc((size_t)nJ + 1, 4);
    for (int32_t k = 0; k < nJ; ++k) P->cp[k + 1] = P->cp[k] + Urows[k].n + 1 + Lrows[k].n;
    P->nnzLU = P->cp[nJ];
    P->ri = (int32_t*)malloc((size_t)P->nnzLU * 4 + 4);
    P->dpos = (int32_t*)malloc((size_t)nJ * 4 + 4);
    P->nnzL = P->nnzU = 0;
    P->max_col = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        int32_t* dst = P->ri + P->cp[k];
        int32_t m = 0;
        for (int32_t z = 0; z < Urows[k].n; ++z) dst[m++] = pinv[Urows[k].a[z]];
        dst[m++] = k;
        for (int32_t z = 0; z < Lrows[k].n; ++z) dst[m++] = pinv[Lrows[k].a[z]];
        qsort(dst, (size_t)m, 4, cmp_i32);
        for (int32_t z = 0; z < m; ++z)
            if (dst[z] == k) P->dpos[k] = P->cp[k] + z;
        P->nnzU += Urows[k].n;
        P->nnzL += Lrows[k].n;
        if (m > P->max_col) P->max_col = m;
    }
    for (int32_t i = 0; i < nJ; ++i) { iv_free(&Lrows[i]); iv_free(&Urows[i]); free(Lval[i]); }
    free(Lrows); free(Urows); free(Lval);
    /* ---- scatter lookup: Ybus slot quadrant -> LU slot (sparse.hpp:237-267 shape) ---- */
    P->lk = (int32_t*)malloc((size_t)4 * nY * 4 + 4);
    for (int32_t r = 0; r < n; ++r)
        for (int32_t q = yp[r]; q < yp[r + 1]; ++q)
            for (int a = 0; a < 4; ++a) {
                int32_t js = jslot[4 * q + a];
                if (js < 0) { P->lk[4 * q + a] = -1; continue; }
                int32_t jr = (a < 2) ? P->jth[r] : P->jvm[r];
                int32_t jc = (a & 1) ? P->jvm[yi[q]] : P->jth[yi[q]];
                int32_t ar = P->row_fwd[jr], ac = P->col_fwd[jc];
                int32_t lo = P->cp[ac], hi = P->cp[ac + 1], hit = -1;
                for (int32_t z = lo; z < hi; ++z)
                    if (P->ri[z] == ar) { hit = z; break; }
                P->lk[4 * q + a] = hit;
            }
    free(jp); free(ji); free(jslot); free(jcp); free(jri); free(j2c);
    /* ---- refactor program: per column, U deps ascending with L destinations ---- */
    int32_t* posmap = (int32_t*)malloc((size_t)nJ * 4 + 4);
    for (int32_t i = 0; i < nJ; ++i) posmap[i] = -1;
    P->dep_ptr = (int32_t*)calloc((size_t)nJ + 1, 4);
    for (int32_t k = 0; k < nJ; ++k) P->dep_ptr[k + 1] = P->dep_ptr[k] + (P->dpos[k] - P->cp[k]);
    int32_t ndep = P->dep_ptr[nJ];
    P->dep_j = (int32_t*)malloc((size_t)ndep * 4 + 4);
    P->dep_pos = (int32_t*)malloc((size_t)ndep * 4 + 4);
    P->upd_ptr = (int32_t*)calloc((size_t)ndep + 1, 4);
    P->D = 0;
    P->max_udeps = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        int32_t d0 = P->dep_ptr[k];
        for (int32_t z = P->cp[k]; z < P->dpos[k]; ++z) {
            int32_t j = P->ri[z];
            P->dep_j[d0 + z - P->cp[k]] = j;
            P->dep_pos[d0 + z - P->cp[k]] = z - P->cp[k];
            P->D += P->cp[j + 1] - P->dpos[j] - 1;
        }
        if (P->dpos[k] - P->cp[k] > P->max_udeps) P->max_udeps = P->dpos[k] - P->cp[k];
    }
    P->upd_dst = (int32_t*)malloc((size_t)P->D * 4 + 4);
    int64_t u = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        for (int32_t z = P->cp[k]; z < P->cp[k + 1]; ++z) posmap[P->ri[z]] = z - P->cp[k];
        for (int32_t d = P->dep_ptr[k]; d < P->dep_ptr[k + 1]; ++d) {
            int32_t j = P->dep_j[d];
            P->upd_ptr[d] = (int32_t)u;
            for (int32_t z = P->dpos[j] + 1; z < P->cp[j + 1]; ++z) {
                int32_t dst = posmap[P->ri[z]];
                if (dst < 0) { rc = fail(2, "frozen pattern not closed (col %d dep %d)", k, j); }
                P->upd_dst[u++] = dst;
            }
        }
        for (int32_t z = P->cp[k]; z < P->cp[k + 1]; ++z) posmap[P->ri[z]] = -1;
    }
    P->upd_ptr[ndep] = (int32_t)u;
    free(posmap);
    if (rc != 0) { orc_plan_destroy(P); return rc; }
    /* ---- level schedules ---- */
    P->lev = (int32_t*)calloc((size_t)nJ + 1, 4);
    int32_t* fl = (int32_t*)calloc((size_t)nJ + 1, 4);
    int32_t* bl = (int32_t*)calloc((size_t)nJ + 1, 4);
    P->levels_lu = P->levels_fs = P->levels_bs = 0;
    for (int32_t k = 0; k < nJ; ++k) {
        int32_t l = 0;
        for (int32_t z = P->cp[k]; z < P->dpos[k]; ++z)
            if (P->lev[P->ri[z]] + 1 > l) l = P->lev[P->ri[z]] + 1;
        P->lev[k] = l;
        if (l + 1 > P->levels_lu) P->levels_lu = l + 1;
        /* FS: rows of L(:,k) depend on k */
        if (fl[k] + 1 > P->levels_fs) P->levels_fs = fl[k] + 1;
        for (int32_t z = P->dpos[k] + 1; z < P->cp[k + 1]; ++z)
            if (fl[k] + 1 > fl[P->ri[z]]) fl[P->ri[z]] = fl[k] + 1;
    }
    for (int32_t k = nJ - 1; k >= 0; --k) {
        if (bl[k] + 1 > P->levels_bs) P->levels_bs = bl[k] + 1;
        for (int32_t z = P->cp[k]; z < P->dpos[k]; ++z)
            if (bl[k] + 1 > bl[P->ri[z]]) bl[P->ri[z]] = bl[k] + 1;
    }
    free(fl); free(bl);
    *out = P;
    return 0;
}

int orc_plan_stats(const orc_plan* P, int64_t* o) {
    memset(o, 0, 16 * sizeof(int64_t));
    o[0] = P->nJ; o[1] = P->nnzJ; o[2] = P->nnzLU; o[3] = P->nnzL; o[4] = P->nnzU; o[5] = P->D;
    o[6] = 2 * P->D + P->nnzL; o[7] = P->levels_lu; o[8] = P->levels_fs; o[9] = P->levels_bs;
    o[10] = P->offdiag_piv; o[11] = P->npvpq; o[12] = P->nnzLU - P->nnzJ; o[13] = P->max_col;
    o[14] = P->max_udeps;
    return 0;
}

int orc_plan_export(const orc_plan* P, int32_t* row_fwd, int32_t* col_fwd, int32_t* col_ptr,
                    int32_t* row_ix, int32_t* level) {
    if (row_fwd) memcpy(row_fwd, P->row_fwd, (size_t)P->nJ * 4);
    if (col_fwd) memcpy(col_fwd, P->col_fwd, (size_t)P->nJ * 4);
    if (col_ptr) memcpy(col_ptr, P->cp, ((size_t)P->nJ + 1) * 4);
    if (row_ix) memcpy(row_ix, P->ri, (size_t)P->nnzLU * 4);
    if (level) memcpy(level, P->lev, (size_t)P->nJ * 4);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Batched numeric kernels on one mini-batch (element-major, MB lanes).      */
/* ------------------------------------------------------------------------- */
typedef struct {
    double *vm, *va, *c, *s; /* [n][MB] */
    double* lu;              /* [nnzLU][MB] */
    double* b;               /* [nJ][MB] */
    double *yre, *yim;       /* [nnzY][MB] when per-task Ybus */
    double *p0, *q0;         /* [n][MB] */
} mb_work;

/* NPM for all lanes into b (permuted rows); returns per-lane
 * max-norm in nrm (NaN counted as +inf). */
static void mb_npm(const orc_plan* P, mb_work* w, int per_task_y, double* nrm) {
    const int32_t n = P->n;
    for (int l = 0; l < MB; ++l) nrm[l] = 0.0;
    for (int32_t r = 0; r < n; ++r) {
        if (r == P->ref) continue;
        double ire[MB], iim[MB];
        for (int l = 0; l < MB; ++l) ire[l] = iim[l] = 0.0;
        for (int32_t q = P->yp[r]; q < P->yp[r + 1]; ++q) {
            int32_t k = P->yi[q];
            const double* vmk = w->vm + (size_t)k * MB;
            const double* ck = w->c + (size_t)k * MB;
            const double* sk = w->s + (size_t)k * MB;
            for (int l = 0; l < MB; ++l) {
                double g = per_task_y ? w->yre[(size_t)q * MB + l] : P->yre[q];
                double b = per_task_y ? w->yim[(size_t)q * MB + l] : P->yim[q];
                double vre = vmk[l] * ck[l], vim = vmk[l] * sk[l];
                ire[l] = fma(g, vre, ire[l]);
                ire[l] = fma(-b, vim, ire[l]);
                iim[l] = fma(g, vim, iim[l]);
                iim[l] = fma(b, vre, iim[l]);
            }
        }
        const double* vmr = w->vm + (size_t)r * MB;
        const double* cr = w->c + (size_t)r * MB;
        const double* sr = w->s + (size_t)r * MB;
        double* bp = w->b + (size_t)P->row_fwd[P->jth[r]] * MB;
        double* bq = P->jvm[r] >= 0 ? w->b + (size_t)P->row_fwd[P->jvm[r]] * MB : NULL;
        for (int l = 0; l < MB; ++l) {
            double vre = vmr[l] * cr[l], vim = vmr[l] * sr[l];
            double Pc = fma(vre, ire[l], vim * iim[l]);
            double fp = Pc - w->p0[(size_t)r * MB + l];
            bp[l] = fp;
            double a = fabs(fp);
            if (isnan(a)) a = INFINITY;
            nrm[l] = fmax(nrm[l], a);
            if (bq) {
                double Qc = fma(vim, ire[l], -(vre * iim[l]));
                double fq = Qc - w->q0[(size_t)r * MB + l];
                bq[l] = fq;
                double aq = fabs(fq);
                if (isnan(aq)) aq = INFINITY;
                nrm[l] = fmax(nrm[l], aq);
            }
        }
    }
}

/* Jacobian scattered straight into the LU tape (fill slots zero). */
static void mb_jacobian(const orc_plan* P, mb_work* w, int per_task_y) {
    memset(w->lu, 0, (size_t)P->nnzLU * MB * sizeof(double));
    for (int32_t r = 0; r < P->n; ++r) {
        if (r == P->ref) continue;
        double ire[MB], iim[MB], Pc[MB], Qc[MB], vre[MB], vim[MB];
        for (int l = 0; l < MB; ++l) ire[l] = iim[l] = 0.0;
        for (int32_t q = P->yp[r]; q < P->yp[r + 1]; ++q) {
            int32_t k = P->yi[q];
            for (int l = 0; l < MB; ++l) {
                double g = per_task_y ? w->yre[(size_t)q * MB + l] : P->yre[q];
                double b = per_task_y ? w->yim[(size_t)q * MB + l] : P->yim[q];
                double vr = w->vm[(size_t)k * MB + l] * w->c[(size_t)k * MB + l];
                double vi = w->vm[(size_t)k * MB + l] * w->s[(size_t)k * MB + l];
                ire[l] = fma(g, vr, ire[l]);
                ire[l] = fma(-b, vi, ire[l]);
                iim[l] = fma(g, vi, iim[l]);
                iim[l] = fma(b, vr, iim[l]);
            }
        }
        for (int l = 0; l < MB; ++l) {
            vre[l] = w->vm[(size_t)r * MB + l] * w->c[(size_t)r * MB + l];
            vim[l] = w->vm[(size_t)r * MB + l] * w->s[(size_t)r * MB + l];
            Pc[l] = fma(vre[l], ire[l], vim[l] * iim[l]);
            Qc[l] = fma(vim[l], ire[l], -(vre[l] * iim[l]));
        }
        for (int32_t q = P->yp[r]; q < P->yp[r + 1]; ++q) {
            int32_t k = P->yi[q];
            const int32_t* lk = P->lk + 4 * (size_t)q;
            for (int l = 0; l < MB; ++l) {
                double g = per_task_y ? w->yre[(size_t)q * MB + l] : P->yre[q];
                double b = per_task_y ? w->yim[(size_t)q * MB + l] : P->yim[q];
                double ck = w->c[(size_t)k * MB + l], sk = w->s[(size_t)k * MB + l];
                double vmk = w->vm[(size_t)k * MB + l];
                double zre, zim, j0, j1, j2, j3;
                jac_entry(g, b, vre[l], vim[l], ck, sk, &zre, &zim);
                if (k != r) {
                    j0 = vmk * zim;
                    j1 = zre;
                    j2 = -(vmk * zre);
                    j3 = zim;
                } else {
                    j0 = fma(vmk, zim, -Qc[l]);
                    j1 = zre + fma(ire[l], ck, iim[l] * sk);
                    j2 = fma(-vmk, zre, Pc[l]);
                    j3 = zim + fma(ire[l], sk, -(iim[l] * ck));
                }
                if (lk[0] >= 0) w->lu[(size_t)lk[0] * MB + l] = j0;
                if (lk[1] >= 0) w->lu[(size_t)lk[1] * MB + l] = j1;
                if (lk[2] >= 0) w->lu[(size_t)lk[2] * MB + l] = j2;
                if (lk[3] >= 0) w->lu[(size_t)lk[3] * MB + l] = j3;
            }
        }
    }
}

/* Alg. 2 on the frozen pattern, in place; flags lanes whose
 * pivot is tiny relative to the column. */
static void mb_refactor(const orc_plan* P, double* lu, double singular_tol, uint8_t* flag) {
    for (int32_t k = 0; k < P->nJ; ++k) {
        double* col = lu + (size_t)P->cp[k] * MB;
        for (int32_t d = P->dep_ptr[k]; d < P->dep_ptr[k + 1]; ++d) {
            int32_t j = P->dep_j[d];
            double xj[MB];
            for (int l = 0; l < MB; ++l) xj[l] = col[(size_t)P->dep_pos[d] * MB + l];
            const double* Lj = lu + ((size_t)P->dpos[j] + 1) * MB;
            const int32_t* dst = P->upd_dst + P->upd_ptr[d];
            int32_t cnt = P->upd_ptr[d + 1] - P->upd_ptr[d];
            for (int32_t z = 0; z < cnt; ++z) {
                double* xi = col + (size_t)dst[z] * MB;
                const double* lz = Lj + (size_t)z * MB;
                for (int l = 0; l < MB; ++l) xi[l] = fma(-xj[l], lz[l], xi[l]);
            }
        }
        int32_t len = P->cp[k + 1] - P->cp[k], dp = P->dpos[k] - P->cp[k];
        double cmax[MB];
        for (int l = 0; l < MB; ++l) cmax[l] = 0.0;
        for (int32_t z = 0; z < len; ++z)
            for (int l = 0; l < MB; ++l) cmax[l] = fmax(cmax[l], fabs(col[(size_t)z * MB + l]));
        double inv[MB];
        for (int l = 0; l < MB; ++l) {
            double piv = col[(size_t)dp * MB + l];
            if (isfinite(cmax[l]) && (piv == 0.0 || fabs(piv) < singular_tol * cmax[l])) flag[l] = 1;
            inv[l] = 1.0 / piv;
        }
        for (int32_t z = dp + 1; z < len; ++z)
            for (int l = 0; l < MB; ++l) col[(size_t)z * MB + l] *= inv[l];
    }
}

/* FS with unit L then BS with U, in place on b. */
static void mb_fsbs(const orc_plan* P, const double* lu, double* b) {
    const int32_t nJ = P->nJ;
    for (int32_t k = 0; k < nJ; ++k) {
        const double* bk = b + (size_t)k * MB;
        for (int32_t z = P->dpos[k] + 1; z < P->cp[k + 1]; ++z) {
            double* bi = b + (size_t)P->ri[z] * MB;
            const double* lz = lu + (size_t)z * MB;
            for (int l = 0; l < MB; ++l) bi[l] = fma(-lz[l], bk[l], bi[l]);
        }
    }
    for (int32_t k = nJ - 1; k >= 0; --k) {
        double* bk = b + (size_t)k * MB;
        const double* uk = lu + (size_t)P->dpos[k] * MB;
        for (int l = 0; l < MB; ++l) bk[l] = bk[l] / uk[l];
        for (int32_t z = P->cp[k]; z < P->dpos[k]; ++z) {
            double* bi = b + (size_t)P->ri[z] * MB;
            const double* uz = lu + (size_t)z * MB;
            for (int l = 0; l < MB; ++l) bi[l] = fma(-uz[l], bk[l], bi[l]);
        }
    }
}

/* V update for active lanes; recompute the unit phasor. */
static void mb_update(const orc_plan* P, mb_work* w, const uint8_t* active) {
    for (int32_t r = 0; r < P->n; ++r) {
        int32_t jt = P->jth[r], jv = P->jvm[r];
        if (jt < 0) continue;
        const double* dt = w->b + (size_t)P->col_fwd[jt] * MB;
        const double* dv = jv >= 0 ? w->b + (size_t)P->col_fwd[jv] * MB : NULL;
        for (int l = 0; l < MB; ++l) {
            if (!active[l]) continue;
            size_t o = (size_t)r * MB + l;
            w->va[o] = w->va[o] - dt[l];
            if (dv) w->vm[o] = w->vm[o] - dv[l];
            orc_sincos(w->va[o], &w->s[o], &w->c[o]);
        }
    }
}

typedef struct {
    const orc_plan* P;
    int32_t n_tasks, n_ysets, n_ssets, n_vsets, max_iter;
    const double *y_re, *y_im, *p0, *q0, *vm0, *va0;
    double tol, singular_tol;
    double *vm_out, *va_out, *max_mis;
    int32_t *iters, *status;
    uint8_t* conv;
    /* refactor-only mode */
    int refactor_only;
    const double *vm_in, *va_in;
    double* lu_out;
    uint8_t* flags_out;
    _Atomic int32_t next;
} solve_job;

static void* solve_worker(void* arg) {
    solve_job* J = (solve_job*)arg;
    const orc_plan* P = J->P;
    const int32_t n = P->n, nY = P->nnzY;
    mb_work w;
    w.vm = (double*)malloc((size_t)n * MB * 8);
    w.va = (double*)malloc((size_t)n * MB * 8);
    w.c = (double*)malloc((size_t)n * MB * 8);
    w.s = (double*)malloc((size_t)n * MB * 8);
    w.p0 = (double*)calloc((size_t)n * MB, 8);
    w.q0 = (double*)calloc((size_t)n * MB, 8);
    w.lu = (double*)malloc((size_t)P->nnzLU * MB * 8);
    w.b = (double*)malloc((size_t)P->nJ * MB * 8 + 8);
    int per_task_y = J->n_ysets > 1;
    w.yre = per_task_y ? (double*)malloc((size_t)nY * MB * 8) : NULL;
    w.yim = per_task_y ? (double*)malloc((size_t)nY * MB * 8) : NULL;
    for (;;) {
        int32_t t0 = atomic_fetch_add(&J->next, MB);
        if (t0 >= J->n_tasks) break;
        int32_t width = J->n_tasks - t0 < MB ? J->n_tasks - t0 : MB;
        /* load lanes; padding lanes replicate the last task and stay inactive */
        for (int l = 0; l < MB; ++l) {
            int32_t t = t0 + (l < width ? l : width - 1);
            for (int32_t i = 0; i < n; ++i) {
                size_t o = (size_t)i * MB + l;
                if (J->refactor_only) {
                    w.vm[o] = J->vm_in[(size_t)i * J->n_tasks + t];
                    w.va[o] = J->va_in[(size_t)i * J->n_tasks + t];
                } else {
                    int32_t tv = J->n_vsets > 1 ? t : 0, ts = J->n_ssets > 1 ? t : 0;
                    w.vm[o] = J->vm0[(size_t)i * J->n_vsets + tv];
                    w.va[o] = J->va0[(size_t)i * J->n_vsets + tv];
                    w.p0[o] = J->p0[(size_t)i * J->n_ssets + ts];
                    w.q0[o] = J->q0[(size_t)i * J->n_ssets + ts];
                }
                orc_sincos(w.va[o], &w.s[o], &w.c[o]);
            }
            if (per_task_y)
                for (int32_t q = 0; q < nY; ++q) {
                    w.yre[(size_t)q * MB + l] = J->y_re[(size_t)q * J->n_ysets + t];
                    w.yim[(size_t)q * MB + l] = J->y_im[(size_t)q * J->n_ysets + t];
                }
        }
        if (J->refactor_only) {
            uint8_t flag[MB] = {0};
            mb_jacobian(P, &w, per_task_y);
            mb_refactor(P, w.lu, J->singular_tol, flag);
            for (int l = 0; l < width; ++l) {
                for (int64_t z = 0; z < P->nnzLU; ++z)
                    J->lu_out[(size_t)z * J->n_tasks + t0 + l] = w.lu[(size_t)z * MB + l];
                J->flags_out[t0 + l] = flag[l];
            }
            continue;
        }
        uint8_t active[MB], conv[MB] = {0};
        int32_t it_out[MB], st[MB];
        double nrm[MB], last[MB];
        for (int l = 0; l < MB; ++l) { active[l] = l < width; it_out[l] = 0; st[l] = 1; }
        mb_npm(P, &w, per_task_y, nrm);
        int any = 0;
        for (int l = 0; l < MB; ++l) {
            last[l] = nrm[l];
            if (active[l] && nrm[l] < J->tol) { active[l] = 0; conv[l] = 1; st[l] = 0; it_out[l] = 0; }
            any |= active[l];
        }
        for (int32_t it = 1; it <= J->max_iter && any; ++it) {
            uint8_t flag[MB] = {0};
            mb_jacobian(P, &w, per_task_y);
            mb_refactor(P, w.lu, J->singular_tol, flag);
            for (int l = 0; l < MB; ++l)
                if (active[l] && flag[l]) { active[l] = 0; st[l] = 2; it_out[l] = it; }
            mb_fsbs(P, w.lu, w.b);
            mb_update(P, &w, active);
            mb_npm(P, &w, per_task_y, nrm);
            any = 0;
            for (int l = 0; l < MB; ++l) {
                if (!active[l]) continue;
                last[l] = nrm[l];
                if (nrm[l] < J->tol) { active[l] = 0; conv[l] = 1; st[l] = 0; it_out[l] = it; }
                else if (it == J->max_iter) { active[l] = 0; st[l] = 1; it_out[l] = it; }
                any |= active[l];
            }
        }
        for (int l = 0; l < width; ++l) {
            int32_t t = t0 + l;
            for (int32_t i = 0; i < n; ++i) {
                J->vm_out[(size_t)i * J->n_tasks + t] = w.vm[(size_t)i * MB + l];
                J->va_out[(size_t)i * J->n_tasks + t] = w.va[(size_t)i * MB + l];
            }
            J->iters[t] = it_out[l];
            J->conv[t] = conv[l];
            J->status[t] = st[l];
            J->max_mis[t] = last[l];
        }
    }
    free(w.vm); free(w.va); free(w.c); free(w.s); free(w.p0); free(w.q0); free(w.lu); free(w.b);
    free(w.yre); free(w.yim);
    return NULL;
}

static void run_pool(solve_job* J, int32_t n_threads) {
    if (n_threads < 1) n_threads = 1;
    int32_t nmb = (J->n_tasks + MB - 1) / MB;
    if (n_threads > nmb) n_threads = nmb;
    atomic_store(&J->next, 0);
    pthread_t* th = (pthread_t*)malloc((size_t)n_threads * sizeof(pthread_t));
    for (int32_t i = 1; i < n_threads; ++i) pthread_create(&th[i], NULL, solve_worker, J);
    solve_worker(J);
    for (int32_t i = 1; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
}

int orc_solve(const orc_plan* P, int32_t n_tasks, const double* y_re, const double* y_im,
              int32_t n_ysets, const double* p0, const double* q0, int32_t n_ssets,
              const double* vm0, const double* va0, int32_t n_vsets, double tol, int32_t max_iter,
              double singular_tol, double* vm_out, double* va_out, int32_t* iterations,
              uint8_t* converged, int32_t* status, double* max_mismatch, int32_t n_threads) {
    if (n_tasks < 0) return fail(3, "n_tasks < 0");
    if ((n_ysets != 1 && n_ysets != n_tasks) || (n_ssets != 1 && n_ssets != n_tasks) ||
        (n_vsets != 1 && n_vsets != n_tasks))
        return fail(3, "set counts must be 1 or n_tasks");
    if (!(tol > 0.0) || max_iter < 1) return fail(3, "tol > 0 and max_iter >= 1 required");
    if (n_tasks == 0) return 0;
    solve_job J;
    memset(&J, 0, sizeof J);
    J.P = P; J.n_tasks = n_tasks; J.n_ysets = n_ysets; J.n_ssets = n_ssets; J.n_vsets = n_vsets;
    J.max_iter = max_iter; J.y_re = y_re; J.y_im = y_im; J.p0 = p0; J.q0 = q0;
    J.vm0 = vm0; J.va0 = va0; J.tol = tol; J.singular_tol = singular_tol;
    J.vm_out = vm_out; J.va_out = va_out; J.max_mis = max_mismatch; J.iters = iterations;
    J.status = status; J.conv = converged;
    run_pool(&J, n_threads);
    return 0;
}

int orc_refactor(const orc_plan* P, int32_t n_tasks, const double* vm, const double* va,
                 double singular_tol, double* lu_out, uint8_t* flags, int32_t n_threads) {
    if (n_tasks <= 0) return 0;
    solve_job J;
    memset(&J, 0, sizeof J);
    J.P = P; J.n_tasks = n_tasks; J.n_ysets = 1; J.singular_tol = singular_tol;
    J.refactor_only = 1; J.vm_in = vm; J.va_in = va; J.lu_out = lu_out; J.flags_out = flags;
    run_pool(&J, n_threads);
    return 0;
}

int orc_mismatch(const orc_plan* P, int32_t n_tasks, const double* p0, const double* q0,
                 const double* vm, const double* va, double* f_out) {
    const int32_t n = P->n;
    double* c = (double*)malloc((size_t)n * 8);
    double* s = (double*)malloc((size_t)n * 8);
    double* vmt = (double*)malloc((size_t)n * 8);
    for (int32_t t = 0; t < n_tasks; ++t) {
        for (int32_t i = 0; i < n; ++i) {
            vmt[i] = vm[(size_t)i * n_tasks + t];
            orc_sincos(va[(size_t)i * n_tasks + t], &s[i], &c[i]);
        }
        for (int32_t r = 0; r < n; ++r) {
            if (r == P->ref) continue;
            double ire, iim, Pc, Qc;
            mismatch_row(P, P->yre, P->yim, vmt, c, s, r, &ire, &iim, &Pc, &Qc);
            f_out[(size_t)P->jth[r] * n_tasks + t] = Pc - p0[(size_t)r * n_tasks + t];
            if (P->jvm[r] >= 0) f_out[(size_t)P->jvm[r] * n_tasks + t] = Qc - q0[(size_t)r * n_tasks + t];
        }
    }
    free(c); free(s); free(vmt);
    return 0;
}

/* calc_branch_flows: S_from = V_f conj(Yff V_f + Yft V_t),
 * S_to = V_t conj(Ytf V_f + Ytt V_t), zero for the task's outaged branch; the
 * operation sequence of the CUDA path (numerics.cuh branch_flow). */
int orc_branch_flows(int32_t n_bus, int32_t n_branch, const int32_t* f, const int32_t* t,
                     const double* adm, int32_t n_tasks, const double* vm, const double* va,
                     const int32_t* outage, double* sf_re, double* sf_im, double* st_re, double* st_im) {
    for (int32_t task = 0; task < n_tasks; ++task) {
        for (int32_t k = 0; k < n_branch; ++k) {
            const size_t o = (size_t)k * n_tasks + task;
            if (outage && outage[task] == k) {
                sf_re[o] = sf_im[o] = st_re[o] = st_im[o] = 0.0;
                continue;
            }
            double sfv, cfv, stv, ctv;
            orc_sincos(va[(size_t)f[k] * n_tasks + task], &sfv, &cfv);
            orc_sincos(va[(size_t)t[k] * n_tasks + task], &stv, &ctv);
            const double vmf = vm[(size_t)f[k] * n_tasks + task], vmt = vm[(size_t)t[k] * n_tasks + task];
            const double vfr = vmf * cfv, vfi = vmf * sfv, vtr = vmt * ctv, vti = vmt * stv;
            const double* a = adm + (size_t)8 * k;
            double ire = 0.0, iim = 0.0;
            ire = fma(a[0], vfr, ire); ire = fma(-a[1], vfi, ire);
            iim = fma(a[0], vfi, iim); iim = fma(a[1], vfr, iim);
            ire = fma(a[2], vtr, ire); ire = fma(-a[3], vti, ire);
            iim = fma(a[2], vti, iim); iim = fma(a[3], vtr, iim);
            sf_re[o] = fma(vfr, ire, vfi * iim);
            sf_im[o] = fma(vfi, ire, -(vfr * iim));
            ire = 0.0; iim = 0.0;
            ire = fma(a[4], vfr, ire); ire = fma(-a[5], vfi, ire);
            iim = fma(a[4], vfi, iim); iim = fma(a[5], vfr, iim);
            ire = fma(a[6], vtr, ire); ire = fma(-a[7], vti, ire);
            iim = fma(a[6], vti, iim); iim = fma(a[7], vtr, iim);
            st_re[o] = fma(vtr, ire, vti * iim);
            st_im[o] = fma(vti, ire, -(vtr * iim));
        }
    }
    (void)n_bus;
    return 0;
}
