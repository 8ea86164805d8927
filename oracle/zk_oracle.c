/*
 * zk_oracle.c -- CPU restatement of the zlinalg hot-path arithmetic.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2112_06465_b200/,
 * libzk.so) links, loads or calls this file.  It is imported by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg purely as the
 * checker the CUDA path is compared against.
 *
 * The reference (`/root/reference/pkg/src/zlinalg`) is pure Python; its
 * floating-point arithmetic lives in numpy's C loops (numpy 2.3.5, pinned by
 * `pkg/pyproject.toml:10` only as `numpy>=1.24`) and in CPython float/complex
 * operators.  This file restates that arithmetic explicitly so that it is the
 * same on every host:
 *
 *   F1(a,b)   numpy complex multiply under the AVX512F/FMA3 dispatch
 *             re = fma(a.re, b.re, -(a.im*b.im)), im = fma(a.re, b.im, a.im*b.re)
 *             (pinned by tests/golden, generated from the
 *             live reference by tests/golden/make_golden.py).
 *   PW_c/PW_r numpy CDOUBLE/DOUBLE pairwise_sum (4 complex / 8 real lanes,
 *             leaves <= 64 complex / 128 real elements).
 *   SEG       np.add.reduceat segment: v[0] + PW(v[1:]).
 *   fold      Python left fold of block partials (vecops.py:156-162).
 *   cdiv/cmul Python Cplx arithmetic (cnum.py:113-134), no FMA.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off -fno-fast-math); fma()
 * from libm is a correctly rounded fused multiply-add on every host.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct { double re, im; } zc;

/* 1 = numpy FMA complex-multiply formula (AVX512F/FMA3 dispatch),
 * 0 = plain formula (each product rounded).  Elision threshold in bytes of
 * the gathered temporary (numpy NPY_MIN_ELIDE_BYTES = 256 KiB). */
static int g_fma = 1;
static int64_t g_elide_bytes = 262144;

void zko_set_arith(int use_fma, int64_t elide_bytes) {
    g_fma = use_fma;
    g_elide_bytes = elide_bytes;
}

/* numpy complex multiply a*b (loops_arithm_fp complex multiply). */
static inline zc f1(zc a, zc b) {
    zc r;
    if (g_fma) {
        r.re = fma(a.re, b.re, -(a.im * b.im));
        r.im = fma(a.re, b.im, a.im * b.re);
    } else {
        double t0 = a.re * b.re, t1 = a.im * b.im, t2 = a.re * b.im, t3 = a.im * b.re;
        r.re = t0 - t1;
        r.im = t2 + t3;
    }
    return r;
}

/* CPython complex multiply (_Py_c_prod) and Cplx.cmul (cnum.py:113-115):
 * every product rounded, no FMA. */
static inline zc cmul_py(zc a, zc b) {
    zc r;
    double t0 = a.re * b.re, t1 = a.im * b.im, t2 = a.re * b.im, t3 = a.im * b.re;
    r.re = t0 - t1;
    r.im = t2 + t3;
    return r;
}

/* Cplx.cdiv, Smith's algorithm with true divisions (cnum.py:118-134). */
static inline zc cdiv_py(zc a, zc b) {
    double c = b.re, d = b.im;
    zc q;
    if (fabs(c) >= fabs(d)) {
        double r = d / c;
        double den = c + d * r;
        q.re = (a.re + a.im * r) / den;
        q.im = (a.im - a.re * r) / den;
    } else {
        double r = c / d;
        double den = c * r + d;
        q.re = (a.re * r + a.im) / den;
        q.im = (a.im * r - a.re) / den;
    }
    return q;
}

static inline int small_py(zc v) { return hypot(v.re, v.im) < 1e-300; } /* krylov.py:209-210 */

/* ---- numpy pairwise sums ------------------------------------------------ */

static zc pw_c(const zc* v, int64_t L) {
    zc s;
    if (L < 4) {                       /* 2L < 8: sequential from -0.0 */
        s.re = -0.0; s.im = -0.0;
        for (int64_t i = 0; i < L; ++i) { s.re += v[i].re; s.im += v[i].im; }
        return s;
    }
    if (L <= 64) {                     /* 2L <= PW_BLOCKSIZE(128): 4 lanes */
        double r0 = v[0].re, r1 = v[1].re, r2 = v[2].re, r3 = v[3].re;
        double i0 = v[0].im, i1 = v[1].im, i2 = v[2].im, i3 = v[3].im;
        int64_t G = L / 4;
        for (int64_t g = 1; g < G; ++g) {
            r0 += v[4 * g + 0].re; i0 += v[4 * g + 0].im;
            r1 += v[4 * g + 1].re; i1 += v[4 * g + 1].im;
            r2 += v[4 * g + 2].re; i2 += v[4 * g + 2].im;
            r3 += v[4 * g + 3].re; i3 += v[4 * g + 3].im;
        }
        s.re = (r0 + r1) + (r2 + r3);
        s.im = (i0 + i1) + (i2 + i3);
        for (int64_t k = 4 * G; k < L; ++k) { s.re += v[k].re; s.im += v[k].im; }
        return s;
    }
    int64_t h = (L - L % 8) / 2;       /* n2 = n/2 - (n/2)%8 doubles */
    zc a = pw_c(v, h), b = pw_c(v + h, L - h);
    s.re = a.re + b.re;
    s.im = a.im + b.im;
    return s;
}

static double pw_r(const double* v, int64_t L) {
    if (L < 8) {
        double s = -0.0;
        for (int64_t i = 0; i < L; ++i) s += v[i];
        return s;
    }
    if (L <= 128) {
        double r[8];
        for (int q = 0; q < 8; ++q) r[q] = v[q];
        int64_t G = L / 8;
        for (int64_t g = 1; g < G; ++g)
            for (int q = 0; q < 8; ++q) r[q] += v[8 * g + q];
        double s = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (int64_t k = 8 * G; k < L; ++k) s += v[k];
        return s;
    }
    int64_t h = L / 2;
    h -= h % 8;
    return pw_r(v, h) + pw_r(v + h, L - h);
}

/* np.add.reduceat segment of length L >= 1. */
static zc seg_c(const zc* v, int64_t L) {
    if (L == 1) return v[0];
    zc p = pw_c(v + 1, L - 1), s;
    s.re = v[0].re + p.re;
    s.im = v[0].im + p.im;
    return s;
}

static double seg_r(const double* v, int64_t L) {
    if (L == 1) return v[0];
    return v[0] + pw_r(v + 1, L - 1);
}

/* ---- level-1 kernels (vecops.py) ----------------------------------------- */

/* zscal: x.data *= complex(alpha)  ->  x = F1(x, alpha)   (vecops.py:124-127) */
void zko_zscal(int64_t n, double ar, double ai, double* x) {
    zc a = {ar, ai};
    zc* v = (zc*)x;
    for (int64_t i = 0; i < n; ++i) v[i] = f1(v[i], a);
}

/* zaxpy: y.data += complex(alpha) * x.data  ->  y = y + F1(alpha, x) (vecops.py:130-134) */
void zko_zaxpy(int64_t n, double ar, double ai, const double* x, double* y) {
    zc a = {ar, ai};
    const zc* xv = (const zc*)x;
    zc* yv = (zc*)y;
    for (int64_t i = 0; i < n; ++i) {
        zc t = f1(a, xv[i]);
        yv[i].re = yv[i].re + t.re;
        yv[i].im = yv[i].im + t.im;
    }
}

/* zaxmy: y.data *= x.data -> y = F1(y, x) (vecops.py:137-141) */
void zko_zaxmy(int64_t n, const double* x, double* y) {
    const zc* xv = (const zc*)x;
    zc* yv = (zc*)y;
    for (int64_t i = 0; i < n; ++i) yv[i] = f1(yv[i], xv[i]);
}

/* Preconditioner.apply (jacobi): out = F1(v, minv) (krylov.py:92-100) */
void zko_jacobi_apply(int64_t n, const double* v, const double* minv, double* out) {
    const zc* vv = (const zc*)v;
    const zc* mv = (const zc*)minv;
    zc* o = (zc*)out;
    for (int64_t i = 0; i < n; ++i) o[i] = f1(vv[i], mv[i]);
}

/* zdot (vecops.py:165-186).  mode 0 = blocked (reduceat + left fold,
 * vecops.py:156-162), mode 1 = sequential (CPython loop, plain product). */
void zko_zdot(int64_t n, const double* x, const double* y, int conjugate, int64_t block,
              int mode, double* out) {
    const zc* xv = (const zc*)x;
    const zc* yv = (const zc*)y;
    if (n == 0) { out[0] = 0.0; out[1] = 0.0; return; }
    if (mode == 1) {
        zc acc = {0.0, 0.0};
        for (int64_t i = 0; i < n; ++i) {
            zc a = xv[i];
            if (conjugate) a.im = -a.im;
            zc p = cmul_py(a, yv[i]);
            acc.re = acc.re + p.re;
            acc.im = acc.im + p.im;
        }
        out[0] = acc.re; out[1] = acc.im;
        return;
    }
    zc* prod = (zc*)malloc(sizeof(zc) * (size_t)block);
    zc total = {0.0, 0.0};
    for (int64_t b0 = 0; b0 < n; b0 += block) {
        int64_t L = n - b0 < block ? n - b0 : block;
        for (int64_t k = 0; k < L; ++k) {
            zc a = xv[b0 + k];
            if (conjugate) a.im = -a.im;  /* np.conj */
            prod[k] = f1(a, yv[b0 + k]);
        }
        zc p = seg_c(prod, L);
        if (b0 == 0) total = p;
        else { total.re = total.re + p.re; total.im = total.im + p.im; }
    }
    free(prod);
    out[0] = total.re; out[1] = total.im;
}

/* znorm2 (vecops.py:189-200): sq = (re*re) + (im*im) as two separate ufunc
 * passes (no FMA), blocked reduceat + fold, math.sqrt. */
double zko_znorm2(int64_t n, const double* x, int64_t block, int mode) {
    const zc* xv = (const zc*)x;
    if (n == 0) return 0.0;
    if (mode == 1) {
        double acc = 0.0;
        for (int64_t i = 0; i < n; ++i) {
            double a = xv[i].re * xv[i].re;
            double b = xv[i].im * xv[i].im;
            acc = acc + (a + b);
        }
        return sqrt(acc);
    }
    double* sq = (double*)malloc(sizeof(double) * (size_t)block);
    double total = 0.0;
    for (int64_t b0 = 0; b0 < n; b0 += block) {
        int64_t L = n - b0 < block ? n - b0 : block;
        for (int64_t k = 0; k < L; ++k) {
            double a = xv[b0 + k].re * xv[b0 + k].re;
            double b = xv[b0 + k].im * xv[b0 + k].im;
            sq[k] = a + b;
        }
        double p = seg_r(sq, L);
        total = (b0 == 0) ? p : total + p;
    }
    free(sq);
    return sqrt(total);
}

/* ---- SpMV (sparse.py:217-232) ------------------------------------------- */

/* y = A x.  prod = A.aa * x.data[A.ja]; numpy elides the gathered temporary
 * when it is >= the elision threshold and then computes F1(x[ja], aa)
 * instead of F1(aa, x[ja]).  Rows sum by reduceat; empty rows stay +0. */
void zko_spmv(int64_t n_rows, int64_t n_cols, const int64_t* ia, const int64_t* ja,
              const double* aa, const double* x, double* y) {
    (void)n_cols;
    const zc* av = (const zc*)aa;
    const zc* xv = (const zc*)x;
    zc* yv = (zc*)y;
    int64_t nnz = n_rows ? ia[n_rows] : 0;
    int swap = nnz * 16 >= g_elide_bytes;
    int64_t maxlen = 0;
    for (int64_t i = 0; i < n_rows; ++i)
        if (ia[i + 1] - ia[i] > maxlen) maxlen = ia[i + 1] - ia[i];
    zc* prod = (zc*)malloc(sizeof(zc) * (size_t)(maxlen > 0 ? maxlen : 1));
    for (int64_t i = 0; i < n_rows; ++i) {
        int64_t lo = ia[i], L = ia[i + 1] - ia[i];
        if (L == 0) { yv[i].re = 0.0; yv[i].im = 0.0; continue; }
        for (int64_t k = 0; k < L; ++k) {
            zc xa = xv[ja[lo + k]];
            prod[k] = swap ? f1(xa, av[lo + k]) : f1(av[lo + k], xa);
        }
        yv[i] = seg_c(prod, L);
    }
    free(prod);
}

/* ---- BiCGStab (krylov.py:213-295, _Run krylov.py:139-206) ---------------- */

enum { ZKO_CONVERGED = 0, ZKO_NOT_CONVERGED = 1, ZKO_BREAKDOWN = 2 };
enum { ZKO_BD_NONE = 0, ZKO_BD_RHO = 1, ZKO_BD_OMEGA = 2, ZKO_BD_PIVOT = 3, ZKO_BD_TT = 4 };

typedef struct {
    int64_t n, n_rows;
    const int64_t *ia, *ja;
    const double* aa;
    const double* b;
    const double* minv;
    double b_norm;
} zko_run;

static void dot_def(int64_t n, const zc* x, const zc* y, zc* out) {
    double o[2];
    zko_zdot(n, (const double*)x, (const double*)y, 1, 4096, 0, o);
    out->re = o[0]; out->im = o[1];
}

static double nrm_def(int64_t n, const zc* x) { return zko_znorm2(n, (const double*)x, 4096, 0); }

/* _Run.true_relative_residual: znorm2(b + F1(-1, A x)) / b_norm */
static double true_rel(zko_run* R, const zc* x, zc* tmp, zc* tmp2) {
    zko_spmv(R->n, R->n, R->ia, R->ja, R->aa, (const double*)x, (double*)tmp);
    memcpy(tmp2, R->b, sizeof(zc) * (size_t)R->n);
    zko_zaxpy(R->n, -1.0, 0.0, (const double*)tmp, (double*)tmp2);
    return nrm_def(R->n, tmp2) / R->b_norm;
}

static void precond(zko_run* R, const zc* v, zc* out) {
    if (R->minv) zko_jacobi_apply(R->n, (const double*)v, R->minv, (double*)out);
    else memcpy(out, v, sizeof(zc) * (size_t)R->n);
}

/* Returns status; x_out[n]; hist_out[maxit+1]; *iters_out = iterations. */
int zko_bicgstab(int64_t n, const int64_t* ia, const int64_t* ja, const double* aa,
                 const double* b, const double* minv, const double* x0, double tol,
                 int64_t maxit, double* x_out, double* hist_out, int64_t* iters_out,
                 int* what_out) {
    zko_run R = {n, n, ia, ja, aa, b, minv, 0.0};
    size_t bytes = sizeof(zc) * (size_t)(n > 0 ? n : 1);
    zc *x = (zc*)x_out, *r = malloc(bytes), *rs = malloc(bytes), *p = malloc(bytes),
       *v = malloc(bytes), *s = malloc(bytes), *t = malloc(bytes), *ph = malloc(bytes),
       *sh = malloc(bytes), *t1 = malloc(bytes), *t2 = malloc(bytes);
    int status = ZKO_NOT_CONVERGED;
    int64_t it = 0;
    *what_out = ZKO_BD_NONE;

    if (x0) memcpy(x, x0, sizeof(zc) * (size_t)n);
    else memset(x, 0, sizeof(zc) * (size_t)n);
    R.b_norm = nrm_def(n, (const zc*)b);
    /* r0 = b.copy(); zaxpy(-1, spmv(A, x0), r0) */
    zko_spmv(n, n, ia, ja, aa, (const double*)x, (double*)t1);
    memcpy(r, b, sizeof(zc) * (size_t)n);
    zko_zaxpy(n, -1.0, 0.0, (const double*)t1, (double*)r);
    double r0_norm = nrm_def(n, r);
    hist_out[0] = R.b_norm > 0.0 ? r0_norm / R.b_norm : 0.0;
    if (R.b_norm == 0.0) {             /* trivial_result: zero rhs */
        memset(x, 0, sizeof(zc) * (size_t)n);
        hist_out[0] = 0.0;
        status = ZKO_CONVERGED;
        goto done;
    }
    if (hist_out[0] <= tol) { status = ZKO_CONVERGED; goto done; }

    memcpy(rs, r, sizeof(zc) * (size_t)n);
    memset(v, 0, sizeof(zc) * (size_t)n);
    memset(p, 0, sizeof(zc) * (size_t)n);
    zc rho = {1.0, 0.0}, alpha = {1.0, 0.0}, omega = {1.0, 0.0};

    while (it < maxit) {
        zc rho_next;
        dot_def(n, rs, r, &rho_next);
        if (small_py(rho)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_RHO; goto done; }
        if (small_py(omega)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_OMEGA; goto done; }
        zc beta = cmul_py(cdiv_py(rho_next, rho), cdiv_py(alpha, omega));
        rho = rho_next;
        zko_zaxpy(n, -omega.re, -omega.im, (const double*)v, (double*)p);
        zko_zscal(n, beta.re, beta.im, (double*)p);
        zko_zaxpy(n, 1.0, 0.0, (const double*)r, (double*)p);
        precond(&R, p, ph);
        zko_spmv(n, n, ia, ja, aa, (const double*)ph, (double*)v);
        zc pivot;
        dot_def(n, rs, v, &pivot);
        if (small_py(pivot)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_PIVOT; goto done; }
        alpha = cdiv_py(rho, pivot);
        memcpy(s, r, sizeof(zc) * (size_t)n);
        zko_zaxpy(n, -alpha.re, -alpha.im, (const double*)v, (double*)s);
        zko_zaxpy(n, alpha.re, alpha.im, (const double*)ph, (double*)x);
        if (nrm_def(n, s) / R.b_norm <= tol) {
            double rel = true_rel(&R, x, t1, t2);
            if (rel <= tol) {
                hist_out[++it] = rel;
                status = ZKO_CONVERGED;
                goto done;
            }
        }
        precond(&R, s, sh);
        zko_spmv(n, n, ia, ja, aa, (const double*)sh, (double*)t);
        zc tt, ts;
        dot_def(n, t, t, &tt);
        if (small_py(tt)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_TT; goto done; }
        dot_def(n, t, s, &ts);
        omega = cdiv_py(ts, tt);
        if (small_py(omega)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_OMEGA; goto done; }
        zko_zaxpy(n, omega.re, omega.im, (const double*)sh, (double*)x);
        /* r = s; zaxpy(-omega, t, r) */
        zc* tmp = r; r = s; s = tmp;
        zko_zaxpy(n, -omega.re, -omega.im, (const double*)t, (double*)r);
        double rel = true_rel(&R, x, t1, t2);
        hist_out[++it] = rel;
        if (rel <= tol) { status = ZKO_CONVERGED; goto done; }
    }
done:
    *iters_out = it;
    free(r); free(rs); free(p); free(v); free(s); free(t); free(ph); free(sh); free(t1); free(t2);
    return status;
}

/* ---- BiCGSTAB(l) and TFQMR (krylov.py:298-489) ------------------------------
 * Breakdown codes shared with the device drivers (include/zk.h ZK_BD_*):
 * 1 rho, 2 omega, 3 shadow pivot, 5 minimal-residual basis vector j
 * (*what_j_out = j), 6 sigma = <r~, v>, 7 alpha, 8 quasi-residual tau. */
enum { ZKO_BD_MR = 5, ZKO_BD_SIGMA = 6, ZKO_BD_ALPHA = 7, ZKO_BD_TAU = 8 };

static int small_r(double v) { return fabs(v) < 1e-300; }
static zc zc_neg(zc a) { zc r = {-a.re, -a.im}; return r; }
static zc zc_add(zc a, zc b) { zc r = {a.re + b.re, a.im + b.im}; return r; }
static zc zc_sub(zc a, zc b) { zc r = {a.re - b.re, a.im - b.im}; return r; }
static zc zc_real(double v) { zc r = {v, 0.0}; return r; }
static void axpy_c(int64_t n, zc a, const zc* x, zc* y) { zko_zaxpy(n, a.re, a.im, (const double*)x, (double*)y); }
static void scal_c(int64_t n, zc a, zc* x) { zko_zscal(n, a.re, a.im, (double*)x); }

/* op(v) = spmv(A, M.apply(v)) (krylov.py:320-321) */
static void op_apply(zko_run* R, const zc* v, zc* tmp, zc* out) {
    precond(R, v, tmp);
    zko_spmv(R->n, R->n, R->ia, R->ja, R->aa, (const double*)tmp, (double*)out);
}

/* _Run.__init__ + trivial_result (krylov.py:147-181).  Returns 1 when the
 * solve is trivially finished (status in *status). */
static int run_setup(zko_run* R, const zc* x0, zc* x, zc* r0, zc* tmp, double tol, double* hist,
                     double* r0_norm, int* status) {
    int64_t n = R->n;
    if (x0) memcpy(x, x0, sizeof(zc) * (size_t)n);
    else memset(x, 0, sizeof(zc) * (size_t)n);
    R->b_norm = nrm_def(n, (const zc*)R->b);
    zko_spmv(n, n, R->ia, R->ja, R->aa, (const double*)x, (double*)tmp);
    memcpy(r0, R->b, sizeof(zc) * (size_t)n);
    zko_zaxpy(n, -1.0, 0.0, (const double*)tmp, (double*)r0);
    *r0_norm = nrm_def(n, r0);
    hist[0] = R->b_norm > 0.0 ? *r0_norm / R->b_norm : 0.0;
    if (R->b_norm == 0.0) {
        memset(x, 0, sizeof(zc) * (size_t)n);
        hist[0] = 0.0;
        *status = ZKO_CONVERGED;
        return 1;
    }
    if (hist[0] <= tol) { *status = ZKO_CONVERGED; return 1; }
    return 0;
}

/* current_x(acc) = x0 + M^-1 acc (krylov.py:323-326) */
static void current_x(zko_run* R, const zc* x0, const zc* acc, zc* tmp, zc* x) {
    if (x0) memcpy(x, x0, sizeof(zc) * (size_t)R->n);
    else memset(x, 0, sizeof(zc) * (size_t)R->n);
    precond(R, acc, tmp);
    axpy_c(R->n, zc_real(1.0), tmp, x);
}

int zko_bicgstab_l(int64_t n, const int64_t* ia, const int64_t* ja, const double* aa,
                   const double* b, const double* minv, const double* x0d, double tol,
                   int64_t maxit, int ell, double* x_out, double* hist, int64_t* iters_out,
                   int* what_out, int* what_j_out) {
    zko_run R = {n, n, ia, ja, aa, b, minv, 0.0};
    const zc* x0 = (const zc*)x0d;
    size_t bytes = sizeof(zc) * (size_t)(n > 0 ? n : 1);
    zc* x = (zc*)x_out;
    zc *tmp = malloc(bytes), *t2 = malloc(bytes), *acc = calloc(1, bytes), *rs = malloc(bytes);
    if (ell < 1) ell = 1;
    zc** r = malloc(sizeof(zc*) * (size_t)(ell + 1));
    zc** u = malloc(sizeof(zc*) * (size_t)(ell + 1));
    for (int i = 0; i <= ell; ++i) { r[i] = calloc(1, bytes); u[i] = calloc(1, bytes); }
    int L1 = ell + 1;
    zc* tau = calloc((size_t)L1 * L1, sizeof(zc));
    double* sigma = calloc((size_t)L1, sizeof(double));
    zc *gp = calloc((size_t)L1, sizeof(zc)), *gm = calloc((size_t)L1, sizeof(zc)), *gpp = calloc((size_t)L1, sizeof(zc));
    int status = ZKO_NOT_CONVERGED;
    int64_t it = 0;
    double r0_norm;
    *what_out = ZKO_BD_NONE;
    *what_j_out = 0;
    if (run_setup(&R, x0, x, r[0], tmp, tol, hist, &r0_norm, &status)) goto done;
    memcpy(rs, r[0], bytes);
    zc rho = zc_real(1.0), alpha = zc_real(0.0), omega = zc_real(1.0);
    while (it < maxit) {
        if (small_py(omega)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_OMEGA; goto done; }
        rho = cmul_py(zc_neg(omega), rho);
        for (int j = 0; j < ell; ++j) {
            zc rho_next;
            dot_def(n, rs, r[j], &rho_next);
            if (small_py(rho)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_RHO; goto done; }
            zc beta = cmul_py(alpha, cdiv_py(rho_next, rho));
            rho = rho_next;
            for (int i = 0; i <= j; ++i) {
                scal_c(n, zc_neg(beta), u[i]);
                axpy_c(n, zc_real(1.0), r[i], u[i]);
            }
            op_apply(&R, u[j], tmp, u[j + 1]);
            zc pivot;
            dot_def(n, rs, u[j + 1], &pivot);
            if (small_py(pivot)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_PIVOT; goto done; }
            alpha = cdiv_py(rho, pivot);
            for (int i = 0; i <= j; ++i) axpy_c(n, zc_neg(alpha), u[i + 1], r[i]);
            op_apply(&R, r[j], tmp, r[j + 1]);
            axpy_c(n, alpha, u[0], acc);
            if (nrm_def(n, r[0]) / R.b_norm <= tol) {
                current_x(&R, x0, acc, tmp, x);
                double rel = true_rel(&R, x, tmp, t2);
                if (rel <= tol) { hist[++it] = rel; status = ZKO_CONVERGED; goto done; }
            }
        }
        for (int j = 1; j <= ell; ++j) {
            for (int i = 1; i < j; ++i) {
                zc d;
                dot_def(n, r[i], r[j], &d);
                zc tij = cdiv_py(d, zc_real(sigma[i]));
                tau[i * L1 + j] = tij;
                axpy_c(n, zc_neg(tij), r[i], r[j]);
            }
            zc sg;
            dot_def(n, r[j], r[j], &sg);
            sigma[j] = sg.re;
            if (small_r(sigma[j])) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_MR; *what_j_out = j; goto done; }
            zc g;
            dot_def(n, r[j], r[0], &g);
            gp[j] = cdiv_py(g, zc_real(sigma[j]));
        }
        for (int j = 0; j <= ell; ++j) gm[j] = zc_real(0.0);
        gm[ell] = gp[ell];
        omega = gm[ell];
        for (int j = ell - 1; j >= 1; --j) {
            zc s = zc_real(0.0);
            for (int i = j + 1; i <= ell; ++i) s = zc_add(s, cmul_py(tau[j * L1 + i], gm[i]));
            gm[j] = zc_sub(gp[j], s);
        }
        for (int j = 1; j < ell; ++j) {
            zc s = zc_real(0.0);
            for (int i = j + 1; i < ell; ++i) s = zc_add(s, cmul_py(tau[j * L1 + i], gm[i + 1]));
            gpp[j] = zc_add(gm[j + 1], s);
        }
        axpy_c(n, gm[1], r[0], acc);
        axpy_c(n, zc_neg(gp[ell]), r[ell], r[0]);
        axpy_c(n, zc_neg(gm[ell]), u[ell], u[0]);
        for (int j = 1; j < ell; ++j) {
            axpy_c(n, zc_neg(gm[j]), u[j], u[0]);
            axpy_c(n, gpp[j], r[j], acc);
            axpy_c(n, zc_neg(gp[j]), r[j], r[0]);
        }
        current_x(&R, x0, acc, tmp, x);
        double rel = true_rel(&R, x, tmp, t2);
        hist[++it] = rel;
        if (rel <= tol) { status = ZKO_CONVERGED; goto done; }
    }
done:
    *iters_out = it;
    for (int i = 0; i <= ell; ++i) { free(r[i]); free(u[i]); }
    free(r); free(u); free(tmp); free(t2); free(acc); free(rs); free(tau); free(sigma); free(gp); free(gm); free(gpp);
    return status;
}

int zko_tfqmr(int64_t n, const int64_t* ia, const int64_t* ja, const double* aa,
              const double* b, const double* minv, const double* x0d, double tol,
              int64_t maxit, double* x_out, double* hist, int64_t* iters_out, int* what_out) {
    zko_run R = {n, n, ia, ja, aa, b, minv, 0.0};
    size_t bytes = sizeof(zc) * (size_t)(n > 0 ? n : 1);
    zc* x = (zc*)x_out;
    zc *r0 = malloc(bytes), *w = malloc(bytes), *y = malloc(bytes), *rs = malloc(bytes), *d = calloc(1, bytes),
       *z = malloc(bytes), *uv = malloc(bytes), *uo = malloc(bytes), *v = malloc(bytes), *t1 = malloc(bytes),
       *t2 = malloc(bytes);
    int status = ZKO_NOT_CONVERGED;
    int64_t it = 0;
    double r0_norm;
    *what_out = ZKO_BD_NONE;
    if (run_setup(&R, (const zc*)x0d, x, r0, t1, tol, hist, &r0_norm, &status)) goto done;
    memcpy(w, r0, bytes);
    memcpy(y, r0, bytes);
    memcpy(rs, r0, bytes);
    precond(&R, y, z);
    zko_spmv(n, n, ia, ja, aa, (const double*)z, (double*)uv);
    memcpy(v, uv, bytes);
    double theta = 0.0, tau = r0_norm;
    zc eta = zc_real(0.0), rho;
    dot_def(n, rs, r0, &rho);
    while (it < maxit) {
        zc sigma;
        dot_def(n, rs, v, &sigma);
        if (small_py(sigma)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_SIGMA; goto done; }
        zc alpha = cdiv_py(rho, sigma);
        if (small_py(alpha)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_ALPHA; goto done; }
        double rel = INFINITY;
        int converged = 0;
        for (int half = 0; half < 2; ++half) {
            if (half == 1) {
                axpy_c(n, zc_neg(alpha), v, y);
                precond(&R, y, z);
                zko_spmv(n, n, ia, ja, aa, (const double*)z, (double*)uv);
            }
            axpy_c(n, zc_neg(alpha), uv, w);
            /* (theta * theta) * eta / alpha: Cplx.__rmul__ = cmul(eta, theta^2), then cdiv */
            scal_c(n, cdiv_py(cmul_py(eta, zc_real(theta * theta)), alpha), d);
            axpy_c(n, zc_real(1.0), z, d);
            if (small_r(tau)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_TAU; goto done; }
            theta = nrm_def(n, w) / tau;
            double c = 1.0 / sqrt(1.0 + theta * theta);
            tau = tau * theta * c;
            eta = cmul_py(alpha, zc_real(c * c));
            axpy_c(n, eta, d, x);
            rel = true_rel(&R, x, t1, t2);
            if (rel <= tol) { converged = 1; break; }
        }
        hist[++it] = rel;
        if (converged) { status = ZKO_CONVERGED; goto done; }
        zc rho_next;
        dot_def(n, rs, w, &rho_next);
        if (small_py(rho)) { status = ZKO_BREAKDOWN; *what_out = ZKO_BD_RHO; goto done; }
        zc beta = cdiv_py(rho_next, rho);
        rho = rho_next;
        scal_c(n, beta, y);
        axpy_c(n, zc_real(1.0), w, y);
        zc* tmp = uo; uo = uv; uv = tmp;  /* u_old = uvec */
        precond(&R, y, z);
        zko_spmv(n, n, ia, ja, aa, (const double*)z, (double*)uv);
        scal_c(n, beta, v);
        axpy_c(n, zc_real(1.0), uo, v);
        scal_c(n, beta, v);
        axpy_c(n, zc_real(1.0), uv, v);
    }
done:
    *iters_out = it;
    free(r0); free(w); free(y); free(rs); free(d); free(z); free(uv); free(uo); free(v); free(t1); free(t2);
    return status;
}
