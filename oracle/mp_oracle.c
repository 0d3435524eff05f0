/*
 * mp_oracle.c -- TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference mixed-precision LOBPCG / PINVIT solver (arXiv 2302.12528 artifact,
 * /root/reference/proj).  It is the CPU checker for the sm_100a product path,
 * never part of it.  Exported over mp_oracle.h with prefix mporc_.
 *
 * Parity pinned (tests/test_oracle.py) against
 *   - the reference itself (oracle/_ref/libmpeig_ref.so, same inputs), and
 *   - the reference's golden vectors (PCG64 outputs, test_precision.cpp:56-71;
 *     to_lower rounding/overflow, :31-54; converged_count prefix cases,
 *     test_eigensolvers.cpp:180-199; analytic Laplacian spectra).
 *
 * Built with -ffp-contract=off so each product and sum rounds separately,
 * like the reference's x86-64 build without -mfma.
 */
#define _POSIX_C_SOURCE 199309L
#include <float.h>
#include <math.h>
#include <setjmp.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#include "mp_oracle.h"

/* ------------------------------------------------------------ infrastructure */
static void* xmalloc(size_t b) {
  void* p = malloc(b ? b : 1);
  if (!p) {
    fprintf(stderr, "mp_oracle: out of memory\n");
    abort();
  }
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) {
    fprintf(stderr, "mp_oracle: out of memory\n");
    abort();
  }
  return p;
}

/* exceptions of the reference (errors.hpp) as a setjmp/longjmp stack */
typedef struct {
  jmp_buf jb;
  int code;
  int64_t idx;
} orc_try;
static orc_try* g_try[256];
static int g_try_n = 0;

static void orc_throw(int code, int64_t idx) {
  if (g_try_n <= 0) {
    fprintf(stderr, "mp_oracle: uncaught error %d\n", code);
    abort();
  }
  orc_try* t = g_try[g_try_n - 1];
  t->code = code;
  t->idx = idx;
  longjmp(t->jb, 1);
}
#define ORC_TRY(t) \
  g_try[g_try_n++] = &(t); \
  if (setjmp((t).jb) == 0)
#define ORC_TRY_END(t) (--g_try_n)
#define ORC_CATCH_POP() (--g_try_n)

/* to_lower (precision.hpp:102-107): round to nearest, finite->inf throws */
static float to_lower_checked(double x) {
  const float y = (float)x;
  if (isfinite(x) && !isfinite((double)y)) orc_throw(MP_E_OVERFLOW, -1);
  return y;
}

/* IterationRecord sink (solver_types.hpp:59-66) writing into mp_result */
typedef struct {
  mp_result* out;
  int64_t m;
  int64_t len;
  int64_t last_dropped;
} rec_sink;

static void sink_push(rec_sink* h, int stage, int64_t m, const double* rv, const double* rn,
                      int64_t n_c) {
  mp_result* o = h->out;
  const int64_t i = h->len++;
  if (!o || i >= o->hist_cap) return;
  if (o->hist_stage) o->hist_stage[i] = stage;
  if (o->hist_nc) o->hist_nc[i] = n_c;
  if (o->hist_dropped) o->hist_dropped[i] = 0;
  if (o->hist_fallback) o->hist_fallback[i] = 0;
  for (int64_t j = 0; j < h->m; ++j) {
    if (o->hist_ritz) o->hist_ritz[i * h->m + j] = j < m ? rv[j] : NAN;
    if (o->hist_resid) o->hist_resid[i * h->m + j] = j < m ? rn[j] : NAN;
  }
}

static void sink_set_last(rec_sink* h, int64_t dropped, int fallback) {
  mp_result* o = h->out;
  const int64_t i = h->len - 1;
  if (!o || i < 0 || i >= o->hist_cap) return;
  if (o->hist_dropped) o->hist_dropped[i] = dropped;
  if (o->hist_fallback) o->hist_fallback[i] = fallback;
}

/* ---------------------------------------------------------------- PCG64 RNG */
/* PCG XSL-RR 128/64 with the published PCG64 constants; seeding and the
 * Box-Muller pairing follow rng.cpp:24-56 */
typedef unsigned __int128 u128;
#define U128(hi, lo) (((u128)(hi) << 64) | (u128)(lo))
static const u128 kMult = U128(2549297995355413924ULL, 4865540595714422341ULL);
static const u128 kInc = U128(6364136223846793005ULL, 1442695040888963407ULL);

typedef struct {
  u128 s;
  double spare;
  int has_spare;
} pcg64;

static pcg64 pcg_seed(uint64_t seed) {
  pcg64 g;
  g.s = 0;
  g.s = g.s * kMult + kInc;
  g.s += (u128)seed;
  g.s = g.s * kMult + kInc;
  g.spare = 0;
  g.has_spare = 0;
  return g;
}

static uint64_t pcg_next(pcg64* g) {
  g->s = g->s * kMult + kInc;
  const uint64_t x = (uint64_t)(g->s >> 64) ^ (uint64_t)g->s;
  const unsigned rot = (unsigned)(g->s >> 122);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

static double pcg_gauss(pcg64* g) {
  if (g->has_spare) {
    g->has_spare = 0;
    return g->spare;
  }
  const double u1 = ((double)(pcg_next(g) >> 11) + 1.0) * 0x1p-53;
  const double u2 = (double)(pcg_next(g) >> 11) * 0x1p-53;
  const double mag = sqrt(-2.0 * log(u1));
  const double two_pi = 6.283185307179586476925286766559;
  g->spare = mag * sin(two_pi * u2);
  g->has_spare = 1;
  return mag * cos(two_pi * u2);
}

/* gaussian_matrix<double> (dense_matrix.hpp:144-161) */
static void gaussian_fill(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  pcg64 g = pcg_seed(seed);
  for (int64_t i = 0; i < rows * cols; ++i) out[i] = pcg_gauss(&g);
}

/* ------------------------------------------------------- precision instances */
static double hypot__d(double a, double b) { return hypot(a, b); }
static float hypot__f(float a, float b) { return hypotf(a, b); }
static double copysign__d(double a, double b) { return copysign(a, b); }
static float copysign__f(float a, float b) { return copysignf(a, b); }

#define R double
#define SFX(x) x##_d
#include "mp_oracle_impl.h"
#undef R
#undef SFX
#define R float
#define SFX(x) x##_f
#include "mp_oracle_impl.h"
#undef R
#undef SFX

/* mixed_qr (ortho.hpp:173-186, Alg. 2): fp32 Householder R_l, V = A R_l^-1,
 * Cholesky QR of V, R = R_chol R_w */
static void mixed_qr_d(int64_t n, int64_t m, const double* A, double* Q, double* Rout) {
  if (n < m) orc_throw(MP_E_DIMENSION, -1);
  float* Al = (float*)xmalloc((size_t)(n * m) * sizeof(float));
  for (int64_t i = 0; i < n * m; ++i) Al[i] = to_lower_checked(A[i]);
  float* Ql = (float*)xmalloc((size_t)(n * m) * sizeof(float));
  float* Rl = (float*)xmalloc((size_t)(m * m) * sizeof(float));
  householder_qr_f(n, m, Al, Ql, Rl);
  free(Al);
  free(Ql);
  double* Rw = (double*)xmalloc((size_t)(m * m) * sizeof(double));
  for (int64_t i = 0; i < m * m; ++i) Rw[i] = (double)Rl[i];
  free(Rl);
  double* V = tri_solve_upper_right_d(n, m, Rw, A);
  double* Rc = (double*)xmalloc((size_t)(m * m) * sizeof(double));
  cholesky_qr_d(n, m, V, Q, Rc);
  free(V);
  if (Rout) {
    double* Rr = matmul_d(m, m, m, Rc, Rw);
    memcpy(Rout, Rr, (size_t)(m * m) * sizeof(double));
    free(Rr);
  }
  free(Rc);
  free(Rw);
}

/* detail::orthonormal_q (eigensolvers.hpp:55-70), in place on W */
static void orthonormal_q_d(int64_t n, int64_t m, double* W, int use_mixed) {
  double* Q = (double*)xmalloc((size_t)(n * m) * sizeof(double));
  if (use_mixed) {
    orc_try t;
    int ok = 0;
    ORC_TRY(t) {
      mixed_qr_d(n, m, W, Q, NULL);
      ORC_TRY_END(t);
      ok = 1;
    }
    else {
      ORC_CATCH_POP();
      if (t.code != MP_E_NOT_PD && t.code != MP_E_OVERFLOW) {
        free(Q);
        orc_throw(t.code, t.idx);
      }
    }
    if (ok) {
      memcpy(W, Q, (size_t)(n * m) * sizeof(double));
      free(Q);
      return;
    }
  }
  householder_qr_d(n, m, W, Q, NULL);
  memcpy(W, Q, (size_t)(n * m) * sizeof(double));
  free(Q);
}

static void orthonormal_q_f(int64_t n, int64_t m, float* W, int use_mixed) {
  (void)use_mixed;  /* the lower stage always uses Householder */
  float* Q = (float*)xmalloc((size_t)(n * m) * sizeof(float));
  householder_qr_f(n, m, W, Q, NULL);
  memcpy(W, Q, (size_t)(n * m) * sizeof(float));
  free(Q);
}

#define R double
#define SFX(x) x##_d
#include "mp_oracle_stage.h"
#undef R
#undef SFX
#define R float
#define SFX(x) x##_f
#include "mp_oracle_stage.h"
#undef R
#undef SFX

/* ------------------------------------------------------------------ systems */
typedef struct {
  int64_t n;
  op_t_d A;
  op_t_f Al;
  double* dinv;
  float* dinvf;
  float* vals_l;
  float* dense_l;
  int64_t* rp;
  int64_t* ci;
  double* vals;
} sys_t;

/* builds CSR for Laplacians is unnecessary: the stencil apply already sums in
 * ascending column order (the CSR order of csr_matrix.hpp:31-58) */
static void sys_make(const mp_problem* p, sys_t* s) {
  memset(s, 0, sizeof(*s));
  s->A.kind = s->Al.kind = p->kind;
  s->A.nx = s->Al.nx = p->nx;
  s->A.ny = s->Al.ny = p->ny;
  s->A.nz = s->Al.nz = p->kind == MP_PROB_LAP2D ? 1 : p->nz;
  if (p->kind == MP_PROB_LAP3D) {
    s->n = p->nx * p->ny * p->nz;
  } else if (p->kind == MP_PROB_LAP2D) {
    s->n = p->nx * p->ny;
  } else {
    s->n = p->n;
  }
  s->A.n = s->Al.n = s->n;
  const int64_t n = s->n;
  s->dinv = (double*)xmalloc((size_t)n * sizeof(double));
  s->dinvf = (float*)xmalloc((size_t)n * sizeof(float));
  if (p->kind == MP_PROB_CSR) {
    const int64_t nnz = p->row_ptr[n];
    s->A.rp = s->Al.rp = p->row_ptr;
    s->A.ci = s->Al.ci = p->col_idx;
    s->A.v = p->vals;
    s->vals_l = (float*)xmalloc((size_t)nnz * sizeof(float));
    for (int64_t q = 0; q < nnz; ++q) s->vals_l[q] = (float)p->vals[q];
    s->Al.v = s->vals_l;
  } else if (p->kind == MP_PROB_DENSE) {
    s->A.D = p->dense;
    s->dense_l = (float*)xmalloc((size_t)(n * n) * sizeof(float));
    for (int64_t q = 0; q < n * n; ++q) s->dense_l[q] = (float)p->dense[q];
    s->Al.D = s->dense_l;
  }
  for (int64_t i = 0; i < n; ++i) {
    double d;
    if (p->kind == MP_PROB_LAP3D)
      d = 6.0;
    else if (p->kind == MP_PROB_LAP2D)
      d = 4.0;
    else if (p->kind == MP_PROB_DENSE)
      d = p->dense[i + i * n];
    else {
      d = 0;
      for (int64_t q = p->row_ptr[i]; q < p->row_ptr[i + 1]; ++q)
        if (p->col_idx[q] == i) d = p->vals[q];
    }
    s->dinv[i] = 1.0 / d;
    s->dinvf[i] = (float)s->dinv[i];
  }
}

static void sys_free(sys_t* s) {
  free(s->dinv);
  free(s->dinvf);
  free(s->vals_l);
  free(s->dense_l);
}

static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

/* spectral_norm_estimate (norm_estimate.hpp:15-24) */
static double norm_estimate(const op_t_d* A, int64_t n, int64_t sr, uint64_t seed) {
  double* om = (double*)xmalloc((size_t)(n * sr) * sizeof(double));
  double* y = (double*)xmalloc((size_t)(n * sr) * sizeof(double));
  gaussian_fill(n, sr, seed, om);
  op_apply_d(A, sr, om, y);
  double dn = 0, yn = 0;
  for (int64_t i = 0; i < n * sr; ++i) dn += fabs(om[i]) * fabs(om[i]);
  for (int64_t i = 0; i < n * sr; ++i) yn += fabs(y[i]) * fabs(y[i]);
  free(om);
  free(y);
  dn = sqrt(dn);
  if (dn == 0) return 0;
  return sqrt(yn) / dn;
}

/* ---------------------------------------------------------------- exports */
int mporc_solve(const mp_problem* prob, int variant, const mp_cfg* c, mp_result* out) {
  orc_try t;
  sys_t sys;
  memset(&sys, 0, sizeof(sys));
  out->status = 0;
  out->msg[0] = 0;
  ORC_TRY(t) {
    sys_make(prob, &sys);
    const int64_t n = sys.n;
    const int64_t m = c->block ? c->block : (3 * c->k + 1) / 2;
    /* SolverConfig::validate (solver_types.hpp:43-56) */
    if (c->k < 1 || m < c->k || 3 * m > n || !(c->tol > 0 && c->tol < 1) ||
        !(c->lower_tol > 0 && c->lower_tol < 1) || c->maxit < 1 || c->sketch_rows < 1)
      orc_throw(MP_E_CONFIG, -1);
    rec_sink hs = {out, m, 0, 0};
    const double t0 = now_s();
    const double est = norm_estimate(&sys.A, n, c->sketch_rows, c->seed ^ 0x9e3779b97f4a7c15ULL);
    double* X = (double*)xmalloc((size_t)(n * m) * sizeof(double));
    if (c->x0)
      memcpy(X, c->x0, (size_t)(n * m) * sizeof(double));
    else
      gaussian_fill(n, m, c->seed, X);
    orthonormal_q_d(n, m, X, 1);
    out->t_setup = now_s() - t0;
    out->t_stage1 = 0;
    out->a_norm_est = est;
    out->iters_lower = 0;
    out->iters_working = 0;
    prec_t_d PW;
    PW.mode = variant == MP_DLOBPCG_DCHOL ? 0 : 1;
    PW.dinv = sys.dinv;
    PW.dinvf = sys.dinvf;
    double* theta = NULL;
    double* resid = NULL;
    double* Xf = NULL;
    int converged = 0;
    if (variant == MP_PINVIT) {
      /* pinvit (eigensolvers.hpp:326-390) with the fp32 Jacobi sandwich */
      double* Xt = X;
      X = NULL;
      double* AX = (double*)xmalloc((size_t)(n * m) * sizeof(double));
      double* th = (double*)xmalloc((size_t)m * sizeof(double));
      for (int64_t iter = 0;; ++iter) {
        orc_try t2;
        ORC_TRY(t2) {
          orthonormal_q_d(n, m, Xt, 1);
          ORC_TRY_END(t2);
        }
        else {
          ORC_CATCH_POP();
          orc_throw(t2.code == MP_E_RANK_DEFICIENT ? MP_E_RANK_COLLAPSE : t2.code, t2.idx);
        }
        op_apply_d(&sys.A, m, Xt, AX);
        ritz_rotate_d(n, m, Xt, AX, th);
        double* Rb = residual_block_d(n, m, AX, Xt, th);
        const int64_t n_c = converged_count_d(n, m, est, Xt, th, Rb, c->tol);
        push_record_d(&hs, 0, n, m, th, Rb, n_c);
        if (n_c >= c->k || iter >= c->maxit) {
          converged = n_c >= c->k;
          out->iters_working = iter;
          theta = (double*)xmalloc((size_t)m * sizeof(double));
          resid = (double*)xmalloc((size_t)m * sizeof(double));
          for (int64_t j = 0; j < m; ++j) {
            theta[j] = th[j];
            resid[j] = col_norm_d(n, Rb + j * n);
          }
          Xf = Xt;
          free(Rb);
          break;
        }
        double* W = (double*)xmalloc((size_t)(n * m) * sizeof(double));
        prec_apply_d(&PW, n, m, Rb, W);
        for (int64_t i = 0; i < n * m; ++i) Xt[i] = Xt[i] - W[i];
        free(W);
        free(Rb);
      }
      free(AX);
      free(th);
    } else {
      const int mixed = variant == MP_MPLOBPCG_SCHOL;
      if (mixed) {
        /* stage 1 in binary32 (drivers.hpp:79-96) */
        const double t1 = now_s();
        float* Xl = (float*)xmalloc((size_t)(n * m) * sizeof(float));
        for (int64_t i = 0; i < n * m; ++i) Xl[i] = to_lower_checked(X[i]);
        prec_t_f PL;
        PL.mode = 0;
        PL.dinv = sys.dinvf;
        PL.dinvf = sys.dinvf;
        stage_out_f s1 = lobpcg_stage_f(&sys.Al, n, Xl, m, c->k, c->maxit, &PL, est, c->lower_tol,
                                        0, 1, 1, &hs);
        free(Xl);
        out->iters_lower = s1.iterations;
        for (int64_t i = 0; i < n * m; ++i) X[i] = (double)s1.X[i];
        free(s1.X);
        free(s1.theta);
        free(s1.resid);
        orthonormal_q_d(n, m, X, 1);
        out->t_stage1 = now_s() - t1;
      }
      stage_out_d s2 = lobpcg_stage_d(&sys.A, n, X, m, c->k, c->maxit, &PW, est, c->tol, mixed, 0,
                                      0, &hs);
      free(X);
      X = NULL;
      out->iters_working = s2.iterations;
      converged = s2.converged;
      theta = s2.theta;
      resid = s2.resid;
      Xf = s2.X;
    }
    out->t_total = now_s() - t0;
    out->converged = converged;
    for (int64_t j = 0; j < c->k; ++j) {
      out->theta[j] = theta[j];
      out->resid[j] = resid[j];
    }
    if (out->X) memcpy(out->X, Xf, (size_t)(n * c->k) * sizeof(double));
    out->hist_len = hs.len;
    free(theta);
    free(resid);
    free(Xf);
    free(X);
    ORC_TRY_END(t);
  }
  else {
    ORC_CATCH_POP();
    out->status = t.code;
    snprintf(out->msg, sizeof(out->msg), "mp_oracle error %d (index %lld)", t.code,
             (long long)t.idx);
  }
  sys_free(&sys);
  return out->status;
}

void mporc_pcg64_u64(uint64_t seed, int64_t count, uint64_t* out) {
  pcg64 g = pcg_seed(seed);
  for (int64_t i = 0; i < count; ++i) out[i] = pcg_next(&g);
}

void mporc_gaussian(int64_t rows, int64_t cols, uint64_t seed, double* out) {
  gaussian_fill(rows, cols, seed, out);
}

double mporc_norm_estimate(const mp_problem* prob, int64_t sketch_rows, uint64_t seed) {
  sys_t s;
  sys_make(prob, &s);
  const double e = norm_estimate(&s.A, s.n, sketch_rows, seed);
  sys_free(&s);
  return e;
}

#define GUARD(body)          \
  do {                       \
    orc_try t_;              \
    ORC_TRY(t_) {            \
      body;                  \
      ORC_TRY_END(t_);       \
    }                        \
    else {                   \
      ORC_CATCH_POP();       \
      return t_.code;        \
    }                        \
    return 0;                \
  } while (0)

int mporc_householder_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  GUARD(householder_qr_d(n, m, A, Q, R));
}

int mporc_householder_qr_f32(int64_t n, int64_t m, const float* A, float* Q, float* R) {
  GUARD(householder_qr_f(n, m, A, Q, R));
}

int mporc_mixed_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  GUARD(mixed_qr_d(n, m, A, Q, R));
}

int mporc_cholesky_qr(int64_t n, int64_t m, const double* A, double* Q, double* R) {
  GUARD(cholesky_qr_d(n, m, A, Q, R));
}

int mporc_small_herm_eig(int64_t n, const double* M, double* vals, double* vecs) {
  GUARD(small_herm_eig_d(n, M, vals, vecs));
}

int mporc_hl_update(int64_t n, int64_t s, int64_t m, const double* S, const double* Cm,
                    double* X, double* P, double* c_pv, int32_t* fallback) {
  GUARD({
    double* cx = (double*)xmalloc((size_t)(s * m) * sizeof(double));
    double* cpv = (double*)xmalloc((size_t)(s * m) * sizeof(double));
    int64_t p = 0;
    *fallback = hl_coeffs_d(s, m, Cm, cx, cpv, &p);
    double* Xn = matmul_d(n, s, m, S, cx);
    memcpy(X, Xn, (size_t)(n * m) * sizeof(double));
    free(Xn);
    if (p) {
      double* Pn = matmul_d(n, s, p, S, cpv);
      memcpy(P, Pn, (size_t)(n * p) * sizeof(double));
      free(Pn);
      memcpy(c_pv, cpv, (size_t)(s * p) * sizeof(double));
    }
    free(cx);
    free(cpv);
  });
}

void mporc_project_out(int64_t n, int64_t b, int64_t w, const double* B, double* W, int passes) {
  project_out_d(n, b, w, B, W, passes);
}

int64_t mporc_ortho_dropping(int64_t n, int64_t w, const double* W, double tol, double* Q) {
  return ortho_dropping_d(n, w, W, tol, Q, NULL);
}

void mporc_apply_op(const mp_problem* prob, int64_t ncols, const double* X, double* Y) {
  sys_t s;
  sys_make(prob, &s);
  op_apply_d(&s.A, ncols, X, Y);
  sys_free(&s);
}

int64_t mporc_converged_count(int64_t n, int64_t m, double a_norm_est, const double* X,
                              const double* theta, const double* Rm, double tol) {
  return converged_count_d(n, m, a_norm_est, X, theta, Rm, tol);
}
