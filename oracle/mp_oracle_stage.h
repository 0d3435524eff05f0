/*
 * mp_oracle_stage.h -- TEST INFRASTRUCTURE ONLY.  Precision-generic LOBPCG
 * stage (eigensolvers.hpp:195-321), included twice by mp_oracle.c after the
 * orthonormal_q_{d,f} helpers are defined (see mp_oracle_impl.h for SFX/R).
 */

typedef struct {
  R* X;            /* n x m, caller frees */
  double* theta;   /* m */
  double* resid;   /* m */
  int64_t iterations;
  int converged;
} SFX(stage_out);

/* orthonormal_q_dropping (eigensolvers.hpp:74-85): Q written into W (n x w);
 * returns the kept column count. */
static int64_t SFX(orthonormal_q_dropping)(int64_t n, int64_t w, R* W, int use_mixed,
                                           int64_t* dropped) {
  *dropped = 0;
  orc_try t;
  int64_t kept = w;
  ORC_TRY(t) {
    SFX(orthonormal_q)(n, w, W, use_mixed);
    ORC_TRY_END(t);
  }
  else {
    ORC_CATCH_POP();
    if (t.code != MP_E_RANK_DEFICIENT) orc_throw(t.code, t.idx);
    const R tol = (R)sqrt((double)(sizeof(R) == 8 ? DBL_EPSILON : FLT_EPSILON));
    R* Q = (R*)xcalloc((size_t)(n * (w > 0 ? w : 1)), sizeof(R));
    kept = SFX(ortho_dropping)(n, w, W, tol, Q, dropped);
    memcpy(W, Q, (size_t)(n * kept) * sizeof(R));
    free(Q);
  }
  return kept;
}

static SFX(stage_out) SFX(lobpcg_stage)(const SFX(op_t) * A, int64_t n, const R* X0, int64_t m,
                                        int64_t k, int64_t maxit, const SFX(prec_t) * P,
                                        double a_norm_est, double tol, int use_mixed_qr,
                                        int stagnation_exit, int tag, rec_sink* hist) {
  SFX(stage_out) out;
  memset(&out, 0, sizeof(out));
  R* X = (R*)xmalloc((size_t)(n * m) * sizeof(R));
  memcpy(X, X0, (size_t)(n * m) * sizeof(R));
  R* AX = (R*)xmalloc((size_t)(n * m) * sizeof(R));
  SFX(op_apply)(A, m, X, AX);
  R* theta = (R*)xmalloc((size_t)m * sizeof(R));
  SFX(ritz_rotate)(n, m, X, AX, theta);
  int64_t p = 0;
  R* P_ = NULL;
  R* AP = NULL;
  double best_metric = INFINITY;
  int64_t since_improvement = 0;
  const int64_t kWindow = 40;

  for (int64_t iter = 0;; ++iter) {
    R* Rb = SFX(residual_block)(n, m, AX, X, theta);
    const int64_t n_c = SFX(converged_count)(n, m, a_norm_est, X, theta, Rb, tol);
    if (stagnation_exit) {
      double metric = 0;
      for (int64_t j = 0; j < k && j < m; ++j) {
        const double denom = (a_norm_est + fabs((double)theta[j])) * (double)SFX(col_norm)(n, X + j * n);
        const double ratio = denom > 0 ? (double)SFX(col_norm)(n, Rb + j * n) / denom : INFINITY;
        if (ratio > metric) metric = ratio;
      }
      if (metric < 0.99 * best_metric) {
        best_metric = metric;
        since_improvement = 0;
      } else {
        ++since_improvement;
      }
    }
    const int done = n_c >= k;
    const int out_of_iters = iter >= maxit;
    const int stalled = stagnation_exit && since_improvement >= kWindow;
    if (done || out_of_iters || stalled) {
      SFX(push_record)(hist, tag, n, m, theta, Rb, n_c);
      hist->last_dropped = 0;
      out.X = X;
      out.theta = (double*)xmalloc((size_t)m * sizeof(double));
      out.resid = (double*)xmalloc((size_t)m * sizeof(double));
      for (int64_t j = 0; j < m; ++j) {
        out.theta[j] = (double)theta[j];
        out.resid[j] = (double)SFX(col_norm)(n, Rb + j * n);
      }
      out.iterations = iter;
      out.converged = done;
      free(Rb);
      free(AX);
      free(theta);
      free(P_);
      free(AP);
      return out;
    }
    /* W = T(R), then project + QR twice (eigensolvers.hpp:266-291) */
    R* W = (R*)xmalloc((size_t)(n * m) * sizeof(R));
    SFX(prec_apply)(P, n, m, Rb, W);
    const int64_t b = m + p;
    R* basis = (R*)xmalloc((size_t)(n * b) * sizeof(R));
    memcpy(basis, X, (size_t)(n * m) * sizeof(R));
    if (p) memcpy(basis + n * m, P_, (size_t)(n * p) * sizeof(R));
    int64_t dropped = 0, more = 0, w = m;
    SFX(project_out)(n, b, w, basis, W, 2);
    w = SFX(orthonormal_q_dropping)(n, w, W, use_mixed_qr, &dropped);
    if (w > 0) {
      SFX(project_out)(n, b, w, basis, W, 1);
      w = SFX(orthonormal_q_dropping)(n, w, W, use_mixed_qr, &more);
      dropped += more;
    }
    free(basis);
    if (w == 0 && p == 0) {
      SFX(push_record)(hist, tag, n, m, theta, Rb, n_c);
      orc_throw(MP_E_RANK_COLLAPSE, -1);
    }
    R* AW = (R*)xmalloc((size_t)(n * (w > 0 ? w : 1)) * sizeof(R));
    SFX(op_apply)(A, w, W, AW);
    const int64_t s = m + p + w;
    R* S = (R*)xmalloc((size_t)(n * s) * sizeof(R));
    R* AS = (R*)xmalloc((size_t)(n * s) * sizeof(R));
    memcpy(S, X, (size_t)(n * m) * sizeof(R));
    memcpy(AS, AX, (size_t)(n * m) * sizeof(R));
    if (p) {
      memcpy(S + n * m, P_, (size_t)(n * p) * sizeof(R));
      memcpy(AS + n * m, AP, (size_t)(n * p) * sizeof(R));
    }
    if (w) {
      memcpy(S + n * (m + p), W, (size_t)(n * w) * sizeof(R));
      memcpy(AS + n * (m + p), AW, (size_t)(n * w) * sizeof(R));
    }
    free(W);
    free(AW);
    R* Ap = SFX(adjoint_matmul)(n, s, s, S, AS);
    SFX(hermitize)(s, Ap);
    R* D = (R*)xmalloc((size_t)s * sizeof(R));
    R* Cv = (R*)xmalloc((size_t)(s * s) * sizeof(R));
    SFX(small_herm_eig)(s, Ap, D, Cv);
    free(Ap);
    R* cx = (R*)xmalloc((size_t)(s * m) * sizeof(R));
    R* cpv = (R*)xmalloc((size_t)(s * m) * sizeof(R));
    int64_t pn = 0;
    const int fb = SFX(hl_coeffs)(s, m, Cv, cx, cpv, &pn);
    hist->last_dropped = dropped;
    SFX(push_record)(hist, tag, n, m, theta, Rb, n_c);
    sink_set_last(hist, dropped, fb);
    free(Rb);
    R* Xn = SFX(matmul)(n, s, m, S, cx);
    R* AXn = SFX(matmul)(n, s, m, AS, cx);
    R* Pn = pn ? SFX(matmul)(n, s, pn, S, cpv) : NULL;
    R* APn = pn ? SFX(matmul)(n, s, pn, AS, cpv) : NULL;
    free(X);
    free(AX);
    free(P_);
    free(AP);
    X = Xn;
    AX = AXn;
    P_ = Pn;
    AP = APn;
    p = pn;
    for (int64_t j = 0; j < m; ++j) theta[j] = D[j];
    free(D);
    free(Cv);
    free(cx);
    free(cpv);
    free(S);
    free(AS);
  }
}
