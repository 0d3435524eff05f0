/*
 * mp_oracle_impl.h -- TEST INFRASTRUCTURE ONLY.  Precision-generic body of the
 * C restatement, included twice by mp_oracle.c with
 *     R = double, SFX(x) = x##_d   (working precision, binary64)
 *     R = float,  SFX(x) = x##_f   (lower precision, binary32)
 * Every routine restates one reference routine (cited); all arrays are
 * column-major (dense_matrix.hpp:38-41), element (i,j) at a[i + j*ld].
 * Arithmetic is sequential with separate rounding (built -ffp-contract=off),
 * which is what the reference does on x86-64 without -mfma.
 */

/* C = A (n x k) * B (k x m); ascending-l axpy order (dense_kernels.hpp:20-34) */
static R* SFX(matmul)(int64_t n, int64_t k, int64_t m, const R* A, const R* B) {
  R* C = (R*)xcalloc((size_t)(n * m), sizeof(R));
  for (int64_t j = 0; j < m; ++j) {
    R* cj = C + j * n;
    for (int64_t l = 0; l < k; ++l) {
      const R b = B[l + j * k];
      const R* al = A + l * n;
      for (int64_t i = 0; i < n; ++i) cj[i] += al[i] * b;
    }
  }
  return C;
}

/* C = A^T B; A n x ka, B n x kb; dot order (dense_kernels.hpp:36-52) */
static R* SFX(adjoint_matmul)(int64_t n, int64_t ka, int64_t kb, const R* A, const R* B) {
  R* C = (R*)xcalloc((size_t)(ka * kb), sizeof(R));
  for (int64_t j = 0; j < kb; ++j)
    for (int64_t i = 0; i < ka; ++i) {
      R s = 0;
      const R* ai = A + i * n;
      const R* bj = B + j * n;
      for (int64_t l = 0; l < n; ++l) s += ai[l] * bj[l];
      C[i + j * ka] = s;
    }
  return C;
}

/* symmetric part in place, (M + M^T)/2 (dense_kernels.hpp:77-88) */
static void SFX(hermitize)(int64_t s, R* M) {
  for (int64_t j = 0; j < s; ++j)
    for (int64_t i = 0; i <= j; ++i) {
      const R v = (M[i + j * s] + M[j + i * s]) / (R)2;
      M[i + j * s] = v;
      M[j + i * s] = v;
    }
}

static R SFX(col_norm)(int64_t n, const R* x) {
  R s = 0;
  for (int64_t i = 0; i < n; ++i) {
    const R a = (R)fabs((double)x[i]);
    s += a * a;
  }
  return (R)sqrt((double)s);
}

/* ---- Householder (ortho.hpp:30-121) --------------------------------------- */
typedef struct {
  int64_t n, m, steps;
  R* Rm;    /* n x m working copy, ends upper trapezoidal */
  R* V;     /* reflector j in column j, rows 0..n-j-1 */
  R* beta;
} SFX(hh_t);

static void SFX(hh_free)(SFX(hh_t) * h) {
  free(h->Rm);
  free(h->V);
  free(h->beta);
}

/* reduce A (n x m) to upper trapezoid; a vanished column -> RankDeficient */
static SFX(hh_t) SFX(householder_reduce)(int64_t n, int64_t m, const R* A) {
  SFX(hh_t) h;
  h.n = n;
  h.m = m;
  h.steps = n < m ? n : m;
  h.Rm = (R*)xmalloc((size_t)(n * m) * sizeof(R));
  memcpy(h.Rm, A, (size_t)(n * m) * sizeof(R));
  h.V = (R*)xcalloc((size_t)(n * (h.steps > 0 ? h.steps : 1)), sizeof(R));
  h.beta = (R*)xcalloc((size_t)(h.steps > 0 ? h.steps : 1), sizeof(R));
  for (int64_t j = 0; j < h.steps; ++j) {
    const int64_t len = n - j;
    R* cj = h.Rm + j * n;
    R nrm2 = 0;
    for (int64_t i = j; i < n; ++i) {
      const R a = (R)fabs((double)cj[i]);
      nrm2 += a * a;
    }
    const R nrm = (R)sqrt((double)nrm2);
    if (nrm == 0) orc_throw(MP_E_RANK_DEFICIENT, j);
    const R x0 = cj[j];
    const R ax0 = (R)fabs((double)x0);
    const R phase = ax0 > 0 ? x0 / ax0 : (R)1;
    R* v = h.V + j * n;
    v[0] = x0 + phase * nrm;
    for (int64_t i = 1; i < len; ++i) v[i] = cj[j + i];
    R vn2 = 0;
    for (int64_t i = 0; i < len; ++i) {
      const R a = (R)fabs((double)v[i]);
      vn2 += a * a;
    }
    h.beta[j] = (R)2 / vn2;
    for (int64_t c = j; c < m; ++c) {
      R* cc = h.Rm + c * n + j;
      R s = 0;
      for (int64_t i = 0; i < len; ++i) s += v[i] * cc[i];
      s *= h.beta[j];
      for (int64_t i = 0; i < len; ++i) cc[i] -= s * v[i];
    }
    cj[j] = -phase * nrm;
    for (int64_t i = j + 1; i < n; ++i) cj[i] = 0;
  }
  return h;
}

/* Q (n x qc) <- H_0 ... H_{steps-1} Q, last reflector first (ortho.hpp:78-92) */
static void SFX(apply_reflectors)(const SFX(hh_t) * h, int64_t qc, R* Q) {
  const int64_t n = h->n;
  for (int64_t jj = h->steps - 1; jj >= 0; --jj) {
    const int64_t len = n - jj;
    const R* v = h->V + jj * n;
    for (int64_t c = 0; c < qc; ++c) {
      R* q = Q + c * n + (n - len);
      R s = 0;
      for (int64_t i = 0; i < len; ++i) s += v[i] * q[i];
      s *= h->beta[jj];
      for (int64_t i = 0; i < len; ++i) q[i] -= s * v[i];
    }
  }
}

/* sign-fix so diag(R) > 0 (ortho.hpp:95-110); R is rr x rc with ld rr */
static void SFX(fix_phases)(int64_t n, int64_t qc, R* Q, int64_t rr, int64_t rc, R* Rmat) {
  (void)qc;
  const int64_t steps = rr < rc ? rr : rc;
  for (int64_t j = 0; j < steps; ++j) {
    const R d = Rmat[j + j * rr];
    if (d == 0) orc_throw(MP_E_RANK_DEFICIENT, j);
    if (d > 0) continue;
    for (int64_t c = j; c < rc; ++c) Rmat[j + c * rr] = -Rmat[j + c * rr];
    for (int64_t i = 0; i < n; ++i) Q[i + j * n] = -Q[i + j * n];
  }
}

/* thin QR, Q n x m, R m x m (ortho.hpp:127-140) */
static void SFX(householder_qr)(int64_t n, int64_t m, const R* A, R* Q, R* Rout) {
  if (n < m) orc_throw(MP_E_DIMENSION, -1);
  SFX(hh_t) h = SFX(householder_reduce)(n, m, A);
  memset(Q, 0, (size_t)(n * m) * sizeof(R));
  for (int64_t j = 0; j < m; ++j) Q[j + j * n] = 1;
  SFX(apply_reflectors)(&h, m, Q);
  R* Rm = (R*)xcalloc((size_t)(m * m), sizeof(R));
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i <= j; ++i) Rm[i + j * m] = h.Rm[i + j * n];
  SFX(hh_free)(&h);
  SFX(fix_phases)(n, m, Q, m, m, Rm);
  if (Rout) memcpy(Rout, Rm, (size_t)(m * m) * sizeof(R));
  free(Rm);
}

/* square-Q QR of a small p x m block (ortho.hpp:114-121): Q p x p */
static void SFX(householder_qr_square)(int64_t p, int64_t m, const R* A, R* Q) {
  SFX(hh_t) h = SFX(householder_reduce)(p, m, A);
  memset(Q, 0, (size_t)(p * p) * sizeof(R));
  for (int64_t j = 0; j < p; ++j) Q[j + j * p] = 1;
  SFX(apply_reflectors)(&h, p, Q);
  R* Rm = (R*)xmalloc((size_t)(p * m) * sizeof(R));
  memcpy(Rm, h.Rm, (size_t)(p * m) * sizeof(R));
  SFX(hh_free)(&h);
  SFX(fix_phases)(p, p, Q, p, m, Rm);
  free(Rm);
}

/* ---- Cholesky / triangular (dense_kernels.hpp:128-224) --------------------- */
static R* SFX(dense_cholesky)(int64_t n, const R* A) {
  R* L = (R*)xcalloc((size_t)(n * n), sizeof(R));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = j; i < n; ++i) {
      R s = A[i + j * n];
      for (int64_t k = 0; k < j; ++k) s -= L[i + k * n] * L[j + k * n];
      if (i == j) {
        if (!isfinite((double)s)) {
          free(L);
          orc_throw(MP_E_OVERFLOW, j);
        }
        if (!(s > 0)) {
          free(L);
          orc_throw(MP_E_NOT_PD, j);
        }
        L[j + j * n] = (R)sqrt((double)s);
      } else {
        L[i + j * n] = s / L[j + j * n];
      }
    }
  return L;
}

/* X U = B for upper U (n x n), B rows x n (TriMode::UpperInverseRight) */
static R* SFX(tri_solve_upper_right)(int64_t rows, int64_t n, const R* U, const R* B) {
  const R tiny = sizeof(R) == 8 ? (R)DBL_MIN : (R)FLT_MIN;
  for (int64_t j = 0; j < n; ++j) {
    const R a = (R)fabs((double)U[j + j * n]);
    if (a == 0 || a < tiny) orc_throw(MP_E_SINGULAR_TRI, j);
  }
  R* X = (R*)xmalloc((size_t)(rows * n) * sizeof(R));
  for (int64_t j = 0; j < n; ++j) {
    R* xj = X + j * rows;
    const R* bj = B + j * rows;
    for (int64_t i = 0; i < rows; ++i) xj[i] = bj[i];
    for (int64_t k = 0; k < j; ++k) {
      const R u = U[k + j * n];
      const R* xk = X + k * rows;
      for (int64_t i = 0; i < rows; ++i) xj[i] -= xk[i] * u;
    }
    const R d = U[j + j * n];
    for (int64_t i = 0; i < rows; ++i) xj[i] /= d;
  }
  return X;
}

/* Cholesky QR: V^T V = L L^T, Q = V L^{-T}, R = L^T (ortho.hpp:145-160) */
static void SFX(cholesky_qr)(int64_t n, int64_t m, const R* V, R* Q, R* Rout) {
  if (n < m) orc_throw(MP_E_DIMENSION, -1);
  R* G = SFX(adjoint_matmul)(n, m, m, V, V);
  SFX(hermitize)(m, G);
  R* L = SFX(dense_cholesky)(m, G);
  free(G);
  R* U = (R*)xcalloc((size_t)(m * m), sizeof(R));
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < m; ++i) U[i + j * m] = L[j + i * m];
  free(L);
  R* X = SFX(tri_solve_upper_right)(n, m, U, V);
  memcpy(Q, X, (size_t)(n * m) * sizeof(R));
  free(X);
  if (Rout) memcpy(Rout, U, (size_t)(m * m) * sizeof(R));
  free(U);
}

/* block_project_out (ortho.hpp:190-200): W -= B (B^T W), `passes` times */
static void SFX(project_out)(int64_t n, int64_t b, int64_t w, const R* B, R* W, int passes) {
  if (b == 0 || passes <= 0) return;
  for (int p = 0; p < passes; ++p) {
    R* G = SFX(adjoint_matmul)(n, b, w, B, W);
    R* BG = SFX(matmul)(n, b, w, B, G);
    for (int64_t i = 0; i < n * w; ++i) W[i] = W[i] - BG[i];
    free(G);
    free(BG);
  }
}

/* two-pass MGS with column dropping (ortho.hpp:205-250); Q n x w capacity */
static int64_t SFX(ortho_dropping)(int64_t n, int64_t w, const R* W, R drop_tol, R* Q,
                                   int64_t* dropped) {
  int64_t kept = 0, drops = 0;
  R* v = (R*)xmalloc((size_t)n * sizeof(R));
  for (int64_t j = 0; j < w; ++j) {
    memcpy(v, W + j * n, (size_t)n * sizeof(R));
    const R n0 = SFX(col_norm)(n, v);
    if (n0 == 0) {
      ++drops;
      continue;
    }
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t q = 0; q < kept; ++q) {
        const R* qv = Q + q * n;
        R s = 0;
        for (int64_t i = 0; i < n; ++i) s += qv[i] * v[i];
        for (int64_t i = 0; i < n; ++i) v[i] -= s * qv[i];
      }
    const R nv = SFX(col_norm)(n, v);
    if (nv <= drop_tol * n0) {
      ++drops;
      continue;
    }
    R* qk = Q + kept * n;
    for (int64_t i = 0; i < n; ++i) qk[i] = v[i] / nv;
    ++kept;
  }
  free(v);
  if (dropped) *dropped = drops;
  return kept;
}

/* ---- small symmetric eigensolver (small_eig.hpp:25-218) -------------------- */
/* implicit-shift QL with Wilkinson shifts; rotations accumulated into V */
static void SFX(tridiag_ql)(int64_t n, R* d, R* e, R* V) {
  if (n == 0) return;
  const R eps = sizeof(R) == 8 ? (R)DBL_EPSILON : (R)FLT_EPSILON;
  int64_t sweeps = 0;
  const int64_t cap = 30 * n;
  for (int64_t l = 0; l < n; ++l) {
    for (;;) {
      int64_t mm = l;
      while (mm + 1 < n) {
        const R dd = (R)fabs((double)d[mm]) + (R)fabs((double)d[mm + 1]);
        if ((R)fabs((double)e[mm]) <= eps * dd) break;
        ++mm;
      }
      if (mm == l) break;
      if (++sweeps > cap) orc_throw(MP_E_NO_CONVERGENCE, -1);
      R g = (d[l + 1] - d[l]) / (2 * e[l]);
      R r = SFX(hypot_)(g, (R)1);
      g = d[mm] - d[l] + e[l] / (g + SFX(copysign_)(r, g));
      R s = 1, c = 1, p = 0;
      int underflowed = 0;
      for (int64_t i1 = mm - 1; i1 >= l; --i1) {
        R f = s * e[i1];
        const R b = c * e[i1];
        r = SFX(hypot_)(f, g);
        e[i1 + 1] = r;
        if (r == 0) {
          d[i1 + 1] -= p;
          e[mm] = 0;
          underflowed = 1;
          break;
        }
        s = f / r;
        c = g / r;
        g = d[i1 + 1] - p;
        r = (d[i1] - g) * s + 2 * c * b;
        p = s * r;
        d[i1 + 1] = g + p;
        g = c * r - b;
        for (int64_t row = 0; row < n; ++row) {
          const R tmp = V[row + (i1 + 1) * n];
          V[row + (i1 + 1) * n] = s * V[row + i1 * n] + c * tmp;
          V[row + i1 * n] = c * V[row + i1 * n] - s * tmp;
        }
      }
      if (underflowed) continue;
      d[l] -= p;
      e[l] = g;
      e[mm] = 0;
    }
  }
}

#ifndef MPORC_EIG_JACOBI
/* full eigendecomposition: Householder tridiagonalisation, QL, stable sort */
static void SFX(small_herm_eig)(int64_t n, const R* M, R* vals, R* vecs) {
  if (n == 0) return;
  R* W = (R*)xmalloc((size_t)(n * n) * sizeof(R));
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < n; ++i) W[i + j * n] = (M[i + j * n] + M[j + i * n]) / (R)2;
  R* Q = (R*)xcalloc((size_t)(n * n), sizeof(R));
  for (int64_t i = 0; i < n; ++i) Q[i + i * n] = 1;
  R* v = (R*)xcalloc((size_t)n, sizeof(R));
  R* p = (R*)xcalloc((size_t)n, sizeof(R));
  R* w = (R*)xcalloc((size_t)n, sizeof(R));
  R* u = (R*)xcalloc((size_t)n, sizeof(R));
  for (int64_t k = 0; k + 2 < n; ++k) {
    const int64_t len = n - k - 1;
    R nrm2 = 0;
    for (int64_t i = 0; i < len; ++i) {
      const R a = (R)fabs((double)W[k + 1 + i + k * n]);
      nrm2 += a * a;
    }
    const R nrm = (R)sqrt((double)nrm2);
    if (nrm == 0) continue;
    const R x0 = W[k + 1 + k * n];
    const R ax0 = (R)fabs((double)x0);
    const R phase = ax0 > 0 ? x0 / ax0 : (R)1;
    const R alpha = -phase * nrm;
    v[0] = x0 + phase * nrm;
    for (int64_t i = 1; i < len; ++i) v[i] = W[k + 1 + i + k * n];
    R vn2 = 0;
    for (int64_t i = 0; i < len; ++i) {
      const R a = (R)fabs((double)v[i]);
      vn2 += a * a;
    }
    const R beta = (R)2 / vn2;
    for (int64_t i = 0; i < len; ++i) p[i] = 0;
    for (int64_t j = 0; j < len; ++j) {
      const R vj = v[j];
      for (int64_t i = 0; i < len; ++i) p[i] += W[k + 1 + i + (k + 1 + j) * n] * vj;
    }
    for (int64_t i = 0; i < len; ++i) p[i] *= beta;
    R vtp = 0;
    for (int64_t i = 0; i < len; ++i) vtp += v[i] * p[i];
    const R kappa = beta * vtp / (R)2;
    for (int64_t i = 0; i < len; ++i) w[i] = p[i] - kappa * v[i];
    for (int64_t j = 0; j < len; ++j)
      for (int64_t i = 0; i < len; ++i)
        W[k + 1 + i + (k + 1 + j) * n] -= v[i] * w[j] + w[i] * v[j];
    W[k + 1 + k * n] = alpha;
    W[k + (k + 1) * n] = alpha;
    for (int64_t i = 2; i <= len; ++i) {
      W[k + i + k * n] = 0;
      W[k + (k + i) * n] = 0;
    }
    for (int64_t r = 0; r < n; ++r) u[r] = 0;
    for (int64_t j = 0; j < len; ++j) {
      const R vj = v[j];
      const R* qj = Q + (k + 1 + j) * n;
      for (int64_t r = 0; r < n; ++r) u[r] += qj[r] * vj;
    }
    for (int64_t j = 0; j < len; ++j) {
      const R f = beta * v[j];
      R* qj = Q + (k + 1 + j) * n;
      for (int64_t r = 0; r < n; ++r) qj[r] -= u[r] * f;
    }
  }
  R* d = (R*)xcalloc((size_t)n, sizeof(R));
  R* e = (R*)xcalloc((size_t)n, sizeof(R));
  for (int64_t i = 0; i < n; ++i) d[i] = W[i + i * n];
  for (int64_t i = 1; i < n; ++i) e[i - 1] = W[i + (i - 1) * n];
  SFX(tridiag_ql)(n, d, e, Q);
  /* stable ascending sort of indices (insertion sort keeps ties in order) */
  int64_t* idx = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    const int64_t key = idx[i];
    int64_t j = i - 1;
    while (j >= 0 && d[key] < d[idx[j]]) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = key;
  }
  for (int64_t j = 0; j < n; ++j) {
    vals[j] = d[idx[j]];
    memcpy(vecs + j * n, Q + idx[j] * n, (size_t)n * sizeof(R));
  }
  free(idx);
  free(d);
  free(e);
  free(W);
  free(Q);
  free(v);
  free(p);
  free(w);
  free(u);
}
#else
/* Sensitivity build only (tests/golden/make_sensitivity.py, -DMPORC_EIG_JACOBI):
 * the same eigendecomposition by cyclic two-sided Jacobi -- a different,
 * equally valid small symmetric eigensolver -- to measure how the reference
 * algorithm's iteration counts react to the rounding of the Rayleigh-Ritz
 * eigenvectors.  Not the reference's algorithm; never used for parity. */
static void SFX(small_herm_eig)(int64_t n, const R* M, R* vals, R* vecs) {
  if (n == 0) return;
  R* W = (R*)xmalloc((size_t)(n * n) * sizeof(R));
  R* V = (R*)xcalloc((size_t)(n * n), sizeof(R));
  for (int64_t j = 0; j < n; ++j) {
    V[j + j * n] = 1;
    for (int64_t i = 0; i < n; ++i) W[i + j * n] = (M[i + j * n] + M[j + i * n]) / (R)2;
  }
  const R eps = sizeof(R) == 8 ? (R)DBL_EPSILON : (R)FLT_EPSILON;
  for (int sweep = 0; sweep < 60; ++sweep) {
    R off = 0, tot = 0;
    for (int64_t j = 0; j < n; ++j)
      for (int64_t i = 0; i < n; ++i) {
        const R a = W[i + j * n] * W[i + j * n];
        tot += a;
        if (i != j) off += a;
      }
    if (off <= eps * eps * tot) break;
    for (int64_t p = 0; p + 1 < n; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        const R apq = W[p + q * n];
        if (apq == 0) continue;
        const R th = (W[q + q * n] - W[p + p * n]) / (2 * apq);
        const R t = (th >= 0 ? (R)1 : (R)-1) / ((R)fabs((double)th) + (R)sqrt((double)(th * th + 1)));
        const R c = (R)1 / (R)sqrt((double)(t * t + 1)), sn = t * c;
        for (int64_t k = 0; k < n; ++k) { /* columns p, q */
          const R wp = W[k + p * n], wq = W[k + q * n];
          W[k + p * n] = c * wp - sn * wq;
          W[k + q * n] = sn * wp + c * wq;
        }
        for (int64_t k = 0; k < n; ++k) { /* rows p, q */
          const R wp = W[p + k * n], wq = W[q + k * n];
          W[p + k * n] = c * wp - sn * wq;
          W[q + k * n] = sn * wp + c * wq;
        }
        for (int64_t k = 0; k < n; ++k) {
          const R vp = V[k + p * n], vq = V[k + q * n];
          V[k + p * n] = c * vp - sn * vq;
          V[k + q * n] = sn * vp + c * vq;
        }
      }
  }
  int64_t* idx = (int64_t*)xmalloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) idx[i] = i;
  for (int64_t i = 1; i < n; ++i) {
    const int64_t key = idx[i];
    int64_t j = i - 1;
    while (j >= 0 && W[key + key * n] < W[idx[j] + idx[j] * n]) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = key;
  }
  for (int64_t j = 0; j < n; ++j) {
    vals[j] = W[idx[j] + idx[j] * n];
    memcpy(vecs + j * n, V + idx[j] * n, (size_t)n * sizeof(R));
  }
  free(idx);
  free(W);
  free(V);
}
#endif

/* ---- Hetmaniuk-Lehoucq update (eigensolvers.hpp:148-174) ------------------- */
/* coefficients only: cx = C(:,0:m) (s x m), cpv = C(:,m:m+p) V (s x p) */
static int SFX(hl_coeffs)(int64_t s, int64_t m, const R* Cm, R* cx, R* cpv, int64_t* p_out) {
  const int64_t p = m < s - m ? m : s - m;
  memcpy(cx, Cm, (size_t)(s * m) * sizeof(R));
  *p_out = p;
  int fallback = 0;
  if (p > 0) {
    const R* cp = Cm + m * s;
    R* topT = (R*)xmalloc((size_t)(p * m) * sizeof(R)); /* p x m = top^T */
    for (int64_t a = 0; a < p; ++a)
      for (int64_t b = 0; b < m; ++b) topT[a + b * p] = cp[b + a * s];
    R* Qs = (R*)xmalloc((size_t)(p * p) * sizeof(R));
    orc_try t;
    ORC_TRY(t) {
      SFX(householder_qr_square)(p, m, topT, Qs);
      R* prod = SFX(matmul)(s, p, p, cp, Qs);
      memcpy(cpv, prod, (size_t)(s * p) * sizeof(R));
      free(prod);
      ORC_TRY_END(t);
    }
    else {
      ORC_CATCH_POP();
      if (t.code != MP_E_RANK_DEFICIENT) orc_throw(t.code, t.idx);
      fallback = 1;
      memcpy(cpv, cp, (size_t)(s * p) * sizeof(R));
    }
    free(topT);
    free(Qs);
  }
  return fallback;
}

/* ---- operators (sparse_kernels.hpp:16-33 and the harness stencil) ---------- */
typedef struct {
  int kind;
  int64_t n, nx, ny, nz;
  const int64_t* rp;
  const int64_t* ci;
  const R* v;   /* CSR values in this precision */
  const R* D;   /* dense n x n in this precision */
} SFX(op_t);

static void SFX(op_apply)(const SFX(op_t) * A, int64_t c, const R* X, R* Y) {
  const int64_t n = A->n;
  for (int64_t j = 0; j < c; ++j) {
    const R* x = X + j * n;
    R* y = Y + j * n;
    if (A->kind == MP_PROB_LAP3D || A->kind == MP_PROB_LAP2D) {
      const int64_t sy = A->nx, sz = A->nx * A->ny;
      const R diag = A->kind == MP_PROB_LAP3D ? (R)6 : (R)4;
      for (int64_t p = 0; p < n; ++p) {
        const int64_t xi = p % A->nx, yi = (p / A->nx) % A->ny, zi = p / sz;
        R s = 0;
        if (A->kind == MP_PROB_LAP3D && zi > 0) s += (R)-1 * x[p - sz];
        if (yi > 0) s += (R)-1 * x[p - sy];
        if (xi > 0) s += (R)-1 * x[p - 1];
        s += diag * x[p];
        if (xi + 1 < A->nx) s += (R)-1 * x[p + 1];
        if (yi + 1 < A->ny) s += (R)-1 * x[p + sy];
        if (A->kind == MP_PROB_LAP3D && zi + 1 < A->nz) s += (R)-1 * x[p + sz];
        y[p] = s;
      }
    } else if (A->kind == MP_PROB_CSR) {
      for (int64_t i = 0; i < n; ++i) {
        R s = 0;
        for (int64_t q = A->rp[i]; q < A->rp[i + 1]; ++q) s += A->v[q] * x[A->ci[q]];
        y[i] = s;
      }
    } else {
      /* herm_product -> matmul, axpy order */
      for (int64_t i = 0; i < n; ++i) y[i] = 0;
      for (int64_t l = 0; l < n; ++l) {
        const R b = x[l];
        const R* al = A->D + l * n;
        for (int64_t i = 0; i < n; ++i) y[i] += al[i] * b;
      }
    }
  }
}

/* Jacobi f_T restated from the harness (Preconditioner::apply shape) */
typedef struct {
  int mode;            /* 0: R .* dinv (this precision); 1: sandwich (R = double only) */
  const R* dinv;
  const float* dinvf;
} SFX(prec_t);

static void SFX(prec_apply)(const SFX(prec_t) * P, int64_t n, int64_t c, const R* Rm, R* W) {
  for (int64_t j = 0; j < c; ++j)
    for (int64_t i = 0; i < n; ++i) {
      const R r = Rm[i + j * n];
      if (P->mode == 0) {
        W[i + j * n] = r * P->dinv[i];
      } else {
        const float rl = to_lower_checked((double)r);
        W[i + j * n] = (R)(rl * P->dinvf[i]);
      }
    }
}

/* converged_count (eigensolvers.hpp:25-43) */
static int64_t SFX(converged_count)(int64_t n, int64_t m, double a_norm_est, const R* X,
                                    const R* theta, const R* Rm, double tol) {
  int64_t n_c = 0;
  for (int64_t j = 0; j < m; ++j) {
    const double rn = (double)SFX(col_norm)(n, Rm + j * n);
    const double xn = (double)SFX(col_norm)(n, X + j * n);
    const double thr = tol * (a_norm_est + fabs((double)theta[j])) * xn;
    if (rn <= thr)
      ++n_c;
    else
      break;
  }
  return n_c;
}

/* ritz_rotate (eigensolvers.hpp:89-102): X <- X V, AX <- AX V, theta */
static void SFX(ritz_rotate)(int64_t n, int64_t m, R* X, R* AX, R* theta) {
  R* Th = SFX(adjoint_matmul)(n, m, m, X, AX);
  SFX(hermitize)(m, Th);
  R* V = (R*)xmalloc((size_t)(m * m) * sizeof(R));
  SFX(small_herm_eig)(m, Th, theta, V);
  R* X2 = SFX(matmul)(n, m, m, X, V);
  R* A2 = SFX(matmul)(n, m, m, AX, V);
  memcpy(X, X2, (size_t)(n * m) * sizeof(R));
  memcpy(AX, A2, (size_t)(n * m) * sizeof(R));
  free(X2);
  free(A2);
  free(V);
  free(Th);
}

/* residual_block (eigensolvers.hpp:104-115) */
static R* SFX(residual_block)(int64_t n, int64_t m, const R* AX, const R* X, const R* theta) {
  R* Rm = (R*)xmalloc((size_t)(n * m) * sizeof(R));
  memcpy(Rm, AX, (size_t)(n * m) * sizeof(R));
  for (int64_t j = 0; j < m; ++j) {
    const R th = theta[j];
    for (int64_t i = 0; i < n; ++i) Rm[i + j * n] -= th * X[i + j * n];
  }
  return Rm;
}

/* record sink helper */
static void SFX(push_record)(rec_sink* h, int stage, int64_t n, int64_t m, const R* theta,
                             const R* Rm, int64_t n_c) {
  double* rv = (double*)xmalloc((size_t)m * sizeof(double));
  double* rn = (double*)xmalloc((size_t)m * sizeof(double));
  for (int64_t j = 0; j < m; ++j) {
    rv[j] = (double)theta[j];
    rn[j] = (double)SFX(col_norm)(n, Rm + j * n);
  }
  sink_push(h, stage, m, rv, rn, n_c);
  free(rv);
  free(rn);
}
