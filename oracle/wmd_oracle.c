/*
 * wmd_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded FP64 CPU implementation of the paper's
 * Sinkhorn-WMD computation (arXiv 2005.06727, Algorithm 1, and
 * the Python walk-through PAPER.md:98 / Table 1). It is the
 * correctness oracle for the CUDA path in paper_2005_06727_b200/ and shares no
 * code, header, table or constant with it. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Deliberately naive: no blocking, no fusion, no reordering beyond what the
 * paper's formulas state; no rescaling of K (plain exp(-lambda*M) in FP64);
 * IEEE round-to-nearest, built without -ffast-math.
 *
 * Inputs are the FP32 arrays the GPU path sees, upcast exactly to double.
 * Parity status of each function: see oracle/__init__.py header and DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_ARG 1
#define ORC_ERR_INDEX 2
#define ORC_ERR_DUP 3
#define ORC_ERR_OOM 4

/* m(i,k) = sqrt(sum_t (E[i,t]-E[k,t])^2)  — PAPER.md:98 ("m(i,j) = sqrt(sum(pow(embedding[i]
 * - embedding[j], 2)))"), Table 1 line "M = cdist(vecs[sel], vecs)".
 * Sequential sum over t ascending, FP64. */
static double euclid(const float* a, const float* b, int32_t d) {
  double s = 0.0;
  for (int32_t t = 0; t < d; ++t) {
    double diff = (double)a[t] - (double)b[t];
    s += diff * diff;
  }
  return sqrt(s);
}

/* M (v_r x V, row-major) for query rows sel[0..v_r). */
int oracle_euclidean_rows(const float* E, int64_t V, int32_t d, const int32_t* sel, int32_t v_r,
                          double* M) {
  if (!E || !sel || !M || V < 1 || d < 1 || v_r < 1) return ORC_ERR_ARG;
  for (int32_t i = 0; i < v_r; ++i) {
    if (sel[i] < 0 || sel[i] >= V) return ORC_ERR_INDEX;
    for (int64_t k = 0; k < V; ++k) M[(int64_t)i * V + k] = euclid(E + (int64_t)sel[i] * d, E + k * d, d);
  }
  return ORC_OK;
}

/* Algorithm 1 line 1 (Table 1): I = (r > 0); r = r(I).
 * The query arrives as (id, weight) pairs; we scatter it into the dense V-vector r the paper
 * uses, then select its nonzero entries in ascending vocabulary order. */
int oracle_select_nonzero(int64_t V, const int32_t* ids, const float* w, int32_t n,
                          int32_t* sel, double* r, int32_t* v_r) {
  if (!ids || !w || !sel || !r || !v_r || V < 1 || n < 1) return ORC_ERR_ARG;
  double* dense = (double*)calloc((size_t)V, sizeof(double));
  unsigned char* seen = (unsigned char*)calloc((size_t)V, 1);
  if (!dense || !seen) { free(dense); free(seen); return ORC_ERR_OOM; }
  int rc = ORC_OK;
  for (int32_t q = 0; q < n; ++q) {
    if (ids[q] < 0 || ids[q] >= V) { rc = ORC_ERR_INDEX; break; }
    if (seen[ids[q]]) { rc = ORC_ERR_DUP; break; }
    seen[ids[q]] = 1;
    dense[ids[q]] = (double)w[q];
  }
  int32_t m = 0;
  if (rc == ORC_OK)
    for (int64_t k = 0; k < V; ++k)
      if (dense[k] > 0.0) { sel[m] = (int32_t)k; r[m] = dense[k]; ++m; }
  *v_r = m;
  free(dense); free(seen);
  return rc;
}

/*
 * Sinkhorn-Knopp WMD of one query against N target documents (Algorithm 1):
 *
 *   I=(r>0); r=r(I); M=M(I,:); K=exp(-lambda*M)                  [PAPER.md:58, Table 1 :116-122]
 *   x = ones(v_r, N)/v_r                                           [PAPER.md:59, :121]
 *   while it < max_iter (and, if tol >= 0, while x changes by > tol):  [PAPER.md:60, :125]
 *       u = 1./x                                                   [:126]
 *       v = c .* (1./(K^T u))        (only where c != 0)          [:62, :128; "c.multiply"]
 *       x = diag(1./r) K v           (p = (1/r)*K precomputed)     [:62, :123, :130]
 *   u = 1./x; v = c .* (1./(K^T u))                                [:64, :132-133]
 *   WMD = sum_i u .* ((K.*M) v)       (sum over query rows)        [:66, :134]
 *
 * dense != 0: K^T u is evaluated for ALL V vocabulary rows (the Python form),
 *             then masked by c's support (c.multiply never forms 0*inf).
 * dense == 0: the SDDMM form: the dot product only where c is nonzero.
 *
 * Iteration semantics: max_iter counts x-updates (Table 1, `while it < max_iter`). If
 * tol >= 0 the loop also stops once max |x_new - x_old| over ALL entries of the v_r x N
 * matrix x is <= tol (the paper's "While x changes", read matrix-wide).
 *
 * Layout: c is CSC of the V x N matrix (col_ptr[N+1], row_idx[nnz], val[nnz]).
 * Outputs: wmd[N]; optional u_out (N x v_r, doc-major: u_out[j*v_r+i]) = final u;
 * optional v_out[nnz] = final v at c's support; optional iters_run (scalar).
 */
int oracle_sinkhorn(int dense, const float* E, int64_t V, int32_t d,
                    const int64_t* col_ptr, const int32_t* row_idx, const float* val, int64_t N,
                    const int32_t* q_ids, const float* q_w, int32_t nq,
                    double lambda, int32_t max_iter, double tol,
                    double* wmd, double* u_out, double* v_out, int32_t* iters_run) {
  if (!E || !col_ptr || !row_idx || !val || !q_ids || !q_w || !wmd) return ORC_ERR_ARG;
  if (V < 1 || d < 1 || N < 1 || nq < 1 || max_iter < 0 || !(lambda > 0.0)) return ORC_ERR_ARG;
  const int64_t nnz = col_ptr[N];
  for (int64_t e = 0; e < nnz; ++e)
    if (row_idx[e] < 0 || row_idx[e] >= V) return ORC_ERR_INDEX;

  int rc = ORC_OK;
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (size_t)nq);
  double* r = (double*)malloc(sizeof(double) * (size_t)nq);
  int32_t v_r = 0;
  if (!sel || !r) { free(sel); free(r); return ORC_ERR_OOM; }
  rc = oracle_select_nonzero(V, q_ids, q_w, nq, sel, r, &v_r);
  if (rc != ORC_OK || v_r < 1) { free(sel); free(r); return rc != ORC_OK ? rc : ORC_ERR_ARG; }

  /* M = M(I,:) (lazily: only the v_r query rows). For the sparse form only the
   * vocabulary columns that c references are needed; each computed column is identical. */
  unsigned char* need = (unsigned char*)calloc((size_t)V, 1);
  double* M = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)V);
  double* K = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)V);
  double* p = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)V);   /* K_over_r */
  double* KM = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)V);  /* K .* M  */
  double* x = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)N);   /* doc-major */
  double* xn = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)N);
  double* u = (double*)malloc(sizeof(double) * (size_t)v_r);
  double* T = (double*)malloc(sizeof(double) * (size_t)V);                 /* K^T u (dense) */
  double* v = (double*)malloc(sizeof(double) * (size_t)(nnz > 0 ? nnz : 1));
  if (!need || !M || !K || !p || !KM || !x || !xn || !u || !T || !v) { rc = ORC_ERR_OOM; goto done; }

  if (dense) memset(need, 1, (size_t)V);
  else for (int64_t e = 0; e < nnz; ++e) need[row_idx[e]] = 1;
  for (int32_t i = 0; i < v_r; ++i)
    for (int64_t k = 0; k < V; ++k) {
      double m = need[k] ? euclid(E + (int64_t)sel[i] * d, E + k * d, d) : 0.0;
      double kk = exp(-lambda * m);                       /* K = np.exp(- M * lamb), :122 */
      M[(int64_t)i * V + k] = m;
      K[(int64_t)i * V + k] = kk;
      p[(int64_t)i * V + k] = (1.0 / r[i]) * kk;          /* p = (1 / r) * K, :123 */
      KM[(int64_t)i * V + k] = kk * m;                    /* (K * M), :134 */
    }

  for (int64_t q = 0; q < (int64_t)v_r * N; ++q) x[q] = 1.0 / (double)v_r;   /* :121 */

  int32_t it = 0;
  for (; it < max_iter; ++it) {
    double change = 0.0;
    for (int64_t j = 0; j < N; ++j) {
      const int64_t b = col_ptr[j], en = col_ptr[j + 1];
      double* xj = x + j * v_r;
      double* xnj = xn + j * v_r;
      for (int32_t i = 0; i < v_r; ++i) u[i] = 1.0 / xj[i];               /* u = 1.0 / x */
      if (dense) {
        for (int64_t k = 0; k < V; ++k) {                                   /* KT @ u, all rows */
          double s = 0.0;
          for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * V + k] * u[i];
          T[k] = s;
        }
        for (int64_t e = b; e < en; ++e) v[e] = (double)val[e] * (1.0 / T[row_idx[e]]);  /* c.multiply(1/.) */
      } else {
        for (int64_t e = b; e < en; ++e) {                                  /* SDDMM */
          const int64_t k = row_idx[e];
          double s = 0.0;
          for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * V + k] * u[i];
          v[e] = (double)val[e] * (1.0 / s);
        }
      }
      for (int32_t i = 0; i < v_r; ++i) {                                   /* x = K_over_r @ v */
        double s = 0.0;
        for (int64_t e = b; e < en; ++e) s += p[(int64_t)i * V + row_idx[e]] * v[e];
        xnj[i] = s;
        double dc = fabs(s - xj[i]);
        if (dc > change || isnan(dc)) change = isnan(dc) ? INFINITY : (dc > change ? dc : change);
      }
    }
    double* t = x; x = xn; xn = t;
    if (tol >= 0.0 && change <= tol) { ++it; break; }
  }
  if (iters_run) *iters_run = it;

  /* Final step: u = 1./x; v = c.*(1./(K^T u)); WMD = sum(u .* ((K.*M) v)) */
  for (int64_t j = 0; j < N; ++j) {
    const int64_t b = col_ptr[j], en = col_ptr[j + 1];
    const double* xj = x + j * v_r;
    for (int32_t i = 0; i < v_r; ++i) u[i] = 1.0 / xj[i];
    if (dense) {
      for (int64_t k = 0; k < V; ++k) {
        double s = 0.0;
        for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * V + k] * u[i];
        T[k] = s;
      }
      for (int64_t e = b; e < en; ++e) v[e] = (double)val[e] * (1.0 / T[row_idx[e]]);
    } else {
      for (int64_t e = b; e < en; ++e) {
        const int64_t k = row_idx[e];
        double s = 0.0;
        for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * V + k] * u[i];
        v[e] = (double)val[e] * (1.0 / s);
      }
    }
    double w = 0.0;
    for (int32_t i = 0; i < v_r; ++i) {
      double s = 0.0;
      for (int64_t e = b; e < en; ++e) s += KM[(int64_t)i * V + row_idx[e]] * v[e];
      w += u[i] * s;
    }
    wmd[j] = w;
    if (u_out) for (int32_t i = 0; i < v_r; ++i) u_out[j * v_r + i] = u[i];
    if (v_out) for (int64_t e = b; e < en; ++e) v_out[e] = v[e];
  }

done:
  free(need); free(M); free(K); free(p); free(KM); free(x); free(xn); free(u); free(T); free(v);
  free(sel); free(r);
  return rc;
}

/* "While x changes" per document (Algorithm 1 l.3).
 * The same sparse Algorithm 1 as oracle_sinkhorn (dense = 0), but each document j stops on its
 * own: after the first x-update t (1 <= t <= max_iter) with
 *        max_i | xnew_ij / x_ij - 1 |  <= tol_rel,
 * i.e. x no longer changes relative to itself (reading R31: the paper gives no
 * tolerance; a relative test is scale free, so the GPU can evaluate it on gauged iterates),
 * or after max_iter updates. tol_rel < 0 never stops early (= oracle_sinkhorn, fixed iters).
 * Then the final step of l.6-7. Documents are independent, so the loop runs
 * document by document. iters_doc[j] (optional) receives the number of x-updates of doc j. */
int oracle_sinkhorn_per_doc(const float* E, int64_t V, int32_t d, const int64_t* col_ptr,
                            const int32_t* row_idx, const float* val, int64_t N,
                            const int32_t* q_ids, const float* q_w, int32_t nq, double lambda,
                            int32_t max_iter, double tol_rel, double* wmd, int32_t* iters_doc) {
  if (!E || !col_ptr || !row_idx || !val || !q_ids || !q_w || !wmd) return ORC_ERR_ARG;
  if (V < 1 || d < 1 || N < 1 || nq < 1 || max_iter < 0 || !(lambda > 0.0)) return ORC_ERR_ARG;
  const int64_t nnz = col_ptr[N];
  for (int64_t e = 0; e < nnz; ++e)
    if (row_idx[e] < 0 || row_idx[e] >= V) return ORC_ERR_INDEX;
  int rc = ORC_OK;
  int32_t* sel = (int32_t*)malloc(sizeof(int32_t) * (size_t)nq);
  double* r = (double*)malloc(sizeof(double) * (size_t)nq);
  int32_t v_r = 0;
  if (!sel || !r) { free(sel); free(r); return ORC_ERR_OOM; }
  rc = oracle_select_nonzero(V, q_ids, q_w, nq, sel, r, &v_r);
  if (rc != ORC_OK || v_r < 1) { free(sel); free(r); return rc != ORC_OK ? rc : ORC_ERR_ARG; }
  int64_t maxlen = 1;
  for (int64_t j = 0; j < N; ++j)
    if (col_ptr[j + 1] - col_ptr[j] > maxlen) maxlen = col_ptr[j + 1] - col_ptr[j];
  double* M = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)maxlen);  /* doc block */
  double* K = (double*)malloc(sizeof(double) * (size_t)v_r * (size_t)maxlen);
  double* x = (double*)malloc(sizeof(double) * (size_t)v_r);
  double* xn = (double*)malloc(sizeof(double) * (size_t)v_r);
  double* u = (double*)malloc(sizeof(double) * (size_t)v_r);
  double* v = (double*)malloc(sizeof(double) * (size_t)maxlen);
  if (!M || !K || !x || !xn || !u || !v) { rc = ORC_ERR_OOM; goto done2; }
  for (int64_t j = 0; j < N; ++j) {
    const int64_t b = col_ptr[j], n = col_ptr[j + 1] - b;
    for (int32_t i = 0; i < v_r; ++i)                    /* M(I, words of j), K = exp(-lambda M) */
      for (int64_t e = 0; e < n; ++e) {
        const double m = euclid(E + (int64_t)sel[i] * d, E + (int64_t)row_idx[b + e] * d, d);
        M[(int64_t)i * n + e] = m;
        K[(int64_t)i * n + e] = exp(-lambda * m);
      }
    for (int32_t i = 0; i < v_r; ++i) x[i] = 1.0 / (double)v_r;             /* :121 */
    int32_t it = 0;
    while (it < max_iter) {
      for (int32_t i = 0; i < v_r; ++i) u[i] = 1.0 / x[i];                   /* u = 1.0 / x */
      for (int64_t e = 0; e < n; ++e) {                                       /* SDDMM */
        double s = 0.0;
        for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * n + e] * u[i];
        v[e] = (double)val[b + e] * (1.0 / s);
      }
      double change = 0.0;
      for (int32_t i = 0; i < v_r; ++i) {                                     /* x = diag(1/r) K v */
        double s = 0.0;
        for (int64_t e = 0; e < n; ++e) s += ((1.0 / r[i]) * K[(int64_t)i * n + e]) * v[e];
        xn[i] = s;
        const double rc_ = fabs(s / x[i] - 1.0);
        change = (rc_ > change || isnan(rc_)) ? (isnan(rc_) ? INFINITY : rc_) : change;
      }
      for (int32_t i = 0; i < v_r; ++i) x[i] = xn[i];
      ++it;
      if (tol_rel >= 0.0 && change <= tol_rel) break;
    }
    if (iters_doc) iters_doc[j] = it;
    for (int32_t i = 0; i < v_r; ++i) u[i] = 1.0 / x[i];                     /* final step */
    for (int64_t e = 0; e < n; ++e) {
      double s = 0.0;
      for (int32_t i = 0; i < v_r; ++i) s += K[(int64_t)i * n + e] * u[i];
      v[e] = (double)val[b + e] * (1.0 / s);
    }
    double w = 0.0;
    for (int32_t i = 0; i < v_r; ++i) {
      double s = 0.0;
      for (int64_t e = 0; e < n; ++e) s += (K[(int64_t)i * n + e] * M[(int64_t)i * n + e]) * v[e];
      w += u[i] * s;
    }
    wmd[j] = w;
  }
done2:
  free(M); free(K); free(x); free(xn); free(u); free(v); free(sel); free(r);
  return rc;
}

/* nnz-balanced document partition ("divided the number of non-zeros in c evenly
 * among the threads and each thread ... determines its starting exploration point inside the
 * CSR using a binary search"), snapped to document boundaries: worker g starts
 * at the first document j with col_ptr[j] >= ceil(g*nnz/P). Written as a plain linear scan. */
int oracle_partition(const int64_t* col_ptr, int64_t N, int32_t P, int64_t* bounds) {
  if (!col_ptr || !bounds || N < 0 || P < 1) return ORC_ERR_ARG;
  const int64_t nnz = col_ptr[N];
  bounds[0] = 0;
  int64_t j = 0;
  for (int32_t g = 1; g < P; ++g) {
    const int64_t target = (g * nnz + P - 1) / P;   /* ceil(g*nnz/P) */
    while (j < N && col_ptr[j] < target) ++j;
    bounds[g] = j;
  }
  bounds[P] = N;
  return ORC_OK;
}
