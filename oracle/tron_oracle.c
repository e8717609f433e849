/*
 * TEST INFRASTRUCTURE ONLY -- see tron_oracle.h.  Plain-C restatement of the
 * reference TRON hot path; each function cites the reference lines it
 * follows (paths relative to /root/reference/proj).  Compile with
 * -ffp-contract=off: the reference's x86-64 build emits no FMA.
 */
#include "tron_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define NB OR_REDUCTION_BLOCKS

/* parallel.hpp:32-34 reduction_block */
static void block_range(size_t len, size_t b, size_t *begin, size_t *end) {
  *begin = len * b / NB;
  *end = len * (b + 1) / NB;
}

/* parallel.hpp:91-98 merge_scalar_tree */
static double merge_scalar_tree(double *s) {
  for (size_t stride = 1; stride < NB; stride *= 2)
    for (size_t i = 0; i + stride < NB; i += 2 * stride) s[i] += s[i + stride];
  return s[0];
}

/* parallel.hpp:101-109 merge_vector_tree */
static void merge_vector_tree(double *partials, size_t n) {
  for (size_t stride = 1; stride < NB; stride *= 2)
    for (size_t i = 0; i + stride < NB; i += 2 * stride) {
      double *dst = partials + i * n;
      const double *src = partials + (i + stride) * n;
      for (size_t j = 0; j < n; ++j) dst[j] += src[j];
    }
}

void or_default_config(or_config *c) { /* tron.hpp:13-27 */
  c->eps = 0.1;
  c->max_outer_iters = 1000;
  c->max_cg_iters = 0;
  c->sigma0 = 1e-4;
  c->eta1 = 0.25;
  c->eta2 = 0.75;
  c->gamma1 = 0.25;
  c->gamma2 = 0.5;
  c->gamma3 = 4.0;
  c->cg_tol = 0.1;
  c->use_preconditioner = 0;
}

/* linalg.cpp:75-86 FeatureMatrix::row_dot */
static double row_dot(const or_matrix *X, size_t i, const double *v) {
  double acc = 0.0;
  if (X->layout == OR_DENSE_ROW_MAJOR) {
    const double *row = X->values + i * X->cols;
    for (size_t j = 0; j < X->cols; ++j) acc += row[j] * v[j];
  } else {
    for (int64_t k = X->row_offsets[i]; k < X->row_offsets[i + 1]; ++k)
      acc += X->values[k] * v[X->col_indices[k]];
  }
  return acc;
}

/* linalg.cpp:88-97 FeatureMatrix::row_axpy */
static void row_axpy(const or_matrix *X, size_t i, double a, double *out) {
  if (X->layout == OR_DENSE_ROW_MAJOR) {
    const double *row = X->values + i * X->cols;
    for (size_t j = 0; j < X->cols; ++j) out[j] += a * row[j];
  } else {
    for (int64_t k = X->row_offsets[i]; k < X->row_offsets[i + 1]; ++k)
      out[X->col_indices[k]] += a * X->values[k];
  }
}

/* linalg.cpp:99-109 FeatureMatrix::row_axpy_squared: out_j += a*v*v */
static void row_axpy_squared(const or_matrix *X, size_t i, double a, double *out) {
  if (X->layout == OR_DENSE_ROW_MAJOR) {
    const double *row = X->values + i * X->cols;
    for (size_t j = 0; j < X->cols; ++j) out[j] += a * row[j] * row[j];
  } else {
    for (int64_t k = X->row_offsets[i]; k < X->row_offsets[i + 1]; ++k) {
      double v = X->values[k];
      out[X->col_indices[k]] += a * v * v;
    }
  }
}

/* linalg.cpp:154-162 matvec (64 row blocks; any order is bit-identical) */
void or_matvec(const or_matrix *X, const double *v, double *out) {
  for (size_t i = 0; i < X->rows; ++i) out[i] = row_dot(X, i, v);
}

/* The scatter flavours of linalg.cpp:175-184 blocked_column_accumulate. */
enum { ACC_ALL_AXPY, ACC_MASKED_AXPY, ACC_ALL_SQ, ACC_MASKED_SQ, ACC_MASKED_HV };

static int blocked_column_accumulate(const or_matrix *X, int kind, const int64_t *I, size_t nI,
                                     const double *u, double *out) {
  const size_t n = X->cols;
  double *partials = (double *)calloc(NB * (n ? n : 1), sizeof(double));
  if (!partials) return OR_ERR_ALLOC;
  const size_t len = (kind == ACC_ALL_AXPY || kind == ACC_ALL_SQ) ? X->rows : nI;
  for (size_t b = 0; b < NB; ++b) {
    size_t begin, end;
    block_range(len, b, &begin, &end);
    double *buf = partials + b * n;
    for (size_t k = begin; k < end; ++k) {
      switch (kind) {
        case ACC_ALL_AXPY: row_axpy(X, k, u[k], buf); break;            /* linalg.cpp:191-194 */
        case ACC_MASKED_AXPY: row_axpy(X, (size_t)I[k], u[I[k]], buf); break; /* :239-245 */
        case ACC_ALL_SQ: row_axpy_squared(X, k, u[k], buf); break;      /* :251-254 */
        case ACC_MASKED_SQ: row_axpy_squared(X, (size_t)I[k], 1.0, buf); break; /* :259-264 */
        case ACC_MASKED_HV: {                                            /* loss.cpp:450-457 */
          size_t i = (size_t)I[k];
          row_axpy(X, i, row_dot(X, i, u), buf);
          break;
        }
      }
    }
  }
  merge_vector_tree(partials, n);
  memcpy(out, partials, n * sizeof(double));
  free(partials);
  return OR_OK;
}

int or_matvec_transpose(const or_matrix *X, const double *u, double *out) {
  return blocked_column_accumulate(X, ACC_ALL_AXPY, NULL, 0, u, out);
}

static int check_index_set(const or_matrix *X, const int64_t *I, size_t nI) {
  for (size_t k = 0; k < nI; ++k)
    if (I[k] < 0 || (size_t)I[k] >= X->rows) return OR_ERR_BOUNDS; /* linalg.cpp:234-238 */
  return OR_OK;
}

int or_masked_matvec_transpose(const or_matrix *X, const int64_t *I, size_t nI, const double *u,
                               double *out) {
  int st = check_index_set(X, I, nI);
  if (st) return st;
  return blocked_column_accumulate(X, ACC_MASKED_AXPY, I, nI, u, out);
}

int or_weighted_sq_col_sums(const or_matrix *X, const double *weights, double *out) {
  return blocked_column_accumulate(X, ACC_ALL_SQ, NULL, 0, weights, out);
}

int or_masked_sq_col_sums(const or_matrix *X, const int64_t *I, size_t nI, double *out) {
  return blocked_column_accumulate(X, ACC_MASKED_SQ, I, nI, NULL, out);
}

/* linalg.cpp:267-286 serial vector ops */
double or_dot(const double *a, const double *b, size_t n) {
  double acc = 0.0;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}
double or_norm2(const double *a, size_t n) { return sqrt(or_dot(a, a, n)); }
static void axpy_inplace(double alpha, const double *a, double *b, size_t n) {
  for (size_t i = 0; i < n; ++i) b[i] += alpha * a[i];
}

/* parallel.cpp:91-100 reduce_sum */
double or_reduce_sum(const double *v, size_t len) {
  double s[NB];
  for (size_t b = 0; b < NB; ++b) {
    size_t begin, end;
    block_range(len, b, &begin, &end);
    double acc = 0.0;
    for (size_t i = begin; i < end; ++i) acc += v[i];
    s[b] = acc;
  }
  return merge_scalar_tree(s);
}

/* loss.hpp:99-102 detail::log1p_exp_neg */
double or_log1p_exp_neg(double t) {
  if (t >= 0.0) return log1p(exp(-t));
  return -t + log1p(exp(t));
}

/* loss.cpp:35-58 logistic_fused_pass; returns f */
double or_logistic_fused_pass(const or_problem *p, const double *w, double *z, double *zhat,
                              double *dvec, double *alpha) {
  const size_t l = p->X.rows;
  or_matvec(&p->X, w, z);
  for (size_t i = 0; i < l; ++i) {
    double t = p->y[i] * z[i];
    double sig = 1.0 / (1.0 + exp(t)); /* exp overflow -> inf -> 0 */
    zhat[i] = -p->y[i] * sig;
    dvec[i] = (1.0 - sig) * sig;
    alpha[i] = or_log1p_exp_neg(t);
  }
  return 0.5 * or_dot(w, w, p->X.cols) + p->C * or_reduce_sum(alpha, l);
}

/* loss.cpp:60-72 logistic_objective */
double or_logistic_objective(const or_problem *p, const double *w) {
  const size_t l = p->X.rows;
  double *z = (double *)malloc((l ? l : 1) * sizeof(double));
  double *alpha = (double *)malloc((l ? l : 1) * sizeof(double));
  or_matvec(&p->X, w, z);
  for (size_t i = 0; i < l; ++i) alpha[i] = or_log1p_exp_neg(p->y[i] * z[i]);
  double f = 0.5 * or_dot(w, w, p->X.cols) + p->C * or_reduce_sum(alpha, l);
  free(z);
  free(alpha);
  return f;
}

/* loss.cpp:74-80 logistic_gradient: g = w + C X' zhat */
int or_logistic_gradient(const or_problem *p, const double *zhat, const double *w, double *g) {
  int st = or_matvec_transpose(&p->X, zhat, g);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) g[j] = w[j] + p->C * g[j];
  return OR_OK;
}

/* loss.cpp:82-92 logistic_hessian_vec: out = v + C X'(D (X v)) */
int or_logistic_hessian_vec(const or_problem *p, const double *dvec, const double *v,
                            double *out) {
  const size_t l = p->X.rows;
  double *a0 = (double *)malloc((l ? l : 1) * sizeof(double));
  if (!a0) return OR_ERR_ALLOC;
  or_matvec(&p->X, v, a0);
  for (size_t i = 0; i < l; ++i) a0[i] *= dvec[i];
  int st = or_matvec_transpose(&p->X, a0, out);
  free(a0);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) out[j] = v[j] + p->C * out[j];
  return OR_OK;
}

/* loss.cpp:94-122 svm_fused_pass: strict active set, ascending */
double or_svm_fused_pass(const or_problem *p, const double *w, double *z, int64_t *active,
                         size_t *n_active) {
  const size_t l = p->X.rows;
  double *hinge_sq = (double *)malloc((l ? l : 1) * sizeof(double));
  or_matvec(&p->X, w, z);
  size_t count = 0;
  for (size_t i = 0; i < l; ++i) {
    double margin = 1.0 - p->y[i] * z[i];
    if (margin > 0.0) {
      active[count++] = (int64_t)i;
      hinge_sq[i] = margin * margin;
    } else {
      hinge_sq[i] = 0.0;
    }
  }
  *n_active = count;
  double f = 0.5 * or_dot(w, w, p->X.cols) + p->C * or_reduce_sum(hinge_sq, l);
  free(hinge_sq);
  return f;
}

/* loss.cpp:129-137 svm_gradient: g = w + 2C sum_{i in I} (z_i - y_i) x_i */
int or_svm_gradient(const or_problem *p, const double *z, const int64_t *active, size_t nI,
                    const double *w, double *g) {
  const size_t l = p->X.rows;
  double *residual = (double *)malloc((l ? l : 1) * sizeof(double));
  if (!residual) return OR_ERR_ALLOC;
  for (size_t i = 0; i < l; ++i) residual[i] = z[i] - p->y[i];
  int st = or_masked_matvec_transpose(&p->X, active, nI, residual, g);
  free(residual);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) g[j] = w[j] + 2.0 * p->C * g[j];
  return OR_OK;
}

/* loss.cpp:139-174 svm_hessian_vec (Indirect; Gathered is bit-identical) */
int or_svm_hessian_vec(const or_problem *p, const int64_t *active, size_t nI, const double *v,
                       double *out) {
  int st = check_index_set(&p->X, active, nI);
  if (st) return st;
  st = blocked_column_accumulate(&p->X, ACC_MASKED_HV, active, nI, v, out);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) out[j] = v[j] + 2.0 * p->C * out[j];
  return OR_OK;
}

/* loss.cpp:176-181 hessian_precond_diag (logistic): 1 + C sum d_i X_ij^2 */
int or_logistic_precond(const or_problem *p, const double *dvec, double *m) {
  int st = or_weighted_sq_col_sums(&p->X, dvec, m);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) m[j] = 1.0 + p->C * m[j];
  return OR_OK;
}

/* loss.cpp:183-188 hessian_precond_diag (L2-SVM): 1 + 2C sum_{i in I} X_ij^2 */
int or_svm_precond(const or_problem *p, const int64_t *active, size_t nI, double *m) {
  int st = or_masked_sq_col_sums(&p->X, active, nI, m);
  if (st) return st;
  for (size_t j = 0; j < p->X.cols; ++j) m[j] = 1.0 + 2.0 * p->C * m[j];
  return OR_OK;
}

/* tron.cpp:37-108 truncated_cg */
int or_truncated_cg(const double *g, size_t n, or_hv_fn hv, void *hv_ctx, double delta,
                    const double *precond, const or_config *cfg, double *d, int *exit_kind,
                    size_t *iters_out, double *model_value) {
  size_t max_iters = cfg->max_cg_iters;
  if (max_iters == 0) max_iters = n < 1000 ? n : 1000;
  size_t nn = n ? n : 1;
  double *r = (double *)malloc(nn * sizeof(double));
  double *z = (double *)malloc(nn * sizeof(double));
  double *p = (double *)malloc(nn * sizeof(double));
  double *hp = (double *)malloc(nn * sizeof(double));
  if (!r || !z || !p || !hp) {
    free(r); free(z); free(p); free(hp);
    return OR_ERR_ALLOC;
  }
  int status = OR_OK;
  int exit_k = OR_CG_CONVERGED;
  size_t iters = 0;
  for (size_t j = 0; j < n; ++j) {
    d[j] = 0.0;
    r[j] = -g[j];
  }
  for (size_t j = 0; j < n; ++j) z[j] = precond ? r[j] / precond[j] : r[j];
  memcpy(p, z, n * sizeof(double));
  double rz = or_dot(r, z, n);
  const double stop = cfg->cg_tol * or_norm2(g, n);

  while (iters < max_iters) {
    if (or_norm2(r, n) <= stop) {
      exit_k = OR_CG_CONVERGED;
      break;
    }
    ++iters;
    hv(hv_ctx, p, hp);
    double php = or_dot(p, hp, n);
    if (!(php > 0.0)) { /* tron.cpp:72-75 */
      status = OR_ERR_NUMERICAL;
      goto done;
    }
    double alpha = rz / php;
    axpy_inplace(alpha, p, d, n);
    if (or_norm2(d, n) > delta) { /* tron.cpp:78-90 boundary */
      axpy_inplace(-alpha, p, d, n);
      double dp = or_dot(d, p, n);
      double dd = or_dot(d, d, n);
      double pp = or_dot(p, p, n);
      double rad = sqrt(dp * dp + pp * (delta * delta - dd));
      double tau = dp >= 0.0 ? (delta * delta - dd) / (dp + rad) : (rad - dp) / pp;
      axpy_inplace(tau, p, d, n);
      axpy_inplace(-tau, hp, r, n);
      exit_k = OR_CG_BOUNDARY;
      break;
    }
    axpy_inplace(-alpha, hp, r, n);
    for (size_t j = 0; j < n; ++j) z[j] = precond ? r[j] / precond[j] : r[j];
    double rz_next = or_dot(r, z, n);
    double beta = rz_next / rz;
    for (size_t j = 0; j < n; ++j) p[j] = z[j] + beta * p[j];
    rz = rz_next;
    exit_k = OR_CG_MAXITERS;
  }
  /* tron.cpp:99-103 exit classification */
  if (iters >= max_iters && exit_k != OR_CG_BOUNDARY && or_norm2(r, n) > stop)
    exit_k = OR_CG_MAXITERS;
  else if (exit_k != OR_CG_BOUNDARY)
    exit_k = OR_CG_CONVERGED;
  /* tron.cpp:106 q(d) = (d'g - d'r)/2 */
  *model_value = 0.5 * (or_dot(d, g, n) - or_dot(d, r, n));
done:
  *exit_kind = exit_k;
  *iters_out = iters;
  free(r); free(z); free(p); free(hp);
  return status;
}

/* tron.cpp:110-125 trust_region_update */
void or_trust_region_update(double sigma, double delta, double step_norm, const or_config *cfg,
                            int *accept, double *next_delta) {
  *accept = sigma > cfg->sigma0;
  if (!*accept) {
    *next_delta = cfg->gamma1 * step_norm;
  } else if (sigma < cfg->eta1) {
    *next_delta = cfg->gamma2 * step_norm;
  } else if (sigma < cfg->eta2) {
    *next_delta = delta;
  } else {
    double grown = cfg->gamma3 * step_norm;
    *next_delta = grown > delta ? grown : delta;
  }
}

/* ---- evaluator: candidate/committed slots (backend.cpp:136-306) ---- */
typedef struct {
  const or_problem *p;
  int loss;
  size_t l, n;
  /* candidate slot */
  double *cz, *czhat, *cdvec, *calpha, *cw;
  int64_t *cact;
  size_t cnact;
  int cvalid;
  /* committed slot */
  double *z, *zhat, *dvec, *alpha, *w;
  int64_t *act;
  size_t nact;
  int valid;
  double *grad, *precond;
  int precond_valid;
} evaluator;

static void swap_d(double **a, double **b) { double *t = *a; *a = *b; *b = t; }

static double ev_eval_candidate(evaluator *e, const double *w) {
  double f;
  if (e->loss == OR_LOGISTIC)
    f = or_logistic_fused_pass(e->p, w, e->cz, e->czhat, e->cdvec, e->calpha);
  else
    f = or_svm_fused_pass(e->p, w, e->cz, e->cact, &e->cnact);
  memcpy(e->cw, w, e->n * sizeof(double));
  e->cvalid = 1;
  return f;
}

static int ev_commit(evaluator *e) {
  swap_d(&e->cz, &e->z);
  swap_d(&e->czhat, &e->zhat);
  swap_d(&e->cdvec, &e->dvec);
  swap_d(&e->calpha, &e->alpha);
  swap_d(&e->cw, &e->w);
  int64_t *t = e->cact; e->cact = e->act; e->act = t;
  size_t tn = e->cnact; e->cnact = e->nact; e->nact = tn;
  e->cvalid = 0;
  e->valid = 1;
  e->precond_valid = 0;
  if (e->loss == OR_LOGISTIC) return or_logistic_gradient(e->p, e->zhat, e->w, e->grad);
  return or_svm_gradient(e->p, e->z, e->act, e->nact, e->w, e->grad);
}

static void ev_hv(void *ctx, const double *v, double *out) {
  evaluator *e = (evaluator *)ctx;
  if (e->loss == OR_LOGISTIC)
    or_logistic_hessian_vec(e->p, e->dvec, v, out);
  else
    or_svm_hessian_vec(e->p, e->act, e->nact, v, out);
}

static const double *ev_precond(evaluator *e) {
  if (!e->precond_valid) {
    if (e->loss == OR_LOGISTIC)
      or_logistic_precond(e->p, e->dvec, e->precond);
    else
      or_svm_precond(e->p, e->act, e->nact, e->precond);
    e->precond_valid = 1;
  }
  return e->precond;
}

static int all_finite(const double *v, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(v[i])) return 0;
  return 1;
}

/* tron.cpp:127-217 solve */
int or_solve(const or_problem *p, int loss, const or_config *cfg, const double *w0, double *w_out,
             or_solve_info *info, or_iteration *trace, size_t trace_cap) {
  const size_t n = p->X.cols, l = p->X.rows;
  const size_t nn = n ? n : 1, ll = l ? l : 1;
  evaluator e;
  memset(&e, 0, sizeof(e));
  e.p = p;
  e.loss = loss;
  e.l = l;
  e.n = n;
  double **lvecs[] = {&e.cz, &e.czhat, &e.cdvec, &e.calpha, &e.z, &e.zhat, &e.dvec, &e.alpha};
  for (size_t k = 0; k < 8; ++k) *lvecs[k] = (double *)calloc(ll, sizeof(double));
  double **nvecs[] = {&e.cw, &e.w, &e.grad, &e.precond};
  for (size_t k = 0; k < 4; ++k) *nvecs[k] = (double *)calloc(nn, sizeof(double));
  e.cact = (int64_t *)calloc(ll, sizeof(int64_t));
  e.act = (int64_t *)calloc(ll, sizeof(int64_t));
  double *w = (double *)calloc(nn, sizeof(double));
  double *g = (double *)calloc(nn, sizeof(double));
  double *d = (double *)calloc(nn, sizeof(double));
  double *wc = (double *)calloc(nn, sizeof(double));
  memset(info, 0, sizeof(*info));
  int status = OR_OK;

  if (w0) memcpy(w, w0, n * sizeof(double));
  double f = ev_eval_candidate(&e, w);
  info->objective_evaluations = 1;
  if (!isfinite(f)) { status = OR_ERR_NUMERICAL; goto out; }
  ev_commit(&e);
  info->gradient_materializations = 1;
  memcpy(g, e.grad, n * sizeof(double));
  if (!all_finite(g, n)) { status = OR_ERR_NUMERICAL; goto out; }
  info->f_initial = f;
  const double gnorm0 = or_norm2(g, n);
  info->gradient_norm_initial = gnorm0;
  double gnorm = gnorm0;
  info->objective = f;
  if (gnorm <= cfg->eps * gnorm0) {
    info->converged = 1;
    goto out;
  }
  double delta = gnorm0;
  while (info->n_iterations < cfg->max_outer_iters) {
    const double *M = cfg->use_preconditioner ? ev_precond(&e) : NULL;
    int cg_exit;
    size_t cg_iters;
    double q;
    if (or_truncated_cg(g, n, ev_hv, &e, delta, M, cfg, d, &cg_exit, &cg_iters, &q) != OR_OK) {
      status = OR_ERR_NUMERICAL;
      goto out;
    }
    double step_norm = or_norm2(d, n);
    memcpy(wc, w, n * sizeof(double));
    axpy_inplace(1.0, d, wc, n);
    double f_cand = ev_eval_candidate(&e, wc);
    info->objective_evaluations++;
    if (!isfinite(f_cand)) { status = OR_ERR_NUMERICAL; goto out; }
    double sigma = (f_cand - f) / q;
    int accept;
    double next_delta;
    or_trust_region_update(sigma, delta, step_norm, cfg, &accept, &next_delta);
    if (trace && info->n_iterations < trace_cap) {
      or_iteration *rec = &trace[info->n_iterations];
      rec->f_candidate = f_cand;
      rec->gradient_norm = gnorm;
      rec->delta = delta;
      rec->sigma = sigma;
      rec->accepted = accept;
      rec->cg_iters = cg_iters;
      rec->cg_exit = cg_exit;
    }
    info->n_iterations++;
    delta = next_delta;
    if (accept) {
      memcpy(w, wc, n * sizeof(double));
      f = f_cand;
      info->objective = f;
      ev_commit(&e);
      info->accepted_steps++;
      info->gradient_materializations++;
      memcpy(g, e.grad, n * sizeof(double));
      if (!all_finite(g, n)) { status = OR_ERR_NUMERICAL; goto out; }
      gnorm = or_norm2(g, n);
      if (gnorm <= cfg->eps * gnorm0) {
        info->converged = 1;
        break;
      }
    }
  }
out:
  memcpy(w_out, w, n * sizeof(double));
  info->status = status;
  for (size_t k = 0; k < 8; ++k) free(*lvecs[k]);
  for (size_t k = 0; k < 4; ++k) free(*nvecs[k]);
  free(e.cact); free(e.act); free(w); free(g); free(d); free(wc);
  return status;
}
