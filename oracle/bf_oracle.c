/* TEST INFRASTRUCTURE — plain-C float64 restatement of the reference
 * algorithms (see bf_oracle.h). Each function cites the reference lines it
 * follows. Parity is pinned two ways (tests/test_oracle.py):
 *   1. against the reference executor itself, compiled in place
 *      (oracle/_ref/libbfref.so, built from /root/reference by oracle/Makefile);
 *   2. against tests/golden/*.npz, produced by tests/golden/make_golden.py from
 *      that same reference build on the acceptance-suite seeds
 *      (tests/acceptance.cpp:114-201).
 */
#include "bf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef void (*row_fn)(void* ctx, int64_t r0, int64_t r1);

typedef struct {
  row_fn fn;
  void* ctx;
  int64_t r0, r1;
} job_t;

static void* run_job(void* p) {
  job_t* j = (job_t*)p;
  j->fn(j->ctx, j->r0, j->r1);
  return NULL;
}

/* Split rows [0, n) over `threads` pthreads. */
static int parallel_rows(row_fn fn, void* ctx, int64_t n, int threads) {
  if (threads <= 1 || n < 2) {
    fn(ctx, 0, n);
    return 0;
  }
  if (threads > n) threads = (int)n;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  job_t* jobs = (job_t*)malloc(sizeof(job_t) * (size_t)threads);
  if (!th || !jobs) {
    free(th);
    free(jobs);
    return 1;
  }
  for (int t = 0; t < threads; ++t) {
    jobs[t].fn = fn;
    jobs[t].ctx = ctx;
    jobs[t].r0 = n * t / threads;
    jobs[t].r1 = n * (t + 1) / threads;
    pthread_create(&th[t], NULL, run_job, &jobs[t]);
  }
  for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
  free(th);
  free(jobs);
  return 0;
}

/* out[i][j] = sum_k a[i][k] * bt[j][k] for one row i (the dot convention:
 * right operand stored transposed, interpreter.hpp:289-294). */
static void row_times_bt(const double* a, const double* bt, double* out, int64_t K, int64_t N) {
  for (int64_t j = 0; j < N; ++j) {
    const double* b = bt + j * K;
    double s = 0.0;
    for (int64_t k = 0; k < K; ++k) s += a[k] * b[k];
    out[j] = s;
  }
}

/* ------------------------------------------------------------------ K1 */
typedef struct {
  const double *X, *Wt, *Vt, *Ut;
  double* O;
  int64_t D, F, N;
  double eps;
} ffn_ctx;

static void ffn_rows(void* p, int64_t r0, int64_t r1) {
  ffn_ctx* c = (ffn_ctx*)p;
  double* xn = (double*)malloc(sizeof(double) * (size_t)c->D);
  double* a = (double*)malloc(sizeof(double) * (size_t)c->F);
  double* b = (double*)malloc(sizeof(double) * (size_t)c->F);
  for (int64_t i = r0; i < r1; ++i) {
    const double* x = c->X + i * c->D;
    /* rmsnorm: inv = 1/sqrt(squaredNorm/k + eps), interpreter.hpp:529-536 */
    double ss = 0.0;
    for (int64_t d = 0; d < c->D; ++d) ss += x[d] * x[d];
    const double inv = 1.0 / sqrt(ss / (double)c->D + c->eps);
    for (int64_t d = 0; d < c->D; ++d) xn[d] = x[d] * inv;
    row_times_bt(xn, c->Wt, a, c->D, c->F);
    row_times_bt(xn, c->Vt, b, c->D, c->F);
    /* swish(a) = a * (1/(1+exp(-a))) (interpreter.hpp:539-541), then Hadamard with b */
    for (int64_t f = 0; f < c->F; ++f) a[f] = a[f] * (1.0 / (1.0 + exp(-a[f]))) * b[f];
    row_times_bt(a, c->Ut, c->O + i * c->N, c->F, c->N);
  }
  free(xn);
  free(a);
  free(b);
}

int bfo_rms_ffn_swiglu(const double* X, const double* Wt, const double* Vt, const double* Ut, double* O, int64_t M,
                       int64_t D, int64_t F, int64_t N, double eps, int threads) {
  ffn_ctx c = {X, Wt, Vt, Ut, O, D, F, N, eps};
  return parallel_rows(ffn_rows, &c, M, threads);
}

/* ------------------------------------------------------------------ K2 */
typedef struct {
  const double *X, *Yt;
  double* O;
  int64_t K, N;
  double eps;
  double* colsum; /* fused form only */
} ln_ctx;

static void ln_dense_rows(void* p, int64_t r0, int64_t r1) {
  ln_ctx* c = (ln_ctx*)p;
  double* xn = (double*)malloc(sizeof(double) * (size_t)c->K);
  const double k = (double)c->K;
  for (int64_t i = r0; i < r1; ++i) {
    const double* x = c->X + i * c->K;
    /* layernorm (interpreter.hpp:512-527): s1 = sum, s2 = squaredNorm,
     * sigma = sqrt(s2/k - mean^2); sigma == 0 -> zero row */
    double s1 = 0.0, s2 = 0.0;
    for (int64_t j = 0; j < c->K; ++j) {
      s1 += x[j];
      s2 += x[j] * x[j];
    }
    const double mean = s1 / k;
    const double sigma = sqrt(s2 / k - mean * mean);
    if (sigma == 0.0) {
      for (int64_t j = 0; j < c->K; ++j) xn[j] = 0.0;
    } else {
      for (int64_t j = 0; j < c->K; ++j) xn[j] = (x[j] - mean) / sigma;
    }
    row_times_bt(xn, c->Yt, c->O + i * c->N, c->K, c->N); /* layernorm(x) * yt^T, :549-551 */
  }
  free(xn);
}

int bfo_layernorm_matmul(const double* X, const double* Yt, double* O, int64_t M, int64_t K, int64_t N, int threads) {
  ln_ctx c = {X, Yt, O, K, N, 0.0, NULL};
  return parallel_rows(ln_dense_rows, &c, M, threads);
}

static void ln_fused_rows(void* p, int64_t r0, int64_t r1) {
  ln_ctx* c = (ln_ctx*)p;
  const double k = (double)c->K;
  for (int64_t i = r0; i < r1; ++i) {
    const double* x = c->X + i * c->K;
    double t1 = 0.0, t2 = 0.0; /* row_sum(X), row_sum(square(X)) */
    for (int64_t j = 0; j < c->K; ++j) {
      t1 += x[j];
      t2 += x[j] * x[j];
    }
    /* mu_neg = 0 - t1/total(K); var = t2/total(K) + (0 - square(t1/total(K)));
     * rstd = recip(sqrt(var))   (R4/R5 rewrite) */
    const double mu_neg = 0.0 - t1 / k;
    const double var = t2 / k + (0.0 - (t1 / k) * (t1 / k)) + c->eps;
    const double rstd = 1.0 / sqrt(var);
    double* o = c->O + i * c->N;
    row_times_bt(x, c->Yt, o, c->K, c->N); /* t3 = dot(X, Yt) on the raw rows */
    for (int64_t j = 0; j < c->N; ++j) o[j] = (o[j] + mu_neg * c->colsum[j]) * rstd; /* add(t3, outer(mu_neg, t4)) */
  }
}

int bfo_layernorm_matmul_fused(const double* X, const double* Yt, double* O, int64_t M, int64_t K, int64_t N,
                               double eps, int threads) {
  double* colsum = (double*)malloc(sizeof(double) * (size_t)N);
  if (!colsum) return 1;
  for (int64_t j = 0; j < N; ++j) { /* t4 = row_sum(Yt[n][k]) */
    double s = 0.0;
    for (int64_t kk = 0; kk < K; ++kk) s += Yt[j * K + kk];
    colsum[j] = s;
  }
  ln_ctx c = {X, Yt, O, K, N, eps, colsum};
  int rc = parallel_rows(ln_fused_rows, &c, M, threads);
  free(colsum);
  return rc;
}

/* ------------------------------------------------------------------ K3 */
typedef struct {
  const double *Q, *K, *Vt;
  double* O;
  int64_t Sq, Skv, D, Dv;
  double scale;
  int64_t chunks;
} attn_ctx;

/* rows index (head, query) pairs: r = h * Sq + i */
static void attn_dense_rows(void* p, int64_t r0, int64_t r1) {
  attn_ctx* c = (attn_ctx*)p;
  double* s = (double*)malloc(sizeof(double) * (size_t)c->Skv);
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t h = r / c->Sq, i = r % c->Sq;
    const double* q = c->Q + (h * c->Sq + i) * c->D;
    const double* Kh = c->K + h * c->Skv * c->D;
    const double* Vh = c->Vt + h * c->Dv * c->Skv;
    double* o = c->O + (h * c->Sq + i) * c->Dv;
    /* s = (q k^T)/sqrt(d); softmax_rows without max subtraction (interpreter.hpp:506-510, 543-547) */
    row_times_bt(q, Kh, s, c->D, c->Skv);
    double sum = 0.0;
    for (int64_t j = 0; j < c->Skv; ++j) {
      s[j] = exp(s[j] * c->scale);
      sum += s[j];
    }
    for (int64_t j = 0; j < c->Skv; ++j) s[j] /= sum;
    row_times_bt(s, Vh, o, c->Skv, c->Dv); /* * vt^T */
  }
  free(s);
}

int bfo_attention(const double* Q, const double* K, const double* Vt, double* O, int64_t BH, int64_t Sq, int64_t Skv,
                  int64_t D, int64_t Dv, double scale, int threads) {
  attn_ctx c = {Q, K, Vt, O, Sq, Skv, D, Dv, scale > 0 ? scale : 1.0 / sqrt((double)D), 1};
  return parallel_rows(attn_dense_rows, &c, BH * Sq, threads);
}

static void attn_safe_rows(void* p, int64_t r0, int64_t r1) {
  attn_ctx* c = (attn_ctx*)p;
  const int64_t hk = c->Skv / c->chunks;
  double* s = (double*)malloc(sizeof(double) * (size_t)hk);
  double* num = (double*)malloc(sizeof(double) * (size_t)c->Dv);
  for (int64_t r = r0; r < r1; ++r) {
    const int64_t h = r / c->Sq, i = r % c->Sq;
    const double* q = c->Q + (h * c->Sq + i) * c->D;
    const double* Kh = c->K + h * c->Skv * c->D;
    const double* Vh = c->Vt + h * c->Dv * c->Skv;
    double* o = c->O + (h * c->Sq + i) * c->Dv;
    double den = 0.0, t = -INFINITY;
    for (int64_t v = 0; v < c->Dv; ++v) num[v] = 0.0;
    for (int64_t ch = 0; ch < c->chunks; ++ch) {
      /* S = (q K_chunk^T) * scale; SEBlock::exp_of row-wise: t_row = max, s = exp(S - t) (:60-71) */
      double mx = -INFINITY;
      for (int64_t j = 0; j < hk; ++j) {
        const double* kr = Kh + (ch * hk + j) * c->D;
        double a = 0.0;
        for (int64_t d = 0; d < c->D; ++d) a += q[d] * kr[d];
        s[j] = a * c->scale;
        if (s[j] > mx) mx = s[j];
      }
      double part = 0.0;
      for (int64_t j = 0; j < hk; ++j) {
        s[j] = exp(s[j] - mx);
        part += s[j];
      }
      /* z = max(t, t_row); rebase = (t == -inf) ? 0 : exp(t - z); fresh = exp(t_row - z) (:163-170) */
      const double z = t > mx ? t : mx;
      const double rebase = (t == -INFINITY) ? 0.0 : exp(t - z);
      const double fresh = exp(mx - z);
      for (int64_t v = 0; v < c->Dv; ++v) {
        const double* vr = Vh + v * c->Skv + ch * hk;
        double a = 0.0;
        for (int64_t j = 0; j < hk; ++j) a += s[j] * vr[j];
        num[v] = num[v] * rebase + a * fresh;
      }
      den = den * rebase + part * fresh;
      t = z;
    }
    for (int64_t v = 0; v < c->Dv; ++v) o[v] = num[v] / den; /* (:172-173) */
  }
  free(s);
  free(num);
}

int bfo_attention_safe(const double* Q, const double* K, const double* Vt, double* O, int64_t BH, int64_t Sq,
                       int64_t Skv, int64_t D, int64_t Dv, double scale, int64_t row_chunks, int threads) {
  if (row_chunks <= 0 || Skv % row_chunks) return 1;
  attn_ctx c = {Q, K, Vt, O, Sq, Skv, D, Dv, scale > 0 ? scale : 1.0 / sqrt((double)D), row_chunks};
  return parallel_rows(attn_safe_rows, &c, BH * Sq, threads);
}
