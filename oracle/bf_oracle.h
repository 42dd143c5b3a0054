/* TEST INFRASTRUCTURE — plain-C float64 restatement of the reference's
 * algorithms on the hot path (used only by tests/, smoke() and bench.py's
 * CPU-baseline leg as the checker; never linked into the product).
 * All matrices are row-major doubles. `threads` partitions output rows over
 * pthreads (1 = serial, like the reference executor). Pinned against the
 * reference itself (oracle/_ref/libbfref.so) and tests/golden/. */
#ifndef BF_ORACLE_H_
#define BF_ORACLE_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ref::rms_ffn_swiglu (interpreter.hpp:553-559), rmsnorm with eps (:529-536), swish (:539-541). */
int bfo_rms_ffn_swiglu(const double* X, const double* Wt, const double* Vt, const double* Ut, double* O, int64_t M,
                       int64_t D, int64_t F, int64_t N, double eps, int threads);

/* ref::layernorm_matmul (interpreter.hpp:549-551): dense layernorm (:512-527, sigma = 0 -> 0 row). */
int bfo_layernorm_matmul(const double* X, const double* Yt, double* O, int64_t M, int64_t K, int64_t N, int threads);

/* The fused K2 program's arithmetic (final snapshot of fuse(lower(layernorm_matmul())),
 * SURVEY.md §2.1): (X Yt^T - mu (x) colsum(Yt)) * recip(sqrt(t2/K - (t1/K)^2 + eps)).
 * sigma = 0 gives inf/NaN like the interpreter walk (README.md:134-136). */
int bfo_layernorm_matmul_fused(const double* X, const double* Yt, double* O, int64_t M, int64_t K, int64_t N,
                               double eps, int threads);

/* ref::attention (interpreter.hpp:543-547): unsafe softmax_rows (:506-510), per head. */
int bfo_attention(const double* Q, const double* K, const double* Vt, double* O, int64_t BH, int64_t Sq, int64_t Skv,
                  int64_t D, int64_t Dv, double scale, int threads);

/* safe_attention_rows (safe_numerics.hpp:147-175): key chunks with row-wise
 * significand/exponent rebasing; finite for any finite input. */
int bfo_attention_safe(const double* Q, const double* K, const double* Vt, double* O, int64_t BH, int64_t Sq,
                       int64_t Skv, int64_t D, int64_t Dv, double scale, int64_t row_chunks, int threads);

/* random_inputs' draw (interpreter.hpp:585-597) is libstdc++-specific (std::normal_distribution);
 * the oracle does not restate it. Golden fixtures carry the drawn values instead. */

#ifdef __cplusplus
}
#endif
#endif
