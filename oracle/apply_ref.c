/* ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * Scalar C restatement, in fp32, of the per-element arithmetic the CUDA
 * kernels perform (paper_2203_06638_b200/csrc/lpp_b200.cu), which in turn
 * restate the reference's fp64 operations:
 *   oracle_apply_sgd  <- ParamStore.sub_assign(start, lr*g)
 *                        (paramstore.py:121-136, _atomics.c:58-74,312-344,
 *                         call site engine.py:355); plus the momentum /
 *                        weight-decay extension the reference lists as an
 *                        extension point
 *   oracle_accum      <- _atomics.accum_cas_f64(dst, start, delta, scale)
 *   oracle_snapshot   <- _atomics.snapshot_f64 (_atomics.c:186-215)
 *   oracle_average    <- _MeanAllReduce.reduce + add_assign(mean - snap)
 *                        (engine.py:199-229, 418-421); np.mean(axis=0) sums
 *                        the worker rows in order and then divides by Q.
 * Compiled with -ffp-contract=off so no FMA contraction changes rounding.
 * Serial, single-writer: bit-exact comparison target for the GPU kernels
 * whenever no two writers touch the same element.
 */
#include <stddef.h>
#include <stdint.h>

static inline float sgd_delta(float g, float x, float* m, float lr, float mu, float wd) {
  float gp = g;
  if (wd != 0.0f) gp = gp + wd * x;
  if (mu != 0.0f) {
    float mm = mu * (*m) + gp;
    *m = mm;
    gp = mm;
  }
  return -(lr * gp);
}

void oracle_apply_sgd(float* x, const float* g, float* m, size_t n, float lr, float mu,
                      float wd) {
  for (size_t e = 0; e < n; ++e) {
    float mv = (mu != 0.0f) ? m[e] : 0.0f;
    float d = sgd_delta(g[e], x[e], &mv, lr, mu, wd);
    if (mu != 0.0f) m[e] = mv;
    x[e] = x[e] + d;
  }
}

int oracle_accum(float* dst, size_t dst_len, size_t start, const float* delta, size_t n,
                 float scale) {
  if (start > dst_len || n > dst_len - start) return -2;
  for (size_t e = 0; e < n; ++e) dst[start + e] = dst[start + e] + scale * delta[e];
  return 0;
}

void oracle_snapshot(const float* src, float* out, size_t n) {
  for (size_t e = 0; e < n; ++e) out[e] = src[e];
}

/* arenas: Q pointers; updates [lo, hi) of every arena in place */
int oracle_average(float** arenas, int Q, size_t lo, size_t hi, float* mean_out) {
  if (Q < 1) return -1;
  for (size_t e = lo; e < hi; ++e) {
    float v[64];
    for (int q = 0; q < Q; ++q) v[q] = arenas[q][e];
    float s = v[0];
    for (int q = 1; q < Q; ++q) s = s + v[q];
    float mean = s / (float)Q;
    for (int q = 0; q < Q; ++q) arenas[q][e] = arenas[q][e] + (mean - v[q]);
    if (mean_out) mean_out[e - lo] = mean;
  }
  return 0;
}
