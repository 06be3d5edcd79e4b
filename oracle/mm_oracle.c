/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the ELEVATE GEMM hot path.
 * Never linked into, loaded by, or called from the product path
 * (paper_2002_02268_b200/); only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg use it.
 *
 * Plain-C restatement of what the reference interpreter computes for the
 * seven scheduled `mm` terms (reference pkg/src/stratir/interp.py):
 *   - scalars are IEEE f64 (Python float): `mult` is a*b, `add` is a+b
 *     (interp.py:145-148); an fp32 x fp32 product is exact in f64;
 *   - `reduce`/`reduceSeq`/`reduceSeqUnroll` are left folds
 *     acc = op(acc)(x) from the init value (interp.py:84-89);
 *   - the baseline term folds acc + a_k*b_k over k in order
 *     (reduceSeq(fun acc p => add(acc)(mult(fst p)(snd p)))(0.0), the term
 *     DFNF;topDown(fuseReduceMap);lowerToC produces);
 *   - the six tiled schedules (paper_2002_02268_b200/schedules.py) split k
 *     by 4 and reorder with liftReduce + absorbReduceInit (rules.py:328-385),
 *     which turns `acc + (0 + p0 + ... + p3)` into `acc + p0 + ... + p3`:
 *     the same sequential fold per output element.
 * Compiled with -ffp-contract=off so the f64 operations round exactly like
 * CPython's, which makes this bit-identical to interp.run on the same
 * inputs (pinned in tests/test_oracle.py against tests/golden/).
 */
#include <stddef.h>
#include <stdlib.h>

/* B^T copy so the k loops read contiguously; the arithmetic is unchanged. */
static double* transpose_b(const float* B, int N, int K) {
  double* t = (double*)malloc((size_t)N * K * sizeof(double));
  for (int k = 0; k < K; ++k)
    for (int j = 0; j < N; ++j) t[(size_t)j * K + k] = (double)B[(size_t)k * N + j];
  return t;
}

/* C[i][j] = sum_k A[i][k]*B[k][j], sequential fold (baseline). */
void oracle_mm_seq_f64(const float* A, const float* B, double* C, int M, int N, int K) {
  double* bt = transpose_b(B, N, K);
  for (int i = 0; i < M; ++i) {
    const float* a = A + (size_t)i * K;
    for (int j = 0; j < N; ++j) {
      const double* b = bt + (size_t)j * K;
      double acc = 0.0;
      for (int k = 0; k < K; ++k) acc = acc + (double)a[k] * b[k];
      C[(size_t)i * N + j] = acc;
    }
  }
  free(bt);
}

/* (|A| |B|)_ij in f64: the magnitude term of the parity bound. */
void oracle_absprod_f64(const float* A, const float* B, double* C, int M, int N, int K) {
  double* bt = transpose_b(B, N, K);
  for (int i = 0; i < M; ++i) {
    const float* a = A + (size_t)i * K;
    for (int j = 0; j < N; ++j) {
      const double* b = bt + (size_t)j * K;
      double acc = 0.0;
      for (int k = 0; k < K; ++k) {
        double x = (double)a[k] * b[k];
        acc += x < 0 ? -x : x;
      }
      C[(size_t)i * N + j] = acc;
    }
  }
  free(bt);
}

/* Binomial filter: what interp.run returns for the
 * naive term -- dot(join(w2d), join(nbh)) folded left over the 9 taps in
 * row-major order from 0.0 -- and for the separated term (separateDot,
 * rules.py:485-513): h_r = ((0 + 1 x_r0) + 2 x_r1) + 1 x_r2 per window row,
 * out = ((0 + w0 h_0) + w1 h_1) + w0 h_2.  Borders clamp (padClamp,
 * interp.py:127-132).  The par schedules evaluate identically. */
static int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

void oracle_bf_naive_f64(const float* img, double* out, int H, int W) {
  static const double w[9] = {0.0625, 0.125, 0.0625, 0.125, 0.25, 0.125, 0.0625, 0.125, 0.0625};
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < W; ++j) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
          acc = acc + w[3 * a + b] * (double)img[(size_t)clampi(i + a - 1, H - 1) * W + clampi(j + b - 1, W - 1)];
      out[(size_t)i * W + j] = acc;
    }
}

void oracle_bf_separated_f64(const float* img, double* out, int H, int W) {
  static const double wh[3] = {1.0, 2.0, 1.0}, wv[3] = {0.0625, 0.125, 0.0625};
  for (int i = 0; i < H; ++i)
    for (int j = 0; j < W; ++j) {
      double acc = 0.0;
      for (int a = 0; a < 3; ++a) {
        const float* row = img + (size_t)clampi(i + a - 1, H - 1) * W;
        double h = 0.0;
        for (int b = 0; b < 3; ++b) h = h + wh[b] * (double)row[clampi(j + b - 1, W - 1)];
        acc = acc + wv[a] * h;
      }
      out[(size_t)i * W + j] = acc;
    }
}
