// Binomial filter (the paper's image-processing case study):
// out = w * clamp_pad(img), w = [1 2 1; 2 4 2; 1 2 1] / 16, one sm_100a kernel
// per ELEVATE binomial schedule (paper_2002_02268_b200/binomial.py):
//
//   naive          mapSeq(mapSeq(dot(join w2d, join nbh)))   thread per pixel,
//                  9 taps read through L1, fold in (di, dj) row-major order
//   naivePar       mapPar on rows                             row band per CTA,
//                  clamped halo tile in SMEM, column sliding window
//   separated      separateDot(w2d, wh, wv)                   thread per pixel,
//                  3 horizontal dots (wh = 1 2 1) then one vertical (wv = w/16)
//   separatedPar   separated + mapPar                         row band per CTA:
//                  each horizontal dot computed once and reused by the three
//                  output rows that need it (the "scanline" reuse)
//
// The banded kernels do the same per-pixel arithmetic as their unbanded
// schedule, so naivePar == naive and separatedPar == separated bitwise.
// All four are HBM-bound: 8 bytes per pixel (read + write), 9-12 FMA.

#include "elv_common.cuh"

namespace elv {
namespace {

__device__ __forceinline__ int clampi(int v, int hi) { return v < 0 ? 0 : (v > hi ? hi : v); }

constexpr float W0 = 0.0625f, W1 = 0.125f, W2 = 0.25f;     // w2d entries
constexpr float WV0 = 0.0625f, WV1 = 0.125f;                // wv = (1 2 1)/16

__global__ void __launch_bounds__(256)
k_bf_naive(const float* __restrict__ img, float* __restrict__ out, int H, int W, int ldi, int ldo) {
  const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
  if (i >= H || j >= W) return;
  const float w[9] = {W0, W1, W0, W1, W2, W1, W0, W1, W0};
  float acc = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float* row = img + (size_t)clampi(i + a - 1, H - 1) * ldi;
#pragma unroll
    for (int b = 0; b < 3; ++b) acc = fmaf(w[3 * a + b], __ldg(row + clampi(j + b - 1, W - 1)), acc);
  }
  out[(size_t)i * ldo + j] = acc;
}

__device__ __forceinline__ float hdot(float x0, float x1, float x2) {
  // dot([1,2,1], row) folded left from 0: ((0 + x0) + 2 x1) + x2
  float h = x0;
  h = fmaf(2.f, x1, h);
  return h + x2;
}

__global__ void __launch_bounds__(256)
k_bf_separated(const float* __restrict__ img, float* __restrict__ out, int H, int W, int ldi, int ldo) {
  const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
  if (i >= H || j >= W) return;
  const int jm = clampi(j - 1, W - 1), jp = clampi(j + 1, W - 1);
  float h[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const float* row = img + (size_t)clampi(i + a - 1, H - 1) * ldi;
    h[a] = hdot(__ldg(row + jm), __ldg(row + j), __ldg(row + jp));
  }
  float acc = WV0 * h[0];
  acc = fmaf(WV1, h[1], acc);
  acc = fmaf(WV0, h[2], acc);
  out[(size_t)i * ldo + j] = acc;
}

// Banded kernels: CTA = BAND rows x 256 columns; the (BAND+2) x (256+2)
// clamped halo is staged in SMEM with coalesced loads, then thread t owns
// column t and slides down the band.
constexpr int BAND = 32, BCOLS = 256;

__device__ __forceinline__ void stage_halo(float (*tile)[BCOLS + 2], const float* __restrict__ img, int H,
                                           int W, int ldi, int r0, int c0) {
  // thread t stages global column c0 + t into tile column t + 1 for all
  // BAND + 2 rows (one coalesced load per row, all rows in flight); threads
  // 0 and 1 also stage the left / right halo columns.  Clamping = padClamp.
  const int t = threadIdx.x;
  const int gj = clampi(c0 + t, W - 1);
  const int hj = t == 0 ? clampi(c0 - 1, W - 1) : clampi(c0 + BCOLS, W - 1);
  float v[BAND + 2], hv[BAND + 2];
#pragma unroll
  for (int rr = 0; rr < BAND + 2; ++rr) {
    const float* row = img + (size_t)clampi(r0 + rr - 1, H - 1) * ldi;
    v[rr] = __ldg(row + gj);
    if (t < 2) hv[rr] = __ldg(row + hj);
  }
#pragma unroll
  for (int rr = 0; rr < BAND + 2; ++rr) {
    tile[rr][t + 1] = v[rr];
    if (t < 2) tile[rr][t == 0 ? 0 : BCOLS + 1] = hv[rr];
  }
}

template <bool SEPARATED>
__global__ void __launch_bounds__(256)
k_bf_band(const float* __restrict__ img, float* __restrict__ out, int H, int W, int ldi, int ldo) {
  __shared__ float tile[BAND + 2][BCOLS + 2];
  const int r0 = blockIdx.y * BAND, c0 = blockIdx.x * BCOLS;
  stage_halo(tile, img, H, W, ldi, r0, c0);
  __syncthreads();
  const int t = threadIdx.x, j = c0 + t;
  if (j >= W) return;
  const int rows = min(BAND, H - r0);
  if (SEPARATED) {
    // horizontal dots once per staged row, reused by three output rows
    float h0 = hdot(tile[0][t], tile[0][t + 1], tile[0][t + 2]);
    float h1 = hdot(tile[1][t], tile[1][t + 1], tile[1][t + 2]);
    for (int r = 0; r < rows; ++r) {
      const float h2 = hdot(tile[r + 2][t], tile[r + 2][t + 1], tile[r + 2][t + 2]);
      float acc = WV0 * h0;
      acc = fmaf(WV1, h1, acc);
      acc = fmaf(WV0, h2, acc);
      out[(size_t)(r0 + r) * ldo + j] = acc;
      h0 = h1;
      h1 = h2;
    }
  } else {
    // 3x3 window slid down the band in registers: 3 SMEM reads per output
    // instead of 9; the taps are folded in the same (a, b) order, so the
    // result is bitwise the unbanded naive kernel's
    const float w[9] = {W0, W1, W0, W1, W2, W1, W0, W1, W0};
    float x[3][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) x[a][b] = tile[a][t + b];
    for (int r = 0; r < rows; ++r) {
#pragma unroll
      for (int b = 0; b < 3; ++b) x[2][b] = tile[r + 2][t + b];
      float acc = 0.f;
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) acc = fmaf(w[3 * a + b], x[a][b], acc);
      out[(size_t)(r0 + r) * ldo + j] = acc;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        x[0][b] = x[1][b];
        x[1][b] = x[2][b];
      }
    }
  }
}

}  // namespace

int launch_binomial(int variant, const float* img, float* out, int H, int W, int ldi, int ldo,
                    cudaStream_t st) {
  switch (variant) {
    case 0: {
      dim3 grid((W + 31) / 32, (H + 7) / 8);
      k_bf_naive<<<grid, dim3(32, 8), 0, st>>>(img, out, H, W, ldi, ldo);
      return check_launch("bf_naive");
    }
    case 2: {
      dim3 grid((W + 31) / 32, (H + 7) / 8);
      k_bf_separated<<<grid, dim3(32, 8), 0, st>>>(img, out, H, W, ldi, ldo);
      return check_launch("bf_separated");
    }
    case 1:
    case 3: {
      dim3 grid((W + BCOLS - 1) / BCOLS, (H + BAND - 1) / BAND);
      if (variant == 1) k_bf_band<false><<<grid, BCOLS, 0, st>>>(img, out, H, W, ldi, ldo);
      else k_bf_band<true><<<grid, BCOLS, 0, st>>>(img, out, H, W, ldi, ldo);
      return check_launch(variant == 1 ? "bf_naive_par" : "bf_separated_par");
    }
    default:
      return set_error(ELV_EVARIANT, "binomial: unknown variant %d", variant);
  }
}

}  // namespace elv
