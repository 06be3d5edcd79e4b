// Host-resident operands: C_h = A_h . B_h with PCIe traffic overlapped with
// the GEMM (elv_gemm_host, include/elevate_b200.h).
//
// This is the reference's calling convention -- interp.run(e, [A, B]) takes
// host values and returns a host value (reference pkg/src/stratir/interp.py:
// 157-162) -- made fast.  Two plans (make_plan): the grid cuts the output
// into R x Nc tiles, the H2D stream brings in B column chunks and A row
// blocks in the order that enables C tiles soonest, the caller's stream
// prepares (packB / tf32 / fp16 split) and multiplies each tile as soon as
// both its operands have landed, and the D2H stream returns each C tile as
// soon as it is written; the growing schedule (tensor-core variants, large
// C) brings A and B in strips and multiplies each landed strip against the
// other operand's resident prefix, so C starts flowing back after a few MB.  PCIe is full duplex
// (measured ~55 GB/s each way, ~100 GB/s both), so for large problems the
// step is bound by the D2H of C (the largest transfer) plus pipeline fill.  Tiles of C are independent (the mapPar axis), and each
// tile's per-element arithmetic is the single-launch kernel's, so the result
// equals elv_gemm's.

#include "elv_common.cuh"

#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <vector>

namespace elv {
namespace {

constexpr size_t kAlign = 256;
inline size_t up(size_t x, size_t a) { return (x + a - 1) / a * a; }
inline int ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

struct HostPlan {
  int R, Nc, nrb, ncb;
  // growing schedule (tensor-core variants, large C): A arrives in R-row
  // strips and B in Nc-column strips; each landed strip is multiplied against
  // everything of the other operand already resident (one GEMM, one D2H), so
  // the resident rectangle grows from the corner and the D2H stream starts
  // after a few MB instead of a whole B chunk.  Operand planes are prepared
  // strip by strip into full-size buffers, so one GEMM reads across strips.
  bool grow;
  bool packed_a;                 // variant 6: pack A per row block (cp.async kernel)
  size_t off_a, off_b, off_c, off_pa, stride_pa, off_pb, stride_pb, total;
};

// Tile sizes.  Small problems: one tile (plain H2D -> GEMM -> D2H).  Large:
// 8-16 row blocks (multiples of the 256-row pair tile) x column chunks of
// about 16384 columns (multiples of 256), so the first C tile is ready after
// a small slice of A and one chunk of B have crossed PCIe and each GEMM
// launch still fills several waves of the persistent grid.  The D2H of C is
// the bound, and a 2D copy's throughput grows with its row segment (32 KB
// rows ~46-51 GB/s, contiguous 57 GB/s).  Measured at 32768 x 32768 x 8192
// (3xTF32, gpurun_out/s2aa): 2048x16384 tiles 91.7 ms, 4096x16384 94.3,
// 2048x8192 96.7, 2048x32768 101.5 (full rows start the D2H too late).
HostPlan make_plan(int v, int M, int N, int K) {
  HostPlan p{};
  const double bytes = 4.0 * ((double)M * K + (double)K * N + (double)M * N);
  const bool tc = v == ELV_PARALLEL_TF32X3 || v == ELV_PARALLEL_FP16X3;
  p.R = M;
  p.Nc = N;
  // Growing schedule for the tensor-core variants once C is large: 1024-row
  // A strips and 4096-column B strips.  Measured (scripts/host_plan_sweep.py,
  // profiles/r1/host_plan_sweep.jsonl, 3xFP16): 32768^2 x 8192 91-93 ms vs
  // 94 ms for the grid, 16384^2 x 8192 29.6 vs 31.3 ms.  Narrower B strips
  // start the D2H sooner but their C blocks are tall, narrow copies (8 KB
  // rows over up to 4 GB of host addresses), which PCIe moves at ~34 GB/s
  // instead of ~45-55 (the trace in profiles/r1/host_pipeline_trace_grow.json).
  p.grow = tc && bytes >= (double)(64 << 20) && (M >= 16384 || N >= 16384);
  if (const char* g = getenv("ELV_HOST_PLAN")) {
    if (!strcmp(g, "grid")) p.grow = false;
    else if (!strcmp(g, "grow")) p.grow = tc;
  }
  if (p.grow) {
    p.R = 1024;
    p.Nc = 4096;
    if (const char* t = getenv("ELV_HOST_STRIPS")) {      // test hook: "R,Nc"
      int r = 0, c = 0;
      if (sscanf(t, "%d,%d", &r, &c) == 2 && r > 0 && c > 0) { p.R = r; p.Nc = c; }
    }
    if (p.R > M) p.R = M;
    if (p.Nc > N) p.Nc = N;
  } else if (bytes >= (double)(64 << 20)) {
    // 3xTF32 is PCIe-bound (GEMM ~ D2H time): finer row blocks start the D2H
    // stream sooner.  The SIMT variants are GEMM-bound (~4.6x the PCIe time):
    // 8 row blocks keep each launch at >= 6 waves of 128x256 tiles.
    const int fine = tc ? 16 : 8;
    const int row_blocks = M >= 8192 ? fine : (M >= 2048 ? 8 : (M >= 512 ? 2 : 1));
    p.R = (int)up((size_t)ceil_div(M, row_blocks), 256);
    if (p.R > M) p.R = M;
    // 3xTF32 (D2H-bound): 16384-column chunks (64 KB copy rows); SIMT
    // (GEMM-bound): 8192, so the first B chunk lands sooner
    const int cw = tc ? 16384 : 8192;
    if (N >= 2 * cw) {
      const int chunks = ceil_div(N, cw);
      p.Nc = (int)up((size_t)ceil_div(N, chunks), 256);
      if (p.Nc > N) p.Nc = N;
    }
  }
  // test hook: ELV_HOST_TILES="R,Nc" forces the tile shape (read per call)
  if (const char* t = getenv("ELV_HOST_TILES")) {
    int r = 0, c = 0;
    if (sscanf(t, "%d,%d", &r, &c) == 2 && r > 0 && c > 0) {
      p.grow = false;
      p.R = r < M ? r : M;
      p.Nc = c < N ? c : N;
    }
  }
  p.nrb = ceil_div(M, p.R);
  p.ncb = ceil_div(N, p.Nc);
  p.packed_a = v == ELV_PARALLEL && parallel_uses_packed_a(p.R, p.Nc);
  size_t o = 0;
  p.off_a = o;  o = up(o + (size_t)M * K * 4, kAlign);
  p.off_b = o;  o = up(o + (size_t)K * N * 4, kAlign);
  p.off_c = o;  o = up(o + (size_t)M * N * 4, kAlign);
  p.stride_pa = 0;
  if (p.grow) {          // full-size plane buffers, filled strip by strip
    const size_t pa = v == ELV_PARALLEL_TF32X3 ? tf32x3_a_planes_bytes(M, K) : fp16x3_a_planes_bytes(M, K);
    const size_t pb = v == ELV_PARALLEL_TF32X3 ? tf32x3_b_planes_bytes(N, K) : fp16x3_b_planes_bytes(N, K);
    p.off_pa = o;  o = up(o + pa, kAlign);
    p.off_pb = o;  o = up(o + pb, kAlign);
    p.total = o + kAlign;
    return p;
  }
  if (v == ELV_PARALLEL_TF32X3) p.stride_pa = up(tf32x3_a_planes_bytes(p.R, K), kAlign);
  else if (v == ELV_PARALLEL_FP16X3) p.stride_pa = up(fp16x3_a_planes_bytes(p.R, K), kAlign);
  else if (p.packed_a) p.stride_pa = up(pack_a_bytes(p.R, K), kAlign);
  p.off_pa = o;  o += p.stride_pa * p.nrb;
  p.stride_pb = 0;
  if (v == ELV_PARALLEL_TF32X3) p.stride_pb = up(tf32x3_b_planes_bytes(p.Nc, K), kAlign);
  else if (v == ELV_PARALLEL_FP16X3) p.stride_pb = up(fp16x3_b_planes_bytes(p.Nc, K), kAlign);
  else if (v >= ELV_ARRAYPACKING) p.stride_pb = up(elv_pack_b_bytes(K, p.Nc), kAlign);
  p.off_pb = o;  o += p.stride_pb * p.ncb;
  p.total = o + kAlign;   // slack for aligning the caller's base pointer
  return p;
}

// The fp16 encoding needs every tile GEMM to qualify (K >= 512, a wave of
// pair tiles); otherwise the whole call uses the tf32 encoding.
int host_variant(int v, int M, int N, int K) {
  if (v != ELV_PARALLEL_FP16X3) return v;
  const HostPlan p = make_plan(ELV_PARALLEL_TF32X3, M, N, K);
  const int rl = M - (p.nrb - 1) * p.R, cl = N - (p.ncb - 1) * p.Nc;
  const bool ok = fp16x3_applicable(p.R, p.Nc, K) && fp16x3_applicable(rl, p.Nc, K) &&
                  fp16x3_applicable(p.R, cl, K) && fp16x3_applicable(rl, cl, K);
  return ok ? v : ELV_PARALLEL_TF32X3;
}

// Per-device copy streams and an event pool (library-internal, created once).
// With ELV_HOST_TRACE=1 a second pool of timing events records when every
// H2D item, tile GEMM and D2H copy finished (elv_gemm_host_trace reads them).
struct DeviceRes {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaStream_t d2h_extra[3] = {nullptr, nullptr, nullptr};   // more copy engines for D2H
  cudaEvent_t end_extra[3] = {nullptr, nullptr, nullptr};
  std::vector<cudaEvent_t> events;
  std::vector<cudaEvent_t> tev;          // trace: [0] entry, then (kind, event) records
  std::vector<int> tkind;                // 0 h2d, 1 tile, 2 d2h
  std::mutex mu;
};
thread_local int g_trace_dev = -1;
DeviceRes g_res[64];

int get_events(DeviceRes& r, size_t n) {
  while (r.events.size() < n) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return set_error(ELV_ECUDA, "gemm_host: cudaEventCreate: %s", cudaGetErrorString(cudaGetLastError()));
    r.events.push_back(e);
  }
  return ELV_OK;
}

#define CK(call, what)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess) return set_error(ELV_ECUDA, "gemm_host: %s: %s", what, cudaGetErrorString(e_)); \
  } while (0)

}  // namespace
}  // namespace elv

using namespace elv;

extern "C" {

size_t elv_gemm_host_workspace_bytes(int variant, int M, int N, int K) {
  if (M < 1 || N < 1 || K < 1 || variant < 0 || variant >= ELV_NUM_VARIANTS) return 0;
  variant = host_variant(variant, M, N, K);
  return make_plan(variant, M, N, K).total;
}

int elv_gemm_host_tiles(int variant, int M, int N, int K, int* rows, int* cols) {
  if (M < 1 || N < 1 || K < 1 || variant < 0 || variant >= ELV_NUM_VARIANTS)
    return set_error(ELV_EINVAL, "gemm_host_tiles: bad arguments");
  variant = host_variant(variant, M, N, K);
  const HostPlan p = make_plan(variant, M, N, K);
  if (rows) *rows = p.R;
  if (cols) *cols = p.Nc;
  return ELV_OK;
}

int elv_gemm_host(int variant, const float* A_h, const float* B_h, float* C_h, int M, int N, int K,
                  int lda, int ldb, int ldc, void* workspace, size_t workspace_bytes, void* stream) {
  if (A_h == nullptr || B_h == nullptr || C_h == nullptr)
    return set_error(ELV_EINVAL, "gemm_host: null matrix pointer");
  if (M < 1 || N < 1 || K < 1)
    return set_error(ELV_EINVAL, "gemm_host: sizes must be positive (M=%d N=%d K=%d)", M, N, K);
  if (lda < K || ldb < N || ldc < N)
    return set_error(ELV_EINVAL, "gemm_host: leading dimension too small (lda=%d ldb=%d ldc=%d)", lda, ldb, ldc);
  if (variant < 0 || variant >= ELV_NUM_VARIANTS) return set_error(ELV_EVARIANT, "unknown variant %d", variant);
  variant = host_variant(variant, M, N, K);
  const HostPlan p = make_plan(variant, M, N, K);
  if (workspace == nullptr || workspace_bytes < p.total)
    return set_error(ELV_EWORKSPACE, "gemm_host: needs %zu workspace bytes, got %zu", p.total, workspace_bytes);
  int dev = 0;
  CK(cudaGetDevice(&dev), "cudaGetDevice");
  if (dev < 0 || dev >= 64) return set_error(ELV_EINVAL, "gemm_host: device %d out of range", dev);
  DeviceRes& r = g_res[dev];
  std::lock_guard<std::mutex> lk(r.mu);
  if (r.h2d == nullptr) {
    CK(cudaStreamCreateWithFlags(&r.h2d, cudaStreamNonBlocking), "create h2d stream");
    CK(cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking), "create d2h stream");
    for (int q = 0; q < 3; ++q) {
      CK(cudaStreamCreateWithFlags(&r.d2h_extra[q], cudaStreamNonBlocking), "create d2h stream");
      CK(cudaEventCreateWithFlags(&r.end_extra[q], cudaEventDisableTiming), "create event");
    }
  }
  // D2H copies of a tile are split by rows over `nd` streams (copy engines)
  int nd = 1;        // measured: 2-3 streams do not raise D2H throughput (gpurun_out/s2aa)
  if (const char* e = getenv("ELV_HOST_D2H_STREAMS")) nd = atoi(e);
  if (nd < 1) nd = 1;
  if (nd > 4) nd = 4;
  cudaStream_t d2hs[4] = {r.d2h, r.d2h_extra[0], r.d2h_extra[1], r.d2h_extra[2]};
  const int ntiles = p.grow ? p.nrb + p.ncb : p.nrb * p.ncb;
  // events: [0] entry, [1] h2d done, [2 .. 2+nrb) A blocks, [.. +ncb) B chunks, [.. +ntiles) tiles
  int rc = get_events(r, 2 + p.nrb + p.ncb + ntiles + (p.grow ? p.nrb + p.ncb : 0));
  if (rc) return rc;
  cudaEvent_t* ev = r.events.data();
  cudaEvent_t ev_entry = ev[0], ev_end = ev[1];
  cudaEvent_t* ev_a = ev + 2;
  cudaEvent_t* ev_b = ev_a + p.nrb;
  cudaEvent_t* ev_t = ev_b + p.ncb;

  cudaStream_t st = (cudaStream_t)stream;
  const bool trace = getenv("ELV_HOST_TRACE") && atoi(getenv("ELV_HOST_TRACE")) != 0;
  size_t ntr = 0;
  auto trace_rec = [&](int kind, cudaStream_t s2) -> int {
    if (!trace) return ELV_OK;
    if (r.tev.size() <= ntr) {
      cudaEvent_t e;
      if (cudaEventCreate(&e) != cudaSuccess) return set_error(ELV_ECUDA, "gemm_host: trace event");
      r.tev.push_back(e);
      r.tkind.push_back(0);
    }
    r.tkind[ntr] = kind;
    if (cudaEventRecord(r.tev[ntr++], s2) != cudaSuccess) return set_error(ELV_ECUDA, "gemm_host: trace record");
    return ELV_OK;
  };
  if (trace) g_trace_dev = dev;
  uint8_t* base = reinterpret_cast<uint8_t*>(up(reinterpret_cast<uintptr_t>(workspace), kAlign));
  float* A_d = reinterpret_cast<float*>(base + p.off_a);
  float* B_d = reinterpret_cast<float*>(base + p.off_b);
  float* C_d = reinterpret_cast<float*>(base + p.off_c);
  auto prep_a = [&](int i) { return base + p.off_pa + p.stride_pa * i; };
  auto prep_b = [&](int j) { return base + p.off_pb + p.stride_pb * j; };

  // the copy streams start after everything already queued on the caller's stream
  CK(cudaEventRecord(ev_entry, st), "record entry");
  if ((rc = trace_rec(-1, st))) return rc;
  CK(cudaStreamWaitEvent(r.h2d, ev_entry, 0), "h2d wait entry");
  for (int q = 0; q < nd; ++q) CK(cudaStreamWaitEvent(d2hs[q], ev_entry, 0), "d2h wait entry");

  if (p.grow) {
    // H2D: B strip 0, then always the operand with less resident (rows vs
    // columns: both K*4 bytes each), so the resident rectangle stays square
    struct Strip { bool is_b; int idx; };
    std::vector<Strip> order;
    {
      int na = 0, nb = 0;
      long long la = 0, lb = 0;
      while (na < p.nrb || nb < p.ncb) {
        const bool take_b = nb < p.ncb && (na == p.nrb || lb <= la);
        if (take_b) { order.push_back({true, nb}); lb += std::min(p.Nc, N - nb * p.Nc); ++nb; }
        else { order.push_back({false, na}); la += std::min(p.R, M - na * p.R); ++na; }
      }
    }
    cudaEvent_t* ev_item = ev_a;            // one per strip, in H2D order
    cudaEvent_t* ev_back = ev_t + ntiles;   // one per strip: its C block is back on the host
    // Pacing (ELV_HOST_PACE=L): strip k's H2D waits until block k-L is back
    // on the host, so the H2D stream runs at most L strips ahead of the D2H
    // stream instead of taking PCIe bandwidth from it early on.
    int pace = 0;
    if (const char* e = getenv("ELV_HOST_PACE")) pace = std::max(0, atoi(e));
    std::vector<int> last_back(order.size(), -1);   // latest block <= k with a D2H
    // strips are enqueued in order on all three streams: H2D, then prepare +
    // GEMM of the block it enables, then the D2H of that block
    const bool f16 = variant == ELV_PARALLEL_FP16X3;
    int d2h_rows = 1 << 30;           // rows per D2H copy (tuning hook)
    if (const char* e = getenv("ELV_HOST_D2H_ROWS")) d2h_rows = std::max(1, atoi(e));
    void* pa = prep_a(0);
    void* pb = prep_b(0);
    int rows_in = 0, cols_in = 0;
    for (size_t k = 0; k < order.size(); ++k) {
      const Strip& it = order[k];
      if (pace > 0 && k >= (size_t)pace && last_back[k - pace] >= 0)
        CK(cudaStreamWaitEvent(r.h2d, ev_back[last_back[k - pace]], 0), "h2d pace");
      if (it.is_b) {
        const int c0 = it.idx * p.Nc, nc = std::min(p.Nc, N - c0);
        CK(cudaMemcpy2DAsync(B_d + c0, (size_t)N * 4, B_h + c0, (size_t)ldb * 4, (size_t)nc * 4, K,
                             cudaMemcpyHostToDevice, r.h2d), "H2D B strip");
      } else {
        const int r0 = it.idx * p.R, nr = std::min(p.R, M - r0);
        CK(cudaMemcpy2DAsync(A_d + (size_t)r0 * K, (size_t)K * 4, A_h + (size_t)r0 * lda, (size_t)lda * 4,
                             (size_t)K * 4, nr, cudaMemcpyHostToDevice, r.h2d), "H2D A strip");
      }
      CK(cudaEventRecord(ev_item[k], r.h2d), "record strip");
      if ((rc = trace_rec(0, r.h2d))) return rc;

      // prepare the strip as it lands, then one GEMM: the strip against the
      // other operand's resident prefix; D2H that block of C
      CK(cudaStreamWaitEvent(st, ev_item[k], 0), "wait strip");
      int r0, nr, c0, nc;
      if (it.is_b) {
        c0 = it.idx * p.Nc; nc = std::min(p.Nc, N - c0);
        rc = f16 ? fp16x3_split_b(B_d + c0, K, nc, N, pb, st, N, c0)
                 : tf32x3_split_b(B_d + c0, K, nc, N, false, pb, st, N, c0);
        if (rc) return rc;
        cols_in += nc;
        r0 = 0; nr = rows_in;
      } else {
        r0 = it.idx * p.R; nr = std::min(p.R, M - r0);
        rc = f16 ? fp16x3_split_a(A_d + (size_t)r0 * K, nr, K, K, pa, st, M, r0)
                 : tf32x3_split_a(A_d + (size_t)r0 * K, nr, K, K, pa, st, M, r0);
        if (rc) return rc;
        rows_in += nr;
        c0 = 0; nc = cols_in;
      }
      last_back[k] = k > 0 ? last_back[k - 1] : -1;
      if (nr == 0 || nc == 0) continue;       // the first strip: nothing to multiply yet
      float* Cb = C_d + (size_t)r0 * N + c0;
      rc = f16 ? fp16x3_gemm_planes(pa, pb, Cb, nr, nc, K, N, st, M, r0, N, c0)
               : tf32x3_gemm_planes(pa, pb, Cb, nr, nc, K, N, st, M, r0, N, c0);
      if (!rc)    // range guard: recompute marked rows / columns of this block
        rc = tc_fixup_planes(f16, pa, pb, A_d + (size_t)r0 * K, K, B_d + c0, N, false, Cb, N, nr, nc, K, st, M, r0,
                             N, c0);
      if (rc) return rc;
      CK(cudaEventRecord(ev_t[k], st), "record block");
      if ((rc = trace_rec(1, st))) return rc;
      CK(cudaStreamWaitEvent(r.d2h, ev_t[k], 0), "d2h wait block");
      for (int a0 = 0; a0 < nr; a0 += d2h_rows) {
        const int h = std::min(d2h_rows, nr - a0);
        CK(cudaMemcpy2DAsync(C_h + (size_t)(r0 + a0) * ldc + c0, (size_t)ldc * 4, C_d + (size_t)(r0 + a0) * N + c0,
                             (size_t)N * 4, (size_t)nc * 4, h, cudaMemcpyDeviceToHost, r.d2h), "D2H C block");
      }
      CK(cudaEventRecord(ev_back[k], r.d2h), "record block back");
      last_back[k] = (int)k;
      if ((rc = trace_rec(2, r.d2h))) return rc;
    }
    CK(cudaEventRecord(ev_end, r.d2h), "record end");
    if (trace) r.tkind.resize(ntr);
    CK(cudaStreamWaitEvent(st, ev_end, 0), "join d2h");
    return ELV_OK;
  }

  // H2D order: start with B chunk 0 and A block 0, then repeatedly bring
  // whichever operand enables more new C tiles per byte (an A block enables
  // one tile per B chunk already present and vice versa), so the GEMM and the
  // D2H stream get work as early as PCIe allows.
  struct Item { bool is_b; int idx; };
  std::vector<Item> order;
  std::vector<int> pos_a(p.nrb), pos_b(p.ncb);
  {
    int na = 0, nb = 0;
    const double a_bytes = (double)p.R * K, b_bytes = (double)K * p.Nc;
    while (na < p.nrb || nb < p.ncb) {
      bool take_b;
      if (nb == 0) take_b = true;
      else if (na == 0) take_b = false;
      else if (na == p.nrb) take_b = true;
      else if (nb == p.ncb) take_b = false;
      else take_b = (double)na / b_bytes > (double)nb / a_bytes;
      if (take_b) { pos_b[nb] = (int)order.size(); order.push_back({true, nb++}); }
      else { pos_a[na] = (int)order.size(); order.push_back({false, na++}); }
    }
  }
  for (const Item& it : order) {
    if (it.is_b) {
      const int c0 = it.idx * p.Nc, nc = N - c0 < p.Nc ? N - c0 : p.Nc;
      CK(cudaMemcpy2DAsync(B_d + c0, (size_t)N * 4, B_h + c0, (size_t)ldb * 4, (size_t)nc * 4, K,
                           cudaMemcpyHostToDevice, r.h2d), "H2D B chunk");
      CK(cudaEventRecord(ev_b[it.idx], r.h2d), "record B chunk");
      if ((rc = trace_rec(0, r.h2d))) return rc;
    } else {
      const int r0 = it.idx * p.R, nr = M - r0 < p.R ? M - r0 : p.R;
      CK(cudaMemcpy2DAsync(A_d + (size_t)r0 * K, (size_t)K * 4, A_h + (size_t)r0 * lda, (size_t)lda * 4,
                           (size_t)K * 4, nr, cudaMemcpyHostToDevice, r.h2d), "H2D A block");
      CK(cudaEventRecord(ev_a[it.idx], r.h2d), "record A block");
      if ((rc = trace_rec(0, r.h2d))) return rc;
    }
  }

  // tiles in the order their operands land (ties: row-major)
  std::vector<int> tiles(ntiles);
  for (int t = 0; t < ntiles; ++t) tiles[t] = t;
  std::stable_sort(tiles.begin(), tiles.end(), [&](int x, int y) {
    const int rx = std::max(pos_a[x / p.ncb], pos_b[x % p.ncb]);
    const int ry = std::max(pos_a[y / p.ncb], pos_b[y % p.ncb]);
    return rx < ry;
  });

  // prepare + multiply tile by tile on the caller's stream
  std::vector<char> have_a(p.nrb, 0), have_b(p.ncb, 0);
  for (int t : tiles) {
    const int i = t / p.ncb, j = t % p.ncb;
    const int r0 = i * p.R, nr = M - r0 < p.R ? M - r0 : p.R;
    const int c0 = j * p.Nc, nc = N - c0 < p.Nc ? N - c0 : p.Nc;
    const float* Ai = A_d + (size_t)r0 * K;
    if (!have_b[j]) {
      CK(cudaStreamWaitEvent(st, ev_b[j], 0), "wait B chunk");
      if (variant == ELV_PARALLEL_TF32X3) rc = tf32x3_split_b(B_d + c0, K, nc, N, false, prep_b(j), st);
      else if (variant == ELV_PARALLEL_FP16X3) rc = fp16x3_split_b(B_d + c0, K, nc, N, prep_b(j), st);
      else if (variant >= ELV_ARRAYPACKING) rc = launch_pack_b(B_d + c0, reinterpret_cast<float*>(prep_b(j)), K, nc, N, st);
      if (rc) return rc;
      have_b[j] = 1;
    }
    if (!have_a[i]) {
      CK(cudaStreamWaitEvent(st, ev_a[i], 0), "wait A block");
      if (variant == ELV_PARALLEL_TF32X3) rc = tf32x3_split_a(Ai, nr, K, K, prep_a(i), st);
      else if (variant == ELV_PARALLEL_FP16X3) rc = fp16x3_split_a(Ai, nr, K, K, prep_a(i), st);
      else if (p.packed_a) rc = launch_pack_a(Ai, reinterpret_cast<float*>(prep_a(i)), nr, K, K, st);
      if (rc) return rc;
      have_a[i] = 1;
    }
    float* Cij = C_d + (size_t)r0 * N + c0;
    if (variant == ELV_PARALLEL_TF32X3 || variant == ELV_PARALLEL_FP16X3) {
      const bool f16 = variant == ELV_PARALLEL_FP16X3;
      rc = f16 ? fp16x3_gemm_planes(prep_a(i), prep_b(j), Cij, nr, nc, K, N, st)
               : tf32x3_gemm_planes(prep_a(i), prep_b(j), Cij, nr, nc, K, N, st);
      if (!rc) rc = tc_fixup_planes(f16, prep_a(i), prep_b(j), Ai, K, B_d + c0, N, false, Cij, N, nr, nc, K, st);
    } else if (variant == ELV_PARALLEL && p.packed_a && parallel_uses_packed_a(nr, nc)) {
      rc = launch_parallel_packed(reinterpret_cast<const float*>(prep_a(i)),
                                  reinterpret_cast<const float*>(prep_b(j)), Cij, nr, nc, K, N, st);
    } else if (variant >= ELV_ARRAYPACKING) {
      rc = launch_simt(variant, Ai, nullptr, reinterpret_cast<const float*>(prep_b(j)), Cij, nr, nc, K, K, 0,
                       N, st);
    } else {
      rc = launch_simt(variant, Ai, B_d + c0, nullptr, Cij, nr, nc, K, K, N, N, st);
    }
    if (rc) return rc;
    CK(cudaEventRecord(ev_t[t], st), "record tile");
    if ((rc = trace_rec(1, st))) return rc;
  }

  // D2H each tile as soon as it is written (row slices over nd streams).
  // Copying whole row blocks instead (longer copy rows, but each waits for
  // its last tile) measured slower: 99.7 vs 94.8 ms (gpurun_out/s2ac).
  for (int t : tiles) {
    const int i = t / p.ncb, j = t % p.ncb;
    const int r0 = i * p.R, nr = M - r0 < p.R ? M - r0 : p.R;
    const int c0 = j * p.Nc, nc = N - c0 < p.Nc ? N - c0 : p.Nc;
    const int per = (nr + nd - 1) / nd;
    for (int q = 0; q < nd; ++q) {
      const int a0 = q * per, a1 = nr < a0 + per ? nr : a0 + per;
      if (a1 <= a0) continue;
      CK(cudaStreamWaitEvent(d2hs[q], ev_t[t], 0), "d2h wait tile");
      CK(cudaMemcpy2DAsync(C_h + (size_t)(r0 + a0) * ldc + c0, (size_t)ldc * 4, C_d + (size_t)(r0 + a0) * N + c0,
                           (size_t)N * 4, (size_t)nc * 4, a1 - a0, cudaMemcpyDeviceToHost, d2hs[q]),
         "D2H C tile");
    }
    if ((rc = trace_rec(2, d2hs[nd - 1]))) return rc;
  }
  CK(cudaEventRecord(ev_end, r.d2h), "record end");
  if (trace) r.tkind.resize(ntr);
  CK(cudaStreamWaitEvent(st, ev_end, 0), "join d2h");
  for (int q = 1; q < nd; ++q) {
    CK(cudaEventRecord(r.end_extra[q - 1], d2hs[q]), "record end");
    CK(cudaStreamWaitEvent(st, r.end_extra[q - 1], 0), "join d2h");
  }
  return ELV_OK;
}

int elv_copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height, int kind,
               void* stream) {
  if (dst == nullptr || src == nullptr || width > dpitch || width > spitch)
    return set_error(ELV_EINVAL, "copy2d: bad arguments");
  if (width == 0 || height == 0) return ELV_OK;
  const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice : kind == 2 ? cudaMemcpyDeviceToHost
                                                                          : cudaMemcpyDeviceToDevice;
  CK(cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, height, k, (cudaStream_t)stream), "copy2d");
  return ELV_OK;
}

/* Diagnostics (ELV_HOST_TRACE=1): after the last elv_gemm_host on this
 * thread has completed, write up to `cap` (kind, ms-since-entry) pairs --
 * kind 0 = an H2D item landed, 1 = a tile's GEMM finished, 2 = a tile's D2H
 * finished -- and return how many. */
int elv_gemm_host_trace(float* out, int cap) {
  if (g_trace_dev < 0) return 0;
  DeviceRes& r = g_res[g_trace_dev];
  std::lock_guard<std::mutex> lk(r.mu);
  int n = 0;
  for (size_t i = 1; i < r.tkind.size() && n < cap; ++i, ++n) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.tev[0], r.tev[i]);
    out[2 * n] = (float)r.tkind[i];
    out[2 * n + 1] = ms;
  }
  return n;
}

}  // extern "C"
