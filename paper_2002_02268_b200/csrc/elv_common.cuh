// Shared internals of libelevate_b200: error plumbing and launch helpers.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <stdio.h>
#include <stdarg.h>
#include <stdlib.h>

#include <utility>

#include "../../include/elevate_b200.h"

namespace elv {

int set_error(int code, const char* fmt, ...);
int check_launch(const char* what);

// Programmatic dependent launch: a GEMM that follows its operand-preparation
// kernel on the stream is launched with programmatic stream serialization,
// so its prologue (TMEM allocation, barrier init, descriptor prefetch) runs
// while the preparation drains; griddep_wait() then blocks until the
// preceding grid has completed and its writes are visible.  Without the
// attribute (or ELV_PDL=0) the wait is a no-op and ordering is the stream's.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void griddep_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl_if(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  return launch_pdl_if(true, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// Preferred L1 / shared-memory carveout of the light-SMEM kernels that run
// next to the big-SMEM GEMMs (prepare kernels before them, the range-guard
// fix-up PDL-scheduled during them): asking for the maximum shared carveout
// keeps every SM in the GEMM's configuration, so a PDL-launched GEMM (or
// fix-up) CTA can become resident beside a finishing neighbour instead of
// waiting for the SM to drain and reconfigure.  Measured slower (the
// prepare kernels lose their L1: 1024^3 3xFP16 call 27.6 -> 29.7 us, bench
// prepass 1.25 -> 1.35 ms; profiles/r2/experiments/carveout_ab.txt), so
// off by default; ELV_PREP_CARVEOUT=1 (read once per process) turns it on.
inline bool prep_carveout_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ELV_PREP_CARVEOUT");
    v = e ? (atoi(e) != 0) : 0;
  }
  return v != 0;
}
#define ELV_PREFER_MAX_SMEM(fn)                                                                          \
  do {                                                                                                   \
    static int elv_carveout_dev_ = -1;                                                                   \
    int elv_cur_dev_ = 0;                                                                                \
    if (prep_carveout_enabled() && cudaGetDevice(&elv_cur_dev_) == cudaSuccess &&                        \
        elv_carveout_dev_ != elv_cur_dev_) {                                                             \
      cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,                           \
                           (int)cudaSharedmemCarveoutMaxShared);                                         \
      elv_carveout_dev_ = elv_cur_dev_;                                                                  \
    }                                                                                                    \
  } while (0)

constexpr int kPanel = 32;          // packB block (rules.py:516 default 32)
constexpr int kPackAlign = 256;     // packed column count padded to 8 panels (widest SIMT tile)

inline size_t packed_cols(int N) { return (size_t)((N + kPackAlign - 1) / kPackAlign) * kPackAlign; }

inline int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// SIMT ladder (simt_gemm.cu)
int launch_simt(int variant, const float* A, const float* B, const float* packedB,
                float* C, int M, int N, int K, int lda, int ldb, int ldc, cudaStream_t st);
int launch_pack_b(const float* B, float* packedB, int K, int N, int ldb, cudaStream_t st);
size_t pack_a_bytes(int M, int K);
int launch_pack_a(const float* A, float* packedA, int M, int K, int lda, cudaStream_t st);
int launch_pack_ab(const float* B, float* packedB, int K, int N, int ldb, const float* A, float* packedA, int M,
                   int lda, cudaStream_t st);
int launch_parallel_packed(const float* packedA, const float* packedB, float* C, int M, int N, int K, int ldc,
                           cudaStream_t st);
bool parallel_uses_packed_a(int M, int N);

// tcgen05 3xTF32 (tf32x3_gemm.cu)
size_t tf32x3_workspace_bytes(int M, int N, int K);
int tf32x3_prepare(const float* A, const float* B, int M, int N, int K, int lda, int ldb,
                   void* ws, size_t ws_bytes, cudaStream_t st);
// compute = the GEMM on the prepared planes + the range-guard fix-up (reads A, B)
int tf32x3_compute(const float* A, const float* B, int lda, int ldb, float* C, int M, int N, int K, int ldc, void* ws,
                   size_t ws_bytes, cudaStream_t st);
size_t tf32x3_a_planes_bytes(int M, int K);
size_t tf32x3_b_planes_bytes(int N, int K);
// optional trailing arguments: the plane buffers hold `total` rows / columns
// and the call covers [r0, r0 + M) / [c0, c0 + N) of them (0, 0: exactly these)
int tf32x3_split_a(const float* A, int M, int K, int lda, void* a_planes, cudaStream_t st, int total = 0,
                   int r0 = 0);
int tf32x3_split_b(const float* B, int K, int N, int ldb, bool packed, void* b_planes, cudaStream_t st,
                   int total = 0, int c0 = 0);
// The range-guard fix-up folded into the GEMM launch: the fp32 operands and
// the split's flags, handed to the 1-CTA tensor-core kernel (small problems),
// which recomputes its own flagged outputs after storing them -- one launch
// fewer.  `applied` is set when the launched kernel took it (the pair kernel
// does not: the caller then runs tc_fixup).
struct FixArgs {
  const float* A;
  int lda;
  const float* B;
  int ldb;
  const unsigned int* flag_a;
  const unsigned int* flag_b;
  int applied;
};
int tf32x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K, int ldc,
                       cudaStream_t st, int a_total = 0, int r0 = 0, int b_total = 0, int c0 = 0,
                       FixArgs* fix = nullptr);
bool tc_fixup_enabled();
int tc_kernel_choice(int M, int N, int sms, int* bn);
const unsigned int* tf32x3_b_planes_flags(const void* b_planes, int N, int K);
bool tf32x3_fused_ok(const float* A, int lda, const float* B, int ldb, int M, int N);
bool tf32x3_fused_a_ok(const float* A, int lda, int M, int N);
int tf32x3_gemm_fused(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N, int K,
                      unsigned int* flag_a, unsigned int* flag_b, cudaStream_t st, const void* b_planes = nullptr,
                      int b_total = 0, int c0 = 0);
int tc_fixup(const float* A, int lda, const float* B, int ldb, bool b_packed, float* C, int ldc, int M, int N, int K,
             const unsigned int* flag_a, const unsigned int* flag_b, cudaStream_t st);
int launch_split_tf32(const float* X, float* hi, float* lo, long long n, cudaStream_t st);
// 3xFP16 encoding of the parallel schedule's tcgen05 kernel (tf32x3_gemm.cu)
bool fp16x3_applicable(int M, int N, int K);
size_t fp16x3_workspace_bytes(int M, int N, int K);
int fp16x3_prepare(const float* A, const float* B, int M, int N, int K, int lda, int ldb, void* ws,
                   size_t ws_bytes, cudaStream_t st);
int fp16x3_compute(const float* A, const float* B, int lda, int ldb, float* C, int M, int N, int K, int ldc, void* ws,
                   size_t ws_bytes, cudaStream_t st);
size_t fp16x3_a_planes_bytes(int M, int K);
size_t fp16x3_b_planes_bytes(int N, int K);
int fp16x3_split_a(const float* A, int M, int K, int lda, void* a_planes, cudaStream_t st, int total = 0,
                   int r0 = 0);
int fp16x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, cudaStream_t st, int total = 0,
                   int c0 = 0, bool packed = false);
int fp16x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K, int ldc,
                       cudaStream_t st, int a_total = 0, int r0 = 0, int b_total = 0, int c0 = 0,
                       FixArgs* fix = nullptr);
unsigned int* fp16x3_planes_flags(const void* buf, int total, int K);
// Range-guard fix-up after a planes GEMM (tf32x3_gemm.cu, k_tc_fixup): the
// rows / columns the splits marked are recomputed from the fp32 operands A
// (rows [r0, r0+M) of the planes' operand, lda) and B (columns [c0, c0+N);
// row-major with ldb, or packedB panels of those columns)
int tc_fixup_planes(bool f16, const void* a_planes, const void* b_planes, const float* A, int lda, const float* B,
                    int ldb, bool b_packed, float* C, int ldc, int M, int N, int K, cudaStream_t st, int a_total = 0,
                    int r0 = 0, int b_total = 0, int c0 = 0);

// binomial filter (stencil.cu)
int launch_binomial(int variant, const float* img, float* out, int H, int W, int ldi, int ldo,
                    cudaStream_t st);

}  // namespace elv
