// extern "C" boundary of libelevate_b200 (declared in include/elevate_b200.h).
//
// Replaces the evaluation of the seven scheduled `mm` terms by the reference
// interpreter (reference pkg/src/stratir/interp.py:157-162, `run`) with
// sm_100a kernels.  Plain pointers, sizes and a cudaStream_t only: no torch
// types cross this boundary.  Errors are reported as negative codes with a
// thread-local message (elv_last_error), never by aborting.

#include "elv_common.cuh"

#include <dlfcn.h>
#include <string.h>
#include <map>
#include <cmath>
#include <algorithm>
#include <mutex>
#include <vector>

namespace elv {

static thread_local char g_err[512] = "";

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ELV_PDL");
    v = e ? (atoi(e) != 0) : 1;
  }
  return v != 0;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  return ELV_OK;
}

// ---------------------------------------------------------------------------
// synthetic inputs: counter-based, identical on the host
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void k_fill_uniform(float* __restrict__ X, long long n, uint64_t key, long long offset) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const uint64_t h = splitmix64(key ^ (uint64_t)(offset + i));
    const int m = (int)(h >> 40);                 // 24 random bits
    X[i] = (float)(m - (1 << 23)) * (1.0f / (float)(1 << 23));   // exact: [-1, 1)
  }
}

// hi = rna_tf32(x); lo = rna_tf32(x - hi)  (x - hi is exact in fp32)
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void k_split_tf32(const float* __restrict__ X, float* __restrict__ hi,
                             float* __restrict__ lo, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float x = X[i];
    const float h = tf32_rna(x);
    hi[i] = h;
    lo[i] = tf32_rna(x - h);
  }
}

int launch_split_tf32(const float* X, float* hi, float* lo, long long n, cudaStream_t st) {
  long long blocks = (n + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  k_split_tf32<<<(unsigned)blocks, 256, 0, st>>>(X, hi, lo, n);
  return check_launch("split_tf32");
}

// ---------------------------------------------------------------------------
// NCCL, resolved lazily with dlopen so the library loads without it.  The
// soname libnccl.so.2 resolves to the copy torch already loaded, if any.
typedef int ncclResult_t_;
typedef struct { char internal[128]; } ncclUniqueId_;
typedef void* ncclComm_t_;
enum { ncclFloat32_ = 7 };
struct NcclApi {
  void* h = nullptr;
  ncclResult_t_ (*CommInitAll)(ncclComm_t_*, int, const int*) = nullptr;
  ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
  ncclResult_t_ (*Broadcast)(const void*, void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*GroupStart)() = nullptr;
  ncclResult_t_ (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t_) = nullptr;
};
static NcclApi g_nccl;
static std::vector<ncclComm_t_> g_comms;
static std::vector<int> g_comm_devs;
static std::mutex g_nccl_mu;

static int nccl_load() {
  if (g_nccl.h) return ELV_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return set_error(ELV_ENCCL, "dlopen(libnccl.so.2) failed: %s", dlerror());
  g_nccl.CommInitAll = (decltype(g_nccl.CommInitAll))dlsym(h, "ncclCommInitAll");
  g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
  g_nccl.Broadcast = (decltype(g_nccl.Broadcast))dlsym(h, "ncclBroadcast");
  g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
  g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
  g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
  if (!g_nccl.CommInitAll || !g_nccl.CommDestroy || !g_nccl.Broadcast || !g_nccl.GroupStart ||
      !g_nccl.GroupEnd)
    return set_error(ELV_ENCCL, "libnccl.so.2 lacks a required symbol");
  g_nccl.h = h;
  return ELV_OK;
}

static int nccl_err(ncclResult_t_ r, const char* what) {
  return set_error(ELV_ENCCL, "%s: %s", what,
                   g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
}

}  // namespace elv

using namespace elv;

static bool bad_ptr(const void* p) { return p == nullptr; }

extern "C" {

const char* elv_last_error(void) { return g_err; }
int elv_abi_version(void) { return ELV_ABI_VERSION; }

const char* elv_variant_name(int v) {
  static const char* names[ELV_NUM_VARIANTS] = {
      "baseline", "blocking", "vectorized", "loopPerm", "arrayPacking",
      "cacheBlocks", "parallel", "parallel_tf32x3", "parallel_fp16x3"};
  return (v >= 0 && v < ELV_NUM_VARIANTS) ? names[v] : "unknown";
}

size_t elv_pack_b_bytes(int K, int N) {
  if (K < 1 || N < 1) return 0;
  return packed_cols(N) * (size_t)K * sizeof(float);
}

size_t elv_gemm_workspace_bytes(int variant, int M, int N, int K) {
  if (M < 1 || N < 1 || K < 1) return 0;
  switch (variant) {
    case ELV_ARRAYPACKING:
    case ELV_CACHEBLOCKS: return elv_pack_b_bytes(K, N);
    case ELV_PARALLEL:
      return elv_pack_b_bytes(K, N) + (parallel_uses_packed_a(M, N) ? pack_a_bytes(M, K) : 0);
    case ELV_PARALLEL_TF32X3: return tf32x3_workspace_bytes(M, N, K);
    case ELV_PARALLEL_FP16X3: return fp16x3_workspace_bytes(M, N, K);
    default: return 0;
  }
}

static int check_args(const float* A, const float* B, const float* C, int M, int N, int K,
                      int lda, int ldb, int ldc, bool need_ldb) {
  if (bad_ptr(A) || bad_ptr(B) || bad_ptr(C))
    return set_error(ELV_EINVAL, "null matrix pointer");
  if (M < 1 || N < 1 || K < 1)
    return set_error(ELV_EINVAL, "sizes must be positive (M=%d N=%d K=%d)", M, N, K);
  if (lda < K || (need_ldb && ldb < N) || ldc < N)
    return set_error(ELV_EINVAL, "leading dimension too small (lda=%d ldb=%d ldc=%d)", lda, ldb, ldc);
  return ELV_OK;
}

int elv_pack_b(const float* B, float* packedB, int K, int N, int ldb, int blk, void* stream) {
  if (blk != kPanel) return set_error(ELV_EINVAL, "pack_b: block %d unsupported (32 only)", blk);
  if (bad_ptr(B) || bad_ptr(packedB)) return set_error(ELV_EINVAL, "pack_b: null pointer");
  if (K < 1 || N < 1 || ldb < N) return set_error(ELV_EINVAL, "pack_b: bad shape");
  return launch_pack_b(B, packedB, K, N, ldb, (cudaStream_t)stream);
}

int elv_split_tf32(const float* X, float* hi, float* lo, long long n, void* stream) {
  if (bad_ptr(X) || bad_ptr(hi) || bad_ptr(lo) || n < 0)
    return set_error(ELV_EINVAL, "split_tf32: bad arguments");
  if (n == 0) return ELV_OK;
  return launch_split_tf32(X, hi, lo, n, (cudaStream_t)stream);
}

int elv_fill_uniform(float* X, long long n, unsigned long long seed, unsigned int tensor_id,
                     long long offset, void* stream) {
  if (bad_ptr(X) || n < 0 || offset < 0) return set_error(ELV_EINVAL, "fill_uniform: bad arguments");
  if (n == 0) return ELV_OK;
  const uint64_t key = (seed << 48) ^ ((uint64_t)tensor_id << 40);
  long long blocks = (n + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  k_fill_uniform<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(X, n, key, offset);
  return check_launch("fill_uniform");
}

int elv_gemm_prepacked(int variant, const float* A, const float* packedB, float* C,
                       int M, int N, int K, int lda, int ldc, void* stream) {
  int rc = check_args(A, packedB, C, M, N, K, lda, 0, ldc, false);
  if (rc) return rc;
  if (variant != ELV_ARRAYPACKING && variant != ELV_CACHEBLOCKS && variant != ELV_PARALLEL)
    return set_error(ELV_EVARIANT, "gemm_prepacked: variant %d does not consume packedB", variant);
  return launch_simt(variant, A, nullptr, packedB, C, M, N, K, lda, 0, ldc, (cudaStream_t)stream);
}

static int check_variant_ws(int variant, int M, int N, int K, void* workspace, size_t workspace_bytes) {
  if (variant < 0 || variant >= ELV_NUM_VARIANTS)
    return set_error(ELV_EVARIANT, "unknown variant %d", variant);
  const size_t need = elv_gemm_workspace_bytes(variant, M, N, K);
  if (need > 0 && (workspace == nullptr || workspace_bytes < need))
    return set_error(ELV_EWORKSPACE, "variant %s needs %zu workspace bytes, got %zu",
                     elv_variant_name(variant), need, workspace_bytes);
  return ELV_OK;
}

int elv_gemm_prepare(int variant, const float* A, const float* B, int M, int N, int K, int lda,
                     int ldb, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_args(A, B, B, M, N, K, lda, ldb, N, true);
  if (!rc) rc = check_variant_ws(variant, M, N, K, workspace, workspace_bytes);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  switch (variant) {
    case ELV_ARRAYPACKING:
    case ELV_CACHEBLOCKS:
      return launch_pack_b(B, static_cast<float*>(workspace), K, N, ldb, st);
    case ELV_PARALLEL:
      if (!parallel_uses_packed_a(M, N)) return launch_pack_b(B, static_cast<float*>(workspace), K, N, ldb, st);
      return launch_pack_ab(B, static_cast<float*>(workspace), K, N, ldb, A,
                            reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + elv_pack_b_bytes(K, N)), M,
                            lda, st);
    case ELV_PARALLEL_TF32X3:
      return tf32x3_prepare(A, B, M, N, K, lda, ldb, workspace, workspace_bytes, st);
    case ELV_PARALLEL_FP16X3:
      return fp16x3_prepare(A, B, M, N, K, lda, ldb, workspace, workspace_bytes, st);
    default:
      return ELV_OK;   // 0..3 read A and B in place
  }
}

int elv_gemm_compute(int variant, const float* A, const float* B, float* C, int M, int N, int K,
                     int lda, int ldb, int ldc, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_args(A, B, C, M, N, K, lda, ldb, ldc, true);
  if (!rc) rc = check_variant_ws(variant, M, N, K, workspace, workspace_bytes);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  switch (variant) {
    case ELV_BASELINE:
    case ELV_BLOCKING:
    case ELV_VECTORIZED:
    case ELV_LOOPPERM:
      return launch_simt(variant, A, B, nullptr, C, M, N, K, lda, ldb, ldc, st);
    case ELV_PARALLEL:
      if (parallel_uses_packed_a(M, N))
        return launch_parallel_packed(
            reinterpret_cast<const float*>(static_cast<const uint8_t*>(workspace) + elv_pack_b_bytes(K, N)),
            static_cast<const float*>(workspace), C, M, N, K, ldc, st);
      return launch_simt(variant, A, nullptr, static_cast<const float*>(workspace), C, M, N, K, lda, 0,
                         ldc, st);
    case ELV_ARRAYPACKING:
    case ELV_CACHEBLOCKS:
      return launch_simt(variant, A, nullptr, static_cast<const float*>(workspace), C, M, N, K, lda, 0,
                         ldc, st);
    case ELV_PARALLEL_TF32X3:
      return tf32x3_compute(A, B, lda, ldb, C, M, N, K, ldc, workspace, workspace_bytes, st);
    case ELV_PARALLEL_FP16X3:
      return fp16x3_compute(A, B, lda, ldb, C, M, N, K, ldc, workspace, workspace_bytes, st);
  }
  return set_error(ELV_EVARIANT, "unknown variant %d", variant);
}

int elv_gemm(int variant, const float* A, const float* B, float* C, int M, int N, int K,
             int lda, int ldb, int ldc, void* workspace, size_t workspace_bytes, void* stream) {
  int rc = check_args(A, B, C, M, N, K, lda, ldb, ldc, true);
  if (rc) return rc;
  rc = elv_gemm_prepare(variant, A, B, M, N, K, lda, ldb, workspace, workspace_bytes, stream);
  if (rc) return rc;
  return elv_gemm_compute(variant, A, B, C, M, N, K, lda, ldb, ldc, workspace, workspace_bytes, stream);
}

size_t elv_tf32x3_a_planes_bytes(int M, int K) {
  return (M < 1 || K < 1) ? 0 : tf32x3_a_planes_bytes(M, K);
}
size_t elv_tf32x3_b_planes_bytes(int N, int K) {
  return (N < 1 || K < 1) ? 0 : tf32x3_b_planes_bytes(N, K);
}

int elv_tf32x3_split_a(const float* A, int M, int K, int lda, void* a_planes, void* stream) {
  if (bad_ptr(A) || bad_ptr(a_planes) || M < 1 || K < 1 || lda < K)
    return set_error(ELV_EINVAL, "tf32x3_split_a: bad arguments");
  return tf32x3_split_a(A, M, K, lda, a_planes, (cudaStream_t)stream);
}

int elv_tf32x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, void* stream) {
  if (bad_ptr(B) || bad_ptr(b_planes) || N < 1 || K < 1 || ldb < N)
    return set_error(ELV_EINVAL, "tf32x3_split_b: bad arguments");
  return tf32x3_split_b(B, K, N, ldb, false, b_planes, (cudaStream_t)stream);
}

int elv_tf32x3_split_b_packed(const float* packedB, int K, int N, void* b_planes, void* stream) {
  if (bad_ptr(packedB) || bad_ptr(b_planes) || N < 1 || K < 1)
    return set_error(ELV_EINVAL, "tf32x3_split_b_packed: bad arguments");
  return tf32x3_split_b(packedB, K, N, 0, true, b_planes, (cudaStream_t)stream);
}

int elv_tf32x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K,
                           int ldc, void* stream) {
  if (bad_ptr(a_planes) || bad_ptr(b_planes) || bad_ptr(C) || M < 1 || N < 1 || K < 1 || ldc < N)
    return set_error(ELV_EINVAL, "tf32x3_gemm_planes: bad arguments");
  return tf32x3_gemm_planes(a_planes, b_planes, C, M, N, K, ldc, (cudaStream_t)stream);
}

size_t elv_fp16x3_a_planes_bytes(int M, int K) { return (M < 1 || K < 1) ? 0 : fp16x3_a_planes_bytes(M, K); }
size_t elv_fp16x3_b_planes_bytes(int N, int K) { return (N < 1 || K < 1) ? 0 : fp16x3_b_planes_bytes(N, K); }
int elv_fp16x3_applicable(int M, int N, int K) { return (M > 0 && N > 0 && K > 0) ? fp16x3_applicable(M, N, K) : 0; }

int elv_fp16x3_split_a(const float* A, int M, int K, int lda, void* a_planes, void* stream) {
  if (bad_ptr(A) || bad_ptr(a_planes) || M < 1 || K < 1 || lda < K)
    return set_error(ELV_EINVAL, "fp16x3_split_a: bad arguments");
  return fp16x3_split_a(A, M, K, lda, a_planes, (cudaStream_t)stream);
}

int elv_fp16x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, void* stream) {
  if (bad_ptr(B) || bad_ptr(b_planes) || N < 1 || K < 1 || ldb < N)
    return set_error(ELV_EINVAL, "fp16x3_split_b: bad arguments");
  return fp16x3_split_b(B, K, N, ldb, b_planes, (cudaStream_t)stream);
}

int elv_fp16x3_split_b_packed(const float* packedB, int K, int N, void* b_planes, void* stream) {
  if (bad_ptr(packedB) || bad_ptr(b_planes) || N < 1 || K < 1)
    return set_error(ELV_EINVAL, "fp16x3_split_b_packed: bad arguments");
  return fp16x3_split_b(packedB, K, N, 0, b_planes, (cudaStream_t)stream, 0, 0, true);
}

int elv_fp16x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K, int ldc,
                           void* stream) {
  if (bad_ptr(a_planes) || bad_ptr(b_planes) || bad_ptr(C) || M < 1 || N < 1 || K < 1 || ldc < N)
    return set_error(ELV_EINVAL, "fp16x3_gemm_planes: bad arguments");
  return fp16x3_gemm_planes(a_planes, b_planes, C, M, N, K, ldc, (cudaStream_t)stream);
}

int elv_tc_kernel_choice(int M, int N, int sms, int* bn) {
  if (M < 1 || N < 1 || sms < 2) return ELV_EINVAL;
  return tc_kernel_choice(M, N, sms, bn);
}

int elv_tf32x3_fused_ok(const float* A, int lda, const float* B, int ldb, int M, int N) {
  if (bad_ptr(A) || bad_ptr(B) || M < 1 || N < 1) return 0;
  return tf32x3_fused_ok(A, lda, B, ldb, M, N) ? 1 : 0;
}

int elv_tf32x3_gemm_fused(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N, int K,
                          unsigned int* flags, void* stream) {
  int rc = check_args(A, B, C, M, N, K, lda, ldb, ldc, true);
  if (rc) return rc;
  if (bad_ptr(flags)) return set_error(ELV_EINVAL, "tf32x3_gemm_fused: null flags");
  if (!tf32x3_fused_ok(A, lda, B, ldb, M, N))
    return set_error(ELV_EINVAL, "tf32x3_gemm_fused: not applicable (needs the pair kernel -- the pair / 1-CTA model -- and 16 B alignment)");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(flags, 0, (size_t)(M + N) * 4, st) != cudaSuccess)
    return set_error(ELV_ECUDA, "tf32x3_gemm_fused: memset");
  rc = tf32x3_gemm_fused(A, lda, B, ldb, C, ldc, M, N, K, flags, flags + M, st);
  if (rc) return rc;
  return tc_fixup(A, lda, B, ldb, false, C, ldc, M, N, K, flags, flags + M, st);
}

int elv_tf32x3_gemm_fused_a(const float* A, int lda, const void* b_planes, const float* B, int ldb, float* C,
                            int ldc, int M, int N, int K, unsigned int* flags_a, void* stream) {
  int rc = check_args(A, B, C, M, N, K, lda, ldb, ldc, true);
  if (rc) return rc;
  if (bad_ptr(flags_a) || bad_ptr(b_planes)) return set_error(ELV_EINVAL, "tf32x3_gemm_fused_a: null pointer");
  if (!tf32x3_fused_a_ok(A, lda, M, N))
    return set_error(ELV_EINVAL, "tf32x3_gemm_fused_a: not applicable (needs the pair kernel -- the pair / 1-CTA model -- and a 16 B aligned A)");
  cudaStream_t st = (cudaStream_t)stream;
  if (cudaMemsetAsync(flags_a, 0, (size_t)M * 4, st) != cudaSuccess)
    return set_error(ELV_ECUDA, "tf32x3_gemm_fused_a: memset");
  const unsigned int* flag_b = tf32x3_b_planes_flags(b_planes, N, K);
  rc = tf32x3_gemm_fused(A, lda, nullptr, 0, C, ldc, M, N, K, flags_a, const_cast<unsigned int*>(flag_b), st,
                         b_planes, N, 0);
  if (rc) return rc;
  return tc_fixup(A, lda, B, ldb, false, C, ldc, M, N, K, flags_a, flag_b, st);
}

int elv_tc_fixup(int encoding, const void* a_planes, const void* b_planes, const float* A, int lda, const float* B,
                 int ldb, int b_packed, float* C, int ldc, int M, int N, int K, void* stream) {
  if (encoding != ELV_PARALLEL_TF32X3 && encoding != ELV_PARALLEL_FP16X3)
    return set_error(ELV_EINVAL, "tc_fixup: encoding must be 7 (tf32) or 8 (fp16)");
  if (bad_ptr(a_planes) || bad_ptr(b_planes) || bad_ptr(A) || bad_ptr(B) || bad_ptr(C) || M < 1 || N < 1 ||
      K < 1 || lda < K || ldc < N || (!b_packed && ldb < N))
    return set_error(ELV_EINVAL, "tc_fixup: bad arguments");
  return tc_fixup_planes(encoding == ELV_PARALLEL_FP16X3, a_planes, b_planes, A, lda, B, ldb, b_packed != 0, C, ldc,
                         M, N, K, (cudaStream_t)stream);
}

const char* elv_binomial_variant_name(int v) {
  static const char* names[ELV_BF_NUM_VARIANTS] = {"naive", "naivePar", "separated", "separatedPar"};
  return (v >= 0 && v < ELV_BF_NUM_VARIANTS) ? names[v] : "unknown";
}

int elv_binomial(int variant, const float* img, float* out, int H, int W, int ld_in, int ld_out,
                 void* stream) {
  if (bad_ptr(img) || bad_ptr(out)) return set_error(ELV_EINVAL, "binomial: null pointer");
  if (H < 1 || W < 1 || ld_in < W || ld_out < W)
    return set_error(ELV_EINVAL, "binomial: bad shape (H=%d W=%d ld_in=%d ld_out=%d)", H, W, ld_in, ld_out);
  if (variant < 0 || variant >= ELV_BF_NUM_VARIANTS)
    return set_error(ELV_EVARIANT, "binomial: unknown variant %d", variant);
  return launch_binomial(variant, img, out, H, W, ld_in, ld_out, (cudaStream_t)stream);
}

int elv_nccl_init(int ndev, const int* devs) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (ndev < 1 || devs == nullptr) return set_error(ELV_EINVAL, "nccl_init: bad device list");
  int rc = nccl_load();
  if (rc) return rc;
  for (auto c : g_comms) g_nccl.CommDestroy(c);
  g_comms.assign(ndev, nullptr);
  g_comm_devs.assign(devs, devs + ndev);
  ncclResult_t_ r = g_nccl.CommInitAll(g_comms.data(), ndev, devs);
  if (r != 0) {
    g_comms.clear();
    g_comm_devs.clear();
    return nccl_err(r, "ncclCommInitAll");
  }
  return ELV_OK;
}

int elv_nccl_destroy(void) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  for (auto c : g_comms) if (g_nccl.CommDestroy) g_nccl.CommDestroy(c);
  g_comms.clear();
  g_comm_devs.clear();
  return ELV_OK;
}

int elv_gemm_rowshard(int variant, int ndev, const int* devs, const float* const* A_shards,
                      float* const* B_per_dev, float* const* packedB_per_dev,
                      float* const* C_shards, const int* rows, int N, int K,
                      void* const* streams) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (variant != ELV_ARRAYPACKING && variant != ELV_CACHEBLOCKS && variant != ELV_PARALLEL)
    return set_error(ELV_EVARIANT, "gemm_rowshard: variant %d not supported (4..6)", variant);
  if (ndev < 1 || !devs || !A_shards || !B_per_dev || !packedB_per_dev || !C_shards || !rows ||
      !streams || N < 1 || K < 1)
    return set_error(ELV_EINVAL, "gemm_rowshard: bad arguments");
  if ((int)g_comms.size() != ndev) return set_error(ELV_ENCCL, "gemm_rowshard: call elv_nccl_init first");
  for (int d = 0; d < ndev; ++d)
    if (g_comm_devs[d] != devs[d]) return set_error(ELV_ENCCL, "gemm_rowshard: device list differs from elv_nccl_init");
  int prev = 0;
  cudaGetDevice(&prev);
  const size_t count = (size_t)K * N;
  // B lives in B_per_dev[0] on devs[0]: broadcast it to every device
  ncclResult_t_ r = g_nccl.GroupStart();
  if (r != 0) return nccl_err(r, "ncclGroupStart");
  for (int d = 0; d < ndev; ++d) {
    cudaSetDevice(devs[d]);
    r = g_nccl.Broadcast(B_per_dev[0], B_per_dev[d], count, ncclFloat32_, 0, g_comms[d],
                         (cudaStream_t)streams[d]);
    if (r != 0) { g_nccl.GroupEnd(); cudaSetDevice(prev); return nccl_err(r, "ncclBroadcast"); }
  }
  r = g_nccl.GroupEnd();
  if (r != 0) { cudaSetDevice(prev); return nccl_err(r, "ncclGroupEnd"); }
  for (int d = 0; d < ndev; ++d) {
    cudaSetDevice(devs[d]);
    if (rows[d] <= 0) continue;
    int rc = launch_pack_b(B_per_dev[d], packedB_per_dev[d], K, N, N, (cudaStream_t)streams[d]);
    if (!rc) rc = launch_simt(variant, A_shards[d], nullptr, packedB_per_dev[d], C_shards[d],
                              rows[d], N, K, K, 0, N, (cudaStream_t)streams[d]);
    if (rc) { cudaSetDevice(prev); return rc; }
  }
  cudaSetDevice(prev);
  return ELV_OK;
}


// ---------------------------------------------------------------------------
// Pipelined single-process row shard (variants 4..8): the C-ABI mirror of
// distributed.PipelinedRowShardGemm for callers without Python.  B (row-major,
// on devs[0]) is packed and NCCL-broadcast in column chunks (the first half
// the size of the others: nothing hides its broadcast); on every device a
// side stream splits each packed chunk into the tensor-core planes as soon as
// it lands (variants 7, 8) while the compute stream multiplies the previous
// chunk; the SIMT variants multiply the packed chunk directly.  Column blocks
// of C are independent and the kernels' per-element arithmetic does not
// depend on the chunking, so C is bitwise elv_gemm's.
static std::vector<std::pair<int, int>> column_chunks(int N, int chunks) {
  const int align = 256;
  const int units = (N + align - 1) / align;
  chunks = std::max(1, std::min(chunks, units));
  std::vector<double> w(chunks, 1.0);
  if (chunks > 1) w[0] = 0.5;
  double tot = 0;
  for (double x : w) tot += x;
  std::vector<int> bounds{0};
  double acc = 0;
  for (int c = 0; c + 1 < chunks; ++c) {
    acc += w[c];
    int b = (int)std::lround(units * acc / tot);
    b = std::min(std::max(b, bounds.back() + 1), units - (chunks - (int)bounds.size()));
    bounds.push_back(b);
  }
  bounds.push_back(units);
  std::vector<std::pair<int, int>> out;
  for (size_t c = 0; c + 1 < bounds.size(); ++c) {
    const int n0 = bounds[c] * align, n1 = std::min(bounds[c + 1] * align, N);
    if (n1 > n0) out.push_back({n0, n1});
  }
  return out;
}

static inline size_t up256(size_t x) { return (x + 255) / 256 * 256; }

// tensor-core encoding the pipeline runs for `variant` (fp16 needs K >= 512 in every chunk GEMM)
static int rowshard_tc(int variant, int rows, int K, const std::vector<std::pair<int, int>>& ch) {
  if (variant == ELV_PARALLEL_FP16X3) {
    for (auto& c : ch)
      if (!fp16x3_applicable(std::max(rows, 1), c.second - c.first, K)) return ELV_PARALLEL_TF32X3;
    return ELV_PARALLEL_FP16X3;
  }
  return variant == ELV_PARALLEL_TF32X3 ? ELV_PARALLEL_TF32X3 : 0;
}

size_t elv_gemm_rowshard_workspace_bytes(int variant, int rows, int N, int K, int chunks) {
  if (rows < 1 || N < 1 || K < 1 || chunks < 1) return 0;
  const auto ch = column_chunks(N, chunks);
  const int tc = rowshard_tc(variant, rows, K, ch);
  if (!tc) return 0;
  const bool f16 = tc == ELV_PARALLEL_FP16X3;
  size_t b = up256(f16 ? fp16x3_a_planes_bytes(rows, K) : tf32x3_a_planes_bytes(rows, K));
  for (auto& c : ch) {
    const int nc = c.second - c.first;
    b += up256(f16 ? fp16x3_b_planes_bytes(nc, K) : tf32x3_b_planes_bytes(nc, K));
  }
  return b;
}

struct RsStreams { cudaStream_t comm = nullptr, prep = nullptr; };
static std::map<int, RsStreams> g_rs_streams;     // per device, created once

int elv_gemm_rowshard_pipelined(int variant, int ndev, const int* devs, const float* const* A_shards,
                                const float* B_root, float* const* packedB_per_dev, float* const* C_shards,
                                const int* rows, int N, int K, int chunks, void* const* workspaces,
                                size_t workspace_bytes, void* const* streams) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (variant < ELV_ARRAYPACKING || variant > ELV_PARALLEL_FP16X3)
    return set_error(ELV_EVARIANT, "gemm_rowshard_pipelined: variant %d not supported (4..8)", variant);
  if (ndev < 1 || !devs || !A_shards || !B_root || !packedB_per_dev || !C_shards || !rows || !streams ||
      N < 1 || K < 1 || chunks < 1)
    return set_error(ELV_EINVAL, "gemm_rowshard_pipelined: bad arguments");
  if ((int)g_comms.size() != ndev) return set_error(ELV_ENCCL, "gemm_rowshard_pipelined: call elv_nccl_init first");
  for (int d = 0; d < ndev; ++d)
    if (g_comm_devs[d] != devs[d])
      return set_error(ELV_ENCCL, "gemm_rowshard_pipelined: device list differs from elv_nccl_init");
  const auto ch = column_chunks(N, chunks);
  const int nch = (int)ch.size();
  int max_rows = 1;
  for (int d = 0; d < ndev; ++d) max_rows = std::max(max_rows, rows[d]);
  const int tc = rowshard_tc(variant, max_rows, K, ch);
  const bool f16 = tc == ELV_PARALLEL_FP16X3;
  if (tc) {
    if (!workspaces) return set_error(ELV_EWORKSPACE, "gemm_rowshard_pipelined: workspaces required");
    for (int d = 0; d < ndev; ++d)
      if (rows[d] > 0 && (!workspaces[d] ||
                          workspace_bytes < elv_gemm_rowshard_workspace_bytes(variant, max_rows, N, K, chunks)))
        return set_error(ELV_EWORKSPACE, "gemm_rowshard_pipelined: workspace too small");
  }
  int prev = 0;
  cudaGetDevice(&prev);
  int rc = ELV_OK;
  std::vector<cudaEvent_t> evs;                    // destroyed at the end (released once their work completes)
  auto event = [&](cudaEvent_t* e) {
    if (cudaEventCreateWithFlags(e, cudaEventDisableTiming) != cudaSuccess) return false;
    evs.push_back(*e);
    return true;
  };
  auto fail = [&](int code) { rc = code; };
  std::vector<RsStreams> S(ndev);
  std::vector<cudaEvent_t> entry(ndev);
  for (int d = 0; d < ndev && !rc; ++d) {
    cudaSetDevice(devs[d]);
    RsStreams& r = g_rs_streams[devs[d]];
    if (!r.comm) {
      if (cudaStreamCreateWithFlags(&r.comm, cudaStreamNonBlocking) != cudaSuccess ||
          cudaStreamCreateWithFlags(&r.prep, cudaStreamNonBlocking) != cudaSuccess)
        fail(set_error(ELV_ECUDA, "gemm_rowshard_pipelined: stream creation"));
    }
    S[d] = r;
    // the side streams start after the caller's earlier work on these buffers
    if (!rc && (!event(&entry[d]) || cudaEventRecord(entry[d], (cudaStream_t)streams[d]) != cudaSuccess ||
                cudaStreamWaitEvent(r.comm, entry[d], 0) != cudaSuccess ||
                cudaStreamWaitEvent(r.prep, entry[d], 0) != cudaSuccess))
      fail(set_error(ELV_ECUDA, "gemm_rowshard_pipelined: entry event"));
  }
  // root: pack each chunk; every device: broadcast it (one NCCL group per chunk)
  std::vector<std::vector<cudaEvent_t>> landed(ndev, std::vector<cudaEvent_t>(nch));
  for (int c = 0; c < nch && !rc; ++c) {
    const int n0 = ch[c].first, nc = ch[c].second - ch[c].first;
    const size_t panel = (size_t)(n0 / 32) * K * 32, count = (size_t)((nc + 255) / 256) * 256 * K;
    cudaSetDevice(devs[0]);
    cudaEvent_t packed;
    if ((rc = launch_pack_b(B_root + n0, packedB_per_dev[0] + panel, K, nc, N, (cudaStream_t)streams[0]))) break;
    if (!event(&packed) || cudaEventRecord(packed, (cudaStream_t)streams[0]) != cudaSuccess) {
      fail(set_error(ELV_ECUDA, "gemm_rowshard_pipelined: pack event"));
      break;
    }
    for (int d = 0; d < ndev; ++d) {
      cudaSetDevice(devs[d]);
      cudaStreamWaitEvent(S[d].comm, packed, 0);
    }
    ncclResult_t_ r = g_nccl.GroupStart();
    if (r != 0) { fail(nccl_err(r, "ncclGroupStart")); break; }
    for (int d = 0; d < ndev && !r; ++d) {
      cudaSetDevice(devs[d]);
      r = g_nccl.Broadcast(packedB_per_dev[0] + panel, packedB_per_dev[d] + panel, count, ncclFloat32_, 0, g_comms[d],
                           S[d].comm);
    }
    const ncclResult_t_ r2 = g_nccl.GroupEnd();
    if (r != 0 || r2 != 0) { fail(nccl_err(r ? r : r2, "ncclBroadcast")); break; }
    for (int d = 0; d < ndev && !rc; ++d) {
      cudaSetDevice(devs[d]);
      if (!event(&landed[d][c]) || cudaEventRecord(landed[d][c], S[d].comm) != cudaSuccess)
        fail(set_error(ELV_ECUDA, "gemm_rowshard_pipelined: broadcast event"));
    }
  }
  // every device: (split chunk c on the side stream) -> GEMM chunk c (+ fix-up)
  for (int d = 0; d < ndev && !rc; ++d) {
    cudaSetDevice(devs[d]);
    cudaStream_t st = (cudaStream_t)streams[d];
    const int m = rows[d];
    if (m <= 0) {
      for (int c = 0; c < nch; ++c) cudaStreamWaitEvent(st, landed[d][c], 0);
      continue;
    }
    const float* P = packedB_per_dev[d];
    float* Cd = C_shards[d];
    if (!tc) {
      for (int c = 0; c < nch && !rc; ++c) {
        const int n0 = ch[c].first, nc = ch[c].second - ch[c].first;
        cudaStreamWaitEvent(st, landed[d][c], 0);
        rc = launch_simt(variant, A_shards[d], nullptr, P + (size_t)(n0 / 32) * K * 32, Cd + n0, m, nc, K, K, 0, N,
                         st);
      }
      continue;
    }
    uint8_t* ws = static_cast<uint8_t*>(workspaces[d]);
    void* ap = ws;
    size_t off = up256(f16 ? fp16x3_a_planes_bytes(max_rows, K) : tf32x3_a_planes_bytes(max_rows, K));
    std::vector<void*> bp(nch);
    std::vector<cudaEvent_t> split(nch);
    for (int c = 0; c < nch && !rc; ++c) {
      const int n0 = ch[c].first, nc = ch[c].second - ch[c].first;
      bp[c] = ws + off;
      off += up256(f16 ? fp16x3_b_planes_bytes(nc, K) : tf32x3_b_planes_bytes(nc, K));
      cudaStreamWaitEvent(S[d].prep, landed[d][c], 0);
      const float* Pc = P + (size_t)(n0 / 32) * K * 32;
      rc = f16 ? fp16x3_split_b(Pc, K, nc, 0, bp[c], S[d].prep, 0, 0, true)
               : tf32x3_split_b(Pc, K, nc, 0, true, bp[c], S[d].prep);
      if (!rc && (!event(&split[c]) || cudaEventRecord(split[c], S[d].prep) != cudaSuccess))
        fail(set_error(ELV_ECUDA, "gemm_rowshard_pipelined: split event"));
    }
    if (rc) break;
    rc = f16 ? fp16x3_split_a(A_shards[d], m, K, K, ap, st) : tf32x3_split_a(A_shards[d], m, K, K, ap, st);
    for (int c = 0; c < nch && !rc; ++c) {
      const int n0 = ch[c].first, nc = ch[c].second - ch[c].first;
      cudaStreamWaitEvent(st, split[c], 0);
      rc = f16 ? fp16x3_gemm_planes(ap, bp[c], Cd + n0, m, nc, K, N, st)
               : tf32x3_gemm_planes(ap, bp[c], Cd + n0, m, nc, K, N, st);
      if (!rc)
        rc = tc_fixup_planes(f16, ap, bp[c], A_shards[d], K, P + (size_t)(n0 / 32) * K * 32, 0, true, Cd + n0, N, m,
                             nc, K, st);
    }
  }
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  cudaSetDevice(prev);
  return rc;
}
}  // extern "C"
