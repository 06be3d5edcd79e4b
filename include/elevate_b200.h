/*
 * elevate_b200.h -- C ABI of the B200 execution backend for the ELEVATE
 * (arXiv 2002.02268) GEMM hot path.
 *
 * The reference has no FFI: its hot path is the Python tree-walking
 * interpreter `stratir.interp.run(e, args)` (reference
 * pkg/src/stratir/interp.py:157-162) evaluating the rewritten `mm` term with
 * f64 scalars on nested lists.  Every entry point below replaces one piece of
 * that evaluation for the seven scheduled `mm` terms; the Python drop-in
 * (`paper_2002_02268_b200.interp.run`) decodes the term and binds these with
 * ctypes.  The shape of the calls follows the reference SPEC's codegen-c
 * contract `void fn(float* out, const float* in0, ...)` (reference
 * SPEC.md:525), extended with sizes, leading dimensions and a stream.
 *
 * Conventions
 *  - All matrices are fp32, row-major, device pointers.  C = A(MxK) . B(KxN).
 *  - The caller owns every buffer (A, B, C, workspace).  The library never
 *    allocates or frees user memory; size workspaces with
 *    elv_gemm_workspace_bytes().
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous on that stream.
 *  - Return value: ELV_OK (0) or a negative ELV_E* code; elv_last_error()
 *    returns a thread-local message for the last failure on this thread.
 *    The Python layer maps ELV_EINVAL/ELV_EVARIANT to the reference's
 *    EvalError (interp.py:16) and ELV_ECUDA/ELV_ENCCL to RuntimeError.
 */
#ifndef ELEVATE_B200_H
#define ELEVATE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ELV_ABI_VERSION 1

enum {
  ELV_OK = 0,
  ELV_EINVAL = -1,      /* bad size / pointer / leading dimension          */
  ELV_EVARIANT = -2,    /* unknown kernel variant                          */
  ELV_ECUDA = -3,       /* CUDA launch or runtime error                    */
  ELV_ENCCL = -4,       /* NCCL error (row-shard driver)                   */
  ELV_EWORKSPACE = -5   /* workspace missing or too small                  */
};

/* Kernel variants: one per ELEVATE/TVM schedule (reference PAPER.md:269-315;
 * SPEC.md:482-488), decoded from the lowered term by the dispatch. */
enum {
  ELV_BASELINE = 0,        /* mapSeq/mapSeq/reduceSeq: one thread per C(i,j)  */
  ELV_BLOCKING = 1,        /* tile(32,32) + split(4): 32x32 SMEM tiles        */
  ELV_VECTORIZED = 2,      /* + vectorize(32): 128-bit loads/stores           */
  ELV_LOOPPERM = 3,        /* + reorder: register outer-product micro-tiles   */
  ELV_ARRAYPACKING = 4,    /* + packB/toMem: GEMM over packedB[N/32][K][32]   */
  ELV_CACHEBLOCKS = 5,     /* + toMem(acc) + unroll: 8x8 register accumulators*/
  ELV_PARALLEL = 6,        /* + mapPar: persistent, double-buffered, 148 SMs  */
  ELV_PARALLEL_TF32X3 = 7, /* parallel term on tcgen05: 3xTF32, TMEM accum    */
  ELV_PARALLEL_FP16X3 = 8, /* same three products on scaled fp16 hi/lo planes:
                              half the bytes, kind::f16 (falls back to 7 for
                              K < 512)                                       */
  ELV_NUM_VARIANTS = 9
};

/* C = A . B with the kernel of `variant`.
 * Replaces interp.run(schedule(mm), [A, B]) (interp.py:157-162) for the
 * decoded schedule.  Variants 4..7 need a workspace (packed / split copies of
 * the operands); pass NULL/0 for 0..3.  Any M, N, K >= 1 (tails predicated).
 */
int elv_gemm(int variant, const float* A, const float* B, float* C,
             int M, int N, int K, int lda, int ldb, int ldc,
             void* workspace, size_t workspace_bytes, void* stream);

/* The two phases of elv_gemm, for callers that time or overlap them:
 * prepare = the operand layout transform into `workspace` (packB for 4..6,
 * the hi/lo split + K-major transpose for 7, nothing for 0..3);
 * compute = the GEMM kernel reading the prepared workspace.
 * elv_gemm == elv_gemm_prepare ; elv_gemm_compute on the same stream. */
int elv_gemm_prepare(int variant, const float* A, const float* B, int M, int N, int K,
                     int lda, int ldb, void* workspace, size_t workspace_bytes, void* stream);
int elv_gemm_compute(int variant, const float* A, const float* B, float* C,
                     int M, int N, int K, int lda, int ldb, int ldc,
                     void* workspace, size_t workspace_bytes, void* stream);

/* Bytes of workspace elv_gemm(variant, ...) needs at this shape. */
size_t elv_gemm_workspace_bytes(int variant, int M, int N, int K);

/* Same as elv_gemm for variants 4..6, but B is already packed by
 * elv_pack_b (used by the row-shard driver after a packedB broadcast). */
int elv_gemm_prepacked(int variant, const float* A, const float* packedB,
                       float* C, int M, int N, int K, int lda, int ldc,
                       void* stream);

/* packedB[p][k][c] = B[k][p*blk + c] (0 past N); p < ceil(N/256)*256/blk.
 * The toMem of the packB rule (reference rules.py:516-549; TVM packedB,
 * PAPER.md:49-50).  blk must be 32. */
int elv_pack_b(const float* B, float* packedB, int K, int N, int ldb, int blk,
               void* stream);
size_t elv_pack_b_bytes(int K, int N);

/* hi = rna_tf32(x), lo = rna_tf32(x - hi), elementwise over n floats. */
int elv_split_tf32(const float* X, float* hi, float* lo, long long n,
                   void* stream);

/* 3xTF32 building blocks (variant 7 split into its pieces, for pipelined and
 * row-sharded callers).  Planes = [hi | lo], each rows x Kp fp32, K-major,
 * Kp = K rounded up to 16, zero padded.  elv_gemm(7) == split_a ; split_b ;
 * gemm_planes.  split_b_packed reads packedB panels (elv_pack_b layout), so
 * a broadcast packedB chunk of Nc columns is split without unpacking. */
size_t elv_tf32x3_a_planes_bytes(int M, int K);
size_t elv_tf32x3_b_planes_bytes(int N, int K);
int elv_tf32x3_split_a(const float* A, int M, int K, int lda, void* a_planes, void* stream);
int elv_tf32x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, void* stream);
int elv_tf32x3_split_b_packed(const float* packedB, int K, int N, void* b_planes,
                              void* stream);
int elv_tf32x3_gemm_planes(const void* a_planes, const void* b_planes, float* C,
                           int M, int N, int K, int ldc, void* stream);

/* 3xTF32 with the split fused into the GEMM (no preparation pass): one
 * tcgen05 pair kernel reads raw fp32 A (M x K, lda) and B (K x N row-major,
 * ldb) by TMA and splits them in shared memory; bitwise the result of
 * split_a ; split_b ; gemm_planes.  Applicable (elv_tf32x3_fused_ok) when the
 * library runs the CTA-pair kernel at this shape (>= 148 256x256 tiles, or a
 * mid-size problem where its modelled mainloop beats the 1-CTA kernel's) and
 * A, B, lda, ldb are 16-byte aligned;
 * elv_gemm / elv_gemm_compute (variant 7) use it then only with
 * ELV_TF32X3_FUSED=1 (measured slower than the planes path).  `flags` is caller
 * scratch of (M + N) u32: zeroed and filled with the range-guard marks, and
 * the range-guard fix-up is run before returning (asynchronously on
 * `stream`). */
int elv_tf32x3_fused_ok(const float* A, int lda, const float* B, int ldb, int M, int N);

/* The tensor-core kernel the library picks by default for an M x N output
 * on a GPU with `sms` SMs (no environment overrides): 1 = the CTA-pair
 * kernel (one 256x256 tile per pair), 0 = the 1-CTA kernel, whose N tile
 * (256 / 128 / 64) is written to *bn when bn is not NULL; ELV_EINVAL for
 * bad sizes.  No device work: callers use it to count launches (the pair
 * kernel's range-guard fix-up is a separate launch). */
int elv_tc_kernel_choice(int M, int N, int sms, int* bn);
int elv_tf32x3_gemm_fused(const float* A, int lda, const float* B, int ldb, float* C, int ldc,
                          int M, int N, int K, unsigned int* flags, void* stream);
/* The same kernel with B already split (elv_tf32x3_split_b / _split_b_packed
 * planes of these N columns, e.g. a broadcast chunk split on arrival): only
 * A is split in the kernel.  B (row-major, ldb) is read only by the
 * range-guard fix-up; flags_a is caller scratch of M u32. */
int elv_tf32x3_gemm_fused_a(const float* A, int lda, const void* b_planes, const float* B, int ldb,
                            float* C, int ldc, int M, int N, int K, unsigned int* flags_a, void* stream);

/* Host-resident operands (the reference's own calling convention:
 * interp.run takes and returns host values, interp.py:157-162).
 * C_h = A_h . B_h; A_h, B_h, C_h are HOST pointers (pinned for overlap).
 * The output is cut into R x Nc tiles: B column chunks and A row blocks
 * cross PCIe on a library H2D stream in first-use order, each tile is
 * prepared and multiplied on `stream` as soon as its operands arrive, and
 * returns on a library D2H stream as soon as it is written.  Asynchronous on
 * `stream` (synchronise it before reading C_h).  Same per-element arithmetic
 * as elv_gemm.  The device workspace holds A, B, C and the per-tile
 * prepared operands: size it with elv_gemm_host_workspace_bytes. */
size_t elv_gemm_host_workspace_bytes(int variant, int M, int N, int K);
int elv_gemm_host(int variant, const float* A_h, const float* B_h, float* C_h,
                  int M, int N, int K, int lda, int ldb, int ldc,
                  void* workspace, size_t workspace_bytes, void* stream);
/* The tile shape elv_gemm_host uses (rows x cols); for the growing schedule
 * (tensor-core variants, large outputs) the A strip rows and B strip columns. */
int elv_gemm_host_tiles(int variant, int M, int N, int K, int* rows, int* cols);
/* Pitched copy (cudaMemcpy2DAsync): kind 1 = host->device, 2 = device->host,
 * 3 = device->device.  Used by the multi-GPU end-to-end path to move column
 * chunks of a row-major matrix. */
int elv_copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t height,
               int kind, void* stream);
/* Diagnostics: with ELV_HOST_TRACE=1 set, after the last elv_gemm_host on
 * this thread completed, write up to `cap` (kind, ms since entry) float pairs
 * (kind 0 = H2D item landed, 1 = tile GEMM done, 2 = tile D2H done). */
int elv_gemm_host_trace(float* out, int cap);

/* 3xFP16 building blocks (variant 8 in pieces, like the 3xTF32 ones above).
 * Planes = [hi | lo] fp16 rows x Kp (Kp = K rounded up to 64, K-major) plus
 * the per-row (A) / per-column (B) power-of-two scales.  split_b takes
 * row-major B (K x N, ldb) and writes B transposed.  gemm_planes requires
 * elv_fp16x3_applicable(M, N, K) (K >= 512). */
size_t elv_fp16x3_a_planes_bytes(int M, int K);
size_t elv_fp16x3_b_planes_bytes(int N, int K);
int elv_fp16x3_applicable(int M, int N, int K);
int elv_fp16x3_split_a(const float* A, int M, int K, int lda, void* a_planes, void* stream);
int elv_fp16x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, void* stream);
/* split_b from packedB panels (elv_pack_b layout) of N columns: what every
 * rank of the row-shard pipeline runs on a broadcast chunk */
int elv_fp16x3_split_b_packed(const float* packedB, int K, int N, void* b_planes, void* stream);
int elv_fp16x3_gemm_planes(const void* a_planes, const void* b_planes, float* C,
                           int M, int N, int K, int ldc, void* stream);

/* Range guard of the tensor-core encodings (variants 7 and 8).  The splits
 * mark every row of A / column of B holding an element outside the
 * encoding's exact window (non-finite; tf32: 0 < |x| < 2^-100; fp16: a
 * scaled value below fp16's normal range, i.e. more than 2^29 below its
 * row / column maximum).  elv_gemm / elv_gemm_compute and elv_gemm_host
 * recompute those rows and columns of C with the SIMT fp32 FMA chain
 * automatically; planes-API callers run elv_tc_fixup after gemm_planes with
 * the same operands in fp32 (A: M x K, lda; B: K x N row-major with ldb, or,
 * with b_packed = 1, packedB panels (elv_pack_b layout) of these N columns).
 * encoding: 7 (tf32 planes) or 8 (fp16 planes).  With nothing marked it is
 * one short launch. */
int elv_tc_fixup(int encoding, const void* a_planes, const void* b_planes, const float* A, int lda,
                 const float* B, int ldb, int b_packed, float* C, int ldc, int M, int N, int K,
                 void* stream);

/* Synthetic inputs: X[i] = U(-1,1) with 24-bit resolution from
 * splitmix64((seed << 48) ^ (tensor_id << 40) ^ (offset + i)); bit-identical
 * to paper_2002_02268_b200.synth.uniform() on the host. */
int elv_fill_uniform(float* X, long long n, unsigned long long seed,
                     unsigned int tensor_id, long long offset, void* stream);

/* Binomial filter, the paper's second data-parallel workload (reference
 * PAPER.md:1618-1770; separateDot rule, reference rules.py:462-513):
 * out = [1 2 1; 2 4 2; 1 2 1]/16 (*) clamp-padded img (pad2D(1) = padClamp,
 * interp.py:127-132; slide2D(3,1); map2D(dot)).  Replaces
 * interp.run(bf_schedule(bf), [img]) for the four binomial schedules.
 * img/out: H x W fp32 row-major device buffers (no aliasing). */
enum {
  ELV_BF_NAIVE = 0,          /* lowerToC(bf)                                  */
  ELV_BF_NAIVE_PAR = 1,      /* topDown(parallel) ; lowerToC                  */
  ELV_BF_SEPARATED = 2,      /* topDown(separateDot) ; lowerToC               */
  ELV_BF_SEPARATED_PAR = 3,  /* separateDot ; parallel ; lowerToC             */
  ELV_BF_NUM_VARIANTS = 4
};
int elv_binomial(int variant, const float* img, float* out, int H, int W,
                 int ld_in, int ld_out, void* stream);
const char* elv_binomial_variant_name(int variant);

/* Row-sharded GEMM over ndev GPUs in ONE process (mapPar(xo) of the parallel
 * schedule as the shard axis): B is broadcast from devs[0] with
 * NCCL (elv_nccl_init must have been called with the same devices), each
 * device packs it and computes its rows C_shards[d] = A_shards[d] . B.
 * rows[d] is the row count of shard d.  packedB_per_dev[d] and B_per_dev[d]
 * are caller-owned device buffers on device devs[d] (B_per_dev[0] == B root). */
int elv_nccl_init(int ndev, const int* devs);
int elv_nccl_destroy(void);
int elv_gemm_rowshard(int variant, int ndev, const int* devs,
                      const float* const* A_shards, float* const* B_per_dev,
                      float* const* packedB_per_dev, float* const* C_shards,
                      const int* rows, int N, int K, void* const* streams);

/* The pipelined row shard for variants 4..8 (the C-ABI mirror of the Python
 * PipelinedRowShardGemm; reference anchor: the mapPar(xo) shard axis,
 * PAPER.md:80).  B_root (K x N row-major on devs[0]) is packed and NCCL-
 * broadcast in `chunks` column chunks into packedB_per_dev[d] (each
 * elv_pack_b_bytes(K, N), on devs[d]); each device splits every chunk as it
 * lands (tensor-core variants, on an internal side stream) and multiplies it
 * on streams[d] while later chunks are still in flight; the tensor-core
 * variants include the range-guard fix-up.  A_shards[d]: rows[d] x K
 * (lda = K); C_shards[d]: rows[d] x N (ldc = N).  workspaces[d] (device
 * devs[d], workspace_bytes each, from elv_gemm_rowshard_workspace_bytes with
 * the largest rows[d]) hold the planes; NULL allowed for variants 4..6.
 * Bitwise equal to elv_gemm on each shard. */
size_t elv_gemm_rowshard_workspace_bytes(int variant, int rows, int N, int K, int chunks);
int elv_gemm_rowshard_pipelined(int variant, int ndev, const int* devs,
                                const float* const* A_shards, const float* B_root,
                                float* const* packedB_per_dev, float* const* C_shards,
                                const int* rows, int N, int K, int chunks,
                                void* const* workspaces, size_t workspace_bytes,
                                void* const* streams);

/* Thread-local message describing the last error on this thread. */
const char* elv_last_error(void);
int elv_abi_version(void);
const char* elv_variant_name(int variant);

#ifdef __cplusplus
}
#endif
#endif /* ELEVATE_B200_H */
