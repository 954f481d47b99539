/*
 * atamul_b200.h — C ABI of the B200-native AtA hot path.
 *
 * The reference (`atamul`, pure Python + NumPy) has no native FFI: its hot
 * path calls NumPy ufuncs / einsum from Python.  Each entry point below
 * replaces one of those arithmetic call sites (cited per function, paths
 * relative to the reference's pkg/src/atamul/).  Plain pointers, extents,
 * leading dimensions (in elements) and a cudaStream_t passed as void*;
 * no torch types.  Every pointer is a DEVICE pointer.  Nothing here
 * allocates: scratch is passed in by the caller (strassen.py:15,
 * "Once the workspace exists, fast_strassen allocates nothing").
 *
 * Return value: 0 on success, a negative ATA_E* code otherwise; the
 * message for the last failure on the calling thread is available through
 * ata_last_error().  The Python layer maps codes onto the reference's
 * exception classes (errors.py:4-37).
 */
#ifndef ATAMUL_B200_H
#define ATAMUL_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (one per reference exception class, errors.py) ---- */
#define ATA_OK 0
#define ATA_E_SHAPE (-1)        /* ShapeMismatchError        errors.py:8  */
#define ATA_E_UNSPLITTABLE (-2) /* UnsplittableError         errors.py:12 */
#define ATA_E_WORKSPACE (-3)    /* WorkspaceUndersizedError  errors.py:16 */
#define ATA_E_UNSUPPORTED (-5)  /* UnsupportedSizeError      errors.py:24 */
#define ATA_E_PROTOCOL (-6)     /* ProtocolError             errors.py:28 */
#define ATA_E_CUDA (-100)       /* CUDA runtime / launch failure          */
#define ATA_E_ARG (-101)        /* invalid argument (null pointer, bad op) */

/* ---- dtype tags ---- */
#define ATA_F64 0
#define ATA_F32 1  /* fp32 storage; products as 3xTF32 (split hi/lo, fp32-level accuracy) */
#define ATA_TF32 2 /* fp32 storage; products as single-pass TF32 (fp32 accumulate)       */

/* ---- plan operations ---- */
#define ATA_OP_GEMM 0   /* D_d[:r,:c] (+)= sign_d*alpha*(sum_i s_i S_i)^T (sum_j t_j T_j) */
#define ATA_OP_SYRK 1   /* lower(D_d) (+)= sign_d*alpha*S^T S, strict upper untouched      */
#define ATA_OP_COMBO 2  /* D_0 = sum_i sign_i * zero-extended S_i  (strassen.py:195-203)    */
#define ATA_OP_UPDATE 3 /* D_d[:r,:c] += sign_d * S_0[:r,:c]       (matrix.py:218-239)      */
#define ATA_OP_FILL 4   /* D_0 = 0                                  (strassen.py:224)        */

/* Operand base selector of a plan reference. */
#define ATA_BASE_A 0  /* the input A                */
#define ATA_BASE_C 1  /* the output C               */
#define ATA_BASE_WS 2 /* the caller's HBM workspace */
#define ATA_BASE_B 3  /* the second operand B (fast_strassen) */

/* GEMM/SYRK use s[0..1], t[0..1] (two zero-extended terms per operand) and up to
 * 8 destinations (post-additions of up to three fused Strassen levels).
 * ATA_OP_COMBO4 reads up to 4 sources s[0..3] (the quadrants of one operand) and
 * writes up to 8 sums d[j] = sum_q c_jq * zero-extended s[q], truncated to d[j]'s
 * extent; c_jq is packed in d[j].region as base-4 digits (digit q: 0 -> 0,
 * 1 -> +1, 2 -> -1); accumulate = 1 restricts every output to its lower
 * triangle (col <= row), which is how split-contraction SYRK partials are summed.  One pass over the quadrants produces all of a Strassen
 * node's operand sums (strassen.py:234-273). */
#define ATA_OP_COMBO4 5
/* ATA_OP_POSTADD7: Strassen post-addition of one node in one pass
 * (strassen.py:238-275 restated as the 4-output form): children P1..P7 are
 * s[0..3], t[0..2] (equal-shape windows, an empty window counts as zero);
 * outputs d[0..3] = (C11, C12, C21, C22) of the node, truncated:
 *   C11 (+)= s0*(P1 + P4 - P5 + P7)   C12 (+)= s1*(P3 + P5)
 *   C21 (+)= s2*(P2 + P4)             C22 (+)= s3*(P1 - P2 + P3 + P6)
 * with accumulate selecting += (into C) or = (into a parent's product buffer). */
#define ATA_OP_POSTADD7 6
/* ATA_OP_ROUND: d[0] = round-to-nearest TF32 of s[0] (fp32 only; equal extents).
 * Emitted once per operand by single-pass-TF32 plans before the tcgen05 products.
 * With accumulate = 2 no pass runs: s[0] is the raw operand the next product group
 * reads directly and d[0] a scratch window (>= 2 * 32 * 192 * cols + 128 scalars)
 * for the CTA-pair kernel's L2 rounding ring, which rounds the operand pieces on
 * chip just before its TMA loads them (auto_plan._ringify decides when the group
 * fits: equal row chunks, two chunks per wave of the persistent grid). */
#define ATA_OP_ROUND 7
/* ata_op.flags.  ATA_OPF_RIDE (COMBO4 only): the op is independent of the product
 * group that follows it in the list -- it neither writes anything those products
 * read or write nor reads anything they write -- so the executor may run it INSIDE
 * that group's launch, on the FP64 leaf kernel's spare warps, instead of as its own
 * HBM pass (the Strassen operand sums of the next leaf group hidden behind this
 * group's tensor-core work).  The executor re-checks the independence and runs the
 * op as an ordinary pass, in list order, whenever it cannot ride. */
#define ATA_OPF_RIDE 1
#define ATA_MAX_TERMS 4
#define ATA_MAX_DESTS 8

/* A rectangular window of one base buffer: element (r, c) lives at
 * base + off + r*ld + c.  Reads outside [rows) x [cols) are zero
 * (the reference's zero-extension, matrix.py:218-239); writes are
 * truncated to [rows) x [cols). */
typedef struct ata_ref {
  int32_t base;  /* ATA_BASE_* */
  int32_t rows;
  int64_t off;   /* element offset from the base pointer */
  int64_t ld;    /* leading dimension (row stride) in elements */
  int32_t cols;
  int32_t region; /* destinations only: 0 = written by this op alone in its launch;
                     r > 0 = a window shared with other ops of the same launch group,
                     accumulated tile by tile in op order (deterministic) */
  double sign;   /* +1 / -1 coefficient */
} ata_ref;

/* One plan operation.  m = contraction length, n x k = output extent. */
typedef struct ata_op {
  int32_t type;          /* ATA_OP_* */
  int32_t m, n, k;
  int32_t ns, nt, nd;    /* term / destination counts */
  int32_t accumulate;    /* GEMM/SYRK: 1 = D += ..., 0 = D = ... */
  int32_t group;         /* consecutive GEMM/SYRK ops with equal group>=0 share one launch */
  int32_t flags;         /* ATA_OPF_* */
  ata_ref s[ATA_MAX_TERMS];
  ata_ref t[ATA_MAX_TERMS];
  ata_ref d[ATA_MAX_DESTS];
} ata_op;

/* ---- library ---- */
const char* ata_last_error(void);
const char* ata_strerror(int code);
int ata_version(void);
int ata_abi_op_size(void); /* sizeof(ata_op), checked by the ctypes layer */

/* ---- leaf kernels ----
 * ata_syrk_lower: lower triangle (incl. diagonal) of C += alpha * A^T A,
 *   A m x n (lda), C n x n (ldc); strict upper never read or written.
 *   Replaces naive_syrk_lower, matrix.py:292-311.
 * ata_gemm_atb: C += alpha * A^T B, A m x n, B m x k, C n x k.
 *   Replaces naive_gemm_atb, matrix.py:269-289 (_accumulate_atb :247-257). */
int ata_syrk_lower(int dtype, const void* A, int64_t lda, int32_t m, int32_t n,
                   void* C, int64_t ldc, double alpha, void* stream);
int ata_gemm_atb(int dtype, const void* A, int64_t lda, const void* B, int64_t ldb,
                 int32_t m, int32_t n, int32_t k, void* C, int64_t ldc, double alpha,
                 void* stream);

/* ---- HBM-bound elementwise kernels ----
 * ata_add_truncated: dst[:r,:c] += scale*src[:r,:c], r/c = min extents;
 *   shapes may differ by at most one row/col.  Replaces add_truncated,
 *   matrix.py:218-239.
 * ata_mirror_lower: C[i,j] = C[j,i] for i<j.  Replaces mirror_lower_to_upper,
 *   matrix.py:373-380.
 * ata_pack_lower / ata_unpack_lower: row-concatenated lower triangle, length
 *   n(n+1)/2.  Replace pack_lower / unpack_lower, matrix.py:353-370; with
 *   accumulate=1 unpack adds (the parent sum of distsim.py:208-216). */
int ata_add_truncated(int dtype, void* dst, int64_t ldd, int32_t dr, int32_t dc,
                      const void* src, int64_t lds, int32_t sr, int32_t sc,
                      double scale, void* stream);
int ata_mirror_lower(int dtype, void* C, int64_t ldc, int32_t n, void* stream);
int ata_pack_lower(int dtype, const void* C, int64_t ldc, int32_t n, void* packed,
                   void* stream);
int ata_unpack_lower(int dtype, const void* packed, int32_t n, void* C, int64_t ldc,
                     int32_t accumulate, void* stream);

/* ---- plan executor ----
 * Runs a flat list of plan ops (built by the host planner from the
 * reference recursion ata.py:97-115 / strassen.py:206-275, or by the
 * auto planner) on one stream.  Bases: A (input), B (second operand, may
 * equal A), C (output), WS (workspace of ws_elems elements).  Every ref is
 * bounds-checked against its base before any launch; ATA_E_WORKSPACE if a
 * workspace ref overruns ws_elems.  `sync` is a caller-owned device int32
 * buffer of sync_ints entries for the persistent kernels' work counter and
 * per-tile turn counters (ata_sync_ints_needed tells how many). */
int ata_run_plan(int dtype, const ata_op* ops, int32_t n_ops, const void* A, int64_t a_elems,
                 const void* B, int64_t b_elems, void* C, int64_t c_elems, void* WS,
                 int64_t ws_elems, void* sync, int64_t sync_ints, double alpha, void* stream);

/* int32 entries of `sync` that ata_run_plan needs for this op list (host-only query). */
int64_t ata_sync_ints_needed(int dtype, const ata_op* ops, int32_t n_ops);

/* Kernel launches the executor has issued since the library was loaded
 * (benchmark accounting; a captured graph replays without new calls). */
int64_t ata_launch_count(void);
/* Product launches that carried riding operand sums (ATA_OPF_RIDE) so far. */
int64_t ata_ride_count(void);

#ifdef __cplusplus
}
#endif
#endif /* ATAMUL_B200_H */
