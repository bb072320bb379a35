/*
 * slicegemm_b200.h -- C ABI of the B200 bitsliced M4RM library (libslicegemm_b200.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference package
 * `slicegemm` (Python) routes its multiply through a backend module chosen by
 * slicegemm/_core.py:15-61 (`_BACKENDS`, `active()`, `set_active()`); each backend exposes
 * the plane kernels and `m4rm_block_<field>` drivers of slicegemm/_core_py.py:24-286 with
 * in-place semantics on per-plane (rows, words) uint64 arrays.  The compiled backend slot
 * (`_core_cy`, slicegemm/_core.py:17-22, built by setup.py:10-19) is what this library fills.
 * Entry points and the reference interface each one replaces:
 *
 *   sg_pack / sg_unpack      BitslicedMatrix.from_dense / to_dense (__init__.py:15)
 *   sg_reduce_canonical      BitslicedMatrix.reduce_canonical;
 *                            f5_reduce / f7_reduce (_core_py.py:143-148, 171-175)
 *   sg_plane_op              the backend's plane kernels f2_add ... f7_reduce (_core_py.py:24-175)
 *   sg_build_table           m4rm.build_table (__init__.py:16)
 *   sg_m4rm_block            m4rm_block_f2/f3/f5/f7 (_core_py.py:205-222, 274-281)
 *   sg_m4rm                  m4rm_multiply(A, B, params) (__init__.py:16), and
 *                            for SG_GF4 ext_multiply over F4 (__init__.py:17)
 *   sg_m4rm_host             the same with host buffers (the call a CPU caller makes)
 *   sg_m4rm_multi            the same over several GPUs of one process (rows sharded, B
 *                            replicated; the reference's row0/row1 partition)
 *   sg_classical             classical_multiply (__init__.py:16)
 *   sg_classical_block       classical_f2/f3/f5/f7/z4/z8 (_core_py.py:292-366)
 *   sg_stream_check          the ValueError of from_dense / to_dense
 *
 * Data layout (identical bits to the reference's BitslicedMatrix planes):
 *   a matrix of `rows` x `n` over a field with R planes is R contiguous planes, each `rows` x
 *   W64 uint64 words, W64 = ceil(n / 64); column c lives in word c >> 6, bit c & 63 (little
 *   endian).  Padding lanes (columns >= n) must be zero.  R = 1 (F2), 2 (F3, GF4, Z4),
 *   3 (F5, F7, GF8, Z8).
 *   F3: plane 0 = unit, plane 1 = sign (0 = 00, 1 = 01, -1 = 11, fields.py:88-101).
 *   F5 / F7: 3-bit binary value, residue = value mod p (redundant, fields.py:103-129).
 *   GF4 = F2[x]/(x^2+x+1): plane 0 = coefficient of 1, plane 1 = coefficient of x (fields.py:215).
 * Pointers passed to the device entry points are CUDA device pointers; `stream` is a
 * cudaStream_t (NULL = the legacy default stream).  Calls are stream-ordered and return
 * before the work completes.  The library never frees caller buffers.
 *
 * Errors: every entry point returns SG_OK (0) or a positive SG_E* code and records a message
 * retrievable with sg_last_error() (thread-local).  No C++ exception crosses the ABI.  The
 * Python layer maps SG_EINVAL / SG_ERANGE / SG_EPATTERN to ValueError (the reference raises
 * ValueError on field / shape mismatch and out-of-range entries, oracle.py:69-79)
 * and everything else to RuntimeError.
 */
#ifndef SLICEGEMM_B200_H
#define SLICEGEMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 1

/* fields (GF4/GF8 = F2[x]/(x^2+x+1), F2[x]/(x^3+x+1) in power-basis planes, fields.py:215-216;
 * Z4/Z8 = the reference's binary rings, fields.py:131-158) */
enum { SG_F2 = 0, SG_F3 = 1, SG_F5 = 2, SG_F7 = 3, SG_GF4 = 4, SG_GF8 = 5, SG_Z4 = 6, SG_Z8 = 7 };

/* status codes */
enum {
  SG_OK = 0,
  SG_EINVAL = 1,       /* bad argument: field, shape, k, null pointer */
  SG_ECUDA = 2,        /* CUDA runtime error (message has the CUDA error string) */
  SG_EUNSUPPORTED = 3, /* valid request this build cannot serve */
  SG_ERANGE = 4,       /* sg_pack: an entry is not a residue of the field */
  SG_EPATTERN = 5,     /* sg_unpack: an F3 lane holds the illegal pattern 10 */
  SG_ENOMEM = 6
};

/* plane-op codes for sg_plane_op (in-place on dst; the reference backend's plane kernels) */
enum {
  SG_OP_F2_ADD = 0,       /* _core_py.py:24  f2_add(d0, s0)                 */
  SG_OP_F3_ADD = 1,       /* _core_py.py:28  f3_add(d0, d1, s0, s1)         */
  SG_OP_F3_SUB = 2,       /* _core_py.py:35  f3_sub                          */
  SG_OP_F3_NEG = 3,       /* _core_py.py:42  f3_neg(p0, p1)                  */
  SG_OP_F5_ADD = 4,       /* _core_py.py:116 f5_add(d0..d2, s0..s2)          */
  SG_OP_F5_SUB = 5,       /* _core_py.py:128 f5_sub                          */
  SG_OP_F5_NEG = 6,       /* _core_py.py:120 f5_neg(p0..p2)                  */
  SG_OP_F5_DOUBLE = 7,    /* _core_py.py:135 f5_double                       */
  SG_OP_F5_REDUCE = 8,    /* _core_py.py:143 f5_reduce                       */
  SG_OP_F7_ADD = 9,       /* _core_py.py:151 f7_add                          */
  SG_OP_F7_SUB = 10,      /* _core_py.py:162 f7_sub(..., tail)               */
  SG_OP_F7_NEG = 11,      /* _core_py.py:155 f7_neg(p0..p2, tail)            */
  SG_OP_F7_DOUBLE = 12,   /* _core_py.py:258 plane rotation                  */
  SG_OP_F7_REDUCE = 13,   /* _core_py.py:171 f7_reduce                       */
  SG_OP_GF4_ADD = 14,     /* coefficientwise F2 add        */
  SG_OP_GF4_MULX = 15,    /* multiply by x mod x^2+x+1                       */
  SG_OP_F5_FOLD5 = 16,    /* kernels.py:205 f5_fold5: dst = s0..s2, src plane 0 = s3 */
  SG_OP_SCALAR_MUL_F3 = 17, /* BitslicedMatrix.scalar_mul, scalar = residue */
  SG_OP_SCALAR_MUL_F5 = 18,
  SG_OP_SCALAR_MUL_F7 = 19,
  SG_OP_SCALAR_MUL_GF4 = 20,
  SG_OP_Z4_ADD = 21,      /* _core_py.py:46 z4_add(d0, d1, s0, s1)          */
  SG_OP_Z4_SUB = 22,      /* _core_py.py:53 z4_sub                           */
  SG_OP_Z4_NEG = 23,      /* _core_py.py:61 z4_neg                           */
  SG_OP_Z8_ADD = 24,      /* _core_py.py:100 z8_add                          */
  SG_OP_Z8_SUB = 25,      /* _core_py.py:110 z8_sub                          */
  SG_OP_Z8_NEG = 26,      /* _core_py.py:104 z8_neg                          */
  SG_OP_GF8_ADD = 27,     /* coefficientwise F2 add                          */
  SG_OP_GF8_MULX = 28,    /* multiply by x mod x^3+x+1                       */
  SG_OP_SCALAR_MUL_Z4 = 29,
  SG_OP_SCALAR_MUL_Z8 = 30,
  SG_OP_SCALAR_MUL_GF8 = 31
};

int sg_abi_version(void);
const char* sg_last_error(void);
int sg_field_planes(int field);

/* dense uint8 residues (row stride ld bytes, device) <-> planes (device).  Stream-ordered like
 * every device entry point: the input check runs inside the kernel and never synchronizes.  An
 * entry that is not a residue (sg_pack) or an F3 lane holding the illegal pattern 10 (sg_unpack)
 * is recorded in a per-(device, stream) status word and reported by the next sg_stream_check on
 * that stream (SG_ERANGE / SG_EPATTERN); the output of such a call is unspecified. */
int sg_pack(int field, const uint8_t* dense, int64_t m, int64_t n, int64_t ld, uint64_t* planes,
            void* stream);
int sg_unpack(int field, const uint64_t* planes, int64_t m, int64_t n, uint8_t* dense, int64_t ld,
              void* stream);
/* Synchronize `stream` (on the current device) and report, then clear, the input-check status of
 * the sg_pack / sg_unpack calls queued on it since the last check: SG_OK, SG_ERANGE or
 * SG_EPATTERN (the reference raises ValueError for both). */
int sg_stream_check(void* stream);
/* every lane to its canonical pattern (no-op for F2, F3, GF4) */
int sg_reduce_canonical(int field, uint64_t* planes, int64_t rows, int64_t n, void* stream);
/* dst (op)= src, lanewise, in place on dst: `dst` and `src` are arrays of R device pointers,
 * one per plane (the reference passes one array per plane, _core_py.py:8-9), each plane
 * `rows` x `words` 64-bit words.  `tail` masks the last word of every row (padding lanes) for
 * SG_OP_F7_NEG / SG_OP_F7_SUB (_core_py.py:155-168); `scalar` is the residue for
 * SG_OP_SCALAR_MUL_*.  src may be NULL for unary ops. */
int sg_plane_op(int op, uint64_t* const* dst, const uint64_t* const* src, int64_t rows,
                int64_t words, uint64_t tail, int scalar, void* stream);

/* C (m x n) = A (m x l) * B (l x n), all device planes; C is written in canonical form and
 * is bit-identical for every k in 1..16 (k > 8 runs with 8-row blocks: same output).
 * workspace may be NULL (library-managed cache, one per (device, stream)). */
int64_t sg_m4rm_workspace_bytes(int field, int64_t m, int64_t l, int64_t n, int k);
int sg_m4rm(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l,
            int64_t n, int k, void* workspace, int64_t workspace_bytes, void* stream);
/* Same with host buffers: copies in, multiplies on `device`, copies C back; synchronous.  The
 * copies overlap the products: A and C move in row pieces, and where the plan allows it
 * (stream-K, warp-specialized TMA schedule) the first piece's product starts before B is up and
 * consumes B's k-chunks as they land (sg_host_streamed_count counts those calls). */
int sg_m4rm_host(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m,
                 int64_t l, int64_t n, int k, int device);

/* Multi-GPU from one process: rows of A and C are split into ngpus contiguous
 * balanced slabs, B goes up once to devices[0] and is replicated to the other devices by peer
 * copies (NVLink / NVSwitch), each device multiplies its slab, and the C slabs come back into
 * the host buffer.  Host buffers as in sg_m4rm_host; synchronous.  The inner dimension is
 * never split, so C is bit-identical for any device list (devices may repeat). */
int sg_m4rm_multi(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m,
                  int64_t l, int64_t n, int k, int ngpus, const int* devices);

/* classical_multiply: the table-free row-accumulate product, a cross-check
 * (O(m l n / 32) word operations); canonical output, same layout as sg_m4rm. */
int sg_classical(int field, const uint64_t* A, const uint64_t* B, uint64_t* C, int64_t m, int64_t l,
                 int64_t n, void* stream);

/* classical_<field>(C planes, A planes, B planes) of the reference backend (_core_py.py:292-366):
 * C (m rows of c_words words) += A (m x l, a_words words per row) * B (l rows of c_words words),
 * in place with the backend's raw semantics (B's rows in order, zero coefficients skipped, no
 * canonical reduction), so the bits equal the pure backend's.  Plane pointer arrays as in
 * sg_plane_op; O(m l n / 32) word operations (a cross-check, not a fast path). */
int sg_classical_block(int field, uint64_t* const* C, int64_t c_words, const uint64_t* const* A,
                       int64_t a_words, const uint64_t* const* B, int64_t m, int64_t l, void* stream);

/* Block-granularity plugin mirror.  Plane pointer arrays as in sg_plane_op.  T has the
 * reference table layout: per plane 2^kp rows x words 64-bit words, entry g = the sum of B rows
 * row_base + t over the set bits t of g (B: b_rows rows of `words` words per plane; rows past
 * b_rows count as zero, the narrow final block of SPEC.md:357). */
int sg_build_table(int field, const uint64_t* const* B, int64_t b_rows, int64_t row_base, int kp,
                   int64_t words, uint64_t* const* T, void* stream);
/* C rows row0..row1 += block (col0, kp) of A times the table T (in place, raw patterns):
 * m4rm_block_<field>(C planes, A planes, col0, kp, T planes, row0, row1). */
int sg_m4rm_block(int field, uint64_t* const* C, int64_t c_words, const uint64_t* const* A,
                  int64_t a_words, int64_t col0, int kp, const uint64_t* const* T, int64_t row0,
                  int64_t row1, void* stream);

/* Introspection and measurement. */
int sg_plan(int field, int64_t m, int64_t l, int64_t n, int k, int* rows_per_cta, int* splits,
            int* ctas, int* kernel_index, int* pipelined, int* threads);
/* force rows per thread / k-splits / threads per CTA (0 = automatic) and the schedule
 * (-1 = automatic; 0 serial, 1 pipelined, 2 warp-specialized).  splits = -1 forces the
 * stream-K launch (one wave of CTAs over tile x k-block units + a compact reduction; k = 8
 * only); sg_plan reports splits = -1 for a stream-K plan. */
int sg_set_plan_override(int rows_per_thread, int splits, int pipe, int threads);
/* Plan for (SM count - sms) SMs, leaving `sms` SMs free for a kernel that must run concurrently
 * (the NCCL broadcast of B's next row block in dist.sharded_multiply); 0 = all SMs. */
int sg_set_sm_reserve(int sms);
int sg_set_timing(int enable);                              /* event-time each internal launch */
int sg_last_timing(double* transpose_ms, double* m4rm_ms, double* reduce_ms);
int64_t sg_launch_count(void);                              /* kernels launched by this library */
int64_t sg_host_streamed_count(void);         /* sg_m4rm_host calls whose product streamed B */
/* compiled M4RM instantiation `index` (0 .. count-1; returns the count, or -1 for a bad index):
 * field, k, rows per thread, lookup threads, schedule, CTAs per SM on `device`, registers per
 * thread, dynamic shared memory bytes (any pointer may be NULL) */
int sg_kernel_info(int index, int device, int* field, int* k, int* rows_per_thread, int* threads,
                   int* schedule, int* occupancy, int* regs, int* smem_bytes);
int sg_probe_peaks(int device, double* lop3_per_clk_sm, double* lds_bytes_per_clk_sm,
                   double* sm_mhz);

#ifdef __cplusplus
}
#endif

#endif /* SLICEGEMM_B200_H */
