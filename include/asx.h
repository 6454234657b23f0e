/*
 * asx.h — C ABI of the B200 α-DFT / α-FFT library (libasx.so).
 *
 * The transform (BASELINE.json north_star):
 *
 *     X[b, m] = sum_{n<N} x[b, n] * exp(-2πi * (a/d) * m * n / N),   m < M
 *
 * with α = a/d an exact reduced rational ("α_b" in SURVEY.md §0).  The
 * reference package names the same family by its density factor
 * DenseFactor(p, q) = 1/α (/root/reference/pkg/src/alpha_spectra/core.py:38-82);
 * its full spectrum has M_ref = p*N/q bins, and M is explicit here so that α
 * values the reference rejects (core.py:95-105) are still computable.
 *
 * Every function returns an int status (asx_status) and never throws across
 * the ABI.  Device pointers are caller-owned; execution is asynchronous on
 * the caller's CUDA stream.  A plan is immutable after create; execute is
 * reentrant for distinct outputs / streams.  There is NO CPU fallback: if no
 * CUDA device is usable every compute entry point returns ASX_ERR_CUDA.
 *
 * Reference interfaces each entry point replaces (file:line in
 * /root/reference/pkg/src/alpha_spectra/):
 *   asx_plan_create      fastpath.py:85-110  plan()  (+ oracle.py:50-67 naive_forward's
 *                        validate_pair / table setup, core.py:95-105)
 *   asx_execute          fastpath.py:162-181 transform_samples(), :184-194 alpha_fft(),
 *                        oracle.py:37-67 _reduced_product()/naive_forward()  (batched)
 *   asx_execute_host     same, with host buffers (H2D / D2H pipelined inside)
 *   asx_plan_query       fastpath.py:63-82 Plan fields, :113-127 predicted_mults/adds
 *   asx_plan_destroy     (Plan is garbage-collected in the reference)
 *   asx_dft_matrix       oracle.py:26-34 dft_matrix()
 *   asx_combine          fastpath.py:130-151 combine()
 *   asx_block_sum        fastpath.py:154-159 leaf_block_sum()
 *   asx_strerror / asx_last_error   core.py:17-31 exception messages
 */
#ifndef ASX_H_
#define ASX_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASX_ABI_VERSION 2  /* 2: asx_plan_info.batch_group */

/* Status codes mirror the reference's exception types / CLI exit codes
 * (cli.py:24-29: 3 = incompatible alpha, 4 = unsupported size). */
typedef enum asx_status {
  ASX_OK = 0,
  ASX_ERR_INVALID = 2,      /* ValueError: bad argument (lengths, strides, dtype) */
  ASX_ERR_INCOMPATIBLE = 3, /* IncompatibleAlphaError (core.py:17-27)             */
  ASX_ERR_UNSUPPORTED = 4,  /* UnsupportedSizeError   (core.py:30-31)             */
  ASX_ERR_CUDA = 10,        /* CUDA runtime failure / no device                    */
  ASX_ERR_OOM = 11          /* device allocation failed                             */
} asx_status;

typedef enum asx_dtype {
  ASX_C64 = 0,  /* complex64 in/out (float2), FP32 arithmetic   */
  ASX_C128 = 1  /* complex128 in/out (double2), FP64 arithmetic */
} asx_dtype;

typedef enum asx_method {
  ASX_AUTO = 0,   /* cheapest applicable method by the plan's cost model            */
  ASX_DIRECT = 1, /* direct α-DFT: dense W[M,N] contraction (oracle.py:37-67)       */
  ASX_FFT = 2,    /* α-FFT even/odd recursion (fastpath.py:130-181)                 */
  ASX_CHIRP = 3   /* chirp-z (Bluestein) factorisation of the same α-DFT            */
} asx_method;

typedef enum asx_leaf {
  ASX_LEAF_NONE = 0,
  ASX_LEAF_SINGLE_SAMPLE = 1, /* fastpath.py:41 (alpha_ref >= 1) */
  ASX_LEAF_BLOCK_SUM = 2      /* fastpath.py:42 (alpha_ref <  1) */
} asx_leaf;

typedef struct asx_plan_info {
  int64_t n;               /* signal length N                                  */
  int64_t m;               /* output bins M                                    */
  int64_t a_num, a_den;    /* reduced α = a/d                                  */
  int64_t m_ref;           /* reference full-spectrum size d*N/a (0 if not integral) */
  int32_t depth;           /* reference recursion depth log2(min(N, m_ref)) (-1 if n/a) */
  int32_t leaf;            /* asx_leaf                                         */
  int32_t method;          /* resolved asx_method                              */
  int32_t dtype;           /* asx_dtype                                        */
  int32_t real_input;      /* 1 if inputs are real (float / double)            */
  int32_t fft_size;        /* inner power-of-two FFT size P (0 for direct)     */
  int64_t predicted_mults; /* fastpath.py:113-121 closed form (-1 if n/a)      */
  int64_t predicted_adds;  /* fastpath.py:124-127 closed form (-1 if n/a)      */
  int64_t workspace_bytes; /* device bytes held by the plan                    */
  int32_t kernels_per_execute; /* launches issued by one asx_execute (four-step
                                  plans: per group of batch_group signals)    */
  int32_t device;
  int64_t batch_group;     /* four-step plans: signals per launch set (the
                              workspace holds this many); 0 = whole batch     */
} asx_plan_info;

typedef struct asx_plan_s* asx_plan_t;

int asx_version(void);

/* Create a plan for length-n signals, α = a_num/a_den (reduced internally),
 * m output bins (m <= 0 selects the reference default m_ref = d*n/a, which
 * must then be an integer or ASX_ERR_INCOMPATIBLE is returned).
 * method ASX_FFT reproduces the reference plan() size rules generalised to
 * integer density (ASX_ERR_UNSUPPORTED otherwise); ASX_DIRECT / ASX_CHIRP
 * accept every rational α.  Tables are built on `device` before return. */
int asx_plan_create(asx_plan_t* plan, int64_t n, int64_t a_num, int64_t a_den,
                    int64_t m, int dtype, int real_input, int method, int device);

/* Batched transform on device memory.  x: batch rows of n samples
 * (complex or real per the plan), row stride x_stride elements; X: batch
 * rows of m complex bins, row stride X_stride elements.  stream is a
 * cudaStream_t (NULL = legacy default stream).  Asynchronous. */
int asx_execute(asx_plan_t plan, const void* x, int64_t x_stride, void* X,
                int64_t X_stride, int64_t batch, void* stream);

/* Same transform on HOST buffers (pinned for overlap): the batch is cut into
 * chunks that are copied host->device, transformed and copied back on a
 * small ring of streams so the copies overlap the kernels.  chunk = rows
 * per chunk; chunk <= 0 picks ~128 MiB chunks that ramp up from 1/8 at the
 * start and down at the end (short pipeline fill and drain).  Synchronous:
 * returns after the last result byte is in X. */
int asx_execute_host(asx_plan_t plan, const void* x, int64_t x_stride, void* X,
                     int64_t X_stride, int64_t batch, int64_t chunk);

int asx_plan_query(asx_plan_t plan, asx_plan_info* info);
int asx_plan_destroy(asx_plan_t plan);

/* W[m_rows, n] with W[r, c] = exp(-2πi * ((a*r*c) mod (d*n)) / (d*n)),
 * row-major into device memory (oracle.py:26-34 with exact reduction). */
int asx_dft_matrix(int64_t n, int64_t a_num, int64_t a_den, int64_t m_rows, int dtype,
                   void* W, void* stream);

/* out[r, :] = [y[r,:] + tw*z[r,:],  y[r,:] - tw*z[r,:]] for r < rows
 * (fastpath.py:130-151); y, z: rows x half, tw: half, out: rows x 2*half. */
int asx_combine(const void* y, const void* z, const void* tw, void* out, int64_t rows,
                int64_t half, int dtype, void* stream);

/* out[r] = sum_j x[r, j] for j < len (fastpath.py:154-159). */
int asx_block_sum(const void* x, void* out, int64_t rows, int64_t len, int dtype,
                  void* stream);

/* Launch shape of the last FFT-family kernel this thread launched: grid,
 * block, dynamic shared memory; *staged bit 0 = rows TMA-staged, bits 1.. =
 * kernel variant (0 plain, 1 chirp tables in tensor memory, 2 the P = 16384
 * complex64 group-local chirp kernel k_chirp_local, 3 the α-FFT with two
 * teams per CTA splitting one signal's residues, 4 the complex128 N = 4096
 * α = 1/2 group-local α-FFT k_afft_local, 6 the P = 8192 complex128
 * group-local chirp kernel k_chirp_local128, 8 the tensor-core direct form
 * k_direct_tc, 14 the P = 16384 complex64 chirp kernel at 32 values per
 * thread k_chirp_r32 -- the config-4 default; ASX_NO_R32=1 at plan creation
 * falls back to k_chirp_local). */
int asx_last_launch(int* grid, int* block, int* smem_bytes, int* staged);

const char* asx_strerror(int status);
/* Message of the last failing call on this thread ("" if none). */
const char* asx_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* ASX_H_ */
