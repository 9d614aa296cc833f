/*
 * sketchmm_b200 — C ABI of the B200-native sketched-product hot path.
 *
 * Plain pointers and sizes only (no torch / CUDA-runtime types in the
 * signatures; `stream` is a cudaStream_t passed as void*).  Device pointers
 * are marked [dev], host pointers [host].  Every entry point returns an int
 * status: SMM_OK (0), SMM_ERR_INVALID (parameter/shape violation — the
 * Python facade maps it to InvalidParameterError, mirroring the reference's
 * validation which always happens before any kernel work), SMM_ERR_CUDA
 * (launch/runtime failure -> RuntimeError) or SMM_ERR_WORKSPACE (caller
 * workspace too small).  smm_last_error() returns a thread-local message.
 * Calls never abort; they are re-entrant per stream (no hidden global state
 * besides per-device attribute caches).  Caller-allocated buffers only.
 *
 * Each entry point replaces a reference interface (paths relative to
 * /root/reference/pkg/src/sketchmm):
 *   smm_hash_tables          hashing.py:134-144 (bucket_table / sign_table via
 *                            bucket_many / sign_many, hashing.py:64-75)
 *   smm_compress_workspace   sketch.py:402-417 (estimate_workspace_bytes; device part)
 *   smm_compress_accumulate  sketch.py:238-260 `_run_kernel` -> the compress kernels
 *                            sketch.py:152-177 / 192-218 (steps 1-3, accumulated
 *                            over an inner-index range [k0, k1) — the k-shard unit)
 *   smm_finalize             sketch.py:178-188 / 219-234 (single inverse transform,
 *                            1/b scale) -> ProductSketch.polys
 *   smm_extract              sketch.py:375-399 `decompress_all` (+ the heavy-hitter
 *                            threshold of experiments.py:136-168 / BASELINE cfg5)
 *   smm_transpose            sketch.py:305-307 (`at = ascontiguousarray(A.T)`)
 *   smm_fwht_batched         transforms.py:37-49 / 100-127 (fwht_inplace, xor_convolve)
 *   smm_fft_batched          transforms.py:52-74 / 130-175 (fft_forward, fft_inverse,
 *                            cyclic_convolve)
 *   smm_query                sketch.py:343-372 (sketch_estimates / decompress_entry,
 *                            batched over (i, j) pairs on the device-resident sketch)
 *   smm_copy2d               np.ascontiguousarray(a, dtype=float64) (sketch.py:282-286):
 *                            the host->device move of the operands, done per k-slab so
 *                            uploads overlap the compress kernel
 */
#ifndef SKETCHMM_B200_H
#define SKETCHMM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SMM_OK 0
#define SMM_ERR_INVALID 1
#define SMM_ERR_CUDA 2
#define SMM_ERR_WORKSPACE 3

/* transform codes match the reference container codes (sketch.py:43) */
#define SMM_VARIANT_FFT 0
#define SMM_VARIANT_FWHT 1

/* Repetitions per kernel launch (the hash functions travel in the kernel
 * parameter block).  Deeper sketches (any odd d up to SMM_MAX_DEPTH_TOTAL, the
 * reference accepts any odd d, sketch.py:75-76) are compressed in groups of
 * SMM_MAX_DEPTH repetitions and extracted by a kernel that reads the hash
 * functions from device memory. */
#define SMM_MAX_DEPTH 63
#define SMM_MAX_DEPTH_TOTAL 511

/* OR into `variant` of the compress entry points: acc is ADDED to instead of
 * overwritten.  With the two-pass FWHT kernel and k-ranges split on multiples of
 * 32, consecutive calls reproduce one call's summation order bit for bit
 * (host-streamed operands: each slab is uploaded while the previous computes). */
#define SMM_FLAG_ACCUMULATE 0x100

#define SMM_LAYOUT_KMAJOR 0
#define SMM_LAYOUT_KMINOR 1

int smm_abi_version(void);
const char *smm_last_error(void);

/* Bucket / sign tables for keys 0..n-1 of hash group `group` (0 = h1, 1 = h2,
 * 2 = s1, 3 = s2).  words_host [host]: the 8*d packed hash words in draw order
 * (hashing.py:146-152).  For groups 0/1 buckets_out [dev] (d x n uint32) is
 * written; for groups 2/3 signs_out [dev] (d x n int8, values +-1). */
int smm_hash_tables(const uint64_t *words_host, int d, int log2b, int group, int64_t n,
                    uint32_t *buckets_out, int8_t *signs_out, void *stream);

/* Which compress kernel family serves these shapes (SMM_KERNEL_*): repetitions
 * computed by the same family are bit-identical however they are stacked, which is
 * how compress_seeds groups seeds (sketch.py:289-302 per seed, experiments.py:216-312). */
#define SMM_KERNEL_FOLD 0   /* v1 fold kernels (b < 2^8, b > 2^20)           */
#define SMM_KERNEL_FWHT2P 1 /* two-pass FWHT, 2^8 <= b <= 2^20               */
#define SMM_KERNEL_FFT2P 2  /* two-pass FFT                                   */
#define SMM_KERNEL_FWHT1P 3 /* one-pass FWHT, b = 2^12, n1 + n2 <= 16384 (launches of <= 7 repetitions) */
#define SMM_KERNEL_FFT1P 4  /* one-pass FFT, b = 2^12, n1 + n2 <= 16384 (launches of <= 7 repetitions) */
int smm_compress_kernel(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                        int *kernel);

/* Device workspace (bytes) needed by smm_compress_accumulate for these shapes. */
int smm_compress_workspace(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0,
                           int64_t k1, int64_t *bytes);

/* Steps 1-3 over inner indices [k0, k1):
 *   at [dev]: row k = column k of A (k-major, leading dimension ld_at >= n1);
 *   bm [dev]: row k = row k of B (leading dimension ld_bm >= n2).
 * acc [dev] is OVERWRITTEN with the pre-inverse accumulator of this k-range:
 *   FWHT: d x b float64;  FFT: d x (b/2+1) complex128 (interleaved re, im).
 * Accumulators of disjoint k-ranges add (the multi-GPU allreduce unit). */
int smm_compress_accumulate(int variant, const double *at, int64_t ld_at, const double *bm,
                            int64_t ld_bm, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                            const uint64_t *words_host, int d, int log2b, void *acc,
                            void *workspace, int64_t workspace_bytes, void *stream);

/* Same as smm_compress_accumulate with explicit operand layouts:
 *   SMM_LAYOUT_KMAJOR: row k holds inner index k (the reference's `at` = A^T and B);
 *   SMM_LAYOUT_KMINOR: row i holds element i, inner index k contiguous (A row-major,
 *                      B^T row-major) — the layout the two-pass FWHT kernel reads.
 * lda/ldb are leading dimensions in that layout.  The library transposes the
 * [k0, k1) slab of an operand whose layout differs from what the selected kernel
 * reads into the workspace (size from smm_compress_workspace_ex). */
int smm_compress_workspace_ex(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0,
                              int64_t k1, int a_layout, int b_layout, int64_t *bytes);
int smm_compress_accumulate_ex(int variant, const double *a, int64_t lda, int a_layout,
                               const double *b, int64_t ldb, int b_layout, int64_t n1, int64_t n2,
                               int64_t k0, int64_t k1, const uint64_t *words_host, int d, int log2b,
                               void *acc, void *workspace, int64_t workspace_bytes, void *stream);

/* Strided 2-D copy between any host/device pointers (cudaMemcpyDefault) on
 * `stream`: `rows` rows of width_bytes, pitches in bytes.  Used to stream a
 * k-slab of a host-resident row-major A (a column block) to the device. */
int smm_copy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width_bytes, int64_t rows,
               void *stream);

/* Step 4: polys [dev] (d x b float64) = inverse transform of acc, times 1/b. */
int smm_finalize(int variant, const void *acc, double *polys, int d, int log2b, void *stream);

/* Step 5 on output rows [r0, r1) (all n2 columns):
 *   est [dev, nullable]: (r1-r0) x n2 float64, leading dimension ld_est;
 *   heavy hitters: |est| > thr (strict != 0) or >= thr; *hh_count [dev] receives
 *   the count; if hh_pairs [dev] is non-NULL, the (i, j) pairs (global row
 *   index, column) are written in row-major order, at most hh_cap pairs.
 *   workspace [dev] of smm_extract_workspace() bytes. */
int smm_extract_workspace(int d, int64_t n1, int64_t n2, int64_t r0, int64_t r1, int64_t *bytes);
int smm_extract(int variant, const double *polys, const uint64_t *words_host, int d, int log2b,
                int64_t n1, int64_t n2, int64_t r0, int64_t r1, double *est, int64_t ld_est,
                double thr, int strict, int64_t *hh_pairs, int64_t hh_cap, int64_t *hh_count,
                void *workspace, int64_t workspace_bytes, void *stream);

/* Heavy-hitter pair list of the LAST smm_extract call made with this workspace:
 * the (i, j) pairs whose bit is set, in row-major order, at most hh_cap pairs
 * (hh_pairs [dev], int64 pairs).  Needs no recomputation of the medians, so a
 * caller can size hh_pairs from *hh_count of the extract call.  Replaces the
 * thresholding loop of experiments.py:136-168. */
int smm_hh_pairs(const void *workspace, int64_t n2, int64_t r0, int64_t r1, int64_t *hh_pairs, int64_t hh_cap,
                 void *stream);

/* Per-entry estimates for `count` (i, j) pairs (ij [dev]: int64 pairs; the caller
 * range-checks them against n1 x n2, as sketch.py:352-355 does): est [dev] the
 * median, reps [dev, nullable] the d signed per-repetition values (count x d). */
int smm_query(int variant, const double *polys, const uint64_t *words_host, int d, int log2b, int64_t n1,
              int64_t n2, const int64_t *ij, int64_t count, double *est, double *reps, void *stream);

/* Number of kernels this library has launched in the process (monotone counter;
 * bench/evidence only). */
int64_t smm_kernel_launches(void);

/* Live per-launch kernel timing (bench evidence): while enabled, every launch of the
 * compress kernel (channel 0: fwht2p / fft2p) and of the extraction kernel
 * (channel 1) is bracketed by CUDA events on its stream.  _read waits for the
 * recorded launches of a channel, returns their summed device time and count, and
 * clears them.  Not a reference interface (the reference has no GPU). */
int smm_kernel_timing(int enable);
int smm_kernel_timing_read(int channel, double *total_ms, int64_t *launches);

/* out[c, r] = in[r, c] for a rows x cols float64 matrix [dev]. */
int smm_transpose(const double *in, int64_t rows, int64_t cols, int64_t ld_in, double *out,
                  int64_t ld_out, void *stream);

/* In-place unnormalized FWHT of `batch` contiguous vectors of length 2^log2n [dev],
 * followed by a multiply by `scale`. */
int smm_fwht_batched(double *x, int64_t batch, int log2n, double scale, void *stream);

/* In-place complex FFT (interleaved complex128) of `batch` contiguous vectors of
 * length 2^log2n [dev]; inverse != 0 uses conjugate twiddles; then * scale. */
int smm_fft_batched(double *z, int64_t batch, int log2n, int inverse, double scale, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SKETCHMM_B200_H */
