// extern "C" entry points declared in include/sketchmm_b200.h.  Validation
// mirrors the reference's parameter checks (sketch.py:68-82, hashing.py:25-32)
// and always happens before any kernel is launched.
#include "plan.cuh"

namespace smm {
const char *last_error();
int hash_tables(const SketchHashes &h, int group, int64_t n, uint32_t *buckets, int8_t *signs, cudaStream_t s);
int64_t fwht_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int G);
int64_t fft_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int Gmax);
bool fwht2p_supported(int log2b, int64_t n1, int64_t n2);
bool fwht1p_supported(int log2b, int d, int64_t n1, int64_t n2, int64_t K);
bool fft1p_supported(int log2b, int d, int64_t n1, int64_t n2, int64_t K);
int64_t fft1p_workspace(int d, int64_t n1, int64_t n2, int64_t K);
int fft1p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb, int64_t n1,
                     int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws, int64_t ws_bytes,
                     cudaStream_t s);
int64_t fwht1p_workspace(int d, int64_t n1, int64_t n2, int64_t K);
int fwht1p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, bool a_kminor, const double *xb,
                      int64_t ldb, bool b_kminor, int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc,
                      bool acc_add, char *ws, int64_t ws_bytes, cudaStream_t s);
int64_t fwht2p_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K);
int fwht2p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb,
                      int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws,
                      int64_t ws_bytes, cudaStream_t s);
int add_inplace(double *dst, const double *src, int64_t n, cudaStream_t s);
bool fft2p_supported(int log2b, int64_t n1, int64_t n2);
int64_t fft2p_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K);
int fft2p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb, int64_t n1,
                     int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws, int64_t ws_bytes,
                     cudaStream_t s);
int fwht_accumulate(const SketchHashes &h, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm,
                    int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc, char *ws, int64_t ws_bytes,
                    cudaStream_t s);
int fft_accumulate(const SketchHashes &h, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm,
                   int64_t n1, int64_t n2, int64_t k0, int64_t k1, cplx *acc, char *ws, int64_t ws_bytes,
                   cudaStream_t s);
int finalize(int variant, const void *acc, double *polys, int d, int log2b, cudaStream_t s);
int64_t extract_workspace(int64_t n2, int64_t r0, int64_t r1);
int extract(int variant, const SketchHashes &h, const double *polys, int64_t n1, int64_t n2, int64_t r0, int64_t r1,
            double *est, int64_t ld_est, double thr, int strict, int64_t *hh_pairs, int64_t hh_cap,
            int64_t *hh_count, char *ws, int64_t ws_bytes, cudaStream_t s);
int hh_pairs(const void *ws, int64_t n2, int64_t r0, int64_t r1, int64_t *pairs, int64_t cap, cudaStream_t s);
int query(int variant, const SketchHashes &h, const double *polys, const int64_t *ij, int64_t count, double *est,
          double *reps, cudaStream_t s);
int64_t launches();
int64_t big_hash_bytes(int d);
int extract_big(int variant, const uint64_t *words, int d, int log2b, const double *polys, int64_t n2, int64_t r0,
                int64_t r1, double *est, int64_t ld_est, double thr, int strict, int64_t *hh_pairs, int64_t hh_cap,
                int64_t *hh_count, char *ws, int64_t ws_bytes, cudaStream_t s);
int query_big(int variant, const uint64_t *words, int d, int log2b, const double *polys, const int64_t *ij,
              int64_t count, double *est, double *reps, cudaStream_t s);
int transpose(const double *in, int64_t rows, int64_t cols, int64_t ld_in, double *out, int64_t ld_out,
              cudaStream_t s);
int fwht_batched(double *x, int64_t batch, int log2n, double scale, cudaStream_t s);
int fft_batched(cplx *z, int64_t batch, int log2n, int inverse, double scale, cudaStream_t s);
}  // namespace smm

using namespace smm;

#define SMM_REQUIRE(cond, ...)   \
  do {                           \
    if (!(cond)) {               \
      set_error(__VA_ARGS__);    \
      return SMM_ERR_INVALID;    \
    }                            \
  } while (0)

// bytes of one pre-inverse accumulator
static int64_t acc_bytes(int variant, int d, int log2b) {
  const int64_t b = (int64_t)1 << log2b;
  return variant == SMM_VARIANT_FWHT ? (int64_t)d * b * 8 : (int64_t)d * (b / 2 + 1) * 16;
}

// Compress / finalize accept any depth (stacked repetitions of several seeds);
// extraction needs an odd d (the median is the middle order statistic).
static int check_sketch(int variant, int d, int log2b, bool need_odd = false) {
  SMM_REQUIRE(variant == SMM_VARIANT_FFT || variant == SMM_VARIANT_FWHT, "unknown transform variant %d", variant);
  SMM_REQUIRE(d >= 1 && d <= SMM_MAX_DEPTH_TOTAL, "d must be in [1, %d], got %d", SMM_MAX_DEPTH_TOTAL, d);
  SMM_REQUIRE(!need_odd || d % 2 == 1, "d must be an odd integer in [1, %d], got %d", SMM_MAX_DEPTH_TOTAL, d);
  SMM_REQUIRE(log2b >= 1 && log2b <= 32, "b must be a power of two in [2, 2**32], got 2**%d", log2b);
  if (variant == SMM_VARIANT_FFT) SMM_REQUIRE(log2b <= 30, "fft variant supports b <= 2**30");
  return SMM_OK;
}

// Hash words of repetitions [t0, t1) in the group-major layout of words_host
// (hashing.py:146-152): the input of one kernel launch of at most SMM_MAX_DEPTH.
static void group_words(const uint64_t *words, int d, int t0, int t1, uint64_t *out) {
  const int dg = t1 - t0;
  for (int g = 0; g < 4; ++g)
    for (int t = 0; t < dg; ++t) {
      out[g * 2 * dg + 2 * t] = words[g * 2 * d + 2 * (t0 + t)];
      out[g * 2 * dg + 2 * t + 1] = words[g * 2 * d + 2 * (t0 + t) + 1];
    }
}

extern "C" {

int smm_abi_version(void) { return 1; }

const char *smm_last_error(void) { return last_error(); }

int smm_hash_tables(const uint64_t *words_host, int d, int log2b, int group, int64_t n, uint32_t *buckets_out,
                    int8_t *signs_out, void *stream) {
  SMM_REQUIRE(words_host != nullptr, "hash words must not be NULL");
  SMM_REQUIRE(d >= 1 && d <= SMM_MAX_DEPTH_TOTAL, "d out of range");
  SMM_REQUIRE(log2b >= 1 && log2b <= 32, "log2b out of range");
  SMM_REQUIRE(group >= 0 && group <= 3, "group must be 0..3");
  SMM_REQUIRE(n >= 0 && n <= ((int64_t)1 << 32), "keys must fit in 32 bits");
  SMM_REQUIRE(group >= 2 || buckets_out != nullptr, "buckets_out is NULL");
  SMM_REQUIRE(group < 2 || signs_out != nullptr, "signs_out is NULL");
  uint64_t gw[8 * SMM_MAX_DEPTH];
  for (int t0 = 0; t0 < d; t0 += SMM_MAX_DEPTH) {  // repetition groups of one launch each
    const int t1 = t0 + SMM_MAX_DEPTH < d ? t0 + SMM_MAX_DEPTH : d;
    group_words(words_host, d, t0, t1, gw);
    SketchHashes h;
    load_hashes(h, gw, t1 - t0, log2b);
    const int rc = hash_tables(h, group, n, buckets_out ? buckets_out + (int64_t)t0 * n : nullptr,
                               signs_out ? signs_out + (int64_t)t0 * n : nullptr, (cudaStream_t)stream);
    if (rc) return rc;
  }
  return SMM_OK;
}

// ---------------------------------------------------------------- compress dispatch
// The two-pass FWHT kernel reads k-minor operands (row = input index, k
// contiguous); the fold kernels (FFT, small/large b) read k-major rows.  An
// operand in the other layout is transposed (only its [k0, k1) slab) into the
// front of the workspace.
// SMM_FLAG_ACCUMULATE: the two-pass kernel continues the k order in acc itself;
// the other kernels reduce into a workspace accumulator that is then added.
struct CompressPlan {
  bool one_pass, fft_one_pass, two_pass, fft_two_pass, acc_add;
  bool ta, tb;  // transpose A / B slab
  int64_t ta_bytes, tb_bytes, tmp_acc_bytes, kernel_bytes;
};

static CompressPlan plan_compress(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t K, int alay,
                                  int blay, bool acc_add) {
  CompressPlan c;
  c.acc_add = acc_add;
  // one-pass on-chip kernels for b = 2^12 with small operands (fwht1p.cu, fft1p.cu); k-major operands
  c.fft_one_pass = variant == SMM_VARIANT_FFT && fft1p_supported(log2b, d, n1, n2, K);
  c.fft_two_pass = !c.fft_one_pass && variant == SMM_VARIANT_FFT && fft2p_supported(log2b, n1, n2);
  c.one_pass = variant == SMM_VARIANT_FWHT && fwht1p_supported(log2b, d, n1, n2, K);
  c.two_pass = !c.one_pass && ((variant == SMM_VARIANT_FWHT && fwht2p_supported(log2b, n1, n2)) || c.fft_two_pass);
  // two-pass kernels read k-minor rows, the others k-major ones; the one-pass kernel could
  // read a k-minor operand in place (8-byte strided copies) but measured slower than
  // transposing it first (cfg5 b = 2^12 d = 3: 2.39 vs 1.58 ms)
  const int want = c.two_pass ? SMM_LAYOUT_KMINOR : SMM_LAYOUT_KMAJOR;
  c.ta = alay != want;
  c.tb = blay != want;
  c.ta_bytes = c.ta ? ((n1 * K * 8 + 255) / 256) * 256 : 0;
  c.tb_bytes = c.tb ? ((n2 * K * 8 + 255) / 256) * 256 : 0;
  if (c.one_pass) c.kernel_bytes = fwht1p_workspace(d, n1, n2, K);
  else if (c.fft_one_pass) c.kernel_bytes = fft1p_workspace(d, n1, n2, K);
  else if (c.fft_two_pass) c.kernel_bytes = fft2p_workspace(d, log2b, n1, n2, K);
  else if (c.two_pass) c.kernel_bytes = fwht2p_workspace(d, log2b, n1, n2, K);
  else if (variant == SMM_VARIANT_FWHT) c.kernel_bytes = fwht_workspace(d, log2b, n1, n2, K, num_sms());
  else c.kernel_bytes = fft_workspace(d, log2b, n1, n2, K, num_sms());
  c.tmp_acc_bytes = (acc_add && !c.two_pass && !c.one_pass && !c.fft_one_pass) ? ((acc_bytes(variant, d, log2b) + 255) / 256) * 256 : 0;
  return c;
}

int smm_compress_workspace_ex(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                              int a_layout, int b_layout, int64_t *bytes) {
  const bool acc_add = (variant & SMM_FLAG_ACCUMULATE) != 0;
  variant &= ~SMM_FLAG_ACCUMULATE;
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(bytes != nullptr, "bytes is NULL");
  SMM_REQUIRE(n1 >= 0 && n2 >= 0 && k0 >= 0 && k1 >= k0, "bad shapes");
  SMM_REQUIRE((a_layout == 0 || a_layout == 1) && (b_layout == 0 || b_layout == 1), "bad layout");
  const int dg = d < SMM_MAX_DEPTH ? d : SMM_MAX_DEPTH;  // one launch's repetitions (workspace reused per group)
  CompressPlan c = plan_compress(variant, dg, log2b, n1, n2, k1 - k0, a_layout, b_layout, acc_add);
  *bytes = c.ta_bytes + c.tb_bytes + c.tmp_acc_bytes + c.kernel_bytes;
  return SMM_OK;
}

int smm_compress_kernel(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                        int *kernel) {
  int rc = check_sketch(variant & ~SMM_FLAG_ACCUMULATE, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(kernel != nullptr, "kernel is NULL");
  SMM_REQUIRE(n1 >= 0 && n2 >= 0 && k0 >= 0 && k1 >= k0, "bad shapes");
  variant &= ~SMM_FLAG_ACCUMULATE;
  const int dg = d < SMM_MAX_DEPTH ? d : SMM_MAX_DEPTH;
  CompressPlan c = plan_compress(variant, dg, log2b, n1, n2, k1 - k0, SMM_LAYOUT_KMAJOR, SMM_LAYOUT_KMAJOR, false);
  *kernel = c.one_pass       ? SMM_KERNEL_FWHT1P
            : c.fft_one_pass ? SMM_KERNEL_FFT1P
            : c.fft_two_pass ? SMM_KERNEL_FFT2P
            : c.two_pass     ? SMM_KERNEL_FWHT2P
                             : SMM_KERNEL_FOLD;
  return SMM_OK;
}

int smm_compress_workspace(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                           int64_t *bytes) {
  return smm_compress_workspace_ex(variant, d, log2b, n1, n2, k0, k1, SMM_LAYOUT_KMAJOR, SMM_LAYOUT_KMAJOR, bytes);
}

int smm_compress_accumulate_ex(int variant, const double *a, int64_t lda, int a_layout, const double *b, int64_t ldb,
                               int b_layout, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                               const uint64_t *words_host, int d, int log2b, void *acc, void *workspace,
                               int64_t workspace_bytes, void *stream) {
  const bool acc_add = (variant & SMM_FLAG_ACCUMULATE) != 0;
  variant &= ~SMM_FLAG_ACCUMULATE;
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(words_host != nullptr && acc != nullptr, "NULL argument");
  SMM_REQUIRE(n1 >= 0 && n2 >= 0 && n1 < ((int64_t)1 << 31) && n2 < ((int64_t)1 << 31), "operand sizes out of range");
  SMM_REQUIRE(k0 >= 0 && k1 >= k0, "inner range [%lld, %lld) invalid", (long long)k0, (long long)k1);
  SMM_REQUIRE((a_layout == 0 || a_layout == 1) && (b_layout == 0 || b_layout == 1), "bad layout");
  SMM_REQUIRE(k1 == k0 || ((a != nullptr || n1 == 0) && (b != nullptr || n2 == 0)), "operand pointer is NULL");
  SMM_REQUIRE(a_layout == SMM_LAYOUT_KMAJOR ? lda >= n1 : lda >= k1, "lda too small for the layout");
  SMM_REQUIRE(b_layout == SMM_LAYOUT_KMAJOR ? ldb >= n2 : ldb >= k1, "ldb too small for the layout");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t K = k1 - k0;
  const int dg = d < SMM_MAX_DEPTH ? d : SMM_MAX_DEPTH;
  CompressPlan c = plan_compress(variant, dg, log2b, n1, n2, K, a_layout, b_layout, acc_add);
  const int64_t need = c.ta_bytes + c.tb_bytes + c.tmp_acc_bytes + c.kernel_bytes;
  if (workspace_bytes < need) {
    set_error("compress workspace too small: %lld < %lld bytes", (long long)workspace_bytes, (long long)need);
    return SMM_ERR_WORKSPACE;
  }
  if (acc_add && K == 0) return SMM_OK;
  char *ws = (char *)workspace;
  // operand views in the layout the chosen kernel reads; offsets so that inner index k0 maps to x[.. + k0]
  const double *xa = a, *xb = b;
  int64_t la = lda, lb = ldb, kk0 = k0, kk1 = k1;
  if (c.ta || c.tb) { kk0 = 0; kk1 = K; }
  if (!(c.ta || c.tb)) {
    // no copies: kernels index with k0 directly
  } else {
    // both operands must share the same k origin: shift the untouched one to its slab
    if (!c.ta) xa = c.two_pass ? a + k0 : a + k0 * lda;
    if (!c.tb) xb = c.two_pass ? b + k0 : b + k0 * ldb;
  }
  if (c.ta) {
    double *t = (double *)ws;
    if (a_layout == SMM_LAYOUT_KMAJOR) rc = transpose(a + k0 * lda, K, n1, lda, t, K, s);  // -> n1 x K
    else rc = transpose(a + k0, n1, K, lda, t, n1, s);                                      // -> K x n1
    if (rc) return rc;
    xa = t;
    la = c.two_pass ? K : n1;
  }
  if (c.tb) {
    double *t = (double *)(ws + c.ta_bytes);
    if (b_layout == SMM_LAYOUT_KMAJOR) rc = transpose(b + k0 * ldb, K, n2, ldb, t, K, s);  // -> n2 x K
    else rc = transpose(b + k0, n2, K, ldb, t, n2, s);                                      // -> K x n2
    if (rc) return rc;
    xb = t;
    lb = c.two_pass ? K : n2;
  }
  char *kws = ws + c.ta_bytes + c.tb_bytes + c.tmp_acc_bytes;
  const int64_t kb = workspace_bytes - c.ta_bytes - c.tb_bytes - c.tmp_acc_bytes;
  // repetition groups of at most SMM_MAX_DEPTH, one launch each, into rows [t0, t1) of acc
  uint64_t gw[8 * SMM_MAX_DEPTH];
  for (int t0 = 0; t0 < d; t0 += SMM_MAX_DEPTH) {
    const int t1 = t0 + SMM_MAX_DEPTH < d ? t0 + SMM_MAX_DEPTH : d;
    group_words(words_host, d, t0, t1, gw);
    SketchHashes h;
    load_hashes(h, gw, t1 - t0, log2b);
    char *accg = (char *)acc + acc_bytes(variant, t0, log2b);
    if (c.one_pass)
      rc = fwht1p_accumulate(h, xa, la, false, xb, lb, false, n1, n2, kk0, kk1, (double *)accg, acc_add, kws, kb,
                             s);  // k-major views (transposed above when needed)
    else if (c.fft_one_pass)
      rc = fft1p_accumulate(h, xa, la, xb, lb, n1, n2, kk0, kk1, (double *)accg, acc_add, kws, kb, s);
    else if (c.fft_two_pass)
      rc = fft2p_accumulate(h, xa, la, xb, lb, n1, n2, kk0, kk1, (double *)accg, acc_add, kws, kb, s);
    else if (c.two_pass)
      rc = fwht2p_accumulate(h, xa, la, xb, lb, n1, n2, kk0, kk1, (double *)accg, acc_add, kws, kb, s);
    else {
      void *dst = acc_add ? (void *)(ws + c.ta_bytes + c.tb_bytes) : (void *)accg;
      if (variant == SMM_VARIANT_FWHT)
        rc = fwht_accumulate(h, xa, la, xb, lb, n1, n2, kk0, kk1, (double *)dst, kws, kb, s);
      else
        rc = fft_accumulate(h, xa, la, xb, lb, n1, n2, kk0, kk1, (cplx *)dst, kws, kb, s);
      if (!rc && acc_add) rc = add_inplace((double *)accg, (const double *)dst, acc_bytes(variant, t1 - t0, log2b) / 8, s);
    }
    if (rc) return rc;
  }
  return SMM_OK;
}

int smm_copy2d(void *dst, int64_t dpitch, const void *src, int64_t spitch, int64_t width_bytes, int64_t rows,
               void *stream) {
  SMM_REQUIRE(width_bytes >= 0 && rows >= 0 && dpitch >= width_bytes && spitch >= width_bytes, "bad copy shape");
  SMM_REQUIRE(width_bytes == 0 || rows == 0 || (dst != nullptr && src != nullptr), "NULL argument");
  if (width_bytes == 0 || rows == 0) return SMM_OK;
  SMM_CUDA_TRY(cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, (size_t)width_bytes, (size_t)rows,
                                 cudaMemcpyDefault, (cudaStream_t)stream),
               "cudaMemcpy2DAsync");
  return SMM_OK;
}

int smm_compress_accumulate(int variant, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm, int64_t n1,
                            int64_t n2, int64_t k0, int64_t k1, const uint64_t *words_host, int d, int log2b,
                            void *acc, void *workspace, int64_t workspace_bytes, void *stream) {
  return smm_compress_accumulate_ex(variant, at, ld_at, SMM_LAYOUT_KMAJOR, bm, ld_bm, SMM_LAYOUT_KMAJOR, n1, n2, k0, k1,
                                    words_host, d, log2b, acc, workspace, workspace_bytes, stream);
}

int smm_finalize(int variant, const void *acc, double *polys, int d, int log2b, void *stream) {
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(acc != nullptr && polys != nullptr, "NULL argument");
  return finalize(variant, acc, polys, d, log2b, (cudaStream_t)stream);
}

int smm_extract_workspace(int d, int64_t n1, int64_t n2, int64_t r0, int64_t r1, int64_t *bytes) {
  SMM_REQUIRE(bytes != nullptr, "bytes is NULL");
  SMM_REQUIRE(d >= 1 && d <= SMM_MAX_DEPTH_TOTAL, "d must be in [1, %d], got %d", SMM_MAX_DEPTH_TOTAL, d);
  SMM_REQUIRE(r0 >= 0 && r1 >= r0 && r1 <= n1 && n2 >= 0, "row range [%lld, %lld) outside %lld rows", (long long)r0,
              (long long)r1, (long long)n1);
  *bytes = extract_workspace(n2, r0, r1) + big_hash_bytes(d);
  return SMM_OK;
}

int smm_extract(int variant, const double *polys, const uint64_t *words_host, int d, int log2b, int64_t n1,
                int64_t n2, int64_t r0, int64_t r1, double *est, int64_t ld_est, double thr, int strict,
                int64_t *hh_pairs, int64_t hh_cap, int64_t *hh_count, void *workspace, int64_t workspace_bytes,
                void *stream) {
  int rc = check_sketch(variant, d, log2b, true);
  if (rc) return rc;
  SMM_REQUIRE(polys != nullptr && words_host != nullptr && hh_count != nullptr, "NULL argument");
  SMM_REQUIRE(r0 >= 0 && r1 >= r0 && r1 <= n1 && n2 >= 0, "row range [%lld, %lld) outside %lld rows", (long long)r0,
              (long long)r1, (long long)n1);
  SMM_REQUIRE(n1 <= ((int64_t)1 << 32) && n2 <= ((int64_t)1 << 32), "keys must fit in 32 bits");
  SMM_REQUIRE(est == nullptr || ld_est >= n2, "ld_est < n2");
  SMM_REQUIRE(hh_cap >= 0, "hh_cap < 0");
  if (d > SMM_MAX_DEPTH)
    return extract_big(variant, words_host, d, log2b, polys, n2, r0, r1, est, ld_est, thr, strict, hh_pairs, hh_cap,
                       hh_count, (char *)workspace, workspace_bytes, (cudaStream_t)stream);
  SketchHashes h;
  load_hashes(h, words_host, d, log2b);
  return extract(variant, h, polys, n1, n2, r0, r1, est, ld_est, thr, strict, hh_pairs, hh_cap, hh_count,
                 (char *)workspace, workspace_bytes, (cudaStream_t)stream);
}

int smm_hh_pairs(const void *workspace, int64_t n2, int64_t r0, int64_t r1, int64_t *hh_pairs, int64_t hh_cap,
                 void *stream) {
  SMM_REQUIRE(workspace != nullptr, "workspace is NULL");
  SMM_REQUIRE(r0 >= 0 && r1 >= r0 && n2 >= 0 && hh_cap >= 0, "bad ranges");
  SMM_REQUIRE(hh_cap == 0 || hh_pairs != nullptr, "hh_pairs is NULL");
  return smm::hh_pairs(workspace, n2, r0, r1, hh_pairs, hh_cap, (cudaStream_t)stream);
}

int smm_query(int variant, const double *polys, const uint64_t *words_host, int d, int log2b, int64_t n1, int64_t n2,
              const int64_t *ij, int64_t count, double *est, double *reps, void *stream) {
  int rc = check_sketch(variant, d, log2b, true);
  if (rc) return rc;
  SMM_REQUIRE(count >= 0, "count < 0");
  SMM_REQUIRE(count == 0 || (polys != nullptr && words_host != nullptr && ij != nullptr && est != nullptr),
              "NULL argument");
  SMM_REQUIRE(n1 <= ((int64_t)1 << 32) && n2 <= ((int64_t)1 << 32), "keys must fit in 32 bits");
  if (d > SMM_MAX_DEPTH) return query_big(variant, words_host, d, log2b, polys, ij, count, est, reps, (cudaStream_t)stream);
  SketchHashes h;
  load_hashes(h, words_host, d, log2b);
  return query(variant, h, polys, ij, count, est, reps, (cudaStream_t)stream);
}

int64_t smm_kernel_launches(void) { return launches(); }

int smm_kernel_timing(int enable) {
  kernel_timing(enable);
  return SMM_OK;
}

int smm_kernel_timing_read(int channel, double *total_ms, int64_t *launches_out) {
  SMM_REQUIRE(total_ms != nullptr && launches_out != nullptr, "NULL argument");
  SMM_REQUIRE(channel == 0 || channel == 1, "channel must be 0 (compress) or 1 (extraction)");
  return kernel_timing_read(channel, total_ms, launches_out);
}

int smm_transpose(const double *in, int64_t rows, int64_t cols, int64_t ld_in, double *out, int64_t ld_out,
                  void *stream) {
  SMM_REQUIRE(rows >= 0 && cols >= 0 && ld_in >= cols && ld_out >= rows, "bad transpose shape");
  SMM_REQUIRE((rows == 0 || cols == 0) || (in != nullptr && out != nullptr), "NULL argument");
  return transpose(in, rows, cols, ld_in, out, ld_out, (cudaStream_t)stream);
}

int smm_fwht_batched(double *x, int64_t batch, int log2n, double scale, void *stream) {
  SMM_REQUIRE(log2n >= 0 && log2n <= 34, "transform length out of range");
  SMM_REQUIRE(batch >= 0 && (batch == 0 || x != nullptr), "NULL argument");
  return fwht_batched(x, batch, log2n, scale, (cudaStream_t)stream);
}

int smm_fft_batched(double *z, int64_t batch, int log2n, int inverse, double scale, void *stream) {
  SMM_REQUIRE(log2n >= 0 && log2n <= 30, "transform length out of range");
  SMM_REQUIRE(batch >= 0 && (batch == 0 || z != nullptr), "NULL argument");
  return fft_batched((cplx *)z, batch, log2n, inverse, scale, (cudaStream_t)stream);
}

}  // extern "C"
