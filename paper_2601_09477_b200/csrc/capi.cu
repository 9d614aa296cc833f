// extern "C" entry points declared in include/sketchmm_b200.h.  Validation
// mirrors the reference's parameter checks (sketch.py:68-82, hashing.py:25-32)
// and always happens before any kernel is launched.
#include "plan.cuh"

namespace smm {
const char *last_error();
int hash_tables(const SketchHashes &h, int group, int64_t n, uint32_t *buckets, int8_t *signs, cudaStream_t s);
int64_t fwht_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int G);
int64_t fft_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K, int Gmax);
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
int64_t launches();
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

static int check_sketch(int variant, int d, int log2b) {
  SMM_REQUIRE(variant == SMM_VARIANT_FFT || variant == SMM_VARIANT_FWHT, "unknown transform variant %d", variant);
  SMM_REQUIRE(d >= 1 && d % 2 == 1 && d <= SMM_MAX_DEPTH, "d must be an odd integer in [1, %d], got %d",
              SMM_MAX_DEPTH, d);
  SMM_REQUIRE(log2b >= 1 && log2b <= 32, "b must be a power of two in [2, 2**32], got 2**%d", log2b);
  if (variant == SMM_VARIANT_FFT) SMM_REQUIRE(log2b <= 30, "fft variant supports b <= 2**30");
  return SMM_OK;
}

extern "C" {

int smm_abi_version(void) { return 1; }

const char *smm_last_error(void) { return last_error(); }

int smm_hash_tables(const uint64_t *words_host, int d, int log2b, int group, int64_t n, uint32_t *buckets_out,
                    int8_t *signs_out, void *stream) {
  SMM_REQUIRE(words_host != nullptr, "hash words must not be NULL");
  SMM_REQUIRE(d >= 1 && d <= SMM_MAX_DEPTH, "d out of range");
  SMM_REQUIRE(log2b >= 1 && log2b <= 32, "log2b out of range");
  SMM_REQUIRE(group >= 0 && group <= 3, "group must be 0..3");
  SMM_REQUIRE(n >= 0 && n <= ((int64_t)1 << 32), "keys must fit in 32 bits");
  SMM_REQUIRE(group >= 2 || buckets_out != nullptr, "buckets_out is NULL");
  SMM_REQUIRE(group < 2 || signs_out != nullptr, "signs_out is NULL");
  SketchHashes h;
  load_hashes(h, words_host, d, log2b);
  return hash_tables(h, group, n, buckets_out, signs_out, (cudaStream_t)stream);
}

int smm_compress_workspace(int variant, int d, int log2b, int64_t n1, int64_t n2, int64_t k0, int64_t k1,
                           int64_t *bytes) {
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(bytes != nullptr, "bytes is NULL");
  SMM_REQUIRE(n1 >= 0 && n2 >= 0 && k0 >= 0 && k1 >= k0, "bad shapes");
  *bytes = variant == SMM_VARIANT_FWHT ? fwht_workspace(d, log2b, n1, n2, k1 - k0, num_sms())
                                       : fft_workspace(d, log2b, n1, n2, k1 - k0, num_sms());
  return SMM_OK;
}

int smm_compress_accumulate(int variant, const double *at, int64_t ld_at, const double *bm, int64_t ld_bm, int64_t n1,
                            int64_t n2, int64_t k0, int64_t k1, const uint64_t *words_host, int d, int log2b,
                            void *acc, void *workspace, int64_t workspace_bytes, void *stream) {
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(words_host != nullptr && acc != nullptr, "NULL argument");
  SMM_REQUIRE(n1 >= 0 && n2 >= 0 && n1 < ((int64_t)1 << 31) && n2 < ((int64_t)1 << 31), "operand sizes out of range");
  SMM_REQUIRE(k0 >= 0 && k1 >= k0, "inner range [%lld, %lld) invalid", (long long)k0, (long long)k1);
  SMM_REQUIRE(k1 == k0 || ((at != nullptr || n1 == 0) && (bm != nullptr || n2 == 0)), "operand pointer is NULL");
  SMM_REQUIRE(ld_at >= n1 && ld_bm >= n2, "leading dimension smaller than row length");
  SketchHashes h;
  load_hashes(h, words_host, d, log2b);
  cudaStream_t s = (cudaStream_t)stream;
  if (variant == SMM_VARIANT_FWHT)
    return fwht_accumulate(h, at, ld_at, bm, ld_bm, n1, n2, k0, k1, (double *)acc, (char *)workspace,
                           workspace_bytes, s);
  return fft_accumulate(h, at, ld_at, bm, ld_bm, n1, n2, k0, k1, (cplx *)acc, (char *)workspace, workspace_bytes,
                        s);
}

int smm_finalize(int variant, const void *acc, double *polys, int d, int log2b, void *stream) {
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(acc != nullptr && polys != nullptr, "NULL argument");
  return finalize(variant, acc, polys, d, log2b, (cudaStream_t)stream);
}

int smm_extract_workspace(int d, int64_t n1, int64_t n2, int64_t r0, int64_t r1, int64_t *bytes) {
  (void)d;
  SMM_REQUIRE(bytes != nullptr, "bytes is NULL");
  SMM_REQUIRE(r0 >= 0 && r1 >= r0 && r1 <= n1 && n2 >= 0, "row range [%lld, %lld) outside %lld rows", (long long)r0,
              (long long)r1, (long long)n1);
  *bytes = extract_workspace(n2, r0, r1);
  return SMM_OK;
}

int smm_extract(int variant, const double *polys, const uint64_t *words_host, int d, int log2b, int64_t n1,
                int64_t n2, int64_t r0, int64_t r1, double *est, int64_t ld_est, double thr, int strict,
                int64_t *hh_pairs, int64_t hh_cap, int64_t *hh_count, void *workspace, int64_t workspace_bytes,
                void *stream) {
  int rc = check_sketch(variant, d, log2b);
  if (rc) return rc;
  SMM_REQUIRE(polys != nullptr && words_host != nullptr && hh_count != nullptr, "NULL argument");
  SMM_REQUIRE(r0 >= 0 && r1 >= r0 && r1 <= n1 && n2 >= 0, "row range [%lld, %lld) outside %lld rows", (long long)r0,
              (long long)r1, (long long)n1);
  SMM_REQUIRE(n1 <= ((int64_t)1 << 32) && n2 <= ((int64_t)1 << 32), "keys must fit in 32 bits");
  SMM_REQUIRE(est == nullptr || ld_est >= n2, "ld_est < n2");
  SMM_REQUIRE(hh_cap >= 0, "hh_cap < 0");
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

int64_t smm_kernel_launches(void) { return launches(); }

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
