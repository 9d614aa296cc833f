// Shared device helpers for the sketched-product kernels (sm_100a).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/sketchmm_b200.h"

namespace smm {

// ---------------------------------------------------------------- errors
void set_error(const char *fmt, ...);
int cuda_status(cudaError_t e, const char *what);
#define SMM_CUDA_TRY(expr, what)                          \
  do {                                                    \
    cudaError_t _e = (expr);                              \
    if (_e != cudaSuccess) return ::smm::cuda_status(_e, what); \
  } while (0)
void count_launch();
#define SMM_LAUNCH_CHECK(what)  \
  do {                          \
    ::smm::count_launch();      \
    SMM_CUDA_TRY(cudaGetLastError(), what); \
  } while (0)

int num_sms();

// Per-launch CUDA-event timing of the dominant kernels, for the bench's roofline
// (smm_kernel_timing): when enabled, a KernelTimer records an event pair on the
// launching stream around one launch of channel 0 (compress kernels) or 1 (extraction).
struct KernelTimer {
  cudaEvent_t ev[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  int channel = 0;
  KernelTimer(int channel, cudaStream_t s);
  ~KernelTimer();  // an unstopped timer (error path) returns its events unrecorded
  void stop();
};
// The L2 cache-policy encodings of createpolicy.fractional evict_last / evict_first,
// computed once per device; the two-pass kernels take them as parameters, so their
// cache-hinted loads and stores read the policy from a uniform register.
int l2_policies(uint64_t &evict_last, uint64_t &evict_first);
void kernel_timing(int on);
int kernel_timing_read(int channel, double *total_ms, int64_t *count);
// keep freed stream-ordered scratch in the device's default pool (transforms.cu)
void keep_pool_memory();

// ---------------------------------------------------------------- hashing
// One drawn hash function (hashing.py:35-51): bucket = ((a*x + c) mod 2^64) >> shift.
struct HashFn {
  unsigned long long a, c;
};

// The 4d hash functions of a sketch, passed by value to kernels.
// words layout (hashing.py:146-152): group g in {h1, h2, s1, s2}, function t:
//   a = words[g*2d + 2t], c = words[g*2d + 2t + 1]
struct SketchHashes {
  HashFn f[4][SMM_MAX_DEPTH];
  int d;
  int log2b;
};

void load_hashes(SketchHashes &h, const uint64_t *words_host, int d, int log2b);

__device__ __forceinline__ uint32_t eval_bucket(HashFn h, uint64_t x, int log2b) {
  // unsigned 64-bit wrap-around is exactly the reference's mod 2^64 (hashing.py:54-56)
  return (uint32_t)((h.a * x + h.c) >> (64 - log2b));
}
// sign bit (1 -> -1.0, 0 -> +1.0): top bit of a*x + c (hashing.py:59-61)
__device__ __forceinline__ uint32_t eval_signbit(HashFn h, uint64_t x) {
  return (uint32_t)((h.a * x + h.c) >> 63);
}
__device__ __forceinline__ double apply_sign(double v, uint32_t signbit) {
  return signbit ? -v : v;
}

// ---------------------------------------------------------------- misc
__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) {
  return {fma(a.re, b.re, -a.im * b.im), fma(a.re, b.im, a.im * b.re)};
}

}  // namespace smm
