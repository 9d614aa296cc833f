// L2 store bandwidth against the written footprint (is the ~7.6 TB/s "L2-resident
// store" ceiling an L2 limit or write-back to HBM?), store width (8 / 16 / 32 bytes
// per thread), and the Y pattern: write a footprint, read it back, repeat.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2write tools/l2write.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__global__ void k_w8(double *buf, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] = (double)(i + r);
}
__global__ void k_w16(double2 *buf, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      buf[i] = make_double2((double)(i + r), 1.0);
}
__global__ void k_w32(double *buf, size_t n4, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
      const double a = (double)(i + r);
      asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(buf + 4 * i), "d"(a), "d"(a), "d"(a), "d"(a)
                   : "memory");
    }
}
__global__ void k_w16_el(double2 *buf, size_t n, int reps, uint64_t pol) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double a = (double)(i + r);
      asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(buf + i), "d"(a), "d"(a), "l"(pol)
                   : "memory");
    }
}
// write the footprint, then read it back (the pass-1 -> pass-2 pattern), reps times
__global__ void k_wr(double2 *buf, size_t n, int reps, double *out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int r = 0; r < reps; ++r) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      buf[i] = make_double2((double)(i + r), 1.0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
      const double2 v = __ldcg(buf + i);
      acc += v.x;
    }
  }
  if (acc == 1.2345) out[0] = acc;
}
// sector-granular pattern: lane = (piece half h, row r): a warp instruction writes / reads 16
// rows x 32 bytes (rows 256 B apart); warp q of each 8-warp group owns bytes [32 q, 32 q + 32)
__global__ void k_w_rows32(double2 *buf, size_t nrows, int reps) {
  const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 7;
  const size_t grp = (size_t)blockIdx.x * (blockDim.x >> 8) + (threadIdx.x >> 8);
  const size_t ngrp = (size_t)gridDim.x * (blockDim.x >> 8);
  for (int r = 0; r < reps; ++r)
    for (size_t row0 = grp * 16; row0 < nrows; row0 += ngrp * 16) {
      const size_t row = row0 + (lane >> 1);
      buf[row * 16 + q * 2 + (lane & 1)] = make_double2((double)(row + r), 1.0);
    }
}
__global__ void k_r_rows32(const double2 *buf, size_t nrows, int reps, double *out) {
  const int lane = threadIdx.x & 31, q = (threadIdx.x >> 5) & 7;
  const size_t grp = (size_t)blockIdx.x * (blockDim.x >> 8) + (threadIdx.x >> 8);
  const size_t ngrp = (size_t)gridDim.x * (blockDim.x >> 8);
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t row0 = grp * 16; row0 < nrows; row0 += ngrp * 16) {
      const size_t row = row0 + (lane >> 1);
      acc += __ldcg(buf + row * 16 + q * 2 + (lane & 1)).x;
    }
  if (acc == 1.2345) out[0] = acc;
}
// strided sector reads: 32 B per row, rows 8 KB apart (a pass-2 read of a k-quad-major Y)
__global__ void k_r_stride8k(const double2 *buf, size_t bytes, int reps, double *out) {
  const int lane = threadIdx.x & 31;
  const size_t w = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const size_t nw = ((size_t)gridDim.x * blockDim.x) >> 5;
  const size_t nchunk = bytes / 32;  // 32-byte pieces; piece c lives at ((c % 256) * 256 + c / 256 % 256) ...
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t c0 = w * 16; c0 < nchunk; c0 += nw * 16) {
      const size_t c = c0 + (lane >> 1);
      const size_t blk = c >> 16, in = c & 65535;
      const size_t piece = (blk << 16) | ((in & 255) << 8) | (in >> 8);  // transpose 256 x 256 pieces
      acc += __ldcg(buf + piece * 2 + (lane & 1)).x;
    }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void k_r16(const double2 *buf, size_t n, int reps, double *out) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) acc += __ldcg(buf + i).x;
  if (acc == 1.2345) out[0] = acc;
}
__global__ void k_polw(uint64_t *p) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  p[0] = pol;
}

template <class F>
float time_ms(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char *w;
  CK(cudaMalloc(&w, (size_t)256 << 20));
  double *out;
  CK(cudaMalloc(&out, 64));
  uint64_t *dpol, pol;
  CK(cudaMalloc(&dpol, 8));
  k_polw<<<1, 1>>>(dpol);
  CK(cudaMemcpy(&pol, dpol, 8, cudaMemcpyDeviceToHost));
  for (size_t mb : {2, 4, 8, 16, 32, 48, 64, 96, 192}) {
    const size_t bytes = mb << 20;
    const int reps = mb <= 96 ? 40 : 4;
    CK(cudaMemset(w, 0, bytes));
    float m8 = time_ms([&] { k_w8<<<sms * 4, 512>>>((double *)w, bytes / 8, reps); });
    float m16 = time_ms([&] { k_w16<<<sms * 4, 512>>>((double2 *)w, bytes / 16, reps); });
    float m32 = time_ms([&] { k_w32<<<sms * 4, 512>>>((double *)w, bytes / 32, reps); });
    float mel = time_ms([&] { k_w16_el<<<sms * 4, 512>>>((double2 *)w, bytes / 16, reps, pol); });
    float mwr = time_ms([&] { k_wr<<<sms * 4, 512>>>((double2 *)w, bytes / 16, reps, out); });
    CK(cudaGetLastError());
    auto tb = [&](float ms, double f) { return (double)bytes * reps * f / ms / 1e9; };
    printf("%4zu MB: st8 %5.2f  st16 %5.2f  st32 %5.2f  st16.evict_last %5.2f TB/s | write+read %5.2f TB/s (both "
           "directions)\n",
           mb, tb(m8, 1), tb(m16, 1), tb(m32, 1), tb(mel, 1), tb(mwr, 2));
  }
  for (size_t mb : {32, 64}) {
    const size_t bytes = mb << 20;
    const int reps = 40;
    float a = time_ms([&] { k_w16<<<sms * 4, 512>>>((double2 *)w, bytes / 16, reps); });
    float b = time_ms([&] { k_w_rows32<<<sms * 4, 512>>>((double2 *)w, bytes / 256, reps); });
    float c = time_ms([&] { k_r16<<<sms * 4, 512>>>((const double2 *)w, bytes / 16, reps, out); });
    float d = time_ms([&] { k_r_rows32<<<sms * 4, 512>>>((const double2 *)w, bytes / 256, reps, out); });
    float e = time_ms([&] { k_r_stride8k<<<sms * 4, 512>>>((const double2 *)w, bytes, reps, out); });
    CK(cudaGetLastError());
    auto tb = [&](float ms) { return (double)bytes * reps / ms / 1e9; };
    printf("%4zu MB: st contiguous %5.2f  st 16 rows x 32 B %5.2f | ld contiguous %5.2f  ld 16 rows x 32 B %5.2f  "
           "ld 32 B at 8 KB stride %5.2f TB/s\n", mb, tb(a), tb(b), tb(c), tb(d), tb(e));
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
