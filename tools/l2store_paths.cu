// Is the ~7.6 TB/s ceiling of L2-resident stores (profiles/r02_l2write.txt) a per-SM
// store-path limit or a chip-wide L2 limit, and do TMA bulk stores (smem -> global,
// cp.async.bulk) get past it?  One CTA per SM (forced by shared-memory size), a 64 MB
// footprint written `reps` times, on all SMs and on half of them.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/l2store_paths tools/l2store_paths.cu
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

constexpr int SMEM = 160 * 1024;  // one CTA per SM

// LSU stores, 16 bytes per thread, each CTA owns a contiguous share of the footprint
__global__ void k_lsu(double2 *buf, size_t n, int reps) {
  extern __shared__ __align__(128) char smc[];
  double2 *sm = (double2 *)smc;
  if (threadIdx.x == 0) sm[0] = make_double2(0, 0);
  const size_t per = n / gridDim.x;
  double2 *my = buf + blockIdx.x * per;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) my[i] = make_double2((double)(i + r), 1.0);
}

// TMA bulk stores of CH-byte chunks from one smem buffer, up to INF groups in flight
template <int CH, int INF>
__global__ void k_bulk(char *buf, size_t bytes, int reps) {
  extern __shared__ __align__(128) char smc[];
  char *sm = smc;
  for (int i = threadIdx.x; i < CH * INF / 16; i += blockDim.x) ((double2 *)sm)[i] = make_double2(i, 1.0);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x != 0) return;
  const size_t per = bytes / gridDim.x / CH * CH;
  char *my = buf + blockIdx.x * per;
  const uint32_t src0 = (uint32_t)__cvta_generic_to_shared(sm);
  int q = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t o = 0; o < per; o += CH) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(my + o),
                   "r"(src0 + (uint32_t)(q * CH)), "n"(CH)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(INF - 1) : "memory");
      q = q + 1 == INF ? 0 : q + 1;
    }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// LSU loads (L2-resident), for the read side of the same question
__global__ void k_ld(const double2 *buf, size_t n, int reps, double *out) {
  extern __shared__ __align__(128) char smc[];
  double2 *sm = (double2 *)smc;
  const size_t per = n / gridDim.x;
  const double2 *my = buf + blockIdx.x * per;
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = threadIdx.x; i < per; i += blockDim.x) acc += __ldcg(my + i).x;
  if (acc == 1.2345) out[0] = acc;
  if (threadIdx.x == 0 && acc == 2.5) sm[0].x = acc;
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
  CK(cudaFuncSetAttribute(k_lsu, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(k_ld, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(k_bulk<8192, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(k_bulk<16384, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(k_bulk<2048, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  CK(cudaFuncSetAttribute(k_bulk<512, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM));
  for (size_t mb : {32, 64, 96}) {
    const size_t bytes = mb << 20;
    const int reps = 40;
    CK(cudaMemset(w, 0, bytes));
    for (int g : {sms, sms / 2, sms / 4}) {
      auto tb = [&](float ms) { return (double)bytes * reps / ms / 1e9; };
      float a = time_ms([&] { k_lsu<<<g, 1024, SMEM>>>((double2 *)w, bytes / 16, reps); });
      float b = time_ms([&] { k_bulk<8192, 8><<<g, 128, SMEM>>>(w, bytes, reps); });
      float c = time_ms([&] { k_bulk<16384, 8><<<g, 128, SMEM>>>(w, bytes, reps); });
      float d = time_ms([&] { k_bulk<2048, 32><<<g, 128, SMEM>>>(w, bytes, reps); });
      float e = time_ms([&] { k_bulk<512, 64><<<g, 128, SMEM>>>(w, bytes, reps); });
      float f = time_ms([&] { k_ld<<<g, 1024, SMEM>>>((const double2 *)w, bytes / 16, reps, out); });
      CK(cudaGetLastError());
      printf("%3zu MB, %3d CTAs (1/SM): st16 LSU %5.2f | bulk 8K x8 %5.2f  16K x8 %5.2f  2K x32 %5.2f  512 x64 %5.2f | "
             "ld16 LSU %5.2f TB/s  (LSU st per SM %.1f B/clk at 1.965 GHz)\n",
             mb, g, tb(a), tb(b), tb(c), tb(d), tb(e), tb(f), tb(a) * 1e12 / g / 1.965e9);
    }
  }
  CK(cudaDeviceSynchronize());
  printf("done\n");
  return 0;
}
