// Do warp shuffles and shared-memory loads share a pipe?  Warps of a CTA run either a
// stream of 64-bit shared loads, a stream of 32-bit shuffles, or both (half the warps each);
// if the mixed run takes about as long as the slower stream alone, they overlap.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/shfl_lds tools/shfl_lds.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_mix(int mode, int iters, double *out) {
  __shared__ double sm[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sm[i] = i;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool do_lds = mode == 0 || (mode == 2 && (warp & 1) == 0);
  double acc = 0;
  if (do_lds) {
    int idx = threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
      double v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = sm[(idx + r * 256) & 4095];
#pragma unroll
      for (int r = 0; r < 8; ++r) acc += v[r];
      idx += 33;
    }
  } else {
    unsigned x = threadIdx.x;
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
      unsigned v[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = __shfl_xor_sync(0xffffffffu, x + r, (r + 1) & 31);
#pragma unroll
      for (int r = 0; r < 8; ++r) x += v[r];
      // 8 shuffles of 32 bits = the lanes' bytes of 4 doubles: match the LDS stream's bytes with 2 rounds
#pragma unroll
      for (int r = 0; r < 8; ++r) v[r] = __shfl_xor_sync(0xffffffffu, x + r, (r + 3) & 31);
#pragma unroll
      for (int r = 0; r < 8; ++r) x ^= v[r];
    }
    acc = x;
  }
  if (acc == 123.456) out[0] = acc;
  (void)lane;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out;
  cudaMalloc(&out, 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[3] = {"LDS.64 only (all warps)", "SHFL only (all warps)", "half LDS + half SHFL"};
  for (int mode = 0; mode < 3; ++mode) {
    const int iters = 4096;
    k_mix<<<sms * 2, 512>>>(mode, iters, out);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k_mix<<<sms * 2, 512>>>(mode, iters, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    // bytes moved per warp-iteration: LDS 8 x 256 B, SHFL 16 x 128 B (same)
    const double bytes = (double)sms * 2 * 16 * iters * 2048;
    printf("%-26s %8.3f ms   %.1f TB/s equivalent (%.1f B/clk/SM at 1965 MHz)\n", names[mode], ms,
           bytes / ms / 1e9, bytes / (ms * 1e-3) / sms / 1.965e9);
  }
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
