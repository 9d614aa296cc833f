// Micro-benchmarks that pin the B200 throughputs the compress kernel design
// depends on: FP64 add/FMA pipe, shared-memory bandwidth for 64-bit accesses,
// warp shuffles, L2-resident and HBM read bandwidth, DSMEM, TMEM (tcgen05.ld/st)
// and FP64 DMMA.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

static int g_sms;

template <typename F>
static float time_ms(F f, int reps = 5) {
  cudaEvent_t a, b; CK(cudaEventCreate(&a)); CK(cudaEventCreate(&b));
  f(); CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    CK(cudaEventRecord(a)); f(); CK(cudaEventRecord(b)); CK(cudaEventSynchronize(b));
    float ms; CK(cudaEventElapsedTime(&ms, a, b)); if (ms < best) best = ms;
  }
  CK(cudaGetLastError());
  return best;
}

// ---------------- FP64 add / fma -----------------
__global__ void k_dadd(double* out, int iters, double s) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = x[j] + s;
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = x[j] - s * 0.5;
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += x[j];
  if (t == 12345.678) out[0] = t;
}
__global__ void k_dfma(double* out, int iters, double s) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], s, 0.25);
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], s, -0.25);
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += x[j];
  if (t == 12345.678) out[0] = t;
}
// butterfly-like: u+v,u-v on register pairs (the FWHT inner op)
__global__ void k_bfly(double* out, int iters) {
  double x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int h = 1; h < 16; h <<= 1)
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (!(j & h)) { double u = x[j], v = x[j + h]; x[j] = u + v; x[j + h] = (u - v) * 0.0625; }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) t += x[j];
  if (t == 12345.678) out[0] = t;
}

// ---------------- shared memory -----------------
__global__ void k_lds64(double* out, int iters) {
  extern __shared__ double sm[];
  int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  double acc = 0;
  int idx = tid;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += sm[(idx + j * 1024) & 8191];
    idx = (idx + 32) & 8191;
  }
  if (acc == 1.2345) out[0] = acc;
}
__global__ void k_sts64(double* out, int iters) {
  extern __shared__ double sm[];
  int tid = threadIdx.x;
  double v = tid;
  int idx = tid;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) sm[(idx + j * 1024) & 8191] = v + j;
    idx = (idx + 32) & 8191;
  }
  __syncthreads();
  if (sm[tid] == 1.2345) out[0] = 1;
}
// random 64-bit gathers from smem (bank-conflicted)
__global__ void k_lds64_rand(double* out, const int* perm, int iters) {
  extern __shared__ double sm[];
  int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = i;
  __syncthreads();
  int p[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) p[j] = perm[(tid * 8 + j) & 8191];
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { acc += sm[p[j]]; p[j] = (p[j] + 97) & 8191; }
  }
  if (acc == 1.2345) out[0] = acc;
}

// ---------------- shuffles -----------------
__global__ void k_shfl(double* out, int iters) {
  unsigned x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] += __shfl_xor_sync(0xffffffffu, x[j], 1 << (j & 3));
  }
  unsigned t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t ^= x[j];
  if (t == 0x12345678u) out[0] = t;
}

// ---------------- global reads -----------------
__global__ void k_read(const double2* __restrict__ p, size_t n2, int reps, double* out) {
  double acc = 0;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
      double2 v = __ldcg(p + i);
      acc += v.x + v.y;
    }
  if (acc == 1.2345) out[0] = acc;
}

// ---------------- DSMEM -----------------
__global__ void __cluster_dims__(4, 1, 1) k_dsmem(double* out, int iters) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  int tid = threadIdx.x;
  for (int i = tid; i < 8192; i += blockDim.x) sm[i] = i;
  cl.sync();
  unsigned r = (cl.block_rank() + 1) % cl.num_blocks();
  double* rem = cl.map_shared_rank(sm, r);
  double acc = 0;
  int idx = tid;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += rem[(idx + j * 1024) & 8191];
    idx = (idx + 32) & 8191;
  }
  cl.sync();
  if (acc == 1.2345) out[0] = acc;
}
__global__ void __cluster_dims__(4, 1, 1) k_dsmem_st(double* out, int iters) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  int tid = threadIdx.x;
  cl.sync();
  unsigned r = (cl.block_rank() + 1) % cl.num_blocks();
  double* rem = cl.map_shared_rank(sm, r);
  int idx = tid;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) rem[(idx + j * 1024) & 8191] = (double)(i + j);
    idx = (idx + 32) & 8191;
  }
  cl.sync();
  if (sm[tid] == 1.2345) out[0] = 1;
}

// ---------------- TMEM -----------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k_tmem(double* out, int iters, int mode) {
  __shared__ uint32_t taddr_s;
  int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" :: "r"(smem_u32(&taddr_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t base = taddr_s + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  uint32_t r[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) r[j] = threadIdx.x * 16 + j;
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 128; c += 16) {
      uint32_t a = base + c;
      if (mode == 0) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                     :: "r"(a), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
                        "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
      } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                       "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                     : "r"(a));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
        for (int j = 0; j < 16; ++j) acc += r[j];
      }
    }
    if (mode == 0) asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(taddr_s));
  if (acc == 0x12345u) out[0] = acc;
}

// ---------------- DMMA -----------------
__global__ void k_dmma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - threadIdx.x * 1e-4;
  double c[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) { c[j][0] = j; c[j][1] = -j; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) t += c[j][0] + c[j][1];
  if (t == 1.2345) out[0] = t;
}
__global__ void k_dmma16(double* out, int iters) {
  double a[8], b[4];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll
  for (int j = 0; j < 4; ++j) b[j] = 1.0 - j * 1e-4;
  double c[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) for (int q = 0; q < 4; ++q) c[j][q] = j + q;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[j][0]), "+d"(c[j][1]), "+d"(c[j][2]), "+d"(c[j][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 2; ++j) for (int q = 0; q < 4; ++q) t += c[j][q];
  if (t == 1.2345) out[0] = t;
}

// ---------------- random 8-byte gathers from an L2-resident table (the extraction pattern) -----------------
__global__ void k_gather(const double *tab, uint32_t mask, int iters, double *out) {
  uint32_t x = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0;
  for (int i = 0; i < iters; ++i) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      x = x * 1664525u + 1013904223u;
      v[j] = __ldg(tab + ((x >> 7) & mask));
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += v[j];
  }
  if (acc == 123.0) out[0] = acc;
}

// ---------------- coalesced 8-byte stores into an L2-resident buffer (the pass-1 Y pattern) -----------------
__global__ void k_write(double *buf, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) buf[i] = (double)(i + r);
}

__global__ void k_write2(double2 *buf, size_t n, int reps) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride)
      buf[i] = make_double2((double)(i + r), 1.0);
}

// one 64 KB bulk copy (TMA engine) from shared memory per iteration and CTA
__global__ void k_bulk_store(char *buf, size_t bytes, int reps) {
  extern __shared__ __align__(128) char smb[];
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((int *)smb)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const size_t tiles = bytes / 65536;
    for (int r = 0; r < reps; ++r)
      for (size_t t = blockIdx.x; t < tiles; t += gridDim.x) {
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 65536;" ::"l"(buf + t * 65536),
                     "r"((uint32_t)__cvta_generic_to_shared(smb))
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

int main() {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  g_sms = prop.multiProcessorCount;
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("device %s sms=%d clock(max)=%.0f MHz smemPerBlockOptin=%zu l2=%d\n", prop.name, g_sms, clk_khz / 1e3,
         prop.sharedMemPerBlockOptin, prop.l2CacheSize);
  double* out; CK(cudaMalloc(&out, 64));
  const int T = 512, B = g_sms * 4;
  {
    int it = 4096;
    float ms = time_ms([&] { k_dadd<<<B, T>>>(out, it, 1.0); });
    double ops = (double)B * T * it * 16;
    printf("DADD      : %.2f Tops/s  (%.1f ops/clk/SM at max clk)\n", ops / ms / 1e9, ops / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
    ms = time_ms([&] { k_dfma<<<B, T>>>(out, it, 1.0001); });
    printf("DFMA      : %.2f Tfma/s (%.1f fma/clk/SM)\n", ops / ms / 1e9, ops / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
    int itb = 1024;
    ms = time_ms([&] { k_bfly<<<B, 256>>>(out, itb); });
    double bops = (double)B * 256 * itb * 4 * 8 * 3;  // add, sub, mul per butterfly
    printf("BFLY(reg) : %.2f Tops/s (add+sub+mul) (%.1f ops/clk/SM)\n", bops / ms / 1e9, bops / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
  }
  {
    CK(cudaFuncSetAttribute(k_lds64, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_sts64, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_lds64_rand, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    int it = 2048;
    float ms = time_ms([&] { k_lds64<<<g_sms * 2, 1024, 65536>>>(out, it); });
    double bytes = (double)g_sms * 2 * 1024 * it * 8 * 8;
    printf("LDS.64    : %.1f TB/s  (%.1f B/clk/SM)\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
    ms = time_ms([&] { k_sts64<<<g_sms * 2, 1024, 65536>>>(out, it); });
    printf("STS.64    : %.1f TB/s  (%.1f B/clk/SM)\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
    int* perm; CK(cudaMalloc(&perm, 8192 * 4));
    int h[8192]; unsigned s = 12345; for (int i = 0; i < 8192; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 8) & 8191; }
    CK(cudaMemcpy(perm, h, sizeof(h), cudaMemcpyHostToDevice));
    ms = time_ms([&] { k_lds64_rand<<<g_sms * 2, 1024, 65536>>>(out, perm, it); });
    printf("LDS.64 rnd: %.1f TB/s  (%.1f B/clk/SM useful)\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
  }
  {
    int it = 4096;
    float ms = time_ms([&] { k_shfl<<<g_sms * 4, 512>>>(out, it); });
    double n = (double)g_sms * 4 * 512 * it * 8;
    printf("SHFL.32   : %.1f Gthread-shfl/s (%.1f lanes/clk/SM)\n", n / ms / 1e6, n / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
  }
  {
    for (size_t mb : {32, 64, 96, 4096}) {
      size_t bytes = mb << 20;
      double2* p; CK(cudaMalloc(&p, bytes)); CK(cudaMemset(p, 0, bytes));
      int reps = mb <= 96 ? 20 : 2;
      float ms = time_ms([&] { k_read<<<g_sms * 8, 512>>>(p, bytes / 16, reps, out); });
      printf("read %4zu MB x%d: %.2f TB/s\n", mb, reps, (double)bytes * reps / ms / 1e9);
      CK(cudaFree(p));
    }
  }
  {
    // 5 x 2^16 doubles (2.6 MB, cfg3's polys) and 2^20 doubles (8 MB)
    for (uint32_t n : {5u * 65536u, 1u << 20}) {
      uint32_t m = 1; while (m < n) m <<= 1; m -= 1;
      double *tab; CK(cudaMalloc(&tab, (size_t)(m + 1) * 8)); CK(cudaMemset(tab, 0, (size_t)(m + 1) * 8));
      int it = 256;
      float ms = time_ms([&] { k_gather<<<g_sms * 8, 256>>>(tab, m, it, out); });
      double g = (double)g_sms * 8 * 256 * it * 8;
      printf("gather8 %4.1f MB: %.1f G/s (%.2f gathers/clk/SM, random 8-byte loads, one line each)\n",
             (m + 1) * 8 / 1048576.0, g / ms / 1e6, g / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
      CK(cudaFree(tab));
    }
    size_t bytes = (size_t)64 << 20;
    double *w; CK(cudaMalloc(&w, bytes));
    float ms = time_ms([&] { k_write<<<g_sms * 8, 512>>>(w, bytes / 8, 20); });
    printf("write  64 MB x20: %.2f TB/s (L2-resident stores, 8 B/thread)\n", (double)bytes * 20 / ms / 1e9);
    ms = time_ms([&] { k_write2<<<g_sms * 8, 512>>>((double2 *)w, bytes / 16, 20); });
    printf("write2 64 MB x20: %.2f TB/s (L2-resident stores, 16 B/thread)\n", (double)bytes * 20 / ms / 1e9);
    CK(cudaFuncSetAttribute(k_bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    ms = time_ms([&] { k_bulk_store<<<g_sms * 2, 128, 65536>>>((char *)w, bytes, 20); });
    printf("bulk   64 MB x20: %.2f TB/s (L2-resident cp.async.bulk stores from smem)\n", (double)bytes * 20 / ms / 1e9);
    CK(cudaFree(w));
  }
  {
    CK(cudaFuncSetAttribute(k_dsmem, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    CK(cudaFuncSetAttribute(k_dsmem_st, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
    int it = 512;
    float ms = time_ms([&] { k_dsmem<<<(g_sms / 4) * 4, 1024, 65536>>>(out, it); });
    double bytes = (double)(g_sms / 4) * 4 * 1024 * it * 8 * 8;
    printf("DSMEM ld  : %.1f TB/s  (%.1f B/clk/SM)\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / ((g_sms / 4) * 4) / (clk_khz * 1e3));
    ms = time_ms([&] { k_dsmem_st<<<(g_sms / 4) * 4, 1024, 65536>>>(out, it); });
    printf("DSMEM st  : %.1f TB/s  (%.1f B/clk/SM)\n", bytes / ms / 1e9, bytes / (ms * 1e-3) / ((g_sms / 4) * 4) / (clk_khz * 1e3));
  }
  {
    int it = 256;
    for (int mode = 0; mode < 2; ++mode) {
      float ms = time_ms([&] { k_tmem<<<g_sms, 256>>>(out, it, mode); });
      double bytes = (double)g_sms * 256 * it * 128 * 4;
      printf("TMEM %s : %.1f TB/s  (%.1f B/clk/SM)\n", mode ? "ld" : "st", bytes / ms / 1e9, bytes / (ms * 1e-3) / g_sms / (clk_khz * 1e3));
    }
  }
  {
    int it = 2048;
    float ms = time_ms([&] { k_dmma<<<g_sms * 4, 256>>>(out, it); });
    double fl = (double)g_sms * 4 * (256 / 32) * it * 4 * (8 * 8 * 4 * 2);
    printf("DMMA m8n8k4 : %.2f TFLOP/s\n", fl / ms / 1e9);
    ms = time_ms([&] { k_dmma16<<<g_sms * 4, 256>>>(out, it); });
    fl = (double)g_sms * 4 * (256 / 32) * it * 2 * (16 * 8 * 16 * 2);
    printf("DMMA m16n8k16: %.2f TFLOP/s\n", fl / ms / 1e9);
  }
  printf("done\n");
  return 0;
}
