// Distributed shared memory (DSMEM) bandwidth on B200 for the exchange patterns a
// cluster-resident two-pass transform would need ("measure bulk DSMEM
// before ruling out a cluster-resident exchange"):
//   bulk   cp.async.bulk.shared::cluster.shared::cta (one elected thread per CTA pushes
//          its smem buffer into a peer CTA's smem, completion on the peer's mbarrier)
//   st16   st.shared::cluster.v2.f64 from every thread (16-byte remote stores, no
//          dependent loads), followed by a cluster barrier per round
//   ld16   ld.shared::cluster.v2.f64 from every thread, 8 independent loads in flight
// for cluster sizes 2, 4 and 8; every CTA sends to rank (r + 1) % size, so every SM's
// DSMEM port is both a source and a sink.  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_bulk tools/dsmem_bulk.cu
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

#define CK(x)                                                                                          \
  do {                                                                                                 \
    cudaError_t e = (x);                                                                               \
    if (e != cudaSuccess) {                                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);                   \
      exit(1);                                                                                         \
    }                                                                                                  \
  } while (0)

constexpr int BUF = 96 * 1024;  // bytes per direction per round (src + dst = 192 KB of smem)
constexpr int CHUNK = 16 * 1024;

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_bulk(double *out, int rounds) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t mbar;
  cg::cluster_group cl = cg::this_cluster();
  unsigned char *src = sm, *dst = sm + BUF;
  for (int i = threadIdx.x; i < BUF / 8; i += blockDim.x) ((double *)src)[i] = i;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  // peer's dst buffer and mbarrier in the cluster shared window
  uint32_t rdst, rbar;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rdst) : "r"(smem_u32(dst)), "r"(peer));
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar) : "r"(smem_u32(&mbar)), "r"(peer));
  uint32_t phase = 0;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x == 0) {
      // expect this round's bytes from the CTA that sends to us, then push ours
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(BUF)
                   : "memory");
    }
    cl.sync();  // every CTA armed its barrier before any bytes of this round land
    if (threadIdx.x == 0) {
#pragma unroll 1
      for (int c = 0; c < BUF; c += CHUNK)
        asm volatile(
            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                rdst + c),
            "r"(smem_u32(src + c)), "r"(CHUNK), "r"(rbar)
            : "memory");
      // wait for our own incoming bytes
      uint32_t done = 0;
      while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(smem_u32(&mbar)), "r"(phase)
            : "memory");
    }
    phase ^= 1;
  }
  cl.sync();
  if (threadIdx.x == 0 && ((double *)dst)[5] == 1.2345) out[0] = 1;
}

__global__ void k_st16(double *out, int rounds) {
  extern __shared__ __align__(128) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  double2 *dst = (double2 *)(sm + BUF);
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  double2 *rem = cl.map_shared_rank(dst, peer);
  const int n = BUF / 16;
  for (int r = 0; r < rounds; ++r) {
#pragma unroll 4
    for (int i = threadIdx.x; i < n; i += blockDim.x) rem[i] = make_double2(r, i);
    cl.sync();
  }
  if (dst[threadIdx.x].x == 1.2345) out[0] = 1;
}

__global__ void k_ld16(double *out, int rounds) {
  extern __shared__ __align__(128) unsigned char sm[];
  cg::cluster_group cl = cg::this_cluster();
  double2 *src = (double2 *)sm;
  const int n = BUF / 16;
  for (int i = threadIdx.x; i < n; i += blockDim.x) src[i] = make_double2(i, -i);
  cl.sync();
  const unsigned peer = (cl.block_rank() + 1) % cl.num_blocks();
  const double2 *rem = cl.map_shared_rank(src, peer);
  double acc = 0;
  for (int r = 0; r < rounds; ++r) {
    for (int i0 = threadIdx.x; i0 < n; i0 += 8 * blockDim.x) {
      double2 v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int i = i0 + j * blockDim.x;
        v[j] = i < n ? rem[i] : make_double2(0, 0);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) acc += v[j].x;
    }
  }
  cl.sync();
  if (acc == 1.2345) out[0] = acc;
}

template <typename K>
static void run(const char *name, K kern, int csize, int sms, double clk_hz, double *out) {
  const int smem = 2 * BUF;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  if (csize > 8) CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg = {};
  int nclusters = sms / csize;
  cfg.gridDim = dim3(nclusters * csize);
  cfg.blockDim = dim3(512);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int maxc = 0;
  CK(cudaOccupancyMaxActiveClusters(&maxc, (void *)kern, &cfg));
  if (maxc < nclusters) {
    nclusters = maxc;
    cfg.gridDim = dim3(nclusters * csize);
  }
  const int rounds = 400;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaLaunchKernelEx(&cfg, kern, out, 10));
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    CK(cudaEventRecord(a));
    CK(cudaLaunchKernelEx(&cfg, kern, out, rounds));
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    best = ms < best ? ms : best;
  }
  const int ctas = nclusters * csize;
  const double bytes = (double)ctas * rounds * BUF;
  printf("%-5s cluster %d (%3d CTAs): %7.2f TB/s  %6.1f B/clk/SM\n", name, csize, ctas, bytes / (best * 1e-3) / 1e12,
         bytes / (best * 1e-3) / ctas / clk_hz);
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  double *out;
  CK(cudaMalloc(&out, 64));
  printf("sms=%d clock(max)=%d MHz; %d KB per CTA per round\n", sms, clk_khz / 1000, BUF / 1024);
  for (int cs : {2, 4, 8}) {
    run("bulk", k_bulk, cs, sms, clk_khz * 1e3, out);
    run("st16", k_st16, cs, sms, clk_khz * 1e3, out);
    run("ld16", k_ld16, cs, sms, clk_khz * 1e3, out);
  }
  printf("done\n");
  return 0;
}
