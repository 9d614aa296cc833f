// L2 die locality probe: does B200's L2 store bandwidth depend on whether the
// writing SM and the written 2 KB chunk sit on the same die?
//   1. SM -> die: latency of dependent L2-hit loads from every SM to one chunk (bimodal)
//   2. chunk -> die: latency from SMs of die 0 to every 2 KB chunk of a 64 MB buffer
//   3. store / load bandwidth when every SM touches only same-die chunks, only
//      other-die chunks, or both (same bytes, L2-resident)
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2die l2die.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e = (x);                                                                       \
    if (e != cudaSuccess) {                                                                    \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);           \
      exit(1);                                                                                 \
    }                                                                                          \
  } while (0)

__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

__device__ __forceinline__ uint64_t ld_cg(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.global.cg.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// buffer words are 0, so v & 0 chains the loads without changing the address
__device__ uint64_t g_zero;  // 0 at run time; unknown to the compiler
__device__ __forceinline__ unsigned chase(const char *base, int nlines, int reps) {
  uint64_t v = 0;
  const uint64_t z = *(volatile uint64_t *)&g_zero;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r)
    for (int l = 0; l < nlines; ++l) v += ld_cg((const uint64_t *)(base + (v * z) + l * 128));
  asm volatile("" ::"l"(v));
  long long t1;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t1) : "l"(v));
  return (unsigned)((t1 - t0) / (reps * nlines)) + (unsigned)(v & 1);
}

__global__ void k_sm_lat(const char *buf, unsigned *lat_sm) {
  extern __shared__ char pad[];
  if (threadIdx.x == 0) {
    pad[0] = 0;
    chase(buf, 16, 2);  // warm
    lat_sm[smid()] = chase(buf, 16, 8);
  }
}

// block b (on SM smid) measures chunks c = b, b + grid, ...
__global__ void k_chunk_lat(const char *buf, int nchunks, unsigned *lat_chunk, int *chunk_sm) {
  extern __shared__ char pad[];
  if (threadIdx.x == 0) {
    pad[0] = 0;
    const unsigned s = smid();
    for (int c = blockIdx.x; c < nchunks; c += gridDim.x) {
      chase(buf + (size_t)c * 2048, 16, 1);
      lat_chunk[c] = chase(buf + (size_t)c * 2048, 16, 3);
      chunk_sm[c] = (int)s;
    }
  }
}

// every block claims a rank among the blocks of its die, then streams 16-byte
// stores (or loads) over its share of the chunk list chosen for that die
__global__ void k_stream(double2 *buf, const int *die_of_sm, const int *lists, const int *list_len,
                         const int *blocks_per_die, int *rank_ctr, int reps, int mode /*0 st, 1 ld*/,
                         int which /*0 near, 1 far, 2 all*/, double *sink) {
  __shared__ int s_rank, s_die;
  if (threadIdx.x == 0) {
    s_die = die_of_sm[smid()];
    s_rank = atomicAdd(&rank_ctr[s_die], 1);
  }
  __syncthreads();
  const int die = s_die, rank = s_rank;
  const int lst = which == 2 ? 2 : (which == 0 ? die : 1 - die);
  const int len = list_len[lst];
  const int *L = lists + (size_t)lst * 65536;
  const int nb = blocks_per_die[die];
  // all-chunks mode: split the whole list between all blocks by (die, rank)
  const int parts = which == 2 ? blocks_per_die[0] + blocks_per_die[1] : nb;
  const int part = which == 2 ? (die ? blocks_per_die[0] + rank : rank) : rank;
  const int lo = (int)((long long)len * part / parts), hi = (int)((long long)len * (part + 1) / parts);
  double acc = 0;
  for (int r = 0; r < reps; ++r)
#pragma unroll 8
    for (int q = lo; q < hi; ++q) {
      double2 *ch = buf + (size_t)L[q] * 128;  // 2 KB = 128 x 16 B
      for (int e = threadIdx.x; e < 128; e += blockDim.x) {
        if (mode == 0) {
          ch[e] = make_double2(r, q);
        } else {
          double2 v = __ldcg(ch + e);
          acc += v.x + v.y;
        }
      }
    }
  if (acc == 1.2345) sink[0] = acc;
}

int main() {
  int nsm;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0));
  const int nchunks = 32768;  // 64 MB: L2-resident
  char *buf;
  CK(cudaMalloc(&buf, (size_t)nchunks * 2048));
  CK(cudaMemset(buf, 0, (size_t)nchunks * 2048));
  unsigned *lat_sm, *lat_chunk;
  int *chunk_sm;
  CK(cudaMalloc(&lat_sm, 1024 * 4));
  CK(cudaMalloc(&lat_chunk, nchunks * 4));
  CK(cudaMalloc(&chunk_sm, nchunks * 4));
  CK(cudaMemset(lat_sm, 0, 1024 * 4));
  const int big = 150 * 1024;
  CK(cudaFuncSetAttribute(k_sm_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  CK(cudaFuncSetAttribute(k_chunk_lat, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  // 1. SM -> die, using a few probe chunks (a chunk is far for one die and near for the other)
  std::vector<int> die_of_sm(nsm, -1);
  std::vector<unsigned> h(1024);
  {
    k_sm_lat<<<nsm, 32, big>>>(buf, lat_sm);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), lat_sm, 1024 * 4, cudaMemcpyDeviceToHost));
    unsigned mn = ~0u, mx = 0;
    for (int s = 0; s < nsm; ++s) mn = std::min(mn, h[s]), mx = std::max(mx, h[s]);
    const unsigned thr = (mn + mx) / 2;
    int n0 = 0;
    for (int s = 0; s < nsm; ++s) {
      die_of_sm[s] = h[s] <= thr ? 0 : 1;
      n0 += die_of_sm[s] == 0;
    }
    printf("SM latency to chunk 0: min %u max %u -> %d SMs near (die 0), %d far (die 1)\n", mn, mx, n0, nsm - n0);
    printf("sm lat:");
    for (int s = 0; s < nsm; ++s) printf(" %u", h[s]);
    printf("\n");
  }
  // 2. chunk -> die: each block classifies chunks relative to its own SM's die
  k_chunk_lat<<<nsm, 32, big>>>(buf, nchunks, lat_chunk, chunk_sm);
  CK(cudaDeviceSynchronize());
  std::vector<unsigned> lc(nchunks);
  std::vector<int> cs(nchunks);
  CK(cudaMemcpy(lc.data(), lat_chunk, nchunks * 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(cs.data(), chunk_sm, nchunks * 4, cudaMemcpyDeviceToHost));
  std::vector<unsigned> sorted(lc);
  std::sort(sorted.begin(), sorted.end());
  printf("chunk latency percentiles: p5 %u p25 %u p50 %u p75 %u p95 %u\n", sorted[nchunks / 20], sorted[nchunks / 4],
         sorted[nchunks / 2], sorted[3 * nchunks / 4], sorted[19 * nchunks / 20]);
  const unsigned cthr = (sorted[nchunks / 10] + sorted[9 * nchunks / 10]) / 2;
  std::vector<int> lists(3 * 65536);
  int len[3] = {0, 0, 0};
  for (int c = 0; c < nchunks; ++c) {
    const int sdie = die_of_sm[cs[c]];
    const int cdie = lc[c] <= cthr ? sdie : 1 - sdie;
    lists[cdie * 65536 + len[cdie]++] = c;
    lists[2 * 65536 + len[2]++] = c;
  }
  printf("chunks: %d on die 0, %d on die 1 (threshold %u cycles)\n", len[0], len[1], cthr);
  // equalise the two die lists so near / far move the same bytes per block
  int *d_lists, *d_len, *d_die, *d_bpd, *d_rank;
  double *sink;
  CK(cudaMalloc(&d_lists, lists.size() * 4));
  CK(cudaMalloc(&d_len, 3 * 4));
  CK(cudaMalloc(&d_die, nsm * 4));
  CK(cudaMalloc(&d_bpd, 2 * 4));
  CK(cudaMalloc(&d_rank, 2 * 4));
  CK(cudaMalloc(&sink, 8));
  CK(cudaMemcpy(d_lists, lists.data(), lists.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_len, len, 3 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_die, die_of_sm.data(), nsm * 4, cudaMemcpyHostToDevice));
  int n0 = 0;
  for (int s = 0; s < nsm; ++s) n0 += die_of_sm[s] == 0;
  for (int bps : {2, 4}) {
    int bpd[2] = {bps * n0, bps * (nsm - n0)};
    CK(cudaMemcpy(d_bpd, bpd, 8, cudaMemcpyHostToDevice));
    const int smem = bps == 2 ? 100 * 1024 : 50 * 1024;
    CK(cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int mode = 0; mode < 2; ++mode)
      for (int which = 0; which < 3; ++which) {
        const int reps = 20;
        float best = 1e30f;
        for (int it = 0; it < 4; ++it) {
          CK(cudaMemset(d_rank, 0, 8));
          CK(cudaEventRecord(e0));
          k_stream<<<bps * nsm, 128, smem>>>((double2 *)buf, d_die, d_lists, d_len, d_bpd, d_rank, reps, mode, which,
                                             sink);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          float ms;
          CK(cudaEventElapsedTime(&ms, e0, e1));
          best = std::min(best, ms);
        }
        CK(cudaGetLastError());
        // bytes: near/far lists are per die; every die-d block covers its die's list once per rep
        double bytes;
        if (which == 2) bytes = (double)len[2] * 2048 * reps;
        else if (which == 0) bytes = ((double)len[0] + len[1]) * 2048 * reps;
        else bytes = ((double)len[1] + len[0]) * 2048 * reps;
        printf("%d blocks/SM %s %-4s: %.2f TB/s (%.3f ms)\n", bps, mode ? "load " : "store",
               which == 0 ? "near" : which == 1 ? "far" : "all", bytes / best / 1e9, best);
      }
  }
  return 0;
}
