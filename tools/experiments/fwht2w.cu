// MEASURED AND DROPPED (kept for the record; not built): warp-independent
// two-pass FWHT compress, b = 2^16.  To try it, add it to csrc/Makefile and
// dispatch to fwht2w_accumulate from fwht2p_accumulate (was: SMM_WID=1).
// cfg3: 85.7 ms with one item per (unit, block/slice, k-quad) and 257.7 ms with
// one warp looping over the 8 k-quads, against 43.2 ms for fwht2p — every warp
// then carries a whole item's serial latency chain (ticket, dependency, gather
// and Y round trips, fences) for 1/8 of the work; fwht2p's CTA items pay that
// chain once for 8 warps.  Results were correct (cfg3 bit-identical).
//
// Warp-independent two-pass FWHT compress (experimental; SMM_WID=1, b = 2^16).
// Reference: sketch.py:152-189, transforms.py:37-49 — same arithmetic as fwht2p.cu
// except the order in which the 32 inner indices of a k-tile are summed.
//
// fwht2p moves 8 warps through every item in lock step (five CTA barriers per
// item).  Here one warp owns a whole item: pass-1 item (unit, block, k-quad) —
// the 256 buckets of a block for 4 inner indices; pass-2 item (unit, slice,
// k-quad).  Lane = (g, kq): kq = lane & 3 picks the inner index 4q + kq, the
// lane group g = lane >> 2 is 3 bucket bits; a thread holds 32 buckets (5 bits).
// The 3-bit exchange goes through the warp's own 8 KB of shared memory under
// __syncwarp, and every warp pulls its own tickets, so the 16 warps of an SM
// progress independently.  Gathers stay sector-complete (4 lanes x 8 B per
// entry), Y keeps fwht2p's layout ([slot][op][bucket][32 k], a warp touching
// 32 B of each row).  The 8 k-quads of a k-tile meet in a staging area; the
// last to arrive folds them in quad order and extends the accumulator in
// k-tile order (counters), so results are deterministic.
#include <cstdlib>

#include "plan.cuh"
#include "twopass.cuh"

namespace smm {

__global__ void csr_count_kernel(SketchHashes h, int64_t n1, int64_t n2, int32_t *cnt, int64_t b);
__global__ void csr_scan_kernel(const int32_t *cnt, int32_t *off, int64_t b);
__global__ void csr_fill_kernel(SketchHashes h, int64_t n1, int64_t n2, const int32_t *off, int32_t *fill,
                                uint32_t *ent, int64_t nmax, int64_t b);
__global__ void csr_sort_kernel(const int32_t *off, uint32_t *ent, int64_t nmax, int64_t b, int rows);

namespace w2 {
using namespace tp;

constexpr int THREADS = 256;  // 8 independent warps per CTA, 2 CTAs per SM
constexpr int WARPS = THREADS / 32;
constexpr int KT = 32;        // unit = one k-tile of 32 inner indices
constexpr int NQ = 8;         // k-quads per k-tile
constexpr int WCELLS = 256 * 4;  // doubles of one warp's exchange area (8 KB)
constexpr int LB = 16;        // slice bits handled (b = 2^16, no fold)
constexpr int NBLK = 256;     // 256-bucket blocks / slices per unit
constexpr int G = NBLK;       // items per unit and pass (each covers the 8 k-quads)

struct Args {
  SketchHashes h;
  const double *X[2];  // k-minor operands
  int64_t ld[2];
  int64_t k0, K;
  int d, U, nslot, lag;
  FastDiv div_d, div_slot;
  const int32_t *off;
  const uint32_t *ent;
  int64_t nmax;
  double *Y;    // [nslot][2][2^16][KT]
  double *acc;  // [d][2^16]
  int *ctr;     // ticket | done1[U] | done2[U] | acc_cnt[d][NBLK]
  int acc_add;
};

// exchange-area cell of (bucket beta within the 256, inner index kq): bank-swizzled so
// that both access patterns below take the minimum two wavefronts per 256 B
__device__ __forceinline__ int cell(int beta, int kq) {
  return (((beta & ~31) | ((beta & 31) ^ ((beta >> 5) & 3))) << 2) | kq;
}

__device__ __forceinline__ void fwht_regs(double (&v)[32], int nbits) {
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    if (q < nbits) {
      const int h = 1 << q;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (!(j & h)) {
          const double x = v[j], y = v[j + h];
          v[j] = x + y;
          v[j + h] = x - y;
        }
    }
  }
}

// phase A (register j = bits 0-4, group g = bits 5-7) -> phase B (register bits 0-2 =
// bits 5-7, register bits 3-4 = bits 3-4, group g = bits 0-2), through the warp's area
__device__ __forceinline__ int beta_b(int r, int g) { return ((r & 7) << 5) | ((r >> 3) << 3) | g; }

__device__ __forceinline__ void exchange(double (&v)[32], double *W, int g, int kq) {
#pragma unroll
  for (int j = 0; j < 32; ++j) W[cell((g << 5) | j, kq)] = v[j];
  __syncwarp();
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = W[cell(beta_b(r, g), kq)];
  __syncwarp();  // the area is rewritten next
}

struct Item {
  int valid, is_p1, u, x;
};

__device__ __forceinline__ Item decode(const Args &p, int64_t pos, int64_t total) {
  // prologue: P1 of units 0..lag-1; then per g: [P1(g + lag) x G][P2(g) x G]
  Item it;
  it.valid = pos < total;
  const int pro = p.U < p.lag ? p.U : p.lag;
  if (pos < (int64_t)pro * G) {
    it.is_p1 = 1;
    it.u = (int)(pos / G);
    it.x = (int)(pos % G);
    return it;
  }
  const int64_t q = pos - (int64_t)pro * G;
  const int full = p.U > p.lag ? p.U - p.lag : 0;
  if (q < (int64_t)full * 2 * G) {
    const int g = (int)(q / (2 * G));
    const int r = (int)(q % (2 * G));
    if (r < G) {
      it.is_p1 = 1;
      it.u = g + p.lag;
      it.x = r;
    } else {
      it.is_p1 = 0;
      it.u = g;
      it.x = r - G;
    }
  } else {
    const int64_t q2 = q - (int64_t)full * 2 * G;
    it.is_p1 = 0;
    it.u = full + (int)(q2 / G);
    it.x = (int)(q2 % G);
  }
  return it;
}

__device__ __forceinline__ void spin_geq(const int *c, int target) {
  if (ld_acquire(c) >= target) return;
  while (ld_acquire(c) < target) __nanosleep(64);
}

// pass 1: block blk of unit (kappa, t), both operands, k-quad by k-quad -> Y
__device__ __forceinline__ void p1(const Args &p, int kappa, int t, int slot, int blk, double *W) {
  const int lane = threadIdx.x & 31, g = lane >> 2, kq = lane & 3;
  const uint64_t pol = policy_evict_last();
#pragma unroll 1
  for (int oq = 0; oq < 2 * NQ; ++oq) {
    const int op = oq / NQ, q = oq % NQ;
    const int64_t kk = (int64_t)kappa * KT + 4 * q + kq;
    const int64_t row = (int64_t)t * 2 + op;
    const int32_t *off = p.off + row * ((1 << LB) + 1) + (int64_t)blk * 256 + g * 32;
    const int e_lo = __ldg(off), e_hi = __ldg(off + 32);
    const uint32_t *ent = p.ent + row * p.nmax + e_lo;
    const int cnt = e_hi - e_lo;
    int cmax = cnt;
#pragma unroll
    for (int m = 4; m < 32; m <<= 1) cmax = max(cmax, __shfl_xor_sync(0xffffffffu, cmax, m));
    const char *Xb = (const char *)(p.X[op] + p.k0 + (kk < p.K ? kk : p.K - 1));
    const uint32_t ldb = (uint32_t)(p.ld[op] * 8);
    uint32_t mask = 0;
    int prevj = -1;
    for (int eb = 0; eb < cmax; eb += 8) {
      uint32_t es[8];
      double x[8];
#pragma unroll
      for (int s = 0; s < 8; ++s) es[s] = eb + s < cnt ? __ldg(ent + eb + s) : 0u;
#pragma unroll
      for (int s = 0; s < 8; ++s)
        x[s] = eb + s < cnt ? __ldg((const double *)(Xb + (uint64_t)(es[s] & 0x03ffffffu) * ldb)) : 0.0;
#pragma unroll
      for (int s = 0; s < 8; ++s) {
        if (eb + s < cnt) {
          const int j = (int)((es[s] >> 26) & 31u);
          const double val = (es[s] >> 31) ? -x[s] : x[s];
          double *c = W + cell((g << 5) | j, kq);
          *c = (j == prevj ? *c : 0.0) + val;  // first entry of a bucket stores (0 + val == val)
          mask |= 1u << j;
          prevj = j;
        }
      }
    }
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = ((mask >> j) & 1u) ? W[cell((g << 5) | j, kq)] : 0.0;
    if (kk >= p.K) {
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = 0.0;
    }
    fwht_regs(v, 5);  // bucket bits 0-4
    __syncwarp();     // every lane has read its cells before they are rewritten
    exchange(v, W, g, kq);
    fwht_regs(v, 3);  // bucket bits 5-7 (register bits 0-2)
    double *Yd = p.Y + (((int64_t)slot * 2 + op) << LB) * KT + (int64_t)blk * 256 * KT + 4 * q + kq;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int beta = beta_b(r, g);
      asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(Yd + (int64_t)beta * KT), "d"(v[r]), "l"(pol)
                   : "memory");
    }
  }
}

// pass 2: slice s of unit (kappa, t), k-quad by k-quad; the quads' sums over their 4
// inner indices are added in quad order, then the accumulator is extended in k-tile order
__device__ __forceinline__ void p2(const Args &p, int kappa, int t, int slot, int s, double *W, uint32_t tq,
                                   int *acc_cnt) {
  const int lane = threadIdx.x & 31, g = lane >> 2, kq = lane & 3;
  const uint64_t pol = policy_evict_first();
  const int rb = ((lane & 1) << 4) | (((lane >> 1) & 1) << 3);  // registers this lane keeps after the quad sum
  double tot[8];
#pragma unroll 1
  for (int q = 0; q < NQ; ++q) {
    double v[32];
#pragma unroll 1
    for (int op = 0; op < 2; ++op) {
      const double *Ys = p.Y + (((int64_t)slot * 2 + op) << LB) * KT + s * KT + 4 * q + kq;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int eta = (g << 5) | j;
        asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;"
                     : "=d"(v[j]) : "l"(Ys + (int64_t)eta * 256 * KT), "l"(pol) : "memory");
      }
      fwht_regs(v, 5);
      exchange(v, W, g, kq);
      fwht_regs(v, 3);
      if (op == 0) {
#pragma unroll
        for (int c = 0; c < 4; ++c) tmem_st8(tq + 16 * c, v + 8 * c);
        tmem_wait_st();
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double fa[8];
      tmem_ld8(tq + 16 * c, fa);
#pragma unroll
      for (int i = 0; i < 8; ++i) v[8 * c + i] = __dmul_rn(v[8 * c + i], fa[i]);
    }
    // sum over the quad's 4 inner indices (lane bits 0-1): lane keeps registers rb | i
    halve_step<1, 16>(v, lane);
    halve_step<2, 8>(v, lane);
#pragma unroll
    for (int i = 0; i < 8; ++i) tot[i] = q == 0 ? v[i] : tot[i] + v[i];
  }
  // every k-quad of this slice is done: drop its Y rows without write-back
  __syncwarp();
  for (int op = 0; op < 2; ++op) {
    const double *Ys = p.Y + (((int64_t)slot * 2 + op) << LB) * KT + s * KT;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double *rowp = Ys + (int64_t)(lane + 32 * i) * 256 * KT;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp) : "memory");
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp + 16) : "memory");
    }
  }
  if (lane == 0 && kappa > 0) spin_geq(acc_cnt, kappa);
  __syncwarp();
  double *a = p.acc + ((int64_t)t << LB) + s;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    double *ai = a + (int64_t)beta_b(rb | i, g) * 256;
    __stcg(ai, (kappa > 0 || p.acc_add) ? __ldcg(ai) + tot[i] : tot[i]);
  }
  __syncwarp();
  if (lane == 0) {
    fence_acq_rel();
    red_add(acc_cnt, 1);
  }
}

__global__ void __launch_bounds__(THREADS, 2) fwht2w_kernel(Args p) {
  extern __shared__ __align__(16) double smem[];
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 64);
  double *W = smem + warp * WCELLS;
  int *ticket = p.ctr;
  int *done1 = p.ctr + 1;             // [U]
  int *done2 = done1 + p.U;           // [U]
  int *acc_cnt = done2 + p.U;         // [d][NBLK]
  const int64_t total = (int64_t)p.U * 2 * G;
  int nxt = 0;
  if (lane == 0) nxt = atomicAdd(ticket, 1);
  while (true) {
    int pos = __shfl_sync(0xffffffffu, nxt, 0);
    const Item it = decode(p, pos, total);
    if (!it.valid) break;
    if (lane == 0) nxt = atomicAdd(ticket, 1);  // the next ticket lands while this item runs
    const int kappa = fdiv(it.u, p.div_d);
    const int t = it.u - kappa * p.d;
    const int slot = fmod_(it.u, p.div_slot);
    const int idx = it.x;
    if (lane == 0) {
      if (it.is_p1) {
        if (it.u >= p.nslot) spin_geq(done2 + (it.u - p.nslot), G);  // Y slot free
      } else {
        spin_geq(done1 + it.u, G);  // the unit's pass 1
      }
    }
    __syncwarp();
    if (it.is_p1) {
      p1(p, kappa, t, slot, idx, W);
      __syncwarp();
      if (lane == 0) {
        fence_acq_rel();
        red_add(done1 + it.u, 1);
      }
    } else {
      p2(p, kappa, t, slot, idx, W, tq, acc_cnt + t * NBLK + idx);
      __syncwarp();
      if (lane == 0) {
        fence_acq_rel();
        red_add(done2 + it.u, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(s_tmem));
}

static inline int64_t pad256(int64_t x) { return ((x + 255) / 256) * 256; }

static void ring(int64_t U, int &lag, int &nslot) {
  lag = 1;
  nslot = 3;  // 3 x 32 MB of Y in the 126 MB L2 (fwht2p's ring at b = 2^16)
  if (nslot > U + 1) nslot = (int)(U + 1 > 2 ? U + 1 : 2);
}

}  // namespace w2

bool fwht2w_enabled(int log2b) {
  static const bool on = getenv("SMM_WID") != nullptr;
  return on && log2b == w2::LB;
}

int64_t fwht2w_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K) {
  using namespace w2;
  (void)log2b;
  const int64_t b = (int64_t)1 << LB;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int64_t U = ((K + KT - 1) / KT) * d;
  int lag, nslot;
  ring(U, lag, nslot);
  int64_t w = 0;
  w += pad256((int64_t)d * 2 * (b + 1) * 4);
  w += pad256((int64_t)d * 2 * b * 4);
  w += pad256((int64_t)d * 2 * nmax * 4);
  w += pad256((int64_t)nslot * 2 * b * KT * 8);
  w += pad256((1 + 2 * U + (int64_t)d * NBLK) * 4);
  return w;
}

int fwht2w_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb,
                      int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws,
                      int64_t ws_bytes, cudaStream_t s) {
  using namespace w2;
  const int d = h.d;
  const int64_t b = (int64_t)1 << LB;
  const int64_t K = k1 - k0;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  if (ws_bytes < fwht2w_workspace(d, LB, n1, n2, K)) {
    set_error("compress workspace too small (warp-independent kernel)");
    return SMM_ERR_WORKSPACE;
  }
  if (K <= 0) {
    if (!acc_add) SMM_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)d * b * 8, s), "acc memset");
    return SMM_OK;
  }
  char *q = ws;
  int32_t *off = (int32_t *)q;
  q += pad256((int64_t)d * 2 * (b + 1) * 4);
  int32_t *cnt = (int32_t *)q;
  q += pad256((int64_t)d * 2 * b * 4);
  uint32_t *ent = (uint32_t *)q;
  q += pad256((int64_t)d * 2 * nmax * 4);
  const int64_t U = ((K + KT - 1) / KT) * d;
  int lag, nslot;
  ring(U, lag, nslot);
  double *Y = (double *)q;
  q += pad256((int64_t)nslot * 2 * b * KT * 8);
  int *ctr = (int *)q;
  const int64_t nctr = 1 + 2 * U + (int64_t)d * NBLK;
  // CSR plan: entries of each (t, op) sorted by (bucket, i)
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * b * 4, s), "csr memset");
  const int64_t nin = (int64_t)d * (n1 + n2);
  int64_t blocks = ceil_div(nin, 256);
  if (blocks > 8192) blocks = 8192;
  if (nin > 0) {
    csr_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, cnt, b);
    SMM_LAUNCH_CHECK("csr_count_kernel");
  }
  csr_scan_kernel<<<d * 2, 1024, 0, s>>>(cnt, off, b);
  SMM_LAUNCH_CHECK("csr_scan_kernel");
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * b * 4, s), "csr memset");
  if (nin > 0) {
    csr_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, off, cnt, ent, nmax, b);
    SMM_LAUNCH_CHECK("csr_fill_kernel");
    int64_t sb = ceil_div((int64_t)d * 2 * b, 256);
    if (sb > 8192) sb = 8192;
    csr_sort_kernel<<<(unsigned)sb, 256, 0, s>>>(off, ent, nmax, b, d * 2);
    SMM_LAUNCH_CHECK("csr_sort_kernel");
  }
  SMM_CUDA_TRY(cudaMemsetAsync(ctr, 0, (size_t)nctr * 4, s), "counter memset");
  Args p;
  p.h = h;
  p.X[0] = xa;
  p.X[1] = xb;
  p.ld[0] = lda;
  p.ld[1] = ldb;
  p.k0 = k0;
  p.K = K;
  p.d = d;
  p.U = (int)U;
  p.nslot = nslot;
  p.lag = lag;
  p.div_d = make_fastdiv((uint32_t)d);
  p.div_slot = make_fastdiv((uint32_t)nslot);
  p.off = off;
  p.ent = ent;
  p.nmax = nmax;
  p.Y = Y;
  p.acc = acc;
  p.ctr = ctr;
  p.acc_add = acc_add ? 1 : 0;
  const size_t smem = (size_t)WARPS * WCELLS * 8;
  SMM_CUDA_TRY(cudaFuncSetAttribute(fwht2w_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "fwht2w smem");
  KernelTimer timer(0, s);
  fwht2w_kernel<<<2 * num_sms(), THREADS, smem, s>>>(p);
  timer.stop();
  SMM_LAUNCH_CHECK("fwht2w_kernel");
  return SMM_OK;
}

}  // namespace smm
