// FWHT compress (steps 1-3) for 2^8 <= b <= 2^20: two-pass, persistent,
// dependency-ordered.  Reference: sketch.py:152-189, transforms.py:37-49.
//
// Why two passes.  A length-b FP64 transform does log2(b) adds per element;
// on B200 the FP64 pipe retires 64 adds/clk/SM while shared memory moves 16
// doubles/clk/SM, so every on-chip element exchange costs as much as ~8 FWHT
// stages and a random-access scatter costs ~3x more.  This kernel therefore
// (1) makes the scatter a *coalesced* pull: lanes carry 32 consecutive inner
// indices k, so each input element i contributes one 256-byte row segment
// X[i, k0:k0+32] of the k-minor operand (A row-major, B^T row-major), scattered
// into the warp's lane-private columns of the exchange area; (2) keeps 5 bucket
// bits in registers (free stages) and moves 3 more through ONE shared-memory
// exchange per pass (pass 1: 8 low bits, pass 2: up to 8 high bits); (3) parks
// the pass-1 result Y (2^LB x 32 doubles per repetition and operand) in the
// 126 MB L2 between the passes, in a (lag + 2)-slot ring; (4) keeps the first
// operand's pass-2 result in TMEM until the product, sums FA*FB over the 32
// lanes and adds it to the d x b accumulator once per k-tile.  b > 2^16 is
// folded into F = b / 2^16 slices (one sign per entry).
// Slices of 2^8..2^16 buckets use the *pair mapping* when the operands allow
// 16-byte rows (see "pair mapping" below): lanes own inner-index pairs, 4 + 4
// bucket bits per pass, bit-identical results with half the memory instructions.
//
// Scheduling: two persistent CTAs per SM pull tickets from a global counter in
// a fixed order [P1(0..lag-1)] [P1(lag) P2(0)] [P1(lag+1) P2(1)] ... where a
// unit u is (k-tile kappa, repetition t, fold slice a).  Every item's
// dependencies (P2(u) needs all P1(u); P1(u) reuses the Y slot of
// P2(u - nslot); P2(kappa, t, s) extends the accumulator after P2(kappa-1, t, s))
// are dispensed earlier, so spinning on them cannot deadlock; accumulator
// updates happen in k order, so results are bit-reproducible.
#include <cstdlib>

#include "plan.cuh"
#include "twopass.cuh"

namespace smm {

constexpr int P_THREADS = 256;
constexpr int KT = 32;
constexpr int P1_BITS = 8;
// P2(u) is dispensed `lag` groups after P1(u) (ring_plan(): 1 at b = 2^16, where 2 was
// measured slower; small transforms have few items per unit and need more units in flight)

// Optional phase profiler: thread 0 of every CTA accumulates clock64 deltas between
// marks, printed by the host after the launch.  Compiled in only with -DSMM_FWHT2P_PROFILE
// (tools/prof_phases.sh builds that variant) and then switched on by SMM_PROFILE=1: the
// runtime test of the marks alone cost the product kernel 2.7 % on cfg3 (40.66 vs 39.55 ms).
__shared__ long long s_prof[16];
__shared__ long long s_prof_last;
__device__ int g_prof_on;
#ifdef SMM_FWHT2P_PROFILE
#define PROF_MARK(k)                                 \
  do {                                               \
    if (g_prof_on && threadIdx.x == 0) {             \
      const long long _n = clock64();                \
      s_prof[k] += _n - s_prof_last;                 \
      s_prof_last = _n;                              \
    }                                                \
  } while (0)
#else
#define PROF_MARK(k) \
  do {               \
  } while (0)
#endif

// ------------------------------------------------------------------ CSR plan
// entries sorted by (bucket, i) per (t, op): off [d][2][b+1], ent [d][2][nmax] = i | sign << 31
__global__ void csr_count_kernel(SketchHashes h, int64_t n1, int64_t n2, int32_t *cnt, int64_t b) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const uint32_t m = eval_bucket(h.f[op][t], (uint64_t)i, h.log2b) & (uint32_t)(b - 1);  // bucket within slice
    atomicAdd(&cnt[((int64_t)t * 2 + op) * b + m], 1);
  }
}

// exclusive scan of one (t, op) row of bucket counts per 1024-thread block: chunks of 4096
// counts, each thread loading 4 consecutive ones as one int4 (coalesced across the block),
// a warp-shuffle scan and one block-wide combine per chunk, the running total carried
// across chunks (b >= 4096 is a multiple of 4096; smaller rows take the scalar tail)
__global__ void csr_scan_kernel(const int32_t *cnt, int32_t *off, int64_t b) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t s_carry;
  const int64_t row = blockIdx.x;  // (t, op)
  const int32_t *c = cnt + row * b;
  int32_t *o = off + row * (b + 1);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_carry = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < b; c0 += 4096) {
    const int64_t i0 = c0 + 4 * (int64_t)threadIdx.x;
    int32_t v[4] = {0, 0, 0, 0};
    if (i0 + 3 < b && (b & 3) == 0) {
      const int4 q = *reinterpret_cast<const int4 *>(c + i0);
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      for (int j = 0; j < 4; ++j) v[j] = i0 + j < b ? c[i0 + j] : 0;
    }
    const int32_t sum = v[0] + v[1] + v[2] + v[3];
    int32_t inc = sum;  // inclusive scan within the warp
#pragma unroll
    for (int dd = 1; dd < 32; dd <<= 1) {
      const int32_t y = __shfl_up_sync(0xffffffffu, inc, dd);
      if (lane >= dd) inc += y;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
      int32_t w = wsum[lane];
#pragma unroll
      for (int dd = 1; dd < 32; dd <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, w, dd);
        if (lane >= dd) w += y;
      }
      wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int32_t carry = s_carry;
    int32_t run = carry + inc - sum + (warp > 0 ? wsum[warp - 1] : 0);
    for (int j = 0; j < 4; ++j) {
      if (i0 + j < b) o[i0 + j] = run;
      run += v[j];
    }
    __syncthreads();  // every thread has read wsum and s_carry
    if (threadIdx.x == 0) s_carry = carry + wsum[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) o[b] = s_carry;
}

__global__ void csr_fill_kernel(SketchHashes h, int64_t n1, int64_t n2, const int32_t *off, int32_t *fill,
                                uint32_t *ent, int64_t nmax, int64_t b) {
  const int64_t per = n1 + n2;
  const int64_t total = (int64_t)h.d * per;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(x / per);
    const int64_t q = x % per;
    const int op = q < n1 ? 0 : 1;
    const int64_t i = op ? q - n1 : q;
    const int64_t row = (int64_t)t * 2 + op;
    const uint32_t m = eval_bucket(h.f[op][t], (uint64_t)i, h.log2b) & (uint32_t)(b - 1);  // bucket within slice
    const uint32_t sb = eval_signbit(h.f[2 + op][t], (uint64_t)i);
    const int32_t pos = off[row * (b + 1) + m] + atomicAdd(&fill[row * b + m], 1);
    // entry: i (26 bits) | bucket & 31 (5 bits) | sign (1 bit)
    ent[row * nmax + pos] = (uint32_t)i | ((m & 31u) << 26) | (sb << 31);
  }
}

// CSR heads for the pair mapping: per (t, op) and 16-bucket group, its range and first 16 entry
// words in one record, so that a pass-1 item's heads are independent loads that cp.async can
// stage in shared memory (fwht2p_kernel: "CSR heads")
__global__ void csr_heads_kernel(const int32_t *off, const uint32_t *ent, int64_t nmax, int64_t b, int rows,
                                 uint32_t *hw, int2 *hr) {
  const int64_t ng = b / 16;
  const int64_t total = (int64_t)rows * ng * 16;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(x & 15);
    const int64_t rg = x >> 4;
    const int64_t row = rg / ng, g = rg % ng;
    const int32_t *o = off + row * (b + 1) + g * 16;
    const int e_lo = o[0], e_hi = o[16];
    hw[x] = e_lo + j < e_hi ? ent[row * nmax + e_lo + j] : 0u;
    if (j == 0) hr[rg] = make_int2(e_lo, e_hi);
  }
}

// ------------------------------------------------------------------ kernel
// x / d for 0 <= x < 2^31 by multiply-high (the scheduler thread decodes an item
// on the critical path of every CTA barrier; 32-bit division costs ~20 instructions)
struct FastDiv {
  uint32_t m, d;
  int s;
};
static FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.s = 0;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (uint32_t)((((1ull << f.s) - d) << 32) / d + 1);
  return f;
}
__device__ __forceinline__ int fdiv(int x, const FastDiv &f) {
  return (int)((__umulhi((uint32_t)x, f.m) + (uint32_t)x) >> f.s);
}
__device__ __forceinline__ int fmod_(int x, const FastDiv &f) { return x - fdiv(x, f) * (int)f.d; }

struct TwoPassArgs {
  SketchHashes h;
  const double *X[2];  // k-minor operands: element (i, k) at X[op][i * ld[op] + k]
  int64_t ld[2];
  int64_t k0, K;
  int B, hb, d, nblk, ntiles, U, nslot;
  int F, LB, df;  // top-level fold: F = b / 2^LB slices of 2^LB buckets; df = d * F
  FastDiv div_df, div_F, div_slot;
  const int32_t *off;
  const uint32_t *ent;
  const uint32_t *hw;  // pair mapping: first 16 entry words of every 16-bucket group [d][2][bsz / 16][16]
  const int2 *hr;      // and the group's CSR range (e_lo, e_hi) [d][2][bsz / 16]
  int64_t nmax, bsz;
  double *Y;   // [nslot][2][b][KT]
  double *acc; // [d][b]
  int *ctr;    // [0] ticket | done1[U] | done2[U] | acc_cnt[d * F * nblk]
  long long *prof;  // [16] phase cycles (nullable)
  int acc_add;      // add to acc (continue an earlier call's k order) instead of overwriting it
  uint64_t pol_last, pol_first;  // L2 cache policies (l2_policies)
  int lag;          // pipeline depth in units (nslot = lag + 2)
  int acc_slow;     // test knob (SMM_ACC_SLOWPATH): every P2 item takes the accumulator slow path
};

__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---- TMEM helpers (32x32b shape: thread <-> TMEM lane, 16 x 32-bit columns = 8 doubles)
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const double *v) {
  uint32_t r[16];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    r[2 * q] = (uint32_t)__double2loint(v[q]);
    r[2 * q + 1] = (uint32_t)__double2hiint(v[q]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, double *v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int q = 0; q < 8; ++q) v[q] = __hiloint2double((int)r[2 * q + 1], (int)r[2 * q]);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// L2 cache-policy hints: Y (the pass-1 -> pass-2 intermediate) is written
// evict_last so it survives in L2 until pass 2, and read evict_first (last use);
// the policy operands come from the kernel parameters (TwoPassArgs::pol_*).
__device__ __forceinline__ void st_hint(double *p, double v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ double ld_hint(const double *p, uint64_t pol) {
  double v;
  asm volatile("ld.global.cg.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol) : "memory");
  return v;
}

// in-register butterflies over register-index bits [qlo, qhi)
__device__ __forceinline__ void reg_fwht32(double (&v)[32], int qlo, int qhi) {
#pragma unroll
  for (int q = 0; q < 5; ++q) {
    if (q >= qlo && q < qhi) {
      const int h = 1 << q;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (!(j & h)) {
          const double x = v[j], y = v[j + h];
          v[j] = x + y;
          v[j + h] = x - y;
        }
      }
    }
  }
}


// Pass 1: pull the 256 buckets [blk*256, blk*256+256) of operand op for the
// 32 inner indices of k-tile kappa, FWHT over the 8 low bucket bits, write Y.
// Warp w owns buckets blk*256 + w*32 + j (j = register index), lanes = k.
// CSR range of one warp's 32 buckets and its first 32 entry words (one per lane), fetched ahead of use
struct PullHead {
  int e_lo, e_hi;
  uint32_t first;
};

__device__ __forceinline__ PullHead pull_head(const TwoPassArgs &p, int t, int op, int blk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blk * 256 + warp * 32;
  const int64_t row = (int64_t)t * 2 + op;
  const int32_t *off = p.off + row * (p.bsz + 1);
  PullHead h;
  h.e_lo = __ldg(off + base);
  h.e_hi = __ldg(off + base + 32);
  h.first = h.e_lo + lane < h.e_hi ? __ldg(p.ent + row * p.nmax + h.e_lo + lane) : 0u;
  return h;
}

// first-batch gathers of an operand, issued ahead of its pull (lanes 0-7 of the head hold the entries)
__device__ __forceinline__ void gather_first(const TwoPassArgs &p, int kappa, int op, const PullHead &hd,
                                             double (&x)[8]) {
  const int64_t kk = (int64_t)kappa * KT + (threadIdx.x & 31);
  const char *Xb = (const char *)(p.X[op] + p.k0 + (kk < p.K ? kk : p.K - 1));
  const uint32_t ldb = (uint32_t)(p.ld[op] * 8);
  const int cnt = hd.e_hi - hd.e_lo;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const uint32_t e = __shfl_sync(0xffffffffu, hd.first, s);
    x[s] = s < cnt ? __ldg((const double *)(Xb + (uint64_t)(e & 0x03ffffffu) * ldb)) : 0.0;
  }
}

__device__ __forceinline__ void p1_operand(const TwoPassArgs &p, int kappa, int t, int a, int slot, int op, int blk,
                                           double *S, const PullHead &hd, double (&xpre)[8], bool have_pre,
                                           const PullHead *next) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // lanes past the end of the inner range read a valid element and are zeroed after the pull
  const int64_t kk = (int64_t)kappa * KT + lane;
  const bool full_tile = (int64_t)kappa * KT + KT <= p.K;  // warp-uniform
  // row address = base + i * (ld * 8): one 32x32->64-bit multiply-add per entry (ld < 2^28)
  const char *Xb = (const char *)(p.X[op] + p.k0 + (kk < p.K ? kk : p.K - 1));
  const uint32_t ldb = (uint32_t)(p.ld[op] * 8);
  const int64_t row = (int64_t)t * 2 + op;
  const uint32_t *ent = p.ent + row * p.nmax;
  const int e_lo = hd.e_lo;
  const int e_hi = hd.e_hi;
  // Scatter into this lane's column of the warp's rows of the exchange area
  // (S[(warp * 32 + j) * 32 + lane], lane-private: no barrier), not into registers:
  // a register target needs a data-dependent jump per entry, which measured ~7 ms
  // of instruction-fetch stalls on cfg3.  Entries are sorted by bucket, so the
  // first entry of a bucket stores and later ones add (CSR order, as before).
  double *col = S + warp * 1024 + lane;
  uint32_t mask = 0;  // buckets with an entry (warp-uniform)
  int prevj = -1;
  uint32_t win = hd.first;  // entry words [wbase, wbase + 32), one per lane
  int wbase = e_lo;
  for (int eb = e_lo; eb < e_hi; eb += 8) {
    if (eb - wbase == 32) {
      wbase = eb;
      win = eb + lane < e_hi ? __ldg(ent + eb + lane) : 0u;
    }
    uint32_t es[8];
    double x[8];
#pragma unroll
    for (int s = 0; s < 8; ++s) es[s] = __shfl_sync(0xffffffffu, win, (eb - wbase) + s);
    if (have_pre && eb == e_lo) {
#pragma unroll
      for (int s = 0; s < 8; ++s) x[s] = xpre[s];
    } else {
#pragma unroll
      for (int s = 0; s < 8; ++s)
        x[s] = eb + s < e_hi
                   ? __ldg((const double *)(Xb + (uint64_t)(es[s] & 0x03ffffffu) * ldb))
                   : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (eb + s < e_hi) {  // warp-uniform
        const int j = (int)((es[s] >> 26) & 31u);
        uint32_t neg = es[s] >> 31;
        if (p.F > 1)  // fold character of slice a: (-1)^popcount(a & (h(i) >> LB))
          neg ^= __popc((eval_bucket(p.h.f[op][t], (uint64_t)(es[s] & 0x03ffffffu), p.B) >> p.LB) & (uint32_t)a) & 1u;
        const double val = neg ? -x[s] : x[s];
        const double old = j == prevj ? col[j * 32] : 0.0;  // 0 + val == val, as the register path
        col[j * 32] = old + val;
        mask |= 1u << j;
        prevj = j;
      }
    }
  }
  double v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = ((mask >> j) & 1u) ? col[j * 32] : 0.0;
  if (!full_tile && kk >= p.K) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.0;
  }
  PROF_MARK(3);
  reg_fwht32(v, 0, 5);  // bucket bits 0-4
  // exchange: warp bits (bucket bits 5-7) <-> register bits 0-2
#pragma unroll
  for (int j = 0; j < 32; ++j) S[(warp * 32 + j) * 32 + lane] = v[j];
  PROF_MARK(4);
  __syncthreads();
  PROF_MARK(5);
#pragma unroll
  for (int r = 0; r < 32; ++r) v[r] = S[((r & 7) * 32 + (warp + 8 * (r >> 3))) * 32 + lane];
  reg_fwht32(v, 0, 3);  // bucket bits 5-7
  PROF_MARK(6);
  // the other operand's first gathers go out before this operand's 64 KB of Y stores
  if (next) gather_first(p, kappa, 1, *next, xpre);
  double *Yd = p.Y + (((int64_t)slot * 2 + op) * p.bsz + (int64_t)blk * 256) * KT + lane;
  const uint64_t pol = p.pol_last;
#pragma unroll
  for (int r = 0; r < 32; ++r) {
    const int bl = (warp + 8 * (r >> 3)) + 32 * (r & 7);
    st_hint(Yd + (int64_t)bl * KT, v[r], pol);
  }
  PROF_MARK(7);
}

__device__ __forceinline__ void p1_item(const TwoPassArgs &p, int kappa, int t, int a, int slot, int blk, double *S,
                                        const PullHead &hd1,
                                        const PullHead &hd0) {
  double xpre[8];
  p1_operand(p, kappa, t, a, slot, 0, blk, S, hd0, xpre, false, &hd1);
  __syncthreads();  // every warp has read operand 0's exchange data from S
  p1_operand(p, kappa, t, a, slot, 1, blk, S, hd1, xpre, true, nullptr);
}

// Pass 2: for slice s (256 buckets: every high-bit value x 2^(8-hb) low values)
// finish the transform of both operands over the hb high bits, multiply, sum
// over the 32 inner indices and extend the accumulator.  Slice bit sigma:
// registers <- sigma 0-4, warp <- sigma 5-7; bucket = hi * 256 + lo.
template <int HB>
__device__ __forceinline__ void p2_item(const TwoPassArgs &p, int kappa, int t, int a_sl, int slot, int s, uint32_t tmem,
                                        const int *acc_flag, int acc_ready, double *S) {
  acc_ready |= kappa == 0;  // k-tile 0 adds to a previous launch's accumulator (stream order)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // acc_ready (block-uniform): the scheduler already acquired the slice's counter, i.e. the
  // accumulator holds k-tiles < kappa; otherwise the update waits at the end (slow path)
  const int wq = warp & 3, wh = warp >> 2;
  constexpr int hb = HB;
  const int hmask = (1 << hb) - 1;
  const int64_t lo0 = (int64_t)s << (P1_BITS - hb);
  // this lane's accumulator bucket after the lane reduction (fixed by the mapping)
  const int rl = tp::lane_sum32_reg(lane);
  const int sg_acc = hb > 5 ? ((rl & 3) | (warp << 2) | ((rl >> 2) << 5)) : (rl | (warp << 5));
  double *a = p.acc + ((int64_t)t * p.F + a_sl) * p.bsz + (int64_t)(sg_acc & hmask) * 256 + lo0 + (sg_acc >> hb);
  // usually the previous k-tile's update of this slice finished long ago: fetch the old value early
  const double acc_old = ((kappa > 0 || p.acc_add) && acc_ready) ? __ldcg(a) : 0.0;
  const uint32_t tq = tmem + ((uint32_t)(32 * wq) << 16);
  const uint32_t col_fa = (uint32_t)(wh * 64);
  double v[32];
  const uint64_t pol = p.pol_first;
  if constexpr (HB > 5) {
    // Operand 0 goes through the shared-memory exchange and into TMEM in chunks of
    // 8 registers, so operand 1's 32 row loads can already fly during that half.
    const double *Y0 = p.Y + ((int64_t)slot * 2 + 0) * p.bsz * KT + lane;
    const double *Y1 = p.Y + ((int64_t)slot * 2 + 1) * p.bsz * KT + lane;
    auto load = [&](const double *Ys) {
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        const int sg = r | (warp << 5);
        v[r] = ld_hint(Ys + ((int64_t)(sg & hmask) * 256 + lo0 + (sg >> hb)) * KT, pol);
      }
    };
    auto discard = [&](const double *Ys) {  // last use of these Y rows: drop them without write-back
      __syncwarp();
      const int sg = lane | (warp << 5);
      const double *row = Ys - lane + ((int64_t)(sg & hmask) * 256 + lo0 + (sg >> hb)) * KT;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(row) : "memory");
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + 16) : "memory");
    };
    load(Y0);
    PROF_MARK(8);
    reg_fwht32(v, 0, 5);
    discard(Y0);
    // exchange: warp bits (sigma 5-7) <-> register bits 2-4
#pragma unroll
    for (int r = 0; r < 32; ++r) S[(warp * 32 + r) * 32 + lane] = v[r];
    load(Y1);
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // registers c + 4 j: the remaining stages run over register bits 2-4 = j bits 0-2
      double f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int r = c + 4 * j;
        f[j] = S[((r >> 2) * 32 + ((r & 3) | (warp << 2))) * 32 + lane];
      }
#pragma unroll
      for (int q = 0; q < hb - 5; ++q) {
        const int h = 1 << q;
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (!(j & h)) {
            const double x = f[j], y = f[j + h];
            f[j] = x + y;
            f[j + h] = x - y;
          }
      }
      tmem_st8(tq + col_fa + 16 * c, f);
    }
    tmem_wait_st();
    __syncthreads();  // S is reused by operand 1's exchange
    reg_fwht32(v, 0, 5);
    discard(Y1);
#pragma unroll
    for (int r = 0; r < 32; ++r) S[(warp * 32 + r) * 32 + lane] = v[r];
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 32; ++r) v[r] = S[((r >> 2) * 32 + ((r & 3) | (warp << 2))) * 32 + lane];
    reg_fwht32(v, 2, 2 + (hb - 5));
    PROF_MARK(9);
    // product FA * FB: TMEM chunk c holds FA of registers c + 4 j
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double fa[8];
      tmem_ld8(tq + col_fa + 16 * c, fa);
#pragma unroll
      for (int j = 0; j < 8; ++j) v[c + 4 * j] = __dmul_rn(v[c + 4 * j], fa[j]);
    }
  } else {
#pragma unroll 1
  for (int op = 0; op < 2; ++op) {
    const double *Ys = p.Y + ((int64_t)slot * 2 + op) * p.bsz * KT + lane;
#pragma unroll
    for (int r = 0; r < 32; ++r) {
      const int sg = r | (warp << 5);
      const int64_t bucket = (int64_t)(sg & hmask) * 256 + lo0 + (sg >> hb);
      v[r] = ld_hint(Ys + bucket * KT, pol);
    }
    PROF_MARK(8);
    reg_fwht32(v, 0, hb < 5 ? hb : 5);
    // last use of these Y rows: drop the L2 lines without write-back
    __syncwarp();
    {
      const int sg = lane | (warp << 5);
      const double *row = Ys - lane + ((int64_t)(sg & hmask) * 256 + lo0 + (sg >> hb)) * KT;
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(row) : "memory");
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + 16) : "memory");
    }
    if (hb > 5) {
      // shared-memory exchange: warp bits (sigma 5-7) <-> register bits 2-4
#pragma unroll
      for (int r = 0; r < 32; ++r) S[(warp * 32 + r) * 32 + lane] = v[r];
      __syncthreads();
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = S[((r >> 2) * 32 + ((r & 3) | (warp << 2))) * 32 + lane];
      reg_fwht32(v, 2, 2 + (hb - 5));
      __syncthreads();  // S is reused by the next exchange
    }
    if (op == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st8(tq + col_fa + 16 * c, v + 8 * c);
      tmem_wait_st();
    }
  }
  PROF_MARK(9);
  // product FA * FB (FB in v)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double fa[8];
    tmem_ld8(tq + col_fa + 16 * c, fa);
#pragma unroll
    for (int q = 0; q < 8; ++q) v[8 * c + q] = __dmul_rn(v[8 * c + q], fa[q]);
  }
  }
  // sum over the 32 inner indices (lanes): lane l ends with register l summed over all lanes
  const double sum = tp::lane_sum32(v, lane);
  if (kappa == 0) {
    // accumulate mode continues a previous call's k order exactly (chunk boundaries are k-tiles)
    __stcg(a, p.acc_add ? acc_old + sum : sum);
  } else if (acc_ready) {
    __stcg(a, acc_old + sum);
  } else {
    // slow path: lane 0 acquires the counter, __syncwarp orders the warp's loads after it
    // (a CTA barrier here measured 15 % slower on cfg3)
    if (lane == 0)
      while (ld_acquire(acc_flag) < kappa) __nanosleep(32);
    __syncwarp();
    __stcg(a, __ldcg(a) + sum);
  }
}

// ------------------------------------------------------------------ pair mapping
// Used when both operands allow 16-byte accesses (even row stride, even k origin
// and inner range, 16-byte aligned base) and the slice is 2^16 wide (hb = 8).
// Lane = (lb, kp): kp = lane & 15 owns the inner-index pair (2 kp, 2 kp + 1) of
// the k-tile as one double2, lb = lane >> 4 is one bucket bit; a thread holds
// 16 buckets x 2 inner indices.  Against the one-k-per-lane mapping above this
// halves the global and shared-memory instructions (every gather, Y store, Y
// load and exchange access moves 16 bytes), and the sum over the 32 inner
// indices starts with the in-thread pair, so the lane reduction has 4 halving
// steps instead of 5.  Bucket bits of a 256-bucket block / slice:
//   phase A: register j = bits 0-3, lb = bit 4, warp = bits 5-7
//   phase B (after the one shared-memory exchange): warp = bits 0-2,
//            lb = bit 3, register j = bits 4-7
// Exchange cell of (beta, kp): S2[beta * 16 + kp] (64 KB, as before).
#ifndef SMM_PGB
#define SMM_PGB 6
#endif
constexpr int PGB = SMM_PGB;  // gather batch (entries per half-warp in flight)
__device__ __forceinline__ double2 ldg_pair(const char *p) { return __ldg((const double2 *)p); }

__device__ __forceinline__ double2 d2_add(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 d2_sub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

__device__ __forceinline__ void reg_fwht16x2(double2 (&v)[16], int nq = 4) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q >= nq) break;
    const int h = 1 << q;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (!(j & h)) {
        const double2 x = v[j], y = v[j + h];
        v[j] = d2_add(x, y);
        v[j + h] = d2_sub(x, y);
      }
  }
}

// CSR range of this lane's half-warp (16 buckets) and its first 16 entry words (one per kp)
__device__ __forceinline__ PullHead pull_head2(const TwoPassArgs &p, int t, int op, int blk) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t base = (int64_t)blk * 256 + warp * 32 + (lane & 16);
  const int64_t row = (int64_t)t * 2 + op;
  const int32_t *off = p.off + row * (p.bsz + 1);
  PullHead h;
  h.e_lo = __ldg(off + base);
  h.e_hi = __ldg(off + base + 16);
  h.first = h.e_lo + (lane & 15) < h.e_hi ? __ldg(p.ent + row * p.nmax + h.e_lo + (lane & 15)) : 0u;
  return h;
}

__device__ __forceinline__ const char *pair_row_base(const TwoPassArgs &p, int kappa, int op) {
  const int64_t kk = (int64_t)kappa * KT + 2 * (threadIdx.x & 15);
  return (const char *)(p.X[op] + p.k0 + (kk < p.K ? kk : p.K - 2));  // K even in pair mode
}

__device__ __forceinline__ void gather_first2(const TwoPassArgs &p, int kappa, int op, const PullHead &hd,
                                              double2 (&x)[PGB]) {
  const char *Xb = pair_row_base(p, kappa, op);
  const uint32_t ldb = (uint32_t)(p.ld[op] * 8);
  const int cnt = hd.e_hi - hd.e_lo;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 0; s < PGB; ++s) {
    const uint32_t e = __shfl_sync(0xffffffffu, hd.first, (lane & 16) | s);
    x[s] = s < cnt ? ldg_pair(Xb + (uint64_t)(e & 0x03ffffffu) * ldb) : make_double2(0.0, 0.0);
  }
}

template <bool FOLD>
__device__ __forceinline__ void p1_operand2(const TwoPassArgs &p, int kappa, int t, int a, int slot, int op, int blk,
                                            double2 *S, const PullHead &hd, double2 (&xpre)[PGB], bool have_pre,
                                            const PullHead *next) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kp = lane & 15, lb = lane >> 4;
  const int64_t kk = (int64_t)kappa * KT + 2 * kp;
  const bool full_tile = (int64_t)kappa * KT + KT <= p.K;  // warp-uniform
  const char *Xb = pair_row_base(p, kappa, op);
  const uint32_t ldb = (uint32_t)(p.ld[op] * 8);
  const int64_t row = (int64_t)t * 2 + op;
  const uint32_t *ent = p.ent + row * p.nmax + hd.e_lo;
  const int cnt = hd.e_hi - hd.e_lo;
  const int cnt_o = __shfl_xor_sync(0xffffffffu, cnt, 16);
  const int cmax = cnt > cnt_o ? cnt : cnt_o;
  // this lane's cells: beta = j | lb << 4 | warp << 5, j = 0..15 (lane-private: no barrier)
  double2 *col = S + (warp * 32 + lb * 16) * 16 + kp;
  uint32_t mask = 0;
  int prevj = -1;
  uint32_t win = hd.first;  // entry words [wbase, wbase + 16) of this half, one per kp
  int wbase = 0;
  for (int eb = 0; eb < cmax; eb += PGB) {
    if (eb - wbase + PGB > 16) {  // window exhausted (16 % PGB == 0, or refetch early)
      wbase = eb;
      win = eb + kp < cnt ? __ldg(ent + eb + kp) : 0u;
    }
    uint32_t es[PGB];
    double2 x[PGB];
#pragma unroll
    for (int s = 0; s < PGB; ++s) es[s] = __shfl_sync(0xffffffffu, win, (lane & 16) | ((eb - wbase) + s));
    if (have_pre && eb == 0) {
#pragma unroll
      for (int s = 0; s < PGB; ++s) x[s] = xpre[s];
    } else {
#pragma unroll
      for (int s = 0; s < PGB; ++s)
        x[s] = eb + s < cnt ? ldg_pair(Xb + (uint64_t)(es[s] & 0x03ffffffu) * ldb) : make_double2(0.0, 0.0);
    }
#pragma unroll
    for (int s = 0; s < PGB; ++s) {
      if (eb + s < cnt) {
        const int j = (int)((es[s] >> 26) & 15u);
        uint32_t neg = es[s] >> 31;
        if (FOLD)  // fold character of slice a: (-1)^popcount(a & (h(i) >> LB))
          neg ^= __popc((eval_bucket(p.h.f[op][t], (uint64_t)(es[s] & 0x03ffffffu), p.B) >> p.LB) & (uint32_t)a) & 1u;
        const double2 val = neg ? make_double2(-x[s].x, -x[s].y) : x[s];
        const double2 old = j == prevj ? col[j * 16] : make_double2(0.0, 0.0);  // 0 + val == val
        col[j * 16] = d2_add(old, val);
        mask |= 1u << j;
        prevj = j;
      }
    }
  }
  double2 v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = ((mask >> j) & 1u) ? col[j * 16] : make_double2(0.0, 0.0);
  if (!full_tile && kk >= p.K) {
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = make_double2(0.0, 0.0);
  }
  PROF_MARK(3);
  reg_fwht16x2(v);  // bucket bits 0-3
#pragma unroll
  for (int j = 0; j < 16; ++j) col[j * 16] = v[j];
  PROF_MARK(4);
  __syncthreads();
  PROF_MARK(5);
  // phase B: beta = warp | lb << 3 | j << 4
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = S[((warp | (lb << 3) | (j << 4)) * 16) + kp];
  reg_fwht16x2(v);  // bucket bits 4-7
  PROF_MARK(6);
  if (next) gather_first2(p, kappa, 1, *next, xpre);
  double *Yd = p.Y + (((int64_t)slot * 2 + op) * p.bsz + (int64_t)blk * 256) * KT + 2 * kp;
  const uint64_t pol = p.pol_last;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int beta = warp | (lb << 3) | (j << 4);
    tp::st2_hint(Yd + (int64_t)beta * KT, v[j].x, v[j].y, pol);
  }
  PROF_MARK(7);
}

template <bool FOLD>
__device__ __forceinline__ void p1_item2(const TwoPassArgs &p, int kappa, int t, int a, int slot, int blk, double2 *S,
                                         const PullHead &hd1, const PullHead &hd0) {
  double2 xpre[PGB];
  p1_operand2<FOLD>(p, kappa, t, a, slot, 0, blk, S, hd0, xpre, false, &hd1);
  __syncthreads();  // every warp has read operand 0's exchange data from S
  p1_operand2<FOLD>(p, kappa, t, a, slot, 1, blk, S, hd1, xpre, true, nullptr);
}

// Pass 2 of slice s, pair mapping: slice position pi (8 bits) is bucket
// (pi & hmask) * 256 + lo0 + (pi >> hb); the hb low bits of pi are transformed
// (phase A bits 0..min(hb, 4)-1, phase B bits 4..hb-1; at hb <= 4 the exchange only
// permutes, which still measured 11 % faster than the one-k-per-lane mapping at hb = 4).
template <int HB>
__device__ __forceinline__ void p2_item2(const TwoPassArgs &p, int kappa, int t, int a_sl, int slot, int s,
                                         uint32_t tmem, const int *acc_flag, int acc_ready, double2 *S) {
  acc_ready |= kappa == 0;  // k-tile 0 adds to a previous launch's accumulator (stream order)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kp = lane & 15, lb = lane >> 4;
  // after the lane reduction lane (lb, kp) of warp w holds eta = w | lb << 3 | kp << 4
  constexpr int hmask = (1 << HB) - 1;
  const int64_t lo0 = (int64_t)s << (P1_BITS - HB);
  auto row_of = [&](int pi) { return (int64_t)(pi & hmask) * 256 + lo0 + (pi >> HB); };
  double *a = p.acc + ((int64_t)t * p.F + a_sl) * p.bsz + row_of(warp | (lb << 3) | (kp << 4));
  const double acc_old = ((kappa > 0 || p.acc_add) && acc_ready) ? __ldcg(a) : 0.0;
  const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t col_fa = (uint32_t)((warp >> 2) * 64);
  const uint64_t pol = p.pol_first;
  double2 *cell = S + (warp * 32 + lb * 16) * 16 + kp;  // phase-A cells of this lane (j * 16 apart)
  double2 v[16];
  // Narrower slices (hb < 8) issue operand 1's row loads before the "exchange area free" barrier
  // of operand 0, so that they fly while the CTA meets there (operand loop unrolled; cfg5
  // b = 2^14 5.18 -> 4.95 ms).  At hb = 8 the same costs 24 bytes of spills and 2 % (36.2 vs
  // 35.5 ms on cfg3): full slices load at the top of each operand's turn.
  constexpr bool EARLY_Y1 = HB < 8;
  const double *Yb = p.Y + ((int64_t)slot * 2) * p.bsz * KT + 2 * kp;
  if constexpr (EARLY_Y1) {
#pragma unroll
    for (int j = 0; j < 16; ++j) tp::ld2_hint(Yb + row_of(j | (lb << 4) | (warp << 5)) * KT, v[j].x, v[j].y, pol);
  }
#pragma unroll(EARLY_Y1 ? 2 : 1)
  for (int op = 0; op < 2; ++op) {
    const double *Ys = Yb + (int64_t)op * p.bsz * KT;
    if constexpr (!EARLY_Y1) {
#pragma unroll
      for (int j = 0; j < 16; ++j) tp::ld2_hint(Ys + row_of(j | (lb << 4) | (warp << 5)) * KT, v[j].x, v[j].y, pol);
    }
    PROF_MARK(8);
    reg_fwht16x2(v, HB < 4 ? HB : 4);  // pi bits 0..min(hb, 4)-1
    // Last use of these Y rows (all read by this warp): drop the L2 lines without write-back.
    // Where the discard is issued matters: ptxas is free to move it right behind the loads
    // (the PTX carries no dependency on their data), and a discard that reaches L2 while the
    // rows are still being read measured 18 % slower on cfg3 (46.8 vs 39.5 ms); at the end of
    // the item it is 2.3 % slower (the dirty lines live longer and are written back).  Full
    // slices (hb = 8) issue it behind the exchange barrier, which no load of the rows can
    // cross (cfg3 -0.5 %, cfg4 / b = 2^18..2^20 -1 %), and so do the narrowest ones (hb <= 2:
    // hardly any butterflies stand between their loads and the discard; b = 2^10 -4 %); the
    // others keep it before the barrier (b = 2^14: 2.9 % faster there).
    // profiles/r02_ab_discard_placement.txt
    constexpr bool LATE_DISCARD = HB >= 8 || HB <= 2;
    const double *rowp = Ys - 2 * kp + row_of(lane | (warp << 5)) * KT;
    if constexpr (!LATE_DISCARD) {
      __syncwarp();
      // predicated on the phase-A results, so that ptxas cannot hoist it to the loads (the bit
      // pattern is a NaN payload no transform produces; a skipped discard would cost nothing)
      if (__double2hiint(v[0].x) != 0x7ff8dead) asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp) : "memory");
      if (__double2hiint(v[15].y) != 0x7ff8dead)
        asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp + 16) : "memory");
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) cell[j * 16] = v[j];
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = S[((warp | (lb << 3) | (j << 4)) * 16) + kp];
    if constexpr (LATE_DISCARD) {
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp) : "memory");
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(rowp + 16) : "memory");
    }
    reg_fwht16x2(v, HB - 4);  // pi bits 4..hb-1
    if (op == 0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_st8(tq + col_fa + 16 * c, (const double *)(v + 4 * c));
      tmem_wait_st();
      if constexpr (EARLY_Y1) {  // operand 1's rows fly while the CTA meets at the barrier
        const double *Y1 = Yb + p.bsz * KT;
#pragma unroll
        for (int j = 0; j < 16; ++j) tp::ld2_hint(Y1 + row_of(j | (lb << 4) | (warp << 5)) * KT, v[j].x, v[j].y, pol);
      }
      __syncthreads();  // S is reused by operand 1's exchange (the next item's waits for [B])
    }
  }
  PROF_MARK(9);
  // product FA * FB, summed over the thread's inner-index pair
  double pr[16];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    double fa[8];
    tmem_ld8(tq + col_fa + 16 * c, fa);
#pragma unroll
    for (int q = 0; q < 4; ++q)  // products rounded, then the pair sum: the first node of lane_sum32's tree
      pr[4 * c + q] = __dadd_rn(__dmul_rn(v[4 * c + q].x, fa[2 * q]), __dmul_rn(v[4 * c + q].y, fa[2 * q + 1]));
  }
  // sum over the 16 pairs (lane bits 3..0 = inner-index bits 4..1): lane kp ends with register kp
  tp::halve_step<8, 8>(pr, lane);
  tp::halve_step<4, 4>(pr, lane);
  tp::halve_step<2, 2>(pr, lane);
  tp::halve_step<1, 1>(pr, lane);
  const double sum = pr[0];
  if (kappa == 0) {
    __stcg(a, p.acc_add ? acc_old + sum : sum);
  } else if (acc_ready) {
    __stcg(a, acc_old + sum);
  } else {
    // slow path: lane 0 acquires the counter, __syncwarp orders the warp's loads after it
    // (a CTA barrier here measured 15 % slower on cfg3)
    if (lane == 0)
      while (ld_acquire(acc_flag) < kappa) __nanosleep(32);
    __syncwarp();
    __stcg(a, __ldcg(a) + sum);
  }
}

struct Item {
  int64_t pos;
  int is_p1, u, idx;
};

__device__ __forceinline__ Item decode_item(const TwoPassArgs &p, int64_t pos, int log2g) {
  // prologue: P1 of units 0..LAG-1; then groups g = 0..U-1: [P1(g+LAG) x nblk][P2(g) x nblk]
  // (the P1 part is absent once g+LAG >= U).  2*nblk is a power of two.
  const int G1 = p.nblk;  // = 2^(log2g - 1)
  const int pro_units = p.U < p.lag ? p.U : p.lag;
  Item it;
  it.pos = pos;
  if (pos < (int64_t)pro_units * G1) {
    it.is_p1 = 1; it.u = (int)(pos >> (log2g - 1)); it.idx = (int)(pos & (G1 - 1));
    return it;
  }
  const int q = (int)(pos - (int64_t)pro_units * G1);
  const int full = p.U > p.lag ? p.U - p.lag : 0;
  const int regular = full << log2g;
  if (q < regular) {
    const int g = q >> log2g;
    const int r = q & ((1 << log2g) - 1);
    if (r < G1) { it.is_p1 = 1; it.u = g + p.lag; it.idx = r; }
    else { it.is_p1 = 0; it.u = g; it.idx = r - G1; }
  } else {
    const int q2 = q - regular;
    it.is_p1 = 0; it.u = full + (q2 >> (log2g - 1)); it.idx = q2 & (G1 - 1);
  }
  return it;
}

// threadIdx.x read afresh (ptxas keeps the kernel-entry copy in a register it spills; the reload
// from local memory missed L1 behind the gather stream: 3 % of all warp samples on cfg3)
__device__ __forceinline__ int tid_now() {
  int t;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(t));
  return t;
}

__device__ __forceinline__ void red_add(int *ptr, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}

// FOLD (pair mapping only): b > 2^16, every entry carries its slice's fold character
template <int HB, bool PAIR, bool FOLD = false>
__global__ void __launch_bounds__(P_THREADS, 2) fwht2p_kernel(TwoPassArgs p) {
  extern __shared__ __align__(16) double S[];  // 8 warps x 32 x 32 doubles = 64 KB
  __shared__ uint32_t s_tmem;
  __shared__ int s_item[12];
  // CSR heads of the next pass-1 item (SMEM_HEADS below), staged by cp.async while the current
  // item computes: no register holds them across the item and no warp waits for their loads
  __shared__ __align__(16) uint32_t s_hw[2][2][256];
  __shared__ __align__(16) int2 s_hr[2][2][16];
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid < 16) s_prof[tid] = 0;
  if (tid == 0) s_prof_last = clock64();
  int *ticket = p.ctr;
  int *done1 = p.ctr + 1;
  int *done2 = done1 + p.U;
  int *acc_cnt = done2 + p.U;  // P2 completions per accumulator slice (t, a, s): k-tiles done
  const int G1 = p.nblk, G2 = p.nblk;  // P1 items: one block, both operands; P2 items: one slice
  const int log2g = 31 - __clz(2 * p.nblk);
  const int64_t total = (int64_t)p.U * (G1 + G2);
  // Scheduling (thread 0) runs one item ahead: the ticket after next is claimed
  // while the current item computes, and every warp prefetches the CSR heads of
  // the next pass-1 item.  Dependencies (thread 0): right before the closing
  // barrier [B] of item i it issues RELAXED loads of the counters that item i+1
  // depends on (P1(u): every P2 of unit u - nslot, whose Y slot it reuses; P2(u):
  // every P1 of unit u, and the slice's accumulator counter, i.e. the previous
  // k-tile's P2 of the same accumulator rows).  After [B] a fence.acquire turns
  // those loads into acquires (PTX acquire pattern: relaxed read, then fence; it
  // does not wait for outstanding stores); a counter not yet complete is polled
  // with ld.acquire.  Barrier [A] then extends the order to the CTA, so every Y /
  // accumulator read of item i+1 happens after its producers' writes.  Item i is
  // published by thread 32 after [B] (fence.release, then the completion adds):
  // the release waits for the item's Y / accumulator stores to drain, so warp 1
  // joins [A] through a barrier of its own with warp 0 and the other six warps
  // start item i+1 meanwhile.  Every dependency was dispensed before the item that
  // waits on it and a publish never waits for anything but its own stores, so
  // waiting cannot deadlock.  Scheduler state lives in shared memory (as
  // registers it would cost every thread ~14 of its 128).
  __shared__ int64_t sh_nxt;
  __shared__ Item sh_itn;
  __shared__ int sh_ver[2];  // highest unit whose completion thread 0 acquired: done1 (P2), done2 (P1)
  __shared__ int s_acc_ok;   // the next P2 item's accumulator counter was acquired complete
  __shared__ int sh_prev_next;  // the previous descriptor's next_p1 (thread 0)
  int64_t &nxt = sh_nxt;
  Item &itn = sh_itn;
  struct Deps {
    const int *ptr[2];
    int tgt[2], val[2];
    int ver[2];
  };
  __shared__ Deps sD;
  auto deps_of = [&](const Item &it, Deps &D) {
    D.ptr[0] = D.ptr[1] = nullptr;
    D.tgt[0] = D.tgt[1] = D.val[0] = D.val[1] = 0;
    D.ver[0] = sh_ver[0];
    D.ver[1] = sh_ver[1];
    if (it.pos >= total) return;
    if (it.is_p1) {
      const int need = it.u - p.nslot;
      if (need > sh_ver[1]) { D.ptr[0] = done2 + need; D.tgt[0] = G2; D.ver[1] = need; }
    } else {
      if (it.u > sh_ver[0]) { D.ptr[0] = done1 + it.u; D.tgt[0] = G1; D.ver[0] = it.u; }
      const int kap = fdiv(it.u, p.div_df);
      if (kap > 0) {
        const int ut = fmod_(it.u, p.div_df);
        D.ptr[1] = acc_cnt + (fdiv(ut, p.div_F) * p.F + fmod_(ut, p.div_F)) * p.nblk + it.idx;
        D.tgt[1] = kap;
      }
    }
  };
  // after the acquire fence (or none): poll the must-precede dependency if incomplete; the
  // accumulator counter is only recorded — if incomplete the P2 item waits for it at its end
  auto deps_settle = [&](Deps &D) {
    if (D.ptr[0] && D.val[0] < D.tgt[0]) {
#ifdef SMM_FWHT2P_PROFILE
      const long long w0 = g_prof_on ? clock64() : 0;
#endif
      while (ld_acquire(D.ptr[0]) < D.tgt[0]) __nanosleep(32);
#ifdef SMM_FWHT2P_PROFILE
      if (g_prof_on) s_prof[11] += clock64() - w0;  // informational
#endif
    }
    sh_ver[0] = D.ver[0];
    sh_ver[1] = D.ver[1];
    s_acc_ok = (!D.ptr[1] || D.val[1] >= D.tgt[1]) ? 1 : 0;
  };
  // item descriptor (thread 0): item `it` (= itn) and the prefetch hint of its successor, decoded
  // from the ticket claimed one item earlier.  Written before [B] of the previous item: every warp
  // read the previous descriptor at that item's start, at least one CTA barrier ago.
  auto describe = [&]() {
    const Item it = itn;
    const Item in = decode_item(p, nxt, log2g);
    const int ut = fmod_(it.u, p.div_df);
    const int un = fmod_(in.u, p.div_df);
    s_item[0] = it.pos < total ? 1 : 0;
    s_item[1] = it.is_p1;
    s_item[2] = it.u;
    s_item[3] = it.idx;
    s_item[4] = fdiv(it.u, p.div_df);
    s_item[5] = fdiv(ut, p.div_F);
    s_item[6] = fmod_(it.u, p.div_slot);
    s_item[10] = fmod_(ut, p.div_F);
    s_item[7] = (in.pos < total && in.is_p1) ? 1 : 0;
    s_item[8] = fdiv(un, p.div_F);
    s_item[9] = in.idx;
    s_item[11] = sh_prev_next;  // this item's CSR heads were fetched during the previous item
    sh_prev_next = s_item[7];
    itn = in;
  };
  if (tid == 0) {
    const int64_t cur = atomicAdd(ticket, 1);
    nxt = atomicAdd(ticket, 1);
    itn = decode_item(p, cur, log2g);
    sh_ver[0] = sh_ver[1] = -1;
    sh_prev_next = 0;
    Deps D;  // the first item's dependencies (usually none)
    deps_of(itn, D);
    deps_settle(D);
    s_acc_ok = 0;
    describe();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  // Both operands' CSR heads of the next pass-1 item are fetched one item ahead.  In registers
  // (hd_next*, the one-k-per-lane mapping) the second-level load (entry words) waits for the
  // first (bucket offsets) and ptxas spills the results at once — a store that waits for them:
  // two L2 round trips at the start of every item (7 % of all warp samples on cfg3).  The pair
  // mapping therefore stages the plan's per-group head records (csr_heads_kernel) in shared
  // memory with cp.async: no register, no wait (cfg3 39.2 -> 38.1 ms, cfg4 501 -> 490 ms,
  // cfg5 b = 2^14 -3.4 %).  profiles/r02_ab_smem_heads.txt
  constexpr bool SMEM_HEADS = PAIR;
  PullHead hd_next, hd_next1;
  bool hd_valid = false;
  int hbuf = 0;  // the s_hw / s_hr buffer holding the next pass-1 item's heads
  while (true) {
    PROF_MARK(13);
    tc_fence_before();
    PROF_MARK(0);
    // [A]: the item descriptor (thread 0, after acquiring the item's dependencies) reaches the
    // CTA.  Warp 1 publishes the previous item (a release fence that waits for that item's
    // stores to drain) and joins through its own barrier, so the other warps start at once.
    if (warp == 1) {
      asm volatile("bar.sync 2, 64;" ::: "memory");
    } else {
      if (warp == 0) asm volatile("bar.arrive 2, 64;" ::: "memory");
      asm volatile("bar.sync 1, 224;" ::: "memory");
    }
    PROF_MARK(1);
    tc_fence_after();
    const int go = s_item[0];
    const int is_p1 = s_item[1], u = s_item[2], idx = s_item[3];
    const int kappa = s_item[4], t = s_item[5], slot = s_item[6], asl = s_item[10];
    const int next_p1 = s_item[7], next_t = s_item[8], next_idx = s_item[9];
    const bool hd_have = s_item[11] != 0;
    const int acc_ok = s_acc_ok && !p.acc_slow;
    if (tid == 0 && go) nxt = itn.pos < total ? (int64_t)atomicAdd(ticket, 1) : itn.pos;
    if (!go) break;
    PullHead hd_cur, hd_cur1;
    auto head = [&](int tt, int op, int blk) { return PAIR ? pull_head2(p, tt, op, blk) : pull_head(p, tt, op, blk); };
    if constexpr (SMEM_HEADS) {
      if (is_p1) {
        if (hd_have) {
          const int g = (tid >> 4);  // this half-warp's 16-bucket group within the block
          const int2 r0 = s_hr[hbuf][0][g], r1 = s_hr[hbuf][1][g];
          hd_cur.e_lo = r0.x; hd_cur.e_hi = r0.y; hd_cur.first = s_hw[hbuf][0][tid];
          hd_cur1.e_lo = r1.x; hd_cur1.e_hi = r1.y; hd_cur1.first = s_hw[hbuf][1][tid];
        } else {
          hd_cur = head(t, 0, idx);
          hd_cur1 = head(t, 1, idx);
        }
      }
      if (next_p1) {  // land while this item computes (waited for before [B])
        hbuf ^= 1;
        if (tid < 144) {
          const int op = tid >= 72 ? 1 : 0;
          const int r = tid - 72 * op;
          const int64_t ng = p.bsz >> 4;
          const int64_t rg = ((int64_t)next_t * 2 + op) * ng + (int64_t)next_idx * 16;
          const void *src = r < 64 ? (const void *)(p.hw + rg * 16 + r * 4) : (const void *)(p.hr + rg + (r - 64) * 2);
          const void *dst = r < 64 ? (const void *)(&s_hw[hbuf][op][r * 4]) : (const void *)(&s_hr[hbuf][op][(r - 64) * 2]);
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
    } else {
      if (is_p1) {
        hd_cur = hd_valid ? hd_next : head(t, 0, idx);
        hd_cur1 = hd_valid ? hd_next1 : head(t, 1, idx);
      }
      hd_valid = next_p1 != 0;
      if (hd_valid) {  // land while this item computes
        hd_next = head(next_t, 0, next_idx);
        hd_next1 = head(next_t, 1, next_idx);
      }
    }
    const int *acc_flag = acc_cnt + (t * p.F + asl) * p.nblk + idx;
    if constexpr (PAIR) {
      if (is_p1) p1_item2<FOLD>(p, kappa, t, asl, slot, idx, (double2 *)S, hd_cur1, hd_cur);
      else p2_item2<HB>(p, kappa, t, asl, slot, idx, tmem, acc_flag, acc_ok, (double2 *)S);
    } else {
      if (is_p1) p1_item(p, kappa, t, asl, slot, idx, S, hd_cur1, hd_cur);
      else p2_item<HB>(p, kappa, t, asl, slot, idx, tmem, acc_flag, acc_ok, S);
    }
    // thread 0: relaxed probe of the next item's dependency counters (acquired by the fence below);
    // the probe state crosses [B] in shared memory, not in (spilled) registers
    const int tid_t = tid_now();
    int pv0 = 0, pv1 = 0;  // the probed values stay in registers (a store of them would wait for the loads before [B])
    if (tid_t == 0) {
      Deps D;
      const Item nx = itn;
      deps_of(nx, D);
      sD = D;
      if (D.ptr[0]) pv0 = ld_relaxed(D.ptr[0]);
      if (D.ptr[1]) pv1 = ld_relaxed(D.ptr[1]);
      describe();  // the next item's descriptor, while the probes fly
    }
    if constexpr (SMEM_HEADS) asm volatile("cp.async.wait_group 0;" ::: "memory");  // the staged heads landed
    tc_fence_before();
    PROF_MARK(2);
    __syncthreads();  // [B]: the block's writes are done; smem / TMEM may be reused
    PROF_MARK(10);
    tc_fence_after();
    if (tid_t == 32) {
      // release this item's writes (covered through [B]), then publish it
      asm volatile("fence.release.gpu;" ::: "memory");
      if (is_p1) red_add(done1 + u, 1);
      else {
        red_add(acc_cnt + (t * p.F + asl) * p.nblk + idx, 1);
        red_add(done2 + u, 1);
      }
    }
    if (tid_t == 0) {
      // acquire the probed counters (PTX acquire pattern: relaxed reads, then an acquire fence;
      // no wait for outstanding stores), poll one that is not yet complete
      asm volatile("fence.acquire.gpu;" ::: "memory");
      Deps D = sD;
      D.val[0] = pv0;
      D.val[1] = pv1;
      deps_settle(D);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (p.prof && tid == 0)
    for (int k = 0; k < 16; ++k) atomicAdd((unsigned long long *)&p.prof[k], (unsigned long long)s_prof[k]);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

// ------------------------------------------------------------------ host
static inline int64_t pad256(int64_t x) { return ((x + 255) / 256) * 256; }

constexpr int MAX_LB = 16;  // per-slice transform bits handled by the two passes (8 + 8)

// The two-pass kernel serves every 2^8 <= b <= 2^20 (b > 2^16 through the top-level
// fold) at any input count below 2^26 (26-bit entry indices); it measured faster than
// the v1 fold kernels (fwht_compress.cu) at every such width and density, so those
// only serve b < 2^8 and b > 2^20.
bool fwht2p_supported(int log2b, int64_t n1, int64_t n2) {
  return log2b >= P1_BITS && log2b <= MAX_LB + 4 && n1 < ((int64_t)1 << 26) && n2 < ((int64_t)1 << 26);
}

// Ring plan.  lag: units between a unit's pass 1 and its pass 2, so that about 4
// items per SM are dispensable (a group dispenses 2 * nblk).  nslot = lag + slack:
// pass 1 of unit u reuses the Y slot of pass 2 of unit u - nslot, so the slack is
// how far pass 2 may trail before a pass-1 item has to wait; it takes whatever the
// ~96 MB L2 budget leaves (small transforms: 2 MB slots at b = 2^12, where slack 6
// measured 3.7 ms and slack 29 2.4 ms on cfg5 b = 2^12, d = 3).  At most U + 1
// slots are ever used.
static void ring_plan(int LB, int64_t U, int &lag, int &nslot) {
  const int nblk = 1 << (LB - P1_BITS);
  const int64_t slot = (int64_t)2 * (1 << LB) * KT * 8;
  int maxslots = (int)(((int64_t)96 << 20) / slot);
  if (maxslots < 3) maxslots = 3;
  lag = (4 * num_sms() + 2 * nblk - 1) / (2 * nblk);
  if (lag > maxslots - 2) lag = maxslots - 2;
  lag = lag < 1 ? 1 : (lag > 64 ? 64 : lag);
  int slack = maxslots - lag;
  slack = slack < 2 ? 2 : slack;
  nslot = lag + slack;
  if (nslot > U + 1) nslot = (int)(U + 1 > lag + 1 ? U + 1 : lag + 1);
}

// geometry: LB-bit slices, F = 2^(log2b - LB) of them (the fold of DESIGN.md §5)
static void fwht2p_geometry(int log2b, int &LB, int &F) {
  LB = log2b < MAX_LB ? log2b : MAX_LB;
  F = 1 << (log2b - LB);
}

int64_t fwht2p_workspace(int d, int log2b, int64_t n1, int64_t n2, int64_t K) {
  int LB, F;
  fwht2p_geometry(log2b, LB, F);
  const int64_t bs = (int64_t)1 << LB;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int64_t ntiles = (K + KT - 1) / KT;
  const int64_t U = ntiles * d * F;
  const int64_t nblk = bs >> P1_BITS;
  int64_t w = 0;
  w += pad256((int64_t)d * 2 * (bs + 1) * 4);  // off
  w += pad256((int64_t)d * 2 * bs * 4);        // cnt / fill
  w += pad256((int64_t)d * 2 * nmax * 4);      // ent
  int lag, nslot;
  ring_plan(LB, U, lag, nslot);
  w += pad256((int64_t)nslot * 2 * bs * KT * 8);  // Y ring
  w += pad256((1 + 2 * U + (int64_t)d * F * nblk) * 4);       // counters
  w += pad256((int64_t)d * 2 * (bs / 16) * 16 * 4);            // CSR heads: first words
  w += pad256((int64_t)d * 2 * (bs / 16) * 8);                 // CSR heads: ranges
  return w;
}

int fwht2p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, const double *xb, int64_t ldb,
                      int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc, bool acc_add, char *ws,
                      int64_t ws_bytes, cudaStream_t s) {
  const int d = h.d, log2b = h.log2b;
  int LB, F;
  fwht2p_geometry(log2b, LB, F);
  const int64_t b = (int64_t)1 << log2b;
  const int64_t bs = (int64_t)1 << LB;
  const int64_t K = k1 - k0;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  if (lda >= ((int64_t)1 << 28) || ldb >= ((int64_t)1 << 28)) {  // row offsets are 32-bit byte strides
    set_error("operand row stride too large for the two-pass kernel");
    return SMM_ERR_INVALID;
  }
  if (ws_bytes < fwht2p_workspace(d, log2b, n1, n2, K)) {
    set_error("compress workspace too small (two-pass)");
    return SMM_ERR_WORKSPACE;
  }
  char *q = ws;
  int32_t *off = (int32_t *)q;
  q += pad256((int64_t)d * 2 * (bs + 1) * 4);
  int32_t *cnt = (int32_t *)q;
  q += pad256((int64_t)d * 2 * bs * 4);
  uint32_t *ent = (uint32_t *)q;
  q += pad256((int64_t)d * 2 * nmax * 4);
  double *Y = (double *)q;
  const int64_t ntiles = (K + KT - 1) / KT;
  const int64_t U = ntiles * d * F;
  int lag, nslot;
  ring_plan(LB, U, lag, nslot);
  q += pad256((int64_t)nslot * 2 * bs * KT * 8);
  int *ctr = (int *)q;
  q += pad256((1 + 2 * U + (int64_t)d * F * (bs >> P1_BITS)) * 4);
  uint32_t *hw = (uint32_t *)q;
  q += pad256((int64_t)d * 2 * (bs / 16) * 16 * 4);
  int2 *hr = (int2 *)q;
  const int nblk = (int)(bs >> P1_BITS);
  if (K <= 0) {
    if (!acc_add) SMM_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)d * b * 8, s), "acc memset");
    return SMM_OK;
  }
  if (U > (int64_t)1 << 30) {
    set_error("inner range too large for one call");
    return SMM_ERR_INVALID;
  }
  // plan (CSR by bucket within the slice)
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * bs * 4, s), "csr memset");
  const int64_t nin = (int64_t)d * (n1 + n2);
  int64_t blocks = ceil_div(nin, 256);
  if (blocks > 8192) blocks = 8192;
  if (nin > 0) {
    csr_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, cnt, bs);
    SMM_LAUNCH_CHECK("csr_count_kernel");
  }
  csr_scan_kernel<<<d * 2, 1024, 0, s>>>(cnt, off, bs);
  SMM_LAUNCH_CHECK("csr_scan_kernel");
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * bs * 4, s), "csr memset");
  if (nin > 0) {
    csr_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, off, cnt, ent, nmax, bs);
    SMM_LAUNCH_CHECK("csr_fill_kernel");
    const int rc = csr_sort(off, ent, nmax, bs, d * 2, s);  // deterministic: increasing i per bucket
    if (rc) return rc;
  }
  {  // pair mapping: the head records the kernel stages in shared memory (SMEM_HEADS)
    const int64_t tot = (int64_t)d * 2 * bs;
    int64_t hblocks = ceil_div(tot, 256);
    if (hblocks > 8192) hblocks = 8192;
    csr_heads_kernel<<<(unsigned)hblocks, 256, 0, s>>>(off, ent, nmax, bs, d * 2, hw, hr);
    SMM_LAUNCH_CHECK("csr_heads_kernel");
  }
  SMM_CUDA_TRY(cudaMemsetAsync(ctr, 0, (size_t)(1 + 2 * U + (int64_t)d * F * nblk) * 4, s), "counter memset");
  TwoPassArgs p;
  p.h = h;
  p.X[0] = xa;
  p.X[1] = xb;
  p.ld[0] = lda;
  p.ld[1] = ldb;
  p.k0 = k0;
  p.K = K;
  p.B = log2b;
  p.hb = LB - P1_BITS;
  p.F = F;
  p.LB = LB;
  p.df = d * F;
  p.d = d;
  p.nblk = nblk;
  p.ntiles = (int)ntiles;
  p.U = (int)U;
  p.nslot = nslot;
  p.div_df = make_fastdiv((uint32_t)(d * F));
  p.div_F = make_fastdiv((uint32_t)F);
  p.div_slot = make_fastdiv((uint32_t)nslot);
  p.off = off;
  p.ent = ent;
  p.hw = hw;
  p.hr = hr;
  p.nmax = nmax;
  p.bsz = bs;
  p.Y = Y;
  p.acc = acc;
  p.ctr = ctr;
  p.prof = nullptr;
  p.acc_add = acc_add ? 1 : 0;
  p.lag = lag;
  static const bool acc_slow = getenv("SMM_ACC_SLOWPATH") != nullptr;
  p.acc_slow = acc_slow ? 1 : 0;
  {
    const int rc = l2_policies(p.pol_last, p.pol_first);
    if (rc) return rc;
  }
#ifdef SMM_FWHT2P_PROFILE
  static const bool prof_on = getenv("SMM_PROFILE") != nullptr;
#else
  static const bool prof_on = false;
  if (getenv("SMM_PROFILE")) {
    static bool said = false;
    if (!said) fprintf(stderr, "[fwht2p] SMM_PROFILE: this build has no phase marks (tools/prof_phases.sh)\n");
    said = true;
  }
#endif
  if (prof_on) {
    cudaMalloc((void **)&p.prof, 16 * sizeof(long long));
    cudaMemset(p.prof, 0, 16 * sizeof(long long));
    int one = 1;
    cudaMemcpyToSymbol(g_prof_on, &one, sizeof(int));
  }
  const size_t smem = (size_t)8 * 32 * 32 * 8;
  // two persistent CTAs per SM (256 threads, 128 registers, 64 KB smem, 128 TMEM columns each):
  // one CTA's barriers and memory latency overlap the other's FP64 work
  const int G = 2 * num_sms();
  // pair mapping: 16-byte operand rows need an even k origin, stride and range and an aligned base
  static const bool pair_off = getenv("SMM_NO_PAIR") != nullptr;
  const bool pair = !pair_off && p.hb >= 0 && (k0 % 2) == 0 && (K % 2) == 0 && (lda % 2) == 0 && (ldb % 2) == 0 &&
                    ((uintptr_t)xa % 16) == 0 && ((uintptr_t)xb % 16) == 0;
  KernelTimer timer(0, s);
  if (pair) switch (p.hb) {
#define SMM_LAUNCH_PAIR(H)                                                                                      \
  case H:                                                                                                       \
    SMM_CUDA_TRY(cudaFuncSetAttribute(fwht2p_kernel<H, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), \
                 "fwht2p smem");                                                                                \
    fwht2p_kernel<H, true><<<G, P_THREADS, smem, s>>>(p);                                                       \
    break;
    SMM_LAUNCH_PAIR(0) SMM_LAUNCH_PAIR(1) SMM_LAUNCH_PAIR(2) SMM_LAUNCH_PAIR(3) SMM_LAUNCH_PAIR(4) SMM_LAUNCH_PAIR(5) SMM_LAUNCH_PAIR(6) SMM_LAUNCH_PAIR(7)
#undef SMM_LAUNCH_PAIR
    case 8:  // 2^16-bucket slices: b = 2^16, or b > 2^16 folded (the fold character is compiled in only there)
      if (p.F > 1) {
        SMM_CUDA_TRY(cudaFuncSetAttribute(fwht2p_kernel<8, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem), "fwht2p smem");
        fwht2p_kernel<8, true, true><<<G, P_THREADS, smem, s>>>(p);
      } else {
        SMM_CUDA_TRY(cudaFuncSetAttribute(fwht2p_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem), "fwht2p smem");
        fwht2p_kernel<8, true><<<G, P_THREADS, smem, s>>>(p);
      }
      break;
    default: break;
  } else switch (p.hb) {
#define SMM_LAUNCH_HB(H)                                                                                 \
  case H:                                                                                                \
    SMM_CUDA_TRY(cudaFuncSetAttribute(fwht2p_kernel<H, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), \
                 "fwht2p smem");                                                                         \
    fwht2p_kernel<H, false><<<G, P_THREADS, smem, s>>>(p);                                               \
    break;
    SMM_LAUNCH_HB(0) SMM_LAUNCH_HB(1) SMM_LAUNCH_HB(2) SMM_LAUNCH_HB(3)
    SMM_LAUNCH_HB(4) SMM_LAUNCH_HB(5) SMM_LAUNCH_HB(6) SMM_LAUNCH_HB(7) SMM_LAUNCH_HB(8)
#undef SMM_LAUNCH_HB
    default:
      set_error("two-pass kernel: unsupported width");
      return SMM_ERR_INVALID;
  }
  timer.stop();
  SMM_LAUNCH_CHECK("fwht2p_kernel");
  if (p.prof) {
    long long h[16];
    cudaMemcpy(h, p.prof, sizeof(h), cudaMemcpyDeviceToHost);
    double tot = 0;
    for (int k = 0; k < 16; ++k)
      if (k != 11 && k != 12) tot += (double)h[k];  // m11 / m12: dependency waits inside m13
    fprintf(stderr, "[fwht2p profile, %% of thread-0 cycles over all CTAs]");
    for (int k = 0; k < 16; ++k)
      if (h[k]) fprintf(stderr, " m%d=%.1f", k, 100.0 * (double)h[k] / tot);
    fprintf(stderr, "\n");
    cudaFree(p.prof);
  }
  return SMM_OK;
}

}  // namespace smm
