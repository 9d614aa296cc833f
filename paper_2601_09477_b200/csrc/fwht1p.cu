// FWHT compress (steps 1-3) for b = 2^12 with small operands (n1 + n2 <= 16384):
// one pass, one inner index at a time per CTA, everything on chip.
// Reference: sketch.py:152-189 (scatter :166-172, FWHT :168 / :173, product :176-177).
//
// Why a second kernel.  For small transforms the two-pass kernel (fwht2p.cu) is bound
// by its cross-CTA dependencies: every unit's pass 2 waits for all of its pass 1, and the
// accumulator of each slice is a chain over the k-tiles.  Here one CTA per SM owns a
// share of the inner-dimension tiles and keeps everything of one inner index k on chip:
//   * the two input columns X_A[k, :] (A^T row k) and X_B[k, :] (B row k) are copied
//     into shared memory with cp.async (n1 + n2 doubles, <= 128 KB) — the signed
//     scatter then gathers from shared memory instead of L2;
//   * the CTA's two halves (256 threads each) transform the two operands side by side:
//     CSR pull into thread-private cells (bucket order = increasing input index, the
//     reference's serial order), 4 butterfly stages in registers, a swizzled shared-
//     memory exchange, 4 more, a second exchange, the last 4 (stages in ascending bit
//     order, as fwht_serial: the transform of one (k, t, op) is bit-identical to the
//     reference's and to fwht2p's);
//   * operand A's transform crosses to operand B's half through tensor memory (warps w
//     and w + 8 share a TMEM lane quadrant), B's half multiplies and extends the tile's
//     accumulator, which lives in TMEM for all d repetitions (d <= 7; deeper sketches
//     run as balanced groups of at most 7 repetitions, one launch each);
//   * the column of k + 1 is copied while the last repetition of k is transformed.
// The accumulator of every W-wide tile of inner indices (W | 32, relative to the call's
// k0) is written to a partial buffer; fwht1p_reduce_kernel adds the tiles in k order:
// acc = ((acc + T0) + T1) + ...  Deterministic, and with k-slabs on multiples of 32 the
// host-streamed path (SMM_FLAG_ACCUMULATE) reproduces one call's bits.
#include "plan.cuh"
#include "twopass.cuh"

namespace smm {

__global__ void csr_count_kernel(SketchHashes h, int64_t n1, int64_t n2, int32_t *cnt, int64_t b);  // fwht2p.cu
__global__ void csr_scan_kernel(const int32_t *cnt, int32_t *off, int64_t b);
__global__ void csr_fill_kernel(SketchHashes h, int64_t n1, int64_t n2, const int32_t *off, int32_t *fill,
                                uint32_t *ent, int64_t nmax, int64_t b);

namespace f1p {
using namespace tp;

constexpr int LB = 12;
constexpr int B = 1 << LB;
constexpr int HT = 256;                     // threads per half (one operand each)
constexpr int CT = 2 * HT;                  // threads per CTA
constexpr int MAXD = 7;                     // TMEM: 64 columns for A's transform + 64 per repetition
constexpr int64_t MAX_COLS = 16384;         // n1 + n2 staged in shared memory
constexpr int WARPS_PER_HALF = HT / 32;
// scatter word of the warp-interleaved CSR: byte offset of input i in the staged column
// (bits 0-16, i < 16384), bucket j within the thread's 16 (bits 17-20), first / last
// entry of its bucket (bits 21 / 22), sign (bit 31).  Padding words point at the zero
// double past the column and carry no flags.
constexpr uint32_t W_OFF = 0x1ffffu, W_FIRST = 1u << 21, W_LAST = 1u << 22, W_SIGN = 1u << 31;

// warp-interleaved CSR (one per (t, op)): entry q of lane l of half-warp w at
// ent2[base[w] + q * 32 + l], padded to the warp's longest range, so every step of a
// warp's scatter loop is one coalesced 128-byte load
struct Tab {
  int32_t base, maxcnt;
};

struct Args {
  const double *X[2];  // element (input i, inner index k) of operand op at X[op][k * ks[op] + i * is[op]]
  int64_t ks[2], is[2];
  int n[2];
  int64_t K;
  int d, W, ntiles;
  const uint32_t *ent2;  // [d][2][...] at row offsets roff[t * 2 + op]
  int64_t roff[2 * MAXD];
  const Tab *tab;        // [d][2][8]
  const uint32_t *bmask;  // [d][2][256]: buckets of each thread's 16 that have an entry
  double *part;          // [ntiles][d][B]
  int vec16;             // both operands allow 16-byte async copies
  int bulk;              // per operand: the column is staged with one TMA bulk copy
};

// exchange layout: one pad double per 16 (every access pattern below is conflict-free,
// and a thread's 16 addresses of one access differ by compile-time constants)
constexpr int XS = B + B / 16;  // doubles per half's exchange area
__device__ __forceinline__ int swz(int u) { return u + (u >> 4); }

__device__ __forceinline__ void bar_half(int h) { asm volatile("bar.sync %0, 256;" ::"r"(1 + h) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id) { asm volatile("bar.arrive %0, 512;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void bar_wait(int id) { asm volatile("bar.sync %0, 512;" ::"r"(id) : "memory"); }

__device__ __forceinline__ void fwht16(double (&v)[16]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int hq = 1 << q;
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (!(j & hq)) {
        const double x = v[j], y = v[j + hq];
        v[j] = x + y;
        v[j + hq] = x - y;
      }
  }
}

// copy column k of operand h into shared memory (cp.async, no registers).  A k-minor
// operand (A row-major) is read with 8-byte copies at stride is: 4x the L2 sectors, but
// the neighbouring inner indices of each sector are the CTA's next columns (L2 hits), and
// no transposed copy of the operand is needed
// A contiguous column with 16-byte alignment is one TMA bulk copy issued by thread 0 of the
// half and counted on the half's mbarrier (the LSU then carries none of the staging traffic)
__device__ __forceinline__ void column_copy(const Args &p, int h, int64_t k, double *col, int ht, uint64_t *bar) {
  const double *src = p.X[h] + k * p.ks[h];
  const int n = p.n[h];
  if (p.bulk & (1 << h)) {
    if (ht == 0 && n > 0) bulk_copy_g2s(col, src, (uint32_t)n * 8u, bar);
    return;
  }
  if (p.is[h] != 1) {
    const int64_t st = p.is[h];
    for (int i = ht; i < n; i += HT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + i * st) : "memory");
    }
  } else if (p.vec16 & (1 << h)) {
    for (int i = 2 * ht; i < n; i += 2 * HT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + i) : "memory");
    }
  } else {
    for (int i = ht; i < n; i += HT) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(col + i);
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src + i) : "memory");
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(CT, 1) fwht1p_kernel(Args p) {
  extern __shared__ __align__(16) double sm[];
  __shared__ uint32_t s_tmem;
  __shared__ __align__(8) uint64_t s_colbar[2];  // per half: bulk column copy landed
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int h = tid >> 8;   // 0: operand A, 1: operand B
  const int ht = tid & 255;
  const int hw = ht >> 5;   // warp within the half
  double *X = sm + h * XS;  // this half's exchange area (34 KB)
  // staged columns, each followed by one zero double (the padding words' target)
  double *col = sm + 2 * XS + (h ? ((p.n[0] + 2) & ~1) : 0);
  if (ht == 0) {
    col[p.n[h]] = 0.0;
    mbar_init(&s_colbar[h], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // byte offset of the zero double past the column (the padding words' target), pinned in a register:
  // ptxas otherwise re-reads p.n[h] with an indexed constant load inside the scatter loop, whose
  // latency the loop then waits for (10 % of the kernel's warp samples)
  uint32_t padw;
  asm volatile("mov.u32 %0, %1;" : "=r"(padw) : "r"((uint32_t)(p.n[h] * 8)));
  const bool bulk = (p.bulk >> h) & 1 && p.n[h] > 0;
  uint32_t colpar = 0;  // phase parity of the next bulk copy
  const uint32_t col_s = (uint32_t)__cvta_generic_to_shared(col);
  // this thread's 16 bucket cells (buckets 16 ht + j at X[j * 256 + ht]: the bank depends on the
  // thread only, so the scatter's cell stores are conflict-free whatever buckets the lanes hit)
  double *cells = X + ht;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t tq = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
  const uint32_t col_fa = (uint32_t)((hw >> 2) * 32);                     // A's transform
  auto col_acc = [&](int t) { return (uint32_t)(64 + t * 64 + (hw >> 2) * 32); };  // tile accumulator of t
  const int d = p.d;
  bool fa_pending = false;  // half A: B's half has not yet consumed the previous transform
  int64_t tile = blockIdx.x;
  int64_t k = tile * p.W;
  if (tile < p.ntiles) {
    __syncthreads();  // the mbarriers are initialised
    column_copy(p, h, k, col, ht, &s_colbar[h]);
  }
  for (; tile < p.ntiles; tile += gridDim.x) {
    const int64_t k_lo = tile * p.W;
    const int64_t k_hi = k_lo + p.W < p.K ? k_lo + p.W : p.K;
    for (k = k_lo; k < k_hi; ++k) {
      if (bulk) {
        mbar_wait(&s_colbar[h], colpar);
        colpar ^= 1u;
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      bar_half(h);  // the column is visible to the whole half; the exchange area is free
      for (int t = 0; t < d; ++t) {
        // ---- signed scatter of column k into this thread's 16 buckets [16 ht, 16 ht + 16):
        // entries in bucket order (increasing input index inside a bucket, the reference's
        // order); a bucket's sum starts from 0.0 at its first entry and is stored at its last
        const Tab tb = p.tab[(t * 2 + h) * WARPS_PER_HALF + hw];
        const uint32_t *e2 = p.ent2 + p.roff[t * 2 + h] + tb.base + lane;
        const uint32_t mask = __ldg(p.bmask + (t * 2 + h) * HT + ht);
        double run = 0.0;
        uint32_t wn[8], wn2[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) wn[r] = r < tb.maxcnt ? __ldg(e2 + r * 32) : padw;
#pragma unroll
        for (int r = 0; r < 8; ++r) wn2[r] = 8 + r < tb.maxcnt ? __ldg(e2 + (8 + r) * 32) : padw;
        for (int q0 = 0; q0 < tb.maxcnt; q0 += 8) {
          uint32_t w[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {  // the next two batches' words are in flight while this one is added
            w[r] = wn[r];
            wn[r] = wn2[r];
            wn2[r] = q0 + 16 + r < tb.maxcnt ? __ldg(e2 + (q0 + 16 + r) * 32) : padw;
          }
          double x[8];
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            double y;
            asm volatile("ld.shared.f64 %0, [%1];" : "=d"(y) : "r"(col_s + (w[r] & W_OFF)));
            // s(i) * a (sketch.py:166-167): the sign bit moved into the double's sign
            x[r] = __hiloint2double(__double2hiint(y) ^ (int)(w[r] & W_SIGN), __double2loint(y));
          }
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            run = ((w[r] & W_FIRST) ? 0.0 : run) + x[r];  // the reference's buckets start at 0.0
            if (w[r] & W_LAST) cells[((w[r] >> 17) & 15u) << 8] = run;
          }
        }
        double v[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = ((mask >> j) & 1u) ? cells[j << 8] : 0.0;
        bar_half(h);  // every cell is read before the exchange reuses the area
        if (t == d - 1) {
          // every gather of column k done by the half (barrier above): copy column k + 1 while k finishes
          int64_t kn = k + 1;
          if (kn >= k_hi) {
            const int64_t tn = tile + gridDim.x;
            kn = tn < p.ntiles ? tn * p.W : -1;
          }
          if (kn >= 0) column_copy(p, h, kn, col, ht, &s_colbar[h]);
        }
        // ---- FWHT over the 12 bucket bits, ascending (fwht_serial's stage order)
        fwht16(v);  // bits 0-3
#pragma unroll
        for (int j = 0; j < 16; ++j) X[swz(16 * ht + j)] = v[j];
        bar_half(h);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = X[swz((ht & 15) | (j << 4) | ((ht >> 4) << 8))];
        fwht16(v);  // bits 4-7
        bar_half(h);
#pragma unroll
        for (int j = 0; j < 16; ++j) X[swz((ht & 15) | (j << 4) | ((ht >> 4) << 8))] = v[j];
        bar_half(h);
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = X[swz(ht | (j << 8))];
        fwht16(v);  // bits 8-11: thread holds buckets ht | j << 8
        // ---- product through TMEM
        if (h == 0) {
          if (fa_pending) {
            bar_wait(4);  // B's half has loaded the previous transform
            tc_fence_after();
          }
          tmem_st8(tq + col_fa, v);
          tmem_st8(tq + col_fa + 16, v + 8);
          tmem_wait_st();
          tc_fence_before();
          bar_arrive(3);
          fa_pending = true;
        } else {
          bar_wait(3);
          tc_fence_after();
          double fa[16];
          tmem_ld8(tq + col_fa, fa);
          tmem_ld8(tq + col_fa + 16, fa + 8);
          tc_fence_before();
          bar_arrive(4);
          double pr[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) pr[j] = __dmul_rn(fa[j], v[j]);  // partial += pa * pb (sketch.py:176-177)
          if (k > k_lo) {
            double acc[16];
            tmem_ld8(tq + col_acc(t), acc);
            tmem_ld8(tq + col_acc(t) + 16, acc + 8);
#pragma unroll
            for (int j = 0; j < 16; ++j) pr[j] = __dadd_rn(acc[j], pr[j]);
          }
          tmem_st8(tq + col_acc(t), pr);
          tmem_st8(tq + col_acc(t) + 16, pr + 8);
          tmem_wait_st();
        }
        bar_half(h);  // the exchange area is reused by the next repetition's scatter
      }
    }
    // ---- the tile's sums to the partial buffer (B's half owns the accumulators)
    if (h == 1) {
      for (int t = 0; t < d; ++t) {
        double acc[16];
        tmem_ld8(tq + col_acc(t), acc);
        tmem_ld8(tq + col_acc(t) + 16, acc + 8);
        double *dst = p.part + ((int64_t)tile * d + t) * B + ht;
#pragma unroll
        for (int j = 0; j < 16; ++j) __stcs(dst + (j << 8), acc[j]);
      }
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  if (h == 0 && fa_pending) bar_wait(4);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// acc[t][u] = ((acc_in + T0) + T1) + ... over the tiles in k order (acc_add), or from T0
__global__ void fwht1p_reduce_kernel(const double *part, int ntiles, int d, double *acc, int acc_add) {
  const int64_t total = (int64_t)d * B;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = x / B, u = x % B;
    const double *pt = part + t * B + u;
    const int64_t stride = (int64_t)d * B;
    double s = acc_add ? acc[x] + pt[0] : pt[0];
    // batches of 32 independent loads, then the additions in tile order (few threads: d x b)
    for (int q0 = 1; q0 < ntiles; q0 += 32) {
      double v[32];
#pragma unroll
      for (int r = 0; r < 32; ++r) v[r] = q0 + r < ntiles ? __ldcg(pt + (int64_t)(q0 + r) * stride) : 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (q0 + r < ntiles) s += v[r];
    }
    acc[x] = s;
  }
}

struct RowOffsets {
  int64_t r[2 * MAXD];
};

// warp-interleaved scatter words of one (t, op) row per block (256 threads = the 8 warps of a half)
__global__ void csr_interleave_kernel(const int32_t *off, const uint32_t *ent, int64_t nmax, uint32_t *ent2,
                                      RowOffsets roff, Tab *tab, uint32_t *bmask, int n0, int n1) {
  __shared__ int s_max[WARPS_PER_HALF];
  const int row = blockIdx.x;
  const int nop = (row & 1) ? n1 : n0;
  const int ht = threadIdx.x, hw = ht >> 5, lane = ht & 31;
  const int32_t *o = off + (int64_t)row * (B + 1);
  const int lo = o[16 * ht], hi = o[16 * ht + 16];
  const int cnt = hi - lo;
  const int mx = __reduce_max_sync(0xffffffffu, cnt);
  if (lane == 0) s_max[hw] = mx;
  __syncthreads();
  int base = 0;
  for (int w = 0; w < hw; ++w) base += 32 * s_max[w];
  if (lane == 0) tab[row * WARPS_PER_HALF + hw] = Tab{base, mx};
  uint32_t *dst = ent2 + roff.r[row] + base + lane;
  const uint32_t *src = ent + (int64_t)row * nmax + lo;
  uint32_t mask = 0;
  for (int q = 0; q < mx; ++q) {
    uint32_t wd = (uint32_t)nop * 8u;  // padding: the zero double past the column
    if (q < cnt) {
      const uint32_t e = src[q];
      const uint32_t j = (e >> 26) & 15u;
      const bool first = q == 0 || ((src[q - 1] >> 26) & 15u) != j;
      const bool last = q == cnt - 1 || ((src[q + 1] >> 26) & 15u) != j;
      wd = ((e & 0x03ffffffu) * 8u) | (j << 17) | (first ? W_FIRST : 0u) | (last ? W_LAST : 0u) | (e & W_SIGN);
      mask |= 1u << j;
    }
    dst[q * 32] = wd;
  }
  bmask[row * HT + ht] = mask;
}

// words of one interleaved row: the sum over the 8 warps of 32 x (their longest range) is at
// most 32 x (the row's entries)
static int64_t ent2_row_bound(int64_t nop) { return 32 * (nop > 0 ? nop : 1); }

}  // namespace f1p

static inline int64_t pad256_(int64_t x) { return ((x + 255) / 256) * 256; }

static int f1p_tile_width(int d, int64_t K) {
  // W | 32: the finest that keeps the partial buffer under 512 MB (load balance over the SMs)
  for (int W : {8, 16, 32}) {
    const int64_t nt = (K + W - 1) / W;
    if (nt * d * f1p::B * 8 <= ((int64_t)512 << 20)) return W;
  }
  return 0;
}

// repetitions per launch: up to MAXD (the TMEM accumulators), deeper sketches in balanced
// groups of at most MAXD, one launch each (cfg5 b = 2^12 d = 9: 4.93 ms through fwht2p,
// 3.61 ms as two one-pass launches)
static int f1p_group(int d) {
  if (d <= f1p::MAXD) return d;
  const int ng = (d + f1p::MAXD - 1) / f1p::MAXD;
  return (d + ng - 1) / ng;
}

bool fwht1p_supported(int log2b, int d, int64_t n1, int64_t n2, int64_t K) {
  static const bool off = getenv("SMM_NO_FWHT1P") != nullptr;
  return !off && log2b == f1p::LB && d >= 1 && d <= SMM_MAX_DEPTH && n1 + n2 <= f1p::MAX_COLS &&
         n1 < f1p::MAX_COLS && n2 < f1p::MAX_COLS && (K == 0 || f1p_tile_width(f1p_group(d), K) > 0);
}

int64_t fwht1p_workspace(int d, int64_t n1, int64_t n2, int64_t K) {
  using namespace f1p;
  d = f1p_group(d);  // one group's workspace, reused by the next group
  const int64_t nmax = n1 > n2 ? n1 : n2;
  const int W = f1p_tile_width(d, K > 0 ? K : 1);
  const int64_t nt = (K + (W ? W : 32) - 1) / (W ? W : 32);
  int64_t w = 0;
  w += pad256_((int64_t)d * 2 * (B + 1) * 4);  // off
  w += pad256_((int64_t)d * 2 * B * 4);        // cnt / fill
  w += pad256_((int64_t)d * 2 * nmax * 4);     // ent
  w += pad256_((int64_t)d * (ent2_row_bound(n1) + ent2_row_bound(n2)) * 4);  // ent2
  w += pad256_((int64_t)d * 2 * WARPS_PER_HALF * sizeof(Tab));
  w += pad256_((int64_t)d * 2 * HT * 4);       // bucket masks
  w += pad256_(nt * d * B * 8);                // partial tile sums
  return w;
}

// operands in either layout (a_kminor / b_kminor: row = input, inner index contiguous;
// else row = inner index); inner range [k0, k1)
int fwht1p_accumulate(const SketchHashes &h, const double *xa, int64_t lda, bool a_kminor, const double *xb,
                      int64_t ldb, bool b_kminor, int64_t n1, int64_t n2, int64_t k0, int64_t k1, double *acc,
                      bool acc_add, char *ws, int64_t ws_bytes, cudaStream_t s) {
  using namespace f1p;
  if (h.d > MAXD) {
    // repetition groups, one launch each, into rows [t0, t0 + dg) of acc (workspace reused;
    // every repetition is independent, so the bits equal one launch's)
    const int dg = f1p_group(h.d);
    for (int t0 = 0; t0 < h.d; t0 += dg) {
      SketchHashes hg;
      hg.d = t0 + dg <= h.d ? dg : h.d - t0;
      hg.log2b = h.log2b;
      for (int g = 0; g < 4; ++g)
        for (int t = 0; t < hg.d; ++t) hg.f[g][t] = h.f[g][t0 + t];
      const int rc = fwht1p_accumulate(hg, xa, lda, a_kminor, xb, ldb, b_kminor, n1, n2, k0, k1,
                                       acc + (int64_t)t0 * B, acc_add, ws, ws_bytes, s);
      if (rc) return rc;
    }
    return SMM_OK;
  }
  const int d = h.d;
  const int64_t K = k1 - k0;
  const int64_t nmax = n1 > n2 ? n1 : n2;
  if (ws_bytes < fwht1p_workspace(d, n1, n2, K)) {
    set_error("compress workspace too small (one-pass)");
    return SMM_ERR_WORKSPACE;
  }
  if (K <= 0) {
    if (!acc_add) SMM_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)d * B * 8, s), "acc memset");
    return SMM_OK;
  }
  const int W = f1p_tile_width(d, K);
  const int64_t nt = (K + W - 1) / W;
  char *q = ws;
  int32_t *off = (int32_t *)q;
  q += pad256_((int64_t)d * 2 * (B + 1) * 4);
  int32_t *cnt = (int32_t *)q;
  q += pad256_((int64_t)d * 2 * B * 4);
  uint32_t *ent = (uint32_t *)q;
  q += pad256_((int64_t)d * 2 * nmax * 4);
  uint32_t *ent2 = (uint32_t *)q;
  q += pad256_((int64_t)d * (ent2_row_bound(n1) + ent2_row_bound(n2)) * 4);
  Tab *tab = (Tab *)q;
  q += pad256_((int64_t)d * 2 * WARPS_PER_HALF * sizeof(Tab));
  uint32_t *bmask = (uint32_t *)q;
  q += pad256_((int64_t)d * 2 * HT * 4);
  double *part = (double *)q;
  // CSR by bucket (fwht2p.cu's plan kernels) and its warp-interleaved copy
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * B * 4, s), "csr memset");
  const int64_t nin = (int64_t)d * (n1 + n2);
  int64_t blocks = ceil_div(nin, 256);
  if (blocks > 8192) blocks = 8192;
  if (nin > 0) {
    csr_count_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, cnt, B);
    SMM_LAUNCH_CHECK("csr_count_kernel");
  }
  csr_scan_kernel<<<d * 2, 1024, 0, s>>>(cnt, off, B);
  SMM_LAUNCH_CHECK("csr_scan_kernel");
  SMM_CUDA_TRY(cudaMemsetAsync(cnt, 0, (size_t)d * 2 * B * 4, s), "csr memset");
  if (nin > 0) {
    csr_fill_kernel<<<(unsigned)blocks, 256, 0, s>>>(h, n1, n2, off, cnt, ent, nmax, B);
    SMM_LAUNCH_CHECK("csr_fill_kernel");
    const int rc = csr_sort(off, ent, nmax, B, d * 2, s);
    if (rc) return rc;
  }
  RowOffsets ro;
  {
    int64_t pos = 0;
    for (int r = 0; r < 2 * d; ++r) {
      ro.r[r] = pos;
      pos += ent2_row_bound((r & 1) ? n2 : n1);
    }
  }
  csr_interleave_kernel<<<2 * d, HT, 0, s>>>(off, ent, nmax, ent2, ro, tab, bmask, (int)n1, (int)n2);
  SMM_LAUNCH_CHECK("csr_interleave_kernel");
  Args p;
  p.ks[0] = a_kminor ? 1 : lda;
  p.is[0] = a_kminor ? lda : 1;
  p.ks[1] = b_kminor ? 1 : ldb;
  p.is[1] = b_kminor ? ldb : 1;
  p.X[0] = xa + k0 * p.ks[0];
  p.X[1] = xb + k0 * p.ks[1];
  p.n[0] = (int)n1;
  p.n[1] = (int)n2;
  p.K = K;
  p.d = d;
  p.W = W;
  p.ntiles = (int)nt;
  p.ent2 = ent2;
  for (int r = 0; r < 2 * MAXD; ++r) p.roff[r] = r < 2 * d ? ro.r[r] : 0;
  p.tab = tab;
  p.bmask = bmask;
  p.part = part;
  p.vec16 = 0;  // per operand: 16-byte copies of contiguous columns
  p.bulk = 0;
  if (p.is[0] == 1 && p.ks[0] % 2 == 0 && n1 % 2 == 0 && (uintptr_t)p.X[0] % 16 == 0) p.vec16 |= 1;
  if (p.is[1] == 1 && p.ks[1] % 2 == 0 && n2 % 2 == 0 && (uintptr_t)p.X[1] % 16 == 0) p.vec16 |= 2;
  static const bool no_bulk = getenv("SMM_NO_BULK_COLUMNS") != nullptr;
  if (!no_bulk) p.bulk = p.vec16;  // contiguous, 16-byte aligned rows of a multiple of 16 bytes
  const size_t smem = (size_t)(2 * XS + ((n1 + 2) & ~1) + n2 + 1) * 8;
  SMM_CUDA_TRY(cudaFuncSetAttribute(fwht1p_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "fwht1p smem");
  int grid = num_sms();
  if (grid > nt) grid = (int)nt;
  {
    KernelTimer timer(0, s);
    fwht1p_kernel<<<grid, CT, smem, s>>>(p);
    timer.stop();
  }
  SMM_LAUNCH_CHECK("fwht1p_kernel");
  fwht1p_reduce_kernel<<<(unsigned)ceil_div((int64_t)d * B, 64), 64, 0, s>>>(part, (int)nt, d, acc, acc_add ? 1 : 0);
  SMM_LAUNCH_CHECK("fwht1p_reduce_kernel");
  return SMM_OK;
}

}  // namespace smm
