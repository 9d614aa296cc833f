// Device helpers shared by the persistent two-pass compress kernels (internal
// linkage: every translation unit gets its own copy).
#pragma once
#include "common.cuh"

namespace smm {
namespace tp {

static __device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
static __device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
static __device__ __forceinline__ void red_add(int *ptr, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;" ::"l"(ptr), "r"(v) : "memory");
}
static __device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// x / d for 0 <= x < 2^31 by multiply-high
struct FastDiv {
  uint32_t m, d;
  int s;
};
static inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  f.d = d;
  f.s = 0;
  while ((1ull << f.s) < d) ++f.s;
  f.m = (uint32_t)((((1ull << f.s) - d) << 32) / d + 1);
  return f;
}
static __device__ __forceinline__ int fdiv(int x, const FastDiv &f) {
  return (int)((__umulhi((uint32_t)x, f.m) + (uint32_t)x) >> f.s);
}
static __device__ __forceinline__ int fmod_(int x, const FastDiv &f) { return x - fdiv(x, f) * (int)f.d; }

// ---- TMEM (32x32b shape: thread <-> TMEM lane, 16 x 32-bit columns = 8 doubles)
static __device__ __forceinline__ void tmem_st8(uint32_t taddr, const double *v) {
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
static __device__ __forceinline__ void tmem_ld8(uint32_t taddr, double *v) {
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
static __device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
static __device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
static __device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- L2 policies: the pass-1 -> pass-2 intermediate is written evict_last and read evict_first
static __device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
static __device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
static __device__ __forceinline__ void st2_hint(double *p, double a, double b, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b), "l"(pol) : "memory");
}
static __device__ __forceinline__ void ld2_hint(const double *p, double &a, double &b, uint64_t pol) {
  asm volatile("ld.global.cg.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(a), "=d"(b) : "l"(p), "l"(pol)
               : "memory");
}

// ---- TMA bulk copy global -> shared, completion counted on an mbarrier (one elected thread
// issues; every consumer waits on the barrier's phase parity)
static __device__ __forceinline__ void mbar_init(uint64_t *bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(bar)), "r"(count)
               : "memory");
}
static __device__ __forceinline__ void bulk_copy_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  // earlier generic-proxy accesses of dst (ordered before this thread by a barrier) come first
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(dst)),
               "l"(src), "r"(bytes), "r"(b)
               : "memory");
}
// two bulk copies counted on one barrier phase (one arrival with the total byte count)
static __device__ __forceinline__ void bulk_copy2_g2s(void *dst0, const void *src0, uint32_t bytes0, void *dst1,
                                                      const void *src1, uint32_t bytes1, uint64_t *bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes0 + bytes1) : "memory");
  if (bytes0)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst0)),
                 "l"(src0), "r"(bytes0), "r"(b)
                 : "memory");
  if (bytes1)
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst1)),
                 "l"(src1), "r"(bytes1), "r"(b)
                 : "memory");
}
static __device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(b), "r"(parity)
        : "memory");
}

// Sum over the 32 lanes of a warp, for each of 32 registers: recursive halving
// through shuffles (31 double shuffles per lane, no shared memory).  Step
// (L, R): lanes differing in lane bit L exchange register halves [0, R) / [R, 2R).
// The lane bits are combined in the order 1, 16, 8, 4, 2 — the same summation
// tree as the pair mapping of fwht2p (in-thread pair (2kp, 2kp+1) first, then
// kp bits 3..0), so both mappings give bit-identical accumulators.  Lane l ends
// with register lane_sum32_reg(l) summed over all lanes.
template <int L, int R, int N>
static __device__ __forceinline__ void halve_step(double (&v)[N], int lane) {
  const bool hi = (lane & L) != 0;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double send = hi ? v[r] : v[r + R];
    const double keep = hi ? v[r + R] : v[r];
    v[r] = keep + __shfl_xor_sync(0xffffffffu, send, L);
  }
}

static __device__ __forceinline__ int lane_sum32_reg(int l) {
  return ((l & 1) << 4) | (((l >> 4) & 1) << 3) | (((l >> 3) & 1) << 2) | (((l >> 2) & 1) << 1) | ((l >> 1) & 1);
}

static __device__ __forceinline__ double lane_sum32(double (&v)[32], int lane) {
  halve_step<1, 16>(v, lane);
  halve_step<16, 8>(v, lane);
  halve_step<8, 4>(v, lane);
  halve_step<4, 2>(v, lane);
  halve_step<2, 1>(v, lane);
  return v[0];
}

}  // namespace tp
}  // namespace smm
