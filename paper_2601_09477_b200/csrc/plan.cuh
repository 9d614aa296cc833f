// Scatter plans: per (repetition t, operand op) the inner-dimension inputs are
// grouped into "rounds" so that the signed scatter-add into a length-l folded
// bucket vector needs neither atomics nor ordering between threads:
//   rank(q) = #{q' < q : c(q') = c(q)},  c(q) = h(q) mod l,
//   round r = { q : rank(q) = r } listed in increasing q.
// Inside a round every bucket is hit at most once; rounds run in order, so each
// bucket accumulates its inputs in increasing index order — the same order as
// the reference's serial scatter loop (sketch.py:166-167, 171-172).  The plan
// depends only on the hash functions, never on k, so it is built once per call.
#pragma once
#include "common.cuh"

namespace smm {

struct PlanView {
  uint32_t *list;    // nin entries, sorted by (round, q)
  int32_t *roff;     // round offsets, nin + 2 entries (roff[r]..roff[r+1])
  uint32_t *empty;   // buckets c in [0, l) with no input, increasing
  int32_t *meta;     // [0] = nrounds, [1] = nempty
};

// FWHT: op 0 = A side (h1/s1, n1 inputs), op 1 = B side (h2/s2, n2 inputs).
// FFT:  one combined op over q in [0, n1+n2): q < n1 -> A input i = q (h1),
//       otherwise B input j = q - n1 (h2).
// Per (t, op) block layout (each piece padded to 256 B):
//   list[nin_max] u32 | roff[nin_max+2] i32 | empty[l] u32 | meta[64] i32 |
//   fill[nin_max+2] i32 (scratch) | rank[nin_max] i32 (scratch)
int64_t plan_bytes_per(int64_t nin_max, int L);
int64_t plan_total_bytes(int d, int nops, int64_t n1, int64_t n2, int L);

// Sorts every bucket segment [off[m], off[m+1]) of `rows` CSR rows of ent (row stride
// nmax, b buckets, off row stride b + 1) by input index (entry bits 0-25): the
// deterministic within-bucket order after an atomic fill (plan.cu).
int csr_sort(const int32_t *off, uint32_t *ent, int64_t nmax, int64_t b, int rows, cudaStream_t s);

// builds all d * nops plans; scratch must hold plan_total_bytes(...)
int build_plans(const SketchHashes &h, int nops, int64_t n1, int64_t n2, int L, char *ws,
                cudaStream_t stream);

__device__ __forceinline__ PlanView plan_view_dev(char *base, int64_t per_bytes, int64_t nin_max, int L,
                                                  int nops, int t, int op) {
  char *p = base + (int64_t)(t * nops + op) * per_bytes;
  PlanView v;
  v.list = (uint32_t *)p;
  p += ((nin_max * 4 + 255) / 256) * 256;
  v.roff = (int32_t *)p;
  p += (((nin_max + 2) * 4 + 255) / 256) * 256;
  v.empty = (uint32_t *)p;
  p += ((((int64_t)1 << L) * 4 + 255) / 256) * 256;
  v.meta = (int32_t *)p;
  return v;
}

}  // namespace smm
