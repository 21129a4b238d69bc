// samplers.cu — k-out, hook-based and BFS sampling (sampling.py:61-172).
#include <climits>
#include <cstring>
#include <cub/cub.cuh>

#include "pipeline.cuh"
#include "samplers.h"

namespace gc {

// ---------------------------------------------------------------- k-out ---
// FIRST_PLUS_RANDOM (sampling.py:72-82): the first edge of every non-isolated
// vertex plus k-1 row offsets drawn on the host with the reference's numpy
// generator, materialised as COO pairs.
__global__ void k_kout_random_pairs(const int64_t* off, const int32_t* tgt, int32_t n, int32_t k,
                                    const int32_t* roff, int32_t* cu, int32_t* cv,
                                    unsigned long long* ctr) {
  unsigned long long cnt = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int64_t b = off[i], e = off[i + 1];
    const int64_t base = i * k;
    if (e == b) {
      for (int j = 0; j < k; ++j) cu[base + j] = cv[base + j] = int32_t(i);  // self pair: no-op
      continue;
    }
    cu[base] = int32_t(i);
    cv[base] = tgt[b];
    for (int j = 1; j < k; ++j) {
      cu[base + j] = int32_t(i);
      cv[base + j] = tgt[b + roff[i * (k - 1) + (j - 1)]];
    }
    cnt += k;
  }
  block_add<kEwBlock>(ctr + C_INSP_SAMPLE, cnt);
}

void run_kout(const gc_csr& g, const gc_spec& s, const UFConfig& c, RowUnionArgs a, bool forest,
              SamplerWs& w, unsigned long long* ctr, cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  if (n == 0) return;
  if (s.kout_mode == GC_KOUT_FIRST_K) {
    // sampling.py:68-71: the first min(k, deg) (smallest) neighbours; a
    // sharded caller restricts the rows to its block (a.row_base/count_host)
    a.list = nullptr;
    a.count_dev = nullptr;
    if (a.count_host <= 0 || a.count_host > n) {
      a.row_base = 0;
      a.count_host = n;
    }
    a.take_max = s.kout_k;
    a.lower_only = 0;
    a.insp = ctr + C_INSP_SAMPLE;
    launch_union_rows(c, forest, a, st);
    return;
  }
  require(s.kout_k == 1 || s.kout_rand_offsets != nullptr, GC_ERR_ARG,
          "FIRST_PLUS_RANDOM needs host-drawn row offsets");
  stamp_flush(ctr, st);  // deferred phase stamps: this path starts with a pair kernel
  (k_kout_random_pairs<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(
      g.offsets, g.targets, n, s.kout_k, s.kout_rand_offsets, w.coo_u, w.coo_v, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  CooUnionArgs ca{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, w.coo_u, w.coo_v, int64_t(n) * s.kout_k,
                  nullptr, a.lu, a.lv, a.lcount};
  launch_union_coo(c, forest, ca, st);
}

// ------------------------------------------------------------ hook-based ---
// Phase 1 (sampling.py:98-108): every non-isolated vertex points at its
// first (smallest) neighbour when that is smaller — write-disjoint, no
// atomics.  The surviving non-isolated roots form the phase-2 list.
__global__ void k_hb_phase1(const int64_t* off, const int32_t* tgt, int64_t lo, int64_t hi, int32_t* P,
                            int32_t* fu, int32_t* fv, int32_t* roots, unsigned long long* ctr,
                            int32_t* lu, int32_t* lv, unsigned long long* lcount, int2* fpair) {
  unsigned long long nz = 0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = lo + int64_t(blockIdx.x) * blockDim.x; base < hi; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool root = false;
    if (v < hi) {
      const int64_t b = off[v], e = off[v + 1];
      if (e > b) {
        ++nz;
        const int32_t first = tgt[b];
        if (first < v) {
          P[v] = first;
          if (fpair) {
            fpair[v] = make_int2(int32_t(v), first);
          } else if (fu) {
            fu[v] = int32_t(v);
            fv[v] = first;
          }
          if (lu) {  // a phase-1 hook always merges two trees (v was a singleton root)
            const unsigned long long i = atomicAdd(lcount, 1ull);
            lu[i] = int32_t(v);
            lv[i] = first;
          }
        } else {
          root = true;
        }
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, root);
    if (bal) {
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(ctr + C_SCRATCH0, static_cast<unsigned long long>(__popc(bal)));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (root) roots[pos + __popc(bal & ((1u << lane) - 1u))] = int32_t(v);
    }
  }
  block_add<kEwBlock>(ctr + C_INSP_SAMPLE, nz);
}

void run_hb(const gc_csr& g, const gc_spec& s, const UFConfig& c, RowUnionArgs a, bool forest,
            SamplerWs& w, unsigned long long* ctr, cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  if (n == 0 || g.m == 0) return;  // sampling.py:95-96
  stamp_flush(ctr, st);  // deferred phase stamps: phase 1 runs first
  GC_CUDA(cudaMemsetAsync(ctr + C_SCRATCH0, 0, 8, st));
  int64_t lo = 0, hi = n;
  if (a.count_host > 0 && a.count_host <= n) {  // sharded caller: its row block
    lo = a.row_base;
    hi = a.row_base + a.count_host;
  }
  (k_hb_phase1<<<grid_for(hi - lo, kEwBlock, 8), kEwBlock, 0, st>>>(g.offsets, g.targets, lo, hi, a.P, a.fu,
                                                                   a.fv, w.q0, ctr, a.lu, a.lv, a.lcount,
                                                                   a.fpair),
   ::gc::count_launch());
  GC_CHECK_LAUNCH();
  // Phase 2 (sampling.py:110-116): union the first N edges of each root
  a.list = w.q0;
  a.count_dev = ctr + C_SCRATCH0;
  a.count_host = n;
  a.row_base = 0;
  a.take_max = s.hb_edges;
  a.lower_only = 0;
  a.insp = ctr + C_INSP_SAMPLE;
  launch_union_rows(c, forest, a, st);
}

}  // namespace gc
