// samplers.cu — k-out, hook-based and BFS sampling (sampling.py:61-172).
#include <climits>
#include <cstring>

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
    // sampling.py:68-71: the first min(k, deg) (smallest) neighbours
    a.list = nullptr;
    a.count_dev = nullptr;
    a.count_host = n;
    a.take_max = s.kout_k;
    a.lower_only = 0;
    a.insp = ctr + C_INSP_SAMPLE;
    launch_union_rows(c, forest, a, st);
    return;
  }
  require(s.kout_k == 1 || s.kout_rand_offsets != nullptr, GC_ERR_ARG,
          "FIRST_PLUS_RANDOM needs host-drawn row offsets");
  (k_kout_random_pairs<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(
      g.offsets, g.targets, n, s.kout_k, s.kout_rand_offsets, w.coo_u, w.coo_v, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  CooUnionArgs ca{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, w.coo_u, w.coo_v, int64_t(n) * s.kout_k,
                  nullptr};
  launch_union_coo(c, forest, ca, st);
}

// ------------------------------------------------------------ hook-based ---
// Phase 1 (sampling.py:98-108): every non-isolated vertex points at its
// first (smallest) neighbour when that is smaller — write-disjoint, no
// atomics.  The surviving non-isolated roots form the phase-2 list.
__global__ void k_hb_phase1(const int64_t* off, const int32_t* tgt, int32_t n, int32_t* P,
                            int32_t* fu, int32_t* fv, int32_t* roots, unsigned long long* ctr) {
  unsigned long long nz = 0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool root = false;
    if (v < n) {
      const int64_t b = off[v], e = off[v + 1];
      if (e > b) {
        ++nz;
        const int32_t first = tgt[b];
        if (first < v) {
          P[v] = first;
          if (fu) {
            fu[v] = int32_t(v);
            fv[v] = first;
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
  GC_CUDA(cudaMemsetAsync(ctr + C_SCRATCH0, 0, 8, st));
  (k_hb_phase1<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(g.offsets, g.targets, n, a.P, a.fu,
                                                             a.fv, w.q0, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  // Phase 2 (sampling.py:110-116): union the first N edges of each root
  a.list = w.q0;
  a.count_dev = ctr + C_SCRATCH0;
  a.count_host = n;
  a.take_max = s.hb_edges;
  a.lower_only = 0;
  a.insp = ctr + C_INSP_SAMPLE;
  launch_union_rows(c, forest, a, st);
}

// ------------------------------------------------------------------- BFS ---
// Level-synchronous BFS from the host-chosen probe source (sampling.py:
// 120-172), direction-optimising: top-down over a frontier queue while the
// frontier is small, bottom-up over a frontier bitmap (n/8 bytes, L2
// resident) once its edges dominate.  The discovery parent of x is the
// smallest frontier vertex adjacent to x — exactly the reference's "first
// occurrence in the sorted frontier's concatenated rows" (np.unique
// return_index, :153-155): top-down takes it with atomicMin, bottom-up by
// scanning x's ascending row and stopping at the first frontier member.
// Both give the same forest, bit for bit.  The sample inspection count is
// the reference's per-level sum of frontier degrees, i.e. the degree sum of
// every reached vertex (:141-144).
constexpr int kBfsBlock = 256;

__device__ __forceinline__ bool test_bit(const uint32_t* bits, int32_t x) {
  return (__ldg(bits + (x >> 5)) >> (x & 31)) & 1u;
}

// frontier statistics of the level being produced: [0] count, [1] degree sum
__global__ void __launch_bounds__(kBfsBlock)
k_bfs_td(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt,
         const int32_t* __restrict__ q, const unsigned long long* qstat, int32_t* lvl, int32_t* par,
         int32_t* qn, unsigned long long* nstat, uint32_t* nbits, int32_t level, int32_t* minv) {
  const int lane = threadIdx.x & 31;
  const int64_t count = int64_t(qstat[0]);
  const int64_t warp0 = (int64_t(blockIdx.x) * kBfsBlock + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * kBfsBlock) >> 5;
  unsigned long long degs = 0;
  int32_t my_min = INT_MAX;
  auto visit = [&](int32_t f, int32_t x) {
    const int32_t lx = ld_acq(lvl + x);
    if (lx != -1 && lx != level + 1) return false;
    if (par) atomicMin(par + x, f);
    return lx == -1 && atomicCAS(lvl + x, -1, level + 1) == -1;
  };
  // warp-aggregated enqueue of newly claimed vertices
  auto push = [&](bool fresh, int32_t x) {
    const unsigned bal = __ballot_sync(0xffffffffu, fresh);
    if (!bal) return;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(nstat, static_cast<unsigned long long>(__popc(bal)));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (fresh) {
      qn[pos + __popc(bal & ((1u << lane) - 1u))] = x;
      atomicOr(nbits + (x >> 5), 1u << (x & 31));
      degs += static_cast<unsigned long long>(off[x + 1] - off[x]);
      my_min = x < my_min ? x : my_min;
    }
  };
  for (int64_t base = warp0 * 32; base < count; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t f = -1;
    int64_t b = 0, d = 0;
    if (i < count) {
      f = q[i];
      b = off[f];
      d = off[f + 1] - b;
    }
    const bool big = d > 32;
    // small rows: lanes walk their own rows in lock-step
    int64_t dm = big ? 0 : d;
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t t = __shfl_xor_sync(0xffffffffu, dm, o);
      dm = t > dm ? t : dm;
    }
    for (int64_t j = 0; j < dm; ++j) {
      int32_t x = 0;
      bool fresh = false;
      if (!big && j < d) {
        x = tgt[b + j];
        fresh = visit(f, x);
      }
      push(fresh, x);
    }
    unsigned mask = __ballot_sync(0xffffffffu, big);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t ff = __shfl_sync(0xffffffffu, f, src);
      const int64_t bb = __shfl_sync(0xffffffffu, b, src);
      const int64_t dd = __shfl_sync(0xffffffffu, d, src);
      for (int64_t j0 = 0; j0 < dd; j0 += 32) {
        const int64_t j = j0 + lane;
        int32_t x = 0;
        bool fresh = false;
        if (j < dd) {
          x = tgt[bb + j];
          fresh = visit(ff, x);
        }
        push(fresh, x);
      }
    }
  }
  block_add<kBfsBlock>(nstat + 1, degs);
  for (int o = 16; o > 0; o >>= 1) {
    const int32_t t = __shfl_xor_sync(0xffffffffu, my_min, o);
    my_min = t < my_min ? t : my_min;
  }
  if (lane == 0 && my_min != INT_MAX) atomicMin(minv, my_min);
}

// bottom-up: every unreached vertex looks for its first frontier neighbour;
// a warp owns 32 consecutive vertices and writes its next-bitmap word whole
__global__ void __launch_bounds__(kBfsBlock)
k_bfs_bu(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n, int32_t* lvl,
         int32_t* par, const uint32_t* __restrict__ cbits, uint32_t* nbits, unsigned long long* nstat,
         int32_t level, int32_t* minv) {
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = 0, degs = 0;
  int32_t my_min = INT_MAX;
  const int64_t stride = int64_t(gridDim.x) * kBfsBlock;
  for (int64_t base = int64_t(blockIdx.x) * kBfsBlock; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool found = false;
    if (v < n && lvl[v] == -1) {
      const int64_t b = off[v], e = off[v + 1];
      for (int64_t j = b; j < e; ++j) {
        const int32_t t = tgt[j];
        if (test_bit(cbits, t)) {
          found = true;
          lvl[v] = level + 1;
          if (par) par[v] = t;
          degs += static_cast<unsigned long long>(e - b);
          break;
        }
      }
    }
    const unsigned word = __ballot_sync(0xffffffffu, found);
    if (lane == 0 && word) nbits[(base + (threadIdx.x & ~31)) >> 5] = word;
    if (found) {
      ++cnt;
      my_min = int32_t(v) < my_min ? int32_t(v) : my_min;
    }
  }
  block_add<kBfsBlock>(nstat, cnt);
  block_add<kBfsBlock>(nstat + 1, degs);
  for (int o = 16; o > 0; o >>= 1) {
    const int32_t t = __shfl_xor_sync(0xffffffffu, my_min, o);
    my_min = t < my_min ? t : my_min;
  }
  if (lane == 0 && my_min != INT_MAX) atomicMin(minv, my_min);
}

// bitmap -> queue (switching back to top-down)
__global__ void k_bits_to_queue(const uint32_t* bits, int32_t n, int32_t* q, unsigned long long* qc) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const bool in = v < n && ((bits[v >> 5] >> (v & 31)) & 1u);
    const unsigned bal = __ballot_sync(0xffffffffu, in);
    if (!bal) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(qc, static_cast<unsigned long long>(__popc(bal)));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (in) q[pos + __popc(bal & ((1u << lane) - 1u))] = int32_t(v);
  }
}

__global__ void k_bfs_seed(const int64_t* off, int32_t* lvl, int32_t* q, unsigned long long* qstat,
                           uint32_t* bits, int32_t s, int32_t* minv, unsigned long long* insp) {
  lvl[s] = 0;
  q[0] = s;
  qstat[0] = 1;
  qstat[1] = static_cast<unsigned long long>(off[s + 1] - off[s]);
  bits[s >> 5] |= 1u << (s & 31);
  *minv = s;
  *insp += qstat[1];
}

// Re-root the discovery tree at the component minimum (sampling.py:161-168)
__global__ void k_bfs_reroot(int32_t* par, const int32_t* minv) {
  int32_t cur = *minv, prev = -1;
  while (cur != -1) {
    int32_t nxt = par[cur];
    if (nxt == INT_MAX) nxt = -1;
    par[cur] = prev;
    prev = cur;
    cur = nxt;
  }
}

// label the component with its minimum (:158-160) and emit forest slots
__global__ void k_bfs_label(const int32_t* lvl, const int32_t* par, const int32_t* minv,
                            int32_t n, int32_t* P, int32_t* fu, int32_t* fv) {
  const int32_t mn = *minv;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    if (lvl[v] < 0) continue;
    P[v] = mn;
    if (fu && v != mn) {
      fu[v] = par[v];
      fv[v] = int32_t(v);
    }
  }
}

void run_bfs(const gc_csr& g, const gc_spec& s, int32_t* P, int32_t* fu, int32_t* fv, SamplerWs& w,
             unsigned long long* ctr, cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  if (n == 0 || g.m == 0) return;  // sampling.py:128-129
  require(s.bfs_source >= 0 && s.bfs_source < n, GC_ERR_ARG, "BFS source out of range");
  const int64_t words = (int64_t(n) + 31) / 32;
  fill(w.lvl, n, -1, st);
  if (fu) fill(w.par, n, INT_MAX, st);
  GC_CUDA(cudaMemsetAsync(w.fb0, 0, words * 4, st));
  GC_CUDA(cudaMemsetAsync(w.fb1, 0, words * 4, st));
  int32_t* minv = reinterpret_cast<int32_t*>(ctr + C_SCRATCH1);
  // frontier stats [count, degree sum] for the two parities live in w.stat
  unsigned long long* fs[2] = {w.stat, w.stat + 2};
  int32_t* q[2] = {w.q0, w.q1};
  uint32_t* fb[2] = {w.fb0, w.fb1};
  GC_CUDA(cudaMemsetAsync(w.stat, 0, 4 * sizeof(unsigned long long), st));
  (k_bfs_seed<<<1, 1, 0, st>>>(g.offsets, w.lvl, q[0], fs[0], fb[0], int32_t(s.bfs_source), minv,
                               ctr + C_INSP_SAMPLE), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  unsigned long long* h = pinned_words();
  GC_CUDA(cudaMemcpyAsync(h, fs[0], 16, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  unsigned long long nf = h[0], mf = h[1];
  int64_t unexplored = g.m - int64_t(mf);
  bool bottom_up = false;
  const int bu_grid = grid_for(n, kBfsBlock, 4);
  for (int32_t level = 0; nf > 0; ++level) {
    const int c = level & 1, nx = c ^ 1;
    // Beamer's heuristic: go bottom-up when the frontier's edges exceed
    // 1/14 of the unexplored ones, back top-down when it shrinks below n/24
    const bool want_bu = bottom_up ? (nf >= uint64_t(n) / 24) : (int64_t(mf) * 14 > unexplored);
    if (!want_bu && bottom_up) {
      // the current frontier only exists as a bitmap: build its queue
      GC_CUDA(cudaMemsetAsync(fs[c], 0, 8, st));
      (k_bits_to_queue<<<grid_for(n, kEwBlock, 4), kEwBlock, 0, st>>>(fb[c], n, q[c], fs[c]),
       ::gc::count_launch());
    }
    bottom_up = want_bu;
    GC_CUDA(cudaMemsetAsync(fs[nx], 0, 16, st));
    GC_CUDA(cudaMemsetAsync(fb[nx], 0, words * 4, st));
    if (bottom_up) {
      (k_bfs_bu<<<bu_grid, kBfsBlock, 0, st>>>(g.offsets, g.targets, n, w.lvl, fu ? w.par : nullptr,
                                               fb[c], fb[nx], fs[nx], level, minv), ::gc::count_launch());
    } else {
      const int64_t blocks64 = (int64_t(nf) * 32 + kBfsBlock - 1) / kBfsBlock / 32 + 1;
      const int blocks = int(blocks64 < int64_t(num_sms()) * 8 ? blocks64 : int64_t(num_sms()) * 8);
      (k_bfs_td<<<blocks, kBfsBlock, 0, st>>>(g.offsets, g.targets, q[c], fs[c], w.lvl, fu ? w.par : nullptr,
                                               q[nx], fs[nx], fb[nx], level, minv), ::gc::count_launch());
    }
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaMemcpyAsync(h, fs[nx], 16, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    nf = h[0];
    mf = h[1];
    unexplored -= int64_t(mf);
    set_ctr_add(ctr, C_INSP_SAMPLE, mf, st);
  }
  if (fu) {
    (k_bfs_reroot<<<1, 1, 0, st>>>(w.par, minv), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
  (k_bfs_label<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(w.lvl, w.par, minv, n, P, fu, fv), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

}  // namespace gc

namespace gc {

// ------------------------------------------------------------------- LDD ---
// Low-diameter decomposition sampler (new; the reference has no LDD,
// driver.py:65-69 — it comes from ConnectIt, which GConn extends,
// PAPER.md:102).  Miller-Peng-Xu exponential-shift clustering:
//   delta_v ~ Exp(beta) from a counter-based hash of (seed, v);
//   v may start its own cluster at round floor(delta_max - delta_v);
//   clusters grow one hop per round.
// A vertex first reached in round r joins the smallest cluster id among its
// claimants that round (its own id if it starts then), so the decomposition
// is deterministic for a given seed.  Output labels are the minimum member
// id of each cluster, so P[v] <= v and every label class is connected: the
// partition refines the true one (validate.py:290-297).
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__device__ __forceinline__ float ldd_delta(uint64_t seed, int64_t v, float beta) {
  const uint64_t h = mix64(seed * 0xd1b54a32d192ed03ull + uint64_t(v));
  const double u = (double((h >> 11) + 1)) * (1.0 / 9007199254740992.0);  // (0, 1]
  return float(-log(u) / double(beta));
}

__global__ void k_ldd_delta_max(int32_t n, uint64_t seed, float beta, int32_t* dmax_bits) {
  float mx = 0.f;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mx = fmaxf(mx, ldd_delta(seed, v, beta));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(dmax_bits, __float_as_int(mx));  // positive floats order as ints
}

__global__ void k_ldd_start(int32_t n, uint64_t seed, float beta, const int32_t* dmax_bits,
                            uint16_t* start, int32_t* lvl, int32_t* cl) {
  const float dmax = __int_as_float(*dmax_bits);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const float r = floorf(dmax - ldd_delta(seed, v, beta));
    start[v] = uint16_t(r < 0.f ? 0.f : (r > 65535.f ? 65535.f : r));
    lvl[v] = -1;
    cl[v] = INT_MAX;
  }
}

// new centres of round r: unclaimed vertices whose start round is r
__global__ void k_ldd_centres(int32_t n, int32_t r, const uint16_t* start, int32_t* lvl, int32_t* cl,
                              int32_t* q, unsigned long long* qc) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    bool push = false;
    if (v < n && start[v] == r) {
      const int32_t lv = ld_acq(lvl + v);
      if (lv == -1 || lv == r) {
        atomicMin(cl + v, int32_t(v));
        push = lv == -1 && atomicCAS(lvl + v, -1, r) == -1;
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, push);
    if (bal) {
      unsigned long long pos = 0;
      if (lane == 0) pos = atomicAdd(qc, static_cast<unsigned long long>(__popc(bal)));
      pos = __shfl_sync(0xffffffffu, pos, 0);
      if (push) q[pos + __popc(bal & ((1u << lane) - 1u))] = int32_t(v);
    }
  }
}

// grow: frontier of round r-1 claims unclaimed neighbours in round r
__global__ void __launch_bounds__(kBfsBlock)
k_ldd_grow(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, const int32_t* q,
           const unsigned long long* qcount, int32_t* lvl, int32_t* cl, int32_t* qn,
           unsigned long long* qncount, int32_t r, unsigned long long* insp) {
  const int lane = threadIdx.x & 31;
  const int64_t count = int64_t(*qcount);
  const int64_t warp0 = (int64_t(blockIdx.x) * kBfsBlock + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * kBfsBlock) >> 5;
  unsigned long long my_insp = 0;
  for (int64_t base = warp0 * 32; base < count; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t c = INT_MAX;
    int64_t b = 0, d = 0;
    if (i < count) {
      const int32_t f = q[i];
      c = cl[f];
      b = off[f];
      d = off[f + 1] - b;
      my_insp += d;
    }
    // lanes walk their rows in lock-step so claims can be warp-aggregated
    int64_t dmax = d;
    for (int o = 16; o > 0; o >>= 1) {
      const int64_t t = __shfl_xor_sync(0xffffffffu, dmax, o);
      dmax = t > dmax ? t : dmax;
    }
    for (int64_t j = 0; j < dmax; ++j) {
      bool push = false;
      int32_t x = 0;
      if (j < d) {
        x = tgt[b + j];
        const int32_t lx = ld_acq(lvl + x);
        if (lx == -1 || lx == r) {
          atomicMin(cl + x, c);
          push = lx == -1 && atomicCAS(lvl + x, -1, r) == -1;
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, push);
      if (bal) {
        unsigned long long pos = 0;
        if (lane == 0) pos = atomicAdd(qncount, static_cast<unsigned long long>(__popc(bal)));
        pos = __shfl_sync(0xffffffffu, pos, 0);
        if (push) qn[pos + __popc(bal & ((1u << lane) - 1u))] = x;
      }
    }
  }
  block_add<kBfsBlock>(insp, my_insp);
}

__global__ void k_ldd_mins(const int32_t* cl, int32_t* mins, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    atomicMin(mins + cl[v], int32_t(v));
}

__global__ void k_ldd_label(const int32_t* cl, const int32_t* mins, int32_t* P, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    P[v] = mins[cl[v]];
}

void run_ldd(const gc_csr& g, const gc_spec& s, int32_t* P, SamplerWs& w, unsigned long long* ctr,
             cudaStream_t st) {
  const int32_t n = int32_t(g.n);
  if (n == 0) return;
  const float beta = s.ldd_beta > 0 ? float(s.ldd_beta) : 0.2f;
  int32_t* dmax = reinterpret_cast<int32_t*>(ctr + C_SCRATCH1);
  GC_CUDA(cudaMemsetAsync(dmax, 0, 4, st));
  const int ge = grid_for(n, kEwBlock, 8);
  (k_ldd_delta_max<<<ge, kEwBlock, 0, st>>>(n, s.seed, beta, dmax), ::gc::count_launch());
  (k_ldd_start<<<ge, kEwBlock, 0, st>>>(n, s.seed, beta, dmax, w.start, w.lvl, w.par), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  unsigned long long* hq = pinned_words();
  GC_CUDA(cudaMemcpyAsync(hq + 1, dmax, 4, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  float dmax_h;
  std::memcpy(&dmax_h, hq + 1, 4);
  const int32_t last_start = int32_t(floorf(dmax_h));
  unsigned long long* qc[2] = {ctr + C_NEXT, ctr + C_SCRATCH0};
  int32_t* q[2] = {w.q0, w.q1};
  GC_CUDA(cudaMemsetAsync(qc[0], 0, 8, st));
  // Rounds are enqueued kLddBatch at a time with fixed grids (the kernels
  // read the frontier size on the device); the host checks termination once
  // per batch.  Rounds past the end are empty launches.
  constexpr int kLddBatch = 8;
  const int grow_grid = num_sms() * 8;
  int ci = 0;
  for (int32_t r = 0;;) {
    for (int k = 0; k < kLddBatch; ++k, ++r) {
      GC_CUDA(cudaMemsetAsync(qc[ci ^ 1], 0, 8, st));
      if (r > 0)
        (k_ldd_grow<<<grow_grid, kBfsBlock, 0, st>>>(g.offsets, g.targets, q[ci], qc[ci], w.lvl, w.par,
                                                     q[ci ^ 1], qc[ci ^ 1], r, ctr + C_INSP_SAMPLE),
         ::gc::count_launch());
      if (r <= last_start)
        (k_ldd_centres<<<ge, kEwBlock, 0, st>>>(n, r, w.start, w.lvl, w.par, q[ci ^ 1], qc[ci ^ 1]),
         ::gc::count_launch());
      ci ^= 1;
    }
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaMemcpyAsync(hq, qc[ci], 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    if (*hq == 0 && r > last_start) break;
  }
  // labels: minimum member id per cluster (q0 is free again: reuse as mins)
  int32_t* mins = w.q0;
  fill(mins, n, INT_MAX, st);
  (k_ldd_mins<<<ge, kEwBlock, 0, st>>>(w.par, mins, n), ::gc::count_launch());
  (k_ldd_label<<<ge, kEwBlock, 0, st>>>(w.par, mins, P, n), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

}  // namespace gc
