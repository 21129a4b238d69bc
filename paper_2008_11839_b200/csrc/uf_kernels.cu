// uf_kernels.cu — union-find batch kernels and the compile-time dispatch
// over the 32-configuration matrix of dset.py:60-76.
//
// union_rows: the shared shape of k-out sampling (sampling.py:61-86),
// HB phase 2 (sampling.py:110-116) and the union-find finish
// (driver.py:333-348).  Work decomposition: a warp owns 32 consecutive
// rows; rows of at most kSmall entries are walked by their own lane (the
// paper's edge-serialization "ER": all edges of a vertex are unioned by one
// thread), larger rows are walked by the whole warp, one
// row at a time (warp-cooperative hub handling).
#include <climits>
#include <cstdlib>

#include "internal.h"
#include "uf.cuh"

namespace gc {

constexpr int kSmall = 32;
constexpr int kRowBlock = 512;  // measured: 512 -> 0.3505 ms, 256 -> 0.3522, 1024 -> 0.3549 (k-out s24)

template <class R>
__global__ void __launch_bounds__(kRowBlock)
k_union_rows(UFState s, const int64_t* __restrict__ off, const int32_t* __restrict__ tgt,
             const int32_t* __restrict__ list, const unsigned long long* count_dev,
             int64_t count_host, int32_t take_max, int32_t lower_only,
             unsigned long long* insp, int64_t row_base) {
  const int lane = threadIdx.x & 31;
  const int64_t warp0 = (int64_t(blockIdx.x) * kRowBlock + threadIdx.x) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * kRowBlock) >> 5;
  int64_t count = count_host;
  if (count_dev) {
    int64_t c = int64_t(*count_dev);
    count = c < count ? c : count;
  }
  unsigned long long my_insp = 0;
  const uint64_t pol = evict_first_policy();
  for (int64_t base = warp0 * 32; base < count; base += nwarps * 32) {
    const int64_t i = base + lane;
    int32_t u = -1;
    int64_t b = 0;
    int32_t take = 0;
    if (i < count) {
      u = list ? ldg32(list + i) : int32_t(row_base + i);
      // offsets stream through (no L1 allocation, L2 evict-first); targets
      // keep the default L1 path, which measured faster for the
      // neighbouring-row reuse within a warp
      b = ld_stream64(off + u, pol);
      const int64_t e = ld_stream64(off + u + 1, pol);
      const int64_t d = e - b;
      take = int32_t(d < take_max ? d : take_max);
      my_insp += take;
    }
    const bool big = take > kSmall;
    if (!big) {
      // the first two targets are fetched together (one DRAM round trip for
      // k-out's default k = 2); later ones on demand
      const int32_t f0 = take > 0 ? ldg32(tgt + b) : 0;
      const int32_t f1 = take > 1 ? ldg32(tgt + b + 1) : 0;
      for (int32_t j = 0; j < take; ++j) {
        const int32_t t = j == 0 ? f0 : j == 1 ? f1 : ldg32(tgt + b + j);
        if (lower_only && t >= u) break;
        R::unite(s, u, t);
      }
    }
    unsigned mask = __ballot_sync(0xffffffffu, big);
    while (mask) {
      const int src = __ffs(mask) - 1;
      mask &= mask - 1;
      const int32_t uu = __shfl_sync(0xffffffffu, u, src);
      const int64_t bb = __shfl_sync(0xffffffffu, b, src);
      const int32_t tk = __shfl_sync(0xffffffffu, take, src);
      for (int32_t j = lane; j < tk; j += 32) {
        const int32_t t = ldg32(tgt + bb + j);
        if (lower_only && t >= uu) break;
        R::unite(s, uu, t);
      }
    }
  }
  if (insp) block_add<kRowBlock>(insp, my_insp);
}

// Edge-parallel form of the all-active lower-only finish for graphs with
// fewer rows than resident threads (RMAT s16: 65k rows on 303k thread slots,
// each lane walking a whole row): one thread per CSR entry, its row by a
// binary search over the (cached) offsets; entry (u, t) is unioned when t < u
// — the same edge set as the row form.
template <class R>
__global__ void __launch_bounds__(256)
k_union_csr_edges(UFState s, const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int32_t n,
                  int64_t m) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m; j += stride) {
    const int32_t t = ldg32(tgt + j);
    int32_t lo = 0, hi = n - 1;  // last row with off[row] <= j
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (__ldg(off + mid) <= j) lo = mid;
      else hi = mid - 1;
    }
    if (t < lo) R::unite(s, lo, t);
  }
}

template <class R>
__global__ void __launch_bounds__(256)
k_union_coo(UFState s, const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
            const uint8_t* __restrict__ skip, int32_t sentinel, unsigned int* bad) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    if (skip && skip[i]) continue;
    const int32_t u = ldg32(us + i), v = ldg32(vs + i);
    if (bad && (uint32_t(u) >= uint32_t(s.n) || uint32_t(v) >= uint32_t(s.n))) {
      atomicOr(bad, 1u);  // malformed pair: never touches the parent array
      continue;
    }
    if (sentinel >= 0) {
      // ensure_init (driver.py:620-625) fused into the insert: every parent
      // a union reads is either one of its own endpoints (initialised right
      // here) or an ancestor, which was a root — hence initialised — when it
      // was linked.  The launcher turns L1-cached reads off for this mode.
      // Both endpoint reads are issued together and handed to the union as
      // its first parent reads (a CAS result is a held value too).
      int32_t pu = ld_acq(s.P + u);
      int32_t pv = ld_acq(s.P + v);
      if (pu == sentinel) {
        const int32_t o = atomicCAS(s.P + u, sentinel, u);
        pu = o == sentinel ? u : o;
      }
      if (pv == sentinel) {
        const int32_t o = atomicCAS(s.P + v, sentinel, v);
        pv = o == sentinel ? v : o;
      }
      R::unite_known(s, u, v, pu, pv);
      continue;
    }
    R::unite(s, u, v);
  }
}

// read-only root chase; an uninitialised slot is its own root (driver.py:556-564)
__device__ __forceinline__ int32_t chase(const int32_t* P, int32_t x, int32_t sentinel) {
  int32_t px = ld_acq(P + x);
  if (px == sentinel) return x;
  while (px != x) {
    x = px;
    px = ld_acq(P + x);
  }
  return x;
}

template <class R>
__global__ void __launch_bounds__(256)
k_incr_racy(UFState s, const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
            const uint8_t* __restrict__ is_query, int32_t sentinel, uint32_t* bits, unsigned int* bad) {
  // a warp owns 32 consecutive ops = one packed result word
  const int lane = threadIdx.x & 31;
  const int64_t words = (k + 31) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < words; w += nwarps) {
    const int64_t i = (w << 5) + lane;
    bool hit = false;
    if (i < k) {
      const int32_t u = us[i], v = vs[i];
      if (bad && (uint32_t(u) >= uint32_t(s.n) || uint32_t(v) >= uint32_t(s.n))) {
        atomicOr(bad, 1u);
      } else if (is_query[i]) {
        hit = chase(s.P, u, sentinel) == chase(s.P, v, sentinel);
      } else {
        atomicCAS(s.P + u, sentinel, u);  // ensure_init (driver.py:620-625)
        atomicCAS(s.P + v, sentinel, v);
        R::unite(s, u, v);
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) bits[w] = word;
  }
}

bool valid_uf(const UFConfig& c) {
  switch (c.unite) {
    case GC_FINISH_ASYNC:
    case GC_FINISH_HOOKS:
    case GC_FINISH_EARLY:
      return c.find >= GC_FIND_NAIVE && c.find <= GC_FIND_COMPRESS && c.splice == GC_SPLICE_NONE;
    case GC_FINISH_REM_LOCK:
    case GC_FINISH_REM_CAS:
      return c.find >= GC_FIND_NAIVE && c.find <= GC_FIND_HALVE &&
             c.splice >= GC_SPLICE_SPLIT_ONE && c.splice <= GC_SPLICE_ATOMIC;
    case GC_FINISH_JTB:
      return (c.find == GC_FIND_NAIVE || c.find == GC_FIND_TWO_TRY) && c.splice == GC_SPLICE_NONE;
    default:
      return false;
  }
}

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int dev = 0;
    GC_CUDA(cudaGetDevice(&dev));
    GC_CUDA(cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev));
  }
  return cached;
}

namespace {

// Functor-style launchers so one dispatch switch serves both kernels.
struct RowsLaunch {
  const RowUnionArgs& a;
  cudaStream_t st;
  template <class R>
  void go() const {
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, a.lu, a.lv, a.lcount};
    s.fpair = a.fpair;
    if (a.all_edges >= 0 && !a.list && a.lower_only && a.count_host == a.n &&
        a.count_host < int64_t(num_sms()) * 2048) {
      if (a.all_edges == 0) return;
      int64_t blocks = (a.all_edges + 255) / 256;
      const int64_t cap = int64_t(num_sms()) * 8 * 16;
      if (blocks > cap) blocks = cap;
      (k_union_csr_edges<R><<<int(blocks), 256, 0, st>>>(s, a.off, a.tgt, a.n, a.all_edges),
       ::gc::count_launch());
      GC_CHECK_LAUNCH();
      return;
    }
    int64_t warps = (a.count_host + 31) / 32;
    int64_t blocks = (warps * 32 + kRowBlock - 1) / kRowBlock;
    // one resident wave, grid-stride over 32-row groups
    const int64_t cap = int64_t(num_sms()) * (2048 / kRowBlock);
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    (k_union_rows<R><<<int(blocks), kRowBlock, 0, st>>>(s, a.off, a.tgt, a.list, a.count_dev,
                                                        a.count_host, a.take_max, a.lower_only,
                                                        a.insp, a.row_base), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

struct CooLaunch {
  const CooUnionArgs& a;
  cudaStream_t st;
  template <class R>
  void go() const {
    if (a.k <= 0) return;
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n, a.lu, a.lv, a.lcount};
    s.weak = a.init_sentinel < 0;
    int64_t blocks = (a.k + 255) / 256;
    const int64_t cap = int64_t(num_sms()) * 8 * 16;
    if (blocks > cap) blocks = cap;
    (k_union_coo<R><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, a.skip, a.init_sentinel, a.bad),
     ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

struct RacyLaunch {
  const CooUnionArgs& a;
  const uint8_t* is_query;
  int32_t sentinel;
  uint32_t* bits;
  cudaStream_t st;
  template <class R>
  void go() const {
    if (a.k <= 0) return;
    UFState s{a.P, a.H, a.L, a.R, a.fu, a.fv, a.n};
    s.weak = false;  // slots are initialised inside this launch
    int64_t blocks = (a.k + 255) / 256;
    const int64_t cap = int64_t(num_sms()) * 8 * 16;
    if (blocks > cap) blocks = cap;
    (k_incr_racy<R><<<int(blocks), 256, 0, st>>>(s, a.us, a.vs, a.k, is_query, sentinel, bits, a.bad),
     ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
};

template <int U, int F, int S, class L>
void go_forest(bool forest, const L& l) {
  if (forest) {
    if constexpr (S != GC_SPLICE_ATOMIC) l.template go<Rule<U, F, S, true>>();
    else throw Error(GC_ERR_CONFIG, "atomic splice is not root-based: no forest recording");
  } else {
    l.template go<Rule<U, F, S, false>>();
  }
}

template <int U, class L>
void go_find_nosplice(const UFConfig& c, bool forest, const L& l) {
  switch (c.find) {
    case GC_FIND_NAIVE: return go_forest<U, GC_FIND_NAIVE, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_SPLIT: return go_forest<U, GC_FIND_SPLIT, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_HALVE: return go_forest<U, GC_FIND_HALVE, GC_SPLICE_NONE>(forest, l);
    case GC_FIND_COMPRESS: return go_forest<U, GC_FIND_COMPRESS, GC_SPLICE_NONE>(forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid find rule");
}

template <int U, int F, class L>
void go_splice(const UFConfig& c, bool forest, const L& l) {
  switch (c.splice) {
    case GC_SPLICE_SPLIT_ONE: return go_forest<U, F, GC_SPLICE_SPLIT_ONE>(forest, l);
    case GC_SPLICE_HALVE_ONE: return go_forest<U, F, GC_SPLICE_HALVE_ONE>(forest, l);
    case GC_SPLICE_ATOMIC: return go_forest<U, F, GC_SPLICE_ATOMIC>(forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid splice rule");
}

template <int U, class L>
void go_rem(const UFConfig& c, bool forest, const L& l) {
  switch (c.find) {
    case GC_FIND_NAIVE: return go_splice<U, GC_FIND_NAIVE>(c, forest, l);
    case GC_FIND_SPLIT: return go_splice<U, GC_FIND_SPLIT>(c, forest, l);
    case GC_FIND_HALVE: return go_splice<U, GC_FIND_HALVE>(c, forest, l);
  }
  throw Error(GC_ERR_CONFIG, "invalid find rule for rem");
}

template <class L>
void dispatch(const UFConfig& c, bool forest, const L& l) {
  if (!valid_uf(c)) throw Error(GC_ERR_CONFIG, "unsupported union-find combination");
  switch (c.unite) {
    case GC_FINISH_ASYNC: return go_find_nosplice<GC_FINISH_ASYNC>(c, forest, l);
    case GC_FINISH_HOOKS: return go_find_nosplice<GC_FINISH_HOOKS>(c, forest, l);
    case GC_FINISH_EARLY: return go_find_nosplice<GC_FINISH_EARLY>(c, forest, l);
    case GC_FINISH_REM_LOCK: return go_rem<GC_FINISH_REM_LOCK>(c, forest, l);
    case GC_FINISH_REM_CAS: return go_rem<GC_FINISH_REM_CAS>(c, forest, l);
    case GC_FINISH_JTB:
      if (c.find == GC_FIND_NAIVE) return go_forest<GC_FINISH_JTB, GC_FIND_NAIVE, GC_SPLICE_NONE>(forest, l);
      return go_forest<GC_FINISH_JTB, GC_FIND_TWO_TRY, GC_SPLICE_NONE>(forest, l);
  }
}

}  // namespace

void launch_union_rows(const UFConfig& cfg, bool forest, const RowUnionArgs& a, cudaStream_t st) {
  if (a.count_host <= 0) return;
  dispatch(cfg, forest || a.lu != nullptr, RowsLaunch{a, st});
}

void launch_union_coo(const UFConfig& cfg, bool forest, const CooUnionArgs& a, cudaStream_t st) {
  dispatch(cfg, forest || a.lu != nullptr, CooLaunch{a, st});
}

void launch_incr_racy(const UFConfig& cfg, const CooUnionArgs& a, const uint8_t* is_query,
                      int32_t sentinel, uint32_t* bits, cudaStream_t st) {
  dispatch(cfg, false, RacyLaunch{a, is_query, sentinel, bits, st});
}

}  // namespace gc
