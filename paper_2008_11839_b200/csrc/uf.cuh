// uf.cuh — the concurrent union / find / splice menu on sm_100a.
//
// Device restatement of dset.py (reference /root/reference/pkg/src/connlab):
//   finds   dset.py:109-172   (naive, compress, split, halve, two-try)
//   splices dset.py:180-214   (split-one, halve-one, atomic splice)
//   unions  dset.py:222-331   (async, hooks, early, rem-lock, rem-cas, jtb)
// The Python reference serializes CAS through 64 striped locks
// (parallel.py:17-36); here every CAS is a native 32-bit atomicCAS on the
// L2-resident parent array and every read is ld.relaxed.gpu.
//
// Conventions kept from the reference (dset.py:9-15): links go from the
// larger root id to the smaller (except JTB), failed compression CASes are
// dropped, and a root loses root status exactly once, so forest recording
// at the winning hook is single-shot.
#pragma once

#include "common.cuh"

namespace gc {

struct UFState {
  int32_t* P;           // parent[n]
  int32_t* H;           // hooks[n] (HOOKS), initialised to n
  int32_t* L;           // locks[n] (REM_LOCK), initialised to 0
  const uint32_t* R;    // ranks[n] (JTB)
  int32_t* fu;          // forest slot u (nullable)
  int32_t* fv;          // forest slot v
  int32_t n;
  int32_t* lu = nullptr;  // optional compact list of merging edges (distributed exchange)
  int32_t* lv = nullptr;
  unsigned long long* lcount = nullptr;
  // forest slots as (u, v) pairs: one 8-byte store per recorded link instead
  // of two 4-byte stores to two arrays (each a random DRAM read-modify-write
  // once the slot arrays outgrow L2); split into fu / fv by one pass at the end
  int2* fpair = nullptr;
  // L1-cacheable first reads (see Reader).  Kernels that initialise slots
  // while other threads union (incremental lazy init) turn them off: a stale
  // L1 line could still hold the uninitialised sentinel, which is not an
  // ancestor of anything.
  bool weak = true;
  // incremental giant filter (nullable): bit x of gbits set => x is
  // connected to the anchor vertex; *ganchor = the anchor component's root
  // as of the batch start (-1: none yet).  Membership only grows, so a set
  // bit never goes stale.
  uint32_t* gbits = nullptr;
  const int32_t* ganchor = nullptr;
  // lock-step async COO kernel: mark merging inserts by index (lflag[i] = 1)
  // instead of appending (u, v) to lu / lv through one shared counter
  uint8_t* lflag = nullptr;
  // giant-filter bitmap accesses carry an L2 evict_last hint (GC_GIANT_KEEP=0:
  // evict_normal)
  bool gkeep = true;
};


template <bool FOREST>
__device__ __forceinline__ void record(const UFState& s, int32_t slot, int32_t u, int32_t v) {
  if constexpr (FOREST) {
    if (s.fpair) {
      s.fpair[slot] = make_int2(u, v);
    } else if (s.fu) {
      s.fu[slot] = u;
      s.fv[slot] = v;
    }
    if (s.lu) {
      // warp-aggregated append: one counter atomic per group of lanes that
      // reach the link together (early incremental batches merge ~every edge)
      const unsigned m = __activemask();
      const int lane = threadIdx.x & 31;
      const int leader = __ffs(int(m)) - 1;
      unsigned long long base = 0;
      if (lane == leader) base = atomicAdd(s.lcount, static_cast<unsigned long long>(__popc(m)));
      base = __shfl_sync(m, base, leader);
      const unsigned long long i = base + __popc(m & ((1u << lane) - 1u));
      s.lu[i] = u;
      s.lv[i] = v;
    }
  }
}

// Parent reads.  The first kWeakReads loads of a union call are plain
// (L1-cacheable) loads: the hub vertices near the roots of large trees are
// read by millions of threads and an L1 hit avoids an L2 round trip to one
// hot line.  Any value read, however stale, is an ancestor of the vertex it
// was read from (parents only move up and decrease), so stale reads can
// cost retries but never merge the wrong sets; every link is still decided
// by a CAS at L2.  After the budget is spent all further reads are
// ld.relaxed.gpu, so each retry loop observes fresh values and terminates
// exactly as the all-strong algorithm does.
constexpr int kWeakReads = 48;

struct Reader {
  int budget;
  __device__ __forceinline__ explicit Reader(bool weak = true) : budget(weak ? kWeakReads : 0) {}
  __device__ __forceinline__ explicit Reader(const UFState& s) : budget(s.weak ? kWeakReads : 0) {}
  __device__ __forceinline__ int32_t operator()(const int32_t* p) {
    if (budget > 0) {
      --budget;
      return ld_weak(p);
    }
    return ld_acq(p);
  }
};

// ---------------------------------------------------------------- finds ---

// `known` (>= 0): a value of P[u] this thread already holds (one it just
// wrote, or read this iteration) — used instead of the first read.  A held
// value is at worst a stale read, which the rules already tolerate.
// `known_w` (>= 0, with `known`): a held value of P[known] as well.
// `first_w` (nullable) receives the value read for P[P[u]] in the first step.
template <int FIND>
__device__ __forceinline__ int32_t find(int32_t u, int32_t* P, Reader& rd, int32_t known = -1,
                                        int32_t known_w = -1, int32_t* first_w = nullptr) {
  if constexpr (FIND == GC_FIND_NAIVE) {
    // dset.py:109-112
    while (true) {
      int32_t pu = rd(P + u);
      if (pu == u) return u;
      u = pu;
    }
  } else if constexpr (FIND == GC_FIND_COMPRESS) {
    // dset.py:115-123: locate the root, then swing the path onto it
    int32_t r = u;
    while (true) {
      int32_t pr = rd(P + r);
      if (pr == r) break;
      r = pr;
    }
    while (true) {
      int32_t j = rd(P + u);
      if (j <= r) break;
      atomicCAS(P + u, j, r);
      u = j;
    }
    return r;
  } else if constexpr (FIND == GC_FIND_SPLIT) {
    // dset.py:126-135
    int32_t v = known >= 0 ? known : rd(P + u);
    int32_t w = known >= 0 && known_w >= 0 ? known_w : rd(P + v);
    if (first_w) *first_w = w;
    while (v != w) {
      atomicCAS(P + u, v, w);
      u = v;
      v = rd(P + u);
      w = rd(P + v);
    }
    return v;
  } else if constexpr (FIND == GC_FIND_HALVE) {
    // dset.py:138-147.  `u = p[u]` after the CAS is the value the CAS left
    // there: w when it succeeded, else the value it found — taken from the
    // CAS result instead of a second dependent read of the same word.
    int32_t v = known >= 0 ? known : rd(P + u);
    int32_t w = known >= 0 && known_w >= 0 ? known_w : rd(P + v);
    if (first_w) *first_w = w;
    while (v != w) {
      const int32_t old = atomicCAS(P + u, v, w);
      u = old == v ? w : old;
      v = rd(P + u);
      w = rd(P + v);
    }
    return v;
  } else {  // GC_FIND_TWO_TRY, dset.py:150-163
    int32_t v = rd(P + u);
    int32_t w = rd(P + v);
    while (v != w) {
      if (!cas(P + u, v, w)) {
        int32_t v2 = rd(P + u);
        int32_t w2 = rd(P + v2);
        if (v2 != w2) atomicCAS(P + u, v2, w2);
      }
      u = v;
      v = rd(P + u);
      w = rd(P + v);
    }
    return v;
  }
}

// -------------------------------------------------------------- splices ---

template <int SPLICE>
__device__ __forceinline__ int32_t splice(int32_t u, int32_t pu_seen, int32_t pv_seen, int32_t* P, Reader& rd) {
  // Rem walks call this with P[u] = pu_seen > pv_seen = P[v] as observed at
  // the loop head; every write below replaces a parent by a smaller id, so
  // concurrent splices can never close a cycle.
  if constexpr (SPLICE == GC_SPLICE_SPLIT_ONE) {
    // dset.py:180-186: returns u's old parent
    const int32_t pu = rd(P + u);
    const int32_t w = rd(P + pu);
    if (pu != w) atomicCAS(P + u, pu, w);
    return pu;
  } else if constexpr (SPLICE == GC_SPLICE_HALVE_ONE) {
    // dset.py:189-195: returns u's old grandparent
    const int32_t pu = rd(P + u);
    const int32_t w = rd(P + pu);
    if (pu != w) atomicCAS(P + u, pu, w);
    return w;
  } else {
    // dset.py:198-207: Rem's splice swings P[u] onto P[v]
    atomicCAS(P + u, pu_seen, pv_seen);
    return pu_seen;
  }
}

// --------------------------------------------------------------- unions ---
// All return true iff this call merged two trees.

template <int FIND, bool FOREST>
__device__ __forceinline__ bool union_async(const UFState& s, int32_t u, int32_t v, int32_t ku = -1,
                                            int32_t kv = -1) {
  // dset.py:222-234.  ku / kv (>= 0): values of P[u] / P[v] the caller just
  // read; for the one-step finds the grandparent reads of both endpoints are
  // then issued together before either walk starts.
  int32_t* P = s.P;
  Reader rd(s);
  int32_t pu, pv;
  if (FIND == GC_FIND_HALVE || FIND == GC_FIND_SPLIT) {
    if (ku >= 0 && kv >= 0) {
      const int32_t wu = ku == u ? u : rd(P + ku);
      const int32_t wv = kv == v ? v : rd(P + kv);
      pu = find<FIND>(u, P, rd, ku, wu);
      pv = find<FIND>(v, P, rd, kv, wv);
    } else {
      pu = find<FIND>(u, P, rd);
      pv = find<FIND>(v, P, rd);
    }
  } else {
    pu = find<FIND>(u, P, rd);
    pv = find<FIND>(v, P, rd);
  }
  while (pu != pv) {
    if (pu < pv) { int32_t t = pu; pu = pv; pv = t; }
    if (rd(P + pu) == pu && cas(P + pu, pu, pv)) {
      record<FOREST>(s, pu, u, v);
      return true;
    }
    pu = find<FIND>(u, P, rd);
    pv = find<FIND>(v, P, rd);
  }
  return false;
}

template <int FIND, bool FOREST>
__device__ __forceinline__ bool union_hooks(const UFState& s, int32_t u, int32_t v) {
  // dset.py:237-252: claim the hook slot, then an uncontended parent write.
  int32_t* P = s.P;
  Reader rd(s);
  const int32_t unhooked = s.n;
  int32_t pu = find<FIND>(u, P, rd);
  int32_t pv = find<FIND>(v, P, rd);
  while (pu != pv) {
    if (pu < pv) { int32_t t = pu; pu = pv; pv = t; }
    if (rd(P + pu) == pu && cas(s.H + pu, unhooked, pv)) {
      record<FOREST>(s, pu, u, v);
      // release: the forest slot is visible before the parent write
      __threadfence();
      st_rlx(P + pu, pv);
      return true;
    }
    pu = find<FIND>(u, P, rd);
    pv = find<FIND>(v, P, rd);
  }
  return false;
}

template <int FIND, bool FOREST>
__device__ __forceinline__ bool union_early(const UFState& s, int32_t u, int32_t v) {
  // dset.py:255-274
  int32_t* P = s.P;
  Reader rd(s);
  int32_t pu = u, pv = v;
  bool merged = false;
  while (pu != pv) {
    if (pu < pv) { int32_t t = pu; pu = pv; pv = t; }
    if (rd(P + pu) == pu && cas(P + pu, pu, pv)) {
      record<FOREST>(s, pu, u, v);
      merged = true;
      break;
    }
    int32_t z = rd(P + pu);
    int32_t w = rd(P + z);
    if (z != w) atomicCAS(P + pu, z, w);
    pu = w;
  }
  if constexpr (FIND != GC_FIND_NAIVE) {
    find<FIND>(u, P, rd);
    find<FIND>(v, P, rd);
  }
  return merged;
}

template <int FIND, int SPLICE, bool FOREST>
__device__ __forceinline__ bool union_rem_lock(const UFState& s, int32_t u, int32_t v) {
  // dset.py:277-300.  A failed re-validation re-derives and loops, as the
  // reference does (the paper's pseudocode returns instead).
  int32_t* P = s.P;
  Reader rd(s);
  int32_t ru = u, rv = v;
  while (true) {
    int32_t pru = rd(P + ru);
    int32_t prv = rd(P + rv);
    if (pru == prv) break;
    if (pru < prv) {
      int32_t t = ru; ru = rv; rv = t;
      t = pru; pru = prv; prv = t;
    }
    if (ru == pru) {
      // per-vertex spin lock; independent thread scheduling guarantees the
      // holder makes progress even when it shares a warp with waiters
      while (atomicCAS(s.L + ru, 0, 1) != 0) __nanosleep(32);
      __threadfence();
      // re-validate with fresh (L2) reads while holding ru's lock
      int32_t pv = ld_acq(P + rv);
      bool linked = (ru == ld_acq(P + ru)) && ru > pv;
      if (linked) {
        st_rlx(P + ru, pv);
        record<FOREST>(s, ru, u, v);
      }
      __threadfence();
      atomicExch(s.L + ru, 0);
      if (linked) return true;
    } else {
      ru = splice<SPLICE>(ru, pru, prv, P, rd);
    }
  }
  if constexpr (FIND != GC_FIND_NAIVE) {
    find<FIND>(u, P, rd);
    find<FIND>(v, P, rd);
  }
  return false;
}

template <int FIND, int SPLICE, bool FOREST>
__device__ __forceinline__ bool union_rem_cas(const UFState& s, int32_t u, int32_t v, int32_t ku = -1,
                                              int32_t kv = -1) {
  // dset.py:303-316 (ku / kv: held values of P[u] / P[v] for the first step)
  int32_t* P = s.P;
  Reader rd(s);
  int32_t ru = u, rv = v;
  bool first = ku >= 0 && kv >= 0;
  while (true) {
    int32_t pru = first ? ku : rd(P + ru);
    int32_t prv = first ? kv : rd(P + rv);
    first = false;
    if (pru == prv) return false;
    if (pru < prv) {
      int32_t t = ru; ru = rv; rv = t;
      t = pru; pru = prv; prv = t;
    }
    if (ru == pru && cas(P + ru, ru, prv)) {
      record<FOREST>(s, ru, u, v);
      if constexpr (FIND != GC_FIND_NAIVE) {
        // P[ru] is now prv and P[rv] was just read as prv; when both
        // endpoints start from prv, the second find reuses the first's
        // read of P[prv]
        const int32_t ku = (u == ru || u == rv) ? prv : -1;
        const int32_t kv = (v == ru || v == rv) ? prv : -1;
        int32_t w = -1;
        find<FIND>(u, P, rd, ku, -1, &w);
        find<FIND>(v, P, rd, kv, (ku >= 0 && kv == ku) ? w : -1);
      }
      return true;
    }
    ru = splice<SPLICE>(ru, pru, prv, P, rd);
  }
}

template <int FIND, bool FOREST>
__device__ __forceinline__ bool union_jtb(const UFState& s, int32_t u, int32_t v) {
  // dset.py:319-331: link the lower (rank, id) root under the higher one
  int32_t* P = s.P;
  Reader rd(s);
  while (true) {
    int32_t ru = find<FIND>(u, P, rd);
    int32_t rv = find<FIND>(v, P, rd);
    if (ru == rv) return false;
    uint32_t kru = s.R[ru], krv = s.R[rv];
    if (kru > krv || (kru == krv && ru > rv)) { int32_t t = ru; ru = rv; rv = t; }
    if (cas(P + ru, ru, rv)) {
      record<FOREST>(s, ru, u, v);
      return true;
    }
  }
}

// Compile-time (union, find, splice) triple.  Only the 32 combinations of
// dset.py:60-76 are ever instantiated (see dispatch.cuh).
template <int UNION, int FIND, int SPLICE, bool FOREST>
struct Rule {
  static constexpr int kUnion = UNION;
  static constexpr int kFind = FIND;
  static constexpr int kSplice = SPLICE;
  static constexpr bool kForest = FOREST;
  __device__ __forceinline__ static bool unite(const UFState& s, int32_t u, int32_t v) {
    if constexpr (UNION == GC_FINISH_ASYNC) return union_async<FIND, FOREST>(s, u, v);
    else if constexpr (UNION == GC_FINISH_HOOKS) return union_hooks<FIND, FOREST>(s, u, v);
    else if constexpr (UNION == GC_FINISH_EARLY) return union_early<FIND, FOREST>(s, u, v);
    else if constexpr (UNION == GC_FINISH_REM_LOCK) return union_rem_lock<FIND, SPLICE, FOREST>(s, u, v);
    else if constexpr (UNION == GC_FINISH_REM_CAS) return union_rem_cas<FIND, SPLICE, FOREST>(s, u, v);
    else return union_jtb<FIND, FOREST>(s, u, v);
  }
  // as unite, with pu0 / pv0 = values of P[u] / P[v] just read (or written)
  __device__ __forceinline__ static bool unite_known(const UFState& s, int32_t u, int32_t v, int32_t pu0,
                                                     int32_t pv0) {
    if constexpr (UNION == GC_FINISH_ASYNC) return union_async<FIND, FOREST>(s, u, v, pu0, pv0);
    else if constexpr (UNION == GC_FINISH_REM_CAS) return union_rem_cas<FIND, SPLICE, FOREST>(s, u, v, pu0, pv0);
    else return unite(s, u, v);
  }
};

}  // namespace gc
