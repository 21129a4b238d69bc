// rounds.cu — Jacobi min-label rounds (minbased.py:124-304) on sm_100a.
//
// Layout: the working edge set is a COO (u, v[, idx], w) built once from the
// active CSR rows (driver.py:325-330 _gather_edges).
//
// Control: the fixpoint test of every family lives on the device.  Each
// round is a fixed kernel sequence bracketed by a 1-thread prologue (count
// the round and its inspections, clear the change flag) and epilogue (set
// `done` when the round changed nothing — that round is counted, as in the
// reference).  Every kernel returns at once when `done` is set, so the host
// enqueues rounds in batches and reads `done` once per batch instead of once
// per round.
#include <climits>
#include <cub/cub.cuh>

#include "pipeline.cuh"
#include "rounds.h"

namespace gc {

namespace {

constexpr int kRB = 256;
constexpr int kBatch = 4;  // rounds enqueued per host check
constexpr unsigned long long kNoWin = ~0ull;

unsigned long long* host_words() { return pinned_words(); }

// device-side round control words (slots of the counter block)
struct Ctl {
  unsigned long long* done;
  unsigned long long* changed;
  unsigned long long* rounds;
  unsigned long long* insp;
  unsigned long long* len;  // [2] working length per parity
  unsigned long long* wt;   // [2] working weight per parity
};

Ctl make_ctl(unsigned long long* ctr) {
  return Ctl{ctr + C_DONE, ctr + C_CHANGED, ctr + C_ROUNDS, ctr + C_RINSP, ctr + C_WLEN0, ctr + C_WWT0};
}

__global__ void k_set(unsigned long long* p, unsigned long long v) { *p = v; }

__global__ void k_ctl_init(Ctl c, unsigned long long len, unsigned long long wt, int nonempty) {
  *c.done = nonempty ? 0ull : 1ull;
  *c.changed = 0;
  *c.rounds = 0;
  *c.insp = 0;
  c.len[0] = c.len[1] = len;
  c.wt[0] = c.wt[1] = wt;
}

// round prologue: count it (insp += len(work) of this round), clear flags;
// with alter, the next parity's length / weight restart at zero
__global__ void k_round_begin(Ctl c, int par, int alter) {
  if (*c.done) return;
  *c.rounds += 1;
  *c.insp += c.wt[par];
  *c.changed = 0;
  if (alter) {
    c.len[par ^ 1] = 0;
    c.wt[par ^ 1] = 0;
  }
}

__global__ void k_round_end(Ctl c) {
  if (*c.done) return;
  if (*c.changed == 0) *c.done = 1;
}

#define GC_SKIP_IF_DONE(ctl) \
  if (*(ctl).done) return

// full-array passes take four entries per thread (16-byte accesses) when
// both arrays are 16-byte aligned, which every caller's buffers are
__device__ __forceinline__ bool aligned16(const void* a, const void* b) {
  return ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

__global__ void k_copy(int32_t* dst, const int32_t* src, int64_t n, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nq = aligned16(dst, src) ? n / 4 : 0;
  for (int64_t q = t0; q < nq; q += stride) reinterpret_cast<int4*>(dst)[q] = reinterpret_cast<const int4*>(src)[q];
  for (int64_t i = 4 * nq + t0; i < n; i += stride) dst[i] = src[i];
}

// ---------------------------------------------------------------- gather ---
__device__ __forceinline__ bool keep_entry(int32_t u, int32_t t, bool all_active, const int32_t* P,
                                           int32_t lmax, bool& twin) {
  twin = all_active || P[t] != lmax;
  if (!twin) return true;
  // label-equal twins never produce a message in any round rule: drop them
  return t > u && (all_active || P[u] != P[t]);
}

// Single-pass gather: a block takes 256 rows, counts their kept entries (all
// active: the sorted suffix t > u, found by binary search), scans the counts
// in the block, reserves its output range with one atomic on a cursor and
// writes.  Replaces count pass + device scan + host read + write pass; the
// entry order is then block-arrival order, which no round rule depends on
// (rounds are Jacobi, forest winners compare CSR indices).
__global__ void __launch_bounds__(kRB)
k_coo_gather(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, const int32_t* __restrict__ P,
             const int32_t* __restrict__ list, int64_t count, int32_t lmax, int all_active, int map_labels,
             Coo out, unsigned long long* cursor) {
  using Scan = cub::BlockScan<int, kRB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  const int64_t stride = int64_t(gridDim.x) * kRB;
  const uint64_t pol = evict_first_policy();
  for (int64_t i0 = int64_t(blockIdx.x) * kRB; i0 < count; i0 += stride) {
    const int64_t i = i0 + threadIdx.x;
    int32_t u = 0;
    int64_t b = 0, e = 0;
    int c = 0;
    // the first 32 entries' keep / twin decisions, so the write pass does
    // not repeat their random label reads (longer rows re-evaluate the rest)
    uint32_t keepm = 0, twinm = 0;
    if (i < count) {
      u = list ? list[i] : int32_t(i);
      // graph data streams through L2 evict-first: the labels stay resident
      b = ld_stream64(off + u, pol);
      e = ld_stream64(off + u + 1, pol);
      if (all_active) {
        int64_t lo = b, hi = e;  // rows are sorted: the kept entries t > u are a suffix
        while (lo < hi) {
          const int64_t mid = (lo + hi) >> 1;
          if (tgt[mid] > u) hi = mid; else lo = mid + 1;
        }
        b = lo;
        c = int(e - lo);
      } else {
        bool twin;
        for (int64_t j = b; j < e; ++j) {
          const bool k = keep_entry(u, tgt[j], false, P, lmax, twin);
          c += k;
          if (j - b < 32) {
            keepm |= uint32_t(k) << (j - b);
            twinm |= uint32_t(twin) << (j - b);
          }
        }
      }
    }
    int rank, total;
    Scan(tmp).ExclusiveSum(c, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(cursor, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    if (c) {
      const int32_t lu = map_labels ? P[u] : u;
      unsigned long long p = base + rank;
      for (int64_t j = b; j < e; ++j) {
        bool twin = true;
        if (!all_active && j - b < 32) {
          if (!(keepm >> (j - b) & 1u)) continue;
          twin = twinm >> (j - b) & 1u;
        }
        const int32_t t = tgt[j];
        if (!all_active && j - b >= 32 && !keep_entry(u, t, false, P, lmax, twin)) continue;
        out.u[p] = lu;
        out.v[p] = map_labels ? P[t] : t;
        out.w[p] = twin ? 2 : 1;
        if (out.idx) out.idx[p] = j;
        ++p;
      }
    }
    __syncthreads();  // base is rewritten next step
  }
}

// The gather's entries from a list of label-crossing pairs (LDD cut edges,
// each unordered pair once): a pair touching L_max becomes (active end,
// L_max end) with weight 1, any other (smaller id, larger id) with weight 2
// — the same entries k_coo_gather keeps (keep_entry), in place.
__global__ void __launch_bounds__(kRB)
k_cut_orient(const int32_t* __restrict__ P, int64_t count, int32_t lmax, int map_labels, Coo out) {
  const int64_t stride = int64_t(gridDim.x) * kRB;
  for (int64_t i = int64_t(blockIdx.x) * kRB + threadIdx.x; i < count; i += stride) {
    int32_t a = out.u[i], b = out.v[i];
    const int32_t la = P[a], lb = P[b];
    uint8_t w = 2;
    int32_t pa = la, pb = lb;
    if (la == lmax) {
      const int32_t t = a; a = b; b = t;
      pa = lb;
      pb = la;
      w = 1;
    } else if (lb == lmax) {
      w = 1;
    } else if (a > b) {
      const int32_t t = a; a = b; b = t;
      pa = lb;
      pb = la;
    }
    out.u[i] = map_labels ? pa : a;
    out.v[i] = map_labels ? pb : b;
    out.w[i] = w;
  }
}

// ----------------------------------------------------------------- forest ---
// Winner commit: root r records the original pair of its smallest winning
// edge index (minbased.py:95-116); the source row of CSR position j is found
// by binary search over the offsets.
__global__ void k_commit_win(unsigned long long* win, int64_t n, const int64_t* off,
                             const int32_t* tgt, int32_t* fu, int32_t* fv, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const unsigned long long j = win[v];
    if (j == kNoWin) continue;
    int64_t lo = 0, hi = n;  // last row with off[row] <= j
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (off[mid] <= int64_t(j)) lo = mid; else hi = mid - 1;
    }
    fu[v] = int32_t(lo);
    fv[v] = tgt[j];
    win[v] = kNoWin;
  }
}

__global__ void k_fill_u64(unsigned long long* a, int64_t n, unsigned long long v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

// ------------------------------------------------------ Shiloach-Vishkin ---
// minbased.py:124-155: hook the larger endpoint label onto the smaller when
// the larger is a root of the snapshot, then fully shortcut.
// SV over a chunked working list.  An edge whose endpoints share a snapshot
// label never sends another message (SV moves only roots and every vertex
// follows its label's chain, so equal labels stay equal), so after each
// round's hook every block compacts its own chunk in place, keeping only the
// differing edges: on a permuted grid 63% / 33% / 15% / 5% of the edges
// remain after rounds 1-4.  Each block owns one chunk for the whole loop (no
// global cursor); counted inspections keep the reference's full per-round
// edge count.
struct Chunks {
  int64_t* start = nullptr;
  int64_t* len = nullptr;
  uint8_t* keep = nullptr;             // per working edge: snapshot labels differ
  unsigned long long* count = nullptr; // [live, kept] per round parity: live[0..1], kept[2..3]
};

__global__ void k_chunk_init(Chunks ch, int nch, int64_t total) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c == 0) ch.count[0] = ch.count[1] = ch.count[2] = ch.count[3] = 0;
  if (c >= nch) return;
  const int64_t per = (total + nch - 1) / nch;
  const int64_t s = int64_t(c) * per < total ? int64_t(c) * per : total;
  const int64_t e = s + per < total ? s + per : total;
  ch.start[c] = s;
  ch.len[c] = e - s;
}

// hook: block b walks its chunk (no barriers, as a grid-stride loop would);
// keep[k] marks the edges whose snapshot labels still differ
__global__ void __launch_bounds__(kRB)
k_sv_hook_chunk(Coo c, Chunks ch, const int32_t* __restrict__ prev, int32_t* cur, uint8_t* keep, int par,
                Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t s = ch.start[blockIdx.x], L = ch.len[blockIdx.x];
  bool any = false;
  int kept = 0;
  for (int64_t t = threadIdx.x; t < L; t += kRB) {
    const int64_t k = s + t;
    const int32_t pu = prev[c.u[k]], pv = prev[c.v[k]];
    const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
    keep[k] = lo != hi;
    kept += lo != hi;
    if (lo != hi && prev[hi] == hi) {
      if (lo < ld_free(cur + hi)) red_min(cur + hi, lo);
      any = true;
    }
  }
  kept = __reduce_add_sync(0xffffffffu, kept);
  if ((threadIdx.x & 31) == 0 && kept) atomicAdd(ch.count + 2 + par, static_cast<unsigned long long>(kept));
  if (threadIdx.x == 0 && L) atomicAdd(ch.count + par, static_cast<unsigned long long>(L));
  if (__syncthreads_or(any) && threadIdx.x == 0) *ctl.changed = 1;
}

// In-place SV (no forest): one label array instead of a snapshot copy per
// round.  During the hook only roots' entries change, so the snapshot value
// of x is x itself when x was a root at the round's start and L[x] (not
// written this round) otherwise; the roots bitmap records the start-of-round
// roots and is rebuilt by the full shortcut that ends every round.  Same
// messages, same rounds and inspections as the snapshot form, without its
// two full-array passes per round.
__device__ __forceinline__ bool root_bit(const uint32_t* __restrict__ roots, int32_t x) {
  return (__ldg(roots + (x >> 5)) >> (x & 31)) & 1u;
}

__global__ void __launch_bounds__(kRB)
k_sv_hook_inplace(Coo c, Chunks ch, int32_t* L, const uint32_t* __restrict__ roots, uint8_t* keep, int par,
                  Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t s = ch.start[blockIdx.x], len = ch.len[blockIdx.x];
  bool any = false;
  int kept = 0;
  for (int64_t t = threadIdx.x; t < len; t += kRB) {
    const int64_t k = s + t;
    const int32_t u = c.u[k], v = c.v[k];
    const int32_t pu = root_bit(roots, u) ? u : ld_free(L + u);
    const int32_t pv = root_bit(roots, v) ? v : ld_free(L + v);
    const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
    keep[k] = lo != hi;
    kept += lo != hi;
    if (lo != hi && root_bit(roots, hi)) {
      if (lo < ld_free(L + hi)) red_min(L + hi, lo);  // stale: one extra red
      any = true;
    }
  }
  kept = __reduce_add_sync(0xffffffffu, kept);
  if ((threadIdx.x & 31) == 0 && kept) atomicAdd(ch.count + 2 + par, static_cast<unsigned long long>(kept));
  if (threadIdx.x == 0 && len) atomicAdd(ch.count + par, static_cast<unsigned long long>(len));
  if (__syncthreads_or(any) && threadIdx.x == 0) *ctl.changed = 1;
}

// full shortcut in place, writing the roots bitmap of the result.  Four
// vertices per thread (one 16-byte load; a stale value is an ancestor, so a
// plain load is safe while other threads shorten their own entries), the
// four first hops issued together, one 16-byte store when any moved; a warp
// covers 128 vertices = four bitmap words, each OR-reduced over its eight
// lanes.  A round without a hook changed nothing, so its shortcut (and
// bitmap) is skipped.  init: only the bitmap of the array as given.
__global__ void __launch_bounds__(kRB)
k_shortcut_roots(int32_t* a, int64_t n, uint32_t* roots, Ctl ctl, int init) {
  if (!init) {
    GC_SKIP_IF_DONE(ctl);
    if (*ctl.changed == 0) return;
  }
  const int lane = threadIdx.x & 31;
  const int64_t nq = (n + 3) / 4;
  const int64_t words = (n + 31) / 32;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < nq; base += stride) {
    const int64_t q = base + threadIdx.x;
    const int64_t v0 = 4 * q;
    unsigned nib = 0;
    if (q < nq) {
      int32_t r[4];
      const bool full = v0 + 3 < n;
      if (full) {
        const int4 x = reinterpret_cast<const int4*>(a)[q];
        r[0] = x.x, r[1] = x.y, r[2] = x.z, r[3] = x.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) r[k] = v0 + k < n ? ld_acq(a + v0 + k) : int32_t(v0 + k);
      }
      bool moved = false;
      if (!init) {
        // the four chains advance in lock step (four loads in flight per
        // hop): the step count is the longest chain, not the sum — a
        // natural-order grid builds chains hundreds of hops long.  Loads are
        // L1-cacheable: roots do not move during the pass and other threads
        // only shorten entries, so a stale value is an ancestor, and most
        // chains end at one hot root (an L2-only load per vertex piled onto
        // one L2 slice)
        int32_t h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = v0 + k < n ? ld_free(a + r[k]) : r[k];  // tail lanes: no read
        unsigned live = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) live |= unsigned(h[k] != r[k]) << k;
        moved = live != 0;
        while (live) {
#pragma unroll
          for (int k = 0; k < 4; ++k) r[k] = (live >> k) & 1u ? h[k] : r[k];
#pragma unroll
          for (int k = 0; k < 4; ++k) h[k] = (live >> k) & 1u ? ld_free(a + r[k]) : h[k];
#pragma unroll
          for (int k = 0; k < 4; ++k) live &= ~(unsigned(h[k] == r[k]) << k);
        }
      }
      if (moved) {
        if (full) reinterpret_cast<int4*>(a)[q] = make_int4(r[0], r[1], r[2], r[3]);
        else
          for (int k = 0; k < 4; ++k)
            if (v0 + k < n) st_rlx(a + v0 + k, r[k]);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) nib |= unsigned(v0 + k < n && r[k] == int32_t(v0 + k)) << k;
    }
    unsigned word = nib << (4 * (lane & 7));
    word |= __shfl_xor_sync(0xffffffffu, word, 1);
    word |= __shfl_xor_sync(0xffffffffu, word, 2);
    word |= __shfl_xor_sync(0xffffffffu, word, 4);
    if ((lane & 7) == 0 && (v0 >> 5) < words) roots[v0 >> 5] = word;
  }
}

// streaming in-place compaction of each chunk by its keep flags (tiles of
// the block; every thread reads its entry before the scan's barrier, and a
// write position never passes a read position)
__global__ void __launch_bounds__(kRB)
k_chunk_compact(Coo c, Chunks ch, const uint8_t* __restrict__ keep, int par, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  // the next round's hook counts into the other parity
  if (blockIdx.x == 0 && threadIdx.x == 0) ch.count[par ^ 1] = ch.count[2 + (par ^ 1)] = 0;
  // compaction pays when at least a third of the live edges closed (the
  // first round never drops any: labels start as the identity)
  const unsigned long long live = ch.count[par], kept = ch.count[2 + par];
  if (3 * (live - kept) < live) return;
  using Scan = cub::BlockScan<int, kRB>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t s = ch.start[blockIdx.x], L = ch.len[blockIdx.x];
  int64_t wpos = 0;
  for (int64_t t0 = 0; t0 < L; t0 += kRB) {
    const int64_t k = s + t0 + threadIdx.x;
    int kp = 0;
    int32_t u = 0, v = 0;
    uint8_t w = 0;
    int64_t id = 0;
    if (t0 + threadIdx.x < L && keep[k]) {
      kp = 1;
      u = c.u[k];
      v = c.v[k];
      w = c.w[k];
      if (c.idx) id = c.idx[k];
    }
    int rank, total;
    Scan(tmp).ExclusiveSum(kp, rank, total);
    if (kp) {
      const int64_t p = s + wpos + rank;
      c.u[p] = u;
      c.v[p] = v;
      c.w[p] = w;
      if (c.idx) c.idx[p] = id;
    }
    wpos += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) ch.len[blockIdx.x] = wpos;
}

// forest winners over the compacted chunks (a winning edge has differing
// snapshot labels, so compaction never drops one)
__global__ void k_sv_win_chunk(Coo c, Chunks ch, const int32_t* __restrict__ prev, const int32_t* cur,
                               unsigned long long* win, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t s = ch.start[blockIdx.x], L = ch.len[blockIdx.x];
  for (int64_t t = threadIdx.x; t < L; t += blockDim.x) {
    const int64_t k = s + t;
    const int32_t pu = prev[c.u[k]], pv = prev[c.v[k]];
    const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
    if (lo != hi && prev[hi] == hi && cur[hi] == lo)
      atomicMin(win + hi, static_cast<unsigned long long>(c.idx[k]));
  }
}

__global__ void k_full_shortcut(int32_t* a, int64_t n, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    int32_t r = ld_free(a + v);
    int32_t q = ld_free(a + r);
    if (q == r) continue;
    while (q != r) {
      r = q;
      q = ld_free(a + r);
    }
    st_rlx(a + v, r);
  }
}

// ------------------------------------------------------------ Liu-Tarjan ---
// minbased.py:163-243.  Messages (recipient <- value) per working edge:
//   Connect  : u <- v, v <- u
//   Parent   : L[u] <- L[v], L[v] <- L[u]
//   Extended : u <- L[v], v <- L[u], L[u] <- L[v], L[v] <- L[u]
template <class F>
__device__ __forceinline__ void lt_messages(int connect, int32_t u, int32_t v, const int32_t* L,
                                            F&& send) {
  if (connect == GC_LT_CONNECT) {
    send(u, v);
    send(v, u);
  } else {
    const int32_t pu = L[u], pv = L[v];
    if (connect == GC_LT_EXTENDED) {
      send(u, pv);
      send(v, pu);
    }
    send(pu, pv);
    send(pv, pu);
  }
}

__global__ void k_lt_connect(Coo c, const unsigned long long* len, const int32_t* __restrict__ L,
                             int32_t* msg, int connect, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t m = int64_t(*len);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += stride) {
    lt_messages(connect, c.u[k], c.v[k], L, [&](int32_t r, int32_t x) {
      if (x < ld_free(msg + r)) red_min(msg + r, x);  // msg only decreases: a stale (L1) value costs one extra red
    });
  }
}

// forest: a root lowered this round records its smallest winning edge index
__global__ void k_lt_win(Coo c, const unsigned long long* len, const int32_t* __restrict__ L,
                         const int32_t* msg, int connect, unsigned long long* win, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t m = int64_t(*len);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += stride) {
    const unsigned long long idx = static_cast<unsigned long long>(c.idx[k]);
    lt_messages(connect, c.u[k], c.v[k], L, [&](int32_t r, int32_t x) {
      if (L[r] == r && msg[r] < r && msg[r] == x) atomicMin(win + r, idx);
    });
  }
}

// update: roots take their message (ROOTS) or everyone does (ALL)
__global__ void k_lt_update(const int32_t* L, int32_t* msg, int64_t n, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nq = aligned16(L, msg) ? n / 4 : 0;
  for (int64_t q = t0; q < nq; q += stride) {
    const int4 l = reinterpret_cast<const int4*>(L)[q];
    const int32_t v = int32_t(4 * q);
    if (l.x == v && l.y == v + 1 && l.z == v + 2 && l.w == v + 3) continue;  // four roots: nothing to take
    int4 m = reinterpret_cast<const int4*>(msg)[q];
    if (l.x != v) m.x = l.x;
    if (l.y != v + 1) m.y = l.y;
    if (l.z != v + 2) m.z = l.z;
    if (l.w != v + 3) m.w = l.w;
    reinterpret_cast<int4*>(msg)[q] = m;
  }
  for (int64_t v = 4 * nq + t0; v < n; v += stride) {
    const int32_t l = L[v];
    if (l != v) msg[v] = l;
  }
}

// shortcut (one step: new[new[v]], full: root of new) + change test vs the
// round's starting labels; writes the next labels into L
__global__ void k_lt_shortcut(int32_t* L, const int32_t* msg, int64_t n, int full, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nq = aligned16(L, msg) ? n / 4 : 0;
  for (int64_t q = t0; q < nq; q += stride) {
    const int4 m4 = reinterpret_cast<const int4*>(msg)[q];
    int32_t x[4] = {m4.x, m4.y, m4.z, m4.w};
    int32_t y[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) y[k] = msg[x[k]];  // four first hops in flight
    if (full) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        while (y[k] != x[k]) {
          x[k] = y[k];
          y[k] = msg[x[k]];
        }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) x[k] = y[k];
    }
    const int4 l = reinterpret_cast<const int4*>(L)[q];
    if (l.x != x[0] || l.y != x[1] || l.z != x[2] || l.w != x[3]) {
      any = true;
      reinterpret_cast<int4*>(L)[q] = make_int4(x[0], x[1], x[2], x[3]);
    }
  }
  for (int64_t v = 4 * nq + t0; v < n; v += stride) {
    int32_t x = msg[v];
    if (full) {
      int32_t y = msg[x];
      while (y != x) {
        x = y;
        y = msg[x];
      }
    } else {
      x = msg[x];
    }
    if (x != L[v]) {
      any = true;
      L[v] = x;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) *ctl.changed = 1;
}

// alter: rewrite working edges to the current labels, drop closed ones.
// Block-aggregated compaction: one global atomic per block.
__global__ void __launch_bounds__(kRB) k_lt_alter(Coo in, const unsigned long long* in_len, Coo out,
                                                  unsigned long long* out_len, unsigned long long* out_wt,
                                                  const int32_t* L, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  using Scan = cub::BlockScan<int, kRB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  const int64_t m = int64_t(*in_len);
  unsigned long long wsum = 0;
  for (int64_t t0 = int64_t(blockIdx.x) * kRB; t0 < m; t0 += int64_t(gridDim.x) * kRB) {
    const int64_t k = t0 + threadIdx.x;
    int32_t a = 0, b = 0;
    int keep = 0;
    if (k < m) {
      a = L[in.u[k]];
      b = L[in.v[k]];
      keep = a != b;
    }
    int rank, total;
    Scan(tmp).ExclusiveSum(keep, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(out_len, static_cast<unsigned long long>(total)) : 0;
    __syncthreads();
    if (keep) {
      const unsigned long long p = base + rank;
      out.u[p] = a;
      out.v[p] = b;
      out.w[p] = in.w[k];
      if (in.idx) out.idx[p] = in.idx[k];
      wsum += in.w[k];
    }
    __syncthreads();
  }
  block_add<kRB>(out_wt, wsum);
}

// --------------------------------------------------------------- Stergiou ---
// minbased.py:251-276: reads only the previous array
__global__ void k_st_init(const int32_t* prev, int32_t* cur, int64_t n, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int32_t p = prev[v];
    const int32_t pp = prev[p];
    cur[v] = pp < p ? pp : p;
  }
}

__global__ void k_st_edges(Coo c, const unsigned long long* len, const int32_t* __restrict__ prev,
                           int32_t* cur, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t m = int64_t(*len);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += stride) {
    const int32_t u = c.u[k], v = c.v[k];
    const int32_t pu = prev[u], pv = prev[v];
    red_min(cur + u, pv);
    red_min(cur + v, pu);
    red_min(cur + pu, pv);
    red_min(cur + pv, pu);
  }
}

__global__ void k_differ(const int32_t* a, const int32_t* b, int64_t n, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    any |= a[v] != b[v];
  if (__syncthreads_or(any) && threadIdx.x == 0) *ctl.changed = 1;
}

// ------------------------------------------------------ label propagation ---
// minbased.py:284-304: lower the larger endpoint label of every differing edge
__global__ void k_lp(Coo c, const unsigned long long* len, const int32_t* __restrict__ snap,
                     int32_t* L, Ctl ctl) {
  GC_SKIP_IF_DONE(ctl);
  const int64_t m = int64_t(*len);
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < m; k += stride) {
    const int32_t u = c.u[k], v = c.v[k];
    const int32_t lu = snap[u], lv = snap[v];
    if (lu > lv) red_min(L + u, lv);
    if (lv > lu) red_min(L + v, lu);
    any |= lu != lv;
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) *ctl.changed = 1;
}

int grid_e(int64_t work) { return grid_for(work, kRB, 8); }

struct ForestOut {
  const int64_t* off = nullptr;
  const int32_t* tgt = nullptr;
  int32_t* fu = nullptr;
  int32_t* fv = nullptr;
  bool on() const { return fu != nullptr; }
};

#define L1(kernel, grid, ...) ((kernel<<<grid, kRB, 0, st>>>(__VA_ARGS__)), ::gc::count_launch())

// Enqueue one round of the configured family (round `r`, parity r & 1).
void enqueue_round(const gc_spec& s, int r, int32_t* P, int64_t nl, Coo* coo, RoundsWs& w, Ctl ctl,
                   int64_t edge_cap, const ForestOut& fo, int32_t*& A, int32_t*& B, const Chunks& ch,
                   cudaStream_t st) {
  const int par = r & 1;
  const int gv = grid_e(nl);
  const int gq = grid_e((nl + 3) / 4);  // quad-vectorised full-array passes
  const int ge = grid_e(edge_cap > 0 ? edge_cap : 1);
  const bool alter = s.finish == GC_FINISH_LT && s.lt_alter;
  Coo& cur = alter ? coo[par] : coo[0];
  const unsigned long long* len = alter ? ctl.len + par : ctl.len;
  ((k_round_begin<<<1, 1, 0, st>>>(ctl, alter ? par : 0, int(alter))), ::gc::count_launch());
  if (s.finish == GC_FINISH_SV && !fo.on()) {
    uint32_t* roots = reinterpret_cast<uint32_t*>(w.b);  // the snapshot buffer is free in this form
    L1(k_sv_hook_inplace, ge, cur, ch, A, roots, ch.keep, par, ctl);
    L1(k_chunk_compact, ge, cur, ch, ch.keep, par, ctl);
    L1(k_shortcut_roots, grid_e((nl + 3) / 4), A, nl, roots, ctl, 0);
  } else if (s.finish == GC_FINISH_SV) {
    L1(k_copy, gq, B, A, nl, ctl);
    L1(k_sv_hook_chunk, ge, cur, ch, A, B, ch.keep, par, ctl);
    if (fo.on()) {
      L1(k_sv_win_chunk, ge, cur, ch, A, B, w.win, ctl);
      L1(k_commit_win, gv, w.win, nl, fo.off, fo.tgt, fo.fu, fo.fv, ctl);
    }
    L1(k_chunk_compact, ge, cur, ch, ch.keep, par, ctl);
    L1(k_full_shortcut, gv, B, nl, ctl);
    std::swap(A, B);
  } else if (s.finish == GC_FINISH_LT) {
    int32_t* msg = w.b;
    L1(k_copy, gq, msg, P, nl, ctl);
    L1(k_lt_connect, ge, cur, len, P, msg, s.lt_connect, ctl);
    if (fo.on()) {
      L1(k_lt_win, ge, cur, len, P, msg, s.lt_connect, w.win, ctl);
      L1(k_commit_win, gv, w.win, nl, fo.off, fo.tgt, fo.fu, fo.fv, ctl);
    }
    if (s.lt_update == GC_LT_UPDATE_ROOTS) L1(k_lt_update, gq, P, msg, nl, ctl);
    L1(k_lt_shortcut, gq, P, msg, nl, int(s.lt_shortcut == GC_LT_SHORTCUT_FULL), ctl);
    if (alter)
      ((k_lt_alter<<<ge, kRB, 0, st>>>(cur, len, coo[par ^ 1], ctl.len + (par ^ 1), ctl.wt + (par ^ 1), P,
                                       ctl)), ::gc::count_launch());
  } else if (s.finish == GC_FINISH_STERGIOU) {
    L1(k_st_init, gv, A, B, nl, ctl);
    L1(k_st_edges, ge, cur, len, A, B, ctl);
    L1(k_differ, gv, A, B, nl, ctl);
    std::swap(A, B);
  } else {
    int32_t* snap = w.a;
    L1(k_copy, gq, snap, P, nl, ctl);
    L1(k_lp, ge, cur, len, snap, P, ctl);
  }
  ((k_round_end<<<1, 1, 0, st>>>(ctl)), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

// The round loop: rounds are enqueued kBatch at a time; the host reads the
// device `done` word once per batch.  Returns (rounds, inspections).
void loop_rounds(const gc_spec& s, int32_t* P, int64_t nl, Coo& work, RoundsWs& w, unsigned long long* ctr,
                 int64_t len, int64_t weight, bool nonempty, const ForestOut& fo, cudaStream_t st,
                 int64_t& rounds_out, int64_t& insp_out) {
  const Ctl ctl = make_ctl(ctr);
  ((k_ctl_init<<<1, 1, 0, st>>>(ctl, static_cast<unsigned long long>(len),
                                static_cast<unsigned long long>(weight), int(nonempty))),
   ::gc::count_launch());
  if (fo.on()) {
    (k_fill_u64<<<grid_e(nl), kRB, 0, st>>>(w.win, nl, kNoWin), ::gc::count_launch());
  }
  GC_CHECK_LAUNCH();
  Coo coo[2] = {work, w.spare};
  if (!fo.on()) coo[1].idx = nullptr;
  int32_t* A = P;
  int32_t* B = w.b;
  unsigned long long* h = host_words();
  // SV: per-block chunks of the working list, compacted in place each round
  Chunks ch;
  const int nch = grid_e(len > 0 ? len : 1);
  if (s.finish == GC_FINISH_SV) {
    require(w.keep != nullptr && w.chunks != nullptr && nch <= kMaxChunks, GC_ERR_OOM, "SV chunk tables missing");
    ch.start = w.chunks;
    ch.len = w.chunks + kMaxChunks;
    ch.keep = w.keep;
    ch.count = reinterpret_cast<unsigned long long*>(w.chunks + 2 * kMaxChunks);
    ((k_chunk_init<<<(nch + 255) / 256, 256, 0, st>>>(ch, nch, len)), ::gc::count_launch());
    // in-place form: the start-of-round roots of the first round
    if (!fo.on())
      ((k_shortcut_roots<<<grid_e((nl + 3) / 4), kRB, 0, st>>>(P, nl, reinterpret_cast<uint32_t*>(w.b), ctl, 1)),
       ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
  for (int r = 0; nonempty;) {
    for (int k = 0; k < kBatch; ++k, ++r) enqueue_round(s, r, P, nl, coo, w, ctl, len, fo, A, B, ch, st);
    GC_CUDA(cudaMemcpyAsync(h, ctl.done, 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    if (h[0]) break;
  }
  // SV / Stergiou ping-pong: at termination both buffers hold the fixpoint
  // (the last executed round changed nothing), so P is already final
  GC_CUDA(cudaMemcpyAsync(h, ctl.rounds, 16, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  rounds_out = int64_t(h[0]);
  insp_out = int64_t(h[1]);
}

}  // namespace

int64_t run_rounds_finish(const gc_csr& g, const gc_spec& s, int32_t* P, const int32_t* list,
                          unsigned long long* ctr, int32_t* fu, int32_t* fv, RoundsWs& w,
                          cudaStream_t st, bool cut_ready) {
  const int32_t n = int32_t(g.n);
  if (n == 0) return 0;
  // active count / gather degree sum / l_max from the device counters
  unsigned long long* h = host_words();
  GC_CUDA(cudaMemcpyAsync(h, ctr, sizeof(unsigned long long) * C_COUNT_, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  const bool all_active = list == nullptr;
  const int64_t count = all_active ? n : int64_t(h[C_N_ACTIVE]);
  const int32_t lmax = all_active ? n : int32_t(h[C_LMAX]);
  const int64_t degsum = all_active ? g.m : int64_t(h[C_INSP_FINISH]);
  if (count == 0) {
    (k_set<<<1, 1, 0, st>>>(ctr + C_INSP_FINISH, 0), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    return 0;
  }
  // gather the working COO (driver.py:325-330), twin-deduplicated, in one
  // pass (the cursor is the first word of the per-row count buffer)
  const bool map_labels = s.finish == GC_FINISH_LT || s.finish == GC_FINISH_LP;
  Coo& work = w.work;
  Coo out = work;
  if (!fu) out.idx = nullptr;
  if (cut_ready && !fu && !all_active) {
    // the sampler's cut edges, exactly the entries the gather keeps: orient
    // and weight them in place
    const int64_t cuts = int64_t(h[C_CUT]);
    if (cuts)
      (k_cut_orient<<<grid_e(cuts), kRB, 0, st>>>(P, cuts, lmax, map_labels, out), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    work.len = cuts;
  } else {
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(w.cnt);
    GC_CUDA(cudaMemsetAsync(cursor, 0, 8, st));
    (k_coo_gather<<<grid_e(count), kRB, 0, st>>>(g.offsets, g.targets, P, list, count, lmax, all_active,
                                                map_labels, out, cursor), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaMemcpyAsync(h, cursor, 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    work.len = int64_t(h[0]);
  }
  work.weight = degsum;
  work.idx = out.idx;
  ForestOut fo;
  if (fu) fo = ForestOut{g.offsets, g.targets, fu, fv};
  int64_t rounds = 0, insp = 0;
  loop_rounds(s, P, n, work, w, ctr, work.len, work.weight, true, fo, st, rounds, insp);
  // LP does not count the gather (driver.py:355-364)
  const int64_t total = (s.finish == GC_FINISH_LP ? 0 : degsum) + insp;
  (k_set<<<1, 1, 0, st>>>(ctr + C_INSP_FINISH, static_cast<unsigned long long>(total)),
   ::gc::count_launch());
  GC_CHECK_LAUNCH();
  return rounds;
}


int64_t run_rounds_coo(const gc_spec& s, int32_t* labels, int64_t nl, Coo& work, RoundsWs& w,
                       unsigned long long* ctr, int counter_slot, cudaStream_t st) {
  int64_t rounds = 0, insp = 0;
  loop_rounds(s, labels, nl, work, w, ctr, work.len, work.weight, true, ForestOut{}, st, rounds, insp);
  (k_set<<<1, 1, 0, st>>>(ctr + counter_slot, static_cast<unsigned long long>(insp)), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  return rounds;
}

}  // namespace gc
