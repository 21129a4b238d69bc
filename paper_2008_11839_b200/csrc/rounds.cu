// rounds.cu — Jacobi min-label rounds (minbased.py:124-304) on sm_100a.
//
// Layout: the working edge set is a COO (u, v[, idx], w) built once from the
// active CSR rows (driver.py:325-330 _gather_edges).  Every round is a short
// fixed kernel sequence; the host reads one change flag per round through a
// pinned word, mirroring the reference's per-round fixpoint test.
#include <climits>
#include <cub/cub.cuh>

#include "pipeline.cuh"
#include "rounds.h"

namespace gc {

namespace {

constexpr int kRB = 256;
constexpr unsigned long long kNoWin = ~0ull;

unsigned long long* host_words() { return pinned_words(); }

__global__ void k_set(unsigned long long* p, unsigned long long v) { *p = v; }
__global__ void k_add(unsigned long long* p, unsigned long long v) { *p += v; }

// ---------------------------------------------------------------- gather ---
__device__ __forceinline__ bool keep_entry(int32_t u, int32_t t, bool all_active, const int32_t* P,
                                           int32_t lmax, bool& twin) {
  twin = all_active || P[t] != lmax;
  return !twin || t > u;
}

__global__ void k_coo_count(const int64_t* off, const int32_t* tgt, const int32_t* P,
                            const int32_t* list, int64_t count, int32_t lmax, int all_active,
                            int64_t* cnt) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= count; i += stride) {
    if (i == count) {
      cnt[i] = 0;
      continue;
    }
    const int32_t u = list ? list[i] : int32_t(i);
    const int64_t b = off[u], e = off[u + 1];
    int64_t c = 0;
    if (all_active) {
      // rows are sorted: the kept entries t > u are a suffix
      int64_t lo = b, hi = e;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (tgt[mid] > u) hi = mid; else lo = mid + 1;
      }
      c = e - lo;
    } else {
      bool twin;
      for (int64_t j = b; j < e; ++j) c += keep_entry(u, tgt[j], false, P, lmax, twin);
    }
    cnt[i] = c;
  }
}

__global__ void k_coo_write(const int64_t* off, const int32_t* tgt, const int32_t* P,
                            const int32_t* list, int64_t count, int32_t lmax, int all_active,
                            int map_labels, const int64_t* pos, Coo out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int32_t u = list ? list[i] : int32_t(i);
    const int32_t lu = map_labels ? P[u] : u;
    int64_t p = pos[i];
    const int64_t b = off[u], e = off[u + 1];
    for (int64_t j = b; j < e; ++j) {
      const int32_t t = tgt[j];
      bool twin;
      if (!keep_entry(u, t, all_active, P, lmax, twin)) continue;
      out.u[p] = lu;
      out.v[p] = map_labels ? P[t] : t;
      out.w[p] = twin ? 2 : 1;
      if (out.idx) out.idx[p] = j;
      ++p;
    }
  }
}

// ----------------------------------------------------------------- forest ---
// Winner commit: root r records the original pair of its smallest winning
// edge index (minbased.py:95-116); the source row of CSR position j is found
// by binary search over the offsets.
__global__ void k_commit_win(unsigned long long* win, int64_t n, const int64_t* off,
                             const int32_t* tgt, int32_t* fu, int32_t* fv) {
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
__global__ void k_sv_hook(Coo c, const int32_t* __restrict__ prev, int32_t* cur,
                          unsigned long long* win, unsigned long long* changed) {
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    const int32_t pu = prev[c.u[k]], pv = prev[c.v[k]];
    const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
    if (lo != hi && prev[hi] == hi) {
      if (lo < ld_acq(cur + hi)) red_min(cur + hi, lo);
      any = true;
    }
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) *changed = 1;
}

__global__ void k_sv_win(Coo c, const int32_t* __restrict__ prev, const int32_t* cur,
                         unsigned long long* win) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    const int32_t pu = prev[c.u[k]], pv = prev[c.v[k]];
    const int32_t lo = pu < pv ? pu : pv, hi = pu < pv ? pv : pu;
    if (lo != hi && prev[hi] == hi && cur[hi] == lo)
      atomicMin(win + hi, static_cast<unsigned long long>(c.idx[k]));
  }
}

__global__ void k_full_shortcut(int32_t* a, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    int32_t r = ld_acq(a + v);
    int32_t q = ld_acq(a + r);
    if (q == r) continue;
    while (q != r) {
      r = q;
      q = ld_acq(a + r);
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

__global__ void k_lt_connect(Coo c, const int32_t* __restrict__ L, int32_t* msg, int connect) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    lt_messages(connect, c.u[k], c.v[k], L, [&](int32_t r, int32_t x) {
      if (x < ld_acq(msg + r)) red_min(msg + r, x);  // msg only decreases
    });
  }
}

// forest: a root lowered this round records its smallest winning edge index
__global__ void k_lt_win(Coo c, const int32_t* __restrict__ L, const int32_t* msg, int connect,
                         unsigned long long* win) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    const unsigned long long idx = static_cast<unsigned long long>(c.idx[k]);
    lt_messages(connect, c.u[k], c.v[k], L, [&](int32_t r, int32_t x) {
      if (L[r] == r && msg[r] < r && msg[r] == x) atomicMin(win + r, idx);
    });
  }
}

// update: roots take their message (ROOTS) or everyone does (ALL)
__global__ void k_lt_update(const int32_t* L, int32_t* msg, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int32_t l = L[v];
    if (l != v) msg[v] = l;
  }
}

// shortcut (one step: new[new[v]], full: root of new) + change test vs the
// round's starting labels; writes the next labels into L
__global__ void k_lt_shortcut(int32_t* L, const int32_t* msg, int64_t n, int full,
                              unsigned long long* changed) {
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
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
  if (__syncthreads_or(any) && threadIdx.x == 0) *changed = 1;
}

// alter: rewrite working edges to the current labels, drop closed ones.
// Block-aggregated compaction: one global atomic per block.
__global__ void __launch_bounds__(kRB) k_lt_alter(Coo in, Coo out, const int32_t* L,
                                                  unsigned long long* ctr) {
  using Scan = cub::BlockScan<int, kRB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long base;
  unsigned long long wsum = 0;
  for (int64_t t0 = int64_t(blockIdx.x) * kRB; t0 < in.len; t0 += int64_t(gridDim.x) * kRB) {
    const int64_t k = t0 + threadIdx.x;
    int32_t a = 0, b = 0;
    int keep = 0;
    if (k < in.len) {
      a = L[in.u[k]];
      b = L[in.v[k]];
      keep = a != b;
    }
    int rank, total;
    Scan(tmp).ExclusiveSum(keep, rank, total);
    if (threadIdx.x == 0) base = total ? atomicAdd(ctr + C_WORK, static_cast<unsigned long long>(total)) : 0;
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
  block_add<kRB>(ctr + C_WORK_W, wsum);
}

// --------------------------------------------------------------- Stergiou ---
// minbased.py:251-276: reads only the previous array
__global__ void k_st_init(const int32_t* prev, int32_t* cur, int64_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const int32_t p = prev[v];
    const int32_t pp = prev[p];
    cur[v] = pp < p ? pp : p;
  }
}

__global__ void k_st_edges(Coo c, const int32_t* __restrict__ prev, int32_t* cur) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    const int32_t u = c.u[k], v = c.v[k];
    const int32_t pu = prev[u], pv = prev[v];
    red_min(cur + u, pv);
    red_min(cur + v, pu);
    red_min(cur + pu, pv);
    red_min(cur + pv, pu);
  }
}

__global__ void k_differ(const int32_t* a, const int32_t* b, int64_t n, unsigned long long* changed) {
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    any |= a[v] != b[v];
  if (__syncthreads_or(any) && threadIdx.x == 0) *changed = 1;
}

// ------------------------------------------------------ label propagation ---
// minbased.py:284-304: lower the larger endpoint label of every differing edge
__global__ void k_lp(Coo c, const int32_t* __restrict__ snap, int32_t* L, unsigned long long* changed) {
  bool any = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < c.len; k += stride) {
    const int32_t u = c.u[k], v = c.v[k];
    const int32_t lu = snap[u], lv = snap[v];
    if (lu > lv) red_min(L + u, lv);
    if (lv > lu) red_min(L + v, lu);
    any |= lu != lv;
  }
  if (__syncthreads_or(any) && threadIdx.x == 0) *changed = 1;
}

int grid_e(int64_t work) { return grid_for(work, kRB, 8); }

bool read_flag(unsigned long long* dev, cudaStream_t st) {
  unsigned long long* h = host_words();
  GC_CUDA(cudaMemcpyAsync(h, dev, 8, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  return *h != 0;
}

struct ForestOut {
  const int64_t* off = nullptr;
  const int32_t* tgt = nullptr;
  int32_t* fu = nullptr;
  int32_t* fv = nullptr;
  bool on() const { return fu != nullptr; }
};

// The round loops.  `insp` accumulates the reference's per-round counts.
int64_t loop_rounds(const gc_spec& s, int32_t* P, int64_t nl, Coo& work, RoundsWs& w,
                    unsigned long long* ctr, int64_t& insp, const ForestOut& fo, cudaStream_t st) {
  unsigned long long* flag = ctr + C_CHANGED;
  int64_t rounds = 0;
  const int gv = grid_e(nl);
  if (fo.on()) {
    (k_fill_u64<<<gv, kRB, 0, st>>>(w.win, nl, kNoWin), ::gc::count_launch());
    GC_CHECK_LAUNCH();
  }
  if (s.finish == GC_FINISH_SV) {
    int32_t* A = P;
    int32_t* B = w.b;
    while (true) {
      ++rounds;
      insp += work.weight;
      GC_CUDA(cudaMemcpyAsync(B, A, size_t(nl) * 4, cudaMemcpyDeviceToDevice, st));
      (k_set<<<1, 1, 0, st>>>(flag, 0), ::gc::count_launch());
      if (work.len) (k_sv_hook<<<grid_e(work.len), kRB, 0, st>>>(work, A, B, w.win, flag), ::gc::count_launch());
      if (fo.on() && work.len) {
        (k_sv_win<<<grid_e(work.len), kRB, 0, st>>>(work, A, B, w.win), ::gc::count_launch());
        (k_commit_win<<<gv, kRB, 0, st>>>(w.win, nl, fo.off, fo.tgt, fo.fu, fo.fv), ::gc::count_launch());
      }
      (k_full_shortcut<<<gv, kRB, 0, st>>>(B, nl), ::gc::count_launch());
      GC_CHECK_LAUNCH();
      const bool changed = read_flag(flag, st);
      int32_t* t = A; A = B; B = t;
      if (!changed) break;
    }
    if (A != P) GC_CUDA(cudaMemcpyAsync(P, A, size_t(nl) * 4, cudaMemcpyDeviceToDevice, st));
    return rounds;
  }
  if (s.finish == GC_FINISH_LT) {
    int32_t* msg = w.b;
    Coo* cur = &work;
    Coo* nxt = &w.spare;
    while (true) {
      ++rounds;
      insp += cur->weight;
      GC_CUDA(cudaMemcpyAsync(msg, P, size_t(nl) * 4, cudaMemcpyDeviceToDevice, st));
      (k_set<<<1, 1, 0, st>>>(flag, 0), ::gc::count_launch());
      if (cur->len) (k_lt_connect<<<grid_e(cur->len), kRB, 0, st>>>(*cur, P, msg, s.lt_connect), ::gc::count_launch());
      if (fo.on() && cur->len) {
        (k_lt_win<<<grid_e(cur->len), kRB, 0, st>>>(*cur, P, msg, s.lt_connect, w.win), ::gc::count_launch());
        (k_commit_win<<<gv, kRB, 0, st>>>(w.win, nl, fo.off, fo.tgt, fo.fu, fo.fv), ::gc::count_launch());
      }
      if (s.lt_update == GC_LT_UPDATE_ROOTS) (k_lt_update<<<gv, kRB, 0, st>>>(P, msg, nl), ::gc::count_launch());
      (k_lt_shortcut<<<gv, kRB, 0, st>>>(P, msg, nl, s.lt_shortcut == GC_LT_SHORTCUT_FULL, flag), ::gc::count_launch());
      GC_CHECK_LAUNCH();
      if (s.lt_alter && cur->len) {
        (k_set<<<1, 1, 0, st>>>(ctr + C_WORK, 0), ::gc::count_launch());
        (k_set<<<1, 1, 0, st>>>(ctr + C_WORK_W, 0), ::gc::count_launch());
        (k_lt_alter<<<grid_e(cur->len), kRB, 0, st>>>(*cur, *nxt, P, ctr), ::gc::count_launch());
        GC_CHECK_LAUNCH();
        unsigned long long* h = host_words();
        GC_CUDA(cudaMemcpyAsync(h + 8, ctr + C_CHANGED, 8, cudaMemcpyDeviceToHost, st));
        GC_CUDA(cudaMemcpyAsync(h + 9, ctr + C_WORK, 16, cudaMemcpyDeviceToHost, st));
        GC_CUDA(cudaStreamSynchronize(st));
        nxt->len = int64_t(h[9]);
        nxt->weight = int64_t(h[10]);
        Coo* t = cur; cur = nxt; nxt = t;
        if (h[8] == 0) break;
      } else {
        if (!read_flag(flag, st)) break;
      }
    }
    if (cur != &work) std::swap(work, w.spare);
    return rounds;
  }
  if (s.finish == GC_FINISH_STERGIOU) {
    int32_t* A = P;
    int32_t* B = w.b;
    while (true) {
      ++rounds;
      insp += work.weight;
      (k_set<<<1, 1, 0, st>>>(flag, 0), ::gc::count_launch());
      (k_st_init<<<gv, kRB, 0, st>>>(A, B, nl), ::gc::count_launch());
      if (work.len) (k_st_edges<<<grid_e(work.len), kRB, 0, st>>>(work, A, B), ::gc::count_launch());
      (k_differ<<<gv, kRB, 0, st>>>(A, B, nl, flag), ::gc::count_launch());
      GC_CHECK_LAUNCH();
      const bool changed = read_flag(flag, st);
      int32_t* t = A; A = B; B = t;
      if (!changed) break;
    }
    if (A != P) GC_CUDA(cudaMemcpyAsync(P, A, size_t(nl) * 4, cudaMemcpyDeviceToDevice, st));
    return rounds;
  }
  // label propagation
  int32_t* snap = w.a;
  while (true) {
    ++rounds;
    insp += work.weight;
    GC_CUDA(cudaMemcpyAsync(snap, P, size_t(nl) * 4, cudaMemcpyDeviceToDevice, st));
    (k_set<<<1, 1, 0, st>>>(flag, 0), ::gc::count_launch());
    if (work.len) (k_lp<<<grid_e(work.len), kRB, 0, st>>>(work, snap, P, flag), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    if (!read_flag(flag, st)) break;
  }
  return rounds;
}

}  // namespace

int64_t run_rounds_finish(const gc_csr& g, const gc_spec& s, int32_t* P, const int32_t* list,
                          unsigned long long* ctr, int32_t* fu, int32_t* fv, RoundsWs& w,
                          cudaStream_t st) {
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
  // gather the working COO (driver.py:325-330), twin-deduplicated:
  // per-row kept counts, exclusive scan, then a write pass
  const bool map_labels = s.finish == GC_FINISH_LT || s.finish == GC_FINISH_LP;
  (k_coo_count<<<grid_e(count + 1), kRB, 0, st>>>(g.offsets, g.targets, P, list, count, lmax,
                                                 all_active, w.cnt), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  size_t tb = w.cub_bytes;
  GC_CUDA(cub::DeviceScan::ExclusiveSum(w.cub_tmp, tb, w.cnt, w.pos, int(count + 1), st));
  GC_CUDA(cudaMemcpyAsync(h, w.pos + count, 8, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  Coo& work = w.work;
  work.len = int64_t(h[0]);
  work.weight = degsum;
  Coo out = work;
  if (!fu) out.idx = nullptr;
  (k_coo_write<<<grid_e(count), kRB, 0, st>>>(g.offsets, g.targets, P, list, count, lmax, all_active,
                                             map_labels, w.pos, out), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  work.idx = out.idx;
  if (!fu) w.spare.idx = nullptr;
  int64_t insp = s.finish == GC_FINISH_LP ? 0 : degsum;  // LP does not count the gather
  ForestOut fo;
  if (fu) fo = ForestOut{g.offsets, g.targets, fu, fv};
  const int64_t rounds = loop_rounds(s, P, n, work, w, ctr, insp, fo, st);
  (k_set<<<1, 1, 0, st>>>(ctr + C_INSP_FINISH, static_cast<unsigned long long>(insp)), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  return rounds;
}

size_t rounds_cub_bytes(int64_t n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, static_cast<int64_t*>(nullptr),
                                static_cast<int64_t*>(nullptr), int(n + 1));
  return b;
}

int64_t run_rounds_coo(const gc_spec& s, int32_t* labels, int64_t nl, Coo& work, RoundsWs& w,
                       unsigned long long* ctr, int counter_slot, cudaStream_t st) {
  int64_t insp = 0;
  const int64_t r = loop_rounds(s, labels, nl, work, w, ctr, insp, ForestOut{}, st);
  (k_add<<<1, 1, 0, st>>>(ctr + counter_slot, static_cast<unsigned long long>(insp)), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  return r;
}

}  // namespace gc
