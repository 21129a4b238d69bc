// incremental.cu — batch-incremental connectivity (driver.py:567-725).
//
// A handle owns the live state: a parent array with the sentinel
// convention (slot value `cap` = uninitialised, driver.py:603-614) for the
// union-find rules, or a cap+1 label array for SV / root-based LT
// (driver.py:615-618).  Each batch runs the insert sub-phase (lazy init by
// CAS sentinel->v, then the union kernel), a stream-ordered barrier, and the
// read-only query sub-phase (driver.py:695-708); racy mode interleaves them
// in one launch (driver.py:674-694).
#include <climits>
#include <cstdlib>
#include <cstring>
#include <cub/cub.cuh>

#include "pipeline.cuh"
#include "rounds.h"

struct gc_incr {
  gc_spec spec;
  int64_t cap;
  bool uf;
  int32_t* state = nullptr;   // cap (UF) or cap+1 (rounds) entries
  int32_t* aux = nullptr;     // hooks / locks
  unsigned long long* ctr = nullptr;
  unsigned int* bad = nullptr;  // sticky device flag: an op had an endpoint outside [0, cap)
  // giant filter (union-find rules): bit x set => x is connected to the
  // anchor; gstate[0] = the anchor component's root (-1: none yet),
  // gstate[1] = the anchor moved to another component (clear the bits)
  uint32_t* gbits = nullptr;
  // 32 bytes: [0] anchor, [1] moved flag, [2..3] u64 count of compacted
  // inserts (~0: passed through), [4] compact the next batch (1) or pass it
  // through (0)
  int32_t* gstate = nullptr;
  int32_t* hmode = nullptr;      // mapped pinned copy of gstate[4] (grid choice only)
  int32_t* hmode_dev = nullptr;
  uint8_t* mflag = nullptr;    // insert_list: per-insert "merged two trees" flags
  int64_t mcap = 0;
  int32_t* cu = nullptr;       // the compacted inserts of the current batch
  int32_t* cv = nullptr;
  int64_t ccap = 0;
  // rounds scratch
  gc::RoundsWs rw;
  int64_t coo_cap = 0;
  cudaStream_t st;
  cudaEvent_t ev[4];
};

namespace gc {
namespace {

constexpr int kIB = 256;

// Read-only root chase of every query (driver.py:556-564, 658-668); a warp
// owns 32 consecutive ops and writes their bits as one packed word
// (__ballot_sync, LSB = lowest op index).  Inserts of a mixed batch (isq[i]
// == 0) read as 0.
__global__ void k_incr_query(const int32_t* P, const int32_t* us, const int32_t* vs,
                             const uint8_t* isq, int64_t len, int32_t sentinel, uint32_t* bits,
                             unsigned int* bad, const uint32_t* gbits) {
  const int lane = threadIdx.x & 31;
  const int64_t words = (len + 31) >> 5;
  const int64_t nwarps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  for (int64_t w = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w < words; w += nwarps) {
    const int64_t i = (w << 5) + lane;
    bool hit = false;
    if (i < len && (!isq || isq[i])) {
      int32_t x = us[i], y = vs[i];
      if (uint32_t(x) >= uint32_t(sentinel) || uint32_t(y) >= uint32_t(sentinel)) {
        atomicOr(bad, 1u);
      } else if (gbits && gbit(gbits[x >> 5], x) && gbit(gbits[y >> 5], y)) {
        hit = true;  // both connected to the giant filter's anchor
      } else {
        int32_t px = P[x];
        if (px != sentinel)
          while (px != x) { x = px; px = P[x]; }
        int32_t py = P[y];
        if (py != sentinel)
          while (py != y) { y = py; py = P[y]; }
        hit = x == y;
      }
    }
    const uint32_t word = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) bits[w] = word;
  }
}

// insert COO for the round finishes; LT maps endpoints through the labels
// once up front (minbased.py:176-177)
__global__ void __launch_bounds__(kIB)
k_incr_coo(const int32_t* us, const int32_t* vs, const uint8_t* isq, int64_t len,
           const int32_t* labels, int map, Coo out, unsigned long long* cnt) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (!isq) {  // insert-only batch: entry i is insert i, no compaction
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride) {
      const int32_t u = us[i], v = vs[i];
      out.u[i] = map ? labels[u] : u;
      out.v[i] = map ? labels[v] : v;
      out.w[i] = 1;
    }
    return;
  }
  // mixed batch: inserts compacted in order within a block, one counter
  // atomic per block step (a per-warp atomic on the one counter serialised)
  using Scan = cub::BlockScan<int, kIB>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ unsigned long long bpos;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < len; base += stride) {
    const int64_t i = base + threadIdx.x;
    const int ins = i < len && !isq[i];
    int rank, total;
    Scan(tmp).ExclusiveSum(ins, rank, total);
    if (threadIdx.x == 0) bpos = total ? atomicAdd(cnt, static_cast<unsigned long long>(total)) : 0ull;
    __syncthreads();
    if (ins) {
      const unsigned long long p = bpos + rank;
      const int32_t u = us[i], v = vs[i];
      out.u[p] = map ? labels[u] : u;
      out.v[p] = map ? labels[v] : v;
      out.w[p] = 1;
    }
    __syncthreads();
  }
}

// lazily initialise fresh endpoints of a label array (driver.py:639-641)
__global__ void k_label_init(int32_t* L, const int32_t* us, const int32_t* vs, const uint8_t* isq,
                             int64_t len, int32_t sentinel) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride) {
    if (isq && isq[i]) continue;
    const int32_t u = us[i], v = vs[i];  // range-checked before the launch
    if (L[u] == sentinel) L[u] = u;
    if (L[v] == sentinel) L[v] = v;
  }
}

__global__ void k_incr_export(const int32_t* S, int64_t cap, int32_t sentinel, int32_t* out) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < cap; v += stride) {
    const int32_t s = S[v];
    out[v] = s == sentinel ? int32_t(v) : s;
  }
}

__global__ void k_incr_count(const int32_t* S, const int32_t* fin, int64_t cap, int32_t sentinel,
                             unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < cap; v += stride)
    c += S[v] != sentinel && fin[v] == v;
  block_add<kIB>(out, c);
}

int g1(int64_t work) { return grid_for(work, kIB, 8); }

// Giant filter upkeep, after every union-find insert sub-phase.  One block
// samples 1024 evenly spaced slots, chases their roots and takes the most
// frequent one (warp-aggregated shared-memory hash, as k_mode_probe).  The
// anchor is re-resolved to its component's current root; it moves to the
// sampled mode only when that component clearly dominates (then the bits,
// which mean "connected to the old anchor", are cleared by the same block).
// Roots of the min-linking rules are component minima, so once the giant
// has formed its root — the anchor — stays put.
__global__ void __launch_bounds__(1024) k_giant_probe(const int32_t* P, int64_t cap, int32_t sentinel,
                                                      int32_t* gstate, volatile int32_t* hmode,
                                                      uint32_t* bits, int64_t words) {
  constexpr int kS = 1024, kSlots = 2 * kS;
  __shared__ int32_t key_[kSlots];
  __shared__ unsigned cnt_[kSlots];
  __shared__ unsigned long long best;
  const int i = threadIdx.x;
  for (int k = i; k < kSlots; k += kS) {
    key_[k] = -1;
    cnt_[k] = 0;
  }
  if (i == 0) best = 0ull;
  const int s = cap < kS ? int(cap) : kS;
  int32_t x = -1;
  if (i < s) {
    x = int32_t((int64_t(i) * cap) / s);
    int32_t p = ld_acq(P + x);
    if (p == sentinel) {
      x = -1;
    } else {
      while (p != x) {
        x = p;
        p = ld_acq(P + x);
      }
    }
  }
  __syncthreads();
  auto slot_of = [](int32_t v) { return int((uint32_t(v) * 2654435761u) >> (32 - 11)); };
  int slot = -1;
  if (x >= 0) {
    const unsigned same = __match_any_sync(__activemask(), x);
    slot = slot_of(x);
    while (true) {
      const int32_t k = atomicCAS(&key_[slot], -1, x);
      if (k == -1 || k == x) break;
      slot = (slot + 1) % kSlots;
    }
    if ((i & 31) == __ffs(int(same)) - 1) atomicAdd(&cnt_[slot], __popc(same));
  }
  __syncthreads();
  if (x >= 0)
    atomicMax(&best, (static_cast<unsigned long long>(cnt_[slot]) << 32) | (0xffffffffull - uint32_t(x)));
  __syncthreads();
  __shared__ int clear;
  if (i == 0) {
    int32_t cur = gstate[0];
    if (cur >= 0) {
      int32_t p = ld_acq(P + cur);
      while (p != cur) {
        cur = p;
        p = ld_acq(P + cur);
      }
    }
    const unsigned cm = unsigned(best >> 32);
    const int32_t m = int32_t(0xffffffffull - (best & 0xffffffffull));
    unsigned cc = 0;
    if (cur >= 0)
      for (int k = slot_of(cur), t = 0; t < kSlots && key_[k] != -1; k = (k + 1) % kSlots, ++t)
        if (key_[k] == cur) {
          cc = cnt_[k];
          break;
        }
    const bool move = cm > 0 && m != cur && (cur < 0 || cm >= 2 * cc + 8);
    gstate[0] = move ? m : cur;
    gstate[1] = move && cur >= 0;
    *reinterpret_cast<unsigned long long*>(gstate + 2) = 0ull;  // the next batch's compaction count
    // compacting costs one pass over the batch plus two bit tests per insert;
    // it pays once about half of the inserts can be dropped (config 4: from
    // the ~12th of 54 batches on)
    if (move) gstate[4] = 0;  // the bits were cleared: pass the next batch through
    if (hmode) *hmode = gstate[4];
    clear = move && cur >= 0;
  }
  __syncthreads();
  // the anchor moved off an old one (rare: the giant overtakes an earlier
  // mode): its bits, which meant "connected to the old anchor", are cleared
  // by this block instead of a separate launch per batch
  if (clear)
    for (int64_t w = i; w < words; w += kS) bits[w] = 0u;
}

// Whether this batch is worth compacting: one block tests the giant bits of
// 1024 evenly spaced inserts of the batch itself.  Compacting costs a pass
// over the batch plus two bit tests per insert (~0.1 ms per 10M) and pays
// once about two thirds of the inserts can be dropped (RMAT s26, 10M
// batches: from about the 12th batch on).
__global__ void __launch_bounds__(1024)
k_giant_decide(const int32_t* us, const int32_t* vs, const uint8_t* isq, int64_t len, int32_t cap,
               const uint32_t* gbits, int32_t* gstate, bool gkeep) {
  __shared__ unsigned both, seen;
  if (threadIdx.x == 0) both = seen = 0u;
  __syncthreads();
  const int32_t anc = gstate[0];
  const int ns = len < 1024 ? int(len) : 1024;
  if (anc >= 0 && int(threadIdx.x) < ns) {
    const int64_t j = (int64_t(threadIdx.x) * len) / ns;
    if (!(isq && isq[j])) {
      const int32_t a = us[j], b = vs[j];
      if (uint32_t(a) < uint32_t(cap) && uint32_t(b) < uint32_t(cap)) {
        atomicAdd(&seen, 1u);
        const uint64_t bpol = bits_policy(gkeep);
        if (gbit(ld_bits(gbits + (a >> 5), bpol), a) && gbit(ld_bits(gbits + (b >> 5), bpol), b)) atomicAdd(&both, 1u);
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) gstate[4] = anc >= 0 && seen > 0 && 3 * both >= 2 * seen;
}

// Giant filter, first step of a union-find insert sub-phase: inserts whose
// two endpoints are both marked as connected to the anchor cannot change
// the partition and are dropped (two bit tests against a cap/8-byte bitmap
// that stays in L2, instead of two random parent reads in a cap*4-byte
// array that does not); the rest — and every insert while no anchor is set
// — are compacted for the union kernel.  A block owns a contiguous chunk
// of the batch, each thread four consecutive inserts per step (16-byte
// loads), survivors are staged in a shared-memory queue that is flushed
// with one counter atomic once half full.  Queries of a mixed batch are
// dropped here too; malformed endpoints set the sticky flag.
constexpr int kGcQ = 2048;
__global__ void __launch_bounds__(kIB)
k_giant_compact(const int32_t* __restrict__ us, const int32_t* __restrict__ vs, const uint8_t* __restrict__ isq,
                int64_t len, int32_t cap, const uint32_t* __restrict__ gbits, int32_t* gstate, int32_t* ou,
                int32_t* ov, unsigned int* bad, bool gkeep) {
  constexpr int kStep = kIB * 4;
  __shared__ int2 q[kGcQ];
  __shared__ int qn;
  __shared__ unsigned long long qbase;
  unsigned long long* ocount = reinterpret_cast<unsigned long long*>(gstate + 2);
  const int32_t anc = gstate[0];
  const bool on = anc >= 0;
  // the anchor is connected to itself: its bit seeds the marking (the other
  // blocks may test it before it lands, which only keeps an insert)
  if (on && blockIdx.x == 0 && threadIdx.x == 0)
    red_or_bits(const_cast<uint32_t*>(gbits) + (anc >> 5), 1u << (anc & 31), bits_policy(gkeep));
  if (!on || !gstate[4]) {  // pass the batch through: the union reads the caller's arrays
    if (blockIdx.x == 0 && threadIdx.x == 0) *reinterpret_cast<unsigned long long*>(gstate + 2) = ~0ull;
    return;
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(us) | reinterpret_cast<uintptr_t>(vs)) & 15) == 0;
  if (threadIdx.x == 0) qn = 0;
  const int64_t per = ((len + gridDim.x - 1) / gridDim.x + kStep - 1) / kStep * kStep;
  const int64_t lo = int64_t(blockIdx.x) * per;
  const int64_t hi = lo + per < len ? lo + per : len;
  const int lane = threadIdx.x & 31;
  auto flush = [&]() {
    __syncthreads();
    const int c = qn;
    if (threadIdx.x == 0) qbase = c ? atomicAdd(ocount, static_cast<unsigned long long>(c)) : 0ull;
    __syncthreads();
    for (int k = threadIdx.x; k < c; k += kIB) {
      ou[qbase + k] = q[k].x;
      ov[qbase + k] = q[k].y;
    }
    __syncthreads();
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
  };
  __syncthreads();
  for (int64_t b = lo; b < hi; b += kStep) {
    const int64_t i0 = b + 4 * int64_t(threadIdx.x);
    int32_t u[4] = {0, 0, 0, 0}, v[4] = {0, 0, 0, 0};
    bool keep[4] = {false, false, false, false};
    if (vec && i0 + 3 < hi) {
      const int4 a = __ldg(reinterpret_cast<const int4*>(us + i0));
      const int4 c = __ldg(reinterpret_cast<const int4*>(vs + i0));
      u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w;
      v[0] = c.x; v[1] = c.y; v[2] = c.z; v[3] = c.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) keep[j] = true;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (i0 + j < hi) {
          u[j] = __ldg(us + i0 + j);
          v[j] = __ldg(vs + i0 + j);
          keep[j] = true;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (!keep[j]) continue;
      if (isq && isq[i0 + j]) keep[j] = false;
      else if (uint32_t(u[j]) >= uint32_t(cap) || uint32_t(v[j]) >= uint32_t(cap)) {
        atomicOr(bad, 1u);
        keep[j] = false;
      }
    }
    if (on) {
      uint32_t wu[4], wv[4];
      const uint64_t bpol = bits_policy(gkeep);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        wu[j] = keep[j] ? ld_bits_nc(gbits + (u[j] >> 5), bpol) : 0u;
        wv[j] = keep[j] ? ld_bits_nc(gbits + (v[j] >> 5), bpol) : 0u;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const bool bu = gbit(wu[j], u[j]), bv = gbit(wv[j], v[j]);
        if (bu && bv) keep[j] = false;
        // survivors carry "bit already set" in bit 31 (the union marks
        // only the endpoints that lack it)
        u[j] |= bu ? int32_t(0x80000000u) : 0;
        v[j] |= bv ? int32_t(0x80000000u) : 0;
      }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const unsigned bal = __ballot_sync(0xffffffffu, keep[j]);
      if (!bal) continue;
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&qn, __popc(bal));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(bal & ((1u << lane) - 1u));
      if (keep[j]) q[pos] = make_int2(u[j], v[j]);
    }
    __syncthreads();
    if (qn >= kGcQ / 2) flush();  // a step adds at most kStep = kGcQ / 2
  }
  flush();
}

// insert_list with the lock-step async kernel: the kernel flags merging
// inserts by index; this pass gathers their (u, v) from the array the
// kernel walked (the giant compaction's survivors, or the caller's batch
// when it was passed through / the filter is off), one counter atomic per
// block flush
__global__ void __launch_bounds__(kIB)
k_merge_compact(const int32_t* __restrict__ cu, const int32_t* __restrict__ cv, const int32_t* __restrict__ us,
                const int32_t* __restrict__ vs, int64_t len, const unsigned long long* kdev,
                const uint8_t* __restrict__ flags, int32_t* ou, int32_t* ov, unsigned long long* ocount) {
  __shared__ int2 q[kGcQ];
  __shared__ int qn;
  __shared__ unsigned long long qbase;
  const unsigned long long c = kdev ? *kdev : ~0ull;
  const bool compacted = c != ~0ull;
  const int64_t k = compacted ? int64_t(c) : len;
  const int32_t* a = compacted ? cu : us;
  const int32_t* b = compacted ? cv : vs;
  if (threadIdx.x == 0) qn = 0;
  const int lane = threadIdx.x & 31;
  const int64_t per = ((k + gridDim.x - 1) / gridDim.x + kIB - 1) / kIB * kIB;
  const int64_t lo = int64_t(blockIdx.x) * per;
  const int64_t hi = lo + per < k ? lo + per : k;
  auto flush = [&]() {
    __syncthreads();
    const int n = qn;
    if (threadIdx.x == 0) qbase = n ? atomicAdd(ocount, static_cast<unsigned long long>(n)) : 0ull;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += kIB) {
      ou[qbase + i] = q[i].x;
      ov[qbase + i] = q[i].y;
    }
    __syncthreads();
    if (threadIdx.x == 0) qn = 0;
    __syncthreads();
  };
  __syncthreads();
  for (int64_t i0 = lo; i0 < hi; i0 += kIB) {
    const int64_t i = i0 + threadIdx.x;
    const bool m = i < hi && flags[i];
    const unsigned bal = __ballot_sync(0xffffffffu, m);
    if (bal) {
      int pos = 0;
      if (lane == 0) pos = atomicAdd(&qn, __popc(bal));
      pos = __shfl_sync(0xffffffffu, pos, 0) + __popc(bal & ((1u << lane) - 1u));
      if (m) q[pos] = make_int2(a[i] & 0x7fffffff, b[i] & 0x7fffffff);
    }
    __syncthreads();
    if (qn > kGcQ - kIB) flush();
  }
  flush();
}

// GC_INCR_GIANT=0 turns the filter off (every insert runs its union)
bool giant_filter_on() {
  static const bool on = [] {
    const char* e = getenv("GC_INCR_GIANT");
    return !(e && e[0] == '0');
  }();
  return on;
}

// compacts the batch into h->cu / h->cv and points the union at it (count
// on the device); the caller runs giant_after once the union is enqueued
// per-insert merge flags of insert_list (lock-step async kernel)
void flags_reserve(gc_incr* h, int64_t len) {
  if (len <= h->mcap) return;
  if (h->mflag) cudaFree(h->mflag);
  h->mflag = nullptr;
  h->mcap = 0;
  GC_CUDA(cudaMalloc(&h->mflag, len));
  h->mcap = len;
}

void giant_reserve(gc_incr* h, int64_t len) {
  if (!h->gbits || len <= h->ccap) return;
  if (h->cu) cudaFree(h->cu);
  if (h->cv) cudaFree(h->cv);
  h->cu = h->cv = nullptr;
  h->ccap = 0;
  GC_CUDA(cudaMalloc(&h->cu, len * 4));
  GC_CUDA(cudaMalloc(&h->cv, len * 4));
  h->ccap = len;
}

void giant_compact(gc_incr* h, CooUnionArgs& a, const uint8_t* isq) {
  if (!h->gbits || a.k <= 0) return;
  giant_reserve(h, a.k);
  static const int per_sm = [] {
    int b = 0;
    GC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k_giant_compact, kIB, 0));
    return b > 0 ? b : 1;
  }();
  int64_t blocks = (a.k + 4 * kIB - 1) / (4 * kIB);
  if (blocks > int64_t(num_sms()) * per_sm) blocks = int64_t(num_sms()) * per_sm;
  (k_giant_decide<<<1, 1024, 0, h->st>>>(a.us, a.vs, isq, a.k, int32_t(h->cap), h->gbits, h->gstate,
                                              giant_keep()),
   ::gc::count_launch());
  (k_giant_compact<<<int(blocks), kIB, 0, h->st>>>(a.us, a.vs, isq, a.k, int32_t(h->cap),
                                                                      h->gbits, h->gstate, h->cu, h->cv, h->bad,
                                                                      giant_keep()),
   ::gc::count_launch());
  GC_CHECK_LAUNCH();
  a.alt.us = a.us;
  a.alt.vs = a.vs;
  a.alt.skip = a.skip;
  a.alt.k = a.k;
  a.us = h->cu;
  a.vs = h->cv;
  a.skip = nullptr;
  a.kdev = reinterpret_cast<const unsigned long long*>(h->gstate + 2);
  a.kdev_wave = h->hmode && *reinterpret_cast<volatile int32_t*>(h->hmode) != 0;
}

void giant_after(gc_incr* h) {
  if (!h->gbits) return;
  const int64_t words = (h->cap + 31) / 32;
  (k_giant_probe<<<1, 1024, 0, h->st>>>(h->state, h->cap, int32_t(h->cap), h->gstate, h->hmode_dev, h->gbits,
                                        words),
   ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

__global__ void k_count_bytes(const uint8_t* a, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) c += a[i] != 0;
  block_add<kIB>(out, c);
}

void ensure_coo(gc_incr* h, int64_t len) {
  if (len <= h->coo_cap) return;
  int64_t cap = len < 1024 ? 1024 : len;
  for (Coo* c : {&h->rw.work, &h->rw.spare}) {
    cudaFree(c->u);
    cudaFree(c->v);
    cudaFree(c->w);
    c->u = c->v = nullptr;
    c->w = nullptr;
    GC_CUDA(cudaMalloc(&c->u, cap * 4));
    GC_CUDA(cudaMalloc(&c->v, cap * 4));
    GC_CUDA(cudaMalloc(&c->w, cap));
    c->idx = nullptr;
  }
  cudaFree(h->rw.keep);
  h->rw.keep = nullptr;
  GC_CUDA(cudaMalloc(&h->rw.keep, cap));
  if (!h->rw.chunks) GC_CUDA(cudaMalloc(&h->rw.chunks, (2 * kMaxChunks + 4) * sizeof(int64_t)));
  h->coo_cap = cap;
}

double elapsed(cudaEvent_t a, cudaEvent_t b) {
  float t = 0;
  GC_CUDA(cudaEventElapsedTime(&t, a, b));
  return t;
}

CooUnionArgs uf_args(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len,
                     const uint8_t* skip) {
  CooUnionArgs a{};
  a.P = h->state;
  a.H = h->spec.finish == GC_FINISH_HOOKS ? h->aux : nullptr;
  a.L = h->spec.finish == GC_FINISH_REM_LOCK ? h->aux : nullptr;
  a.R = h->spec.jtb_ranks;
  a.n = int32_t(h->cap);
  a.us = us;
  a.vs = vs;
  a.k = len;
  a.skip = skip;
  a.bad = h->bad;
  a.gbits = h->gbits;
  a.ganchor = h->gstate;
  return a;
}

// The sticky input flag: kernels skip ops with an endpoint outside
// [0, cap) and set h->bad; every synchronising entry point reads it with its
// own completion sync (fetch before, raise after) and reports
// GC_ERR_MALFORMED once, then clears it.
unsigned int* bad_word() { return reinterpret_cast<unsigned int*>(pinned_words() + 32); }
void fetch_bad(gc_incr* h) {
  GC_CUDA(cudaMemcpyAsync(bad_word(), h->bad, 4, cudaMemcpyDeviceToHost, h->st));
}
void raise_bad(gc_incr* h) {
  unsigned int* w = bad_word();
  if (*w) {
    *w = 0;
    GC_CUDA(cudaMemsetAsync(h->bad, 0, 4, h->st));
    throw Error(GC_ERR_MALFORMED, "an op endpoint lies outside [0, capacity) (op skipped)");
  }
}

// insert sub-phase; returns added inspections (driver.py:627-649)
void insert_phase(gc_incr* h, const int32_t* us, const int32_t* vs, const uint8_t* isq, int64_t len,
                  int64_t n_ins, gc_stats* stats) {
  cudaStream_t st = h->st;
  const int32_t sentinel = int32_t(h->cap);
  if (h->uf) {
    CooUnionArgs a = uf_args(h, us, vs, len, isq);
    // lazy init fused into the union launch (measured +44% inserts/s at
    // RMAT s26 over a separate init pass)
    a.init_sentinel = sentinel;
    giant_compact(h, a, isq);
    launch_union_coo(UFConfig{h->spec.finish, h->spec.find, h->spec.splice}, false, a, st);
    giant_after(h);
    if (stats) stats->insp_finish += n_ins;
    return;
  }
  // the label-array kernels index with the endpoints directly
  check_ids(us, len, h->cap, st, "op endpoint");
  check_ids(vs, len, h->cap, st, "op endpoint");
  ensure_coo(h, len);
  (k_label_init<<<g1(len), kIB, 0, st>>>(h->state, us, vs, isq, len, sentinel), ::gc::count_launch());
  unsigned long long* cnt = h->ctr + C_SCRATCH0;
  GC_CUDA(cudaMemsetAsync(cnt, 0, 8, st));
  Coo w = h->rw.work;
  (k_incr_coo<<<g1(len), kIB, 0, st>>>(us, vs, isq, len, h->state, h->spec.finish == GC_FINISH_LT,
                                      w, cnt), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  h->rw.work.len = n_ins;
  h->rw.work.weight = n_ins;
  GC_CUDA(cudaMemsetAsync(h->ctr + C_INSP_FINISH, 0, 8, st));
  const int64_t r = run_rounds_coo(h->spec, h->state, h->cap + 1, h->rw.work, h->rw, h->ctr,
                                   C_INSP_FINISH, st);
  unsigned long long* hw = pinned_words();
  GC_CUDA(cudaMemcpyAsync(hw, h->ctr + C_INSP_FINISH, 8, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  if (stats) {
    stats->rounds += r;
    stats->insp_finish += n_ins + int64_t(hw[0]);
  }
}

int64_t count_inserts(const uint8_t* isq, int64_t len, cudaStream_t st, unsigned long long* ctr) {
  if (!isq) return len;
  unsigned long long* c = ctr + C_SCRATCH1;
  GC_CUDA(cudaMemsetAsync(c, 0, 8, st));
  (k_count_bytes<<<g1(len), kIB, 0, st>>>(isq, len, c), ::gc::count_launch());
  GC_CHECK_LAUNCH();
  unsigned long long* hw = pinned_words();
  GC_CUDA(cudaMemcpyAsync(hw, c, 8, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  return len - int64_t(hw[0]);
}

}  // namespace

}  // namespace gc

using namespace gc;

extern "C" {

int gc_incr_create(int64_t capacity, const gc_spec* spec, void* stream, gc_incr** out) {
  return guarded([&] {
    require(spec && out, GC_ERR_ARG, "null argument");
    require(capacity >= 0 && capacity < (int64_t(1) << 31) - 1, GC_ERR_MALFORMED,
            "capacity outside [0, 2^31 - 1)");
    const bool uf = spec->finish >= GC_FINISH_ASYNC && spec->finish <= GC_FINISH_JTB;
    const bool ok = uf || spec->finish == GC_FINISH_SV ||
                    (spec->finish == GC_FINISH_LT && spec->lt_update == GC_LT_UPDATE_ROOTS);
    require(ok, GC_ERR_CONFIG, "incremental needs a root-based finish");
    if (uf) require(valid_uf(UFConfig{spec->finish, spec->find, spec->splice}), GC_ERR_CONFIG,
                    "unsupported union-find combination");
    require(spec->finish != GC_FINISH_JTB || spec->jtb_ranks, GC_ERR_ARG, "JTB needs ranks");
    gc_incr* h = new gc_incr();
    h->spec = *spec;
    h->cap = capacity;
    h->uf = uf;
    h->st = static_cast<cudaStream_t>(stream);
    try {
      const int64_t slots = uf ? capacity : capacity + 1;
      GC_CUDA(cudaMalloc(&h->state, (slots > 0 ? slots : 1) * 4));
      GC_CUDA(cudaMalloc(&h->ctr, sizeof(unsigned long long) * C_COUNT_));
      GC_CUDA(cudaMalloc(&h->bad, 16));
      GC_CUDA(cudaMemsetAsync(h->ctr, 0, sizeof(unsigned long long) * C_COUNT_, h->st));
      GC_CUDA(cudaMemsetAsync(h->bad, 0, 16, h->st));
      fill(h->state, slots, int32_t(capacity), h->st);  // every slot = sentinel
      if (spec->finish == GC_FINISH_HOOKS || spec->finish == GC_FINISH_REM_LOCK) {
        GC_CUDA(cudaMalloc(&h->aux, (capacity > 0 ? capacity : 1) * 4));
        fill(h->aux, capacity, spec->finish == GC_FINISH_HOOKS ? int32_t(capacity) : 0, h->st);
      }
      // the giant filter: union-find rules whose roots are component minima
      if (uf && spec->finish != GC_FINISH_JTB && capacity > 0 && giant_filter_on()) {
        const int64_t words = (capacity + 31) / 32;
        GC_CUDA(cudaMalloc(&h->gbits, words * 4));
        GC_CUDA(cudaMalloc(&h->gstate, 32));
        GC_CUDA(cudaMemsetAsync(h->gbits, 0, words * 4, h->st));
        GC_CUDA(cudaMemsetAsync(h->gstate, 0xff, 4, h->st));  // no anchor yet
        GC_CUDA(cudaMemsetAsync(h->gstate + 1, 0, 28, h->st));
        GC_CUDA(cudaHostAlloc(&h->hmode, 4, cudaHostAllocMapped));
        *h->hmode = 0;
        GC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h->hmode_dev), h->hmode, 0));
      }
      if (!uf) {
        GC_CUDA(cudaMalloc(&h->rw.a, (capacity + 1) * 4));
        GC_CUDA(cudaMalloc(&h->rw.b, (capacity + 1) * 4));
      }
      for (auto& e : h->ev) GC_CUDA(cudaEventCreate(&e));
      GC_CUDA(cudaStreamSynchronize(h->st));
    } catch (...) {
      gc_incr_destroy(h);
      throw;
    }
    *out = h;
  });
}

void gc_incr_destroy(gc_incr* h) {
  if (!h) return;
  cudaFree(h->state);
  cudaFree(h->aux);
  cudaFree(h->ctr);
  cudaFree(h->bad);
  cudaFree(h->gbits);
  cudaFree(h->gstate);
  cudaFree(h->cu);
  cudaFree(h->cv);
  if (h->hmode) cudaFreeHost(h->hmode);
  cudaFree(h->mflag);
  cudaFree(h->rw.a);
  cudaFree(h->rw.b);
  for (Coo* c : {&h->rw.work, &h->rw.spare}) {
    cudaFree(c->u);
    cudaFree(c->v);
    cudaFree(c->w);
  }
  cudaFree(h->rw.keep);
  cudaFree(h->rw.chunks);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  delete h;
}

int64_t gc_incr_capacity(gc_incr* h) { return h ? h->cap : -1; }

int gc_incr_set_stream(gc_incr* h, void* stream) {
  return guarded([&] {
    require(h != nullptr, GC_ERR_ARG, "null handle");
    cudaStream_t ns = static_cast<cudaStream_t>(stream);
    if (ns == h->st) return;
    // everything enqueued on the old stream happens before later work on
    // the new one
    GC_CUDA(cudaEventRecord(h->ev[3], h->st));
    GC_CUDA(cudaStreamWaitEvent(ns, h->ev[3], 0));
    h->st = ns;
  });
}

int gc_incr_reserve(gc_incr* h, int64_t batch_len) {
  return guarded([&] {
    require(h != nullptr && batch_len >= 0, GC_ERR_ARG, "bad reserve");
    if (!h->uf && batch_len > 0) ensure_coo(h, batch_len);
    if (h->uf && batch_len > 0) {
      giant_reserve(h, batch_len);
      if (h->spec.finish == GC_FINISH_ASYNC && h->spec.find != GC_FIND_COMPRESS && coo_mlp() > 0)
        flags_reserve(h, batch_len);
    }
  });
}

int gc_incr_batch(gc_incr* h, const int32_t* us, const int32_t* vs, const uint8_t* is_query,
                  int64_t len, uint32_t* bits_out, int racy, gc_stats* stats) {
  return guarded([&] {
    require(h && len >= 0, GC_ERR_ARG, "bad arguments");
    if (len == 0) return;
    require(us && vs && bits_out, GC_ERR_ARG, "null batch arrays");
    cudaStream_t st = h->st;
    const int32_t sentinel = int32_t(h->cap);
    if (racy) {
      require(h->uf, GC_ERR_CONFIG, "racy mode interleaves single ops and only works with union-find finishes");
      require(h->spec.splice != GC_SPLICE_ATOMIC, GC_ERR_CONFIG,
              "the splice rule moves non-roots across trees mid-union: use batched mode");
      const int64_t n_ins = count_inserts(is_query, len, st, h->ctr);
      GC_CUDA(cudaEventRecord(h->ev[0], st));
      launch_incr_racy(UFConfig{h->spec.finish, h->spec.find, h->spec.splice},
                       uf_args(h, us, vs, len, nullptr), is_query, sentinel, bits_out, st);
      GC_CUDA(cudaEventRecord(h->ev[1], st));
      fetch_bad(h);
      GC_CUDA(cudaStreamSynchronize(st));
      raise_bad(h);
      if (stats) {
        stats->t_sample_ms += elapsed(h->ev[0], h->ev[1]);
        stats->insp_finish += n_ins;
      }
      return;
    }
    const int64_t n_ins = count_inserts(is_query, len, st, h->ctr);
    GC_CUDA(cudaEventRecord(h->ev[0], st));
    if (n_ins) insert_phase(h, us, vs, is_query, len, n_ins, stats);
    GC_CUDA(cudaEventRecord(h->ev[1], st));
    (k_incr_query<<<g1(len), kIB, 0, st>>>(h->state, us, vs, is_query, len, sentinel, bits_out, h->bad,
                                          h->gbits), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaEventRecord(h->ev[2], st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(st));
    raise_bad(h);
    if (stats) {
      stats->t_sample_ms += elapsed(h->ev[0], h->ev[1]);
      stats->t_finish_ms += elapsed(h->ev[1], h->ev[2]);
    }
  });
}

int gc_incr_insert(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len, gc_stats* stats) {
  return guarded([&] {
    require(h && len >= 0, GC_ERR_ARG, "bad arguments");
    if (len == 0) return;
    require(us && vs, GC_ERR_ARG, "null batch arrays");
    GC_CUDA(cudaEventRecord(h->ev[0], h->st));
    insert_phase(h, us, vs, nullptr, len, len, stats);
    GC_CUDA(cudaEventRecord(h->ev[1], h->st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(h->st));
    raise_bad(h);
    if (stats) stats->t_sample_ms += elapsed(h->ev[0], h->ev[1]);
  });
}

int gc_incr_insert_async(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len, gc_stats* stats) {
  return guarded([&] {
    require(h && len >= 0, GC_ERR_ARG, "bad arguments");
    if (len == 0) return;
    require(us && vs, GC_ERR_ARG, "null batch arrays");
    if (!h->uf) {  // the round finishes synchronise inside every batch anyway
      GC_CUDA(cudaEventRecord(h->ev[0], h->st));
      insert_phase(h, us, vs, nullptr, len, len, stats);
      GC_CUDA(cudaEventRecord(h->ev[1], h->st));
      fetch_bad(h);
      GC_CUDA(cudaStreamSynchronize(h->st));
      raise_bad(h);
      if (stats) stats->t_sample_ms += elapsed(h->ev[0], h->ev[1]);
      return;
    }
    // union-find inserts: enqueue and return (the stream orders batches;
    // queries, labels and the state copy synchronise and report a malformed
    // endpoint seen by any earlier batch); no per-batch timing
    insert_phase(h, us, vs, nullptr, len, len, stats);
  });
}

int gc_incr_insert_list(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len, int32_t* out_u,
                        int32_t* out_v, unsigned long long* out_count, gc_stats* stats) {
  return guarded([&] {
    require(h && len >= 0 && out_u && out_v && out_count, GC_ERR_ARG, "bad arguments");
    require(h->uf && h->spec.splice != GC_SPLICE_ATOMIC, GC_ERR_CONFIG,
            "recording merging edges needs a root-based union-find rule");
    if (len == 0) return;
    require(us && vs, GC_ERR_ARG, "null batch arrays");
    cudaStream_t st = h->st;
    GC_CUDA(cudaEventRecord(h->ev[0], st));
    CooUnionArgs a = uf_args(h, us, vs, len, nullptr);
    a.init_sentinel = int32_t(h->cap);
    a.lu = out_u;
    a.lv = out_v;
    a.lcount = out_count;
    // the lock-step async kernel flags merging inserts by index (a shared
    // append counter serialised the early batches, where ~every insert
    // merges: RMAT s26 batch 1, 1.73 ms vs 0.60 for a plain insert)
    const bool flagged = h->spec.finish == GC_FINISH_ASYNC && h->spec.find != GC_FIND_COMPRESS && coo_mlp() > 0;
    if (flagged) {
      flags_reserve(h, len);
      GC_CUDA(cudaMemsetAsync(h->mflag, 0, len, st));
      a.lu = a.lv = nullptr;
      a.lcount = nullptr;
      a.lflag = h->mflag;
    }
    giant_compact(h, a, nullptr);
    launch_union_coo(UFConfig{h->spec.finish, h->spec.find, h->spec.splice}, false, a, st);
    if (flagged) {
      GC_CUDA(cudaMemsetAsync(out_count, 0, 8, st));
      (k_merge_compact<<<num_sms() * 4, kIB, 0, st>>>(h->cu, h->cv, us, vs, len, a.kdev, h->mflag, out_u, out_v,
                                                      out_count), ::gc::count_launch());
      GC_CHECK_LAUNCH();
    }
    giant_after(h);
    GC_CUDA(cudaEventRecord(h->ev[1], st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(st));
    raise_bad(h);
    if (stats) {
      stats->t_sample_ms += elapsed(h->ev[0], h->ev[1]);
      stats->insp_finish += len;
    }
  });
}

int gc_incr_query(gc_incr* h, const int32_t* us, const int32_t* vs, int64_t len, uint32_t* bits_out,
                  gc_stats* stats) {
  return guarded([&] {
    require(h && len >= 0, GC_ERR_ARG, "bad arguments");
    if (len == 0) return;
    require(us && vs && bits_out, GC_ERR_ARG, "null batch arrays");
    GC_CUDA(cudaEventRecord(h->ev[0], h->st));
    (k_incr_query<<<g1(len), kIB, 0, h->st>>>(h->state, us, vs, nullptr, len, int32_t(h->cap), bits_out,
                                             h->bad, h->gbits), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaEventRecord(h->ev[1], h->st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(h->st));
    raise_bad(h);
    if (stats) stats->t_finish_ms += elapsed(h->ev[0], h->ev[1]);
  });
}

int gc_incr_state(gc_incr* h, int32_t* state_out) {
  return guarded([&] {
    require(h && state_out, GC_ERR_ARG, "bad arguments");
    const int64_t slots = h->uf ? h->cap : h->cap + 1;
    if (slots > 0)
      GC_CUDA(cudaMemcpyAsync(state_out, h->state, slots * 4, cudaMemcpyDeviceToDevice, h->st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(h->st));
    raise_bad(h);
  });
}

int gc_incr_state_view(gc_incr* h, int32_t** state, int64_t* slots) {
  return guarded([&] {
    require(h && state && slots, GC_ERR_ARG, "bad arguments");
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(h->st));
    raise_bad(h);
    *state = h->state;
    *slots = h->uf ? h->cap : h->cap + 1;
  });
}

int gc_incr_labels(gc_incr* h, int32_t* labels_out, int64_t* components) {
  return guarded([&] {
    require(h && components, GC_ERR_ARG, "bad arguments");
    *components = 0;
    const int64_t cap = h->cap;
    if (cap == 0) return;
    require(labels_out, GC_ERR_ARG, "null labels");
    cudaStream_t st = h->st;
    int32_t* mins = nullptr;
    GC_CUDA(cudaMallocAsync(&mins, cap * 4, st));
    GC_CUDA(cudaMemsetAsync(h->ctr, 0, sizeof(unsigned long long) * C_COUNT_, st));
    (k_incr_export<<<g1(cap), kIB, 0, st>>>(h->state, cap, int32_t(cap), labels_out), ::gc::count_launch());
    run_finalize(labels_out, int32_t(cap), mins, h->ctr, st);
    GC_CUDA(cudaMemsetAsync(h->ctr + C_SCRATCH0, 0, 8, st));
    (k_incr_count<<<g1(cap), kIB, 0, st>>>(h->state, labels_out, cap, int32_t(cap), h->ctr + C_SCRATCH0), ::gc::count_launch());
    GC_CHECK_LAUNCH();
    unsigned long long* hw = pinned_words();
    GC_CUDA(cudaMemcpyAsync(hw, h->ctr + C_SCRATCH0, 8, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaFreeAsync(mins, st));
    fetch_bad(h);
    GC_CUDA(cudaStreamSynchronize(st));
    raise_bad(h);
    *components = int64_t(hw[0]);
  });
}

}  // extern "C"
