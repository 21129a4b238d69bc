// pipeline.cu — elementwise phases of the two-phase pipeline
// (driver.py:454-500): set initialisation, compression, most-frequent label,
// active gather, finalisation and canonical relabelling.
#include <atomic>

#include "pipeline.cuh"

namespace gc {

__global__ void k_init_sets(int32_t* P, int32_t* H, int32_t* L, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    P[v] = int32_t(v);
    if (H) H[v] = n;
    if (L) L[v] = 0;
  }
}

__global__ void k_compress(int32_t* P, int32_t n) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t v = int32_t(i);
    int32_t p = ld_acq(P + v);
    if (p == v) continue;
    int32_t r = p;
    while (true) {
      const int32_t q = ld_acq(P + r);
      if (q == r) break;
      r = q;
    }
    if (r != p) st_rlx(P + v, r);
  }
}

constexpr int kProbe = 1024;

__global__ void __launch_bounds__(kProbe) k_mode_probe(const int32_t* P, int32_t n,
                                                       unsigned long long* ctr) {
  __shared__ int32_t lab[kProbe];
  __shared__ unsigned long long best;
  const int s = n < kProbe ? n : kProbe;
  const int i = threadIdx.x;
  if (i == 0) best = 0ull;
  if (i < s) lab[i] = ld_acq(P + (int64_t(i) * n) / s);
  __syncthreads();
  if (i < s) {
    const int32_t me = lab[i];
    unsigned c = 0;
    for (int j = 0; j < s; ++j) c += lab[j] == me;
    const unsigned long long key =
        (static_cast<unsigned long long>(c) << 32) | (0xffffffffull - uint32_t(me));
    atomicMax(&best, key);
  }
  __syncthreads();
  if (i == 0) {
    ctr[C_CAND] = s ? (0xffffffffull - (best & 0xffffffffull)) : 0ull;
    ctr[C_CAND_COUNT] = 0;
  }
}

__global__ void k_count_eq(const int32_t* P, int32_t n, unsigned long long* ctr) {
  const int32_t cand = int32_t(ctr[C_CAND]);
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    c += P[v] == cand;
  block_add<kEwBlock>(ctr + C_CAND_COUNT, c);
}

__device__ __forceinline__ bool majority(const unsigned long long* ctr, int32_t n) {
  return 2ull * ctr[C_CAND_COUNT] > static_cast<unsigned long long>(n);
}

__global__ void k_hist_zero(int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) hist[v] = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctr[C_SCRATCH0] = 0;
}

__global__ void k_hist_add(const int32_t* P, int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const bool ok = v < n;
    const unsigned act = __ballot_sync(0xffffffffu, ok);
    if (!ok) continue;
    const int32_t lab = P[v];
    // warp aggregation: one atomic per distinct label in the warp
    const unsigned same = __match_any_sync(act, lab);
    const int leader = __ffs(same) - 1;
    if ((threadIdx.x & 31) == leader) atomicAdd(hist + lab, __popc(same));
  }
}

__global__ void k_hist_argmax(const int32_t* hist, int32_t n, unsigned long long* ctr) {
  if (majority(ctr, n)) return;
  __shared__ unsigned long long best;
  if (threadIdx.x == 0) best = 0ull;
  __syncthreads();
  unsigned long long mine = 0ull;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride) {
    const unsigned long long key = (static_cast<unsigned long long>(uint32_t(hist[v])) << 32) |
                                   (0xffffffffull - uint64_t(v));
    mine = key > mine ? key : mine;
  }
  atomicMax(&best, mine);
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(ctr + C_SCRATCH0, best);
}

__global__ void k_mode_finish(int32_t n, unsigned long long* ctr) {
  if (n == 0) {
    ctr[C_LMAX] = 0;
    ctr[C_LMAX_COUNT] = 0;
  } else if (majority(ctr, n)) {
    ctr[C_LMAX] = ctr[C_CAND];
    ctr[C_LMAX_COUNT] = ctr[C_CAND_COUNT];
  } else {
    const unsigned long long k = ctr[C_SCRATCH0];
    ctr[C_LMAX] = 0xffffffffull - (k & 0xffffffffull);
    ctr[C_LMAX_COUNT] = k >> 32;
  }
}

__global__ void k_gather_active(const int32_t* P, int32_t n, const int64_t* off, int32_t* list,
                                unsigned long long* ctr) {
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  unsigned long long degsum = 0;
  const int lane = threadIdx.x & 31;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t base = int64_t(blockIdx.x) * blockDim.x; base < n; base += stride) {
    const int64_t v = base + threadIdx.x;
    const bool act = v < n && P[v] != lmax;
    const unsigned bal = __ballot_sync(0xffffffffu, act);
    if (bal == 0) continue;
    unsigned long long pos = 0;
    if (lane == 0) pos = atomicAdd(ctr + C_N_ACTIVE, static_cast<unsigned long long>(__popc(bal)));
    pos = __shfl_sync(0xffffffffu, pos, 0);
    if (act) {
      list[pos + __popc(bal & ((1u << lane) - 1u))] = int32_t(v);
      degsum += static_cast<unsigned long long>(off[v + 1] - off[v]);
    }
  }
  block_add<kEwBlock>(ctr + C_INSP_FINISH, degsum);
}

__global__ void k_finalize(int32_t* P, int32_t n, unsigned long long* ctr) {
  unsigned long long roots = 0;
  bool noncanon = false, cyc = false;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const int32_t v = int32_t(i);
    int32_t r = ld_acq(P + v);
    if (r == v) {
      ++roots;
      continue;
    }
    int64_t steps = 0;
    while (true) {
      const int32_t q = ld_acq(P + r);
      if (q == r) break;
      r = q;
      if (++steps > n) { cyc = true; break; }
    }
    st_rlx(P + v, r);
    noncanon |= r > v;
  }
  block_add<kEwBlock>(ctr + C_COMPONENTS, roots);
  if (__syncthreads_or(noncanon) && threadIdx.x == 0) ctr[C_NONCANON] = 1;
  if (cyc) ctr[C_CYCLE] = 1;
}

__global__ void k_canon_init(int32_t* mins, int32_t n, const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    mins[v] = INT_MAX;
}

__global__ void k_canon_min(const int32_t* P, int32_t* mins, int32_t n,
                            const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    atomicMin(mins + P[v], int32_t(v));
}

__global__ void k_canon_apply(int32_t* P, const int32_t* mins, int32_t n,
                              const unsigned long long* ctr) {
  if (ctr[C_NONCANON] == 0) return;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    P[v] = mins[P[v]];
}

__global__ void k_ic_census(const int32_t* P, int32_t n, const int64_t* off, const int32_t* tgt,
                            const int32_t* list, unsigned long long* ctr) {
  const int32_t lmax = int32_t(ctr[C_LMAX]);
  const int64_t count = list ? int64_t(ctr[C_N_ACTIVE]) : int64_t(n);
  unsigned long long ic = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride) {
    const int32_t u = list ? list[i] : int32_t(i);
    const int32_t pu = P[u];
    for (int64_t j = off[u]; j < off[u + 1]; ++j) {
      const int32_t pt = P[tgt[j]];
      // over all rows: count crossing entries; over the active rows only,
      // the reverse entries from L_max-labelled rows are added back
      ic += list ? (pu != pt) + (pt == lmax) : (pu != pt);
    }
  }
  block_add<kEwBlock>(ctr + C_IC, ic);
}

__global__ void k_fill(int32_t* a, int64_t n, int32_t v) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) a[i] = v;
}

__global__ void k_count_ne(const int32_t* a, int64_t n, int32_t v, unsigned long long* out) {
  unsigned long long c = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    c += a[i] != v;
  block_add<kEwBlock>(out, c);
}

namespace {
std::atomic<long long> g_launches{0};
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

long long launch_total() { return g_launches.load(); }

unsigned long long* pinned_words() {
  static thread_local unsigned long long* p = nullptr;
  if (!p) GC_CUDA(cudaMallocHost(&p, 64 * sizeof(unsigned long long)));
  return p;
}

__global__ void k_set_ctr(unsigned long long* ctr, int idx, unsigned long long v) { ctr[idx] = v; }

void set_ctr(unsigned long long* ctr, int idx, unsigned long long v, cudaStream_t st) {
  (k_set_ctr<<<1, 1, 0, st>>>(ctr, idx, v), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void fill(int32_t* a, int64_t n, int32_t v, cudaStream_t st) {
  if (n <= 0) return;
  (k_fill<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(a, n, v), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void run_mode(int32_t* P, int32_t n, int32_t* hist, unsigned long long* ctr, cudaStream_t st) {
  if (n > 0) {
    const int g = grid_for(n, kEwBlock, 8);
    (k_mode_probe<<<1, kProbe, 0, st>>>(P, n, ctr), ::gc::count_launch());
    (k_count_eq<<<g, kEwBlock, 0, st>>>(P, n, ctr), ::gc::count_launch());
    (k_hist_zero<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
    (k_hist_add<<<g, kEwBlock, 0, st>>>(P, hist, n, ctr), ::gc::count_launch());
    (k_hist_argmax<<<g, kEwBlock, 0, st>>>(hist, n, ctr), ::gc::count_launch());
  }
  (k_mode_finish<<<1, 1, 0, st>>>(n, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

void run_finalize(int32_t* P, int32_t n, int32_t* mins, unsigned long long* ctr, cudaStream_t st) {
  if (n <= 0) return;
  const int g = grid_for(n, kEwBlock, 8);
  (k_finalize<<<g, kEwBlock, 0, st>>>(P, n, ctr), ::gc::count_launch());
  (k_canon_init<<<g, kEwBlock, 0, st>>>(mins, n, ctr), ::gc::count_launch());
  (k_canon_min<<<g, kEwBlock, 0, st>>>(P, mins, n, ctr), ::gc::count_launch());
  (k_canon_apply<<<g, kEwBlock, 0, st>>>(P, mins, n, ctr), ::gc::count_launch());
  GC_CHECK_LAUNCH();
}

}  // namespace gc

extern "C" long long gc_launch_count(void) { return gc::launch_total(); }
