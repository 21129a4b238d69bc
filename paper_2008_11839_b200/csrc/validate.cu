// validate.cu — device routes behind the reference's DisjointSets probes
// (dset.py:381-399) and its validation helpers (validate.py:178-259): batched
// finds with the configured compaction, canonical min-member relabelling of
// an arbitrary labelling, and the "every recorded edge exists" clause of
// check_forest.  None of these are on the timed path; they make the
// drop-in API complete at BASELINE sizes, where the reference's per-edge
// Python loops take minutes.
#include <climits>

#include "internal.h"
#include "pipeline.cuh"
#include "uf.cuh"

namespace gc {

namespace {

template <int FIND>
__global__ void k_find_batch(int32_t* P, const int32_t* __restrict__ xs, int64_t k, int32_t* roots) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    Reader rd;
    roots[i] = find<FIND>(xs ? ldg32(xs + i) : int32_t(i), P, rd);
  }
}

// (u, v) present in row u of the sorted CSR?  Records the smallest failing
// index (the witness of validate.py:200-206 is the first missing edge).
__global__ void k_edges_exist(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int64_t n,
                              const int32_t* __restrict__ us, const int32_t* __restrict__ vs, int64_t k,
                              unsigned long long* first_missing) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < k; i += stride) {
    const int32_t u = us[i], v = vs[i];
    bool ok = u >= 0 && u < n && v >= 0 && v < n;
    if (ok) {
      int64_t lo = off[u], hi = off[u + 1];
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (tgt[mid] < v) lo = mid + 1;
        else hi = mid;
      }
      ok = lo < off[u + 1] && tgt[lo] == v;
    }
    if (!ok) atomicMin(first_missing, static_cast<unsigned long long>(i));
  }
}

__global__ void k_set_noncanon(unsigned long long* ctr) { ctr[C_NONCANON] = 1; }

// any id of a[0..len) outside [0, bound) sets *bad (one warp vote, one atomic
// per warp that saw a bad id)
__global__ void k_check_ids(const int32_t* __restrict__ a, int64_t len, uint32_t bound, unsigned int* bad) {
  unsigned f = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < len; i += stride)
    f |= uint32_t(a[i]) >= bound;
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(bad, 1u);
}

// CSR shape check (the Graph contract, graphs.py:43-51): offsets start at 0,
// never decrease, end at m; every target lies in [0, n).  bad[0] collects
// flags: 1 offsets, 2 targets.
__global__ void k_check_csr(const int64_t* __restrict__ off, const int32_t* __restrict__ tgt, int64_t n, int64_t m,
                            int aligned, unsigned int* bad) {
  unsigned flags = 0;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const int64_t t0 = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t v = t0; v <= n; v += stride) {
    const int64_t o = off[v];
    if ((v == 0 && o != 0) || (v == n && o != m) || (v < n && off[v + 1] < o) || o < 0 || o > m) flags |= 1u;
  }
  const int64_t mq = aligned ? m / 4 : 0;
  for (int64_t i = t0; i < mq; i += stride) {
    const int4 t = reinterpret_cast<const int4*>(tgt)[i];
    if (uint32_t(t.x) >= uint64_t(n) || uint32_t(t.y) >= uint64_t(n) || uint32_t(t.z) >= uint64_t(n) ||
        uint32_t(t.w) >= uint64_t(n))
      flags |= 2u;
  }
  for (int64_t i = 4 * mq + t0; i < m; i += stride)
    if (uint32_t(tgt[i]) >= uint64_t(n)) flags |= 2u;
  flags = __reduce_or_sync(0xffffffffu, flags);
  if ((threadIdx.x & 31) == 0 && flags) atomicOr(bad, flags);
}

__global__ void k_class_min(const int32_t* __restrict__ L, int32_t n, int32_t* mins) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    atomicMin(mins + L[v], int32_t(v));
}

// refinement (validate.py:290-297): every vertex shares its oracle label
// with its class's minimum member; the smallest violating vertex wins
__global__ void k_refines(const int32_t* __restrict__ L, const int32_t* __restrict__ mins,
                          const int32_t* __restrict__ orc, int32_t n, unsigned long long* first_bad) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t v = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; v < n; v += stride)
    if (orc[v] != orc[mins[L[v]]]) atomicMin(first_bad, static_cast<unsigned long long>(v));
}

}  // namespace

void check_ids(const int32_t* a, int64_t len, int64_t bound, cudaStream_t st, const char* what) {
  if (len <= 0) return;
  require(a != nullptr, GC_ERR_ARG, std::string("null ") + what);
  unsigned int* h = reinterpret_cast<unsigned int*>(pinned_words());
  static thread_local unsigned int* d = nullptr;
  if (!d) GC_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), 16));
  GC_CUDA(cudaMemsetAsync(d, 0, 4, st));
  (k_check_ids<<<grid_for(len, kEwBlock, 8), kEwBlock, 0, st>>>(a, len, uint32_t(bound), d), count_launch());
  GC_CHECK_LAUNCH();
  GC_CUDA(cudaMemcpyAsync(h, d, 4, cudaMemcpyDeviceToHost, st));
  GC_CUDA(cudaStreamSynchronize(st));
  require(h[0] == 0, GC_ERR_MALFORMED, std::string(what) + " outside [0, " + std::to_string(bound) + ")");
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_find_batch(int32_t* parent, int64_t n, const int32_t* xs, int64_t k, int32_t find_kind,
                  int32_t* roots_out, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31) && k >= 0, GC_ERR_ARG, "bad size");
    require(parent != nullptr || n == 0, GC_ERR_ARG, "null parent");
    require(roots_out != nullptr || k == 0, GC_ERR_ARG, "null output");
    require(xs != nullptr || k <= n, GC_ERR_ARG, "k > n without a query list");
    if (k == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(k, kEwBlock, 8);
    switch (find_kind) {
      case GC_FIND_NAIVE: (k_find_batch<GC_FIND_NAIVE><<<g, kEwBlock, 0, st>>>(parent, xs, k, roots_out), count_launch()); break;
      case GC_FIND_SPLIT: (k_find_batch<GC_FIND_SPLIT><<<g, kEwBlock, 0, st>>>(parent, xs, k, roots_out), count_launch()); break;
      case GC_FIND_HALVE: (k_find_batch<GC_FIND_HALVE><<<g, kEwBlock, 0, st>>>(parent, xs, k, roots_out), count_launch()); break;
      case GC_FIND_COMPRESS: (k_find_batch<GC_FIND_COMPRESS><<<g, kEwBlock, 0, st>>>(parent, xs, k, roots_out), count_launch()); break;
      case GC_FIND_TWO_TRY: (k_find_batch<GC_FIND_TWO_TRY><<<g, kEwBlock, 0, st>>>(parent, xs, k, roots_out), count_launch()); break;
      default: throw Error(GC_ERR_CONFIG, "unknown find rule");
    }
    GC_CHECK_LAUNCH();
  });
}

int gc_canonical_labels(int32_t* labels, int64_t n, void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(n >= 0 && n < (int64_t(1) << 31), GC_ERR_MALFORMED, "bad length");
    if (n == 0) return;
    require(labels != nullptr, GC_ERR_ARG, "null labels");
    Arena a(ws, ws_bytes);
    unsigned long long* ctr = a.take<unsigned long long>(C_COUNT_);
    int32_t* mins = a.take<int32_t>(n);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int g = grid_for(n, kEwBlock, 8);
    const int32_t nn = int32_t(n);
    (k_set_noncanon<<<1, 1, 0, st>>>(ctr), count_launch());
    (k_canon_init<<<g, kEwBlock, 0, st>>>(mins, nn, ctr), count_launch());
    (k_canon_min<<<g, kEwBlock, 0, st>>>(labels, mins, nn, ctr), count_launch());
    (k_canon_apply<<<g, kEwBlock, 0, st>>>(labels, mins, nn, ctr), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_edges_exist(const gc_csr* g, const int32_t* us, const int32_t* vs, int64_t k,
                   unsigned long long* first_missing, void* stream) {
  return guarded([&] {
    require(g != nullptr && first_missing != nullptr, GC_ERR_ARG, "null argument");
    require(k >= 0, GC_ERR_ARG, "negative count");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    GC_CUDA(cudaMemsetAsync(first_missing, 0xff, sizeof(unsigned long long), st));
    if (k == 0) return;
    (k_edges_exist<<<grid_for(k, kEwBlock, 8), kEwBlock, 0, st>>>(g->offsets, g->targets, g->n, us, vs, k,
                                                                 first_missing), count_launch());
    GC_CHECK_LAUNCH();
  });
}

int gc_label_census(const gc_csr* g, const int32_t* labels, const int32_t* oracle, int64_t* out_host,
                    void* ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    require(g != nullptr && out_host != nullptr, GC_ERR_ARG, "null argument");
    require(g->n >= 0 && g->n < (int64_t(1) << 31), GC_ERR_MALFORMED, "vertex count outside [0, 2^31)");
    const int32_t n = int32_t(g->n);
    out_host[0] = 0;
    out_host[1] = 0;
    out_host[2] = 0;
    out_host[3] = -1;
    if (n == 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    check_ids(labels, n, n, st, "label");
    if (oracle) check_ids(oracle, n, n, st, "oracle label");
    Arena a(ws, ws_bytes);
    unsigned long long* ctr = a.take<unsigned long long>(C_COUNT_);
    int32_t* hist = a.take<int32_t>(n);
    GC_CUDA(cudaMemsetAsync(ctr, 0, sizeof(unsigned long long) * C_COUNT_, st));
    // most_frequent_label (sampling.py:29-35): probe + exact histogram
    run_mode(const_cast<int32_t*>(labels), n, hist, ctr, st);
    if (g->m)
      (k_ic_census<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(labels, n, g->offsets, g->targets, nullptr,
                                                                 ctr), count_launch());
    if (oracle) {
      fill(hist, n, INT_MAX, st);
      GC_CUDA(cudaMemsetAsync(ctr + C_SCRATCH1, 0xff, 8, st));
      (k_class_min<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(labels, n, hist), count_launch());
      (k_refines<<<grid_for(n, kEwBlock, 8), kEwBlock, 0, st>>>(labels, hist, oracle, n, ctr + C_SCRATCH1),
       count_launch());
    }
    GC_CHECK_LAUNCH();
    unsigned long long c[C_COUNT_];
    GC_CUDA(cudaMemcpyAsync(c, ctr, sizeof(c), cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    out_host[0] = int64_t(c[C_LMAX]);
    out_host[1] = int64_t(c[C_LMAX_COUNT]);
    out_host[2] = g->m ? int64_t(c[C_IC]) : 0;
    out_host[3] = oracle && c[C_SCRATCH1] != ~0ull ? int64_t(c[C_SCRATCH1]) : -1;
  });
}

int gc_check_csr(const gc_csr* g, void* stream) {
  return guarded([&] {
    require(g != nullptr, GC_ERR_ARG, "null graph");
    require(g->n >= 0 && g->n < (int64_t(1) << 31), GC_ERR_MALFORMED, "vertex count outside [0, 2^31)");
    require(g->m >= 0, GC_ERR_MALFORMED, "negative edge count");
    require(g->offsets != nullptr || g->n == 0, GC_ERR_ARG, "null offsets");
    require(g->targets != nullptr || g->m == 0, GC_ERR_ARG, "null targets");
    if (g->offsets == nullptr) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    unsigned int* h = reinterpret_cast<unsigned int*>(pinned_words());
    // one device word per host thread, allocated once (a stream-ordered
    // allocation would go back to the OS at every synchronisation)
    static thread_local unsigned int* d = nullptr;
    if (!d) GC_CUDA(cudaMalloc(reinterpret_cast<void**>(&d), 16));
    GC_CUDA(cudaMemsetAsync(d, 0, 4, st));
    const int64_t work = g->n + 1 > g->m / 4 ? g->n + 1 : g->m / 4;
    const int aligned = reinterpret_cast<uintptr_t>(g->targets) % 16 == 0;
    (k_check_csr<<<grid_for(work, kEwBlock, 4), kEwBlock, 0, st>>>(g->offsets, g->targets, g->n, g->m, aligned,
                                                                  d), count_launch());
    GC_CHECK_LAUNCH();
    GC_CUDA(cudaMemcpyAsync(h, d, 4, cudaMemcpyDeviceToHost, st));
    GC_CUDA(cudaStreamSynchronize(st));
    require(!(h[0] & 1u), GC_ERR_MALFORMED, "CSR offsets must start at 0, never decrease and end at m");
    require(!(h[0] & 2u), GC_ERR_MALFORMED, "CSR target outside [0, n)");
  });
}

}  // extern "C"
