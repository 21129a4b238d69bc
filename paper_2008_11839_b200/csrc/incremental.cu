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
                             unsigned int* bad) {
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
    launch_union_coo(UFConfig{h->spec.finish, h->spec.find, h->spec.splice}, false, a, st);
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
    (k_incr_query<<<g1(len), kIB, 0, st>>>(h->state, us, vs, is_query, len, sentinel, bits_out, h->bad),
     ::gc::count_launch());
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
    launch_union_coo(UFConfig{h->spec.finish, h->spec.find, h->spec.splice}, false, a, st);
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
                                             h->bad), ::gc::count_launch());
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
