// internal.h — host-side launchers shared between the libgconn translation
// units.  Nothing here crosses the C ABI.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <cuda_runtime.h>

#include "../../include/gconn.h"

namespace gc {

// Error carried to the ABI boundary and converted to a status code there.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define GC_CUDA(expr)                                                          \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess)                                                     \
      throw ::gc::Error(GC_ERR_CUDA, std::string(#expr) + ": " +               \
                                         cudaGetErrorString(_e));              \
  } while (0)

#define GC_CHECK_LAUNCH() GC_CUDA(cudaGetLastError())

inline void require(bool ok, int code, const std::string& msg) {
  if (!ok) throw Error(code, msg);
}

// Bump allocator over the caller's workspace (256-byte aligned slices).
struct Arena {
  char* base;
  size_t cap;
  size_t used = 0;
  Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(int64_t count) {
    size_t bytes = (size_t(count < 0 ? 0 : count) * sizeof(T) + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    if (base == nullptr || used + bytes > cap)
      throw Error(GC_ERR_OOM, "workspace too small: need more than " +
                                  std::to_string(used + bytes) + " bytes, have " +
                                  std::to_string(cap));
    T* p = reinterpret_cast<T*>(base + used);
    used += bytes;
    return p;
  }
};

// Sizing twin of Arena: counts bytes without a buffer.
struct Sizer {
  size_t used = 0;
  template <typename T>
  T* take(int64_t count) {
    size_t bytes = (size_t(count < 0 ? 0 : count) * sizeof(T) + 255) & ~size_t(255);
    if (bytes == 0) bytes = 256;
    used += bytes;
    return nullptr;
  }
};

// Device counters block (one allocation, zeroed per call).
enum Counter : int {
  C_INSP_SAMPLE = 0,
  C_INSP_FINISH,
  C_LMAX,          // most frequent label
  C_LMAX_COUNT,
  C_CAND,          // candidate label from the probe
  C_CAND_COUNT,
  C_N_ACTIVE,
  C_COMPONENTS,
  C_NONCANON,      // any label[v] > v after the pointer jump
  C_CHANGED,       // round-based change flag
  C_WORK,          // working-edge count (LT alter)
  C_WORK_W,        // weighted working-edge count (reference semantics)
  C_IC,            // label-crossing directed edges
  C_NEXT,          // frontier size (BFS/LDD)
  C_SCRATCH0,
  C_SCRATCH1,
  C_CYCLE,         // finalize walk exceeded n steps (cyclic input labels)
  C_DONE,          // round loops: fixpoint reached
  C_ROUNDS,        // round loops: rounds executed
  C_RINSP,         // round loops: accumulated per-round inspections
  C_WLEN0,         // round loops: working length, parity 0 / 1
  C_WLEN1,
  C_WWT0,          // round loops: working weight, parity 0 / 1
  C_WWT1,
  C_MODE_EXACT,    // the sampler computed the exact mode itself (C_CAND is L_max)
  C_CUT,           // LDD: cut edges emitted into the rounds finish's COO
  C_STAMP0,        // 10 %globaltimer stamps of the static pipeline's phases
  C_COUNT_ = C_STAMP0 + 10
};

struct UFConfig {
  int unite;   // gc_finish_kind (ASYNC..JTB)
  int find;    // gc_find_kind
  int splice;  // gc_splice_kind
};

bool valid_uf(const UFConfig& c);

// Union over vertex rows (k-out, HB phase 2, union-find finish).
//   list == nullptr  -> vertices [0, count_host)
//   count_dev != nullptr -> the list length is read on device (bounded by count_host)
//   take_max: first min(take_max, deg) entries of each row
//   lower_only: only entries t < u (both endpoints active, dedup of twins)
//   insp: += sum over rows of min(take_max, deg)
struct RowUnionArgs {
  int32_t* P;
  int32_t* H;
  int32_t* L;
  const uint32_t* R;
  int32_t* fu;
  int32_t* fv;
  int32_t n;
  const int64_t* off;
  const int32_t* tgt;
  const int32_t* list;
  const unsigned long long* count_dev;
  int64_t count_host;
  int32_t take_max;
  int32_t lower_only;
  unsigned long long* insp;
  int32_t* lu = nullptr;  // optional compact list of the edges that merged two trees
  int32_t* lv = nullptr;
  unsigned long long* lcount = nullptr;
  int64_t row_base = 0;   // list == nullptr: rows [row_base, row_base + count_host)
  int2* fpair = nullptr;   // forest slots as pairs (see UFState::fpair)
  int64_t all_edges = -1;  // >= 0: the rows are the whole graph with this many entries
                           // (all-active lower-only finish; small graphs go edge-parallel)
  unsigned long long* stamps = nullptr;  // non-null: the kernel takes the pending phase stamps
                                         // (take_stamps) at entry into these slots
};
void launch_union_rows(const UFConfig& cfg, bool forest, const RowUnionArgs& a, cudaStream_t st);
// pending deferred phase stamps (pipeline.cu), cleared by the call
unsigned take_stamps();

// The caller's batch arrays for a giant-filter compaction that passed the
// batch through (see k_union_coo_async_mlp).
struct GiantPass {
  const int32_t* us = nullptr;
  const int32_t* vs = nullptr;
  const uint8_t* skip = nullptr;
  int64_t k = 0;
};

// Union over COO pairs (union_edge_list, incremental inserts).
struct CooUnionArgs {
  int32_t* P;
  int32_t* H;
  int32_t* L;
  const uint32_t* R;
  int32_t* fu;
  int32_t* fv;
  int32_t n;
  const int32_t* us;
  const int32_t* vs;
  int64_t k;
  const uint8_t* skip;   // optional: entries with skip[i] != 0 are not unions (queries)
  int32_t* lu = nullptr;  // optional: compact list of the edges that merged two trees
  int32_t* lv = nullptr;
  unsigned long long* lcount = nullptr;
  int32_t init_sentinel = -1;  // >= 0: lazily initialise both endpoints first (incremental)
  unsigned int* bad = nullptr;  // non-null: pairs with an endpoint outside [0, n) are skipped
                                // and set *bad (the incremental handle's sticky input flag)
  uint32_t* gbits = nullptr;         // incremental giant filter (see UFState::gbits)
  const int32_t* ganchor = nullptr;
  const unsigned long long* kdev = nullptr;  // non-null (async giant filter): the compaction's
                                             // survivor count, ~0 = use `alt`
  GiantPass alt;
  bool kdev_wave = false;  // the batch is expected to be compacted: one-wave grid
  uint8_t* lflag = nullptr;  // lock-step async kernel: lflag[i] = 1 when pair i merged two trees
};
void launch_union_coo(const UFConfig& cfg, bool forest, const CooUnionArgs& a, cudaStream_t st);

// Racy incremental batch (driver.py:674-694): each op is either a lazy-init
// + union (is_query[i] == 0) or a read-only root-chase query, interleaved in
// one launch.  sentinel marks uninitialised slots.  bits: one bit per op,
// packed LSB-first into 32-bit words (a warp's ballot per word).
void launch_incr_racy(const UFConfig& cfg, const CooUnionArgs& a, const uint8_t* is_query,
                      int32_t sentinel, uint32_t* bits, cudaStream_t st);

int num_sms();
// unions per thread of the lock-step async COO kernel (GC_COO_MLP, 0 = one per thread)
int coo_mlp();
// giant-filter bitmap accesses with an L2 evict_last hint (GC_GIANT_KEEP=0: off)
bool giant_keep();

// Kernel launches issued by libgconn (process-wide, exported through
// gc_launch_count for the bench's gpu_launches claim).
void count_launch();
void add_launches(long long k);
long long launch_total();

// Thread-local last-error string behind gc_last_error().
void set_last_error(const char* msg);

// Run f, converting any exception into a status code (nothing crosses the ABI).
template <class F>
int guarded(F&& f) {
  try {
    f();
    return GC_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return GC_ERR_OOM;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GC_ERR_CUDA;
  } catch (...) {
    set_last_error("unknown error");
    return GC_ERR_CUDA;
  }
}

// Synchronous range check: every a[i] in [0, bound), else GC_ERR_MALFORMED
// naming `what` (one streaming pass; entry points whose kernels would index
// with the values call it before launching them).
void check_ids(const int32_t* a, int64_t len, int64_t bound, cudaStream_t st, const char* what);

// 64 pinned host words per thread for flag / count read-backs.
unsigned long long* pinned_words();

}  // namespace gc
