// pipeline.cuh — elementwise kernels shared by the static, forest and
// incremental drivers (initialisation, compression, most-frequent label,
// active gather, finalisation, canonicalisation).
#pragma once

#include <climits>

#include "common.cuh"
#include "internal.h"

namespace gc {

constexpr int kEwBlock = 256;

// P[v] = v; optional hook / lock arrays (DisjointSets.__init__, dset.py:353-379)
__global__ void k_init_sets(int32_t* P, int32_t* H, int32_t* L, int32_t n, unsigned long long* stamps = nullptr,
                            unsigned stamp_mask = 0u);

// Full compression to the fixpoint (sampling.py:38-47 compress_all).
__global__ void k_compress(int32_t* P, int32_t n);

// Most-frequent label (sampling.py:29-35): probe a strided sample for the
// candidate, count it exactly; a strict majority is provably the argmax,
// otherwise an exact histogram decides (ties -> smaller label).
__global__ void k_mode_probe(const int32_t* P, int32_t n, unsigned long long* ctr, int walk, unsigned stamp_mask = 0u);
__global__ void k_count_eq(const int32_t* P, int32_t n, unsigned long long* ctr);
__global__ void k_hist_zero(int32_t* hist, int32_t n, unsigned long long* ctr);
__global__ void k_hist_add(const int32_t* P, int32_t* hist, int32_t n, unsigned long long* ctr);
__global__ void k_hist_argmax(const int32_t* hist, int32_t n, unsigned long long* ctr);

// Active vertices: label != l_max (driver.py:473), plus sum of their degrees
// (the finish inspection count, driver.py:335-336).
__global__ void k_gather_active(const int32_t* P, int32_t n, const int64_t* off, int32_t* list,
                                unsigned long long* ctr, int only_fallback);

// Pointer jump to the root in place; counts roots and flags labels that are
// not their class minimum (label_finalization, driver.py:420-429).
__global__ void k_finalize(int32_t* P, int32_t n, unsigned long long* ctr, unsigned stamp_mask = 0u);
// canonical_labels (validate.py:251-259), skipped on device when the
// finalize pass proved labels already canonical.
__global__ void k_canon_init(int32_t* mins, int32_t n, const unsigned long long* ctr);
__global__ void k_canon_min(const int32_t* P, int32_t* mins, int32_t n, const unsigned long long* ctr);
__global__ void k_canon_apply(int32_t* P, const int32_t* mins, int32_t n, const unsigned long long* ctr);

// Label-crossing directed edges over the active rows (driver.py:406-417 ic),
// computed outside the timed phases.
__global__ void k_ic_census(const int32_t* P, int32_t n, const int64_t* off, const int32_t* tgt,
                            const int32_t* list, unsigned long long* ctr);

__global__ void k_fill(int32_t* a, int64_t n, int32_t v);
__global__ void k_root_bitmap(const int32_t* P, int32_t n, uint32_t* bits);
__global__ void k_root_flags_list(const int32_t* P, const int32_t* list, const unsigned long long* ctr,
                                  uint8_t* flags);
__global__ void k_root_transitions_list(const int32_t* P, const int32_t* list, const unsigned long long* ctr,
                                        const uint8_t* flags, int32_t* out_u, int32_t* out_v,
                                        unsigned long long* out_count);
__global__ void k_root_transitions(const int32_t* P, const uint32_t* before, int32_t n, int32_t* out_u,
                                   int32_t* out_v, unsigned long long* count);
__global__ void k_count_ne(const int32_t* a, int64_t n, int32_t v, unsigned long long* out);

// Host helpers
void run_mode(int32_t* P, int32_t n, int32_t* hist, unsigned long long* ctr, cudaStream_t st);
// Post-sampling: candidate probe, (compress +) candidate count + optimistic
// active gather in one pass, exact-mode fallback.  Leaves L_max, the active
// list, its size and degree sum in the counters.
void run_post_sample(int32_t* P, int32_t n, const int64_t* off, int32_t* list, int32_t* hist,
                     unsigned long long* ctr, bool compress, cudaStream_t st, bool exact_mode = false);
// Active gather for a known L_max (finish_phase).
void run_gather(int32_t* P, int32_t n, const int64_t* off, int32_t* list, unsigned long long* ctr,
                cudaStream_t st);
// Pointer jump (+ canonical relabel when labels may not be class minima).
void run_finalize(int32_t* P, int32_t n, int32_t* mins, unsigned long long* ctr, cudaStream_t st,
                  bool maybe_noncanon = true, const int32_t* list = nullptr);
void fill(int32_t* a, int64_t n, int32_t v, cudaStream_t st);
void set_ctr(unsigned long long* ctr, int idx, unsigned long long v, cudaStream_t st);
void zero_ctr(unsigned long long* ctr, int words, cudaStream_t st);
void stamp(unsigned long long* ctr, int i, cudaStream_t st);
void stamp_defer(int i);
void stamp_flush(unsigned long long* ctr, cudaStream_t st);
// the pending (deferred) stamps, handed to the next kernel launch that takes
// them at entry (entry_stamp); clears them
unsigned take_stamps();
void set_ctr_add(unsigned long long* ctr, int idx, unsigned long long v, cudaStream_t st);

}  // namespace gc
