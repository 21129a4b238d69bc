// samplers.h — sampling-phase launchers (sampling.py:61-172 + the new LDD
// sampler).  Each leaves P holding labels that refine the true partition.
#pragma once

#include "internal.h"

namespace gc {

struct SamplerWs {
  int32_t* coo_u = nullptr;   // k-out random mode pairs
  int32_t* coo_v = nullptr;
  unsigned long long* key = nullptr;  // BFS / LDD claim word: (round << 32) | parent-or-cluster
  int32_t* q0 = nullptr;      // frontier queues (HB: phase-2 roots)
  int32_t* q1 = nullptr;
  uint32_t* fb0 = nullptr;    // BFS frontier bitmaps
  uint32_t* fb1 = nullptr;
  uint32_t* vis = nullptr;    // BFS visited bitmap (union of all frontiers so far)
  unsigned long long* stat = nullptr;  // frontier [count, degree sum] x 2
  uint16_t* start = nullptr;  // LDD start round per vertex
  int32_t* order = nullptr;   // LDD vertices bucketed by start round
  unsigned int* boff = nullptr;    // LDD bucket offsets [kLddMaxRounds + 2]
  unsigned int* cursor = nullptr;  // LDD scatter cursors
  // LDD cut-edge emission (set by a labels-only rounds finish; the
  // finish's working COO arrays): every pair of adjacent vertices in
  // different clusters, once; cut_done when the sampler produced it
  int32_t* cut_u = nullptr;
  int32_t* cut_v = nullptr;
  unsigned long long* cut_count = nullptr;
  bool cut_done = false;
};

constexpr int kLddMaxRounds = 4094;

template <class A>
void sampler_carve(A& a, SamplerWs& w, int64_t n, int64_t m, const gc_spec& s) {
  (void)m;
  if (s.sample == GC_SAMPLE_KOUT && s.kout_mode == GC_KOUT_FIRST_PLUS_RANDOM) {
    w.coo_u = a.template take<int32_t>(n * int64_t(s.kout_k));
    w.coo_v = a.template take<int32_t>(n * int64_t(s.kout_k));
  }
  if (s.sample == GC_SAMPLE_HB) w.q0 = a.template take<int32_t>(n);  // phase-2 roots
  if (s.sample == GC_SAMPLE_BFS || s.sample == GC_SAMPLE_LDD) {
    w.key = a.template take<unsigned long long>(n);
    w.q0 = a.template take<int32_t>(n);
    w.q1 = a.template take<int32_t>(n);
    w.stat = a.template take<unsigned long long>(8);
  }
  if (s.sample == GC_SAMPLE_BFS) {
    w.fb0 = a.template take<uint32_t>((n + 31) / 32);
    w.fb1 = a.template take<uint32_t>((n + 31) / 32);
    w.vis = a.template take<uint32_t>((n + 31) / 32);
  }
  if (s.sample == GC_SAMPLE_LDD) {
    w.fb0 = a.template take<uint32_t>((n + 31) / 32);  // sorted-frontier bitmap
    w.start = a.template take<uint16_t>(n);
    w.order = a.template take<int32_t>(n);
    w.boff = a.template take<unsigned int>(kLddMaxRounds + 4);
    w.cursor = a.template take<unsigned int>(kLddMaxRounds + 4);
  }
}

void run_kout(const gc_csr& g, const gc_spec& s, const UFConfig& c, RowUnionArgs a, bool forest,
              SamplerWs& w, unsigned long long* ctr, cudaStream_t st);
void run_hb(const gc_csr& g, const gc_spec& s, const UFConfig& c, RowUnionArgs a, bool forest,
            SamplerWs& w, unsigned long long* ctr, cudaStream_t st);
void run_bfs(const gc_csr& g, const gc_spec& s, int32_t* P, int32_t* fu, int32_t* fv, SamplerWs& w,
             unsigned long long* ctr, cudaStream_t st);
// true when the persistent packed form also left the exact mode in
// ctr[C_CAND] (+ C_MODE_EXACT): the pipeline then skips its probe / histogram
bool run_ldd(const gc_csr& g, const gc_spec& s, int32_t* P, SamplerWs& w, unsigned long long* ctr,
             cudaStream_t st);

}  // namespace gc
