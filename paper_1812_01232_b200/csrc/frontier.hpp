// GPU-resident frontier (frontier.cu): an unordered node pool in HBM with an
// order-preserving 64-bit key per node (the lower bound); each wave
// radix-selects the W smallest keys, expands them, and appends the surviving
// children. Expanded nodes become holes; holes and stale nodes are compacted
// away when they dominate the pool.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "gosma_capi.h"

namespace gosma {

constexpr unsigned long long kHoleKey = ~0ull;

struct RouteStats {
  double pruned_volume = 0.0;
  double resolved_volume = 0.0;
  unsigned long long floor_key = ~0ull;  // order key of the min resolved lower bound
  double scratch = 0.0;
};

unsigned long long host_order_key(double v);

// A child whose upper bound beats every earlier child of its wave and the
// incumbent (process_wave's refinement candidates, solver.cpp:409-431).
struct ImprovingChild {
  double upper;
  unsigned long long index;
  gosma_node node;  // the child itself (no per-record copy afterwards)
};
double key_to_double(unsigned long long k);

struct Frontier {
  // node pool
  gosma_node* nodes = nullptr;
  int8_t* split = nullptr;
  double* vol = nullptr;
  unsigned long long* key = nullptr;
  size_t size = 0;   // slots in use (live + holes + stale)
  size_t holes = 0;  // expanded slots
  size_t cap = 0;
  size_t cap_limit = 0;  // memory budget in nodes (0: none)
  // selection
  unsigned int* sel = nullptr;
  size_t sel_cap = 0;
  unsigned int* hist = nullptr;  // radix-select histogram (4096 bins)
  unsigned int* bsel = nullptr;  // boundary-bin candidates of a selection
  size_t bsel_cap = 0;
  unsigned int* cidx = nullptr;  // compaction move lists (holes, live tail)
  size_t cidx_cap = 0;
  // a lower bound of the smallest live key (set by min_key; keys only rise
  // through selection/append, so it stays valid until an import)
  unsigned long long known_min = 0;
  // candidate list: pool indices of all live keys < tau (0: invalid)
  unsigned int* cand = nullptr;
  unsigned int* cand_tmp = nullptr;
  size_t cand_n = 0, cand_cap = 0;
  unsigned long long tau = 0;
  unsigned long long rebuilds = 0;  // candidate-list rebuilds (profiling)
  // depth-first stack (select_deepest): pool indices of deep live nodes, the
  // kept children of each depth-first wave pushed on top, so a wave pops the
  // deepest nodes without scanning the pool; refilled by one scan when short,
  // dropped whenever pool indices move (compaction, folds, imports) or the
  // waves go best-first again
  unsigned int* dstk = nullptr;
  size_t dstk_n = 0, dstk_cap = 0;
  bool dstk_ok = false, deep_active = false;
  unsigned long long deep_fills = 0;  // stack refills (profiling)
  void drop_deep() { dstk_ok = false; dstk_n = 0; }
  bool prof = false;                // synchronising sub-phase timers
  double t_sub[6] = {0, 0, 0, 0, 0, 0};  // rebuild, descend, pick, list; grow, route
  size_t max_bin = 0, max_cand = 0;
  unsigned long long kids_total = 0, kids_kept = 0;  // routed / appended children
  std::vector<unsigned int> h_hist;
  // children of one wave
  gosma_node* kids = nullptr;
  double* kid_lower = nullptr;
  double* kid_upper = nullptr;
  int8_t* kid_split = nullptr;
  double* kid_vol = nullptr;
  int* keep = nullptr;
  unsigned int* kept_idx = nullptr;
  size_t kid_cap = 0;
  // distinct translation cuboids of one wave (translation-cached bounds)
  unsigned int* tcnt = nullptr;  // per selected parent: 1 (rotation split) or 8
  unsigned int* toff = nullptr;  // exclusive scan of tcnt (n_sel + 1 entries)
  int* tidx = nullptr;           // child -> cuboid slot
  gosma_node* tnodes = nullptr;  // cuboid slots (translation part used)
  double* tself = nullptr;       // 4 doubles per cuboid: self LB, self UB, err, flag
  int* rot_list = nullptr;       // selection indices with a rotation split
  int* trans_list = nullptr;     // children 8k+c of translation-split selections
  unsigned long long* list_counts = nullptr;  // {rotation parents, translation children}
  // reductions / scratch
  RouteStats* stats = nullptr;
  unsigned long long* counter = nullptr;
  RouteStats* h_stats = nullptr;
  unsigned long long* h_counter = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;

  cudaError_t reserve(size_t cap_nodes, size_t wave);
  cudaError_t ensure_kids(size_t n_sel);
  void release();
  cudaError_t ensure_temp(size_t bytes);
  cudaError_t grow(size_t need, cudaStream_t s);
  // Host upload of initial nodes.
  cudaError_t upload(const gosma_node* h_nodes, const int8_t* h_split, const double* h_vol,
                     size_t n, cudaStream_t s);
  // min key over the pool (kHoleKey if empty)
  cudaError_t min_key(cudaStream_t s, unsigned long long* out);
  // selects up to `want` slots with key < limit (the smallest first); writes
  // their indices to sel, marks them holes, returns the count.
  cudaError_t descend(size_t want, unsigned long long limit, double fill, cudaStream_t s,
                      unsigned long long* lo, unsigned long long* hi, size_t* below,
                      size_t* bin, const unsigned int* idx, size_t n_items, const double* rank);
  cudaError_t rebuild_candidates(size_t want_total, cudaStream_t s);
  cudaError_t select_smallest(size_t want, unsigned long long limit, cudaStream_t s, size_t* n);
  // depth-first order under memory pressure: the smallest volumes below limit
  cudaError_t select_deepest(size_t want, unsigned long long limit, cudaStream_t s, size_t* n);
  cudaError_t deep_scan(size_t want_total, unsigned long long limit, cudaStream_t s,
                        unsigned int* out, size_t* n_out);
  cudaError_t expand_selected(size_t n_sel, cudaStream_t s);
  cudaError_t expand_selected_cached(size_t n_sel, cudaStream_t s, size_t* n_cuboids);
  // rotation-split selections (rot_list) and translation-split children (trans_list)
  // rotation-split selections / translation-split children lists; their
  // counts stay on the device (list_counts, read by the bound kernels)
  cudaError_t wave_lists(size_t n_sel, cudaStream_t s);
  // the selected records (sel[0..n)) into contiguous device buffers
  cudaError_t gather_selected(size_t n, cudaStream_t s, gosma_node* out_nodes, int8_t* out_split,
                              double* out_vol);
  // device-side import of n records
  cudaError_t upload_device(const gosma_node* d_nodes, const int8_t* d_split, const double* d_vol,
                            size_t n, cudaStream_t s);
  // children i with upper[i] < min(bound, upper[0..i-1]) in index order: the
  // branches the reference's in-order wave loop would refine (before its
  // refinements lower the incumbent further)
  cudaError_t improving_children(size_t n_kids, double bound, cudaStream_t s,
                                 std::vector<ImprovingChild>* out);
  double* kid_pmin = nullptr;  // exclusive prefix minimum of kid_upper
  size_t pmin_cap = 0;
  ImprovingChild* rec = nullptr;  // device record list (rec_cap entries, grown on demand)
  size_t rec_cap = 0;
  // route children against d* (prune) and finish (bound >= finish: to the
  // floor with the unsplittable ones), append survivors
  cudaError_t route_append(size_t n_kids, double dstar, double finish, cudaStream_t s,
                           RouteStats* out);
  // drop holes and nodes with key >= limit; returns the dropped (non-hole) volume
  cudaError_t compact(unsigned long long limit, cudaStream_t s, double* dropped_volume);
  // keep the `keep_n` smallest keys (capacity folding); returns folded volume
  // and the smallest folded lower bound
  cudaError_t fold_to(size_t keep_n, cudaStream_t s, double* folded_volume, double* folded_min);
  size_t live_upper_bound() const { return size - holes; }
  cudaError_t live_volume(cudaStream_t s, double* out);
};

}  // namespace gosma
