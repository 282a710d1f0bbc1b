// K2-K4: the GPU-resident branch-and-bound frontier.
//
// Reference: solve() (core/src/solver.cpp:312-688) keeps a best-first binary
// heap on the host and pops batch_size/8 nodes per wave. Here the frontier is
// an unordered pool in HBM with an order-preserving 64-bit key per node (its
// lower bound). Each wave radix-selects the W smallest keys below a limit
// (12-bit digit histograms, refined until the boundary bin is narrow), expands
// them into 8 children each (subdivide_adaptive, se3.cpp:107-147, using the
// split decision the bound kernel fused), bounds the children with K1, and
// routes them by stream compaction (solver.cpp:396-405): prune, resolve
// (unsplittable: certified floor), or append to the pool tail. Expanded slots
// become holes; holes and stale nodes (lower >= d*) are compacted away when
// they dominate the pool. Volumes travel with the nodes (children carry an
// exact eighth; solver.cpp:379-405, 597-608).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <unordered_map>

#include "frontier.hpp"

namespace gosma {

namespace {

constexpr int kBins = 4096;

// First error of a chain of asynchronous calls.
inline cudaError_t chain(cudaError_t e, cudaError_t next) { return e != cudaSuccess ? e : next; }

// Device (and pinned host) blocks freed by a frontier are cached by exact
// size per device instead of returned to the driver: cudaMalloc / cudaFree of
// a few hundred MB cost milliseconds each, which dominated short solves
// (create + destroy ~0.14 s against ~0.02 s of waves). A freed block waits for
// the device to go idle before it can be handed out again (cudaFree's own
// semantics); the cache keeps at most kCacheBytes per device, oldest first
// out. gosma_release_cached_memory empties it.
struct CachedBlock {
  int device;
  bool host;
  size_t bytes;
  void* p;
};
constexpr size_t kCacheBytes = size_t(8) << 30;
std::mutex g_cache_mu;
std::vector<CachedBlock> g_cache;                // oldest first
std::unordered_map<void*, CachedBlock> g_live;   // blocks handed out by dmalloc / hmalloc

void* cache_take(int dev, bool host, size_t bytes) {
  std::lock_guard<std::mutex> lk(g_cache_mu);
  for (size_t k = g_cache.size(); k-- > 0;) {
    const CachedBlock& b = g_cache[k];
    if (b.device == dev && b.host == host && b.bytes == bytes) {
      void* p = b.p;
      g_cache.erase(g_cache.begin() + static_cast<long>(k));
      g_live[p] = CachedBlock{dev, host, bytes, p};
      return p;
    }
  }
  return nullptr;
}

void release_block(const CachedBlock& b) {
  if (b.host)
    cudaFreeHost(b.p);
  else
    cudaFree(b.p);
}

cudaError_t cached_alloc(void** p, size_t bytes, bool host) {
  *p = nullptr;
  if (bytes == 0) bytes = 1;
  int dev = 0;
  cudaGetDevice(&dev);
  if ((*p = cache_take(dev, host, bytes))) return cudaSuccess;
  const cudaError_t e = host ? cudaMallocHost(p, bytes) : cudaMalloc(p, bytes);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_cache_mu);
  g_live[*p] = CachedBlock{dev, host, bytes, *p};
  return cudaSuccess;
}

void cached_free(void* p) {
  if (!p) return;
  CachedBlock b;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    auto it = g_live.find(p);
    if (it == g_live.end()) return;
    b = it->second;
    g_live.erase(it);
  }
  int cur = 0;
  cudaGetDevice(&cur);
  if (cur != b.device) cudaSetDevice(b.device);
  cudaDeviceSynchronize();  // no kernel may still use it when it is handed out again
  if (cur != b.device) cudaSetDevice(cur);
  std::vector<CachedBlock> evict;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_cache.push_back(b);
    size_t total = 0;
    for (const CachedBlock& c : g_cache)
      if (c.device == b.device) total += c.bytes;
    for (size_t k = 0; k < g_cache.size() && total > kCacheBytes;) {
      if (g_cache[k].device == b.device) {
        total -= g_cache[k].bytes;
        evict.push_back(g_cache[k]);
        g_cache.erase(g_cache.begin() + static_cast<long>(k));
      } else {
        ++k;
      }
    }
  }
  for (const CachedBlock& c : evict) release_block(c);
}

template <typename T>
cudaError_t dmalloc(T** p, size_t bytes) {
  return cached_alloc(reinterpret_cast<void**>(p), bytes, false);
}

template <typename T>
cudaError_t hmalloc(T** p, size_t bytes) {
  return cached_alloc(reinterpret_cast<void**>(p), bytes, true);
}

void dfree(void* p) { cached_free(p); }

// Returns a dmalloc'd block to the driver (parked sets being replaced).
void hard_free(void* p) {
  if (!p) return;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    g_live.erase(p);
  }
  cudaFree(p);
}

// Frees the cached blocks of `device` (gosma_release_cached_memory).
void purge_cache(int device) {
  std::vector<CachedBlock> out;
  {
    std::lock_guard<std::mutex> lk(g_cache_mu);
    for (size_t k = 0; k < g_cache.size();) {
      if (g_cache[k].device == device) {
        out.push_back(g_cache[k]);
        g_cache.erase(g_cache.begin() + static_cast<long>(k));
      } else {
        ++k;
      }
    }
  }
  for (const CachedBlock& c : out) release_block(c);
}

// The four pool arrays of a released frontier are parked (one set per device)
// instead of freed: unmapping tens of GB costs tenths of a second, and the
// next solve on the device reuses them. gosma_release_cached_memory frees.
struct ParkedPool {
  int device = -1;
  size_t cap = 0;
  gosma_node* nodes = nullptr;
  int8_t* split = nullptr;
  double* vol = nullptr;
  unsigned long long* key = nullptr;
};
std::mutex g_park_mu;
std::vector<ParkedPool> g_parked;

// Child buffers of a wave, parked the same way.
struct ParkedWave {
  int device = -1;
  size_t cap = 0;
  void* buf[10] = {nullptr, nullptr, nullptr, nullptr, nullptr,
                   nullptr, nullptr, nullptr, nullptr, nullptr};
};
std::vector<ParkedWave> g_parked_wave;

void free_parked_wave(ParkedWave& w) {
  for (void* b : w.buf) hard_free(b);
  w = ParkedWave{};
}

void free_parked(ParkedPool& p) {
  hard_free(p.nodes);
  hard_free(p.split);
  hard_free(p.vol);
  hard_free(p.key);
  p = ParkedPool{};
}

// A parked set of at least `need` nodes on the current device, if any.
bool take_parked(size_t need, ParkedPool* out) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_park_mu);
  for (size_t k = 0; k < g_parked.size(); ++k) {
    if (g_parked[k].device == dev && g_parked[k].cap >= need) {
      *out = g_parked[k];
      g_parked.erase(g_parked.begin() + static_cast<long>(k));
      return true;
    }
  }
  return false;
}

void park(ParkedPool p) {
  if (!p.nodes) return;
  cudaGetDevice(&p.device);
  cudaDeviceSynchronize();
  std::lock_guard<std::mutex> lk(g_park_mu);
  for (ParkedPool& q : g_parked) {
    if (q.device == p.device) {  // keep the larger set per device
      if (q.cap >= p.cap) {
        free_parked(p);
      } else {
        free_parked(q);
        q = p;
      }
      return;
    }
  }
  g_parked.push_back(p);
}

__host__ __device__ __forceinline__ unsigned long long order_key_bits(unsigned long long b) {
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ unsigned long long order_key(double v) {
  return order_key_bits(static_cast<unsigned long long>(__double_as_longlong(v)));
}

inline unsigned grid_for(size_t n, unsigned block) {
  return static_cast<unsigned>(std::max<size_t>(1, (n + block - 1) / block));
}

inline unsigned grid_cap(size_t n, unsigned block) {
  return static_cast<unsigned>(std::min<size_t>(grid_for(n, block), 148 * 8));
}

// Histogram of digit (key >> shift) & mask among keys < limit whose bits above
// `prefix_shift` equal `prefix` (prefix_shift 64: no prefix).
// With `rank` set, the slots with key < limit are ranked by the bits of
// rank[i] (a positive double: the node volume) instead of by their key (the
// depth-first order, smallest volumes first).
__global__ void digit_hist(const unsigned long long* key, const unsigned int* idx, size_t n,
                           unsigned long long limit, int shift, int bits,
                           unsigned long long prefix, int prefix_shift, unsigned int* hist,
                           const double* rank) {
  __shared__ unsigned int sh[kBins];
  const int nb = 1 << bits;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t slot = idx ? idx[i] : i;
    unsigned long long k = key[slot];
    if (k >= limit) continue;
    if (rank) k = __double_as_longlong(rank[slot]);
    if (prefix_shift < 64 && (k >> prefix_shift) != prefix) continue;
    atomicAdd(&sh[(k >> shift) & static_cast<unsigned long long>(nb - 1)], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], sh[b]);
}

struct KeyBelow {
  const unsigned long long* key;
  unsigned long long lo, hi;  // select lo <= key < hi
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    const unsigned long long k = key[i];
    return k >= lo && k < hi;
  }
};

// Depth-first order: key < limit with the volume's bits in [lo, hi).
struct VolRange {
  const unsigned long long* key;
  const double* vol;
  unsigned long long lo, hi, limit;
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    if (key[i] >= limit) return false;
    const unsigned long long r = __double_as_longlong(vol[i]);
    return r >= lo && r < hi;
  }
};

// Live node below the limit (holes carry kHoleKey, which no limit reaches).
struct KeyBelowLimit {
  const unsigned long long* key;
  unsigned long long limit;
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    return key[i] < limit;
  }
};

__global__ void iota_u32(unsigned int* out, unsigned int first, size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) out[i] = first + static_cast<unsigned int>(i);
}

// Appended children (slot < end, read on the device) whose key is below tau.
struct NewCandidate {
  const unsigned long long* key;
  unsigned long long tau;
  size_t base;
  const unsigned long long* count;  // appended children (int in the low word)
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    return i < base + static_cast<size_t>(*reinterpret_cast<const int*>(count)) && key[i] < tau;
  }
};

struct NotHole {
  const unsigned long long* key;
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    return key[i] != kHoleKey;
  }
};

__global__ void min_key_gather(const unsigned long long* key, const unsigned int* idx, size_t n,
                               unsigned long long* out) {
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long best = kHoleKey;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[idx[i]];
    if (k < best) best = k;
  }
  const unsigned long long r = BR(tmp).Reduce(best, cub::Min());
  if (threadIdx.x == 0 && r != kHoleKey) atomicMin(out, r);
}

__global__ void mark_holes(unsigned long long* key, const unsigned int* sel, size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) key[sel[i]] = kHoleKey;
}

// subdivide_adaptive (se3.cpp:107-147): 8 children per selected node.
// With `toff` set, also emits the wave's distinct translation cuboids for the
// translation-cached bound kernels: a rotation split keeps the parent's cuboid
// for all 8 children (one slot), a translation split makes 8 new ones.
__global__ void expand(const gosma_node* front, const int8_t* split, const double* vol,
                       const unsigned int* sel, size_t n_sel, gosma_node* kids, double* kid_vol,
                       const unsigned int* toff, int* tidx, gosma_node* tnodes) {
  const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (t >= n_sel * 8) return;
  const size_t p = sel[t / 8];
  const int c = static_cast<int>(t % 8);
  const int sx = (c & 4) ? 1 : -1, sy = (c & 2) ? 1 : -1, sz = (c & 1) ? 1 : -1;
  gosma_node k = front[p];
  if (split[p] == 1) {
    const double h = 0.5 * k.rhw;
    k.rc[0] += h * sx;
    k.rc[1] += h * sy;
    k.rc[2] += h * sz;
    k.rhw = h;
  } else {
    const double h0 = 0.5 * k.thw[0], h1 = 0.5 * k.thw[1], h2 = 0.5 * k.thw[2];
    k.tc[0] += h0 * sx;
    k.tc[1] += h1 * sy;
    k.tc[2] += h2 * sz;
    k.thw[0] = h0;
    k.thw[1] = h1;
    k.thw[2] = h2;
  }
  kids[t] = k;  // lower inherited: the parent's bound is valid on any subset
  kid_vol[t] = vol[p] / 8.0;
  if (toff) {
    const bool rot = split[p] == 1;
    const unsigned slot = toff[t / 8] + (rot ? 0u : static_cast<unsigned>(c));
    tidx[t] = static_cast<int>(slot);
    if (!rot || c == 0) tnodes[slot] = k;
  }
}

// Work lists of a wave: rotation-split parents (siblings kernel) and the
// children of translation-split parents (full kernel). Order is irrelevant:
// every item writes its own output slots.
__global__ void split_lists(const int8_t* split, const unsigned int* sel, size_t n_sel,
                            int* rot, int* trans_kids, unsigned long long* counts) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k >= n_sel) return;
  if (split[sel[k]] == 1) {
    rot[atomicAdd(&counts[0], 1ull)] = static_cast<int>(k);
  } else {
    const int b = static_cast<int>(atomicAdd(&counts[1], 8ull));
    for (int c = 0; c < 8; ++c) trans_kids[b + c] = static_cast<int>(8 * k + c);
  }
}

__global__ void keys_of(const gosma_node* nodes, size_t n, unsigned long long* key) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k < n) key[k] = order_key(nodes[k].lower);
}

__global__ void gather_sel(const gosma_node* nodes, const int8_t* split, const double* vol,
                           const unsigned int* sel, size_t n, gosma_node* on, int8_t* os,
                           double* ov) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k >= n) return;
  const unsigned int i = sel[k];
  on[k] = nodes[i];
  os[k] = split[i];
  ov[k] = vol[i];
}

__global__ void cuboid_counts(const int8_t* split, const unsigned int* sel, size_t n_sel,
                              unsigned int* cnt) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k < n_sel) cnt[k] = split[sel[k]] == 1 ? 1u : 8u;
  if (k == n_sel) cnt[k] = 0u;
}

// Route evaluated children (solver.cpp:396-405).
// finish: children with a bound >= finish (the wave's limit d* - eps) are
// finished for the certificate: no wave will expand them, and their only
// effect on it is the minimum bound among those still below d* -- which is
// the minimum over all of them, since pruning removes the largest first. They
// go to the floor like unsplittable children instead of the pool (the
// certificate min(d*, frontier min, floor) is unchanged).
__global__ void route(gosma_node* kids, const double* lower, const int8_t* split,
                      const double* kid_vol, size_t n, double dstar, double finish, int* keep,
                      RouteStats* stats) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double pv = 0.0, rv = 0.0;
  unsigned long long fl = ~0ull;
  int flag = 0;
  if (i < n) {
    const double lo = lower[i];
    kids[i].lower = lo;
    if (!(lo < dstar)) {
      pv = kid_vol[i];
    } else if (split[i] < 0 || !(lo < finish)) {
      rv = kid_vol[i];
      fl = order_key(lo);
    } else {
      flag = 1;
    }
    keep[i] = flag;
  }
  typedef cub::BlockReduce<double, 256> BR;
  typedef cub::BlockReduce<unsigned long long, 256> BU;
  __shared__ typename BR::TempStorage t1;
  __shared__ typename BU::TempStorage t2;
  const double spv = BR(t1).Sum(pv);
  __syncthreads();
  const double srv = BR(t1).Sum(rv);
  const unsigned long long mfl = BU(t2).Reduce(fl, cub::Min());
  if (threadIdx.x == 0) {
    if (spv != 0.0) atomicAdd(&stats->pruned_volume, spv);
    if (srv != 0.0) atomicAdd(&stats->resolved_volume, srv);
    if (mfl != ~0ull) atomicMin(&stats->floor_key, mfl);
  }
}

// Appends the flagged children at the pool tail.
__global__ void append_kids(const gosma_node* kids, const int8_t* ksplit, const double* kvol,
                            const unsigned int* idx, size_t n, gosma_node* dst, int8_t* dsplit,
                            double* dvol, unsigned long long* dkey) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned int k = idx[i];
  const gosma_node nd = kids[k];
  dst[i] = nd;
  dsplit[i] = ksplit[k];
  dvol[i] = kvol[k];
  dkey[i] = order_key(nd.lower);
}

__global__ void append_kids_counted(const gosma_node* kids, const int8_t* ksplit,
                                    const double* kvol, const unsigned int* idx,
                                    const unsigned long long* count, gosma_node* dst,
                                    int8_t* dsplit, double* dvol, unsigned long long* dkey) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k >= static_cast<size_t>(*reinterpret_cast<const int*>(count))) return;
  const gosma_node nd = kids[idx[k]];
  dst[k] = nd;
  dsplit[k] = ksplit[idx[k]];
  dvol[k] = kvol[idx[k]];
  dkey[k] = order_key(nd.lower);
}

__global__ void gather_pool(const gosma_node* src, const int8_t* ssplit, const double* svol,
                            const unsigned long long* skey, const unsigned int* idx, size_t n,
                            gosma_node* dst, int8_t* dsplit, double* dvol,
                            unsigned long long* dkey) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned int k = idx[i];
  dst[i] = src[k];
  dsplit[i] = ssplit[k];
  dvol[i] = svol[k];
  dkey[i] = skey[k];
}

// Marks stale slots (key >= limit) as holes and sums their volume.
__global__ void drop_stale(unsigned long long* key, const double* vol, size_t n,
                           unsigned long long limit, double* out) {
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[i];
    if (k != kHoleKey && k >= limit) {
      acc += vol[i];
      key[i] = kHoleKey;
    }
  }
  const double sum = BR(tmp).Sum(acc);
  if (threadIdx.x == 0 && sum != 0.0) atomicAdd(out, sum);
}

// Live (non-hole) slots at index >= live and holes at index < live.
struct TailLive {
  const unsigned long long* key;
  unsigned int live;
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    return i >= live && key[i] != kHoleKey;
  }
};
struct HeadHole {
  const unsigned long long* key;
  unsigned int live;
  __device__ __forceinline__ bool operator()(const unsigned int& i) const {
    return i < live && key[i] == kHoleKey;
  }
};

__global__ void count_live(const unsigned long long* key, size_t n, unsigned long long* out) {
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    c += key[i] != kHoleKey ? 1 : 0;
  const unsigned long long sum = BR(tmp).Sum(c);
  if (threadIdx.x == 0 && sum) atomicAdd(out, sum);
}

// Moves the live tail into the head holes (in place, order not preserved).
__global__ void move_tail(gosma_node* nodes, int8_t* split, double* vol, unsigned long long* key,
                          const unsigned int* dst, const unsigned int* src,
                          const unsigned long long* count) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k >= static_cast<size_t>(*reinterpret_cast<const int*>(count))) return;
  const unsigned int d = dst[k], s = src[k];
  nodes[d] = nodes[s];
  split[d] = split[s];
  vol[d] = vol[s];
  key[d] = key[s];
}

// Sum of volumes of non-hole slots with key >= limit.
__global__ void dropped_volume(const unsigned long long* key, const double* vol, size_t n,
                               unsigned long long limit, double* out) {
  typedef cub::BlockReduce<double, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[i];
    if (k != kHoleKey && k >= limit) acc += vol[i];
  }
  const double s = BR(tmp).Sum(acc);
  if (threadIdx.x == 0 && s != 0.0) atomicAdd(out, s);
}

__global__ void min_key_at_least(const unsigned long long* key, size_t n,
                                 unsigned long long tau, unsigned long long* out) {
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long best = kHoleKey;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[i];
    if (k >= tau && k < best) best = k;
  }
  const unsigned long long r = BR(tmp).Reduce(best, cub::Min());
  if (threadIdx.x == 0 && r != kHoleKey) atomicMin(out, r);
}

// Children whose upper bound is below the exclusive prefix minimum (records).
__global__ void flag_records(const double* upper, const double* pmin, const gosma_node* kids,
                             size_t n, ImprovingChild* out, unsigned long long* count,
                             unsigned cap) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double u = upper[i];
    if (u < pmin[i]) {
      const unsigned long long k = atomicAdd(count, 1ull);
      if (k < cap) out[k] = ImprovingChild{u, i, kids[i]};
    }
  }
}

struct MinOp {
  __device__ __forceinline__ double operator()(double a, double b) const { return fmin(a, b); }
};

}  // namespace

unsigned long long host_order_key(double v) {
  unsigned long long b;
  std::memcpy(&b, &v, 8);
  return order_key_bits(b);
}

double key_to_double(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

// Child buffers for n_sel selected parents (8 children each): a small set
// first, then grown on demand (at least doubling); a finished solver parks
// them for the next solve on the device.
cudaError_t Frontier::ensure_kids(size_t n_sel) {
  const size_t need = 8 * n_sel;
  if (need <= kid_cap) return cudaSuccess;
  // geometric growth from a small first block (short solves never map a
  // full wave's worth; depth-first waves grow it further)
  const size_t nk = std::max(need, kid_cap ? 2 * kid_cap : (size_t(1) << 16));
  void** slots[10] = {reinterpret_cast<void**>(&tidx),      reinterpret_cast<void**>(&tnodes),
                      reinterpret_cast<void**>(&tself),     reinterpret_cast<void**>(&kids),
                      reinterpret_cast<void**>(&kid_lower), reinterpret_cast<void**>(&kid_upper),
                      reinterpret_cast<void**>(&kid_split), reinterpret_cast<void**>(&kid_vol),
                      reinterpret_cast<void**>(&keep),      reinterpret_cast<void**>(&kept_idx)};
  const size_t elem[10] = {4, sizeof(gosma_node), 4 * sizeof(double), sizeof(gosma_node), 8, 8,
                           1, 8, 4, 4};
  for (void** p : slots) {
    dfree(*p);
    *p = nullptr;
  }
  kid_cap = 0;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_park_mu);
    for (size_t k = 0; k < g_parked_wave.size(); ++k) {
      ParkedWave& w = g_parked_wave[k];
      if (w.device == dev && w.cap >= nk) {
        for (int i = 0; i < 10; ++i) *slots[i] = w.buf[i];
        kid_cap = w.cap;
        g_parked_wave.erase(g_parked_wave.begin() + static_cast<long>(k));
        return cudaSuccess;
      }
    }
  }
  cudaError_t e;
  for (int i = 0; i < 10; ++i)
    if ((e = dmalloc(slots[i], nk * elem[i])) != cudaSuccess) return e;
  kid_cap = nk;
  return cudaSuccess;
}

cudaError_t Frontier::reserve(size_t cap_nodes, size_t wave) {
  cudaError_t e = cudaSuccess;
  if (cap_nodes > cap) {
    if ((e = dmalloc(&nodes, cap_nodes * sizeof(gosma_node))) != cudaSuccess) return e;
    if ((e = dmalloc(&split, cap_nodes)) != cudaSuccess) return e;
    if ((e = dmalloc(&vol, cap_nodes * sizeof(double))) != cudaSuccess) return e;
    if ((e = dmalloc(&key, cap_nodes * 8)) != cudaSuccess) return e;
    cap = cap_nodes;
  }
  if (wave > sel_cap) {
    dfree(sel);
    dfree(tcnt);
    dfree(toff);
    dfree(rot_list);
    dfree(trans_list);
    if ((e = dmalloc(&rot_list, wave * 4)) != cudaSuccess) return e;
    if ((e = dmalloc(&trans_list, wave * 8 * 4)) != cudaSuccess) return e;
    if ((e = dmalloc(&sel, wave * 4)) != cudaSuccess) return e;
    if ((e = dmalloc(&tcnt, (wave + 1) * 4)) != cudaSuccess) return e;
    if ((e = dmalloc(&toff, (wave + 1) * 4)) != cudaSuccess) return e;
    sel_cap = wave;
  }
  if (!stats) {
    if ((e = dmalloc(&stats, sizeof(RouteStats))) != cudaSuccess) return e;
    if ((e = dmalloc(&counter, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    if ((e = dmalloc(&hist, kBins * sizeof(unsigned int))) != cudaSuccess) return e;
    if ((e = dmalloc(&list_counts, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    if ((e = hmalloc(&h_stats, sizeof(RouteStats))) != cudaSuccess) return e;
    if ((e = hmalloc(&h_counter, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    h_hist.resize(kBins);
  }
  return e;
}

void Frontier::release() {
  if (cap >= (size_t(1) << 24)) {  // >= 16M nodes (1.7 GB): keep for the next solve
    ParkedPool p;
    p.cap = cap;
    p.nodes = nodes;
    p.split = split;
    p.vol = vol;
    p.key = key;
    park(p);
  } else {
    dfree(nodes);
    dfree(split);
    dfree(vol);
    dfree(key);
  }
  dfree(sel);
  dfree(hist);
  if (kid_cap >= (size_t(1) << 20)) {  // keep a full wave's child buffers for the next solve
    ParkedWave w;
    cudaGetDevice(&w.device);
    w.cap = kid_cap;
    void* bufs[10] = {tidx, tnodes, tself, kids, kid_lower, kid_upper, kid_split, kid_vol, keep,
                      kept_idx};
    for (int i = 0; i < 10; ++i) w.buf[i] = bufs[i];
    cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_park_mu);
    bool placed = false;
    for (ParkedWave& q : g_parked_wave) {
      if (q.device == w.device) {
        if (q.cap >= w.cap) {
          free_parked_wave(w);
        } else {
          free_parked_wave(q);
          q = w;
        }
        placed = true;
        break;
      }
    }
    if (!placed) g_parked_wave.push_back(w);
  } else {
    dfree(kids);
    dfree(kid_lower);
    dfree(kid_upper);
    dfree(kid_split);
    dfree(kid_vol);
    dfree(keep);
    dfree(kept_idx);
    dfree(tidx);
    dfree(tnodes);
    dfree(tself);
  }
  dfree(tcnt);
  dfree(toff);
  tcnt = toff = nullptr;
  tidx = nullptr;
  tnodes = nullptr;
  tself = nullptr;
  dfree(bsel);
  bsel = nullptr;
  dfree(rot_list);
  dfree(trans_list);
  dfree(list_counts);
  rot_list = trans_list = nullptr;
  list_counts = nullptr;
  bsel_cap = 0;
  dfree(cidx);
  cidx = nullptr;
  cidx_cap = 0;
  dfree(kid_pmin);
  kid_pmin = nullptr;
  pmin_cap = 0;
  dfree(rec);
  rec = nullptr;
  rec_cap = 0;
  dfree(cand);
  dfree(cand_tmp);
  cand = cand_tmp = nullptr;
  cand_n = cand_cap = 0;
  tau = 0;
  known_min = 0;
  dfree(dstk);
  dstk = nullptr;
  dstk_cap = 0;
  drop_deep();
  deep_active = false;
  dfree(stats);
  dfree(counter);
  dfree(temp);
  dfree(h_stats);
  dfree(h_counter);
  nodes = nullptr;
  split = nullptr;
  vol = nullptr;
  key = nullptr;
  sel = nullptr;
  hist = nullptr;
  kids = nullptr;
  kid_lower = kid_upper = nullptr;
  kid_split = nullptr;
  kid_vol = nullptr;
  keep = nullptr;
  kept_idx = nullptr;
  stats = nullptr;
  counter = nullptr;
  temp = nullptr;
  h_stats = nullptr;
  h_counter = nullptr;
  size = holes = cap = sel_cap = kid_cap = temp_bytes = 0;
}

cudaError_t Frontier::ensure_temp(size_t bytes) {
  if (bytes <= temp_bytes) return cudaSuccess;
  dfree(temp);
  temp = nullptr;
  bytes = std::max(bytes, temp_bytes + temp_bytes / 2);  // geometric growth
  const cudaError_t e = dmalloc(&temp, bytes);
  if (e == cudaSuccess) temp_bytes = bytes;
  return e;
}

cudaError_t Frontier::grow(size_t need, cudaStream_t s) {
  if (need <= cap) return cudaSuccess;
  // geometric growth (x4); past half the budget, straight to the budget
  size_t c = std::max(need, 4 * cap);
  if (cap_limit && c > cap_limit / 2) c = std::max(need, cap_limit);
  gosma_node* n2 = nullptr;
  int8_t* s2 = nullptr;
  double* v2 = nullptr;
  unsigned long long* k2 = nullptr;
  cudaError_t e;
  ParkedPool pk;
  if (take_parked(need, &pk)) {
    n2 = pk.nodes;
    s2 = pk.split;
    v2 = pk.vol;
    k2 = pk.key;
    c = pk.cap;
  } else {
    if ((e = dmalloc(&n2, c * sizeof(gosma_node))) != cudaSuccess) return e;
    if ((e = dmalloc(&s2, c)) != cudaSuccess) return e;
    if ((e = dmalloc(&v2, c * sizeof(double))) != cudaSuccess) return e;
    if ((e = dmalloc(&k2, c * 8)) != cudaSuccess) return e;
  }
  e = cudaSuccess;
  if (size) {
    e = chain(e, cudaMemcpyAsync(n2, nodes, size * sizeof(gosma_node), cudaMemcpyDeviceToDevice,
                                 s));
    e = chain(e, cudaMemcpyAsync(s2, split, size, cudaMemcpyDeviceToDevice, s));
    e = chain(e, cudaMemcpyAsync(v2, vol, size * sizeof(double), cudaMemcpyDeviceToDevice, s));
    e = chain(e, cudaMemcpyAsync(k2, key, size * 8, cudaMemcpyDeviceToDevice, s));
  }
  if ((e = chain(e, cudaStreamSynchronize(s))) != cudaSuccess) return e;
  dfree(nodes);
  dfree(split);
  dfree(vol);
  dfree(key);
  nodes = n2;
  split = s2;
  vol = v2;
  key = k2;
  cap = c;
  return cudaSuccess;
}

cudaError_t Frontier::upload(const gosma_node* h_nodes, const int8_t* h_split,
                             const double* h_vol, size_t n, cudaStream_t s) {
  drop_deep();
  cudaError_t e;
  if ((e = grow(size + n, s)) != cudaSuccess) return e;
  std::vector<unsigned long long> k(n);
  for (size_t i = 0; i < n; ++i) k[i] = host_order_key(h_nodes[i].lower);
  known_min = 0;  // imported keys may lie below the cached minimum
  tau = 0;
  e = cudaMemcpyAsync(nodes + size, h_nodes, n * sizeof(gosma_node), cudaMemcpyHostToDevice, s);
  e = chain(e, cudaMemcpyAsync(split + size, h_split, n, cudaMemcpyHostToDevice, s));
  e = chain(e, cudaMemcpyAsync(vol + size, h_vol, n * sizeof(double), cudaMemcpyHostToDevice, s));
  e = chain(e, cudaMemcpyAsync(key + size, k.data(), n * 8, cudaMemcpyHostToDevice, s));
  e = chain(e, cudaStreamSynchronize(s));
  if (e == cudaSuccess) size += n;
  return e;
}

cudaError_t Frontier::min_key(cudaStream_t s, unsigned long long* out) {
  if (size == 0) {
    *out = kHoleKey;
    return cudaSuccess;
  }
  cudaError_t e;
  // every live key below tau is a candidate: their minimum is the pool minimum
  if (tau != 0 && (cand_n > 0 || tau == kHoleKey)) {
    unsigned long long init = kHoleKey;
    std::memcpy(h_counter, &init, 8);
    if ((e = cudaMemcpyAsync(counter, h_counter, 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return e;
    if (cand_n) min_key_gather<<<grid_cap(cand_n, 256), 256, 0, s>>>(key, cand, cand_n, counter);
    cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
    e = cudaStreamSynchronize(s);
    *out = h_counter[0];
    if (e == cudaSuccess && (*out != kHoleKey || tau == kHoleKey)) {
      if (*out != kHoleKey) known_min = *out;
      return cudaSuccess;
    }
    if (e != cudaSuccess) return e;
  }
  size_t need = 0;
  cub::DeviceReduce::Min(nullptr, need, key, counter, static_cast<int>(size), s);
  e = ensure_temp(need);
  if (e != cudaSuccess) return e;
  cub::DeviceReduce::Min(temp, need, key, counter, static_cast<int>(size), s);
  cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  *out = h_counter[0];
  if (e == cudaSuccess && *out != kHoleKey) known_min = *out;
  return e;
}

// Radix descent over 12-bit digit histograms: the largest bin boundary lo
// with count(key < lo) = below <= want (refined until below >= fill * want or
// the digits run out), and hi = the end of the boundary bin (capped at limit).
cudaError_t Frontier::descend(size_t want, unsigned long long limit, double fill, cudaStream_t s,
                              unsigned long long* lo, unsigned long long* hi, size_t* below_out,
                              size_t* bin_out, const unsigned int* idx, size_t n_items,
                              const double* rank) {
  // Digit schedule over the 64-bit key: 12,12,12,12,12,4 bits.
  // Every live key lies in [known_min, limit): the digits start below their
  // common high bits (one 12-bit level usually resolves a wave).
  int pshift = 64;  // bits >= pshift are fixed to `prefix` (64: none)
  unsigned long long prefix = 0;
  if (!rank && known_min > 0 && known_min < limit) {
    const unsigned long long x = known_min ^ (limit - 1);
    pshift = std::max(12, x ? 64 - __builtin_clzll(x) : 0);
    prefix = pshift >= 64 ? 0ull : (known_min >> pshift);
  }
  unsigned long long lo_key = 0, hi_key = rank ? kHoleKey : limit;
  size_t below = 0;  // count of keys < lo_key
  size_t bin = 0;    // count of keys in [lo_key, hi_key)
  cudaError_t e;
  while (pshift > 0) {
    const int bits = std::min(12, pshift);
    const int shift = pshift - bits;
    if ((e = cudaMemsetAsync(hist, 0, kBins * 4, s)) != cudaSuccess) return e;
    digit_hist<<<grid_cap(n_items, 256), 256, 0, s>>>(key, idx, n_items, limit, shift, bits,
                                                      prefix, pshift, hist, rank);
    const int nb = 1 << bits;
    if ((e = cudaMemcpyAsync(h_hist.data(), hist, nb * 4, cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    const unsigned long long base = pshift >= 64 ? 0ull : (prefix << pshift);
    size_t cum = below;
    int b = 0;
    for (; b < nb; ++b) {
      if (cum + h_hist[b] > want) break;
      cum += h_hist[b];
    }
    const unsigned long long cap = rank ? kHoleKey : limit;  // ranked values are not keys
    if (b == nb) {  // everything under this prefix fits
      const unsigned long long end = pshift >= 64 ? 0ull : base + (1ull << pshift);
      lo_key = hi_key = (end == 0 || end > cap) ? cap : end;
      below = cum;
      bin = 0;
      break;
    }
    bin = h_hist[b];
    lo_key = base + (static_cast<unsigned long long>(b) << shift);
    const unsigned long long end = lo_key + (1ull << shift);
    hi_key = (end == 0 || end > cap) ? cap : end;
    below = cum;
    if (static_cast<double>(below) >= fill * static_cast<double>(want) || shift == 0) break;
    prefix = (pshift >= 64 ? 0ull : (prefix << bits)) | static_cast<unsigned long long>(b);
    pshift = shift;
  }
  *lo = lo_key;
  *hi = hi_key;
  *below_out = below;
  if (bin_out) *bin_out = bin;
  return cudaSuccess;
}

// Candidate list: the pool indices of every live key below tau (tau = 0:
// invalid, kHoleKey: the list holds the whole live pool). Waves select from
// it, so a wave touches O(candidates) memory instead of the whole pool.
cudaError_t Frontier::rebuild_candidates(size_t want_total, cudaStream_t s) {
  ++rebuilds;
  tau = 0;
  cand_n = 0;
  if (size == 0) {
    tau = kHoleKey;
    return cudaSuccess;
  }
  unsigned long long lo = 0, hi = kHoleKey;
  size_t below = 0, bin = 0;
  cudaError_t e = descend(want_total, kHoleKey, 0.5, s, &lo, &hi, &below, &bin, nullptr, size, nullptr);
  if (e != cudaSuccess) return e;
  const unsigned long long t = below > 0 ? lo : hi;  // massive ties: keep the boundary bin
  const size_t count = below > 0 ? below : bin;
  const size_t cap_need = count + 16 * std::max<size_t>(sel_cap, 1);
  if (cap_need > cand_cap) {
    dfree(cand);
    dfree(cand_tmp);
    cand = cand_tmp = nullptr;
    if ((e = dmalloc(&cand, cap_need * 4)) != cudaSuccess) return e;
    if ((e = dmalloc(&cand_tmp, cap_need * 4)) != cudaSuccess) return e;
    cand_cap = cap_need;
  }
  if (count) {
    cub::CountingInputIterator<unsigned int> it(0);
    KeyBelow p{key, 0ull, t};
    size_t need = 0;
    cub::DeviceSelect::If(nullptr, need, it, cand, counter, static_cast<int>(size), p, s);
    if ((e = ensure_temp(need)) != cudaSuccess) return e;
    cub::DeviceSelect::If(temp, need, it, cand, counter, static_cast<int>(size), p, s);
  }
  cand_n = count;
  tau = t;
  return cudaGetLastError();
}

namespace {
struct SubTimer {
  Frontier* F;
  cudaStream_t s;
  std::chrono::steady_clock::time_point t;
  SubTimer(Frontier* f, cudaStream_t st) : F(f), s(st) {
    if (F->prof) {
      cudaStreamSynchronize(s);
      t = std::chrono::steady_clock::now();
    }
  }
  void lap(int k) {
    if (!F->prof) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    F->t_sub[k] += std::chrono::duration<double>(now - t).count();
    t = now;
  }
};
}  // namespace

cudaError_t Frontier::select_smallest(size_t want, unsigned long long limit, cudaStream_t s,
                                      size_t* n_out) {
  deep_active = false;  // best-first again: the depth-first stack is refilled next time
  drop_deep();
  SubTimer tm(this, s);
  *n_out = 0;
  if (size == 0 || want == 0) return cudaSuccess;
  want = std::min(want, sel_cap);
  cudaError_t e;
  const size_t target = std::max<size_t>(8 * want, size_t(1) << 20);
  if (tau == 0 && (e = rebuild_candidates(target, s)) != cudaSuccess) return e;
  tm.lap(0);
  unsigned long long lo_key = 0, hi_key = limit;
  size_t below = 0, bin_count = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    if (cand_n == 0) {
      lo_key = hi_key = limit;
      below = bin_count = 0;
    } else if ((e = descend(want, limit, 0.5, s, &lo_key, &hi_key, &below, &bin_count, cand,
                            cand_n, nullptr)) != cudaSuccess) {
      return e;
    }
    // too few candidates below the limit while the pool may hold more: refill
    const bool short_of_want = hi_key == lo_key && below < want;
    if (attempt == 0 && short_of_want && tau < limit && tau != kHoleKey) {
      tm.lap(1);
      if ((e = rebuild_candidates(target, s)) != cudaSuccess) return e;
      tm.lap(0);
      continue;
    }
    break;
  }
  tm.lap(1);
  // candidates with key < lo_key (count `below` <= want), then the first ones
  // (in candidate order) of the boundary bin [lo_key, hi_key); both counts are
  // known from the histograms, so the stable selections need no host sync.
  size_t need = 0;
  KeyBelow p1{key, 0ull, lo_key};
  cub::DeviceSelect::If(nullptr, need, cand, sel, counter, static_cast<int>(cand_n), p1, s);
  if ((e = ensure_temp(need)) != cudaSuccess) return e;
  const size_t n1 = below;
  if (n1 > 0) cub::DeviceSelect::If(temp, need, cand, sel, counter, static_cast<int>(cand_n), p1, s);
  size_t n2 = 0;
  if (n1 < want && hi_key > lo_key && bin_count > 0) {
    n2 = std::min(want - n1, bin_count);
    if (bin_count > bsel_cap) {
      dfree(bsel);
      bsel = nullptr;
      const size_t c = std::max(bin_count, 2 * bsel_cap);
      if ((e = dmalloc(&bsel, c * 4)) != cudaSuccess) return e;
      bsel_cap = c;
    }
    KeyBelow p2{key, lo_key, hi_key};
    cub::DeviceSelect::If(temp, need, cand, bsel, counter, static_cast<int>(cand_n), p2, s);
    if ((e = cudaMemcpyAsync(sel + n1, bsel, n2 * 4, cudaMemcpyDeviceToDevice, s)) !=
        cudaSuccess)
      return e;
  }
  const size_t n = n1 + n2;
  max_bin = std::max(max_bin, bin_count);
  max_cand = std::max(max_cand, cand_n);
  tm.lap(2);
  if (n) {
    mark_holes<<<grid_for(n, 256), 256, 0, s>>>(key, sel, n);
    holes += n;
    // drop the expanded slots from the candidate list
    NotHole ph{key};
    size_t need2 = 0;
    cub::DeviceSelect::If(nullptr, need2, cand, cand_tmp, counter, static_cast<int>(cand_n), ph,
                          s);
    if ((e = ensure_temp(need2)) != cudaSuccess) return e;
    cub::DeviceSelect::If(temp, need2, cand, cand_tmp, counter, static_cast<int>(cand_n), ph, s);
    std::swap(cand, cand_tmp);
    cand_n -= n;
  }
  tm.lap(3);
  *n_out = n;
  return cudaGetLastError();
}

// Depth-first order (memory pressure): the `want` live nodes below `limit`
// with the SMALLEST volumes, i.e. the deepest. Every node below d* - eps has
// to be expanded before the gap closes whatever the order (children's bounds
// are max(core, parent)), so the order changes neither the work nor the
// certificate, only the pool's peak size: depth-first keeps ~(8 W x depth)
// nodes open. Full-pool radix descent on the volume bits (no candidate list).
// The want_total deepest live nodes below the limit (one pool scan) into
// out[0 .. *n_out): the smallest volumes; the boundary depth contributes its
// first nodes in pool order.
cudaError_t Frontier::deep_scan(size_t want_total, unsigned long long limit, cudaStream_t s,
                                unsigned int* out, size_t* n_out) {
  *n_out = 0;
  if (size == 0 || want_total == 0) return cudaSuccess;
  cudaError_t e;
  unsigned long long lo_key = 0, hi_key = kHoleKey;
  size_t below = 0, bin_count = 0;
  // one histogram pass: the first 12 bits of a positive double are its
  // exponent, and a level deeper divides the volume by 8 (three exponent
  // steps), so the first digit already separates depths; the nodes of one
  // depth share their volume bits, so refining the boundary bin would only
  // cost passes (the boundary depth contributes its first nodes in pool order)
  if ((e = descend(want_total, limit, 0.0, s, &lo_key, &hi_key, &below, &bin_count, nullptr,
                   size, vol)) != cudaSuccess)
    return e;
  cub::CountingInputIterator<unsigned int> it(0);
  size_t need = 0;
  VolRange p1{key, vol, 0ull, lo_key, limit};
  cub::DeviceSelect::If(nullptr, need, it, out, counter, static_cast<int>(size), p1, s);
  if ((e = ensure_temp(need)) != cudaSuccess) return e;
  const size_t n1 = below;
  if (n1 > 0) cub::DeviceSelect::If(temp, need, it, out, counter, static_cast<int>(size), p1, s);
  size_t n2 = 0;
  if (n1 < want_total && hi_key > lo_key && bin_count > 0) {
    n2 = std::min(want_total - n1, bin_count);
    if (bin_count > bsel_cap) {
      dfree(bsel);
      bsel = nullptr;
      const size_t c = std::max(bin_count, 2 * bsel_cap);
      if ((e = dmalloc(&bsel, c * 4)) != cudaSuccess) return e;
      bsel_cap = c;
    }
    VolRange p2{key, vol, lo_key, hi_key, limit};
    cub::DeviceSelect::If(temp, need, it, bsel, counter, static_cast<int>(size), p2, s);
    if ((e = cudaMemcpyAsync(out + n1, bsel, n2 * 4, cudaMemcpyDeviceToDevice, s)) != cudaSuccess)
      return e;
  }
  *n_out = n1 + n2;
  return cudaGetLastError();
}

cudaError_t Frontier::select_deepest(size_t want, unsigned long long limit, cudaStream_t s,
                                     size_t* n_out) {
  *n_out = 0;
  deep_active = true;
  if (size == 0 || want == 0) return cudaSuccess;
  want = std::min(want, sel_cap);
  cudaError_t e;
  static const bool use_stack = [] {  // GOSMA_DEEP_STACK=0: scan every wave (A/B)
    const char* v = std::getenv("GOSMA_DEEP_STACK");
    return !(v && std::string(v) == "0");
  }();
  size_t n = 0;
  if (!use_stack) {
    if ((e = deep_scan(want, limit, s, sel, &n)) != cudaSuccess) return e;
  } else {
    for (int attempt = 0; attempt < 4 && n == 0; ++attempt) {
      if (!dstk_ok || dstk_n == 0) {
        // refill: the 8 waves' worth deepest live nodes (one pool scan)
        const size_t fill = 8 * want;
        const size_t cap_need = fill + 32 * want;  // room for the pushed children
        if (cap_need > dstk_cap) {
          dfree(dstk);
          dstk = nullptr;
          dstk_cap = 0;
          if ((e = dmalloc(&dstk, cap_need * 4)) != cudaSuccess) return e;
          dstk_cap = cap_need;
        }
        ++deep_fills;
        if ((e = deep_scan(fill, limit, s, dstk, &dstk_n)) != cudaSuccess) return e;
        dstk_ok = true;
        if (dstk_n == 0) break;  // nothing live below the limit
      }
      // pop the top window (the most recently pushed, i.e. deepest, nodes);
      // entries that became holes or stale since they were pushed drop out
      const size_t w = std::min(want, dstk_n);
      KeyBelowLimit pk{key, limit};
      size_t need = 0;
      cub::DeviceSelect::If(nullptr, need, dstk + (dstk_n - w), sel, counter,
                            static_cast<int>(w), pk, s);
      if ((e = ensure_temp(need)) != cudaSuccess) return e;
      cub::DeviceSelect::If(temp, need, dstk + (dstk_n - w), sel, counter, static_cast<int>(w),
                            pk, s);
      if ((e = cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      n = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
      dstk_n -= w;
    }
  }
  if (n) {
    mark_holes<<<grid_for(n, 256), 256, 0, s>>>(key, sel, n);
    holes += n;
    if (tau != 0 && cand_n) {  // the candidate list must not hold holes
      NotHole ph{key};
      size_t need2 = 0;
      cub::DeviceSelect::If(nullptr, need2, cand, cand_tmp, counter, static_cast<int>(cand_n), ph,
                            s);
      if ((e = ensure_temp(need2)) != cudaSuccess) return e;
      cub::DeviceSelect::If(temp, need2, cand, cand_tmp, counter, static_cast<int>(cand_n), ph,
                            s);
      if ((e = cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
        return e;
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      std::swap(cand, cand_tmp);
      cand_n = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
    }
  }
  *n_out = n;
  return cudaGetLastError();
}

cudaError_t Frontier::expand_selected(size_t n_sel, cudaStream_t s) {
  if (n_sel == 0) return cudaSuccess;
  expand<<<grid_for(n_sel * 8, 256), 256, 0, s>>>(nodes, split, vol, sel, n_sel, kids, kid_vol,
                                                   nullptr, nullptr, nullptr);
  return cudaGetLastError();
}

cudaError_t Frontier::gather_selected(size_t n, cudaStream_t s, gosma_node* out_nodes,
                                      int8_t* out_split, double* out_vol) {
  if (n == 0) return cudaSuccess;
  gather_sel<<<grid_for(n, 256), 256, 0, s>>>(nodes, split, vol, sel, n, out_nodes, out_split,
                                              out_vol);
  return cudaGetLastError();
}

cudaError_t Frontier::upload_device(const gosma_node* d_nodes, const int8_t* d_split,
                                    const double* d_vol, size_t n, cudaStream_t s) {
  drop_deep();
  cudaError_t e;
  if ((e = grow(size + n, s)) != cudaSuccess) return e;
  e = cudaMemcpyAsync(nodes + size, d_nodes, n * sizeof(gosma_node), cudaMemcpyDeviceToDevice, s);
  e = chain(e, cudaMemcpyAsync(split + size, d_split, n, cudaMemcpyDeviceToDevice, s));
  e = chain(e, cudaMemcpyAsync(vol + size, d_vol, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (e != cudaSuccess) return e;
  keys_of<<<grid_for(n, 256), 256, 0, s>>>(nodes + size, n, key + size);
  e = chain(cudaGetLastError(), cudaStreamSynchronize(s));
  if (e != cudaSuccess) return e;
  size += n;
  known_min = 0;  // imported keys may lie below the cached minimum
  tau = 0;
  return cudaSuccess;
}

cudaError_t Frontier::wave_lists(size_t n_sel, cudaStream_t s) {
  if (n_sel == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(list_counts, 0, 2 * sizeof(unsigned long long), s);
  if (e != cudaSuccess) return e;
  split_lists<<<grid_for(n_sel, 256), 256, 0, s>>>(split, sel, n_sel, rot_list, trans_list,
                                                    list_counts);
  return cudaGetLastError();
}

cudaError_t Frontier::expand_selected_cached(size_t n_sel, cudaStream_t s, size_t* n_cuboids) {
  *n_cuboids = 0;
  if (n_sel == 0) return cudaSuccess;
  cuboid_counts<<<grid_for(n_sel + 1, 256), 256, 0, s>>>(split, sel, n_sel, tcnt);
  size_t need = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, need, tcnt, toff, static_cast<int>(n_sel + 1), s);
  cudaError_t e = ensure_temp(need);
  if (e != cudaSuccess) return e;
  cub::DeviceScan::ExclusiveSum(temp, need, tcnt, toff, static_cast<int>(n_sel + 1), s);
  expand<<<grid_for(n_sel * 8, 256), 256, 0, s>>>(nodes, split, vol, sel, n_sel, kids, kid_vol,
                                                   toff, tidx, tnodes);
  unsigned int total = 0;
  if ((e = cudaMemcpyAsync(h_counter, toff + n_sel, sizeof(unsigned int),
                           cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  std::memcpy(&total, h_counter, sizeof(unsigned int));
  *n_cuboids = total;
  return cudaGetLastError();
}

cudaError_t Frontier::improving_children(size_t n_kids, double bound, cudaStream_t s,
                                         std::vector<ImprovingChild>* out) {
  out->clear();
  if (n_kids == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (n_kids > pmin_cap) {
    dfree(kid_pmin);
    kid_pmin = nullptr;
    pmin_cap = 0;
    if ((e = dmalloc(&kid_pmin, kid_cap * sizeof(double))) != cudaSuccess) return e;
    pmin_cap = kid_cap;
  }
  if (!rec) {
    if ((e = dmalloc(&rec, 4096 * sizeof(ImprovingChild))) != cudaSuccess) return e;
    rec_cap = 4096;
  }
  size_t bytes = 0;
  cub::DeviceScan::ExclusiveScan(nullptr, bytes, kid_upper, kid_pmin, MinOp(), bound,
                                 static_cast<int>(n_kids), s);
  if ((e = ensure_temp(bytes)) != cudaSuccess) return e;
  bytes = temp_bytes;
  if ((e = cub::DeviceScan::ExclusiveScan(temp, bytes, kid_upper, kid_pmin, MinOp(), bound,
                                          static_cast<int>(n_kids), s)) != cudaSuccess)
    return e;
  // every record is kept (the list grows and the flags are re-run when a wave
  // has more than fit), so the replay below is the reference's in-order one
  for (int pass = 0; pass < 2; ++pass) {
    if ((e = cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
    flag_records<<<grid_cap(n_kids, 256), 256, 0, s>>>(kid_upper, kid_pmin, kids, n_kids, rec,
                                                       counter, static_cast<unsigned>(rec_cap));
    if ((e = cudaMemcpyAsync(h_counter, counter, sizeof(unsigned long long),
                             cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    if (*h_counter <= rec_cap) break;
    dfree(rec);
    rec = nullptr;
    rec_cap = 0;
    const size_t c = static_cast<size_t>(*h_counter) * 2;
    if ((e = dmalloc(&rec, c * sizeof(ImprovingChild))) != cudaSuccess) return e;
    rec_cap = c;
  }
  const size_t m = std::min<size_t>(*h_counter, rec_cap);
  out->resize(m);
  if (m && (e = cudaMemcpy(out->data(), rec, m * sizeof(ImprovingChild),
                           cudaMemcpyDeviceToHost)) != cudaSuccess)
    return e;
  std::sort(out->begin(), out->end(),
            [](const ImprovingChild& a, const ImprovingChild& b) { return a.index < b.index; });
  return cudaSuccess;
}

cudaError_t Frontier::route_append(size_t n_kids, double dstar, double finish, cudaStream_t s,
                                   RouteStats* out) {
  SubTimer tm(this, s);
  cudaError_t e;
  RouteStats zero;
  std::memcpy(h_stats, &zero, sizeof(RouteStats));
  if ((e = cudaMemcpyAsync(stats, h_stats, sizeof(RouteStats), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return e;
  // room for every child, so the append needs no host round trip
  if ((e = grow(size + n_kids, s)) != cudaSuccess) return e;
  tm.lap(4);
  if (n_kids) {
    route<<<grid_for(n_kids, 256), 256, 0, s>>>(kids, kid_lower, kid_split, kid_vol, n_kids,
                                                dstar, finish, keep, stats);
    size_t need = 0;
    cub::CountingInputIterator<unsigned int> it(0);
    cub::DeviceSelect::Flagged(nullptr, need, it, keep, kept_idx, counter,
                               static_cast<int>(n_kids), s);
    if ((e = ensure_temp(need)) != cudaSuccess) return e;
    cub::DeviceSelect::Flagged(temp, need, it, keep, kept_idx, counter, static_cast<int>(n_kids),
                               s);
    append_kids_counted<<<grid_for(n_kids, 256), 256, 0, s>>>(
        kids, kid_split, kid_vol, kept_idx, counter, nodes + size, split + size, vol + size,
        key + size);
    if (tau != 0 && cand_n + n_kids > cand_cap) tau = 0;  // list full: rebuild next wave
    if (tau != 0) {
      // appended children below tau join the candidate list (count -> counter[1])
      cub::CountingInputIterator<unsigned int> ia(static_cast<unsigned int>(size));
      NewCandidate pc{key, tau, size, counter};
      size_t need2 = 0;
      cub::DeviceSelect::If(nullptr, need2, ia, cand + cand_n, counter + 1,
                            static_cast<int>(n_kids), pc, s);
      if ((e = ensure_temp(need2)) != cudaSuccess) return e;
      cub::DeviceSelect::If(temp, need2, ia, cand + cand_n, counter + 1, static_cast<int>(n_kids),
                            pc, s);
    }
    if ((e = cudaMemcpyAsync(h_counter, counter, 16, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
  }
  if ((e = cudaMemcpyAsync(h_stats, stats, sizeof(RouteStats), cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  tm.lap(5);
  *out = *h_stats;
  if (n_kids) {
    const size_t kept = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
    // depth-first waves: the kept children (the deepest nodes) go on top of
    // the stack, so the next wave pops them without a pool scan
    if (deep_active && dstk_ok && kept) {
      if (dstk_n + kept <= dstk_cap) {
        iota_u32<<<grid_for(kept, 256), 256, 0, s>>>(dstk + dstk_n,
                                                     static_cast<unsigned int>(size), kept);
        dstk_n += kept;
      } else {
        drop_deep();
      }
    }
    size += kept;
    kids_total += n_kids;
    kids_kept += kept;
    if (tau != 0) cand_n += static_cast<size_t>(*reinterpret_cast<int*>(h_counter + 1));
  }
  return cudaGetLastError();
}

// Drops holes and stale nodes (key >= limit) in place: stale slots become
// holes (their volume is returned), then the live tail is moved into the head
// holes; no reallocation, traffic proportional to the moved nodes.
cudaError_t Frontier::compact(unsigned long long limit, cudaStream_t s, double* dropped) {
  drop_deep();  // slots move
  *dropped = 0.0;
  if (size == 0) return cudaSuccess;
  cudaError_t e;
  RouteStats zero;
  std::memcpy(h_stats, &zero, sizeof(RouteStats));
  if ((e = cudaMemcpyAsync(stats, h_stats, sizeof(RouteStats), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return e;
  if ((e = cudaMemsetAsync(counter, 0, 16, s)) != cudaSuccess) return e;
  if (limit < kHoleKey)
    drop_stale<<<grid_cap(size, 256), 256, 0, s>>>(key, vol, size, limit, &stats->scratch);
  count_live<<<grid_cap(size, 256), 256, 0, s>>>(key, size, counter);
  cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_stats, stats, sizeof(RouteStats), cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  const size_t live = static_cast<size_t>(h_counter[0]);
  *dropped = h_stats->scratch;
  // holes below `live` and live slots at or above it are equally many (<= m)
  const size_t m = size - live;
  if (live > 0 && m > 0) {
    if (2 * m > cidx_cap) {
      dfree(cidx);
      cidx = nullptr;
      if ((e = dmalloc(&cidx, 2 * m * 4)) != cudaSuccess) return e;
      cidx_cap = 2 * m;
    }
    cub::CountingInputIterator<unsigned int> it(0);
    const HeadHole ph{key, static_cast<unsigned int>(live)};
    const TailLive pt{key, static_cast<unsigned int>(live)};
    size_t need = 0, need2 = 0;
    cub::DeviceSelect::If(nullptr, need, it, cidx, counter, static_cast<int>(live), ph, s);
    cub::DeviceSelect::If(nullptr, need2, it + live, cidx + m, counter + 1,
                          static_cast<int>(size - live), pt, s);
    if ((e = ensure_temp(std::max(need, need2))) != cudaSuccess) return e;
    cub::DeviceSelect::If(temp, need, it, cidx, counter, static_cast<int>(live), ph, s);
    cub::DeviceSelect::If(temp, need2, it + live, cidx + m, counter + 1,
                          static_cast<int>(size - live), pt, s);
    move_tail<<<grid_for(m, 256), 256, 0, s>>>(nodes, split, vol, key, cidx, cidx + m, counter);
  }
  size = live;
  holes = 0;
  tau = 0;  // slots moved: the candidate list is rebuilt on the next selection
  return cudaGetLastError();
}

// enforce_capacity (solver.cpp:433-447): keeps the ~keep_n best live nodes
// and folds the rest into the resolved set; their volume and minimum lower
// bound are returned (the caller adds them to the ledger and floor_lower).
cudaError_t Frontier::live_volume(cudaStream_t s, double* out) {
  *out = 0.0;
  if (size == 0) return cudaSuccess;
  RouteStats zero;
  std::memcpy(h_stats, &zero, sizeof(RouteStats));
  cudaError_t e = cudaMemcpyAsync(stats, h_stats, sizeof(RouteStats), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  // live = non-hole keys >= 0: dropped_volume with limit 0 sums every live slot
  dropped_volume<<<grid_cap(size, 256), 256, 0, s>>>(key, vol, size, 0ull, &stats->scratch);
  cudaMemcpyAsync(h_stats, stats, sizeof(RouteStats), cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *out = h_stats->scratch;
  return cudaSuccess;
}

cudaError_t Frontier::fold_to(size_t keep_n, cudaStream_t s, double* folded_volume,
                              double* folded_min) {
  drop_deep();  // slots move
  *folded_volume = 0.0;
  *folded_min = INFINITY;
  double none = 0.0;
  cudaError_t e = compact(kHoleKey, s, &none);  // drop holes: the pool is live nodes only
  if (e != cudaSuccess || size <= keep_n) return e;
  unsigned long long lo = 0, hi = kHoleKey;
  size_t below = 0;
  if ((e = descend(keep_n, kHoleKey, 0.9, s, &lo, &hi, &below, nullptr, nullptr, size, nullptr)) !=
      cudaSuccess)
    return e;
  // fold every key >= tau; with massive ties below the first boundary keep the bin
  const unsigned long long cut = below > 0 ? lo : hi;
  if (cut >= kHoleKey) return cudaSuccess;
  unsigned long long kmin = kHoleKey;
  if ((e = cudaMemcpyAsync(counter, &kmin, 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return e;
  min_key_at_least<<<grid_cap(size, 256), 256, 0, s>>>(key, size, cut, counter);
  if ((e = cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  kmin = h_counter[0];
  if (kmin == kHoleKey) return cudaSuccess;
  *folded_min = key_to_double(kmin);
  return compact(cut, s, folded_volume);
}

}  // namespace gosma

extern "C" int gosma_release_cached_memory(int device) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  {
    std::lock_guard<std::mutex> lk(gosma::g_park_mu);
    for (size_t k = 0; k < gosma::g_parked.size();) {
      if (gosma::g_parked[k].device == device) {
        gosma::free_parked(gosma::g_parked[k]);
        gosma::g_parked.erase(gosma::g_parked.begin() + static_cast<long>(k));
      } else {
        ++k;
      }
    }
    for (size_t k = 0; k < gosma::g_parked_wave.size();) {
      if (gosma::g_parked_wave[k].device == device) {
        gosma::free_parked_wave(gosma::g_parked_wave[k]);
        gosma::g_parked_wave.erase(gosma::g_parked_wave.begin() + static_cast<long>(k));
      } else {
        ++k;
      }
    }
  }
  gosma::purge_cache(device);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaSetDevice(cur);
  return e == cudaSuccess ? GOSMA_OK : GOSMA_ECUDA;
}
