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
#include <cstdint>
#include <cstring>

#include "frontier.hpp"

namespace gosma {

namespace {

constexpr int kBins = 4096;

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
__global__ void digit_hist(const unsigned long long* key, size_t n, unsigned long long limit,
                           int shift, int bits, unsigned long long prefix, int prefix_shift,
                           unsigned int* hist) {
  __shared__ unsigned int sh[kBins];
  const int nb = 1 << bits;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) sh[b] = 0;
  __syncthreads();
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = key[i];
    if (k >= limit) continue;
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

__global__ void cuboid_counts(const int8_t* split, const unsigned int* sel, size_t n_sel,
                              unsigned int* cnt) {
  const size_t k = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (k < n_sel) cnt[k] = split[sel[k]] == 1 ? 1u : 8u;
  if (k == n_sel) cnt[k] = 0u;
}

// Route evaluated children (solver.cpp:396-405).
__global__ void route(gosma_node* kids, const double* lower, const int8_t* split,
                      const double* kid_vol, size_t n, double dstar, int* keep,
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
    } else if (split[i] < 0) {
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

__global__ void min_upper_key(const double* upper, size_t n, ArgMin* out) {
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long best = ~0ull;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double u = upper[i];
    if (u < INFINITY) best = min(best, order_key(u));
  }
  const unsigned long long r = BR(tmp).Reduce(best, cub::Min());
  if (threadIdx.x == 0 && r != ~0ull) atomicMin(&out->key, r);
}

// First index attaining the minimal key (deterministic argmin).
__global__ void first_index_of_key(const double* upper, size_t n, ArgMin* out) {
  const unsigned long long k = out->key;
  if (k == ~0ull) return;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    if (order_key(upper[i]) == k) atomicMin(&out->index, static_cast<unsigned long long>(i));
  }
}

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

cudaError_t Frontier::reserve(size_t cap_nodes, size_t wave) {
  cudaError_t e = cudaSuccess;
  if (cap_nodes > cap) {
    if ((e = cudaMalloc(&nodes, cap_nodes * sizeof(gosma_node))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&split, cap_nodes)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&vol, cap_nodes * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&key, cap_nodes * 8)) != cudaSuccess) return e;
    cap = cap_nodes;
  }
  if (wave > sel_cap) {
    cudaFree(sel);
    cudaFree(tcnt);
    cudaFree(toff);
    if ((e = cudaMalloc(&sel, wave * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&tcnt, (wave + 1) * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&toff, (wave + 1) * 4)) != cudaSuccess) return e;
    sel_cap = wave;
  }
  const size_t nk = wave * 8;
  if (nk > kid_cap) {
    cudaFree(kids);
    cudaFree(kid_lower);
    cudaFree(kid_upper);
    cudaFree(kid_split);
    cudaFree(kid_vol);
    cudaFree(keep);
    cudaFree(kept_idx);
    cudaFree(tidx);
    cudaFree(tnodes);
    cudaFree(tself);
    if ((e = cudaMalloc(&tidx, nk * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&tnodes, nk * sizeof(gosma_node))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&tself, nk * 4 * sizeof(double))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kids, nk * sizeof(gosma_node))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kid_lower, nk * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kid_upper, nk * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kid_split, nk)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kid_vol, nk * 8)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&keep, nk * 4)) != cudaSuccess) return e;
    if ((e = cudaMalloc(&kept_idx, nk * 4)) != cudaSuccess) return e;
    kid_cap = nk;
  }
  if (!stats) {
    if ((e = cudaMalloc(&stats, sizeof(RouteStats))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&amin, sizeof(ArgMin))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&counter, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    if ((e = cudaMalloc(&hist, kBins * sizeof(unsigned int))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&h_stats, sizeof(RouteStats))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&h_amin, sizeof(ArgMin))) != cudaSuccess) return e;
    if ((e = cudaMallocHost(&h_counter, 2 * sizeof(unsigned long long))) != cudaSuccess) return e;
    h_hist.resize(kBins);
  }
  return e;
}

void Frontier::release() {
  cudaFree(nodes);
  cudaFree(split);
  cudaFree(vol);
  cudaFree(key);
  cudaFree(sel);
  cudaFree(hist);
  cudaFree(kids);
  cudaFree(kid_lower);
  cudaFree(kid_upper);
  cudaFree(kid_split);
  cudaFree(kid_vol);
  cudaFree(keep);
  cudaFree(kept_idx);
  cudaFree(tcnt);
  cudaFree(toff);
  cudaFree(tidx);
  cudaFree(tnodes);
  cudaFree(tself);
  tcnt = toff = nullptr;
  tidx = nullptr;
  tnodes = nullptr;
  tself = nullptr;
  cudaFree(stats);
  cudaFree(amin);
  cudaFree(counter);
  cudaFree(temp);
  cudaFreeHost(h_stats);
  cudaFreeHost(h_amin);
  cudaFreeHost(h_counter);
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
  amin = nullptr;
  counter = nullptr;
  temp = nullptr;
  h_stats = nullptr;
  h_amin = nullptr;
  h_counter = nullptr;
  size = holes = cap = sel_cap = kid_cap = temp_bytes = 0;
}

cudaError_t Frontier::ensure_temp(size_t bytes) {
  if (bytes <= temp_bytes) return cudaSuccess;
  cudaFree(temp);
  temp = nullptr;
  const cudaError_t e = cudaMalloc(&temp, bytes);
  if (e == cudaSuccess) temp_bytes = bytes;
  return e;
}

cudaError_t Frontier::grow(size_t need, cudaStream_t s) {
  if (need <= cap) return cudaSuccess;
  const size_t c = std::max(need, 2 * cap);
  gosma_node* n2 = nullptr;
  int8_t* s2 = nullptr;
  double* v2 = nullptr;
  unsigned long long* k2 = nullptr;
  cudaError_t e;
  if ((e = cudaMalloc(&n2, c * sizeof(gosma_node))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&s2, c)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&v2, c * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&k2, c * 8)) != cudaSuccess) return e;
  if (size) {
    cudaMemcpyAsync(n2, nodes, size * sizeof(gosma_node), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(s2, split, size, cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(v2, vol, size * sizeof(double), cudaMemcpyDeviceToDevice, s);
    cudaMemcpyAsync(k2, key, size * 8, cudaMemcpyDeviceToDevice, s);
  }
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  cudaFree(nodes);
  cudaFree(split);
  cudaFree(vol);
  cudaFree(key);
  nodes = n2;
  split = s2;
  vol = v2;
  key = k2;
  cap = c;
  return cudaSuccess;
}

cudaError_t Frontier::upload(const gosma_node* h_nodes, const int8_t* h_split,
                             const double* h_vol, size_t n, cudaStream_t s) {
  cudaError_t e;
  if ((e = grow(size + n, s)) != cudaSuccess) return e;
  std::vector<unsigned long long> k(n);
  for (size_t i = 0; i < n; ++i) k[i] = host_order_key(h_nodes[i].lower);
  cudaMemcpyAsync(nodes + size, h_nodes, n * sizeof(gosma_node), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(split + size, h_split, n, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(vol + size, h_vol, n * sizeof(double), cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(key + size, k.data(), n * 8, cudaMemcpyHostToDevice, s);
  size += n;
  return cudaStreamSynchronize(s);
}

cudaError_t Frontier::min_key(cudaStream_t s, unsigned long long* out) {
  if (size == 0) {
    *out = kHoleKey;
    return cudaSuccess;
  }
  size_t need = 0;
  cub::DeviceReduce::Min(nullptr, need, key, counter, static_cast<int>(size), s);
  cudaError_t e = ensure_temp(need);
  if (e != cudaSuccess) return e;
  cub::DeviceReduce::Min(temp, need, key, counter, static_cast<int>(size), s);
  cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
  e = cudaStreamSynchronize(s);
  *out = h_counter[0];
  return e;
}

cudaError_t Frontier::select_smallest(size_t want, unsigned long long limit, cudaStream_t s,
                                      size_t* n_out) {
  *n_out = 0;
  if (size == 0 || want == 0) return cudaSuccess;
  want = std::min(want, sel_cap);
  // Digit schedule over the 64-bit key: 12,12,12,12,12,4 bits.
  static const int kShift[6] = {52, 40, 28, 16, 4, 0};
  static const int kBits[6] = {12, 12, 12, 12, 12, 4};
  unsigned long long prefix = 0, lo_key = 0, hi_key = limit;
  size_t below = 0;  // count of keys < lo_key
  cudaError_t e;
  for (int lvl = 0; lvl < 6; ++lvl) {
    const int shift = kShift[lvl], bits = kBits[lvl];
    const int pshift = shift + bits;  // bits above this digit form the prefix
    if ((e = cudaMemsetAsync(hist, 0, kBins * 4, s)) != cudaSuccess) return e;
    digit_hist<<<grid_cap(size, 256), 256, 0, s>>>(key, size, limit, shift, bits, prefix,
                                                   lvl == 0 ? 64 : pshift, hist);
    const int nb = 1 << bits;
    if ((e = cudaMemcpyAsync(h_hist.data(), hist, nb * 4, cudaMemcpyDeviceToHost, s)) !=
        cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    const unsigned long long base = (lvl == 0) ? 0ull : (prefix << pshift);
    size_t cum = below;
    int b = 0;
    for (; b < nb; ++b) {
      if (cum + h_hist[b] > want) break;
      cum += h_hist[b];
    }
    if (b == nb) {  // everything under this prefix fits
      if (lvl == 0) {
        lo_key = hi_key = limit;
      } else {
        const unsigned long long end = base + (1ull << pshift);
        lo_key = hi_key = (end == 0 || end > limit) ? limit : end;
      }
      below = cum;
      break;
    }
    lo_key = base + (static_cast<unsigned long long>(b) << shift);
    const unsigned long long end = lo_key + (1ull << shift);
    hi_key = (end == 0 || end > limit) ? limit : end;
    below = cum;
    if (below >= want / 2 || lvl == 5) break;
    prefix = (lvl == 0 ? 0ull : (prefix << bits)) | static_cast<unsigned long long>(b);
  }
  // keys < lo_key (count `below` <= want), then fill from [lo_key, hi_key)
  cub::CountingInputIterator<unsigned int> it(0);
  size_t need = 0;
  KeyBelow p1{key, 0ull, lo_key};
  cub::DeviceSelect::If(nullptr, need, it, sel, counter, static_cast<int>(size), p1, s);
  if ((e = ensure_temp(need)) != cudaSuccess) return e;
  size_t n1 = 0;
  if (below > 0) {
    cub::DeviceSelect::If(temp, need, it, sel, counter, static_cast<int>(size), p1, s);
    cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    n1 = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
  }
  size_t n2 = 0;
  if (n1 < want && hi_key > lo_key) {
    // fill from the boundary bin, chunked through kept_idx (kid_cap slots)
    KeyBelow p2{key, lo_key, hi_key};
    size_t done = 0;
    while (done < size && n1 + n2 < want) {
      const size_t chunk = std::min(size - done, kid_cap);
      cub::CountingInputIterator<unsigned int> it2(static_cast<unsigned int>(done));
      size_t need2 = 0;
      cub::DeviceSelect::If(nullptr, need2, it2, kept_idx, counter, static_cast<int>(chunk), p2,
                            s);
      if ((e = ensure_temp(need2)) != cudaSuccess) return e;
      cub::DeviceSelect::If(temp, need2, it2, kept_idx, counter, static_cast<int>(chunk), p2, s);
      cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
      if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
      const size_t got = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
      const size_t take = std::min(got, want - n1 - n2);
      if (take)
        cudaMemcpyAsync(sel + n1 + n2, kept_idx, take * 4, cudaMemcpyDeviceToDevice, s);
      n2 += take;
      done += chunk;
    }
  }
  const size_t n = n1 + n2;
  if (n) {
    mark_holes<<<grid_for(n, 256), 256, 0, s>>>(key, sel, n);
    holes += n;
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

cudaError_t Frontier::best_child(size_t n_kids, cudaStream_t s, int* index, double* value) {
  ArgMin init;
  cudaError_t e = cudaMemcpyAsync(amin, &init, sizeof(ArgMin), cudaMemcpyHostToDevice, s);
  if (e != cudaSuccess) return e;
  const unsigned g = grid_cap(n_kids, 256);
  min_upper_key<<<g, 256, 0, s>>>(kid_upper, n_kids, amin);
  first_index_of_key<<<g, 256, 0, s>>>(kid_upper, n_kids, amin);
  if ((e = cudaMemcpyAsync(h_amin, amin, sizeof(ArgMin), cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  if (h_amin->key == ~0ull || h_amin->index == ~0ull) {
    *index = -1;
    *value = INFINITY;
    return cudaSuccess;
  }
  *index = static_cast<int>(h_amin->index);
  *value = key_to_double(h_amin->key);
  return cudaSuccess;
}

cudaError_t Frontier::route_append(size_t n_kids, double dstar, cudaStream_t s,
                                   RouteStats* out) {
  cudaError_t e;
  RouteStats zero;
  if ((e = cudaMemcpyAsync(stats, &zero, sizeof(RouteStats), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return e;
  size_t kept = 0;
  if (n_kids) {
    route<<<grid_for(n_kids, 256), 256, 0, s>>>(kids, kid_lower, kid_split, kid_vol, n_kids,
                                                dstar, keep, stats);
    size_t need = 0;
    cub::CountingInputIterator<unsigned int> it(0);
    cub::DeviceSelect::Flagged(nullptr, need, it, keep, kept_idx, counter,
                               static_cast<int>(n_kids), s);
    if ((e = ensure_temp(need)) != cudaSuccess) return e;
    cub::DeviceSelect::Flagged(temp, need, it, keep, kept_idx, counter, static_cast<int>(n_kids),
                               s);
    if ((e = cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    kept = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
    if ((e = grow(size + kept, s)) != cudaSuccess) return e;
    if (kept) {
      append_kids<<<grid_for(kept, 256), 256, 0, s>>>(kids, kid_split, kid_vol, kept_idx, kept,
                                                      nodes + size, split + size, vol + size,
                                                      key + size);
    }
  }
  if ((e = cudaMemcpyAsync(h_stats, stats, sizeof(RouteStats), cudaMemcpyDeviceToHost, s)) !=
      cudaSuccess)
    return e;
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  *out = *h_stats;
  size += kept;
  return cudaGetLastError();
}

cudaError_t Frontier::compact(unsigned long long limit, cudaStream_t s, double* dropped) {
  *dropped = 0.0;
  if (size == 0) return cudaSuccess;
  cudaError_t e;
  RouteStats zero;
  if ((e = cudaMemcpyAsync(stats, &zero, sizeof(RouteStats), cudaMemcpyHostToDevice, s)) !=
      cudaSuccess)
    return e;
  dropped_volume<<<grid_cap(size, 256), 256, 0, s>>>(key, vol, size, limit, &stats->scratch);
  // surviving slots: key < limit (holes carry the maximal key)
  unsigned int* idx = nullptr;
  if ((e = cudaMalloc(&idx, size * 4)) != cudaSuccess) return e;
  cub::CountingInputIterator<unsigned int> it(0);
  KeyBelow p{key, 0ull, limit};
  size_t need = 0;
  cub::DeviceSelect::If(nullptr, need, it, idx, counter, static_cast<int>(size), p, s);
  if ((e = ensure_temp(need)) != cudaSuccess) return e;
  cub::DeviceSelect::If(temp, need, it, idx, counter, static_cast<int>(size), p, s);
  cudaMemcpyAsync(h_counter, counter, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(h_stats, stats, sizeof(RouteStats), cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  const size_t n = static_cast<size_t>(*reinterpret_cast<int*>(h_counter));
  *dropped = h_stats->scratch;
  gosma_node* n2 = nullptr;
  int8_t* s2 = nullptr;
  double* v2 = nullptr;
  unsigned long long* k2 = nullptr;
  const size_t c = std::max<size_t>(n + n / 4, 1024);  // shrink-to-fit with headroom
  if ((e = cudaMalloc(&n2, c * sizeof(gosma_node))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&s2, c)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&v2, c * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&k2, c * 8)) != cudaSuccess) return e;
  if (n)
    gather_pool<<<grid_for(n, 256), 256, 0, s>>>(nodes, split, vol, key, idx, n, n2, s2, v2, k2);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  cudaFree(idx);
  cudaFree(nodes);
  cudaFree(split);
  cudaFree(vol);
  cudaFree(key);
  nodes = n2;
  split = s2;
  vol = v2;
  key = k2;
  size = n;
  cap = c;
  holes = 0;
  return cudaGetLastError();
}

cudaError_t Frontier::fold_to(size_t keep_n, cudaStream_t s, double* folded_volume,
                              double* folded_min) {
  *folded_volume = 0.0;
  *folded_min = INFINITY;
  double none = 0.0;
  cudaError_t e = compact(kHoleKey, s, &none);  // drop holes: the pool is live nodes only
  if (e != cudaSuccess || size <= keep_n) return e;
  // full sort of the keys (rare path)
  unsigned long long *k0 = nullptr, *k1 = nullptr;
  unsigned int *i0 = nullptr, *i1 = nullptr;
  if ((e = cudaMalloc(&k0, size * 8)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&k1, size * 8)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&i0, size * 4)) != cudaSuccess) return e;
  if ((e = cudaMalloc(&i1, size * 4)) != cudaSuccess) return e;
  cudaMemcpyAsync(k0, key, size * 8, cudaMemcpyDeviceToDevice, s);
  std::vector<unsigned int> iota(size);
  for (size_t i = 0; i < size; ++i) iota[i] = static_cast<unsigned int>(i);
  cudaMemcpyAsync(i0, iota.data(), size * 4, cudaMemcpyHostToDevice, s);
  cub::DoubleBuffer<unsigned long long> kb(k0, k1);
  cub::DoubleBuffer<unsigned int> vb(i0, i1);
  size_t need = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, need, kb, vb, static_cast<int>(size), 0, 64, s);
  if ((e = ensure_temp(need)) != cudaSuccess) return e;
  cub::DeviceRadixSort::SortPairs(temp, need, kb, vb, static_cast<int>(size), 0, 64, s);
  unsigned long long kmin = 0;
  std::vector<unsigned int> ord(size);
  std::vector<double> hv(size);
  cudaMemcpyAsync(&kmin, kb.Current() + keep_n, 8, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(ord.data(), vb.Current(), size * 4, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(hv.data(), vol, size * 8, cudaMemcpyDeviceToHost, s);
  if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
  double fv = 0.0;
  for (size_t i = keep_n; i < size; ++i) fv += hv[ord[i]];
  *folded_volume = fv;
  *folded_min = key_to_double(kmin);
  const size_t nf = size - keep_n;
  mark_holes<<<grid_for(nf, 256), 256, 0, s>>>(key, vb.Current() + keep_n, nf);
  holes += nf;
  e = compact(kHoleKey, s, &none);
  cudaFree(k0);
  cudaFree(k1);
  cudaFree(i0);
  cudaFree(i1);
  return e;
}

}  // namespace gosma
