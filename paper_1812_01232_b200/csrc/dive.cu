// Discovery-dive beam on the device (dive.hpp; solver.cpp:459-568).
//
// Per iteration, on one stream and without a host round trip:
//   beam_expand   beam entry e -> children 8e..8e+7 (subdivide_adaptive order,
//                 se3.cpp:124-145), the iteration's skip value (the worst
//                 sector candidate) and the stop test (empty beam / budget);
//   K1            bounds of the children on the blurred context (the item
//                 count is read on the device);
//   offer_*       per sector, the first child (in index order) with the
//                 smallest finite upper bound below the sector's candidate -
//                 exactly the host's sequential `offer` loop - becomes the
//                 candidate (upper bounds of children with lower >= skip are
//                 +inf, as evaluate_branch_batch's skip gives them);
//   beam_select   per sector the `quota` splittable children with the lowest
//                 (lower, index) - the host's stable sort + quota - packed in
//                 sector order into the other beam buffer.
// Two iterations (beam A -> B -> A) are captured into one CUDA graph and
// replayed; after the stop flag is set every kernel is a no-op.
#include "dive.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "capi_internal.hpp"

namespace gosma {

namespace {

constexpr unsigned long long kNone = ~0ull;

struct DiveVars {
  unsigned long long used;    // children bounded so far (incl. the host part)
  unsigned long long budget;  // children budget
  double skip;                // this iteration's skip_upper_at
  double floor;               // is_splittable floor
  long long nkids;            // children this iteration (0 once stopped)
  unsigned count[2];          // beam sizes (ping-pong)
  int stop;
  int it_left;                // iterations left (the host loop's kMaxIt)
};

struct DiveDev {
  DiveVars* v;
  DiveEntry* beam[2];
  gosma_node* kids;
  unsigned* ksec;
  double* lo;
  double* up;
  int8_t* sp;
  DiveBest* best;
  unsigned long long* key;
  unsigned long long* idx;
  unsigned* cnt;   // beam entries per sector (this beam)
  unsigned* off;   // their offsets
  unsigned* ncnt;  // entries per sector of the next beam
  unsigned* sel;
  int R, quota;
  unsigned cap_beam, cap_kids;
};

__device__ __forceinline__ unsigned long long okey(double v) {
  // order-preserving map of a double to an unsigned key (finite values)
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
  return (b >> 63) ? ~b : (b | (1ull << 63));
}

__device__ __forceinline__ gosma_node child_d(const gosma_node& p, int split_rot, int c) {
  // solver.cpp child_of / subdivide_adaptive child order (se3.cpp:124-145)
  const int sx = (c & 4) ? 1 : -1, sy = (c & 2) ? 1 : -1, sz = (c & 1) ? 1 : -1;
  gosma_node k = p;
  if (split_rot == 1) {
    const double h = 0.5 * p.rhw;
    k.rc[0] = p.rc[0] + h * sx;
    k.rc[1] = p.rc[1] + h * sy;
    k.rc[2] = p.rc[2] + h * sz;
    k.rhw = h;
  } else {
    for (int a = 0; a < 3; ++a) {
      const double h = 0.5 * p.thw[a];
      k.tc[a] = p.tc[a] + h * (a == 0 ? sx : (a == 1 ? sy : sz));
      k.thw[a] = h;
    }
  }
  return k;
}

__device__ __forceinline__ bool splittable_d(const gosma_node& n, double floor) {
  return n.rhw > floor || fmax(fmax(n.thw[0], n.thw[1]), n.thw[2]) > floor;
}

__global__ void beam_expand(DiveDev d, int from) {
  DiveVars& v = *d.v;
  const unsigned n = v.count[from];
  const bool halt = v.stop || v.it_left <= 0 || n == 0 || v.used + 8ull * n > v.budget;
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t == 0) {  // (stop / it_left are updated by offer_commit_select: read-only here)
    v.nkids = halt ? 0 : 8ll * n;
    double skip = -INFINITY;  // the worst sector candidate (+inf until all are seeded)
    for (int s = 0; s < d.R; ++s) skip = fmax(skip, d.best[s].value);
    v.skip = skip;
  }
  if (halt || t >= 8u * n) return;
  const DiveEntry& e = d.beam[from][t >> 3];
  d.kids[t] = child_d(e.node, e.split, static_cast<int>(t & 7));
  d.ksec[t] = e.sector;
}

__device__ __forceinline__ bool offers(const DiveDev& d, long long i) {
  const double u = d.up[i];
  return !(d.lo[i] >= d.v->skip) && isfinite(u) && u < d.best[d.ksec[i]].value;
}

__global__ void offer_min(DiveDev d) {
  const long long n = d.v->nkids;
  for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (offers(d, i)) atomicMin(&d.key[d.ksec[i]], okey(d.up[i]));
}

__global__ void offer_idx(DiveDev d) {
  const long long n = d.v->nkids;
  for (long long i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x)
    if (offers(d, i) && okey(d.up[i]) == d.key[d.ksec[i]])
      atomicMin(&d.idx[d.ksec[i]], static_cast<unsigned long long>(i));
}

// Single CTA: commit the sector candidates, then select the next beam.
__global__ void __launch_bounds__(1024) offer_commit_select(DiveDev d, int to) {
  DiveVars& v = *d.v;
  const long long n = v.nkids;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int s = threadIdx.x; s < d.R; s += blockDim.x) {
    const unsigned long long i = d.idx[s];
    if (i != kNone) d.best[s] = DiveBest{d.up[i], d.kids[i]};
    d.key[s] = kNone;
    d.idx[s] = kNone;
  }
  // per sector: the quota smallest (lower, index) splittable children; a
  // sector's children are contiguous (the beam is in sector order)
  for (int s = warp; s < d.R; s += nw) {
    unsigned c = 0;
    if (n > 0) {
      // [a, b): children of sector s - 8 per beam entry of the sector, whose
      // offset and count the previous selection left in off / cnt
      const long long a = 8ll * d.off[s];
      const long long b = a + 8ll * d.cnt[s];
      // this lane's candidates (a sector has at most quota * 8 <= 128
      // children: <= 4 per lane), read once
      constexpr int kPer = 4;
      double cl[kPer];
      long long ci[kPer];
      for (int k = 0; k < kPer; ++k) {
        const long long i = a + lane + 32ll * k;
        const bool ok = i < b && splittable_d(d.kids[i], v.floor);
        cl[k] = ok ? d.lo[i] : INFINITY;
        ci[k] = ok ? i : -1;
      }
      double pl = -INFINITY;
      long long pi = -1;
      for (; c < static_cast<unsigned>(d.quota); ++c) {
        double bl = INFINITY;
        long long bi = -1;
#pragma unroll
        for (int k = 0; k < kPer; ++k) {
          const long long i = ci[k];
          if (i < 0) continue;
          const double l = cl[k];
          const bool after = l > pl || (l == pl && i > pi);
          const bool better = bi < 0 || l < bl || (l == bl && i < bi);
          if (after && better) {
            bl = l;
            bi = i;
          }
        }
        // warp argmin over (lower, index)
        for (int o = 16; o > 0; o >>= 1) {
          const double ol = __shfl_xor_sync(0xffffffffu, bl, o);
          const long long oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (oi >= 0 && (bi < 0 || ol < bl || (ol == bl && oi < bi))) {
            bl = ol;
            bi = oi;
          }
        }
        if (bi < 0) break;
        if (lane == 0) d.sel[static_cast<unsigned>(s) * d.quota + c] = static_cast<unsigned>(bi);
        pl = bl;
        pi = bi;
      }
    }
    if (lane == 0) d.ncnt[s] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned total = 0;
    for (int s = 0; s < d.R; ++s) {
      d.off[s] = total;
      d.cnt[s] = d.ncnt[s];
      total += d.ncnt[s];
    }
    v.count[to] = total;
    v.used += static_cast<unsigned long long>(n);
    if (n == 0)
      v.stop = 1;
    else
      --v.it_left;
  }
  __syncthreads();
  for (int s = warp; s < d.R; s += nw) {
    const unsigned c = d.cnt[s], o = d.off[s];
    for (unsigned r = lane; r < c; r += 32) {
      const unsigned i = d.sel[static_cast<unsigned>(s) * d.quota + r];
      DiveEntry e;
      e.node = d.kids[i];
      e.node.lower = d.lo[i];
      e.split = d.sp[i];
      e.sector = static_cast<unsigned>(s);
      d.beam[to][o + r] = e;
    }
  }
}

size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

// Carves the device block; returns its size (p == nullptr: size only).
size_t carve(char* p, int R, int quota, DiveDev* d) {
  const size_t cb = static_cast<size_t>(R) * quota, ck = 8 * cb;
  size_t off = 0;
  auto take = [&](size_t bytes) -> char* {
    char* q = p ? p + off : nullptr;
    off += align256(bytes);
    return q;
  };
  d->v = reinterpret_cast<DiveVars*>(take(sizeof(DiveVars)));
  d->beam[0] = reinterpret_cast<DiveEntry*>(take(cb * sizeof(DiveEntry)));
  d->beam[1] = reinterpret_cast<DiveEntry*>(take(cb * sizeof(DiveEntry)));
  d->kids = reinterpret_cast<gosma_node*>(take(ck * sizeof(gosma_node)));
  d->ksec = reinterpret_cast<unsigned*>(take(ck * sizeof(unsigned)));
  d->lo = reinterpret_cast<double*>(take(ck * sizeof(double)));
  d->up = reinterpret_cast<double*>(take(ck * sizeof(double)));
  d->sp = reinterpret_cast<int8_t*>(take(ck));
  d->best = reinterpret_cast<DiveBest*>(take(R * sizeof(DiveBest)));
  d->key = reinterpret_cast<unsigned long long*>(take(R * 8));
  d->idx = reinterpret_cast<unsigned long long*>(take(R * 8));
  d->cnt = reinterpret_cast<unsigned*>(take(R * 4));
  d->off = reinterpret_cast<unsigned*>(take(R * 4));
  d->ncnt = reinterpret_cast<unsigned*>(take(R * 4));
  d->sel = reinterpret_cast<unsigned*>(take(cb * 4));
  d->R = R;
  d->quota = quota;
  d->cap_beam = static_cast<unsigned>(cb);
  d->cap_kids = static_cast<unsigned>(ck);
  return off;
}

cudaError_t launch_iteration(gosma_ctx* ctx, const DiveDev& d, int from, cudaStream_t s) {
  const unsigned ck = d.cap_kids;
  beam_expand<<<(ck + 255) / 256, 256, 0, s>>>(d, from);
  EvalArgs a{};
  a.nodes = reinterpret_cast<const double*>(d.kids);
  a.n = ck;
  a.n_dev = &d.v->nkids;
  a.skip_upper_at = INFINITY;  // applied in offers(): the same +inf upper bounds
  a.lower = d.lo;
  a.upper = d.up;
  a.split_rot = d.sp;
  a.work = work_counter(ctx, s);
  cudaError_t e = launch_eval_bounds(ctx->dev, a, ctx->sm_count, s);
  if (e != cudaSuccess) return e;
  const unsigned g = std::min<unsigned>((ck + 255) / 256, 4u * ctx->sm_count);
  offer_min<<<g, 256, 0, s>>>(d);
  offer_idx<<<g, 256, 0, s>>>(d);
  offer_commit_select<<<1, 1024, 0, s>>>(d, 1 - from);
  return cudaGetLastError();
}

}  // namespace

int dive_beam_device(gosma_ctx* ctx, const std::vector<DiveEntry>& beam,
                     const std::vector<DiveBest>& best0, unsigned long long used0,
                     unsigned long long budget, int max_it, int quota, double floor,
                     DiveBeamResult* out) {
  const int R = static_cast<int>(best0.size());
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  cudaError_t e = cudaSuccess;
  DiveDev d{};
  const size_t bytes = carve(nullptr, R, quota, &d);
  if (!ctx->dive_buf || ctx->dive_bytes < bytes || ctx->dive_sectors != R ||
      ctx->dive_quota != quota) {
    if (ctx->dive_graph) cudaGraphExecDestroy(ctx->dive_graph);
    ctx->dive_graph = nullptr;
    cudaFree(ctx->dive_buf);
    ctx->dive_buf = nullptr;
    ctx->dive_bytes = 0;
    if ((e = cudaMalloc(&ctx->dive_buf, bytes)) != cudaSuccess) return cuda_error(e, "dive beam");
    ctx->dive_bytes = bytes;
    ctx->dive_sectors = R;
    ctx->dive_quota = quota;
  }
  carve(static_cast<char*>(ctx->dive_buf), R, quota, &d);
  if (beam.size() > d.cap_beam) return set_error(GOSMA_EINVAL, "dive beam larger than its quota");
  if (quota > 16) return set_error(GOSMA_EINVAL, "dive quota above 16 (4 candidates per lane)");
  // state: vars, beam A, sector candidates, empty argmin slots
  DiveVars v{};
  v.used = used0;
  v.budget = budget;
  v.floor = floor;
  v.count[0] = static_cast<unsigned>(beam.size());
  v.it_left = max_it;
  std::vector<unsigned long long> none(R, kNone);
  if ((e = cudaMemcpyAsync(d.v, &v, sizeof v, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (!beam.empty() && (e = cudaMemcpyAsync(d.beam[0], beam.data(),
                                             beam.size() * sizeof(DiveEntry),
                                             cudaMemcpyHostToDevice, s)) != cudaSuccess) ||
      (e = cudaMemcpyAsync(d.best, best0.data(), R * sizeof(DiveBest), cudaMemcpyHostToDevice,
                           s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.key, none.data(), R * 8, cudaMemcpyHostToDevice, s)) !=
          cudaSuccess ||
      (e = cudaMemcpyAsync(d.idx, none.data(), R * 8, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_error(e, "dive upload");
  // the initial beam's per-sector counts and offsets (it is in sector order)
  std::vector<unsigned> cnt(R, 0), off(R, 0);
  for (const DiveEntry& en : beam) ++cnt[en.sector];
  for (int k = 1; k < R; ++k) off[k] = off[k - 1] + cnt[k - 1];
  if ((e = cudaMemcpyAsync(d.cnt, cnt.data(), R * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(d.off, off.data(), R * 4, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)  // cnt / off are host locals
    return cuda_error(e, "dive upload");
  const bool prof = std::getenv("GOSMA_PROFILE") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  if (!ctx->dive_graph) {
    // first use: one plain iteration pair fills the launch caches, then capture
    cudaGraph_t graph = nullptr;
    if ((e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal)) != cudaSuccess)
      return cuda_error(e, "dive capture");
    const cudaError_t e1 = launch_iteration(ctx, d, 0, s);
    const cudaError_t e2 = e1 == cudaSuccess ? launch_iteration(ctx, d, 1, s) : e1;
    e = cudaStreamEndCapture(s, &graph);
    if (e2 != cudaSuccess) e = e2;
    if (e == cudaSuccess) e = cudaGraphInstantiate(&ctx->dive_graph, graph, 0);
    if (graph) cudaGraphDestroy(graph);
    if (e != cudaSuccess) {
      ctx->dive_graph = nullptr;
      return cuda_error(e, "dive graph");
    }
  }
  const auto t1 = std::chrono::steady_clock::now();
  for (int it = 0; it < max_it; it += 2)  // two iterations per graph; it_left stops exactly
    if ((e = cudaGraphLaunch(ctx->dive_graph, s)) != cudaSuccess)
      return cuda_error(e, "dive graph launch");
  out->best.resize(R);
  if ((e = cudaMemcpyAsync(out->best.data(), d.best, R * sizeof(DiveBest), cudaMemcpyDeviceToHost,
                           s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(&v, d.v, sizeof v, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
      (e = cudaStreamSynchronize(s)) != cudaSuccess)
    return cuda_error(e, "dive download");
  out->used = v.used;
  if (prof)
    std::fprintf(stderr, "[gosma profile] dive beam (device): capture %.2f ms, run %.2f ms\n",
                 1e3 * std::chrono::duration<double>(t1 - t0).count(),
                 1e3 * std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count());
  return GOSMA_OK;
}

}  // namespace gosma
