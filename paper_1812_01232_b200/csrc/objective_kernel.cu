// FP64 objective value + gradient on the GPU:
// objective_value / objective_gradient (core/src/objective.cpp:175-334).
//
// * objgrad_block: one CTA evaluates one pose (model rows in shared memory,
//   FP64 throughout: the refiner tests |g| < 1e-6; pair terms below the
//   reference's margin, K < a + b - 64, objective.cpp:17, are skipped exactly
//   as on the host).
// * K6 (objgrad_kernel): a batch of poses, each spread over a grid row of CTAs
//   (CTAs = slices of the pair partners, partial sums added on the host in a
//   fixed order) - gosma_objective_batch.
// * refine_kernel: the GPU-resident local refiner. One CTA (or a cluster of
//   CTAs, each taking a partner slice, totals exchanged through distributed
//   shared memory) runs one start's whole L-BFGS ladder (local_refine /
//   wolfe_search / clamp_to_domain, solver.cpp:37-258) - the discovery dive's
//   SMA ladder and the wave refinements for large mixtures.
//
// Gradient algebra (objective.cpp:254-334), rearranged so no 3x3 matrix is
// stored: J_i v = u_i (u_i.v)(-2 d_i / s2_i) - (v - u_i (u_i.v)) (k_i / d_i)
// is linear in v, so every J_i / R^T / Jl^T product is applied once per row
// (or once per pose) to an accumulated vector. Self pairs are visited as
// ordered pairs (i != j), each side adding its own half of the gradient.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "objective_device.hpp"
#include "objective_math.hpp"
#include "refine_core.hpp"

namespace gosma {

namespace {

constexpr unsigned kFullMask = 0xffffffffu;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

using objmath::RowD;
using objmath::jv;
using objmath::log_z_d;
using objmath::log_z_deriv_d;
using objmath::pair_terms;

// CTA totals of 7 values (fixed tree: warp shuffles, then one warp per value
// over the warps' partials); red holds 7 x 32 + 8 doubles.
__device__ __forceinline__ void block_sum7(double* v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int k = 0; k < 7; ++k) v[k] = wsum(v[k]);
  __syncthreads();
  if (lane == 0)
    for (int k = 0; k < 7; ++k) red[32 * k + warp] = v[k];
  __syncthreads();
  for (int k = warp; k < 7; k += nw) {
    const double t = wsum(lane < nw ? red[32 * k + lane] : 0.0);
    if (lane == 0) red[224 + k] = t;
  }
  __syncthreads();
  for (int k = 0; k < 7; ++k) v[k] = red[224 + k];
}

// CTA minimum (exact, order-free) of a double / an int; red as above.
__device__ __forceinline__ double block_min_d(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(kFullMask, v, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmin(t, red[w]);
  return t;
}
__device__ __forceinline__ int block_min_i(int v, double* red) {
  v = __reduce_min_sync(kFullMask, v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = static_cast<double>(v);
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < static_cast<int>(blockDim.x >> 5); ++w) t = fmin(t, red[w]);
  return static_cast<int>(t);
}

// One CTA evaluates pose x over partner slice `slice` of S: thread = model
// row (strided; with split_rows, row x chunk of the slice), the slice = a
// contiguous range of partners (self rows j != i, then image columns). Every
// thread returns the CTA total {f, g[6]} of the slice in o[0..6]
// (deterministic fixed-tree reduction).
#ifdef GOSMA_OBJ_NOINLINE
__device__ __noinline__
#else
__device__
#endif
    void objgrad_block(const DevModel64& m, const double* x, int slice, int S,
                              RowD* rows, double* red, double* o, bool split_rows = false) {
  const double r0 = x[0], r1 = x[1], r2 = x[2];
  const double t0 = x[3], t1 = x[4], t2 = x[5];
  // check_feasible (objective.cpp:160-166)
  int hit = 0;
  for (int i = threadIdx.x; i < m.n_all; i += blockDim.x) {
    const double dx = m.all_means[3 * i] - t0, dy = m.all_means[3 * i + 1] - t1,
                 dz = m.all_means[3 * i + 2] - t2;
    hit |= sqrt(dx * dx + dy * dy + dz * dz) < m.zeta;
  }
  if (__syncthreads_or(hit)) {
    o[0] = slice == 0 ? INFINITY : 0.0;
    for (int k = 1; k < 7; ++k) o[k] = 0.0;
    return;
  }
  // Rodrigues R (se3.cpp:21-31) and the left Jacobian (objective.cpp:240-250),
  // computed by the CTA's last warp only (FP64 sin / cos / divisions would
  // otherwise occupy the FP64 pipe once per thread) and published in shared
  // memory; every reader comes after the first class's row barrier below, and
  // the last reads precede the trailing barrier of this evaluation.
  __shared__ double rjl[18];
  if (threadIdx.x >= blockDim.x - 32) {
    double R[9], Jl[9];
    objmath::rotation_and_jacobian(r0, r1, r2, R, Jl);
    if (threadIdx.x == blockDim.x - 32)
      for (int e = 0; e < 9; ++e) {
        rjl[e] = R[e];
        rjl[9 + e] = Jl[e];
      }
  }
  const double* const R = rjl;
  const double* const Jl = rjl + 9;
  double fval = 0.0, gt0 = 0.0, gt1 = 0.0, gt2 = 0.0, cr0 = 0.0, cr1 = 0.0, cr2 = 0.0;
  for (int c = 0; c < m.n_classes; ++c) {
    const ClassSpan cs = m.cls[c];
    const double w = m.cls_w[c];
    __syncthreads();
    for (int il = threadIdx.x; il < cs.n1; il += blockDim.x) {
      const int i = cs.o1 + il;
      rows[il] = objmath::make_row(m.mu[3 * i], m.mu[3 * i + 1], m.mu[3 * i + 2], m.sigma2[i],
                                   m.phi1[i], t0, t1, t2);
    }
    __syncthreads();
    // this slice's partners: [p0, p1) over self rows (0..n1-1) then columns
    const int np = cs.n1 + cs.n2;
    const int p0 = np * slice / S;  // np < 2^20, S <= 32: no overflow
    const int p1 = np * (slice + 1) / S;
    // work items: (row, chunk of the slice's partners); split_rows spreads a
    // row over nq threads (n1 * nq <= CTA size: one balanced pass) so one
    // CTA alone fills its SM (the refiner)
    const int nq =
        split_rows ? max(1, min(static_cast<int>(blockDim.x) / cs.n1, p1 - p0)) : 1;
    for (int wi = threadIdx.x; wi < cs.n1 * nq; wi += blockDim.x) {
      const int il = wi % cs.n1, q = wi / cs.n1;
      const int q0 = p0 + (p1 - p0) * q / nq;
      const int q1 = p0 + (p1 - p0) * (q + 1) / nq;
      const RowD a = rows[il];
      const double uix = a.ux * a.d, uiy = a.uy * a.d, uiz = a.uz * a.d;  // u_i
      const double cu = 2.0 * a.zl * a.is2;
      double fself = 0.0, fcross = 0.0;
      if (slice == 0 && q == 0) {  // diagonal (objective.cpp:201-203, 268-274)
        const double term = 0.5 * a.k / tanh(a.k);
        fself += a.phi * a.phi * term;
        const double dlog = 2.0 * (log_z_deriv_d(2.0 * a.k) - a.zl);
        const double sd = a.phi * a.phi * term * dlog * (-2.0 * a.is2);
        gt0 += w * uix * sd;
        gt1 += w * uiy * sd;
        gt2 += w * uiz * sd;
      }
      const double vix = a.ux * a.k, viy = a.uy * a.k, viz = a.uz * a.k;
      // self pairs, ordered (i != j): this row's half of each pair
      double sx = 0.0, sy = 0.0, sz = 0.0, su = 0.0;
      const int s_end = min(q1, cs.n1);
      for (int jl = q0; jl < s_end; ++jl) {
        if (jl == il) continue;
        const RowD b = rows[jl];
        const double ex = vix + b.ux * b.k, ey = viy + b.uy * b.k, ez = viz + b.uz * b.k;
        const double K = sqrt(ex * ex + ey * ey + ez * ez);
        if (K < a.k + b.k - objmath::kNegligible) continue;
        double eK, zl;
        pair_terms(K, a.lz + b.lz, eK, zl);
        const double term = 2.0 * a.phi * b.phi * eK;
        fself += 0.5 * term;
        if (K > 1e-12) {
          const double s = zl * term / K;
          sx += ex * s;
          sy += ey * s;
          sz += ez * s;
        }
        su += term;
      }
      // cross pairs (objective.cpp:212-220, 300-326)
      const double wx = R[0] * vix + R[1] * viy + R[2] * viz;
      const double wy = R[3] * vix + R[4] * viy + R[5] * viz;
      const double wz = R[6] * vix + R[7] * viy + R[8] * viz;
      double hx = 0.0, hy = 0.0, hz = 0.0, hu = 0.0;
      for (int jp = max(q0, cs.n1); jp < q1; ++jp) {
        const int j = cs.o2 + (jp - cs.n1);
        const double ex = wx + m.b[3 * j], ey = wy + m.b[3 * j + 1], ez = wz + m.b[3 * j + 2];
        const double K = sqrt(ex * ex + ey * ey + ez * ez);
        if (K < a.k + m.kappa2[j] - objmath::kNegligible) continue;
        double eK, zl;
        pair_terms(K, a.lz + m.log_z2[j], eK, zl);
        const double term = a.phi * m.phi2[j] * eK;
        fcross += term;
        double qx = 0.0, qy = 0.0, qz = 0.0;
        if (K > 1e-12) {
          const double iK = 1.0 / K;
          qx = ex * iK;
          qy = ey * iK;
          qz = ez * iK;
        }
        const double s = zl * (-2.0 * term);
        hx += qx * s;
        hy += qy * s;
        hz += qz * s;
        hu += -2.0 * term;
        // (w x what) for the rotation gradient (Jl^T applied per pose)
        cr0 += w * (wy * qz - wz * qy) * s;
        cr1 += w * (wz * qx - wx * qz) * s;
        cr2 += w * (wx * qy - wy * qx) * s;
      }
      double ox, oy, oz;
      jv(a, sx, sy, sz, ox, oy, oz);  // self: J_i (sum/K) zl(K) term + u_i (2 zl_i/s2_i) term
      gt0 += w * (ox + uix * cu * su);
      gt1 += w * (oy + uiy * cu * su);
      gt2 += w * (oz + uiz * cu * su);
      const double px = R[0] * hx + R[3] * hy + R[6] * hz;  // R^T what
      const double py = R[1] * hx + R[4] * hy + R[7] * hz;
      const double pz = R[2] * hx + R[5] * hy + R[8] * hz;
      jv(a, px, py, pz, ox, oy, oz);
      gt0 += w * (ox + uix * cu * hu);
      gt1 += w * (oy + uiy * cu * hu);
      gt2 += w * (oz + uiz * cu * hu);
      fval += w * (fself - 2.0 * fcross);
    }
  }
  double v[7] = {fval, gt0, gt1, gt2, cr0, cr1, cr2};
  block_sum7(v, red);
  o[0] = v[0];
  o[1] = Jl[0] * v[4] + Jl[3] * v[5] + Jl[6] * v[6];
  o[2] = Jl[1] * v[4] + Jl[4] * v[5] + Jl[7] * v[6];
  o[3] = Jl[2] * v[4] + Jl[5] * v[5] + Jl[8] * v[6];
  o[4] = v[1];
  o[5] = v[2];
  o[6] = v[3];
  __syncthreads();  // rows / red are reused by the next evaluation
}

// Grid: x = partner slice, y = request. Per-slice partial {f, g[6]} go to
// out[(q * S + s) * 7]; the host sums slices in order (deterministic).
__global__ void __launch_bounds__(256)
    objgrad_kernel(const DevModel64* models, const ObjRequest* req, double* out, int max_n1) {
  extern __shared__ double smem_d[];
  RowD* rows = reinterpret_cast<RowD*>(smem_d);
  double* red = smem_d + static_cast<size_t>(max_n1) * (sizeof(RowD) / sizeof(double));
  const int q = blockIdx.y, slice = blockIdx.x, S = gridDim.x;
  const ObjRequest rq = req[q];
  double o[7];
  objgrad_block(models[rq.model], rq.x, slice, S, rows, red, o);
  if (threadIdx.x == 0)
    for (int k = 0; k < 7; ++k) out[(static_cast<size_t>(q) * S + slice) * 7 + k] = o[k];
}


// ---- GPU-resident local refinement ------------------------
// One CTA runs one start's L-BFGS ladder end to end: local_refine /
// wolfe_search / clamp_to_domain (core/src/solver.cpp:37-258; host version in
// csrc/sma.cpp) with every objective + gradient evaluated by the whole CTA
// (objgrad_block). All threads execute the same control code on identical
// values (the reductions broadcast), so control flow stays uniform across the
// CTA without shared control state.

// Value + gradient of one pose by a cluster of CTAs: CTA rank r takes partner
// slice r of C (objgrad_block), the C partial totals meet in distributed
// shared memory and every CTA sums them in rank order, so all CTAs of the
// cluster hold identical values and take identical control decisions.
struct CtaObjective {
  const DevModel64* m;
  const RefineDomain* dom;
  RowD* rows;
  double* red;
  double* xch;  // this CTA's partial totals (7), read by the cluster
  double* tot;  // cluster totals (7)
  long long* count;
  bool have = false;
  double x[6], f, g[6];
  __device__ const double* grad() const { return g; }
  __device__ bool project(double* p);
  __device__ void eval(const double* xx) {
    bool same = have;
    for (int k = 0; k < 6; ++k) same = same && xx[k] == x[k];
    if (same) return;
    ++*count;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const int C = static_cast<int>(cl.num_blocks());
    double o[7];
    objgrad_block(*m, xx, static_cast<int>(cl.block_rank()), C, rows, red, o, true);
    if (C > 1) {
      if (threadIdx.x == 0)
        for (int k = 0; k < 7; ++k) xch[k] = o[k];
      cl.sync();
      if (threadIdx.x < 7) {
        double t = 0.0;
        for (int r = 0; r < C; ++r) t += cl.map_shared_rank(xch, r)[threadIdx.x];
        tot[threadIdx.x] = t;
      }
      cl.sync();  // totals visible; every rank done reading xch
      for (int k = 0; k < 7; ++k) o[k] = tot[k];
    }
    for (int k = 0; k < 6; ++k) x[k] = xx[k];
    f = o[0];
    for (int k = 0; k < 6; ++k) g[k] = std::isinf(o[0]) ? 0.0 : o[1 + k];
    have = true;
  }
  __device__ double value(const double* xx) {
    eval(xx);
    return f;
  }
};

// clamp_to_domain (solver.cpp:48-95); the box and standoff-ball scans are
// spread over the CTA (nearest box: smallest distance, then lowest index;
// first offending mean: lowest index), every thread gets the same result.
__device__ bool clamp_to_domain_d(const DevModel64& m, const RefineDomain& dom, double* v,
                                  double* red) {
  for (int k = 0; k < 3; ++k)
    v[k] = fmin(fmax(v[k], dom.rc[k] - dom.rhw), dom.rc[k] + dom.rhw);
  constexpr int kNone = 0x7fffffff;
  double my_d = INFINITY;
  int my_b = kNone;
  for (int b = threadIdx.x; b < dom.n_boxes; b += blockDim.x) {
    const double* bx = dom.boxes + 6 * b;
    double s2 = 0.0;
    for (int k = 0; k < 3; ++k) {
      const double o = fmax(fabs(v[3 + k] - bx[k]) - bx[3 + k], 0.0);
      s2 += o * o;
    }
    const double d = sqrt(s2);
    if (d < my_d) {
      my_d = d;
      my_b = b;
    }
  }
  const double best_d = block_min_d(my_d, red);
  const int best = block_min_i(my_d == best_d ? my_b : kNone, red);
  if (best == kNone) return false;
  const double* bx = dom.boxes + 6 * best;
  double p[3];
  for (int k = 0; k < 3; ++k) p[k] = fmin(fmax(v[3 + k], bx[k] - bx[3 + k]), bx[k] + bx[3 + k]);
  for (int projection = 0; projection <= 8; ++projection) {
    int mine = kNone;
    for (int i = threadIdx.x; i < m.n_all && mine == kNone; i += blockDim.x) {
      const double dx = m.all_means[3 * i] - p[0], dy = m.all_means[3 * i + 1] - p[1],
                   dz = m.all_means[3 * i + 2] - p[2];
      if (sqrt(dx * dx + dy * dy + dz * dz) < m.zeta) mine = i;
    }
    const int off = block_min_i(mine, red);
    if (off == kNone) {
      for (int k = 0; k < 3; ++k) v[3 + k] = p[k];
      return true;
    }
    if (projection == 8) break;
    const double* mu = m.all_means + 3 * off;
    double dir[3] = {p[0] - mu[0], p[1] - mu[1], p[2] - mu[2]};
    const double n = sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
    if (n > 1e-12) {
      for (double& c : dir) c /= n;
    } else {
      dir[0] = 1.0;
      dir[1] = dir[2] = 0.0;
    }
    for (int k = 0; k < 3; ++k)
      p[k] = fmin(fmax(mu[k] + dir[k] * (m.zeta * (1.0 + 1e-9)), bx[k] - bx[3 + k]),
                  bx[k] + bx[3 + k]);
  }
  return false;
}

__device__ bool CtaObjective::project(double* p) { return clamp_to_domain_d(*m, *dom, p, red); }

// The CTA's one copy of the L-BFGS curvature pairs in shared memory: every
// thread computes the same pairs; thread 0 stores them and all threads read
// them back (broadcast loads) - per-thread copies would be 1 KB of local
// memory per thread (0.5 MB per CTA, spilled through L2 on every two-loop
// recursion).
struct LbfgsHistory {
  double S[refine::kMem][6], Y[refine::kMem][6], Rho[refine::kMem];
  __device__ void put(int slot, const double* s, const double* y, double rho) {
    __syncthreads();  // every thread is past its reads of the history
    if (threadIdx.x == 0) {
      for (int k = 0; k < 6; ++k) {
        S[slot][k] = s[k];
        Y[slot][k] = y[k];
      }
      Rho[slot] = rho;
    }
    __syncthreads();
  }
};

// One start's local refinement on one CTA (cluster): the shared controller
// (refine_core.hpp) over the CTA-wide FP64 objective.
__device__ void local_refine_d(const DevModel64& m, const RefineDomain& dom, RowD* rows,
                               double* red, double* xch, double* tot, LbfgsHistory& H,
                               double* xio, double* fout, long long* count) {
  CtaObjective ob{&m, &dom, rows, red, xch, tot, count};
  refine::lbfgs_refine(ob, H, xio, fout);
}

#ifndef GOSMA_REFINE_THREADS
#define GOSMA_REFINE_THREADS 512
#endif
constexpr int kRefineThreads = GOSMA_REFINE_THREADS;

__global__ void __launch_bounds__(kRefineThreads)
    refine_kernel(const DevModel64* models, const RefineJob* jobs, RefineDomain dom,
                  RefineOut* out, int max_n1) {
  extern __shared__ double smem_d[];
  __shared__ double xch[8], tot[8];
  __shared__ LbfgsHistory hist;
  RowD* rows = reinterpret_cast<RowD*>(smem_d);
  double* red = smem_d + static_cast<size_t>(max_n1) * (sizeof(RowD) / sizeof(double));
  namespace cg = cooperative_groups;
  const cg::cluster_group cl = cg::this_cluster();
  const int job = blockIdx.x / static_cast<int>(cl.num_blocks());
  const RefineJob jb = jobs[job];
  double x[6] = {jb.x[0], jb.x[1], jb.x[2], jb.x[3], jb.x[4], jb.x[5]};
  double f = INFINITY;
  long long count = 0;
  for (int st = 0; st < jb.stages; ++st)
    local_refine_d(models[jb.model[st]], dom, rows, red, xch, tot, hist, x, &f, &count);
  if (threadIdx.x == 0 && cl.block_rank() == 0) {
    RefineOut o;
    o.value = f;
    for (int k = 0; k < 6; ++k) o.x[k] = x[k];
    o.evals = count;
    out[job] = o;
  }
}

}  // namespace

cudaError_t launch_refine(const DevModel64* models, const RefineJob* jobs, int n,
                          const RefineDomain& dom, RefineOut* out, int max_n1, int cluster,
                          cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = objgrad_smem_bytes(max_n1);
  if (smem > 48 * 1024) {  // per call: the attribute is per device, the call is cheap
    const cudaError_t e = cudaFuncSetAttribute(
        refine_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  cluster = std::max(1, std::min(cluster, 8));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(n * cluster));
  cfg.blockDim = dim3(kRefineThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(cluster);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, refine_kernel, models, jobs, dom, out, max_n1);
}

size_t objgrad_smem_bytes(int max_n1) {
  return static_cast<size_t>(max_n1) * sizeof(RowD) + (7 * 32 + 8) * sizeof(double);
}

int objgrad_slices(int max_pairs_per_row) {
  // ~16 partners per thread and slice, at most 32 slices
  return std::max(1, std::min(32, max_pairs_per_row / 16));
}

cudaError_t launch_objgrad(const DevModel64* models, const ObjRequest* req, int n, int slices,
                           double* partial, int max_n1, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = objgrad_smem_bytes(max_n1);
  if (smem > 48 * 1024) {  // per call: the attribute is per device, the call is cheap
    const cudaError_t e = cudaFuncSetAttribute(
        objgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
  }
  const int threads = std::min(256, std::max(32, (max_n1 + 31) / 32 * 32));
  objgrad_kernel<<<dim3(slices, n), threads, smem, s>>>(models, req, partial, max_n1);
  return cudaGetLastError();
}

}  // namespace gosma
