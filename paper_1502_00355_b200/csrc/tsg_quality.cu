// Quality audit on the device (include/tsg.h: tsg_quality_tri_alpha, tsg_quality_vertex_minima).
//
// The host-side audits of the reference — compute_all_qualities / refresh_tri_alphas
// (proj/src/quality.cpp:27-32, proj/include/trismooth/quality.hpp:68-74), reduce_vertex_minima
// (proj/src/quality.cpp:60-65, quality.hpp:78-89) and the reductions of quality_summary /
// `trismooth quality` (proj/bindings/module.cpp:157-185, proj/tools/main.cpp:151-208) — as
// stand-alone calls on caller-owned host arrays: no tsg_mesh, no topology build.  Each call
// stages its inputs into stream-ordered device allocations, runs one pass over the triangles
// (or vertices), and copies the results back.
//
// Bit-exactness: α is triangle_alpha in the reference's operand order with explicit _rn
// intrinsics (tsg_device.cuh, alpha_plain).  The reductions reproduce the reference's
// sequential folds, not just their values:
//   * min / max follow std::min(lo, q) / std::max(hi, q) from lo = 2.0, hi = -2.0: NaN never
//     replaces, ties keep the FIRST occurrence (so the sign of a zero extreme is that of the
//     first zero in triangle order).  Device: atomic min/max of an order key with -0 folded
//     onto +0, then an atomic min of the first index holding that value;
//   * the histogram bin is static_cast<int>((q + 1.0) * 10.0) clamped to [0, 19] — NaN lands
//     in bin 0 on both sides (x86 cvttsd2si gives INT_MIN, the device conversion 0);
//   * vertex minima are the per-vertex fold `q < lowest ? q : lowest` from +inf, NaN for a
//     vertex without incident triangles (kUnsetQuality), exactly as written.
// The mean is NOT reduced here: its sequential sum is order-sensitive, so callers sum the
// returned α field in triangle order on the host (as smooth() does).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>

#include "tsg.h"
#include "tsg_device.cuh"
#include "tsg_internal.hpp"

namespace {

using tsg::Arith;
using tsg::alpha_plain;

constexpr int kBins = TSG_QUALITY_BINS;
constexpr int kThreads = 256;

__device__ __forceinline__ unsigned long long order_key(double d) {
  if (d == 0.0) d = 0.0;  // -0 and +0 are one value for the fold (the first one wins)
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

struct AuditScratch {
  unsigned long long lo_key, hi_key;  // order keys of the extreme values
  unsigned long long lo_first, hi_first;  // first triangle holding them (~0: none)
  unsigned long long nonpos;
  unsigned long long bins[kBins];
};

__global__ void __launch_bounds__(kThreads) audit_alpha(const double2* __restrict__ xy,
                                                        const int32_t* __restrict__ tri, int64_t nt,
                                                        double* __restrict__ alpha, AuditScratch* acc) {
  __shared__ unsigned long long sbins[kBins];
  for (int i = threadIdx.x; i < kBins; i += blockDim.x) sbins[i] = 0;
  __syncthreads();
  unsigned long long lo = order_key(2.0), hi = order_key(-2.0), np = 0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 p1 = xy[tri[3 * t]], p2 = xy[tri[3 * t + 1]], p3 = xy[tri[3 * t + 2]];
    const double q = alpha_plain<double>(p1.x, p1.y, p2.x, p2.y, p3.x, p3.y);
    alpha[t] = q;
    if (q == q) {  // NaN never replaces an extreme
      const unsigned long long k = order_key(q);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
    np += q <= 0.0 ? 1 : 0;
    int b = __double2int_rz(__dmul_rn(__dadd_rn(q, 1.0), 10.0));
    b = b < 0 ? 0 : (b > kBins - 1 ? kBins - 1 : b);
    atomicAdd(&sbins[b], 1ULL);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
    np += __shfl_xor_sync(0xffffffffu, np, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&acc->lo_key, lo);
    atomicMax(&acc->hi_key, hi);
    if (np) atomicAdd(&acc->nonpos, np);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += blockDim.x)
    if (sbins[i]) atomicAdd(&acc->bins[i], sbins[i]);
}

// First triangle whose α equals the extreme value (value equality: -0 == +0).
__global__ void __launch_bounds__(kThreads) audit_first(const double* __restrict__ alpha, int64_t nt,
                                                        AuditScratch* acc) {
  const unsigned long long lo = acc->lo_key, hi = acc->hi_key;
  unsigned long long flo = ~0ULL, fhi = ~0ULL;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double q = alpha[t];
    if (q != q) continue;
    const unsigned long long k = order_key(q);
    if (k == lo && static_cast<unsigned long long>(t) < flo) flo = t;
    if (k == hi && static_cast<unsigned long long>(t) < fhi) fhi = t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long a = __shfl_xor_sync(0xffffffffu, flo, o);
    const unsigned long long b = __shfl_xor_sync(0xffffffffu, fhi, o);
    flo = a < flo ? a : flo;
    fhi = b < fhi ? b : fhi;
  }
  if ((threadIdx.x & 31) == 0) {
    if (flo != ~0ULL) atomicMin(&acc->lo_first, flo);
    if (fhi != ~0ULL) atomicMin(&acc->hi_first, fhi);
  }
}

__global__ void __launch_bounds__(kThreads) audit_vertex_minima(const int64_t* __restrict__ inc_off,
                                                                const int32_t* __restrict__ inc,
                                                                const double* __restrict__ alpha, int64_t nv,
                                                                double* __restrict__ out) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = inc_off[v], e = inc_off[v + 1];
    if (b == e) {
      out[v] = __longlong_as_double(0x7ff8000000000000LL);  // kUnsetQuality
      continue;
    }
    double lowest = __longlong_as_double(0x7ff0000000000000LL);  // +inf
    for (int64_t j = b; j < e; ++j) {
      const double q = alpha[inc[j]];
      lowest = q < lowest ? q : lowest;
    }
    out[v] = lowest;
  }
}

unsigned grid_of(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

// Stream-ordered device allocations released on every return path.
struct DevBufs {
  cudaStream_t s;
  void* p[6] = {};
  int n = 0;
  explicit DevBufs(cudaStream_t st) : s(st) {}
  ~DevBufs() {
    for (int i = 0; i < n; ++i) cudaFreeAsync(p[i], s);
  }
  cudaError_t alloc(void** out, size_t bytes) {
    cudaError_t e = cudaMallocAsync(out, bytes ? bytes : 8, s);
    if (e == cudaSuccess) p[n++] = *out;
    return e;
  }
};

}  // namespace

extern "C" {

tsg_status tsg_quality_tri_alpha(tsg_context* ctx, int64_t nv, const double* xy, int64_t nt, const int32_t* tri,
                                 double* alpha_out, tsg_quality_report* report) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || nv < 0 || nt < 0 || (nv > 0 && !xy) || (nt > 0 && (!tri || !alpha_out)))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_tri_alpha: bad arguments");
  for (int64_t i = 0; i < 3 * nt; ++i)
    if (tri[i] < 0 || tri[i] >= nv)
      return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_tri_alpha: triangle corner index out of range");
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  DevBufs d(s);
  double2* dxy = nullptr;
  int32_t* dtri = nullptr;
  double* dalpha = nullptr;
  AuditScratch* dacc = nullptr;
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dxy), sizeof(double2) * nv));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dtri), sizeof(int32_t) * 3 * nt));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dalpha), sizeof(double) * nt));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dacc), sizeof(AuditScratch)));
  AuditScratch init{};
  init.lo_key = ~0ULL;
  init.hi_key = 0;
  init.lo_first = init.hi_first = ~0ULL;
  TSG_CUDA(cudaMemcpyAsync(dacc, &init, sizeof init, cudaMemcpyHostToDevice, s));
  if (nv) TSG_CUDA(cudaMemcpyAsync(dxy, xy, sizeof(double2) * nv, cudaMemcpyHostToDevice, s));
  if (nt) TSG_CUDA(cudaMemcpyAsync(dtri, tri, sizeof(int32_t) * 3 * nt, cudaMemcpyHostToDevice, s));
  audit_alpha<<<grid_of(nt), kThreads, 0, s>>>(dxy, dtri, nt, dalpha, dacc);
  TSG_LAUNCHED();
  audit_first<<<grid_of(nt), kThreads, 0, s>>>(dalpha, nt, dacc);
  TSG_LAUNCHED();
  if (nt) TSG_CUDA(cudaMemcpyAsync(alpha_out, dalpha, sizeof(double) * nt, cudaMemcpyDeviceToHost, s));
  AuditScratch h{};
  TSG_CUDA(cudaMemcpyAsync(&h, dacc, sizeof h, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  if (report) {
    // the folds start from 2.0 / -2.0; a first index exists iff some α reached the extreme
    report->min_alpha = h.lo_first != ~0ULL ? alpha_out[h.lo_first] : 2.0;
    report->max_alpha = h.hi_first != ~0ULL ? alpha_out[h.hi_first] : -2.0;
    report->non_positive = static_cast<int64_t>(h.nonpos);
    for (int i = 0; i < kBins; ++i) report->histogram[i] = static_cast<int64_t>(h.bins[i]);
  }
  return TSG_OK;
}

tsg_status tsg_quality_vertex_minima(tsg_context* ctx, int64_t nv, const int64_t* inc_off, const int32_t* inc,
                                     int64_t nt, const double* alpha, double* vmin_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || nv < 0 || nt < 0 || (nv > 0 && (!inc_off || !vmin_out)))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_vertex_minima: bad arguments");
  if (nv == 0) return TSG_OK;
  if (inc_off[0] != 0) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_vertex_minima: offsets must start at 0");
  for (int64_t v = 0; v < nv; ++v)
    if (inc_off[v + 1] < inc_off[v])
      return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_vertex_minima: offsets decreasing");
  const int64_t m = inc_off[nv];
  if (m > 0 && (!inc || (nt > 0 && !alpha)))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_vertex_minima: bad arguments");
  for (int64_t j = 0; j < m; ++j)
    if (inc[j] < 0 || inc[j] >= nt)
      return tsg_abi::fail(TSG_ERR_INVALID, "tsg_quality_vertex_minima: triangle id out of range");
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  DevBufs d(s);
  int64_t* doff = nullptr;
  int32_t* dinc = nullptr;
  double *dalpha = nullptr, *dout = nullptr;
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&doff), sizeof(int64_t) * (nv + 1)));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dinc), sizeof(int32_t) * m));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dalpha), sizeof(double) * nt));
  TSG_CUDA(d.alloc(reinterpret_cast<void**>(&dout), sizeof(double) * nv));
  TSG_CUDA(cudaMemcpyAsync(doff, inc_off, sizeof(int64_t) * (nv + 1), cudaMemcpyHostToDevice, s));
  if (m) TSG_CUDA(cudaMemcpyAsync(dinc, inc, sizeof(int32_t) * m, cudaMemcpyHostToDevice, s));
  if (nt && alpha) TSG_CUDA(cudaMemcpyAsync(dalpha, alpha, sizeof(double) * nt, cudaMemcpyHostToDevice, s));
  audit_vertex_minima<<<grid_of(nv), kThreads, 0, s>>>(doff, dinc, dalpha, nv, dout);
  TSG_LAUNCHED();
  TSG_CUDA(cudaMemcpyAsync(vmin_out, dout, sizeof(double) * nv, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}

}  // extern "C"
