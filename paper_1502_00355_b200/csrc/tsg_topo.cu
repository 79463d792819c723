// Mesh topology on the device: tsg_topology (include/tsg.h).
//
// The reference builds its adjacency on one host thread (find_neighbors / build_adjacency /
// determine_constraints, proj/src/topology.cpp:12-95): a raw list with two entries per
// incidence (int32 offsets: it overflows at 6 nt > 2^31), per-vertex sort + dedup
// with multiplicities, and "pinned iff isolated or some multiplicity != 2".  Here the same three
// outputs come from radix sorts on the device:
//   * incident rows: the 3 nt (corner vertex, triangle) pairs sorted by vertex — a stable sort,
//     and the pairs are generated in triangle order, so every row is ascending (Adjacency::incident);
//   * unique neighbour rows: the 6 nt directed corner pairs (v, u) as 64-bit keys v << 32 | u,
//     sorted, run-length encoded: the runs are the rows' entries in ascending u, the run lengths
//     their multiplicities (Adjacency::unique + multiplicity);
//   * boundary: isolated (no run) or some multiplicity != 2.
// Offsets are int64 and no raw list is materialised, so cfg5-sized meshes (nt = 512M) build.
// Results equal gpu::build_topology / find_neighbors bit for bit (tests/test_gpu_topology.py).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_run_length_encode.cuh>
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "tsg.h"
#include "tsg_internal.hpp"

namespace {

constexpr int kThreads = 256;

unsigned grid_of(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

__global__ void corner_pairs(const int32_t* __restrict__ tri, int64_t nt, uint32_t* __restrict__ cv,
                             int32_t* __restrict__ ct, unsigned long long* __restrict__ pairs,
                             int64_t* __restrict__ inc_cnt) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t a = static_cast<uint32_t>(tri[3 * t]), b = static_cast<uint32_t>(tri[3 * t + 1]),
                   c = static_cast<uint32_t>(tri[3 * t + 2]);
    const uint32_t v[3] = {a, b, c};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      cv[3 * t + k] = v[k];
      ct[3 * t + k] = static_cast<int32_t>(t);
      atomicAdd(reinterpret_cast<unsigned long long*>(inc_cnt + v[k]), 1ULL);
      const unsigned long long hi = static_cast<unsigned long long>(v[k]) << 32;
      pairs[6 * t + 2 * k] = hi | v[(k + 1) % 3];
      pairs[6 * t + 2 * k + 1] = hi | v[(k + 2) % 3];
    }
  }
}

__global__ void row_counts(const unsigned long long* __restrict__ keys, const int32_t* __restrict__ mult,
                           const int64_t* __restrict__ nruns, int32_t* __restrict__ nbr, int64_t* __restrict__ cnt,
                           uint8_t* __restrict__ boundary) {
  const int64_t n = *nruns;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const unsigned long long k = keys[i];
    const uint32_t v = static_cast<uint32_t>(k >> 32);
    nbr[i] = static_cast<int32_t>(k & 0xffffffffULL);
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + v), 1ULL);
    if (mult[i] != 2) boundary[v] = 1;
  }
}

__global__ void mark_isolated(const int64_t* __restrict__ cnt, int64_t nv, uint8_t* __restrict__ boundary) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x)
    if (cnt[v] == 0) boundary[v] = 1;
}

// Hilbert index of (x, y) on a 2^16 x 2^16 lattice (the host hilbert_d, tsg_prep.cpp).
__device__ uint32_t hilbert_d_dev(uint32_t x, uint32_t y) {
  uint32_t d = 0;
  for (uint32_t s = 1u << 15; s > 0; s >>= 1) {
    const uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
    d += s * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = 0xffffu - x;
        y = 0xffffu - y;
      }
      const uint32_t t = x;
      x = y;
      y = t;
    }
  }
  return d;
}

__global__ void hilbert_keys(const double2* __restrict__ xy, int64_t nv, double xmin, double ymin, double sx, double sy,
                             unsigned long long* __restrict__ keys) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double2 p = xy[v];
    const double fx = isfinite(p.x) ? __dmul_rn(__dsub_rn(p.x, xmin), sx) : 0.0;
    const double fy = isfinite(p.y) ? __dmul_rn(__dsub_rn(p.y, ymin), sy) : 0.0;
    const uint32_t qx = static_cast<uint32_t>(fx < 0.0 ? 0.0 : (fx > 65535.0 ? 65535.0 : fx));
    const uint32_t qy = static_cast<uint32_t>(fy < 0.0 ? 0.0 : (fy > 65535.0 ? 65535.0 : fy));
    keys[v] = (static_cast<unsigned long long>(hilbert_d_dev(qx, qy)) << 32) | static_cast<unsigned long long>(v);
  }
}

__global__ void keys_to_order(const unsigned long long* __restrict__ keys, int64_t nv, int64_t* __restrict__ order) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    order[i] = static_cast<int64_t>(keys[i] & 0xffffffffULL);
}

int end_bit_for(int64_t nv) {
  int b = 1;
  while (b < 32 && (int64_t{1} << b) < nv) ++b;
  return b;
}

}  // namespace

extern "C" tsg_status tsg_topology(tsg_context* ctx, int64_t nv, int64_t nt, const int32_t* tri, int64_t* nbr_off,
                                   int32_t* nbr, int64_t nbr_cap, int64_t* inc_off, int32_t* inc, uint8_t* boundary,
                                   int64_t* n_nbr_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || nv <= 0 || nt < 0 || nv >= (int64_t{1} << 31) || (nt > 0 && !tri) || !nbr_off || !inc_off ||
      !boundary || !n_nbr_out || (nt > 0 && (!inc || !nbr)))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: bad arguments");
  for (int64_t i = 0; i < 3 * nt; ++i)
    if (tri[i] < 0 || tri[i] >= nv) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: corner index out of range");
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int64_t m3 = 3 * nt, m6 = 6 * nt;
  const int vbits = end_bit_for(nv);
  // device buffers (stream-ordered; freed on every path by the guard)
  struct Bufs {
    cudaStream_t s;
    std::vector<void*> p;
    ~Bufs() {
      for (void* q : p) cudaFreeAsync(q, s);
    }
    cudaError_t get(void** out, size_t bytes) {
      cudaError_t e = cudaMallocAsync(out, bytes ? bytes : 8, s);
      if (e == cudaSuccess) p.push_back(*out);
      return e;
    }
  } B{s, {}};
  int32_t *d_tri = nullptr, *d_ct = nullptr, *d_ct2 = nullptr, *d_mult = nullptr, *d_nbr = nullptr;
  uint32_t *d_cv = nullptr, *d_cv2 = nullptr;
  unsigned long long *d_pairs = nullptr, *d_pairs2 = nullptr, *d_ukeys = nullptr;
  int64_t *d_inc_cnt = nullptr, *d_inc_off = nullptr, *d_cnt = nullptr, *d_off = nullptr, *d_nruns = nullptr;
  uint8_t* d_bnd = nullptr;
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_tri), sizeof(int32_t) * m3));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_cv), sizeof(uint32_t) * m3));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_cv2), sizeof(uint32_t) * m3));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_ct), sizeof(int32_t) * m3));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_ct2), sizeof(int32_t) * m3));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_pairs), sizeof(unsigned long long) * m6));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_pairs2), sizeof(unsigned long long) * m6));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_inc_cnt), sizeof(int64_t) * (nv + 1)));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_inc_off), sizeof(int64_t) * (nv + 1)));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_cnt), sizeof(int64_t) * (nv + 1)));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_off), sizeof(int64_t) * (nv + 1)));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_nruns), sizeof(int64_t)));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_bnd), nv));
  TSG_CUDA(cudaMemsetAsync(d_inc_cnt, 0, sizeof(int64_t) * (nv + 1), s));
  TSG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(int64_t) * (nv + 1), s));
  TSG_CUDA(cudaMemsetAsync(d_bnd, 0, nv, s));
  if (nt) TSG_CUDA(cudaMemcpyAsync(d_tri, tri, sizeof(int32_t) * m3, cudaMemcpyHostToDevice, s));
  corner_pairs<<<grid_of(nt), kThreads, 0, s>>>(d_tri, nt, d_cv, d_ct, d_pairs, d_inc_cnt);
  TSG_LAUNCHED();

  // incident rows: stable sort of (vertex, triangle) by vertex
  size_t tmp_bytes = 0, need = 0;
  TSG_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, need, d_cv, d_cv2, d_ct, d_ct2, m3, 0, vbits, s));
  tmp_bytes = need;
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, need, d_pairs, d_pairs2, m6, 0, 32 + vbits, s));
  tmp_bytes = std::max(tmp_bytes, need);
  TSG_CUDA(cub::DeviceRunLengthEncode::Encode(nullptr, need, d_pairs2, d_pairs, d_ct, d_nruns, m6, s));
  tmp_bytes = std::max(tmp_bytes, need);
  TSG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, need, d_inc_cnt, d_inc_off, nv + 1, s));
  tmp_bytes = std::max(tmp_bytes, need);
  void* d_tmp = nullptr;
  TSG_CUDA(B.get(&d_tmp, tmp_bytes));
  need = tmp_bytes;
  TSG_CUDA(cub::DeviceRadixSort::SortPairs(d_tmp, need, d_cv, d_cv2, d_ct, d_ct2, m3, 0, vbits, s));
  need = tmp_bytes;
  TSG_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, need, d_inc_cnt, d_inc_off, nv + 1, s));

  // unique neighbour rows with multiplicities: sort the directed pairs, run-length encode
  need = tmp_bytes;
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(d_tmp, need, d_pairs, d_pairs2, m6, 0, 32 + vbits, s));
  d_ukeys = d_pairs;  // the runs overwrite the (consumed) unsorted keys
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_mult), sizeof(int32_t) * m6));
  need = tmp_bytes;
  TSG_CUDA(cub::DeviceRunLengthEncode::Encode(d_tmp, need, d_pairs2, d_ukeys, d_mult, d_nruns, m6, s));
  int64_t h_runs = 0;
  TSG_CUDA(cudaMemcpyAsync(&h_runs, d_nruns, sizeof h_runs, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  if (h_runs > nbr_cap) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: nbr capacity too small");
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_nbr), sizeof(int32_t) * h_runs));
  row_counts<<<grid_of(h_runs), kThreads, 0, s>>>(d_ukeys, d_mult, d_nruns, d_nbr, d_cnt, d_bnd);
  TSG_LAUNCHED();
  mark_isolated<<<grid_of(nv), kThreads, 0, s>>>(d_cnt, nv, d_bnd);
  TSG_LAUNCHED();
  need = tmp_bytes;
  TSG_CUDA(cub::DeviceScan::ExclusiveSum(d_tmp, need, d_cnt, d_off, nv + 1, s));

  TSG_CUDA(cudaMemcpyAsync(nbr_off, d_off, sizeof(int64_t) * (nv + 1), cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(inc_off, d_inc_off, sizeof(int64_t) * (nv + 1), cudaMemcpyDeviceToHost, s));
  if (h_runs) TSG_CUDA(cudaMemcpyAsync(nbr, d_nbr, sizeof(int32_t) * h_runs, cudaMemcpyDeviceToHost, s));
  if (m3) TSG_CUDA(cudaMemcpyAsync(inc, d_ct2, sizeof(int32_t) * m3, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(boundary, d_bnd, nv, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  *n_nbr_out = h_runs;
  return TSG_OK;
}

// tsg_hilbert_order on the device: same keys (bounding box and quantisation on the host, exact
// fp64 without contraction), radix-sorted; identical order.
extern "C" tsg_status tsg_hilbert_order_device(tsg_context* ctx, int64_t nv, const double* xy, int64_t* order_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || nv <= 0 || nv >= (int64_t{1} << 32) || !xy || !order_out)
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_hilbert_order_device: bad arguments");
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  for (int64_t v = 0; v < nv; ++v) {
    xmin = std::min(xmin, xy[2 * v]);
    xmax = std::max(xmax, xy[2 * v]);
    ymin = std::min(ymin, xy[2 * v + 1]);
    ymax = std::max(ymax, xy[2 * v + 1]);
  }
  const double sx = xmax > xmin ? 65535.0 / (xmax - xmin) : 0.0;
  const double sy = ymax > ymin ? 65535.0 / (ymax - ymin) : 0.0;
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  struct Bufs {
    cudaStream_t s;
    std::vector<void*> p;
    ~Bufs() {
      for (void* q : p) cudaFreeAsync(q, s);
    }
    cudaError_t get(void** out, size_t bytes) {
      cudaError_t e = cudaMallocAsync(out, bytes ? bytes : 8, s);
      if (e == cudaSuccess) p.push_back(*out);
      return e;
    }
  } B{s, {}};
  double2* d_xy = nullptr;
  unsigned long long *k1 = nullptr, *k2 = nullptr;
  int64_t* d_order = nullptr;
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_xy), sizeof(double2) * nv));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&k1), 8 * nv));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&k2), 8 * nv));
  TSG_CUDA(B.get(reinterpret_cast<void**>(&d_order), 8 * nv));
  TSG_CUDA(cudaMemcpyAsync(d_xy, xy, sizeof(double2) * nv, cudaMemcpyHostToDevice, s));
  hilbert_keys<<<grid_of(nv), kThreads, 0, s>>>(d_xy, nv, xmin, ymin, sx, sy, k1);
  TSG_LAUNCHED();
  size_t bytes = 0;
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k1, k2, nv, 0, 64, s));
  void* tmp = nullptr;
  TSG_CUDA(B.get(&tmp, bytes));
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, k1, k2, nv, 0, 64, s));
  keys_to_order<<<grid_of(nv), kThreads, 0, s>>>(k2, nv, d_order);
  TSG_LAUNCHED();
  TSG_CUDA(cudaMemcpyAsync(order_out, d_order, 8 * nv, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}
