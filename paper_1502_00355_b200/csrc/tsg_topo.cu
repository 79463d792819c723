// Mesh topology on the device: tsg_topology (include/tsg.h).
//
// The reference builds its adjacency on one host thread (find_neighbors / build_adjacency /
// determine_constraints, proj/src/topology.cpp:12-95): a raw list with two entries per
// incidence (int32 offsets: it overflows at 6 nt > 2^31), per-vertex sort + dedup
// with multiplicities, and "pinned iff isolated or some multiplicity != 2".  Here the same three
// outputs come from radix sorts on the device:
//   * incident rows: the 3 nt (corner vertex, triangle) pairs sorted by vertex — a stable sort,
//     and the pairs are generated in triangle order, so every row is ascending (Adjacency::incident);
//   * unique neighbour rows, per vertex from its incident rows: the two other corners of every
//     incident triangle (the reference's raw row, in some order), sorted and run-length counted —
//     in registers / local memory for rows of up to kLocalCand candidates (thread per vertex),
//     through a segmented sort for the few longer rows (hubs) — giving the rows in ascending id
//     and the multiplicities (Adjacency::unique + multiplicity);
//   * boundary: isolated or some multiplicity != 2.
// Offsets are int64, no raw list is materialised and no device-wide sort exceeds 3 nt items,
// so cfg5-sized meshes (nt = 512M: 1.5e9 corners) build.
// Results equal gpu::build_topology / find_neighbors bit for bit (tests/test_gpu_topology.py).
#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/device/device_scan.cuh>
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "tsg.h"
#include "tsg_internal.hpp"
#include "tsg_layout_dev.hpp"

namespace {

constexpr int kThreads = 256;

unsigned grid_of(int64_t n) {
  const int64_t g = (n + kThreads - 1) / kThreads;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 32 ? 148 * 32 : g));
}

// (Also the range check of every corner: *bad = 1 when one lies outside [0, nv).)
__global__ void corner_keys(const int32_t* __restrict__ tri, int64_t nt, int64_t nv, uint32_t* __restrict__ cv,
                            int32_t* __restrict__ ct, unsigned long long* __restrict__ inc_cnt,
                            unsigned long long* __restrict__ bad) {
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t v = static_cast<uint32_t>(tri[3 * t + k]);
      cv[3 * t + k] = v;
      ct[3 * t + k] = static_cast<int32_t>(t);
      if (v < static_cast<uint64_t>(nv))
        atomicAdd(inc_cnt + v, 1ULL);
      else
        *bad = 1;
    }
  }
}

constexpr int kLocalCand = 64;  // candidates sorted in a thread's local array (valence <= 32)

// The two other corners of each incident triangle of v.
__device__ __forceinline__ int gather_candidates(const int32_t* __restrict__ tri, const int32_t* __restrict__ inc,
                                                 int64_t b, int64_t e, int32_t v, int32_t* c) {
  int n = 0;
  for (int64_t i = b; i < e; ++i) {
    const int32_t* tv = tri + 3 * static_cast<int64_t>(inc[i]);
#pragma unroll
    for (int k = 0; k < 3; ++k)
      if (tv[k] != v) c[n++] = tv[k];
  }
  return n;
}

// Sorted candidates -> unique values (optional output), count, and "some multiplicity != 2".
__device__ __forceinline__ int unique_runs(const int32_t* c, int n, int32_t* out, bool& odd) {
  int u = 0;
  for (int i = 0; i < n;) {
    int j = i + 1;
    while (j < n && c[j] == c[i]) ++j;
    if (out) out[u] = c[i];
    odd = odd || (j - i) != 2;
    ++u;
    i = j;
  }
  return u;
}

// Thread per vertex: rows of up to kLocalCand candidates; longer rows are flagged for the
// segmented path.  Pass 0 counts (and classifies), pass 1 writes the values.
__global__ void local_rows(const int32_t* __restrict__ tri, const unsigned long long* __restrict__ inc_off,
                           const int32_t* __restrict__ inc, int64_t nv, int pass, unsigned long long* __restrict__ cnt,
                           uint8_t* __restrict__ boundary, uint8_t* __restrict__ big,
                           const unsigned long long* __restrict__ off, int32_t* __restrict__ nbr) {
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t b = static_cast<int64_t>(inc_off[v]), e = static_cast<int64_t>(inc_off[v + 1]);
    if (2 * (e - b) > kLocalCand) {
      if (pass == 0) big[v] = 1;
      continue;
    }
    int32_t c[kLocalCand];
    const int n = gather_candidates(tri, inc, b, e, static_cast<int32_t>(v), c);
    for (int i = 1; i < n; ++i) {  // insertion sort (about a dozen entries)
      const int32_t x = c[i];
      int j = i - 1;
      while (j >= 0 && c[j] > x) {
        c[j + 1] = c[j];
        --j;
      }
      c[j + 1] = x;
    }
    bool odd = false;
    if (pass == 0) {
      big[v] = 0;
      cnt[v] = static_cast<unsigned long long>(unique_runs(c, n, nullptr, odd));
      boundary[v] = (n == 0 || odd) ? 1 : 0;
    } else {
      unique_runs(c, n, nbr + off[v], odd);
    }
  }
}

// Long rows (hubs): candidates into a buffer segmented by big vertex, sorted by CUB, then counted
// / written by a thread per big vertex.
__global__ void big_candidates(const int32_t* __restrict__ tri, const unsigned long long* __restrict__ inc_off,
                               const int32_t* __restrict__ inc, const int32_t* __restrict__ bigv, int64_t nbig,
                               const unsigned long long* __restrict__ cand_off, int32_t* __restrict__ cand) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nbig;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = bigv[i];
    gather_candidates(tri, inc, static_cast<int64_t>(inc_off[v]), static_cast<int64_t>(inc_off[v + 1]), v,
                      cand + cand_off[i]);
  }
}

__global__ void big_rows(const int32_t* __restrict__ cand, const unsigned long long* __restrict__ cand_off,
                         const int32_t* __restrict__ bigv, int64_t nbig, int pass, unsigned long long* __restrict__ cnt,
                         uint8_t* __restrict__ boundary, const unsigned long long* __restrict__ off,
                         int32_t* __restrict__ nbr) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nbig;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = bigv[i];
    const int32_t* c = cand + cand_off[i];
    const int n = static_cast<int>(cand_off[i + 1] - cand_off[i]);
    bool odd = false;
    if (pass == 0) {
      cnt[v] = static_cast<unsigned long long>(unique_runs(c, n, nullptr, odd));
      boundary[v] = (n == 0 || odd) ? 1 : 0;
    } else {
      unique_runs(c, n, nbr + off[v], odd);
    }
  }
}

__global__ void big_cand_counts(const unsigned long long* __restrict__ inc_off, const int32_t* __restrict__ bigv,
                                int64_t nbig, unsigned long long* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nbig;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v = bigv[i];
    out[i] = 2 * (inc_off[v + 1] - inc_off[v]);
  }
}

__global__ void iota32(int64_t n, int32_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<int32_t>(i);
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

// Stream-ordered device allocations released on every return path.
struct DevBufs {
  cudaStream_t s;
  std::vector<void*> p;
  ~DevBufs() {
    for (void* q : p) cudaFreeAsync(q, s);
  }
  template <class T>
  cudaError_t get(T** out, int64_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, static_cast<size_t>(n > 0 ? n : 1) * sizeof(T), s);
    if (e == cudaSuccess) {
      p.push_back(q);
      *out = static_cast<T*>(q);
    }
    return e;
  }
};

int end_bit_for(int64_t nv) {
  int b = 1;
  while (b < 32 && (int64_t{1} << b) < nv) ++b;
  return b;
}

}  // namespace

namespace {

// The topology on the device (buffers owned by B): triangles uploaded, unique-neighbour rows,
// incident rows, boundary flags.  Shared by tsg_topology (downloads them) and
// tsg_mesh_upload_triangles (hands them to the device layout without a host round trip).
struct TopoDev {
  const int32_t* tri = nullptr;  // 3 nt
  const unsigned long long* off = nullptr;      // nv + 1 (int64 values)
  const int32_t* nbr = nullptr;  // off[nv]
  const unsigned long long* inc_off = nullptr;  // nv + 1
  const int32_t* inc = nullptr;  // 3 nt
  const uint8_t* bnd = nullptr;  // nv
  int64_t n_nbr = 0;
};

tsg_status topology_device(tsg_context* ctx, int64_t nv, int64_t nt, const int32_t* tri, DevBufs& B, TopoDev& out) {
  cudaStream_t s = ctx->stream;
  const int64_t m3 = 3 * nt;
  const int vbits = end_bit_for(nv);
  DevBufs Tmp{s, {}};  // temporaries; the outputs come from the caller's B
  auto cub_call = [&](auto&& f) -> cudaError_t {
    size_t bytes = 0;
    cudaError_t e = f(nullptr, bytes);
    if (e != cudaSuccess) return e;
    char* t = nullptr;
    if ((e = Tmp.get(&t, static_cast<int64_t>(bytes))) != cudaSuccess) return e;
    return f(t, bytes);
  };
  int32_t *d_tri, *d_ct, *d_inc;
  uint32_t *d_cv, *d_cv2;
  unsigned long long *d_inc_cnt, *d_inc_off, *d_cnt, *d_off;
  uint8_t *d_bnd, *d_big;
  TSG_CUDA(B.get(&d_tri, m3));
  TSG_CUDA(Tmp.get(&d_cv, m3));
  TSG_CUDA(Tmp.get(&d_cv2, m3));
  TSG_CUDA(Tmp.get(&d_ct, m3));
  TSG_CUDA(B.get(&d_inc, m3));
  TSG_CUDA(Tmp.get(&d_inc_cnt, nv + 1));
  TSG_CUDA(B.get(&d_inc_off, nv + 1));
  TSG_CUDA(Tmp.get(&d_cnt, nv + 1));
  TSG_CUDA(B.get(&d_off, nv + 1));
  TSG_CUDA(B.get(&d_bnd, nv));
  TSG_CUDA(Tmp.get(&d_big, nv));
  TSG_CUDA(cudaMemsetAsync(d_inc_cnt, 0, 8 * (nv + 1), s));
  TSG_CUDA(cudaMemsetAsync(d_cnt, 0, 8 * (nv + 1), s));
  if (nt) TSG_CUDA(cudaMemcpyAsync(d_tri, tri, 4 * m3, cudaMemcpyHostToDevice, s));
  {
    unsigned long long* d_bad = nullptr;
    unsigned long long h_bad = 0;
    TSG_CUDA(Tmp.get(&d_bad, 1));
    TSG_CUDA(cudaMemsetAsync(d_bad, 0, 8, s));
    corner_keys<<<grid_of(nt), kThreads, 0, s>>>(d_tri, nt, nv, d_cv, d_ct, d_inc_cnt, d_bad);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(&h_bad, d_bad, 8, cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    if (h_bad) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: corner index out of range");
  }
  // incident rows: stable sort of (vertex, triangle) by vertex (pairs generated in triangle order)
  TSG_CUDA(cub_call([&](void* t, size_t& b) {
    return cub::DeviceRadixSort::SortPairs(t, b, d_cv, d_cv2, d_ct, d_inc, static_cast<int>(m3), 0, vbits, s);
  }));
  TSG_CUDA(cub_call([&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, d_inc_cnt, d_inc_off, nv + 1, s);
  }));
  // unique rows: pass 0 counts and classifies
  local_rows<<<grid_of(nv), kThreads, 0, s>>>(d_tri, d_inc_off, d_inc, nv, 0, d_cnt, d_bnd, d_big, nullptr, nullptr);
  TSG_LAUNCHED();
  int32_t *d_iota, *d_bigv;
  int64_t* d_nbig;
  TSG_CUDA(Tmp.get(&d_iota, nv));
  TSG_CUDA(Tmp.get(&d_bigv, nv));
  TSG_CUDA(Tmp.get(&d_nbig, 1));
  iota32<<<grid_of(nv), kThreads, 0, s>>>(nv, d_iota);
  TSG_LAUNCHED();
  TSG_CUDA(cub_call([&](void* t, size_t& b) {
    return cub::DeviceSelect::Flagged(t, b, d_iota, d_big, d_bigv, d_nbig, nv, s);
  }));
  int64_t nbig = 0;
  TSG_CUDA(cudaMemcpyAsync(&nbig, d_nbig, 8, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  unsigned long long *d_coff = nullptr, *d_ccnt = nullptr;
  int32_t *d_cand = nullptr, *d_cand2 = nullptr;
  if (nbig > 0) {
    TSG_CUDA(Tmp.get(&d_ccnt, nbig + 1));
    TSG_CUDA(Tmp.get(&d_coff, nbig + 1));
    TSG_CUDA(cudaMemsetAsync(d_ccnt + nbig, 0, 8, s));
    big_cand_counts<<<grid_of(nbig), kThreads, 0, s>>>(d_inc_off, d_bigv, nbig, d_ccnt);
    TSG_LAUNCHED();
    TSG_CUDA(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, d_ccnt, d_coff, nbig + 1, s); }));
    unsigned long long ncand = 0;
    TSG_CUDA(cudaMemcpyAsync(&ncand, d_coff + nbig, 8, cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    if (ncand >= (1ULL << 31)) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: hub rows exceed 2^31 entries");
    TSG_CUDA(Tmp.get(&d_cand, static_cast<int64_t>(ncand)));
    TSG_CUDA(Tmp.get(&d_cand2, static_cast<int64_t>(ncand)));
    big_candidates<<<grid_of(nbig), kThreads, 0, s>>>(d_tri, d_inc_off, d_inc, d_bigv, nbig, d_coff, d_cand);
    TSG_LAUNCHED();
    TSG_CUDA(cub_call([&](void* t, size_t& b) {
      return cub::DeviceSegmentedSort::SortKeys(t, b, d_cand, d_cand2, static_cast<int>(ncand), static_cast<int>(nbig),
                                                d_coff, d_coff + 1, s);
    }));
    big_rows<<<grid_of(nbig), kThreads, 0, s>>>(d_cand2, d_coff, d_bigv, nbig, 0, d_cnt, d_bnd, nullptr, nullptr);
    TSG_LAUNCHED();
  }
  TSG_CUDA(cub_call([&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, d_cnt, d_off, nv + 1, s); }));
  unsigned long long h_total = 0;
  TSG_CUDA(cudaMemcpyAsync(&h_total, d_off + nv, 8, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  int32_t* d_nbr;
  TSG_CUDA(B.get(&d_nbr, static_cast<int64_t>(h_total)));
  local_rows<<<grid_of(nv), kThreads, 0, s>>>(d_tri, d_inc_off, d_inc, nv, 1, d_cnt, d_bnd, d_big, d_off, d_nbr);
  TSG_LAUNCHED();
  if (nbig > 0) {
    big_rows<<<grid_of(nbig), kThreads, 0, s>>>(d_cand2, d_coff, d_bigv, nbig, 1, d_cnt, d_bnd, d_off, d_nbr);
    TSG_LAUNCHED();
  }
  static_assert(sizeof(unsigned long long) == sizeof(int64_t), "offset width");
  out.tri = d_tri;
  out.off = d_off;
  out.nbr = d_nbr;
  out.inc_off = d_inc_off;
  out.inc = d_inc;
  out.bnd = d_bnd;
  out.n_nbr = static_cast<int64_t>(h_total);
  return TSG_OK;
}

}  // namespace

extern "C" tsg_status tsg_topology(tsg_context* ctx, int64_t nv, int64_t nt, const int32_t* tri, int64_t* nbr_off,
                                   int32_t* nbr, int64_t nbr_cap, int64_t* inc_off, int32_t* inc, uint8_t* boundary,
                                   int64_t* n_nbr_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || nv <= 0 || nt < 0 || nv >= (int64_t{1} << 31) || 3 * nt >= (int64_t{1} << 31) || (nt > 0 && !tri) ||
      !nbr_off || !inc_off || !boundary || !n_nbr_out || (nt > 0 && (!inc || !nbr)))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: bad arguments");
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  const int64_t m3 = 3 * nt;
  DevBufs B{s, {}};
  TopoDev T;
  if (tsg_status st = topology_device(ctx, nv, nt, tri, B, T)) return st;
  if (T.n_nbr > nbr_cap) return tsg_abi::fail(TSG_ERR_INVALID, "tsg_topology: nbr capacity too small");
  const unsigned long long h_total = static_cast<unsigned long long>(T.n_nbr);
  const unsigned long long *d_off = T.off, *d_inc_off = T.inc_off;
  const int32_t *d_nbr = T.nbr, *d_inc = T.inc;
  const uint8_t* d_bnd = T.bnd;
  TSG_CUDA(cudaMemcpyAsync(nbr_off, d_off, 8 * (nv + 1), cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(inc_off, d_inc_off, 8 * (nv + 1), cudaMemcpyDeviceToHost, s));
  if (h_total) TSG_CUDA(cudaMemcpyAsync(nbr, d_nbr, 4 * h_total, cudaMemcpyDeviceToHost, s));
  if (m3) TSG_CUDA(cudaMemcpyAsync(inc, d_inc, 4 * m3, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(boundary, d_bnd, nv, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  *n_nbr_out = static_cast<int64_t>(h_total);
  return TSG_OK;
}

// Upload from points and triangles only: the topology stays on the device and feeds the device
// layout directly (no host round trip of the ~100 B/node of adjacency).  The desc's topology
// arrays are ignored; xy, tri, counts, layout, precision and order are read.
extern "C" tsg_status tsg_mesh_upload_triangles(tsg_context* ctx, const tsg_mesh_desc* d, tsg_mesh** out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || !d || !out || !d->xy || !d->tri) return tsg_abi::fail(TSG_ERR_INVALID, "null argument");
  const int64_t nv = d->nv, nt = d->nt;
  if (nv <= 0 || nt <= 0 || nv >= (int64_t{1} << 31) || 3 * nt >= (int64_t{1} << 31))
    return tsg_abi::fail(TSG_ERR_INVALID, "tsg_mesh_upload_triangles: bad counts");
  TSG_CUDA(cudaSetDevice(ctx->device));
  DevBufs B{ctx->stream, {}};
  TopoDev T;
  if (tsg_status st = topology_device(ctx, nv, nt, d->tri, B, T)) return st;
  tsg::DeviceInputs din;
  din.nbr_off = reinterpret_cast<const int64_t*>(T.off);
  din.nbr = T.nbr;
  din.inc_off = reinterpret_cast<const int64_t*>(T.inc_off);
  din.inc = T.inc;
  din.tri = T.tri;
  din.boundary = T.bnd;
  din.nnb = T.n_nbr;
  din.ninc = 3 * nt;
  return tsg_internal::mesh_upload_impl(ctx, d, &din, out);
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
  DevBufs B{s, {}};
  double2* d_xy = nullptr;
  unsigned long long *k1 = nullptr, *k2 = nullptr;
  int64_t* d_order = nullptr;
  TSG_CUDA(B.get(&d_xy, nv));
  TSG_CUDA(B.get(&k1, nv));
  TSG_CUDA(B.get(&k2, nv));
  TSG_CUDA(B.get(&d_order, nv));
  TSG_CUDA(cudaMemcpyAsync(d_xy, xy, sizeof(double2) * nv, cudaMemcpyHostToDevice, s));
  hilbert_keys<<<grid_of(nv), kThreads, 0, s>>>(d_xy, nv, xmin, ymin, sx, sy, k1);
  TSG_LAUNCHED();
  size_t bytes = 0;
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, k1, k2, nv, 0, 64, s));
  char* tmp = nullptr;
  TSG_CUDA(B.get(&tmp, static_cast<int64_t>(bytes)));
  TSG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, k1, k2, nv, 0, 64, s));
  keys_to_order<<<grid_of(nv), kThreads, 0, s>>>(k2, nv, d_order);
  TSG_LAUNCHED();
  TSG_CUDA(cudaMemcpyAsync(order_out, d_order, 8 * nv, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}
