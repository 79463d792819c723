// Device-side layout preparation: the arrays build_host_mesh (tsg_prep.cpp)
// makes on the host — slot order with degree-sorted tile windows, compact CSR over slots, fan
// records, link cycles, device triangle order, incident CSR over slots, tier lists and the
// tile records of tile_update — built with kernels and CUB sorts / scans on the GPU, bit for
// bit the same (tsg_debug_layout_check compares every array; tests/test_gpu_layout.py).
//
//   slot order   segmented stable sort of each 1024-slot window of the locality order by
//                descending degree key (boundary -> 0)              build_host_mesh "slot order"
//   rows         thread per movable slot: neighbour slots, (i1, i2, k) fan records, fan16 ring
//                positions, link-cycle successor walk (rows <= 31)  "rows, fans, cycles"
//   triangles    radix sort of (min corner slot << 32 | t)           "triangle order"
//   incident     gather + segmented sort of each slot's triangle ranks
//   tiers        stable flagged selects; `large` stable-sorted by descending degree
//   tiles        per tile: group bases of the degree groups (stable rank among equal degrees),
//                the sorted unique external slots (segmented sort + first-of-run flags + select),
//                entry-major words with local indices (binary search in the tile's externals)
// Host-side consumers (Form B schedules, halo plans, tsg_mesh_slots, the side schedule model)
// get copies of order / rank / off / nbr / fan / tier lists.
#include <cuda_runtime.h>

#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>
#include <cub/device/device_select.cuh>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <type_traits>
#include <vector>

#include "tsg_device.cuh"
#include "tsg_layout_dev.hpp"

namespace tsg {

namespace {

constexpr int kT = 256;

unsigned blocks(int64_t n) {
  const int64_t g = (n + kT - 1) / kT;
  return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 64 ? 148 * 64 : g));
}

#define FOR_I(n) \
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < (n); i += static_cast<int64_t>(gridDim.x) * blockDim.x)

// Degree sort key of the slot windows (descending degree: key = 32767 - degree key).
__global__ void k_window_keys(const int64_t* __restrict__ order, const uint8_t* __restrict__ boundary,
                              const int64_t* __restrict__ nbr_off, int64_t nv, uint16_t* __restrict__ key) {
  FOR_I(nv) {
    const int64_t v = order[i];
    const int64_t d = boundary[v] ? 0 : nbr_off[v + 1] - nbr_off[v];
    key[i] = static_cast<uint16_t>(32767 - (d > 32767 ? 32767 : d));
  }
}

__global__ void k_rank(const int64_t* __restrict__ order, int64_t nv, int64_t* __restrict__ rank) {
  FOR_I(nv) rank[order[i]] = i;
}

__global__ void k_iota64(int64_t n, int64_t* __restrict__ out) {
  FOR_I(n) out[i] = i;
}

// deg[s] (movable rows only) + the structural checks of build_host_mesh.
__global__ void k_degrees(const int64_t* __restrict__ order, const uint8_t* __restrict__ boundary,
                          const int64_t* __restrict__ nbr_off, const int64_t* __restrict__ inc_off, int64_t nv,
                          uint32_t* __restrict__ deg, unsigned long long* __restrict__ bad) {
  FOR_I(nv) {
    const int64_t v = order[i];
    uint32_t d = 0;
    if (!boundary[v]) {
      const int64_t dn = nbr_off[v + 1] - nbr_off[v], di = inc_off[v + 1] - inc_off[v];
      if (dn != di || dn <= 0 || dn >= 32768) atomicMin(bad, static_cast<unsigned long long>(v));
      d = static_cast<uint32_t>(dn > 0 && dn < 32768 ? dn : 0);
    }
    deg[i] = d;
  }
}

__global__ void k_tri_keys(const int32_t* __restrict__ tri, const int64_t* __restrict__ rank, int64_t nt,
                           unsigned long long* __restrict__ key) {
  FOR_I(nt) {
    int64_t m = rank[tri[3 * i]];
    const int64_t b = rank[tri[3 * i + 1]], c = rank[tri[3 * i + 2]];
    m = b < m ? b : m;
    m = c < m ? c : m;
    key[i] = (static_cast<unsigned long long>(m) << 32) | static_cast<unsigned long long>(i);
  }
}

__global__ void k_tri_order(const unsigned long long* __restrict__ key, int64_t nt, int64_t* __restrict__ tri_order,
                            int64_t* __restrict__ tri_rank) {
  FOR_I(nt) {
    const int64_t t = static_cast<int64_t>(key[i] & 0xffffffffULL);
    tri_order[i] = t;
    tri_rank[t] = i;
  }
}

__global__ void k_tri_slots(const int32_t* __restrict__ tri, const int64_t* __restrict__ tri_order,
                            const int64_t* __restrict__ rank, int64_t nt, int32_t* __restrict__ out) {
  FOR_I(nt) {
    const int64_t t = tri_order[i];
#pragma unroll
    for (int k = 0; k < 3; ++k) out[3 * i + k] = static_cast<int32_t>(rank[tri[3 * t + k]]);
  }
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Rows of movable slots: neighbour slots, fan records, fan16, link cycle (build_host_mesh).
__global__ void k_rows(const int64_t* __restrict__ order, const int64_t* __restrict__ rank,
                       const uint32_t* __restrict__ deg, const uint32_t* __restrict__ off,
                       const int64_t* __restrict__ nbr_off, const int32_t* __restrict__ nbr,
                       const int64_t* __restrict__ inc_off, const int32_t* __restrict__ inc,
                       const int32_t* __restrict__ tri, int64_t nv, Tiers tiers, uint32_t* __restrict__ out_nbr,
                       uint32_t* __restrict__ out_fan, uint16_t* __restrict__ out_fan16, uint8_t* __restrict__ cycpos,
                       uint8_t* __restrict__ cycrot, uint8_t* __restrict__ has_cycle,
                       unsigned long long* __restrict__ broken) {
  FOR_I(nv) {
    const int64_t s = i;
    has_cycle[s] = 0;
    const int32_t n = static_cast<int32_t>(deg[s]);
    if (n == 0) continue;
    const int64_t v = order[s];
    const int32_t* row = nbr + nbr_off[v];
    const uint32_t o = off[s];
    for (int32_t j = 0; j < n; ++j) out_nbr[o + j] = static_cast<uint32_t>(rank[row[j]]);
    const bool want_cycle = n <= kMaxCycleDeg;
    int8_t succ[kMaxCycleDeg], indeg[kMaxCycleDeg], rot[kMaxCycleDeg];
    bool cycle_ok = want_cycle;
    if (want_cycle)
      for (int32_t j = 0; j < n; ++j) succ[j] = -1, indeg[j] = 0;
    const int tier = tiers.tier(static_cast<uint32_t>(n));
    bool bad = false;
    int64_t j = 0;
    for (int64_t e = inc_off[v]; e < inc_off[v + 1]; ++e, ++j) {
      const int32_t* tv = tri + 3 * static_cast<int64_t>(inc[e]);
      const int k = tv[0] == v ? 0 : tv[1] == v ? 1 : 2;
      const int32_t a = tv[(k + 1) % 3], c = tv[(k + 2) % 3];
      const int64_t pa = lower_bound_i32(row, n, a), pc = lower_bound_i32(row, n, c);
      if (tv[k] != v || pa == n || row[pa] != a || pc == n || row[pc] != c) {
        bad = true;
        break;
      }
      const uint32_t ia = static_cast<uint32_t>(pa), ic = static_cast<uint32_t>(pc);
      if (cycle_ok) {
        if (succ[ia] >= 0 || indeg[ic] > 0) {
          cycle_ok = false;
        } else {
          succ[ia] = static_cast<int8_t>(ic);
          indeg[ic] = 1;
          rot[ia] = static_cast<int8_t>(k);
        }
      }
      if (tier < 2) {
        uint32_t p[3];
        p[k] = static_cast<uint32_t>(tier == 0 ? tiers.small_max : tiers.medium_max);
        p[(k + 1) % 3] = ia;
        p[(k + 2) % 3] = ic;
        out_fan16[o + j] = static_cast<uint16_t>(p[0] | (p[1] << 5) | (p[2] << 10));
      } else {
        out_fan16[o + j] = 0;
      }
      out_fan[o + j] = fan_pack(ia, ic, static_cast<uint32_t>(k));
    }
    if (bad) {
      atomicMin(broken, static_cast<unsigned long long>(v));
      continue;
    }
    if (cycle_ok) {
      int32_t p = 0, steps = 0;
      do {
        cycpos[o + steps] = static_cast<uint8_t>(p);
        cycrot[o + steps] = static_cast<uint8_t>(rot[p]);
        p = succ[p];
        ++steps;
      } while (p > 0 && steps < n);
      if (p == 0 && steps == n) has_cycle[s] = 1;
    }
  }
}

__global__ void k_inc_counts(const int64_t* __restrict__ order, const int64_t* __restrict__ inc_off, int64_t nv,
                             uint64_t* __restrict__ cnt) {
  FOR_I(nv) {
    const int64_t v = order[i];
    cnt[i] = static_cast<uint64_t>(inc_off[v + 1] - inc_off[v]);
  }
}

__global__ void k_vinc(const int64_t* __restrict__ order, const int64_t* __restrict__ inc_off,
                       const int32_t* __restrict__ inc, const int64_t* __restrict__ tri_rank,
                       const uint64_t* __restrict__ vinc_off, int64_t nv, uint32_t* __restrict__ vinc) {
  FOR_I(nv) {
    const int64_t v = order[i];
    uint64_t o = vinc_off[i];
    for (int64_t e = inc_off[v]; e < inc_off[v + 1]; ++e) vinc[o++] = static_cast<uint32_t>(tri_rank[inc[e]]);
  }
}

__global__ void k_tier_flags(const uint32_t* __restrict__ deg, int64_t nv, Tiers tiers, uint8_t* __restrict__ fm,
                             uint8_t* __restrict__ fh, uint8_t* __restrict__ fl, uint16_t* __restrict__ lkey) {
  FOR_I(nv) {
    const uint32_t d = deg[i];
    const int t = d ? tiers.tier(d) : -1;
    fm[i] = t == 1;
    fh[i] = t == 2;
    fl[i] = d > static_cast<uint32_t>(kMaxCycleDeg);
    lkey[i] = static_cast<uint16_t>(32767 - (d > 32767 ? 32767 : d));
  }
}

// Per tile: tmeta of the small rows (group bases in ascending valence, stable rank inside a
// group) and the tile's word count.  One CTA per tile; degrees staged in shared memory.
__global__ void __launch_bounds__(kT) k_tile_meta(const uint32_t* __restrict__ deg, int64_t nv, int kTile,
                                                  uint32_t* __restrict__ tmeta, uint32_t* __restrict__ words) {
  __shared__ uint8_t d_s[kTileMax];
  __shared__ uint32_t count[kMaxCycleDeg + 1], gbase[kMaxCycleDeg + 2];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  const int n = static_cast<int>(nv - base < kTile ? nv - base : kTile);
  for (int i = threadIdx.x; i <= kMaxCycleDeg; i += blockDim.x) count[i] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < kTile; i += blockDim.x) {
    const uint32_t d = i < n ? deg[base + i] : 0u;
    const uint8_t ds = static_cast<uint8_t>(d >= 1 && d <= static_cast<uint32_t>(kMaxCycleDeg) ? d : 0);
    d_s[i] = ds;
    if (ds) atomicAdd(&count[ds], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t w = 0;
    for (int d = 1; d <= kMaxCycleDeg; ++d) {
      gbase[d] = w;
      w += static_cast<uint32_t>(d) * count[d];
    }
    words[blockIdx.x] = (w + 3) / 4 * 4;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const uint8_t d = d_s[i];
    if (!d) {
      tmeta[base + i] = 0u;
      continue;
    }
    uint32_t k = 0;
    for (int q = 0; q < i; ++q) k += d_s[q] == d;
    tmeta[base + i] = (gbase[d] + k) | (static_cast<uint32_t>(d) << kMetaDegShift) | (count[d] << kMetaStrideShift);
  }
}

// External-slot candidates: for every row entry of a small row, the neighbour slot if it lies
// outside the row's tile, else UINT32_MAX (dropped after the sort).
__global__ void k_ext_candidates(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ off,
                                 const uint32_t* __restrict__ nbr, int64_t nv, int kTile, uint32_t* __restrict__ cand) {
  FOR_I(nv) {
    const uint32_t d = deg[i];
    const uint32_t o = off[i], o1 = off[i + 1];
    const bool small = d >= 1 && d <= static_cast<uint32_t>(kMaxCycleDeg);
    const int64_t base = (i / kTile) * kTile, end = base + kTile;
    for (uint32_t e = o; e < o1; ++e) {
      const int64_t u = nbr[e];
      cand[e] = small && (u < base || u >= end) ? static_cast<uint32_t>(u) : 0xffffffffu;
    }
  }
}

// First entries of runs of equal candidates inside each tile segment.
__global__ void __launch_bounds__(kT) k_ext_firsts(const uint32_t* __restrict__ cand,
                                                   const uint32_t* __restrict__ seg_of_tile_begin, int64_t ntiles,
                                                   uint8_t* __restrict__ first, uint32_t* __restrict__ per_tile) {
  const int64_t t = blockIdx.x;  // one CTA per tile segment
  if (t >= ntiles) return;
  const uint32_t b = seg_of_tile_begin[t], e = seg_of_tile_begin[t + 1];
  uint32_t local = 0;
  for (uint32_t i = b + threadIdx.x; i < e; i += blockDim.x) {
    const uint32_t x = cand[i];
    const bool f = x != 0xffffffffu && (i == b || cand[i - 1] != x);
    first[i] = f;
    local += f;
  }
  // block reduce
  __shared__ uint32_t red[kT / 32];
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = local;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < kT / 32; ++w) s += red[w];
    per_tile[t] = s;
  }
}

// The tile's unique external slots (run firsts of its sorted candidates) at ext_off[t].
__global__ void __launch_bounds__(kT) k_ext_compact(const uint32_t* __restrict__ cand, const uint8_t* __restrict__ first,
                                                    const uint32_t* __restrict__ tbound,
                                                    const uint32_t* __restrict__ ext_off, uint32_t* __restrict__ ext) {
  using Scan = cub::BlockScan<uint32_t, kT>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t t = blockIdx.x;
  const uint32_t b = tbound[t], e = tbound[t + 1];
  uint32_t out = ext_off[t];
  for (uint32_t c = b; c < e; c += kT) {
    const uint32_t i = c + threadIdx.x;
    const uint32_t f = i < e ? first[i] : 0u;
    uint32_t pos, total;
    Scan(tmp).ExclusiveSum(f, pos, total);
    if (f) ext[out + pos] = cand[i];
    out += total;
    __syncthreads();
  }
}

__global__ void k_tile_bounds(const uint32_t* __restrict__ off, int64_t nv, int64_t ntiles, int kTile,
                              uint32_t* __restrict__ b) {
  FOR_I(ntiles + 1) {
    const int64_t s = i * kTile;
    b[i] = off[s < nv ? s : nv];
  }
}

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t n, uint32_t x) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// Entry-major words of the small rows (build_tiles).
__global__ void k_tile_words(const uint32_t* __restrict__ deg, const uint32_t* __restrict__ off,
                             const uint32_t* __restrict__ nbr, const uint8_t* __restrict__ cycpos,
                             const uint8_t* __restrict__ cycrot, const uint8_t* __restrict__ has_cycle,
                             const uint32_t* __restrict__ tmeta, const uint32_t* __restrict__ tile_rec,
                             const uint32_t* __restrict__ ext_off, const uint32_t* __restrict__ ext, int64_t nv,
                             int kTile, uint32_t* __restrict__ trec) {
  FOR_I(nv) {
    const uint32_t d = deg[i];
    if (!(d >= 1 && d <= static_cast<uint32_t>(kMaxCycleDeg))) continue;
    const int64_t t = i / kTile, base = t * kTile, end = base + kTile;
    const uint32_t* E = ext + ext_off[t];
    const uint32_t ne = ext_off[t + 1] - ext_off[t];
    auto local = [&](uint32_t u) -> uint32_t {
      if (static_cast<int64_t>(u) >= base && static_cast<int64_t>(u) < end) return static_cast<uint32_t>(u - base);
      return static_cast<uint32_t>(kTile) + lower_bound_u32(E, ne, u);
    };
    const uint32_t meta = tmeta[i];
    const uint32_t stride = meta >> kMetaStrideShift;
    uint32_t* r = trec + tile_rec[t] + (meta & kMetaBaseMask);
    const uint32_t o0 = off[i];
    const bool cyc = has_cycle[i] != 0;
    for (uint32_t j = 0; j < d; ++j) {
      const uint32_t row = local(nbr[o0 + j]);
      const uint32_t cy = cyc ? local(nbr[o0 + cycpos[o0 + j]]) : kNoLocal;
      const uint32_t k = cyc ? cycrot[o0 + j] : 0u;
      r[j * stride] = row | (cy << kWordCycleShift) | (k << kWordRotShift);
    }
  }
}

__global__ void k_window_offsets(int64_t ntiles, int64_t nv, int kTile, int64_t* __restrict__ seg) {
  FOR_I(ntiles + 1) seg[i] = i * kTile < nv ? i * kTile : nv;
}

__global__ void k_iota32(int64_t n, int32_t* __restrict__ out) {
  FOR_I(n) out[i] = static_cast<int32_t>(i);
}

__global__ void k_widen(const uint32_t* __restrict__ in, int64_t n, uint64_t* __restrict__ out) {
  FOR_I(n) out[i] = in[i];
}

__global__ void k_narrow(const uint64_t* __restrict__ in, int64_t n, uint32_t* __restrict__ out) {
  FOR_I(n) out[i] = static_cast<uint32_t>(in[i]);
}

// Segment offsets [s0, s0 + count] relative to the first (one chunked CUB call).
template <class Off>
__global__ void k_rel_offsets(const Off* __restrict__ off, int64_t s0, int64_t count, uint32_t* __restrict__ rel) {
  FOR_I(count + 1) rel[i] = static_cast<uint32_t>(off[s0 + i] - off[s0]);
}

// Segmented sorts in chunks of segments (each call well under 2^31 items and its own temp
// storage): CUB's segmented sort at 1.5e9 items (cfg5) faulted on the device.
// TSG_SEG_CHUNK overrides the segments per chunk (tests exercise many chunks at small sizes).
int64_t seg_chunk(int64_t dflt) {
  static const int64_t env = [] {
    const char* e = std::getenv("TSG_SEG_CHUNK");
    return e ? std::max<int64_t>(1, std::atoll(e)) : 0;
  }();
  return env ? env : dflt;
}

template <class Off, class K, class V>
cudaError_t seg_sort(cudaStream_t s, const K* kin, K* kout, const V* vin, V* vout, const Off* off, int64_t nseg,
                     int64_t per_chunk, bool stable) {
  uint32_t* rel = nullptr;
  cudaError_t e = cudaMallocAsync(&rel, 4 * (per_chunk + 1), s);
  if (e != cudaSuccess) return e;
  for (int64_t s0 = 0; s0 < nseg && e == cudaSuccess; s0 += per_chunk) {
    const int64_t cnt = std::min(per_chunk, nseg - s0);
    Off ends[2];
    if ((e = cudaMemcpyAsync(&ends[0], off + s0, sizeof(Off), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
    if ((e = cudaMemcpyAsync(&ends[1], off + s0 + cnt, sizeof(Off), cudaMemcpyDeviceToHost, s)) != cudaSuccess) break;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) break;
    const int64_t b = static_cast<int64_t>(ends[0]), n = static_cast<int64_t>(ends[1]) - b;
    if (n <= 0) continue;
    k_rel_offsets<<<blocks(cnt + 1), kT, 0, s>>>(off, s0, cnt, rel);
    if ((e = cudaGetLastError()) != cudaSuccess) break;
    size_t bytes = 0;
    void* tmp = nullptr;
    auto call = [&](void* t, size_t& bb) -> cudaError_t {
      if constexpr (std::is_same_v<V, void>) {
        return cub::DeviceSegmentedSort::SortKeys(t, bb, kin + b, kout + b, static_cast<int>(n), static_cast<int>(cnt),
                                                  rel, rel + 1, s);
      } else if (stable) {
        return cub::DeviceSegmentedSort::StableSortPairs(t, bb, kin + b, kout + b, vin + b, vout + b,
                                                         static_cast<int>(n), static_cast<int>(cnt), rel, rel + 1, s);
      } else {
        return cub::DeviceSegmentedSort::SortPairs(t, bb, kin + b, kout + b, vin + b, vout + b, static_cast<int>(n),
                                                   static_cast<int>(cnt), rel, rel + 1, s);
      }
    };
    if ((e = call(nullptr, bytes)) != cudaSuccess) break;
    if ((e = cudaMallocAsync(&tmp, bytes ? bytes : 8, s)) != cudaSuccess) break;
    e = call(tmp, bytes);
    cudaFreeAsync(tmp, s);
  }
  cudaFreeAsync(rel, s);
  return e;
}

// ---------------------------------------------------------------------------------------------

struct Arena {
  cudaStream_t s;
  std::vector<void*> tmp;
  ~Arena() {
    for (void* p : tmp) cudaFreeAsync(p, s);
  }
  template <class T>
  cudaError_t get(T** p, int64_t n) {
    void* q = nullptr;
    cudaError_t e = cudaMallocAsync(&q, static_cast<size_t>(n > 0 ? n : 1) * sizeof(T), s);
    if (e == cudaSuccess) {
      tmp.push_back(q);
      *p = static_cast<T*>(q);
    }
    return e;
  }
};

// CUB temp storage sized by a query call, then the real call.
template <class F>
cudaError_t cub_call(Arena& A, F&& f) {
  size_t bytes = 0;
  cudaError_t e = f(nullptr, bytes);
  if (e != cudaSuccess) return e;
  void* t = nullptr;
  e = A.get(reinterpret_cast<char**>(&t), static_cast<int64_t>(bytes));
  if (e != cudaSuccess) return e;
  return f(t, bytes);
}

template <class T>
cudaError_t to_host(std::vector<T>& h, const T* d, int64_t n, cudaStream_t s) {
  h.resize(static_cast<size_t>(n));
  if (n == 0) return cudaSuccess;
  return cudaMemcpyAsync(h.data(), d, sizeof(T) * n, cudaMemcpyDeviceToHost, s);
}

#define DL_CUDA(x)                                                                  \
  do {                                                                              \
    cudaError_t e_ = (x);                                                           \
    if (e_ != cudaSuccess) return std::string("CUDA: ") + #x + ": " + cudaGetErrorString(e_); \
  } while (0)

}  // namespace

// TSG_PREP_TIMING=1: per-phase wall times of the device layout on stderr (stream synchronised
// at each mark; profiling aid).
struct DevPhaseTimer {
  cudaStream_t s;
  bool on = std::getenv("TSG_PREP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tsg layout] %-24s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

std::string build_device_layout(cudaStream_t s, const tsg_mesh_desc& d, const Tiers& tiers, HostMesh& hm,
                                DeviceLayout& L, int32_t tile, bool host_rows, const DeviceInputs* din) {
  const int64_t nv = d.nv, nt = d.nt;
  if (tile < 256 || tile > kTileMax || tile % 256) return "tile size must be a multiple of 256 in [256, 1536]";
  const int kTile = tile;
  if (nv <= 0 || nt <= 0) return "mesh must have vertices and triangles";
  if (nv >= (int64_t{1} << 31) - 1) return "vertex count exceeds 2^31-1";
  if (nt >= (int64_t{1} << 32)) return "triangle count exceeds 2^32";
  Arena A{s, {}};
  DevPhaseTimer pt{s};
  hm = HostMesh{};
  hm.nv = nv;
  hm.nt = nt;
  hm.tile = tile;
  const int64_t nnb = din ? din->nnb : d.nbr_off[nv], ninc = din ? din->ninc : d.inc_off[nv];
  const int64_t ntiles = (nv + kTile - 1) / kTile;

  // ---- inputs on the device
  int64_t *nbr_off, *inc_off, *rank;
  int32_t *nbr, *inc, *tri_in;
  uint8_t* bnd;
  DL_CUDA(A.get(&nbr_off, nv + 1));
  DL_CUDA(A.get(&inc_off, nv + 1));
  DL_CUDA(A.get(&nbr, nnb));
  DL_CUDA(A.get(&inc, ninc));
  DL_CUDA(A.get(&tri_in, 3 * nt));
  DL_CUDA(A.get(&bnd, nv));
  DL_CUDA(A.get(&rank, nv));
  {
    const cudaMemcpyKind kind = din ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    DL_CUDA(cudaMemcpyAsync(nbr_off, din ? din->nbr_off : d.nbr_off, 8 * (nv + 1), kind, s));
    DL_CUDA(cudaMemcpyAsync(inc_off, din ? din->inc_off : d.inc_off, 8 * (nv + 1), kind, s));
    if (nnb) DL_CUDA(cudaMemcpyAsync(nbr, din ? din->nbr : d.nbr, 4 * nnb, kind, s));
    if (ninc) DL_CUDA(cudaMemcpyAsync(inc, din ? din->inc : d.inc, 4 * ninc, kind, s));
    DL_CUDA(cudaMemcpyAsync(tri_in, din ? din->tri : d.tri, 12 * nt, kind, s));
    DL_CUDA(cudaMemcpyAsync(bnd, din ? din->boundary : d.boundary, nv, kind, s));
  }

  pt.mark("inputs");
  // ---- slot order: degree-sorted windows of the locality order (stable), rank
  int64_t* order;
  DL_CUDA(A.get(&order, nv));
  if (d.order) {
    int64_t *given, *seg;
    uint16_t *key, *key2;
    DL_CUDA(A.get(&given, nv));
    DL_CUDA(A.get(&key, nv));
    DL_CUDA(A.get(&key2, nv));
    DL_CUDA(A.get(&seg, ntiles + 1));
    DL_CUDA(cudaMemcpyAsync(given, d.order, 8 * nv, cudaMemcpyHostToDevice, s));
    k_window_keys<<<blocks(nv), kT, 0, s>>>(given, bnd, nbr_off, nv, key);
    DL_CUDA(cudaGetLastError());
    k_window_offsets<<<blocks(ntiles + 1), kT, 0, s>>>(ntiles, nv, kTile, seg);
    DL_CUDA(cudaGetLastError());
    DL_CUDA(seg_sort(s, key, key2, given, order, seg, ntiles, seg_chunk(65536), true));
  } else {
    k_iota64<<<blocks(nv), kT, 0, s>>>(nv, order);
    DL_CUDA(cudaGetLastError());
  }
  k_rank<<<blocks(nv), kT, 0, s>>>(order, nv, rank);
  DL_CUDA(cudaGetLastError());

  pt.mark("slot order");
  // ---- row lengths, checks, compact offsets
  uint32_t* deg;
  unsigned long long* flags;  // [0] inconsistent vertex, [1] broken rows vertex
  DL_CUDA(A.get(&deg, nv + 1));
  DL_CUDA(A.get(&flags, 2));
  DL_CUDA(cudaMemsetAsync(flags, 0xff, 16, s));
  DL_CUDA(cudaMemsetAsync(deg + nv, 0, 4, s));
  k_degrees<<<blocks(nv), kT, 0, s>>>(order, bnd, nbr_off, inc_off, nv, deg, flags);
  DL_CUDA(cudaGetLastError());
  uint64_t *off64, *deg64;
  DL_CUDA(A.get(&off64, nv + 1));
  DL_CUDA(A.get(&deg64, nv + 1));
  k_widen<<<blocks(nv + 1), kT, 0, s>>>(deg, nv + 1, deg64);
  DL_CUDA(cudaGetLastError());
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) {
    return cub::DeviceScan::ExclusiveSum(t, b, deg64, off64, nv + 1, s);
  }));
  unsigned long long hflags[2];
  uint64_t total = 0;
  uint32_t maxdeg = 0;
  uint32_t* dmax;
  DL_CUDA(A.get(&dmax, 1));
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, deg, dmax, nv, s); }));
  DL_CUDA(cudaMemcpyAsync(hflags, flags, sizeof hflags, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaMemcpyAsync(&total, off64 + nv, 8, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaMemcpyAsync(&maxdeg, dmax, 4, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaStreamSynchronize(s));
  if (hflags[0] != ~0ULL)
    return "movable vertex " + std::to_string(hflags[0]) +
           " has inconsistent neighbour / incident counts (or degree >= 32768)";
  if (total >= 0xffffffffULL) return "adjacency exceeds 2^32 entries";
  hm.max_deg = static_cast<int32_t>(maxdeg);
  DL_CUDA(cudaMalloc(&L.off, 4 * (nv + 1)));
  k_narrow<<<blocks(nv + 1), kT, 0, s>>>(off64, nv + 1, L.off);
  DL_CUDA(cudaGetLastError());

  pt.mark("row lengths");
  // ---- device triangle order
  int64_t* tri_rank;
  DL_CUDA(A.get(&tri_rank, nt));
  DL_CUDA(cudaMalloc(&L.tri_order, 8 * nt));
  if (d.order) {
    unsigned long long *tk, *tk2;
    DL_CUDA(A.get(&tk, nt));
    DL_CUDA(A.get(&tk2, nt));
    k_tri_keys<<<blocks(nt), kT, 0, s>>>(tri_in, rank, nt, tk);
    DL_CUDA(cudaGetLastError());
    int hi = 1;
    while (hi < 31 && (int64_t{1} << hi) < nv) ++hi;
    DL_CUDA(cub_call(A, [&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, tk, tk2, nt, 0, 32 + hi, s);
    }));
    k_tri_order<<<blocks(nt), kT, 0, s>>>(tk2, nt, L.tri_order, tri_rank);
    DL_CUDA(cudaGetLastError());
  } else {
    k_iota64<<<blocks(nt), kT, 0, s>>>(nt, L.tri_order);
    DL_CUDA(cudaGetLastError());
    k_iota64<<<blocks(nt), kT, 0, s>>>(nt, tri_rank);
    DL_CUDA(cudaGetLastError());
  }
  DL_CUDA(cudaMalloc(&L.tri, 12 * nt));
  k_tri_slots<<<blocks(nt), kT, 0, s>>>(tri_in, L.tri_order, rank, nt, L.tri);
  DL_CUDA(cudaGetLastError());

  pt.mark("triangle order");
  // ---- rows: neighbour slots, fan records, fan16, link cycles
  DL_CUDA(cudaMalloc(&L.nbr, 4 * (total ? total : 1)));
  DL_CUDA(cudaMalloc(&L.fan, 4 * (total ? total : 1)));
  DL_CUDA(cudaMalloc(&L.fan16, 2 * (total ? total : 1)));
  uint8_t *cycpos, *cycrot, *has_cycle;
  DL_CUDA(A.get(&cycpos, static_cast<int64_t>(total)));
  DL_CUDA(A.get(&cycrot, static_cast<int64_t>(total)));
  DL_CUDA(A.get(&has_cycle, nv));
  DL_CUDA(cudaMemsetAsync(cycpos, 0, total ? total : 1, s));
  DL_CUDA(cudaMemsetAsync(cycrot, 0, total ? total : 1, s));
  k_rows<<<blocks(nv), kT, 0, s>>>(order, rank, deg, L.off, nbr_off, nbr, inc_off, inc, tri_in, nv, tiers, L.nbr,
                                    L.fan, L.fan16, cycpos, cycrot, has_cycle, flags + 1);
  DL_CUDA(cudaGetLastError());

  pt.mark("rows");
  // ---- incident CSR over slots (device triangle ids, ascending per row)
  uint64_t *icnt, *ioff64;
  DL_CUDA(A.get(&icnt, nv + 1));
  DL_CUDA(A.get(&ioff64, nv + 1));
  DL_CUDA(cudaMemsetAsync(icnt + nv, 0, 8, s));
  k_inc_counts<<<blocks(nv), kT, 0, s>>>(order, inc_off, nv, icnt);
  DL_CUDA(cudaGetLastError());
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, icnt, ioff64, nv + 1, s); }));
  uint64_t itotal = 0;
  DL_CUDA(cudaMemcpyAsync(&itotal, ioff64 + nv, 8, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaMemcpyAsync(&hflags[1], flags + 1, 8, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaStreamSynchronize(s));
  if (hflags[1] != ~0ULL) return "incident / neighbour lists disagree at vertex " + std::to_string(hflags[1]);
  if (itotal >= 0xffffffffULL) return "incidence exceeds 2^32 entries";
  DL_CUDA(cudaMalloc(&L.vinc_off, 4 * (nv + 1)));
  k_narrow<<<blocks(nv + 1), kT, 0, s>>>(ioff64, nv + 1, L.vinc_off);
  DL_CUDA(cudaGetLastError());
  {
    uint32_t* vtmp;
    DL_CUDA(A.get(&vtmp, static_cast<int64_t>(itotal)));
    DL_CUDA(cudaMalloc(&L.vinc, 4 * (itotal ? itotal : 1)));
    k_vinc<<<blocks(nv), kT, 0, s>>>(order, inc_off, inc, tri_rank, ioff64, nv, vtmp);
    DL_CUDA(cudaGetLastError());
    DL_CUDA(seg_sort(s, vtmp, L.vinc, static_cast<const void*>(nullptr), static_cast<void*>(nullptr), L.vinc_off, nv,
                     seg_chunk(1 << 20), false));
  }

  pt.mark("incident CSR");
  // ---- tier lists (slot order), `large` by descending valence (stable)
  {
    uint8_t *fm, *fh, *fl;
    uint16_t *lkey, *lkey2;
    int64_t* nsel;
    int32_t *iota, *ltmp;
    DL_CUDA(A.get(&fm, nv));
    DL_CUDA(A.get(&fh, nv));
    DL_CUDA(A.get(&fl, nv));
    DL_CUDA(A.get(&lkey, nv));
    DL_CUDA(A.get(&lkey2, nv));
    DL_CUDA(A.get(&nsel, 3));
    DL_CUDA(A.get(&iota, nv));
    DL_CUDA(A.get(&ltmp, nv));
    k_tier_flags<<<blocks(nv), kT, 0, s>>>(deg, nv, tiers, fm, fh, fl, lkey);
    DL_CUDA(cudaGetLastError());
    k_iota32<<<blocks(nv), kT, 0, s>>>(nv, iota);
    DL_CUDA(cudaGetLastError());
    int32_t *med, *hub, *lrg;
    DL_CUDA(A.get(&med, nv));
    DL_CUDA(A.get(&hub, nv));
    DL_CUDA(A.get(&lrg, nv));
    DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, iota, fm, med, nsel, nv, s); }));
    DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, iota, fh, hub, nsel + 1, nv, s); }));
    DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, iota, fl, ltmp, nsel + 2, nv, s); }));
    DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceSelect::Flagged(t, b, lkey, fl, lkey2, nsel + 2, nv, s); }));
    int64_t hn[3];
    DL_CUDA(cudaMemcpyAsync(hn, nsel, sizeof hn, cudaMemcpyDeviceToHost, s));
    DL_CUDA(cudaStreamSynchronize(s));
    uint16_t* lk3;
    DL_CUDA(A.get(&lk3, hn[2]));
    if (hn[2] > 0)
      DL_CUDA(cub_call(A, [&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, lkey2, lk3, ltmp, lrg, hn[2], 0, 16, s);
      }));
    DL_CUDA(to_host(hm.medium, med, hn[0], s));
    DL_CUDA(to_host(hm.hubs, hub, hn[1], s));
    DL_CUDA(to_host(hm.large, lrg, hn[2], s));
  }

  pt.mark("tier lists");
  // ---- tiles: meta words, sorted external slots, entry-major words
  uint32_t *words, *ext_cnt, *tbound, *cand, *cand2;
  uint8_t* first;
  DL_CUDA(cudaMalloc(&L.tmeta, 4 * nv));
  DL_CUDA(A.get(&words, ntiles + 1));
  DL_CUDA(A.get(&ext_cnt, ntiles + 1));
  DL_CUDA(A.get(&tbound, ntiles + 1));
  DL_CUDA(A.get(&cand, static_cast<int64_t>(total)));
  DL_CUDA(A.get(&cand2, static_cast<int64_t>(total)));
  DL_CUDA(A.get(&first, static_cast<int64_t>(total)));
  DL_CUDA(cudaMemsetAsync(words + ntiles, 0, 4, s));
  DL_CUDA(cudaMemsetAsync(ext_cnt + ntiles, 0, 4, s));
  k_tile_meta<<<static_cast<unsigned>(ntiles), kT, 0, s>>>(deg, nv, kTile, L.tmeta, words);
  DL_CUDA(cudaGetLastError());
  k_ext_candidates<<<blocks(nv), kT, 0, s>>>(deg, L.off, L.nbr, nv, kTile, cand);
  DL_CUDA(cudaGetLastError());
  k_tile_bounds<<<blocks(ntiles + 1), kT, 0, s>>>(L.off, nv, ntiles, kTile, tbound);
  DL_CUDA(cudaGetLastError());
  DL_CUDA(seg_sort(s, cand, cand2, static_cast<const void*>(nullptr), static_cast<void*>(nullptr), tbound, ntiles,
                   seg_chunk(16384), false));
  k_ext_firsts<<<static_cast<unsigned>(ntiles), kT, 0, s>>>(cand2, tbound, ntiles, first, ext_cnt);
  DL_CUDA(cudaGetLastError());
  DL_CUDA(cudaMalloc(&L.ext_off, 4 * (ntiles + 1)));
  DL_CUDA(cudaMalloc(&L.tile_rec, 4 * (ntiles + 1)));
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, ext_cnt, L.ext_off, ntiles + 1, s); }));
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceScan::ExclusiveSum(t, b, words, L.tile_rec, ntiles + 1, s); }));
  uint32_t hext = 0, hwords = 0, mx[2] = {0, 0};
  uint32_t* dmx;
  DL_CUDA(A.get(&dmx, 2));
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, ext_cnt, dmx, ntiles, s); }));
  DL_CUDA(cub_call(A, [&](void* t, size_t& b) { return cub::DeviceReduce::Max(t, b, words, dmx + 1, ntiles, s); }));
  DL_CUDA(cudaMemcpyAsync(&hext, L.ext_off + ntiles, 4, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaMemcpyAsync(&hwords, L.tile_rec + ntiles, 4, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaMemcpyAsync(mx, dmx, 8, cudaMemcpyDeviceToHost, s));
  DL_CUDA(cudaStreamSynchronize(s));
  if (kTile + static_cast<int64_t>(mx[0]) >= static_cast<int64_t>(kNoLocal))
    return "a tile references more than " + std::to_string(kNoLocal - kTile - 1) + " external vertices";
  if (mx[1] > kMetaBaseMask + 1) return "tile words exceed the meta offset field";
  hm.max_ext = static_cast<int32_t>(mx[0]);
  hm.max_rec_words = static_cast<int32_t>(mx[1]);
  DL_CUDA(cudaMalloc(&L.ext, sizeof(uint32_t) * static_cast<size_t>(hext ? hext : 1)));
  k_ext_compact<<<static_cast<unsigned>(ntiles), kT, 0, s>>>(cand2, first, tbound, L.ext_off, L.ext);
  DL_CUDA(cudaGetLastError());
  DL_CUDA(cudaMalloc(&L.trec, sizeof(uint32_t) * static_cast<size_t>(hwords ? hwords : 1)));
  DL_CUDA(cudaMemsetAsync(L.trec, 0, sizeof(uint32_t) * static_cast<size_t>(hwords ? hwords : 1), s));
  k_tile_words<<<blocks(nv), kT, 0, s>>>(deg, L.off, L.nbr, cycpos, cycrot, has_cycle, L.tmeta, L.tile_rec, L.ext_off,
                                         L.ext, nv, kTile, L.trec);
  DL_CUDA(cudaGetLastError());

  pt.mark("tiles");
  // ---- host copies the host side reads (Form B schedules, halo plans, slots, tier sizes)
  DL_CUDA(to_host(hm.off, L.off, nv + 1, s));
  if (host_rows) {
    DL_CUDA(to_host(hm.order, order, nv, s));
    DL_CUDA(to_host(hm.rank, rank, nv, s));
    DL_CUDA(to_host(hm.nbr, L.nbr, static_cast<int64_t>(total), s));
    DL_CUDA(to_host(hm.fan, L.fan, static_cast<int64_t>(total), s));
    DL_CUDA(to_host(hm.tri_order, L.tri_order, nt, s));
  }
  if (d.order) {
    DL_CUDA(cudaMalloc(&L.order, 8 * nv));
    DL_CUDA(cudaMemcpyAsync(L.order, order, 8 * nv, cudaMemcpyDeviceToDevice, s));
  } else {
    cudaFree(L.tri_order);
    L.tri_order = nullptr;
  }
  DL_CUDA(cudaStreamSynchronize(s));
  pt.mark("host copies");
  return "";
}

// Every HostMesh array of the device build, downloaded (tests: compared with build_host_mesh).
std::string download_layout(cudaStream_t s, const DeviceLayout& L, HostMesh& hm) {
  const int64_t nv = hm.nv, nt = hm.nt;
  const int64_t kTile = hm.tile;
  DL_CUDA(cudaStreamSynchronize(s));
  hm.fan16.resize(hm.nbr.size());
  if (!hm.nbr.empty()) DL_CUDA(cudaMemcpy(hm.fan16.data(), L.fan16, 2 * hm.nbr.size(), cudaMemcpyDeviceToHost));
  hm.tri.resize(3 * nt);
  DL_CUDA(cudaMemcpy(hm.tri.data(), L.tri, 12 * nt, cudaMemcpyDeviceToHost));
  hm.vinc_off.resize(nv + 1);
  DL_CUDA(cudaMemcpy(hm.vinc_off.data(), L.vinc_off, 4 * (nv + 1), cudaMemcpyDeviceToHost));
  hm.vinc.resize(hm.vinc_off[nv]);
  if (!hm.vinc.empty()) DL_CUDA(cudaMemcpy(hm.vinc.data(), L.vinc, 4 * hm.vinc.size(), cudaMemcpyDeviceToHost));
  const int64_t ntiles = (nv + kTile - 1) / kTile;
  hm.tmeta.resize(nv);
  DL_CUDA(cudaMemcpy(hm.tmeta.data(), L.tmeta, 4 * nv, cudaMemcpyDeviceToHost));
  hm.tile_rec.resize(ntiles + 1);
  DL_CUDA(cudaMemcpy(hm.tile_rec.data(), L.tile_rec, 4 * (ntiles + 1), cudaMemcpyDeviceToHost));
  hm.ext_off.resize(ntiles + 1);
  DL_CUDA(cudaMemcpy(hm.ext_off.data(), L.ext_off, 4 * (ntiles + 1), cudaMemcpyDeviceToHost));
  hm.ext.resize(hm.ext_off[ntiles]);
  if (!hm.ext.empty()) DL_CUDA(cudaMemcpy(hm.ext.data(), L.ext, 4 * hm.ext.size(), cudaMemcpyDeviceToHost));
  hm.trec.resize(hm.tile_rec[ntiles]);
  if (!hm.trec.empty()) DL_CUDA(cudaMemcpy(hm.trec.data(), L.trec, 4 * hm.trec.size(), cudaMemcpyDeviceToHost));
  return "";
}

void free_layout(DeviceLayout& L) {
  for (void* p : {static_cast<void*>(L.off), static_cast<void*>(L.nbr), static_cast<void*>(L.fan),
                  static_cast<void*>(L.fan16), static_cast<void*>(L.tmeta), static_cast<void*>(L.tile_rec),
                  static_cast<void*>(L.ext_off), static_cast<void*>(L.ext), static_cast<void*>(L.trec),
                  static_cast<void*>(L.vinc_off), static_cast<void*>(L.vinc), static_cast<void*>(L.tri),
                  static_cast<void*>(L.order), static_cast<void*>(L.tri_order)})
    cudaFree(p);
  L = DeviceLayout{};
}

}  // namespace tsg
