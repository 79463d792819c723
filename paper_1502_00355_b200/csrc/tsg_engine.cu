// libtsg.so — the C ABI (include/tsg.h) over the sm_100a Smart Laplacian kernels.
//
// Device residency: one tsg_mesh holds the slot-ordered topology (compact CSR + fan records,
// incident CSR, device triangles), two coordinate buffers and the per-pass stats.  The pass
// loop runs as a CUDA graph whose body is one pass and whose WHILE condition is set on the
// device by the finalize kernel, so a whole smooth() is one graph launch and no host
// round-trip happens between passes (reference loop: proj/src/smoothing.cpp:98-141).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <map>
#include <type_traits>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "tsg.h"
#include "tsg_flow.cuh"
#include "tsg_peer.cuh"
#include "tsg_kernels.cuh"
#include "tsg_internal.hpp"
#include "tsg_layout_dev.hpp"
#include "tsg_prep.hpp"

namespace {

using tsg_abi::fail;
using tsg_abi::g_err;

// Valence tiers: thread-per-vertex (<= 12, CTA of 128, every slot in Form A), thread-per-vertex
// over a list (13..31, CTA of 64: larger per-thread ring), CTA-per-vertex hubs (>= 32).
constexpr int kMaxSmallDeg = 10;
constexpr int kMaxMedDeg = 31;
constexpr tsg::Tiers kTiers{kMaxSmallDeg, kMaxMedDeg};
constexpr int kGraphUnroll = 4;  // passes per WHILE-body iteration (graph_unroll)
constexpr int kHubCap = 4096;     // hub entries staged in shared memory
constexpr int kTileThreads = 256;  // tile_update: threads per 1024-slot tile
constexpr int kTileExtCap = 2048;  // ... external coordinates staged in shared memory
constexpr int kTileRecCap = 12288;  // ... row words staged in shared memory (multiple of 4)
// formb_chunk_update: record double buffer + per-thread pass-start / view rings (f64 pairs)
constexpr int kChunkRecSmem = 2 * 256 * tsg::kChunkRecWords * 4 + 2 * tsg::kChunkRecMaxDeg * 256 * 16;
#ifndef TSG_WARP_TIER_WARPS
#define TSG_WARP_TIER_WARPS 1
#endif
constexpr int kWarpTierWarps = TSG_WARP_TIER_WARPS;  // warp-per-row tier: warps per CTA (1: finest dispatch in the tail; -0.6 % vs 8, measured)
constexpr int kWarpTierCap = 256;  // ... row entries staged in shared memory per warp
#ifndef TSG_HUB_FAST_MIN
#define TSG_HUB_FAST_MIN 256
#endif
constexpr int kHubFastMin = TSG_HUB_FAST_MIN;  // rows above this valence get a CTA each
constexpr int kSideWarps = 4;   // side_rows: warps per CTA (one per SM sub-partition), one CTA per SM
constexpr int kSideRegs = 32;   // ... registers per thread (fits beside 3 tile CTAs of 80 registers)

template <class T>
tsg_status dalloc(T** p, size_t count, int64_t* bytes) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
  if (e != cudaSuccess) return fail(TSG_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  *bytes += static_cast<int64_t>(count * sizeof(T));
  return TSG_OK;
}

template <class T>
tsg_status upload(T** p, const std::vector<T>& v, int64_t* bytes, cudaStream_t s) {
  tsg_status st = dalloc(p, v.size(), bytes);
  if (st) return st;
  if (!v.empty()) {
    cudaError_t e = cudaMemcpyAsync(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return fail(TSG_ERR_CUDA, std::string("cudaMemcpyAsync: ") + cudaGetErrorString(e));
  }
  return TSG_OK;
}

// Gather original-order f64 pairs into slot order (both buffers) and back.
// Largest coordinate magnitude as ordered u64 bits (NaN counts as +inf): per-thread maximum,
// then one warp reduction and one atomic per warp at the end of the grid-stride loop.
__device__ __forceinline__ double abs_max2(double x, double y) {
  return (x != x || y != y) ? INFINITY : fmax(fabs(x), fabs(y));
}
__device__ __forceinline__ void commit_maxabs(double m, unsigned long long* maxabs) {
  unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(m));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long c = __shfl_xor_sync(0xffffffffu, b, o);
    b = c > b ? c : b;
  }
  if ((threadIdx.x & 31) == 0 && b) atomicMax(maxabs, b);
}

template <typename R, bool kSoA>
__global__ void coords_from_orig(const double* __restrict__ xy, const int64_t* __restrict__ order,
                                 int64_t nv, tsg::Coords<R, kSoA> b0, tsg::Coords<R, kSoA> b1,
                                 unsigned long long* maxabs) {
  double m = 0.0;
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nv;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t v = order ? order[s] : s;
    const double2 q = reinterpret_cast<const double2*>(xy)[v];  // one 16-B gather (staging buffers are cudaMalloc'd)
    const double x = q.x, y = q.y;
    const auto p = tsg::Arith<R>::make(static_cast<R>(x), static_cast<R>(y));
    b0.store(s, p);
    b1.store(s, p);
    m = fmax(m, abs_max2(x, y));
  }
  commit_maxabs(m, maxabs);
}

template <typename R, bool kSoA>
__global__ void coords_to_orig(tsg::Coords<R, kSoA> b, const int32_t* __restrict__ rank,
                               int64_t nv, double* __restrict__ xy) {
  // Gather by original id (coalesced writes, random 16-byte reads): measured cheaper than the
  // scatter by slot (random partial-sector writes read the sectors back: cfg3 339 vs 564 us).
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const auto p = b.load_mut(rank ? rank[v] : v);
    reinterpret_cast<double2*>(xy)[v] = make_double2(static_cast<double>(p.x), static_cast<double>(p.y));
  }
}

// Current coordinates -> original-order f64 pairs, the current buffer chosen on the device
// from the pass counter (ping-pong: the last pass wrote buffer (pass & 1) ? buf1 : buf0).
template <typename R, bool kSoA>
__global__ void coords_to_orig_parity(tsg::Coords<R, kSoA> b0, tsg::Coords<R, kSoA> b1, int32_t swap,
                                      const tsg::PassState* st, const int32_t* __restrict__ rank, int64_t nv,
                                      double* __restrict__ xy) {
  const tsg::Coords<R, kSoA> b = (swap == tsg::kSwapPingPong && (st->pass & 1)) ? b1 : b0;
  for (int64_t v = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; v < nv;
       v += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const auto p = b.load_mut(rank ? rank[v] : v);
    reinterpret_cast<double2*>(xy)[v] = make_double2(static_cast<double>(p.x), static_cast<double>(p.y));
  }
}

// rank[order[s]] = s: the slot of each original vertex (for the gathers above).
__global__ void rank_of_order(const int64_t* __restrict__ order, int64_t nv, int32_t* __restrict__ rank) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nv;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x)
    rank[order[s]] = static_cast<int32_t>(s);
}

__global__ void save_state(const tsg::PassState* st, tsg::PassState* out) { *out = *st; }
__global__ void set_state(tsg::PassState* st, int32_t pass, int32_t stop) { *st = tsg::PassState{pass, 1, stop, 0}; }

// Start of a smooth: pass state, per-pass stat slots, and the side_rows ticket pair (normally
// left zeroed by each launch's last warp; reset here too so an aborted run cannot leak into the
// next).
__global__ void reset_pass_state(tsg::PassState* st, int32_t* slot_acc, unsigned long long* slot_md, int64_t n,
                                 uint32_t* side_ctr) {
  const int64_t i0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (i0 == 0) {
    *st = tsg::PassState{0, 0, 0, 0};
    side_ctr[0] = 0;
    side_ctr[1] = 0;
  }
  for (int64_t i = i0; i < n; i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    slot_acc[i] = 0;
    slot_md[i] = 0ull;
  }
}

__global__ void zero_u64(unsigned long long* p) { *p = 0ull; }

// Stop rule over the per-pass totals of a dataflow launch of np passes (the reference's order,
// proj/src/smoothing.cpp:132-141): the first pass with no moves, or with a maximum displacement
// below tol_abs, ends the smooth; else MaxIters.  One warp; the pass state it writes is what
// finalize_pass would have left (the batch API reads the final buffer parity from it).  Only
// used where passes after the stopping one cannot change the coordinates (tol_abs == 0: the
// stop can only be NoMoves, after which every pass is a no-op).
__global__ void flow_stop_state(const int32_t* slot_acc, const unsigned long long* slot_md, int32_t np, double tol_abs,
                                tsg::PassState* st) {
  const int lane = threadIdx.x;
  int32_t it = np, stop = tsg::kStopMaxIters;
  for (int32_t p = 0; p < np; ++p) {
    int32_t a = slot_acc[static_cast<int64_t>(p) * tsg::kStatSlots + lane];
    unsigned long long b = slot_md[static_cast<int64_t>(p) * tsg::kStatSlots + lane];
    a = __reduce_add_sync(0xffffffffu, a);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long q = __shfl_xor_sync(0xffffffffu, b, o);
      b = q > b ? q : b;
    }
    if (a == 0) {
      it = p + 1;
      stop = tsg::kStopNoMoves;
      break;
    }
    if (__longlong_as_double(static_cast<long long>(b)) < tol_abs) {
      it = p + 1;
      stop = tsg::kStopDisplacement;
      break;
    }
  }
  if (lane == 0) *st = tsg::PassState{it, 1, stop, 0};
}

template <typename R>
__global__ void to_double_scatter(const R* __restrict__ in, const int64_t* __restrict__ order,
                                  int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[order ? order[i] : i] = static_cast<double>(in[i]);
}

// Halo exchange: current coordinates of the send slots -> packed f64 pairs, and packed pairs
// -> both buffers of the (locally pinned) halo slots.
template <typename R, bool kSoA>
__global__ void halo_pack(tsg::Coords<R, kSoA> cur, const int32_t* __restrict__ slots, int64_t n,
                          double* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const auto p = cur.load_mut(slots[i]);
    out[2 * i] = static_cast<double>(p.x);
    out[2 * i + 1] = static_cast<double>(p.y);
  }
}

template <typename R, bool kSoA>
__global__ void halo_unpack(tsg::Coords<R, kSoA> b0, tsg::Coords<R, kSoA> b1, const int32_t* __restrict__ slots,
                            int64_t n, const double* __restrict__ in, unsigned long long* maxabs) {
  double m = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = in[2 * i], y = in[2 * i + 1];
    const auto p = tsg::Arith<R>::make(static_cast<R>(x), static_cast<R>(y));
    b0.store(slots[i], p);
    b1.store(slots[i], p);
    m = fmax(m, abs_max2(x, y));
  }
  commit_maxabs(m, maxabs);
}

__global__ void scatter_i8(const int8_t* __restrict__ in, const int64_t* __restrict__ order,
                           int64_t n, int8_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[order ? order[i] : i] = in[i];
}

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

__global__ void selftest_alpha(int64_t n, uint64_t seed, int steps, unsigned long long* max_err,
                               unsigned long long* nonfinite) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double c[6];
    const uint64_t h = mix64(seed ^ static_cast<uint64_t>(i));
    const double scale = __longlong_as_double(static_cast<long long>((1023ULL + (h % 61) - 30) << 52));
    for (int k = 0; k < 6; ++k)
      c[k] = (static_cast<double>(mix64(h + 7 * k + 1) >> 11) * 0x1.0p-53 - 0.5) * scale;
    if ((h >> 60) == 0) {  // near-degenerate: third corner almost on the first edge
      const double t = static_cast<double>(mix64(h + 99) >> 11) * 0x1.0p-53;
      c[4] = c[0] + t * (c[2] - c[0]) + 1e-9 * scale;
      c[5] = c[1] + t * (c[3] - c[1]);
    }
    const double e = tsg::alpha_plain<double>(c[0], c[1], c[2], c[3], c[4], c[5]);
    const double f = steps == 1 ? tsg::alpha_fast<double, 1>(c[0], c[1], c[2], c[3], c[4], c[5])
                                : tsg::alpha_fast<double, 2>(c[0], c[1], c[2], c[3], c[4], c[5]);
    if (!(fabs(f) <= 2.0)) {
      atomicAdd(nonfinite, 1ULL);
      continue;
    }
    if (fabs(e) <= 1.0) {
      const double d = fabs(f - e);
      atomicMax(max_err, static_cast<unsigned long long>(__double_as_longlong(d)));
    }
  }
}

unsigned grid_for(int64_t n, int block) {
  const int64_t g = (n + block - 1) / block;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(g, 148 * 64)));
}

// The cycle path's fast α/K (ring_pair, v at a random rotation of the triangle) against the
// reference's literal α / K: max |t - α_ref/K| in α/K units (error analysis: kGuardCycle).
__global__ void selftest_alpha_cycle(int64_t n, uint64_t seed, unsigned long long* max_err,
                                     unsigned long long* nonfinite) {
  constexpr double K = tsg::Arith<double>::kAlpha;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double c[6];
    const uint64_t h = mix64(seed ^ static_cast<uint64_t>(i));
    const double scale = __longlong_as_double(static_cast<long long>((1023ULL + (h % 61) - 30) << 52));
    const double off = (h >> 40) & 1 ? 0.0 : scale * 37.0;  // also away from the origin
    for (int k = 0; k < 6; ++k)
      c[k] = off + (static_cast<double>(mix64(h + 7 * k + 1) >> 11) * 0x1.0p-53 - 0.5) * scale;
    if ((h >> 60) == 0) {  // near-degenerate: third corner almost on the first edge
      const double t = static_cast<double>(mix64(h + 99) >> 11) * 0x1.0p-53;
      c[4] = c[0] + t * (c[2] - c[0]) + 1e-9 * scale;
      c[5] = c[1] + t * (c[3] - c[1]);
    }
    const double e = tsg::alpha_plain<double>(c[0], c[1], c[2], c[3], c[4], c[5]);
    const int r = static_cast<int>((h >> 20) % 3);  // v = p_r, then the cyclic successors
    const double2 v = make_double2(c[2 * r], c[2 * r + 1]);
    const double2 a = make_double2(c[2 * ((r + 1) % 3)], c[2 * ((r + 1) % 3) + 1]);
    const double2 b = make_double2(c[2 * ((r + 2) % 3)], c[2 * ((r + 2) % 3) + 1]);
    double tp, tc;
    tsg::ring_pair<double>(tsg::ring_edge<double>(a, v, v), tsg::ring_edge<double>(b, v, v), tp, tc);
    if (!(fabs(tp) <= 1.0)) {
      atomicAdd(nonfinite, 1ULL);
      continue;
    }
    if (fabs(e) <= 1.0) {
      const double d = fabs(fma(tp, K, -e)) / K;
      atomicMax(max_err, static_cast<unsigned long long>(__double_as_longlong(d)));
    }
  }
}

// Partitioned driver (tsg_dist_*): this partition's totals of the current pass, {accepted,
// max displacement} as two doubles (exact: counts < 2^53), for the cross-partition all-gather
// (0 / 0 once the global stop fired: the pass did not run).
__global__ void dist_fold(const tsg::PassState* st, const int32_t* slot_acc, const unsigned long long* slot_md,
                          double* out) {
  const int lane = threadIdx.x;
  const int q = st->pass;
  const bool done = st->done != 0;
  int32_t acc = done ? 0 : slot_acc[q * tsg::kStatSlots + lane];
  unsigned long long mdb = done ? 0ull : slot_md[q * tsg::kStatSlots + lane];
  acc = __reduce_add_sync(0xffffffffu, acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, mdb, o);
    mdb = other > mdb ? other : mdb;
  }
  if (lane == 0) {
    out[0] = static_cast<double>(acc);
    out[1] = __longlong_as_double(static_cast<long long>(mdb));
  }
}

// The reference's stop rule (smoothing.cpp:132-141) on the totals of all partitions (the
// all-gathered {accepted, max displacement} pairs: sum and max); advances the device pass
// counter exactly like finalize_pass.
__global__ void dist_finalize(tsg::PassState* st, const double* gathered, int32_t n_parts, int32_t* pass_acc,
                              unsigned long long* pass_md, double tol_abs, int32_t max_iters) {
  if (st->done) return;
  const int q = st->pass;
  long long acc = 0;
  double md = 0.0;
  for (int r = 0; r < n_parts; ++r) {
    acc += static_cast<long long>(gathered[2 * r]);
    md = gathered[2 * r + 1] > md ? gathered[2 * r + 1] : md;
  }
  pass_acc[q] = static_cast<int32_t>(acc);
  pass_md[q] = static_cast<unsigned long long>(__double_as_longlong(md));
  st->pass = q + 1;
  if (acc == 0) {
    st->done = 1;
    st->stop = tsg::kStopNoMoves;
  } else if (md < tol_abs) {
    st->done = 1;
    st->stop = tsg::kStopDisplacement;
  } else if (q + 1 >= max_iters) {
    st->done = 1;
    st->stop = tsg::kStopMaxIters;
  }
}

// Halo copies of the partitioned driver: the current buffer is chosen on the device (the pass
// just executed wrote N = buffer ((pass & 1) ? buf0 : buf1) in ping-pong mode, buf0 in copy
// mode); nothing is copied once the global stop fired.
template <typename R, bool kSoA>
__global__ void dist_halo_pack(tsg::Coords<R, kSoA> b0, tsg::Coords<R, kSoA> b1, int32_t swap,
                               const tsg::PassState* st, const int32_t* __restrict__ slots, int64_t n,
                               double* __restrict__ out) {
  if (st->done) return;
  const tsg::Coords<R, kSoA> cur = (swap == tsg::kSwapCopy || (st->pass & 1)) ? b0 : b1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const auto p = cur.load_mut(slots[i]);
    out[2 * i] = static_cast<double>(p.x);
    out[2 * i + 1] = static_cast<double>(p.y);
  }
}

template <typename R, bool kSoA>
__global__ void dist_halo_unpack(tsg::Coords<R, kSoA> b0, tsg::Coords<R, kSoA> b1, const tsg::PassState* st,
                                 const int32_t* __restrict__ slots, int64_t n, const double* __restrict__ in,
                                 unsigned long long* maxabs) {
  if (st->done) return;
  double m = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double x = in[2 * i], y = in[2 * i + 1];
    const auto p = tsg::Arith<R>::make(static_cast<R>(x), static_cast<R>(y));
    b0.store(slots[i], p);
    b1.store(slots[i], p);
    m = fmax(m, abs_max2(x, y));
  }
  commit_maxabs(m, maxabs);
}

// The dynamic shared-memory limit of a kernel is a per-function, per-device setting shared by
// every mesh: only ever raise it (a later mesh needing less must not lower the limit an earlier
// mesh's launches rely on).
// Slots per tile the tile kernel is compiled for (tsg_mesh_upload picks one per mesh).
constexpr int kTileSizes[] = {768, 1024, 1280};

bool tile_supported(int tile) {
  for (int t : kTileSizes)
    if (t == tile) return true;
  return false;
}

// f(std::integral_constant<int, tile>) for a supported tile size.
template <class F>
void with_tile(int tile, F&& f) {
  switch (tile) {
    case 768: f(std::integral_constant<int, 768>{}); break;
    case 1024: f(std::integral_constant<int, 1024>{}); break;
    default: f(std::integral_constant<int, 1280>{}); break;
  }
}

template <class K>
cudaError_t raise_smem_limit(K* fn, int bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, int> limit;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  int& cur = limit[{dev, reinterpret_cast<const void*>(fn)}];
  if (bytes <= cur) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) cur = bytes;
  return e;
}

struct GraphCache {
  bool valid = false;
  int32_t form = -1, strategy = -1, chunks = -1, swap = -1, max_iters = -1;
  bool peer = false;
  double tol_abs = 0.0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels_per_pass = 0;
  void reset() {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    exec = nullptr;
    graph = nullptr;
    valid = false;
  }
};

}  // namespace


struct tsg_mesh {
  tsg_context* ctx = nullptr;
  tsg::HostMesh hm;
  int32_t layout = 0, prec = 0;
  size_t rsize = 8;
  int64_t bytes = 0;
  void* buf[2] = {nullptr, nullptr};
  void* init = nullptr;  // slot-ordered copy of the coordinates given at upload / set_coords
  uint16_t* d_fan16 = nullptr;
  uint32_t *d_tmeta = nullptr, *d_tile_rec = nullptr, *d_ext_off = nullptr, *d_tile_ext = nullptr;
  uint32_t* d_trec = nullptr;
  uint32_t *d_off = nullptr, *d_nbr = nullptr, *d_fan = nullptr, *d_vinc_off = nullptr,
           *d_vinc = nullptr;
  int32_t *d_tri = nullptr, *d_hubs = nullptr, *d_medium = nullptr, *d_large = nullptr;
  uint32_t* d_side_ctr = nullptr;  // side_rows ticket pair (zero between launches)
  int32_t num_sms = 0;
  // Rows above the cycle tiers: persistent side_rows kernel beside the tile grid, or per-tier
  // grids after it (tsg_mesh_side_schedule; AUTO decides from the estimated work at upload).
  int32_t side_mode = TSG_SIDE_AUTO;
  bool side_persist_auto = false;
  int64_t n_side_cta = 0;  // persistent mode: leading rows too long for one warp (hub CTAs)
  unsigned long long* d_maxabs = nullptr;  // bits of max |coordinate|
  int64_t *d_order = nullptr, *d_tri_order = nullptr;
  bool host_rows_pending = false;  // hm.order / rank / nbr / fan not yet downloaded (ensure_host_rows)
  int32_t* d_rank = nullptr;       // original id -> slot (ensure_rank; null without a locality order)
  uint32_t* d_tflow = nullptr;     // tile_flow: done[ntiles] + item counter
  bool forma_flow_auto = false;    // AUTO picks tile_flow for Form A (tsg_mesh_upload)
  void* d_alpha = nullptr;
  double* d_xy_stage = nullptr;  // 2*nv original-order doubles
  double* d_batch_in[2] = {nullptr, nullptr};   // tsg_smooth_host_batch staging (lazy)
  double* d_batch_out[2] = {nullptr, nullptr};
  tsg::PassState* h_batch_state = nullptr;      // pinned, per batch item
  tsg::PassState* d_batch_state = nullptr;
  int32_t h_batch_cap = 0;
  double* d_vmin = nullptr;
  int8_t *d_decision = nullptr, *d_decision_orig = nullptr;
  tsg::PassState* d_state = nullptr;
  int32_t* d_acc = nullptr;            // per-pass totals (written by finalize_pass)
  unsigned long long* d_md = nullptr;
  int32_t* d_sacc = nullptr;           // per-pass stat slots (kStatSlots each)
  unsigned long long* d_smd = nullptr;
  unsigned long long* d_rare = nullptr;  // diagnostics: rare-path decisions per pass
  unsigned long long* d_ext = nullptr;  // extrema scratch (3)
  int32_t cap = 0;
  int cur = 0;
  int32_t hub_max_deg = 0;
  int64_t n_hub_fast = 0;  // leading entries of hm.large with deg > kWarpTierCap
  int64_t dist_launches = 0;  // kernels enqueued by tsg_dist_* since tsg_dist_begin
  // Form B schedule cache
  int32_t fb_chunks = 0;
  uint32_t* d_nbr_fresh = nullptr;
  int32_t *d_fb_nodes = nullptr, *d_fb_hubs = nullptr, *d_fb_medium = nullptr;  // level-set schedule
  std::vector<tsg::Phase> fb_levels;
  int32_t *d_cb_order = nullptr, *d_cb_lvl = nullptr, *d_cb_chunk = nullptr;  // chunk schedule
  uint32_t* d_cb_rec = nullptr;
  uint32_t* d_flow_rec = nullptr;   // dataflow schedule (tsg_flow.cuh): records in level order
  uint32_t* d_flow_done = nullptr;  // per slot: passes completed in the running launch
  void* d_flow_save = nullptr;      // round-start coordinates (displacement-stop replay)
  int64_t flow_n = 0;
  int64_t fb_nchunks = 0;
  bool fb_use_chunks = false;  // narrow levels: one CTA per chunk instead of a launch per level
  bool fb_auto_flow = false;   // AUTO picks the dataflow kernel for tsg_smooth (cost model)
  int32_t fb_mode = TSG_FORMB_AUTO;
  int64_t fb_bytes = 0;
  GraphCache gc;
  // Halo exchange plan (multi-GPU partitions): slots sent to / received from peers.
  int32_t* d_send_slots = nullptr;
  int32_t* d_recv_slots = nullptr;
  int64_t n_send = 0, n_recv = 0;
  double* d_halo_stage = nullptr;  // 2 * max(n_send, n_recv) doubles (host-pointer transfers)
  // Peer-memory partitioned driver (tsg_peer.cuh): this rank, the peers' mapped buffers and
  // sync blocks, and the push plan (own slot -> peer, peer slot).
  int32_t peer_rank = 0, peer_world = 0;
  tsg::PeerSync* d_peer_sync = nullptr;
  tsg::PeerEntry* d_peer_tab = nullptr;
  int32_t* d_push_peer = nullptr;
  uint32_t *d_push_src = nullptr, *d_push_dst = nullptr;  // rows of valence > 31 (peer_push)
  int64_t n_push = 0;
  uint32_t *d_fpush_mask = nullptr, *d_fpush_off = nullptr, *d_fpush_peer = nullptr, *d_fpush_dst = nullptr;  // tile rows
  uint32_t peer_tick = 0;  // last tick of the previous peer run (identical on every rank)
  uint32_t h_peer_tick0 = 0;  // host copy of this run's start tick (source of an async copy)
};

#define TSG_LOCK_MESH(m) tsg_abi::CtxLock tsg_ctx_lock_((m) ? (m)->ctx : nullptr)

namespace {

void free_form_b(tsg_mesh* m) {
  cudaFree(m->d_nbr_fresh);
  cudaFree(m->d_fb_nodes);
  cudaFree(m->d_fb_hubs);
  cudaFree(m->d_fb_medium);
  m->d_fb_nodes = m->d_fb_hubs = m->d_fb_medium = nullptr;
  m->fb_levels.clear();
  cudaFree(m->d_cb_order);
  cudaFree(m->d_cb_lvl);
  cudaFree(m->d_cb_chunk);
  cudaFree(m->d_cb_rec);
  cudaFree(m->d_flow_rec);
  cudaFree(m->d_flow_done);
  cudaFree(m->d_flow_save);
  m->d_cb_order = m->d_cb_lvl = m->d_cb_chunk = nullptr;
  m->d_cb_rec = m->d_flow_rec = m->d_flow_done = nullptr;
  m->d_flow_save = nullptr;
  m->flow_n = 0;
  m->d_nbr_fresh = nullptr;
  m->bytes -= m->fb_bytes;
  m->fb_bytes = 0;
  m->fb_chunks = 0;
  m->fb_nchunks = 0;
}

// The device layout leaves order / rank / rows / fan records on the device; host-side builders
// (Form B schedules, halo plans, slot lookups, peer pushes) download them on first use.
tsg_status ensure_host_rows(tsg_mesh* m) {
  if (!m->host_rows_pending) return TSG_OK;
  auto& hm = m->hm;
  const int64_t nv = hm.nv, nrow = hm.off[nv];
  cudaStream_t s = m->ctx->stream;
  hm.order.resize(nv);
  if (m->d_order) {
    TSG_CUDA(cudaMemcpyAsync(hm.order.data(), m->d_order, 8 * nv, cudaMemcpyDeviceToHost, s));
  } else {
    for (int64_t v = 0; v < nv; ++v) hm.order[v] = v;
  }
  hm.nbr.resize(nrow);
  hm.fan.resize(nrow);
  if (nrow) {
    TSG_CUDA(cudaMemcpyAsync(hm.nbr.data(), m->d_nbr, 4 * nrow, cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaMemcpyAsync(hm.fan.data(), m->d_fan, 4 * nrow, cudaMemcpyDeviceToHost, s));
  }
  TSG_CUDA(cudaStreamSynchronize(s));
  hm.rank.resize(nv);
  for (int64_t sl = 0; sl < nv; ++sl) hm.rank[hm.order[sl]] = sl;
  m->host_rows_pending = false;
  return TSG_OK;
}

tsg_status ensure_form_b(tsg_mesh* m, int32_t chunks) {
  if (m->fb_chunks == chunks) return TSG_OK;
  tsg_status st0 = ensure_host_rows(m);
  if (st0) return st0;
  free_form_b(m);
  m->gc.reset();
  tsg::FormBSchedule sch;
  const std::string err = tsg::build_form_b(m->hm, chunks, kTiers, sch);
  if (!err.empty()) return fail(TSG_ERR_INVALID, err);
  int64_t b = 0;
  cudaStream_t s = m->ctx->stream;
  tsg_status st;
  if ((st = upload(&m->d_nbr_fresh, sch.nbr_fresh, &b, s))) return st;
  if ((st = upload(&m->d_fb_nodes, sch.nodes, &b, s))) return st;
  if ((st = upload(&m->d_fb_hubs, sch.hubs, &b, s))) return st;
  if ((st = upload(&m->d_fb_medium, sch.medium, &b, s))) return st;
  if ((st = upload(&m->d_cb_order, sch.cb_order, &b, s))) return st;
  if ((st = upload(&m->d_cb_lvl, sch.lvl_off, &b, s))) return st;
  if ((st = upload(&m->d_cb_chunk, sch.chunk_lvl, &b, s))) return st;
  if ((st = upload(&m->d_cb_rec, sch.cb_rec, &b, s))) return st;
  if ((st = upload(&m->d_flow_rec, sch.flow_rec, &b, s))) return st;
  m->flow_n = static_cast<int64_t>(sch.flow_rec.size() / tsg::kChunkRecWords);
  TSG_CUDA(cudaMalloc(&m->d_flow_done, sizeof(uint32_t) * m->hm.nv));
  TSG_CUDA(cudaMemsetAsync(m->d_flow_done, 0xff, sizeof(uint32_t) * m->hm.nv, s));  // pinned: ~0u
  TSG_CUDA(cudaMalloc(&m->d_flow_save, 2 * m->hm.nv * m->rsize));
  b += static_cast<int64_t>(sizeof(uint32_t) * m->hm.nv + 2 * m->hm.nv * m->rsize);
  TSG_CUDA(cudaStreamSynchronize(s));
  m->fb_nchunks = static_cast<int64_t>(sch.chunk_lvl.size()) - 1;
  {
    // Per-level cost models fitted on B200 (cfg1 W = 1, 8; cfg2 W = 16, 148; cfg3 W = 64, 148):
    //   launch per level:        ~6 us + 8e-5 us x (vertices in the level)
    //   one CTA per chunk:       ~2.4 us + 0.04 us x (vertices of one chunk in the level)
    // e.g. cfg3 W = 148 (1025 levels, 106 per chunk): chunks 7.9 ms vs levels 10.5 ms per pass;
    // cfg3 W = 64 (163 per chunk): levels 12.8 vs chunks 17.0; cfg2 W = 148: levels 0.10 vs 0.28.
    const int64_t movable = static_cast<int64_t>(sch.cb_order.size());
    const int64_t nlev = static_cast<int64_t>(sch.levels.size());
    const double w_total = nlev ? double(movable) / nlev : 0.0;
    const double w_chunk = nlev && m->fb_nchunks ? w_total / double(m->fb_nchunks) : 0.0;
    const bool chunks_faster = nlev > 0 && 2.4 + 0.04 * w_chunk < 6.0 + 8e-5 * w_total;
    m->fb_use_chunks = (m->fb_mode == TSG_FORMB_AUTO || m->fb_mode == TSG_FORMB_FLOW) ? chunks_faster
                                                                                  : m->fb_mode == TSG_FORMB_CHUNKS;
    // Dataflow kernel (tsg_smooth only), fitted on B200: per pass ~ max(0.36 us x levels (the
    // pipelined critical path: cfg1 serial, 195 levels -> 69 us), 0.68 ns x movable vertices
    // (throughput: cfg2 1M, W = 1 / 148 -> 0.72 / 0.64 ms)).  Per-level launches: 6 us x levels +
    // 8e-5 us x movable; per-chunk CTAs as above.
    const double levels_us = 6.0 * nlev + 8e-5 * movable;
    const double chunks_us = nlev * (2.4 + 0.04 * w_chunk);
    const double flow_us = std::max(0.36 * nlev, 6.8e-4 * movable);
    m->fb_auto_flow = nlev > 0 && flow_us < std::min(levels_us, chunks_us);
    if (std::getenv("TSG_DIAG"))
      std::fprintf(stderr, "[tsg] Form B W=%d: %lld levels, %lld chunks, mean level width %.0f (%.1f per chunk) -> %s\n",
                   chunks, static_cast<long long>(nlev), static_cast<long long>(m->fb_nchunks),
                   w_total, w_chunk,
                   m->fb_auto_flow ? "flow" : m->fb_use_chunks ? "chunks" : "levels");
  }
  m->fb_levels = std::move(sch.levels);
  m->fb_bytes = b;
  m->bytes += b;
  m->fb_chunks = chunks;
  return TSG_OK;
}

template <typename R, bool kSoA>
tsg::Coords<R, kSoA> coords_of(const tsg_mesh* m, int i) {
  return tsg::Coords<R, kSoA>{static_cast<R*>(m->buf[i]), m->hm.nv};
}

// Diagnostics (TSG_DIAG=1): per-pass rare-path counts and node-kernel times printed by the
// stream driver to stderr.  Not part of the ABI; used to tune the fast-path guard.
bool diag_enabled() {
  static const bool on = std::getenv("TSG_DIAG") != nullptr;
  return on;
}

// The device inverse of the slot order (write-back gathers), built on first use.
tsg_status ensure_rank(tsg_mesh* m) {
  if (!m->d_order || m->d_rank) return TSG_OK;
  const int64_t nv = m->hm.nv;
  TSG_CUDA(cudaMalloc(&m->d_rank, sizeof(int32_t) * nv));
  rank_of_order<<<grid_for(nv, 256), 256, 0, m->ctx->stream>>>(m->d_order, nv, m->d_rank);
  TSG_LAUNCHED();
  return TSG_OK;
}

// Everything templated on the coordinate type and layout.
template <typename R, bool kSoA>
struct Engine {
  using Args = tsg::PassArgs<R, kSoA>;
  using R2 = typename tsg::Arith<R>::R2;

  static Args base_args(tsg_mesh* m, const tsg_smooth_cfg& c) {
    Args a{};
    a.buf0 = coords_of<R, kSoA>(m, 0);
    a.buf1 = coords_of<R, kSoA>(m, 1);
    a.swap = c.swap;
    a.off = m->d_off;
    a.nbr = c.form == TSG_FORM_B ? m->d_nbr_fresh : m->d_nbr;
    a.fan = m->d_fan;
    a.fan16 = m->d_fan16;
    a.vinc_off = m->d_vinc_off;
    a.vinc = m->d_vinc;
    a.alpha = static_cast<const R*>(m->d_alpha);
    a.st = m->d_state;
    a.slot_acc = m->d_sacc;
    a.slot_md = m->d_smd;
    a.decision = nullptr;
    a.rare = diag_enabled() ? m->d_rare : nullptr;
    a.maxabs = m->d_maxabs;
    return a;
  }

  // Events for fork/join (reused round-robin; a graph capture keeps its own edges, a plain
  // launch sequence only needs each event until the matching wait has been enqueued).
  static tsg_status next_event(tsg_context* ctx, cudaEvent_t* ev) {
    if (ctx->fork_next == ctx->fork_events.size()) {
      cudaEvent_t e;
      TSG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      ctx->fork_events.push_back(e);
    }
    *ev = ctx->fork_events[ctx->fork_next++];
    return TSG_OK;
  }

  template <bool kFormB, bool kTwoPhase>
  static tsg_status launch_phase(tsg_mesh* m, const Args& base, const int32_t* small, int64_t ns,
                                 const int32_t* medium, int64_t nmed,
                                 const int32_t* hubs, int64_t nh, int32_t hub_cap, cudaStream_t s,
                                 int64_t* kernels) {
    tsg_context* ctx = m->ctx;
    const bool fork = ns > 0 && (nmed > 0 || nh > 0);
    cudaStream_t t = s;  // stream of the medium / hub tiers
    if (fork) {
      cudaEvent_t e;
      tsg_status st = next_event(ctx, &e);
      if (st) return st;
      TSG_CUDA(cudaEventRecord(e, s));
      TSG_CUDA(cudaStreamWaitEvent(ctx->side, e, 0));
      t = ctx->side;
    }
    if (nh > 0) {  // longest-latency tier first
      Args a = base;
      a.list = hubs;
      a.count = nh;
      const size_t smem = static_cast<size_t>(hub_cap) * sizeof(R2) * (kFormB ? 2 : 1);
      tsg::hub_update<R, kSoA, kFormB, kTwoPhase><<<static_cast<unsigned>(nh), tsg::kHubBlock, smem, t>>>(a, hub_cap);
      TSG_LAUNCHED();
      ++*kernels;
    }
    if (nmed > 0) {
      constexpr int kMedBlock = 64;
      Args a = base;
      a.list = medium;
      a.count = nmed;
      tsg::node_update<R, kSoA, kFormB, kTwoPhase, kMaxMedDeg, kMedBlock>
          <<<static_cast<unsigned>((nmed + kMedBlock - 1) / kMedBlock), kMedBlock, 0, t>>>(a);
      TSG_LAUNCHED();
      ++*kernels;
    }
    if (ns > 0) {
      Args a = base;
      a.list = small;
      a.count = ns;
      tsg::node_update<R, kSoA, kFormB, kTwoPhase, kMaxSmallDeg, tsg::kNodeBlock>
          <<<static_cast<unsigned>((ns + tsg::kNodeBlock - 1) / tsg::kNodeBlock), tsg::kNodeBlock, 0, s>>>(a);
      TSG_LAUNCHED();
      ++*kernels;
    }
    if (fork) {
      cudaEvent_t e;
      tsg_status st = next_event(ctx, &e);
      if (st) return st;
      TSG_CUDA(cudaEventRecord(e, ctx->side));
      TSG_CUDA(cudaStreamWaitEvent(s, e, 0));
    }
    return TSG_OK;
  }

  // Form A, fused: tile-staged cycle sweep (thread per vertex) over every slot with deg <=
  // kMaxCycleDeg; warp per vertex above, on the side stream.
  // graph: the pass is being captured into the WHILE graph (the persistent side kernel needs the
  // graph's dispatch order, see below; plain stream launches use the per-tier grids).
  static tsg_status launch_form_a_fused(tsg_mesh* m, const Args& base, cudaStream_t s, int64_t* kernels,
                                        bool graph) {
    tsg_context* ctx = m->ctx;
    const int64_t nv = m->hm.nv, nlarge = static_cast<int64_t>(m->hm.large.size());
    const int64_t nhub = m->n_hub_fast, nwarp = nlarge - nhub;
    // The side tiers run on one stream forked (and joined) inside the captured graph, concurrently
    // with the tile grid (measured alternatives: serial tiers -4 %, hub and warp tiers on two
    // streams -1 %).
    cudaStream_t th = s, tw = s;
    if (nlarge > 0) th = tw = ctx->side;
    cudaStream_t forked[1];
    int nf = 0;
    if (nlarge > 0) forked[nf++] = ctx->side;
    for (int i = 0; i < nf; ++i) {
      cudaStream_t t = forked[i];
      cudaEvent_t e;
      tsg_status st = next_event(ctx, &e);
      if (st) return st;
      TSG_CUDA(cudaEventRecord(e, s));
      TSG_CUDA(cudaStreamWaitEvent(t, e, 0));
    }
    {
      Args a = base;
      a.list = nullptr;
      a.count = nv;
      const tsg::TileArgs ta = tile_args(m);
      const unsigned ntiles = static_cast<unsigned>((nv + ta.tile - 1) / ta.tile);
      const size_t smem = tsg::tile_smem_bytes<R>(ta.tile, ta.ext_cap, ta.rec_cap);
      const bool staged = tiles_staged(m);
      with_tile(ta.tile, [&](auto K) {
        if (staged)
          tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, true, K><<<ntiles, kTileThreads, smem, s>>>(a, ta);
        else
          tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, false, K><<<ntiles, kTileThreads, smem, s>>>(a, ta);
      });
      TSG_LAUNCHED();
      ++*kernels;
    }
    // The persistent side kernel is enqueued AFTER the tile grid: in the captured graph the two
    // forked branches are then dispatched side kernel first (measured: all of its CTAs resident
    // at t = 0, the tile grid from 0.1 us, profiles/r01s3c_cfg3_timeline.txt); enqueued before
    // the tile grid, it was dispatched behind it and ran alone after it (0.70 ms per pass).  The
    // stream driver and the partitioned driver's plain launches have no such order (there it ran
    // after the tile grid: 0.69 ms per pass), so there AUTO uses the per-tier grids (a forced
    // TSG_SIDE_PERSIST still applies: tests, profiling).
    const bool persist = nlarge > 0 && (m->side_mode == TSG_SIDE_PERSIST || (graph && side_persistent(m)));
    if (persist) {
      Args a = base;
      a.list = m->d_large + m->n_side_cta;
      a.count = nlarge - m->n_side_cta;
      if (a.count > 0) {
        tsg::side_rows<R, kSoA, kSideWarps, kWarpTierCap, kSideRegs>
            <<<static_cast<unsigned>(m->num_sms), kSideWarps * 32, 0, tw>>>(a, m->d_side_ctr);
        TSG_LAUNCHED();
        ++*kernels;
      }
    }
    const int64_t n_cta = persist ? m->n_side_cta : nhub;  // rows with a CTA each
    // Side tiers launched after the tile kernel (its CTAs are dispatched first: +1 %, measured).
    if (n_cta > 0) {  // the longest rows (a prefix of the degree-descending list): CTA per hub
      Args a = base;
      a.list = m->d_large;
      a.count = n_cta;
      const int32_t cap = hub_fast_cap(m);
      tsg::hub_fast_update<R, kSoA><<<static_cast<unsigned>(n_cta), tsg::kHubFastBlock, cap * sizeof(R2), th>>>(a, cap);
      TSG_LAUNCHED();
      ++*kernels;
    }
    if (!persist && nwarp > 0) {
      Args a = base;
      a.list = m->d_large + nhub;
      a.count = nwarp;
      tsg::warp_update<R, kSoA, kWarpTierWarps, kWarpTierCap>
          <<<static_cast<unsigned>((nwarp + kWarpTierWarps - 1) / kWarpTierWarps), kWarpTierWarps * 32, 0, tw>>>(a);
      TSG_LAUNCHED();
      ++*kernels;
    }
    for (int i = 0; i < nf; ++i) {  // join
      cudaStream_t t = forked[i];
      cudaEvent_t e;
      tsg_status st = next_event(ctx, &e);
      if (st) return st;
      TSG_CUDA(cudaEventRecord(e, t));
      TSG_CUDA(cudaStreamWaitEvent(s, e, 0));
    }
    return TSG_OK;
  }

  template <bool kFormB, bool kTwoPhase>
  static tsg_status enqueue_pass_t(tsg_mesh* m, const tsg_smooth_cfg& c, cudaStream_t s,
                                   double tol_abs, cudaGraphConditionalHandle h, int use_handle,
                                   int8_t* decision, cudaEvent_t ev_begin, cudaEvent_t ev_end,
                                   int64_t* kernels, bool with_finalize = true) {
    const int64_t nv = m->hm.nv;
    m->ctx->fork_next = 0;  // fork/join events are reusable once their waits are enqueued
    if (c.swap == TSG_SWAP_COPY)
      TSG_CUDA(cudaMemcpyAsync(m->buf[1], m->buf[0], 2 * nv * sizeof(R), cudaMemcpyDeviceToDevice, s));
    if (kTwoPhase && !(kFormB && m->fb_use_chunks)) {
      tsg::tri_alpha<R, kSoA><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
          coords_of<R, kSoA>(m, 0), coords_of<R, kSoA>(m, 1), c.swap, m->d_state, m->d_tri,
          m->hm.nt, static_cast<R*>(m->d_alpha));
      TSG_LAUNCHED();
      ++*kernels;
    }
    Args base = base_args(m, c);
    base.decision = decision;
    const int32_t hub_cap = std::max(1, std::min(m->hub_max_deg, kHubCap));
    if (ev_begin) TSG_CUDA(cudaEventRecord(ev_begin, s));
    if (!kFormB && !kTwoPhase) {
      tsg_status st = launch_form_a_fused(m, base, s, kernels, use_handle != 0);
      if (st) return st;
    } else if (!kFormB) {
      tsg_status st = launch_phase<false, kTwoPhase>(m, base, nullptr, nv, m->d_medium,
                                                     static_cast<int64_t>(m->hm.medium.size()), m->d_hubs,
                                                     static_cast<int64_t>(m->hm.hubs.size()),
                                                     hub_cap, s, kernels);
      if (st) return st;
    } else if (m->fb_use_chunks) {
      // Form B, both strategies (equal thresholds): one CTA per chunk.
      tsg::formb_chunk_update<R, kSoA><<<static_cast<unsigned>(m->fb_nchunks), 256, kChunkRecSmem, s>>>(
          base, m->d_cb_order, m->d_cb_lvl, m->d_cb_chunk, m->d_cb_rec);
      TSG_LAUNCHED();
      ++*kernels;
    } else {
      for (const tsg::Phase& L : m->fb_levels) {
        tsg_status st = launch_phase<true, kTwoPhase>(m, base, m->d_fb_nodes + L.small_begin,
                                                      L.small_count, m->d_fb_medium + L.medium_begin,
                                                      L.medium_count, m->d_fb_hubs + L.hub_begin,
                                                      L.hub_count, hub_cap, s, kernels);
        if (st) return st;
      }
    }
    if (ev_end) TSG_CUDA(cudaEventRecord(ev_end, s));
    if (!with_finalize) return TSG_OK;  // partitioned driver: the stop rule runs on global totals
    tsg::finalize_pass<<<1, 32, 0, s>>>(m->d_state, m->d_sacc, m->d_smd, m->d_acc, m->d_md, tol_abs,
                                        c.max_iters, h, use_handle);
    TSG_LAUNCHED();
    ++*kernels;
    return TSG_OK;
  }

  static bool side_persistent(const tsg_mesh* m) {
    return m->side_mode == TSG_SIDE_PERSIST || (m->side_mode == TSG_SIDE_AUTO && m->side_persist_auto);
  }

  static int32_t hub_fast_cap(const tsg_mesh* m) {
    return std::max(1, std::min(m->hm.max_deg, kHubCap));
  }

  static bool tiles_staged(const tsg_mesh* m) {
    return m->hm.max_ext <= kTileExtCap && m->hm.max_rec_words <= kTileRecCap;
  }

  static tsg::TileArgs tile_args(const tsg_mesh* m) {
    tsg::TileArgs t{};
    t.meta = m->d_tmeta;
    t.rec = m->d_trec;
    t.tile_rec = m->d_tile_rec;
    t.ext_off = m->d_ext_off;
    t.ext = m->d_tile_ext;
    // Even, so that the words after the staged coordinates stay 16-byte aligned for fp32 pairs
    // (bulk copies and uint4 stores).
    t.ext_cap = (std::min(m->hm.max_ext, kTileExtCap) + 1) & ~1;
    t.rec_cap = std::min(m->hm.max_rec_words, kTileRecCap);
    t.small_max = kMaxSmallDeg;
    t.medium_max = kMaxMedDeg;
    t.tile = m->hm.tile;
    t.nv = m->hm.nv;
    if (m->peer_world > 1 && m->d_fpush_mask)
      t.push = tsg::TilePush{m->d_fpush_mask, m->d_fpush_off, m->d_fpush_peer, m->d_fpush_dst, m->d_peer_tab};
    return t;
  }

  // Tile CTAs resident per SM (registers and the mesh's shared memory).
  static tsg_status tile_blocks_per_sm(tsg_mesh* m, int* out) {
    const tsg::TileArgs ta = tile_args(m);
    const size_t smem = tsg::tile_smem_bytes<R>(ta.tile, ta.ext_cap, ta.rec_cap);
    const bool staged = tiles_staged(m);
    cudaError_t e = cudaSuccess;
    with_tile(ta.tile, [&](auto K) {
      if (staged)
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            out, tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, true, K>, kTileThreads, smem);
      else
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            out, tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, false, K>, kTileThreads, smem);
    });
    TSG_CUDA(e);
    return TSG_OK;
  }

  // Opt-in shared memory for the hub kernels (done outside any stream capture).
  static tsg_status prepare(tsg_mesh* m) {
    TSG_CUDA(raise_smem_limit(tsg::formb_chunk_update<R, kSoA>, kChunkRecSmem));
    TSG_CUDA(raise_smem_limit(tsg::hub_fast_update<R, kSoA>, static_cast<int>(hub_fast_cap(m) * sizeof(R2))));
    {
      const tsg::TileArgs ta = tile_args(m);
      const int smem = static_cast<int>(tsg::tile_smem_bytes<R>(ta.tile, ta.ext_cap, ta.rec_cap));
      if (std::getenv("TSG_DIAG"))
        std::fprintf(stderr, "[tsg] tile %d slots, smem %d B (ext_cap %d, rec_cap %d words), large rows %zu (hub CTAs %lld)\n",
                     ta.tile, smem, ta.ext_cap, ta.rec_cap, m->hm.large.size(), static_cast<long long>(m->n_hub_fast));
      cudaError_t e = cudaSuccess;
      with_tile(ta.tile, [&](auto K) {
        e = raise_smem_limit(tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, true, K>, smem);
        if (e == cudaSuccess) e = raise_smem_limit(tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, false, K>, smem);
      });
      TSG_CUDA(e);
    }
    // Kernels that run concurrently on one SM must agree on its L1 / shared-memory split: the
    // tile and side-tier kernels all ask for the maximum shared-memory carveout, so that a
    // side-tier CTA does not pin an SM to a smaller split that excludes the tile kernel's CTAs.
    {
      const int kMax = cudaSharedmemCarveoutMaxShared;
      cudaError_t e = cudaSuccess;
      with_tile(m->hm.tile, [&](auto K) {
        e = cudaFuncSetAttribute(tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, true, K>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, kMax);
        if (e == cudaSuccess)
          e = cudaFuncSetAttribute(tsg::tile_update<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, false, K>,
                                   cudaFuncAttributePreferredSharedMemoryCarveout, kMax);
      });
      TSG_CUDA(e);
      TSG_CUDA(cudaFuncSetAttribute(tsg::hub_fast_update<R, kSoA>, cudaFuncAttributePreferredSharedMemoryCarveout, kMax));
      TSG_CUDA(cudaFuncSetAttribute(tsg::warp_update<R, kSoA, kWarpTierWarps, kWarpTierCap>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, kMax));
      TSG_CUDA(cudaFuncSetAttribute(tsg::side_rows<R, kSoA, kSideWarps, kWarpTierCap, kSideRegs>,
                                    cudaFuncAttributePreferredSharedMemoryCarveout, kMax));
    }
    const int32_t hub_cap = std::max(1, std::min(m->hub_max_deg, kHubCap));
    const int smem1 = static_cast<int>(hub_cap * sizeof(R2)), smem2 = 2 * smem1;
    TSG_CUDA(raise_smem_limit(tsg::hub_update<R, kSoA, false, false>, smem1));
    TSG_CUDA(raise_smem_limit(tsg::hub_update<R, kSoA, false, true>, smem1));
    TSG_CUDA(raise_smem_limit(tsg::hub_update<R, kSoA, true, false>, smem2));
    TSG_CUDA(raise_smem_limit(tsg::hub_update<R, kSoA, true, true>, smem2));
    return TSG_OK;
  }

  static tsg_status enqueue_pass(tsg_mesh* m, const tsg_smooth_cfg& c, cudaStream_t s, double tol_abs,
                                 cudaGraphConditionalHandle h, int use_handle, int8_t* decision,
                                 cudaEvent_t e0, cudaEvent_t e1, int64_t* kernels, bool fin = true) {
    // UpdateStrategy changes the reference's schedule, never its results: TwoPhase reads the
    // threshold from the α field refreshed at the end of the previous pass
    // (proj/src/smoothing.cpp:119-120), Fused recomputes the same minimum from the pass-start
    // coordinates (proj/tests/acceptance.cpp:146-193 checks Fused == TwoPhase
    // bitwise).  Both run the fused kernels here: the per-pass α sweep and its 8-byte-per-
    // triangle field are not needed, and the final field is computed once for write-back
    // (tsg_tri_alpha).  TSG_TWOPHASE_SWEEP=1 keeps the literal two-phase schedule (tests).
    static const bool literal = std::getenv("TSG_TWOPHASE_SWEEP") != nullptr;
    const bool fb = c.form == TSG_FORM_B, tp = literal && c.strategy == TSG_STRATEGY_TWOPHASE;
    if (fb && tp) return enqueue_pass_t<true, true>(m, c, s, tol_abs, h, use_handle, decision, e0, e1, kernels, fin);
    if (fb) return enqueue_pass_t<true, false>(m, c, s, tol_abs, h, use_handle, decision, e0, e1, kernels, fin);
    if (tp) return enqueue_pass_t<false, true>(m, c, s, tol_abs, h, use_handle, decision, e0, e1, kernels, fin);
    return enqueue_pass_t<false, false>(m, c, s, tol_abs, h, use_handle, decision, e0, e1, kernels, fin);
  }

  static tsg_status set_coords(tsg_mesh* m, const double* xy_host) {
    cudaStream_t s = m->ctx->stream;
    const int64_t nv = m->hm.nv;
    TSG_CUDA(cudaMemcpyAsync(m->d_xy_stage, xy_host, 2 * nv * sizeof(double), cudaMemcpyHostToDevice, s));
    TSG_CUDA(cudaMemsetAsync(m->d_maxabs, 0, sizeof(unsigned long long), s));
    coords_from_orig<R, kSoA><<<grid_for(nv, 256), 256, 0, s>>>(m->d_xy_stage, m->d_order, nv,
                                                                coords_of<R, kSoA>(m, 0),
                                                                coords_of<R, kSoA>(m, 1), m->d_maxabs);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(m->init, m->buf[0], 2 * nv * sizeof(R), cudaMemcpyDeviceToDevice, s));
    m->cur = 0;
    return TSG_OK;
  }

  static tsg_status get_coords(tsg_mesh* m, double* xy_host) {
    cudaStream_t s = m->ctx->stream;
    const int64_t nv = m->hm.nv;
    if (tsg_status st = ensure_rank(m)) return st;
    coords_to_orig<R, kSoA><<<grid_for(nv, 256), 256, 0, s>>>(coords_of<R, kSoA>(m, m->cur), m->d_rank,
                                                              nv, m->d_xy_stage);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(xy_host, m->d_xy_stage, 2 * nv * sizeof(double), cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    return TSG_OK;
  }

  // Current coordinates into buf0 (both buffers equal afterwards for pinned vertices anyway).
  // Batch: staged original-order input -> both buffers (on the context stream).
  static tsg_status batch_load(tsg_mesh* m, const double* stage) {
    cudaStream_t s = m->ctx->stream;
    const int64_t nv = m->hm.nv;
    zero_u64<<<1, 1, 0, s>>>(m->d_maxabs);  // (a kernel: see smooth_enqueue_graph)
    coords_from_orig<R, kSoA><<<grid_for(nv, 256), 256, 0, s>>>(stage, m->d_order, nv, coords_of<R, kSoA>(m, 0),
                                                                coords_of<R, kSoA>(m, 1), m->d_maxabs);
    TSG_LAUNCHED();
    m->cur = 0;
    return TSG_OK;
  }
  static tsg_status batch_store(tsg_mesh* m, int32_t swap, double* stage) {
    cudaStream_t s = m->ctx->stream;
    const int64_t nv = m->hm.nv;
    if (tsg_status st = ensure_rank(m)) return st;
    coords_to_orig_parity<R, kSoA><<<grid_for(nv, 256), 256, 0, s>>>(coords_of<R, kSoA>(m, 0), coords_of<R, kSoA>(m, 1),
                                                                     swap, m->d_state, m->d_rank, nv, stage);
    TSG_LAUNCHED();
    return TSG_OK;
  }

  static tsg_status normalize(tsg_mesh* m) {
    if (m->cur != 0) {
      TSG_CUDA(cudaMemcpyAsync(m->buf[0], m->buf[1], 2 * m->hm.nv * sizeof(R), cudaMemcpyDeviceToDevice,
                               m->ctx->stream));
      m->cur = 0;
    }
    return TSG_OK;
  }

  // One launch of the Form B dataflow kernel over passes [p0, p0 + np) (tsg_flow.cuh).
  // Cooperative launch: every CTA is co-resident (the kernel's progress argument needs it).
  static tsg_status flow_launch(tsg_mesh* m, int32_t p0, int32_t np, int64_t* kernels) {
    cudaStream_t s = m->ctx->stream;
    const int64_t n = m->flow_n;
    if (n == 0 || np <= 0) return TSG_OK;
    tsg::flow_reset<<<grid_for(n, 256), 256, 0, s>>>(m->d_flow_rec, n, m->d_flow_done);
    TSG_LAUNCHED();
    int per_sm = 0, sms = 0;
    constexpr size_t smem = tsg::flow_smem_bytes<R>();
    TSG_CUDA(raise_smem_limit(tsg::formb_flow<R, kSoA>, static_cast<int>(smem)));
    TSG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tsg::formb_flow<R, kSoA>, tsg::kFlowBlock, smem));
    TSG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, m->ctx->device));
    const int64_t cap = static_cast<int64_t>(std::max(per_sm, 1)) * sms;
    const int64_t want = (n + tsg::kFlowBlock - 1) / tsg::kFlowBlock;
    const unsigned grid = static_cast<unsigned>(std::min(cap, want));
    tsg::FlowArgs<R> f{};
    f.buf0 = static_cast<R*>(m->buf[0]);
    f.buf1 = static_cast<R*>(m->buf[1]);
    f.nv = m->hm.nv;
    f.rec = m->d_flow_rec;
    f.off = m->d_off;
    f.nbr = m->d_nbr_fresh;
    f.fan = m->d_fan;
    f.done = m->d_flow_done;
    f.n = n;
    f.p0 = p0;
    f.np = np;
    f.slot_acc = m->d_sacc;
    f.slot_md = m->d_smd;
    f.maxabs = m->d_maxabs;
    void* args[] = {&f};
    TSG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(tsg::formb_flow<R, kSoA>), dim3(grid),
                                         dim3(tsg::kFlowBlock), args, smem, s));
    *kernels += 2;
    return TSG_OK;
  }

  // One launch of the Form A (tile, pass) dataflow kernel over passes [p0, p0 + np)
  // (tile_flow, tsg_kernels.cuh).  Cooperative launch: the kernel's progress argument needs
  // every CTA co-resident.
  static tsg_status tile_flow_launch(tsg_mesh* m, const tsg_smooth_cfg& c, int32_t p0, int32_t np,
                                     int64_t* kernels) {
    cudaStream_t s = m->ctx->stream;
    const int64_t ntiles = (m->hm.nv + m->hm.tile - 1) / m->hm.tile;
    if (np <= 0 || ntiles == 0) return TSG_OK;
    if (!m->d_tflow) TSG_CUDA(cudaMalloc(&m->d_tflow, sizeof(uint32_t) * (ntiles + 1)));
    TSG_CUDA(cudaMemsetAsync(m->d_tflow, 0, sizeof(uint32_t) * (ntiles + 1), s));
    Args a = base_args(m, c);
    a.swap = TSG_SWAP_PINGPONG;  // the driver normalises copy mode afterwards (bit-identical)
    a.list = nullptr;
    a.count = m->hm.nv;
    tsg::TileArgs ta = tile_args(m);
    ta.flow = tsg::TileFlow{m->d_tflow, m->d_tflow + ntiles, p0, np, ntiles};
    const size_t smem = tsg::tile_smem_bytes<R>(ta.tile, ta.ext_cap, ta.rec_cap);
    cudaError_t e = cudaSuccess;
    with_tile(ta.tile, [&](auto K) {
      auto* fn = tsg::tile_flow<R, kSoA, kTileThreads, tsg::kMaxCycleDeg, K>;
      int per_sm = 0;
      if ((e = raise_smem_limit(fn, static_cast<int>(smem))) != cudaSuccess) return;
      if ((e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout,
                                    cudaSharedmemCarveoutMaxShared)) != cudaSuccess)
        return;
      if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kTileThreads, smem)) != cudaSuccess) return;
      const int64_t cap = static_cast<int64_t>(std::max(per_sm, 1)) * std::max(m->num_sms, 1);
      const unsigned grid = static_cast<unsigned>(std::min(cap, ntiles * np));
      void* args[] = {&a, &ta};
      e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fn), dim3(grid), dim3(kTileThreads), args, smem, s);
    });
    TSG_CUDA(e);
    ++*kernels;
    return TSG_OK;
  }

  static tsg_status peer_push(tsg_mesh* m, cudaStream_t s, int64_t* kernels) {
    if (m->n_push == 0) return TSG_OK;
    tsg::peer_push<R, kSoA><<<grid_for(m->n_push, 256), 256, 0, s>>>(
        m->d_state, coords_of<R, kSoA>(m, 0), coords_of<R, kSoA>(m, 1), m->d_push_peer, m->d_push_src,
        m->d_push_dst, m->n_push, m->d_peer_tab);
    TSG_LAUNCHED();
    ++*kernels;
    return TSG_OK;
  }

  static tsg_status refresh_alpha(tsg_mesh* m) {
    cudaStream_t s = m->ctx->stream;
    tsg::tri_alpha<R, kSoA><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
        coords_of<R, kSoA>(m, m->cur), coords_of<R, kSoA>(m, m->cur), 0, nullptr, m->d_tri, m->hm.nt,
        static_cast<R*>(m->d_alpha));
    TSG_LAUNCHED();
    return TSG_OK;
  }
};

template <class F>
tsg_status dispatch(const tsg_mesh* m, F&& f) {
  if (m->prec == TSG_F64) {
    if (m->layout == TSG_LAYOUT_SOA) return f(Engine<double, true>{});
    return f(Engine<double, false>{});
  }
  if (m->layout == TSG_LAYOUT_SOA) return f(Engine<float, true>{});
  return f(Engine<float, false>{});
}

tsg_status validate_cfg(const tsg_smooth_cfg* c) {
  if (!c) return fail(TSG_ERR_INVALID, "null config");
  if (c->form != TSG_FORM_A && c->form != TSG_FORM_B) return fail(TSG_ERR_INVALID, "form must be A or B");
  if (c->strategy != TSG_STRATEGY_FUSED && c->strategy != TSG_STRATEGY_TWOPHASE)
    return fail(TSG_ERR_INVALID, "strategy must be fused or twophase");
  if (c->swap != TSG_SWAP_PINGPONG && c->swap != TSG_SWAP_COPY)
    return fail(TSG_ERR_INVALID, "swap must be pingpong or copy");
  if (c->chunks < 1) return fail(TSG_ERR_INVALID, "workers must be >= 1");
  if (c->max_iters < 1) return fail(TSG_ERR_INVALID, "max_iters must be >= 1");
  if (!(c->move_tol >= 0.0)) return fail(TSG_ERR_INVALID, "move_tol must be >= 0");
  if (c->driver < TSG_DRIVER_GRAPH || c->driver > TSG_DRIVER_STREAM)
    return fail(TSG_ERR_INVALID, "driver must be graph or stream");
  return TSG_OK;
}

tsg_status ensure_stats_capacity(tsg_mesh* m, int32_t n) {
  if (m->cap >= n) return TSG_OK;
  cudaFree(m->d_acc);
  cudaFree(m->d_md);
  cudaFree(m->d_sacc);
  cudaFree(m->d_smd);
  m->d_acc = nullptr;
  m->d_md = nullptr;
  m->d_sacc = nullptr;
  m->d_smd = nullptr;
  TSG_CUDA(cudaMalloc(&m->d_acc, sizeof(int32_t) * n));
  TSG_CUDA(cudaMalloc(&m->d_md, sizeof(unsigned long long) * n));
  TSG_CUDA(cudaMalloc(&m->d_sacc, sizeof(int32_t) * n * tsg::kStatSlots));
  TSG_CUDA(cudaMalloc(&m->d_smd, sizeof(unsigned long long) * n * tsg::kStatSlots));
  cudaFree(m->d_rare);
  m->d_rare = nullptr;
  TSG_CUDA(cudaMalloc(&m->d_rare, sizeof(unsigned long long) * (n + 16)));
  m->cap = n;
  m->gc.reset();  // graph captured old pointers
  return TSG_OK;
}

}  // namespace

// ----------------------------------------------------------------------------- C ABI

extern "C" {

int32_t tsg_abi_version(void) { return TSG_ABI_VERSION; }

const char* tsg_last_error(void) { return g_err.c_str(); }

int32_t tsg_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
  return n;
}

tsg_status tsg_context_create(int32_t device, tsg_context** out) {
  if (!out) return fail(TSG_ERR_INVALID, "null out");
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0)
    return fail(TSG_ERR_NODEVICE, std::string("no CUDA device: ") + cudaGetErrorString(e));
  if (device < 0 || device >= n) return fail(TSG_ERR_INVALID, "device index out of range");
  TSG_CUDA(cudaSetDevice(device));
  auto ctx = std::make_unique<tsg_context>();
  ctx->device = device;
  TSG_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
  TSG_CUDA(cudaEventCreate(&ctx->ev0));
  TSG_CUDA(cudaEventCreate(&ctx->ev1));
  TSG_CUDA(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
  TSG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking));
  TSG_CUDA(cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking));
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t* e : {&ctx->ev_in_ready[b], &ctx->ev_in_free[b], &ctx->ev_out_ready[b], &ctx->ev_out_free[b]})
      TSG_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  // Mesh prep allocates its temporaries from the device's default pool (cudaMallocAsync); with
  // the default release threshold (0) every synchronisation unmaps them and the next phase maps
  // them again — measured: cfg3 device layout 0.4..1.7 s run to run.  Keep them in the pool.
  {
    cudaMemPool_t pool;
    TSG_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    TSG_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  }
  *out = ctx.release();
  return TSG_OK;
}

tsg_status tsg_context_destroy(tsg_context* ctx) {
  if (!ctx) return TSG_OK;
  cudaSetDevice(ctx->device);
  for (cudaEvent_t e : ctx->pass_events) cudaEventDestroy(e);
  cudaEventDestroy(ctx->ev0);
  cudaEventDestroy(ctx->ev1);
  for (cudaEvent_t e : ctx->fork_events) cudaEventDestroy(e);
  cudaStreamDestroy(ctx->side);
  cudaStreamDestroy(ctx->copy_in);
  cudaStreamDestroy(ctx->copy_out);
  for (int b = 0; b < 2; ++b)
    for (cudaEvent_t e : {ctx->ev_in_ready[b], ctx->ev_in_free[b], ctx->ev_out_ready[b], ctx->ev_out_free[b]})
      cudaEventDestroy(e);
  cudaStreamDestroy(ctx->stream);
  delete ctx;
  return TSG_OK;
}

void* tsg_context_stream(tsg_context* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

tsg_status tsg_hilbert_order(int64_t nv, const double* xy, int64_t* order_out) {
  if (nv < 0 || (nv > 0 && (!xy || !order_out))) return fail(TSG_ERR_INVALID, "bad arguments");
  tsg::hilbert_order(nv, xy, order_out);
  return TSG_OK;
}

tsg_status tsg_selftest_alpha(tsg_context* ctx, int64_t n, uint64_t seed, int32_t newton_steps,
                              double* max_abs_err_out, int64_t* nonfinite_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || n < 0) return fail(TSG_ERR_INVALID, "bad arguments");
  TSG_CUDA(cudaSetDevice(ctx->device));
  unsigned long long* d = nullptr;
  TSG_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
  TSG_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ctx->stream));
  selftest_alpha<<<grid_for(n, 256), 256, 0, ctx->stream>>>(n, seed, newton_steps, d, d + 1);
  TSG_LAUNCHED();
  unsigned long long h[2];
  TSG_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d);
  if (max_abs_err_out) std::memcpy(max_abs_err_out, &h[0], sizeof(double));
  if (nonfinite_out) *nonfinite_out = static_cast<int64_t>(h[1]);
  return TSG_OK;
}

tsg_status tsg_selftest_alpha_cycle(tsg_context* ctx, int64_t n, uint64_t seed, double* max_abs_err_out,
                                    int64_t* nonfinite_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || n < 0) return fail(TSG_ERR_INVALID, "bad arguments");
  TSG_CUDA(cudaSetDevice(ctx->device));
  unsigned long long* d = nullptr;
  TSG_CUDA(cudaMalloc(&d, 2 * sizeof(unsigned long long)));
  TSG_CUDA(cudaMemsetAsync(d, 0, 2 * sizeof(unsigned long long), ctx->stream));
  selftest_alpha_cycle<<<grid_for(n, 256), 256, 0, ctx->stream>>>(n, seed, d, d + 1);
  TSG_LAUNCHED();
  unsigned long long h[2];
  TSG_CUDA(cudaMemcpyAsync(h, d, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(ctx->stream));
  cudaFree(d);
  if (max_abs_err_out) std::memcpy(max_abs_err_out, &h[0], sizeof(double));
  if (nonfinite_out) *nonfinite_out = static_cast<int64_t>(h[1]);
  return TSG_OK;
}

namespace {

// TSG_PREP_TIMING=1: wall times of the upload phases on stderr (stream synchronised per mark).
struct UploadTimer {
  cudaStream_t s;
  bool on = std::getenv("TSG_PREP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tsg upload] %-24s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Shared memory of one tile CTA: dynamic (tile_smem_bytes) + ~3 KB static + 1 KB reserved.
size_t tile_smem_estimate(const tsg::HostMesh& hm, int rsize) {
  return 2 * static_cast<size_t>(rsize) * (hm.tile + ((std::min(hm.max_ext, kTileExtCap) + 1) & ~1)) +
         4 * static_cast<size_t>(std::min(hm.max_rec_words, kTileRecCap)) + 4 * static_cast<size_t>(hm.tile) + 4096;
}

// kTileMinBlocks tile CTAs still fit one SM's 228 KB.
bool tile_fits(const tsg::HostMesh& hm, int rsize) {
  return tsg::kTileMinBlocks * tile_smem_estimate(hm, rsize) <= 228 * 1024;
}

// Slots per tile (a compiled size, kTileSizes).  Larger tiles stage fewer external
// coordinates per vertex (halo ~ perimeter / area); smaller tiles balance the last waves of the
// grid better.  Measured on one B200, 3 CTAs per SM (profiles/r02/tile_sizes.txt):
//   cfg3 16M f64  768 31.9 / 1024 34.0 / 1280 35.5 G/s;  cfg4 64M f64 1024 38.8 / 1280 40.4;
//   cfg3 f32 1024 41.7 / 1280 43.9;  cfg2 1M f64 768 22.5 / 1024 22.0 / 1280 21.1;
//   cfg2 1M f32 768 31.6 / 1024 32.3 / 1280 29.6.
// So: 1280 once the grid runs >= 8 waves of 1280-slot tiles; below that 1024 for fp32 meshes
// of at least one wave and 768 otherwise.  TSG_TILE forces a size (tests, measurements); upload
// falls back to kTile when a larger tile exceeds a layout or shared-memory limit.
// Meshes small enough that the per-pass launch's wave tail and launch cost are a large share of
// a pass: at most kFlowWaves waves of 1280-slot tiles.  Measured, random Delaunay fp64
// (profiles/r02/flow_sizes.txt; per-pass graph at its own tile size vs the dataflow launch):
// 1M 22.7 -> 30.4, 2M 26.0 -> 32.4, 4M 29.1 -> 33.9, 8M 34.6 -> 34.8 G node-upd/s; cfg4 64M
// 40.3 -> 35.6 (a tile can wait on a neighbour tile far away in the item order, and the
// per-pass graph's tail is already < 1 %).
constexpr double kFlowWaves = 12.0;
bool flow_sized(int64_t nv, int num_sms) {
  return static_cast<double>(nv) <= kFlowWaves * std::max(1, num_sms) * tsg::kTileMinBlocks * 1280.0;
}
// The dataflow launch's tile: 1280 slots once the mesh fills a wave of them, else 768 (more,
// shorter items for meshes that do not fill the GPU).
int32_t flow_tile(int64_t nv, int num_sms) {
  return static_cast<double>(nv) >= static_cast<double>(std::max(1, num_sms)) * tsg::kTileMinBlocks * 1280.0 ? 1280
                                                                                                             : 768;
}

int32_t choose_tile(int64_t nv, int num_sms, int rsize) {
  if (const char* e = std::getenv("TSG_TILE")) return tile_supported(std::atoi(e)) ? std::atoi(e) : -1;
  const double slots = static_cast<double>(std::max(1, num_sms)) * tsg::kTileMinBlocks;
  const double nvd = static_cast<double>(nv);
  if (nvd >= 8.0 * slots * 1280) return 1280;
  if (rsize == 4 && nvd >= slots * 1024) return 1024;
  return 768;
}

}  // namespace

tsg_status tsg_mesh_upload(tsg_context* ctx, const tsg_mesh_desc* d, tsg_mesh** out) {
  TSG_LOCK_CTX(ctx);
  return tsg_internal::mesh_upload_impl(ctx, d, nullptr, out);
}

}  // extern "C"

// din: the topology already on the device (tsg_mesh_upload_triangles, tsg_topo.cu); the desc's
// CSR arrays are then not read.
tsg_status tsg_internal::mesh_upload_impl(tsg_context* ctx, const tsg_mesh_desc* d, const tsg::DeviceInputs* din,
                                          tsg_mesh** out) {
  if (!ctx || !d || !out) return fail(TSG_ERR_INVALID, "null argument");
  if (!d->xy || !d->tri || (!din && (!d->nbr_off || !d->nbr || !d->inc_off || !d->inc || !d->boundary)))
    return fail(TSG_ERR_INVALID, "mesh description has null arrays");
  if (d->layout != TSG_LAYOUT_AOS && d->layout != TSG_LAYOUT_SOA)
    return fail(TSG_ERR_INVALID, "layout must be aos or soa");
  if (d->precision != TSG_F64 && d->precision != TSG_F32)
    return fail(TSG_ERR_INVALID, "precision must be f64 or f32");
  TSG_CUDA(cudaSetDevice(ctx->device));
  auto m = std::make_unique<tsg_mesh>();
  m->ctx = ctx;
  m->layout = d->layout;
  m->prec = d->precision;
  m->rsize = d->precision == TSG_F64 ? 8 : 4;
  cudaStream_t s = ctx->stream;
  int64_t* b = &m->bytes;
  tsg_status st;
  UploadTimer ut{s};
  TSG_CUDA(cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int32_t tile_graph = choose_tile(d->nv, m->num_sms, m->rsize);
  if (tile_graph < 0) return fail(TSG_ERR_INVALID, "TSG_TILE must be one of 768, 1024, 1280");
  // Small meshes smooth Form A through the (tile, pass) dataflow launch when every movable row
  // fits the tile kernel; that launch has no wave tail and prefers 1280-slot tiles.  The tile
  // size is chosen before the tiers are known: a mesh that turns out to have side rows is
  // rebuilt at the per-pass graph's size.
  const bool tile_forced = std::getenv("TSG_TILE") != nullptr;
  const bool flow_size = flow_sized(d->nv, m->num_sms);
  int32_t tile = tile_graph;
  if (!tile_forced && flow_size) tile = flow_tile(d->nv, m->num_sms);
  auto staged = [&] { return m->hm.max_ext <= kTileExtCap && m->hm.max_rec_words <= kTileRecCap; };
  // Device layout: built on the GPU (tsg_layout_dev.cu, default) or on the host
  // (build_host_mesh, TSG_HOST_PREP=1); identical arrays either way.
  static const bool host_prep = std::getenv("TSG_HOST_PREP") != nullptr;
  if (host_prep && din) return fail(TSG_ERR_INVALID, "TSG_HOST_PREP=1 needs the host topology (tsg_mesh_upload)");
  if (!host_prep) {
    std::string err = tsg::validate_desc(*d, din == nullptr);
    if (!err.empty()) return fail(TSG_ERR_INVALID, err);
    ut.mark("validate");
    tsg::DeviceLayout L;
    auto build = [&](int32_t t) {
      tsg::free_layout(L);
      tile = t;
      err = tsg::build_device_layout(s, *d, kTiers, m->hm, L, t, false, din);
    };
    auto cuda_err = [&] { return err.rfind("CUDA: ", 0) == 0; };
    build(tile);
    if (!tile_forced && tile != tile_graph && !cuda_err() && (!err.empty() || !m->hm.large.empty() || !staged()))
      build(tile_graph);
    // Larger tiles can overflow the 15-bit word offsets (rows of high valence) or the shared
    // memory of kTileMinBlocks CTAs: fall back to kTile, whose limits every mesh meets.
    if (tile != tsg::kTile && !cuda_err() && (!err.empty() || !tile_fits(m->hm, m->rsize))) build(tsg::kTile);
    if (!err.empty()) {
      tsg::free_layout(L);
      return fail(err.rfind("CUDA: ", 0) == 0 ? TSG_ERR_CUDA : TSG_ERR_INVALID, err);
    }
    const auto& h = m->hm;
    const int64_t ntiles = (h.nv + h.tile - 1) / h.tile;
    m->d_off = L.off;
    m->d_nbr = L.nbr;
    m->d_fan = L.fan;
    m->d_fan16 = L.fan16;
    m->d_tmeta = L.tmeta;
    m->d_tile_rec = L.tile_rec;
    m->d_ext_off = L.ext_off;
    m->d_tile_ext = L.ext;
    m->d_trec = L.trec;
    m->d_vinc_off = L.vinc_off;
    m->d_vinc = L.vinc;
    m->d_tri = L.tri;
    m->d_order = L.order;
    m->d_tri_order = L.tri_order;
    m->host_rows_pending = true;
    const int64_t nrow = static_cast<int64_t>(h.off[h.nv]);
    *b += 4 * (h.nv + 1) + 10 * nrow + 4 * h.nv + 8 * (ntiles + 1) + 12 * h.nt + 4 * (h.nv + 1) + 12 * h.nt +
          (L.order ? 8 * (h.nv + h.nt) : 0);
    if ((st = upload(&m->d_hubs, h.hubs, b, s))) return st;
    if ((st = upload(&m->d_medium, h.medium, b, s))) return st;
    if ((st = upload(&m->d_large, h.large, b, s))) return st;
  } else {
    std::string err = tsg::build_host_mesh(*d, kTiers, m->hm, tile);
    if (!tile_forced && tile != tile_graph && (!err.empty() || !m->hm.large.empty() || !staged()))
      err = tsg::build_host_mesh(*d, kTiers, m->hm, tile = tile_graph);
    if (tile != tsg::kTile && (!err.empty() || !tile_fits(m->hm, m->rsize)))
      err = tsg::build_host_mesh(*d, kTiers, m->hm, tile = tsg::kTile);
    if (!err.empty()) return fail(TSG_ERR_INVALID, err);
    const auto& h = m->hm;
    if ((st = upload(&m->d_off, h.off, b, s))) return st;
    if ((st = upload(&m->d_nbr, h.nbr, b, s))) return st;
    if ((st = upload(&m->d_fan, h.fan, b, s))) return st;
    if ((st = upload(&m->d_fan16, h.fan16, b, s))) return st;
    if ((st = upload(&m->d_tmeta, h.tmeta, b, s))) return st;
    if ((st = upload(&m->d_tile_rec, h.tile_rec, b, s))) return st;
    if ((st = upload(&m->d_ext_off, h.ext_off, b, s))) return st;
    if ((st = upload(&m->d_tile_ext, h.ext, b, s))) return st;
    if ((st = upload(&m->d_trec, h.trec, b, s))) return st;
    if ((st = upload(&m->d_vinc_off, h.vinc_off, b, s))) return st;
    if ((st = upload(&m->d_vinc, h.vinc, b, s))) return st;
    if ((st = upload(&m->d_tri, h.tri, b, s))) return st;
    if ((st = upload(&m->d_hubs, h.hubs, b, s))) return st;
    if ((st = upload(&m->d_medium, h.medium, b, s))) return st;
    if ((st = upload(&m->d_large, h.large, b, s))) return st;
    if (d->order) {
      if ((st = upload(&m->d_order, h.order, b, s))) return st;
      if ((st = upload(&m->d_tri_order, h.tri_order, b, s))) return st;
    }
  }
  ut.mark("layout");
  m->forma_flow_auto = flow_size && m->hm.large.empty() && staged();
  const auto& hm = m->hm;
  const int64_t nv = hm.nv, nt = hm.nt;
  for (void** p : {&m->buf[0], &m->buf[1], &m->init}) {
    TSG_CUDA(cudaMalloc(p, 2 * nv * m->rsize));
    *b += 2 * nv * m->rsize;
  }
  TSG_CUDA(cudaMalloc(&m->d_alpha, nt * m->rsize));
  *b += nt * m->rsize;
  if ((st = dalloc(&m->d_xy_stage, 2 * nv, b))) return st;
  if ((st = dalloc(&m->d_vmin, nv, b))) return st;
  if ((st = dalloc(&m->d_decision, nv, b))) return st;
  if ((st = dalloc(&m->d_decision_orig, nv, b))) return st;
  if ((st = dalloc(&m->d_state, 1, b))) return st;
  if ((st = dalloc(&m->d_maxabs, 1, b))) return st;
  if ((st = dalloc(&m->d_ext, 3, b))) return st;
  if ((st = dalloc(&m->d_side_ctr, 2, b))) return st;
  TSG_CUDA(cudaMemsetAsync(m->d_side_ctr, 0, 2 * sizeof(uint32_t), s));
  for (int32_t s2 : hm.hubs) m->hub_max_deg = std::max<int32_t>(m->hub_max_deg, hm.off[s2 + 1] - hm.off[s2]);
  while (m->n_hub_fast < static_cast<int64_t>(hm.large.size()) &&
         hm.off[hm.large[m->n_hub_fast] + 1] - hm.off[hm.large[m->n_hub_fast]] > static_cast<uint32_t>(kHubFastMin))
    ++m->n_hub_fast;
  {
    // AUTO side schedule: the persistent side_rows kernel when its estimated time fits inside
    // the tile grid's.  Calibrated on cfg3 (B200): the tile grid runs ~36 G vertices/s on 148
    // SMs; a side warp (32 registers, beside the tile grid) takes ~0.09 us per row entry plus
    // ~40 entries' worth per row; one warp per SM sub-partition.  Rows whose single-warp time
    // would exceed half the tile grid's keep a CTA each (hub_fast_update after the tile grid).
    const double sms = std::max(1, m->num_sms);
    const double tile_us = static_cast<double>(hm.nv) / 36e3 * (148.0 / sms);
    double entries = 0.0;
    for (int32_t r : hm.large) entries += static_cast<double>(hm.off[r + 1] - hm.off[r]) + 40.0;
    const double side_us = 0.09 * entries / (kSideWarps * sms);
    const double row_cap = std::max<double>(kHubFastMin, 0.5 * tile_us / 0.16);
    while (m->n_side_cta < static_cast<int64_t>(hm.large.size()) &&
           hm.off[hm.large[m->n_side_cta] + 1] - hm.off[hm.large[m->n_side_cta]] > row_cap)
      ++m->n_side_cta;
    // ... and only when one side CTA fits in the shared memory left by kTileMinBlocks tile CTAs
    // (dynamic + ~3 KB static + 1 KB reserved each; 228 KB per SM).
    const size_t pair = 2 * m->rsize;
    const size_t tile_smem = tile_smem_estimate(hm, m->rsize);
    const size_t side_smem = kSideWarps * static_cast<size_t>(kWarpTierCap) * pair + 1024;
    const bool fits = tsg::kTileMinBlocks * tile_smem + side_smem <= 228 * 1024;
    m->side_persist_auto = !hm.large.empty() && side_us <= tile_us && fits;
    if (std::getenv("TSG_DIAG"))
      std::fprintf(stderr, "[tsg] side rows %zu: est %.0f us vs tile grid %.0f us -> %s (%lld CTA rows)\n",
                   hm.large.size(), side_us, tile_us, m->side_persist_auto ? "persistent" : "kernels",
                   static_cast<long long>(m->n_side_cta));
  }
  ut.mark("buffers, side schedule");
  if ((st = ensure_stats_capacity(m.get(), 128))) return st;
  st = dispatch(m.get(), [&](auto E) { return decltype(E)::set_coords(m.get(), d->xy); });
  if (st) return st;
  st = dispatch(m.get(), [&](auto E) { return decltype(E)::prepare(m.get()); });
  if (st) return st;
  if (m->side_persist_auto) {
    // The persistent side kernel lives in the registers and shared memory that kTileMinBlocks
    // tile CTAs leave on an SM; a tile kernel that fits more CTAs (fp32: 58 registers, 4 CTAs)
    // leaves no room, and the side kernel would only run where tile CTAs end (measured, cfg3
    // fp32: 0.366 ms per pass persistent vs 0.344 ms with the per-tier grids after the tiles).
    int per_sm = 0;
    st = dispatch(m.get(), [&](auto E) { return decltype(E)::tile_blocks_per_sm(m.get(), &per_sm); });
    if (st) return st;
    if (per_sm > tsg::kTileMinBlocks) m->side_persist_auto = false;
    if (std::getenv("TSG_DIAG"))
      std::fprintf(stderr, "[tsg] tile CTAs per SM %d -> side rows %s\n", per_sm,
                   m->side_persist_auto ? "persistent" : "kernels");
  }
  TSG_CUDA(cudaStreamSynchronize(s));
  ut.mark("coords, prepare");
  {
    // the prep temporaries kept in the default pool during the upload go back to the device
    cudaMemPool_t pool;
    TSG_CUDA(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
    TSG_CUDA(cudaMemPoolTrimTo(pool, 0));
  }
  *out = m.release();
  return TSG_OK;
}

extern "C" {

tsg_status tsg_mesh_free(tsg_mesh* m) {
  TSG_LOCK_MESH(m);
  if (!m) return TSG_OK;
  cudaSetDevice(m->ctx->device);
  m->gc.reset();
  free_form_b(m);
  void* ptrs[] = {m->buf[0], m->buf[1], m->init, m->d_off, m->d_nbr, m->d_fan, m->d_fan16, m->d_tmeta, m->d_tile_rec, m->d_ext_off, m->d_tile_ext, m->d_trec, m->d_vinc_off, m->d_vinc,
                  m->d_tri, m->d_hubs, m->d_medium, m->d_large, m->d_maxabs, m->d_order, m->d_tri_order, m->d_alpha, m->d_xy_stage,
                  m->d_vmin, m->d_decision, m->d_decision_orig, m->d_state, m->d_acc, m->d_md, m->d_sacc, m->d_smd,
                  m->d_ext, m->d_side_ctr, m->d_rare, m->d_send_slots, m->d_recv_slots, m->d_halo_stage,
                  m->d_peer_sync, m->d_peer_tab, m->d_push_peer, m->d_push_src, m->d_push_dst,
                  m->d_fpush_mask, m->d_fpush_off, m->d_fpush_peer, m->d_fpush_dst, m->d_tflow, m->d_rank};
  for (void* p : ptrs) cudaFree(p);
  for (int b = 0; b < 2; ++b) {
    cudaFree(m->d_batch_in[b]);
    cudaFree(m->d_batch_out[b]);
  }
  cudaFreeHost(m->h_batch_state);
  cudaFree(m->d_batch_state);
  delete m;
  return TSG_OK;
}

int64_t tsg_mesh_device_bytes(const tsg_mesh* m) { return m ? m->bytes : 0; }

tsg_status tsg_mesh_set_coords(tsg_mesh* m, const double* xy) {
  if (!m || !xy) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg_status st = dispatch(m, [&](auto E) { return decltype(E)::set_coords(m, xy); });
  if (st) return st;
  TSG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  return TSG_OK;
}

tsg_status tsg_mesh_restore_coords(tsg_mesh* m) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  const size_t bytes = 2 * m->hm.nv * m->rsize;
  TSG_CUDA(cudaMemcpyAsync(m->buf[0], m->init, bytes, cudaMemcpyDeviceToDevice, m->ctx->stream));
  TSG_CUDA(cudaMemcpyAsync(m->buf[1], m->init, bytes, cudaMemcpyDeviceToDevice, m->ctx->stream));
  m->cur = 0;
  return TSG_OK;
}

tsg_status tsg_mesh_get_coords(tsg_mesh* m, double* xy_out) {
  TSG_LOCK_MESH(m);
  if (!m || !xy_out) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  return dispatch(m, [&](auto E) { return decltype(E)::get_coords(m, xy_out); });
}

tsg_status tsg_tri_alpha(tsg_mesh* m, double* alpha_out) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  tsg_status st = dispatch(m, [&](auto E) { return decltype(E)::refresh_alpha(m); });
  if (st) return st;
  if (alpha_out) {
    // device triangle i holds original triangle tri_order[i]
    double* tmp = m->d_xy_stage;  // 2*nv doubles; triangles may exceed it
    double* dst = nullptr;
    bool own = false;
    if (m->hm.nt <= 2 * m->hm.nv) {
      dst = tmp;
    } else {
      TSG_CUDA(cudaMalloc(&dst, m->hm.nt * sizeof(double)));
      own = true;
    }
    if (m->prec == TSG_F64)
      to_double_scatter<double><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
          static_cast<const double*>(m->d_alpha), m->d_tri_order, m->hm.nt, dst);
    else
      to_double_scatter<float><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
          static_cast<const float*>(m->d_alpha), m->d_tri_order, m->hm.nt, dst);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(alpha_out, dst, m->hm.nt * sizeof(double), cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    if (own) cudaFree(dst);
  } else {
    TSG_CUDA(cudaStreamSynchronize(s));
  }
  return TSG_OK;
}

tsg_status tsg_vertex_minima(tsg_mesh* m, double* vmin_out) {
  TSG_LOCK_MESH(m);
  if (!m || !vmin_out) return fail(TSG_ERR_INVALID, "null argument");
  tsg_status st = tsg_tri_alpha(m, nullptr);
  if (st) return st;
  cudaStream_t s = m->ctx->stream;
  const int64_t nv = m->hm.nv;
  if (m->prec == TSG_F64)
    tsg::vertex_min<double><<<grid_for(nv, 256), 256, 0, s>>>(m->d_vinc_off, m->d_vinc,
                                                              static_cast<const double*>(m->d_alpha), nv, m->d_vmin);
  else
    tsg::vertex_min<float><<<grid_for(nv, 256), 256, 0, s>>>(m->d_vinc_off, m->d_vinc,
                                                             static_cast<const float*>(m->d_alpha), nv, m->d_vmin);
  TSG_LAUNCHED();
  to_double_scatter<double><<<grid_for(nv, 256), 256, 0, s>>>(m->d_vmin, m->d_order, nv, m->d_xy_stage);
  TSG_LAUNCHED();
  TSG_CUDA(cudaMemcpyAsync(vmin_out, m->d_xy_stage, nv * sizeof(double), cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}

tsg_status tsg_alpha_extrema(tsg_mesh* m, double* min_out, double* max_out, int64_t* nonpos_out) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_status st = tsg_tri_alpha(m, nullptr);
  if (st) return st;
  cudaStream_t s = m->ctx->stream;
  const unsigned long long init[3] = {~0ULL, 0ULL, 0ULL};
  TSG_CUDA(cudaMemcpyAsync(m->d_ext, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (m->prec == TSG_F64)
    tsg::alpha_extrema<double><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
        static_cast<const double*>(m->d_alpha), m->hm.nt, m->d_ext, m->d_ext + 1, m->d_ext + 2);
  else
    tsg::alpha_extrema<float><<<grid_for(m->hm.nt, 256), 256, 0, s>>>(
        static_cast<const float*>(m->d_alpha), m->hm.nt, m->d_ext, m->d_ext + 1, m->d_ext + 2);
  TSG_LAUNCHED();
  unsigned long long h[3];
  TSG_CUDA(cudaMemcpyAsync(h, m->d_ext, sizeof(h), cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  auto unkey = [](unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffULL) : ~k;
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
  };
  if (min_out) *min_out = unkey(h[0]);
  if (max_out) *max_out = unkey(h[1]);
  if (nonpos_out) *nonpos_out = static_cast<int64_t>(h[2]);
  return TSG_OK;
}

}  // extern "C"

namespace {

// Passes per WHILE-body iteration (TSG_GRAPH_UNROLL overrides, 1..16).  Measured on B200:
// Form A without side rows (cfg2, 1M Delaunay) 45.8 -> 43.7 us per pass at 4; with the
// persistent side kernel (cfg3) unrolling loses its dispatch order (0.459 -> 0.573 ms), so 1.
int graph_unroll(const tsg_mesh* m, const tsg_smooth_cfg* c) {
  static const int env = [] {
    const char* e = std::getenv("TSG_GRAPH_UNROLL");
    return e ? std::max(1, std::min(16, std::atoi(e))) : 0;
  }();
  if (env) return env;
  const bool side_rows = c->form == TSG_FORM_A && !m->hm.large.empty();
  return c->max_iters >= 8 && !side_rows ? kGraphUnroll : 1;
}

// Resets the pass state and enqueues a whole smooth() as one launch of the cached
// conditional-WHILE graph on the context stream (no synchronisation).
tsg_status smooth_enqueue_graph(tsg_mesh* m, const tsg_smooth_cfg* c, int64_t* kernels_per_pass) {
  tsg_context* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  tsg_status st;
  if (c->form == TSG_FORM_B && (st = ensure_form_b(m, c->chunks))) return st;
  if ((st = ensure_stats_capacity(m, c->max_iters))) return st;
  const double tol_abs = c->move_tol * c->bbox_diag;  // smoothing.cpp:136, same rounding
  // (zeroed by a kernel: memsets may be served by a copy engine, where they would queue behind
  // the host<->device copies tsg_smooth_host_batch overlaps with this stream)
  reset_pass_state<<<grid_for(int64_t{tsg::kStatSlots} * c->max_iters, 256), 256, 0, s>>>(
      m->d_state, m->d_sacc, m->d_smd, int64_t{tsg::kStatSlots} * c->max_iters, m->d_side_ctr);
  TSG_LAUNCHED();
  GraphCache& g = m->gc;
  if (!(g.valid && !g.peer && g.form == c->form && g.strategy == c->strategy && g.chunks == c->chunks &&
        g.swap == c->swap && g.max_iters == c->max_iters && g.tol_abs == tol_abs)) {
    g.reset();
    TSG_CUDA(cudaGraphCreate(&g.graph, 0));
    cudaGraphConditionalHandle h;
    TSG_CUDA(cudaGraphConditionalHandleCreate(&h, g.graph, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t node;
    TSG_CUDA(cudaGraphAddNode(&node, g.graph, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    TSG_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    // The WHILE body holds `unroll` passes: the conditional re-launch of the body is paid once
    // per `unroll` passes.  After the stop rule fires inside the body, the remaining passes of the
    // body are empty (every node kernel and finalize_pass return on `done`).
    const int unroll = graph_unroll(m, c);
    int64_t k = 0;
    for (int u = 0; u < unroll && !st; ++u)
      st = dispatch(m, [&](auto E) {
        return decltype(E)::enqueue_pass(m, *c, s, tol_abs, h, 1, nullptr, nullptr, nullptr, &k);
      });
    k /= unroll;
    cudaGraph_t captured = nullptr;
    cudaError_t e = cudaStreamEndCapture(s, &captured);
    if (st) return st;
    if (e != cudaSuccess) return fail(TSG_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e));
    TSG_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
    g.valid = true;
    g.peer = false;
    g.form = c->form;
    g.strategy = c->strategy;
    g.chunks = c->chunks;
    g.swap = c->swap;
    g.max_iters = c->max_iters;
    g.tol_abs = tol_abs;
    g.kernels_per_pass = k;
  }
  *kernels_per_pass = g.kernels_per_pass;
  TSG_CUDA(cudaGraphLaunch(g.exec, s));
  return TSG_OK;
}

// Partitioned Form A over peer memory: the conditional-WHILE graph whose body is the pass's node
// kernels, peer_push and peer_sync (tsg_peer.cuh).  Built (stats capacity, capture,
// instantiation) before any rank's start barrier spins: those calls may synchronise the device,
// which must not happen while a peer on the same device waits for this rank
// (tsg_peer_prepare does it ahead of the first run).
tsg_status peer_graph(tsg_mesh* m, const tsg_smooth_cfg* c) {
  cudaStream_t s = m->ctx->stream;
  tsg_status st;
  if ((st = ensure_stats_capacity(m, c->max_iters))) return st;
  const double tol_abs = c->move_tol * c->bbox_diag;
  tsg_smooth_cfg cc = *c;
  cc.swap = TSG_SWAP_PINGPONG;  // see tsg_peer.cuh: copy mode maps to ping-pong (same results)
  GraphCache& g = m->gc;
  if (g.valid && g.peer && g.form == cc.form && g.strategy == cc.strategy && g.max_iters == cc.max_iters &&
      g.tol_abs == tol_abs)
    return TSG_OK;
  g.reset();
  TSG_CUDA(cudaGraphCreate(&g.graph, 0));
  cudaGraphConditionalHandle h;
  TSG_CUDA(cudaGraphConditionalHandleCreate(&h, g.graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  TSG_CUDA(cudaGraphAddNode(&node, g.graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  TSG_CUDA(cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  int64_t k = 0;
  st = dispatch(m, [&](auto E) {
    tsg_status r = decltype(E)::enqueue_pass(m, cc, s, tol_abs, h, 1, nullptr, nullptr, nullptr, &k, false);
    if (r) return r;
    return decltype(E)::peer_push(m, s, &k);
  });
  if (!st) {
    tsg::peer_sync<<<1, 32, 0, s>>>(m->d_state, m->d_sacc, m->d_smd, m->d_peer_sync, m->d_peer_tab, m->peer_rank,
                                    m->peer_world, m->d_acc, m->d_md, tol_abs, c->max_iters, h, 0);
    ++k;
  }
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &captured);
  if (st) return st;
  if (e != cudaSuccess) return fail(TSG_ERR_CUDA, std::string("capture: ") + cudaGetErrorString(e));
  TSG_CUDA(cudaGraphInstantiate(&g.exec, g.graph, 0));
  g.valid = true;
  g.peer = true;
  g.form = cc.form;
  g.strategy = cc.strategy;
  g.chunks = cc.chunks;
  g.swap = cc.swap;
  g.max_iters = cc.max_iters;
  g.tol_abs = tol_abs;
  g.kernels_per_pass = k;
  return TSG_OK;
}

// Start barrier, then one launch of the peer graph (no synchronising call in between).
tsg_status smooth_enqueue_peer(tsg_mesh* m, const tsg_smooth_cfg* c, int64_t* kernels_per_pass) {
  cudaStream_t s = m->ctx->stream;
  tsg_status st;
  if ((st = peer_graph(m, c))) return st;
  const double tol_abs = c->move_tol * c->bbox_diag;
  reset_pass_state<<<grid_for(int64_t{tsg::kStatSlots} * c->max_iters, 256), 256, 0, s>>>(
      m->d_state, m->d_sacc, m->d_smd, int64_t{tsg::kStatSlots} * c->max_iters, m->d_side_ctr);
  TSG_LAUNCHED();
  m->h_peer_tick0 = m->peer_tick + 1;
  TSG_CUDA(cudaMemcpyAsync(&m->d_peer_sync->tick0, &m->h_peer_tick0, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
  TSG_CUDA(cudaMemsetAsync(&m->d_peer_sync->error, 0, sizeof(int32_t), s));
  tsg::peer_sync<<<1, 32, 0, s>>>(m->d_state, m->d_sacc, m->d_smd, m->d_peer_sync, m->d_peer_tab, m->peer_rank,
                                  m->peer_world, m->d_acc, m->d_md, tol_abs, c->max_iters,
                                  cudaGraphConditionalHandle{}, 1);
  TSG_LAUNCHED();
  *kernels_per_pass = m->gc.kernels_per_pass;
  TSG_CUDA(cudaGraphLaunch(m->gc.exec, s));
  return TSG_OK;
}

// Form B through the dataflow kernel: rounds of up to kFlowRound passes per launch when the
// displacement stop is live (move_tol > 0), else every pass in one launch.  The stop rule
// (proj/src/smoothing.cpp:132-141) is applied to each round's per-pass totals in the
// reference's order; a NoMoves pass leaves the state unchanged, so the passes the launch ran
// after it are no-ops; a Displacement stop inside a round replays the round from its saved
// start up to the stopping pass (deterministic, so identical statistics).
constexpr int32_t kFlowRound = 64;

bool flow_selected(const tsg_mesh* m, const tsg_smooth_cfg* c) {
  if (c->form != TSG_FORM_B) return false;
  if (m->fb_mode == TSG_FORMB_FLOW) return true;
  // AUTO: the dataflow kernel where the level schedules are latency-bound — deep, narrow level
  // structures (cfg1 serial Form B: 195 levels of ~50 vertices per pass); wide levels stay on
  // the per-level / per-chunk launches (cost model in ensure_form_b).
  return m->fb_mode == TSG_FORMB_AUTO && m->flow_n > 0 && m->fb_auto_flow;
}

// Form A through the (tile, pass) dataflow kernel (tile_flow): meshes whose every movable row
// is in the tile kernel (no side rows), all staged, one GPU, the graph driver.  TSG_FORMA_FLOW
// = 0 / 1 forces it off / on where it applies; AUTO takes it where the per-pass launch's wave
// tail and launch cost are a large share of the pass.
bool tile_flow_selected(const tsg_mesh* m, const tsg_smooth_cfg* c) {
  if (c->form != TSG_FORM_A || c->driver != TSG_DRIVER_GRAPH || m->peer_world > 1) return false;
  if (!m->hm.large.empty() || !Engine<double, false>::tiles_staged(m)) return false;
  static const bool sweep = std::getenv("TSG_TWOPHASE_SWEEP") != nullptr;
  if (c->strategy == TSG_STRATEGY_TWOPHASE && sweep) return false;
  const int64_t ntiles = (m->hm.nv + m->hm.tile - 1) / m->hm.tile;
  if (ntiles * static_cast<int64_t>(c->max_iters) >= (int64_t{1} << 31)) return false;
  if (const char* e = std::getenv("TSG_FORMA_FLOW")) return std::atoi(e) != 0;
  // AUTO keeps the per-pass graph when the displacement stop is live: its stop rule runs on the
  // device after every pass, while the dataflow launch speculates rounds of 64 passes and replays
  // the stopping one (measured, 1M nodes converging in 72 passes: 136 passes of work, 4.6 vs
  // 3.2 ms; the maximum displacement falls off abruptly, so the stopping pass is not predictable
  // from its decay).
  return m->forma_flow_auto && c->move_tol * c->bbox_diag == 0.0;
}

tsg_status smooth_flow(tsg_mesh* m, const tsg_smooth_cfg* c, double tol_abs, int32_t* it_out, int32_t* stop_out,
                       std::vector<int32_t>& acc, std::vector<unsigned long long>& md, int64_t* kernels) {
  const bool form_a = c->form == TSG_FORM_A;
  auto launch = [&](int32_t p0, int32_t np) {
    return dispatch(m, [&](auto E) {
      return form_a ? decltype(E)::tile_flow_launch(m, *c, p0, np, kernels) : decltype(E)::flow_launch(m, p0, np, kernels);
    });
  };
  cudaStream_t s = m->ctx->stream;
  const int32_t P = c->max_iters;
  const int32_t round = tol_abs > 0.0 ? kFlowRound : P;
  const size_t coord_bytes = 2 * static_cast<size_t>(m->hm.nv) * m->rsize;
  acc.assign(P, 0);
  md.assign(P, 0ULL);
  std::vector<int32_t> sa;
  std::vector<unsigned long long> sm;
  int32_t p0 = 0;
  *it_out = P;
  *stop_out = tsg::kStopMaxIters;
  while (p0 < P) {
    const int32_t np = std::min(round, P - p0);
    const bool may_replay = tol_abs > 0.0 && np > 1;
    if (may_replay && !m->d_flow_save) TSG_CUDA(cudaMalloc(&m->d_flow_save, coord_bytes));
    if (may_replay)
      TSG_CUDA(cudaMemcpyAsync(m->d_flow_save, m->buf[p0 & 1], coord_bytes, cudaMemcpyDeviceToDevice, s));
    tsg_status st = launch(p0, np);
    if (st) return st;
    sa.resize(static_cast<size_t>(np) * tsg::kStatSlots);
    sm.resize(static_cast<size_t>(np) * tsg::kStatSlots);
    TSG_CUDA(cudaMemcpyAsync(sa.data(), m->d_sacc + static_cast<size_t>(p0) * tsg::kStatSlots,
                             sizeof(int32_t) * sa.size(), cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaMemcpyAsync(sm.data(), m->d_smd + static_cast<size_t>(p0) * tsg::kStatSlots,
                             sizeof(unsigned long long) * sm.size(), cudaMemcpyDeviceToHost, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    int32_t stop_at = -1;
    for (int32_t j = 0; j < np && stop_at < 0; ++j) {
      int32_t a = 0;
      unsigned long long b = 0;
      for (int k = 0; k < tsg::kStatSlots; ++k) {
        a += sa[static_cast<size_t>(j) * tsg::kStatSlots + k];
        b = std::max(b, sm[static_cast<size_t>(j) * tsg::kStatSlots + k]);
      }
      acc[p0 + j] = a;
      md[p0 + j] = b;
      double d;
      std::memcpy(&d, &b, sizeof d);
      if (a == 0) {
        stop_at = j;
        *stop_out = tsg::kStopNoMoves;
      } else if (d < tol_abs) {
        stop_at = j;
        *stop_out = tsg::kStopDisplacement;
      }
    }
    if (stop_at >= 0) {
      if (*stop_out == tsg::kStopDisplacement && stop_at + 1 < np) {
        TSG_CUDA(cudaMemcpyAsync(m->buf[p0 & 1], m->d_flow_save, coord_bytes, cudaMemcpyDeviceToDevice, s));
        st = launch(p0, stop_at + 1);
        if (st) return st;
      }
      *it_out = p0 + stop_at + 1;
      break;
    }
    p0 += np;
  }
  return TSG_OK;
}

}  // namespace

extern "C" {

tsg_status tsg_smooth(tsg_mesh* m, const tsg_smooth_cfg* c, tsg_smooth_stats* stats,
                      int32_t* accepted_per_pass, double* max_disp_per_pass, int32_t capacity) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg_context* ctx = m->ctx;
  cudaStream_t s = ctx->stream;
  if (c->form == TSG_FORM_B && (st = ensure_form_b(m, c->chunks))) return st;
  if ((st = ensure_stats_capacity(m, c->max_iters))) return st;
  st = dispatch(m, [&](auto E) { return decltype(E)::normalize(m); });
  if (st) return st;
  const double tol_abs = c->move_tol * c->bbox_diag;  // smoothing.cpp:136, same rounding
  TSG_CUDA(cudaMemsetAsync(m->d_state, 0, sizeof(tsg::PassState), s));
  TSG_CUDA(cudaMemsetAsync(m->d_sacc, 0, sizeof(int32_t) * tsg::kStatSlots * c->max_iters, s));
  TSG_CUDA(cudaMemsetAsync(m->d_smd, 0, sizeof(unsigned long long) * tsg::kStatSlots * c->max_iters, s));
  if (diag_enabled()) TSG_CUDA(cudaMemsetAsync(m->d_rare, 0, sizeof(unsigned long long) * (m->cap + 16), s));

  if (flow_selected(m, c) || tile_flow_selected(m, c)) {
    std::vector<int32_t> acc;
    std::vector<unsigned long long> md;
    int32_t it = 0, stop = 0;
    int64_t kernels = 0;
    TSG_CUDA(cudaEventRecord(ctx->ev0, s));
    if ((st = smooth_flow(m, c, tol_abs, &it, &stop, acc, md, &kernels))) return st;
    TSG_CUDA(cudaEventRecord(ctx->ev1, s));
    // final coordinates are in buf[it & 1]; copy mode keeps them in buf[0]
    if (c->swap == TSG_SWAP_COPY && (it & 1)) {
      st = dispatch(m, [&](auto E) {
        m->cur = 1;
        return decltype(E)::normalize(m);
      });
      if (st) return st;
    } else {
      m->cur = c->swap == TSG_SWAP_PINGPONG ? (it & 1) : 0;
    }
    const tsg::PassState hs{it, 1, stop, 0};
    TSG_CUDA(cudaMemcpyAsync(m->d_state, &hs, sizeof hs, cudaMemcpyHostToDevice, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    float total_ms = 0.f;
    TSG_CUDA(cudaEventElapsedTime(&total_ms, ctx->ev0, ctx->ev1));
    const int32_t n = std::min(capacity, it);
    for (int32_t p = 0; p < n; ++p) {
      if (accepted_per_pass) accepted_per_pass[p] = acc[p];
      if (max_disp_per_pass) std::memcpy(max_disp_per_pass + p, &md[p], sizeof(double));
    }
    if (stats) {
      stats->iterations = it;
      stats->stop = stop;
      stats->node_updates = m->hm.nv * static_cast<int64_t>(it);
      stats->device_ms = total_ms;
      stats->node_kernel_ms = total_ms;
      stats->launches = kernels;
      stats->schedule = TSG_SCHEDULE_FLOW;
    }
    return TSG_OK;
  }

  int64_t kernels_per_pass = 0;
  double node_ms = -1.0;
  int64_t launches = 0;
  const bool peer = m->peer_world > 1;
  if (peer) {
    if (c->form != TSG_FORM_A) return fail(TSG_ERR_INVALID, "the peer-memory partitioned driver runs Form A");
    TSG_CUDA(cudaEventRecord(ctx->ev0, s));
    if ((st = smooth_enqueue_peer(m, c, &kernels_per_pass))) return st;
    TSG_CUDA(cudaEventRecord(ctx->ev1, s));
    launches = 2;  // the start barrier and the graph
  } else if (c->driver == TSG_DRIVER_GRAPH) {
    TSG_CUDA(cudaEventRecord(ctx->ev0, s));
    if ((st = smooth_enqueue_graph(m, c, &kernels_per_pass))) return st;
    TSG_CUDA(cudaEventRecord(ctx->ev1, s));
  } else {
    // Plain launches; kernels early-exit once done is set.  Per-pass events bracket the
    // node-update launches so the bench can time the node kernel alone.
    const size_t need = 2 * static_cast<size_t>(c->max_iters);
    while (ctx->pass_events.size() < need) {
      cudaEvent_t e;
      TSG_CUDA(cudaEventCreate(&e));
      ctx->pass_events.push_back(e);
    }
    TSG_CUDA(cudaEventRecord(ctx->ev0, s));
    int32_t host_state[4] = {0, 0, 0, 0};
    int q = 0;
    for (; q < c->max_iters; ++q) {
      int64_t k = 0;
      st = dispatch(m, [&](auto E) {
        return decltype(E)::enqueue_pass(m, *c, s, tol_abs, cudaGraphConditionalHandle{}, 0, nullptr,
                                         ctx->pass_events[2 * q], ctx->pass_events[2 * q + 1], &k);
      });
      if (st) return st;
      kernels_per_pass = k;
      if ((q & 7) == 7 || q + 1 == c->max_iters) {
        TSG_CUDA(cudaMemcpyAsync(host_state, m->d_state, sizeof(host_state), cudaMemcpyDeviceToHost, s));
        TSG_CUDA(cudaStreamSynchronize(s));
        if (host_state[1]) {
          ++q;
          break;
        }
      }
    }
    TSG_CUDA(cudaEventRecord(ctx->ev1, s));
    TSG_CUDA(cudaStreamSynchronize(s));
    launches = kernels_per_pass * q;
  }
  TSG_CUDA(cudaStreamSynchronize(s));
  tsg::PassState hs;
  TSG_CUDA(cudaMemcpy(&hs, m->d_state, sizeof hs, cudaMemcpyDeviceToHost));
  float total_ms = 0.f;
  TSG_CUDA(cudaEventElapsedTime(&total_ms, ctx->ev0, ctx->ev1));
  const int32_t it = hs.pass;
  if (c->driver == TSG_DRIVER_STREAM) {
    node_ms = 0.0;  // node-update launches of the passes that ran (events bracket them)
    for (int p = 0; p < it; ++p) {
      float ms = 0.f;
      TSG_CUDA(cudaEventElapsedTime(&ms, ctx->pass_events[2 * p], ctx->pass_events[2 * p + 1]));
      node_ms += ms;
    }
    if (diag_enabled()) {
      std::vector<unsigned long long> rare(it);
      std::vector<int32_t> accd(it);
      TSG_CUDA(cudaMemcpy(rare.data(), m->d_rare + 16, sizeof(unsigned long long) * it, cudaMemcpyDeviceToHost));
      TSG_CUDA(cudaMemcpy(accd.data(), m->d_acc, sizeof(int32_t) * it, cudaMemcpyDeviceToHost));
      for (int p = 0; p < it; ++p) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->pass_events[2 * p], ctx->pass_events[2 * p + 1]);
        std::fprintf(stderr, "[tsg diag] pass %d node_ms %.4f accepted %d rare %llu\n", p, ms, accd[p], rare[p]);
      }
      unsigned long long hist[16];
      TSG_CUDA(cudaMemcpy(hist, m->d_rare, sizeof hist, cudaMemcpyDeviceToHost));
      for (int b = 0; b < 16; ++b) std::fprintf(stderr, "[tsg diag] |hyp-thr| 2^%d: %llu\n", b - 60, hist[b]);
    }
  }
  if (peer) {
    int32_t err = 0;
    TSG_CUDA(cudaMemcpy(&err, &m->d_peer_sync->error, sizeof err, cudaMemcpyDeviceToHost));
    m->peer_tick += 1 + static_cast<uint32_t>(it);
    if (err) return fail(TSG_ERR_CUDA, "peer barrier timed out (a rank did not reach the same pass)");
    m->cur = it & 1;
  } else if (c->swap == TSG_SWAP_PINGPONG) {
    m->cur = it & 1;
  } else {
    m->cur = 0;
  }
  const int32_t n = std::min(capacity, it);
  if (accepted_per_pass && n > 0)
    TSG_CUDA(cudaMemcpy(accepted_per_pass, m->d_acc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  if (max_disp_per_pass && n > 0) {
    std::vector<unsigned long long> bits(n);
    TSG_CUDA(cudaMemcpy(bits.data(), m->d_md, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
    std::memcpy(max_disp_per_pass, bits.data(), sizeof(double) * n);
  }
  if (stats) {
    stats->iterations = it;
    stats->stop = hs.stop;
    stats->node_updates = m->hm.nv * static_cast<int64_t>(it);
    stats->device_ms = total_ms;
    stats->node_kernel_ms = node_ms;
    stats->launches = peer ? 2 + kernels_per_pass * it
                      : c->driver == TSG_DRIVER_GRAPH ? kernels_per_pass * it : launches;
    stats->schedule = peer ? TSG_SCHEDULE_PEER : c->driver == TSG_DRIVER_GRAPH ? TSG_SCHEDULE_GRAPH : TSG_SCHEDULE_STREAM;
  }
  return TSG_OK;
}

tsg_status tsg_smooth_host_batch(tsg_mesh* m, int32_t n, const double* const* xy_in, const tsg_smooth_cfg* c,
                                 double* const* xy_out, int32_t* iterations_out, int32_t* stop_out) {
  TSG_LOCK_MESH(m);
  if (!m || n < 0 || (n > 0 && (!xy_in || !xy_out))) return fail(TSG_ERR_INVALID, "bad batch arguments");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  if (c->driver != TSG_DRIVER_GRAPH) return fail(TSG_ERR_INVALID, "the batch API runs the graph driver");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg_context* ctx = m->ctx;
  const int64_t nv = m->hm.nv;
  const size_t bytes = 2 * static_cast<size_t>(nv) * sizeof(double);
  for (int b = 0; b < 2; ++b) {
    if (!m->d_batch_in[b]) TSG_CUDA(cudaMalloc(&m->d_batch_in[b], bytes));
    if (!m->d_batch_out[b]) TSG_CUDA(cudaMalloc(&m->d_batch_out[b], bytes));
  }
  if (m->h_batch_cap < n) {
    cudaFreeHost(m->h_batch_state);
    cudaFree(m->d_batch_state);
    m->h_batch_state = nullptr;
    m->d_batch_state = nullptr;
    TSG_CUDA(cudaHostAlloc(&m->h_batch_state, sizeof(tsg::PassState) * n, cudaHostAllocDefault));
    TSG_CUDA(cudaMalloc(&m->d_batch_state, sizeof(tsg::PassState) * n));
    m->h_batch_cap = n;
  }
  cudaStream_t s = ctx->stream;
  // Form A through tile_flow when it is selected and the stop rule cannot fire after a pass
  // that changed the coordinates (move_tol == 0); otherwise the graph.
  const bool flow = tile_flow_selected(m, c) && c->move_tol * c->bbox_diag == 0.0;
  // The other dataflow cases (Form B's formb_flow; Form A with a live displacement stop) run
  // their rounds with the stop rule on the host: item by item, copies still on their streams.
  const bool flow_sync = !flow && (tile_flow_selected(m, c) || (c->form == TSG_FORM_B &&
                                                                (st = ensure_form_b(m, c->chunks)) == TSG_OK &&
                                                                flow_selected(m, c)));
  if (st) return st;
  if ((flow || flow_sync) && (st = ensure_stats_capacity(m, c->max_iters))) return st;
  // Item k uses staging slot k & 1.  The copy engines serve host<->device copies in issue
  // order, so the loop issues the input copy of item k+1 BEFORE the result copy of item k:
  //   copy_in : H2D(k+1)            (after item k-1 released the slot)
  //   compute : reorder in (k), smooth graph (k), reorder out (k) (after item k-2's result left)
  //   copy_out: D2H(k)
  // H2D(k+1) then runs during the passes of item k, D2H(k) during those of item k+1.
  auto h2d = [&](int32_t k) -> tsg_status {
    const int b = k & 1;
    if (k >= 2) TSG_CUDA(cudaStreamWaitEvent(ctx->copy_in, ctx->ev_in_free[b], 0));
    TSG_CUDA(cudaMemcpyAsync(m->d_batch_in[b], xy_in[k], bytes, cudaMemcpyHostToDevice, ctx->copy_in));
    TSG_CUDA(cudaEventRecord(ctx->ev_in_ready[b], ctx->copy_in));
    return TSG_OK;
  };
  if (n > 0 && (st = h2d(0))) return st;
  for (int32_t k = 0; k < n; ++k) {
    const int b = k & 1;
    if (k + 1 < n && (st = h2d(k + 1))) return st;
    TSG_CUDA(cudaStreamWaitEvent(s, ctx->ev_in_ready[b], 0));
    st = dispatch(m, [&](auto E) { return decltype(E)::batch_load(m, m->d_batch_in[b]); });
    if (st) return st;
    TSG_CUDA(cudaEventRecord(ctx->ev_in_free[b], s));
    int64_t kpp = 0;
    int32_t swap = c->swap;
    if (flow) {
      // every pass in one dataflow launch, the stop rule on the device (tol_abs == 0)
      reset_pass_state<<<grid_for(tsg::kStatSlots * c->max_iters, 256), 256, 0, s>>>(
          m->d_state, m->d_sacc, m->d_smd, static_cast<int64_t>(tsg::kStatSlots) * c->max_iters, m->d_side_ctr);
      TSG_LAUNCHED();
      st = dispatch(m, [&](auto E) { return decltype(E)::tile_flow_launch(m, *c, 0, c->max_iters, &kpp); });
      if (st) return st;
      flow_stop_state<<<1, 32, 0, s>>>(m->d_sacc, m->d_smd, c->max_iters, 0.0, m->d_state);
      TSG_LAUNCHED();
      swap = TSG_SWAP_PINGPONG;  // the final coordinates are in buf[iterations & 1]
    } else if (flow_sync) {
      reset_pass_state<<<grid_for(tsg::kStatSlots * c->max_iters, 256), 256, 0, s>>>(
          m->d_state, m->d_sacc, m->d_smd, static_cast<int64_t>(tsg::kStatSlots) * c->max_iters, m->d_side_ctr);
      TSG_LAUNCHED();
      std::vector<int32_t> acc;
      std::vector<unsigned long long> md;
      int32_t it = 0, stop = 0;
      if ((st = smooth_flow(m, c, c->move_tol * c->bbox_diag, &it, &stop, acc, md, &kpp))) return st;
      set_state<<<1, 1, 0, s>>>(m->d_state, it, stop);
      TSG_LAUNCHED();
      swap = TSG_SWAP_PINGPONG;
    } else if ((st = smooth_enqueue_graph(m, c, &kpp))) {
      return st;
    }
    if (k >= 2) TSG_CUDA(cudaStreamWaitEvent(s, ctx->ev_out_free[b], 0));
    st = dispatch(m, [&](auto E) { return decltype(E)::batch_store(m, swap, m->d_batch_out[b]); });
    if (st) return st;
    save_state<<<1, 1, 0, s>>>(m->d_state, m->d_batch_state + k);
    TSG_LAUNCHED();
    TSG_CUDA(cudaEventRecord(ctx->ev_out_ready[b], s));
    TSG_CUDA(cudaStreamWaitEvent(ctx->copy_out, ctx->ev_out_ready[b], 0));
    TSG_CUDA(cudaMemcpyAsync(xy_out[k], m->d_batch_out[b], bytes, cudaMemcpyDeviceToHost, ctx->copy_out));
    TSG_CUDA(cudaEventRecord(ctx->ev_out_free[b], ctx->copy_out));
  }
  TSG_CUDA(cudaMemcpyAsync(m->h_batch_state, m->d_batch_state, sizeof(tsg::PassState) * n, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(ctx->copy_out));
  TSG_CUDA(cudaStreamSynchronize(s));
  for (int32_t k = 0; k < n; ++k) {
    if (iterations_out) iterations_out[k] = m->h_batch_state[k].pass;
    if (stop_out) stop_out[k] = m->h_batch_state[k].stop;
  }
  if (n > 0) m->cur = (flow || flow_sync || c->swap == TSG_SWAP_PINGPONG) ? (m->h_batch_state[n - 1].pass & 1) : 0;
  return TSG_OK;
}

tsg_status tsg_smooth_host(tsg_mesh* m, const double* xy_in, const tsg_smooth_cfg* c, double* xy_out,
                           tsg_smooth_stats* stats, int32_t* accepted_per_pass,
                           double* max_disp_per_pass, int32_t capacity) {
  TSG_LOCK_MESH(m);
  if (!m || !xy_in || !xy_out) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg_status st = dispatch(m, [&](auto E) { return decltype(E)::set_coords(m, xy_in); });
  if (st) return st;
  if ((st = tsg_smooth(m, c, stats, accepted_per_pass, max_disp_per_pass, capacity))) return st;
  return tsg_mesh_get_coords(m, xy_out);
}

tsg_status tsg_pass_lockstep(tsg_mesh* m, int32_t form, int32_t chunks, int8_t* decision_out,
                             int32_t* accepted_out, double* max_disp_out) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_smooth_cfg c{};
  c.form = form;
  c.strategy = TSG_STRATEGY_FUSED;
  c.chunks = chunks;
  c.swap = TSG_SWAP_PINGPONG;
  c.max_iters = 1;
  c.driver = TSG_DRIVER_STREAM;
  c.move_tol = 0.0;
  c.bbox_diag = 0.0;
  tsg_status st = validate_cfg(&c);
  if (st) return st;
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  if (form == TSG_FORM_B && (st = ensure_form_b(m, chunks))) return st;
  st = dispatch(m, [&](auto E) { return decltype(E)::normalize(m); });
  if (st) return st;
  TSG_CUDA(cudaMemsetAsync(m->d_state, 0, sizeof(tsg::PassState), s));
  TSG_CUDA(cudaMemsetAsync(m->d_sacc, 0, sizeof(int32_t) * tsg::kStatSlots, s));
  TSG_CUDA(cudaMemsetAsync(m->d_smd, 0, sizeof(unsigned long long) * tsg::kStatSlots, s));
  TSG_CUDA(cudaMemsetAsync(m->d_decision, 0xff, m->hm.nv, s));
  int64_t k = 0;
  st = dispatch(m, [&](auto E) {
    return decltype(E)::enqueue_pass(m, c, s, 0.0, cudaGraphConditionalHandle{}, 0, m->d_decision,
                                     nullptr, nullptr, &k);
  });
  if (st) return st;
  m->cur = 1;
  if (decision_out) {
    scatter_i8<<<grid_for(m->hm.nv, 256), 256, 0, s>>>(m->d_decision, m->d_order, m->hm.nv,
                                                       m->d_decision_orig);
    TSG_LAUNCHED();
    TSG_CUDA(cudaMemcpyAsync(decision_out, m->d_decision_orig, m->hm.nv, cudaMemcpyDeviceToHost, s));
  }
  int32_t acc = 0;
  unsigned long long md = 0;
  TSG_CUDA(cudaMemcpyAsync(&acc, m->d_acc, sizeof acc, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(&md, m->d_md, sizeof md, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  if (accepted_out) *accepted_out = acc;
  if (max_disp_out) std::memcpy(max_disp_out, &md, sizeof(double));
  return TSG_OK;
}

tsg_status tsg_pass(tsg_mesh* m, const tsg_smooth_cfg* c, int32_t* accepted_out, double* max_disp_out) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  if (c->form == TSG_FORM_B && (st = ensure_form_b(m, c->chunks))) return st;
  if ((st = ensure_stats_capacity(m, 2))) return st;
  if (c->swap == TSG_SWAP_COPY) {
    st = dispatch(m, [&](auto E) { return decltype(E)::normalize(m); });
    if (st) return st;
  }
  const int32_t q = c->swap == TSG_SWAP_PINGPONG ? m->cur : 0;  // pass index = buffer parity
  const tsg::PassState init{q, 0, 0, 0};
  TSG_CUDA(cudaMemcpyAsync(m->d_state, &init, sizeof init, cudaMemcpyHostToDevice, s));
  TSG_CUDA(cudaMemsetAsync(m->d_sacc + q * tsg::kStatSlots, 0, sizeof(int32_t) * tsg::kStatSlots, s));
  TSG_CUDA(cudaMemsetAsync(m->d_smd + q * tsg::kStatSlots, 0, sizeof(unsigned long long) * tsg::kStatSlots, s));
  tsg_smooth_cfg one = *c;
  one.max_iters = q + 1;
  one.driver = TSG_DRIVER_STREAM;
  int64_t k = 0;
  st = dispatch(m, [&](auto E) {
    return decltype(E)::enqueue_pass(m, one, s, -1.0, cudaGraphConditionalHandle{}, 0, nullptr, nullptr,
                                     nullptr, &k);
  });
  if (st) return st;
  int32_t acc = 0;
  unsigned long long md = 0;
  TSG_CUDA(cudaMemcpyAsync(&acc, m->d_acc + q, sizeof acc, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaMemcpyAsync(&md, m->d_md + q, sizeof md, cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  m->cur = c->swap == TSG_SWAP_PINGPONG ? (q ^ 1) : 0;
  if (accepted_out) *accepted_out = acc;
  if (max_disp_out) std::memcpy(max_disp_out, &md, sizeof(double));
  return TSG_OK;
}

tsg_status tsg_halo_plan(tsg_mesh* m, const int64_t* send_ids, int64_t n_send, const int64_t* recv_ids,
                         int64_t n_recv) {
  TSG_LOCK_MESH(m);
  if (!m || n_send < 0 || n_recv < 0 || (n_send && !send_ids) || (n_recv && !recv_ids))
    return fail(TSG_ERR_INVALID, "bad halo plan");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if (tsg_status st = ensure_host_rows(m)) return st;
  std::vector<int32_t> ss(n_send), rs(n_recv);
  for (int64_t i = 0; i < n_send; ++i) {
    if (send_ids[i] < 0 || send_ids[i] >= m->hm.nv) return fail(TSG_ERR_INVALID, "send id out of range");
    ss[i] = static_cast<int32_t>(m->hm.rank[send_ids[i]]);
  }
  for (int64_t i = 0; i < n_recv; ++i) {
    if (recv_ids[i] < 0 || recv_ids[i] >= m->hm.nv) return fail(TSG_ERR_INVALID, "recv id out of range");
    rs[i] = static_cast<int32_t>(m->hm.rank[recv_ids[i]]);
  }
  cudaFree(m->d_send_slots);
  cudaFree(m->d_recv_slots);
  cudaFree(m->d_halo_stage);
  m->d_send_slots = m->d_recv_slots = nullptr;
  m->d_halo_stage = nullptr;
  int64_t b = 0;
  tsg_status st;
  if ((st = upload(&m->d_send_slots, ss, &b, m->ctx->stream))) return st;
  if ((st = upload(&m->d_recv_slots, rs, &b, m->ctx->stream))) return st;
  if ((st = dalloc(&m->d_halo_stage, 2 * std::max<int64_t>(1, std::max(n_send, n_recv)), &b))) return st;
  TSG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  m->n_send = n_send;
  m->n_recv = n_recv;
  return TSG_OK;
}

tsg_status tsg_mesh_side_schedule(tsg_mesh* m, int32_t mode) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  if (mode < TSG_SIDE_AUTO || mode > TSG_SIDE_PERSIST) return fail(TSG_ERR_INVALID, "unknown side-row schedule");
  if (m->side_mode != mode) {
    m->side_mode = mode;
    m->gc.reset();  // re-captured by the next call
  }
  return TSG_OK;
}

tsg_status tsg_mesh_formb_schedule(tsg_mesh* m, int32_t mode) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  if (mode < TSG_FORMB_AUTO || mode > TSG_FORMB_FLOW) return fail(TSG_ERR_INVALID, "unknown Form B schedule");
  if (m->fb_mode != mode) {
    m->fb_mode = mode;
    m->fb_chunks = 0;  // rebuilt (and the graph re-captured) by the next Form B call
    m->gc.reset();
  }
  return TSG_OK;
}

tsg_status tsg_dist_begin(tsg_mesh* m, const tsg_smooth_cfg* c) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  if (c->form != TSG_FORM_A) return fail(TSG_ERR_INVALID, "the partitioned driver supports Form A");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  if ((st = ensure_stats_capacity(m, c->max_iters + 1))) return st;
  st = dispatch(m, [&](auto E) { return decltype(E)::normalize(m); });  // current coordinates in buf0
  if (st) return st;
  m->dist_launches = 0;
  TSG_CUDA(cudaMemsetAsync(m->d_state, 0, sizeof(tsg::PassState), s));
  TSG_CUDA(cudaMemsetAsync(m->d_sacc, 0, sizeof(int32_t) * tsg::kStatSlots * (c->max_iters + 1), s));
  TSG_CUDA(cudaMemsetAsync(m->d_smd, 0, sizeof(unsigned long long) * tsg::kStatSlots * (c->max_iters + 1), s));
  return TSG_OK;
}

tsg_status tsg_dist_pass(tsg_mesh* m, const tsg_smooth_cfg* c, double* stats_dev) {
  TSG_LOCK_MESH(m);
  if (!m || !stats_dev) return fail(TSG_ERR_INVALID, "null argument");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  int64_t k = 0;
  st = dispatch(m, [&](auto E) {
    return decltype(E)::enqueue_pass(m, *c, s, -1.0, cudaGraphConditionalHandle{}, 0, nullptr, nullptr, nullptr, &k,
                                     false);
  });
  if (st) return st;
  dist_fold<<<1, 32, 0, s>>>(m->d_state, m->d_sacc, m->d_smd, stats_dev);
  TSG_LAUNCHED();
  m->dist_launches += k + 1;
  return TSG_OK;
}

tsg_status tsg_dist_halo_pack(tsg_mesh* m, const tsg_smooth_cfg* c, double* out_dev) {
  TSG_LOCK_MESH(m);
  if (!m || !c || (m->n_send && !out_dev)) return fail(TSG_ERR_INVALID, "bad halo pack arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if (m->n_send == 0) return TSG_OK;
  cudaStream_t s = m->ctx->stream;
  const unsigned g = grid_for(m->n_send, 256);
  if (m->prec == TSG_F64) {
    if (m->layout == TSG_LAYOUT_SOA)
      dist_halo_pack<double, true><<<g, 256, 0, s>>>(coords_of<double, true>(m, 0), coords_of<double, true>(m, 1), c->swap, m->d_state, m->d_send_slots, m->n_send, out_dev);
    else
      dist_halo_pack<double, false><<<g, 256, 0, s>>>(coords_of<double, false>(m, 0), coords_of<double, false>(m, 1), c->swap, m->d_state, m->d_send_slots, m->n_send, out_dev);
  } else {
    if (m->layout == TSG_LAYOUT_SOA)
      dist_halo_pack<float, true><<<g, 256, 0, s>>>(coords_of<float, true>(m, 0), coords_of<float, true>(m, 1), c->swap, m->d_state, m->d_send_slots, m->n_send, out_dev);
    else
      dist_halo_pack<float, false><<<g, 256, 0, s>>>(coords_of<float, false>(m, 0), coords_of<float, false>(m, 1), c->swap, m->d_state, m->d_send_slots, m->n_send, out_dev);
  }
  TSG_LAUNCHED();
  ++m->dist_launches;
  return TSG_OK;
}

tsg_status tsg_dist_halo_unpack(tsg_mesh* m, const double* in_dev) {
  TSG_LOCK_MESH(m);
  if (!m || (m->n_recv && !in_dev)) return fail(TSG_ERR_INVALID, "bad halo unpack arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if (m->n_recv == 0) return TSG_OK;
  cudaStream_t s = m->ctx->stream;
  const unsigned g = grid_for(m->n_recv, 256);
  if (m->prec == TSG_F64) {
    if (m->layout == TSG_LAYOUT_SOA)
      dist_halo_unpack<double, true><<<g, 256, 0, s>>>(coords_of<double, true>(m, 0), coords_of<double, true>(m, 1), m->d_state, m->d_recv_slots, m->n_recv, in_dev, m->d_maxabs);
    else
      dist_halo_unpack<double, false><<<g, 256, 0, s>>>(coords_of<double, false>(m, 0), coords_of<double, false>(m, 1), m->d_state, m->d_recv_slots, m->n_recv, in_dev, m->d_maxabs);
  } else {
    if (m->layout == TSG_LAYOUT_SOA)
      dist_halo_unpack<float, true><<<g, 256, 0, s>>>(coords_of<float, true>(m, 0), coords_of<float, true>(m, 1), m->d_state, m->d_recv_slots, m->n_recv, in_dev, m->d_maxabs);
    else
      dist_halo_unpack<float, false><<<g, 256, 0, s>>>(coords_of<float, false>(m, 0), coords_of<float, false>(m, 1), m->d_state, m->d_recv_slots, m->n_recv, in_dev, m->d_maxabs);
  }
  TSG_LAUNCHED();
  ++m->dist_launches;
  return TSG_OK;
}

tsg_status tsg_dist_finalize(tsg_mesh* m, const tsg_smooth_cfg* c, const double* gathered_dev, int32_t n_parts) {
  TSG_LOCK_MESH(m);
  if (!m || !c || !gathered_dev || n_parts < 1) return fail(TSG_ERR_INVALID, "bad finalize arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  const double tol_abs = c->move_tol * c->bbox_diag;  // smoothing.cpp:136, same rounding
  dist_finalize<<<1, 1, 0, m->ctx->stream>>>(m->d_state, gathered_dev, n_parts, m->d_acc, m->d_md, tol_abs,
                                            c->max_iters);
  TSG_LAUNCHED();
  ++m->dist_launches;
  return TSG_OK;
}

tsg_status tsg_dist_status(tsg_mesh* m, int32_t* iterations, int32_t* done, int32_t* stop) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg::PassState hs;
  TSG_CUDA(cudaMemcpyAsync(&hs, m->d_state, sizeof hs, cudaMemcpyDeviceToHost, m->ctx->stream));
  TSG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  if (iterations) *iterations = hs.pass;
  if (done) *done = hs.done;
  if (stop) *stop = hs.stop;
  return TSG_OK;
}

tsg_status tsg_dist_end(tsg_mesh* m, const tsg_smooth_cfg* c, int32_t* accepted_per_pass, double* max_disp_per_pass,
                        int32_t capacity, int32_t* iterations_out, int32_t* stop_out, int64_t* launches_out) {
  TSG_LOCK_MESH(m);
  if (!m || !c) return fail(TSG_ERR_INVALID, "null argument");
  int32_t it = 0, done = 0, stop = 0;
  tsg_status st = tsg_dist_status(m, &it, &done, &stop);
  if (st) return st;
  if (c->swap == TSG_SWAP_PINGPONG) m->cur = it & 1;
  else m->cur = 0;
  const int32_t n = std::min(capacity, it);
  if (accepted_per_pass && n > 0)
    TSG_CUDA(cudaMemcpy(accepted_per_pass, m->d_acc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  if (max_disp_per_pass && n > 0) {
    std::vector<unsigned long long> bits(n);
    TSG_CUDA(cudaMemcpy(bits.data(), m->d_md, sizeof(unsigned long long) * n, cudaMemcpyDeviceToHost));
    std::memcpy(max_disp_per_pass, bits.data(), sizeof(double) * n);
  }
  if (iterations_out) *iterations_out = it;
  if (stop_out) *stop_out = stop;
  if (launches_out) *launches_out = m->dist_launches;
  return TSG_OK;
}

tsg_status tsg_halo_pack(tsg_mesh* m, double* out, int32_t out_is_host) {
  TSG_LOCK_MESH(m);
  if (!m || (m->n_send && !out)) return fail(TSG_ERR_INVALID, "bad halo pack arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  if (m->n_send == 0) return TSG_OK;
  double* dst = out_is_host ? m->d_halo_stage : out;
  if (m->prec == TSG_F64) {
    if (m->layout == TSG_LAYOUT_SOA)
      halo_pack<double, true><<<grid_for(m->n_send, 256), 256, 0, s>>>(coords_of<double, true>(m, m->cur), m->d_send_slots, m->n_send, dst);
    else
      halo_pack<double, false><<<grid_for(m->n_send, 256), 256, 0, s>>>(coords_of<double, false>(m, m->cur), m->d_send_slots, m->n_send, dst);
  } else {
    if (m->layout == TSG_LAYOUT_SOA)
      halo_pack<float, true><<<grid_for(m->n_send, 256), 256, 0, s>>>(coords_of<float, true>(m, m->cur), m->d_send_slots, m->n_send, dst);
    else
      halo_pack<float, false><<<grid_for(m->n_send, 256), 256, 0, s>>>(coords_of<float, false>(m, m->cur), m->d_send_slots, m->n_send, dst);
  }
  TSG_LAUNCHED();
  if (out_is_host)
    TSG_CUDA(cudaMemcpyAsync(out, dst, 2 * m->n_send * sizeof(double), cudaMemcpyDeviceToHost, s));
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}

tsg_status tsg_halo_unpack(tsg_mesh* m, const double* in, int32_t in_is_host) {
  TSG_LOCK_MESH(m);
  if (!m || (m->n_recv && !in)) return fail(TSG_ERR_INVALID, "bad halo unpack arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  cudaStream_t s = m->ctx->stream;
  if (m->n_recv == 0) return TSG_OK;
  const double* src = in;
  if (in_is_host) {
    TSG_CUDA(cudaMemcpyAsync(m->d_halo_stage, in, 2 * m->n_recv * sizeof(double), cudaMemcpyHostToDevice, s));
    src = m->d_halo_stage;
  }
  const unsigned g = grid_for(m->n_recv, 256);
  if (m->prec == TSG_F64) {
    if (m->layout == TSG_LAYOUT_SOA)
      halo_unpack<double, true><<<g, 256, 0, s>>>(coords_of<double, true>(m, 0), coords_of<double, true>(m, 1), m->d_recv_slots, m->n_recv, src, m->d_maxabs);
    else
      halo_unpack<double, false><<<g, 256, 0, s>>>(coords_of<double, false>(m, 0), coords_of<double, false>(m, 1), m->d_recv_slots, m->n_recv, src, m->d_maxabs);
  } else {
    if (m->layout == TSG_LAYOUT_SOA)
      halo_unpack<float, true><<<g, 256, 0, s>>>(coords_of<float, true>(m, 0), coords_of<float, true>(m, 1), m->d_recv_slots, m->n_recv, src, m->d_maxabs);
    else
      halo_unpack<float, false><<<g, 256, 0, s>>>(coords_of<float, false>(m, 0), coords_of<float, false>(m, 1), m->d_recv_slots, m->n_recv, src, m->d_maxabs);
  }
  TSG_LAUNCHED();
  TSG_CUDA(cudaStreamSynchronize(s));
  return TSG_OK;
}

// ---- peer-memory partitioned driver (tsg_peer.cuh) ----

tsg_status tsg_peer_local(tsg_mesh* m, void** buf0, void** buf1, void** sync, int64_t* nv) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if (!m->d_peer_sync) {
    TSG_CUDA(cudaMalloc(&m->d_peer_sync, sizeof(tsg::PeerSync)));
    TSG_CUDA(cudaMemset(m->d_peer_sync, 0, sizeof(tsg::PeerSync)));
    m->bytes += sizeof(tsg::PeerSync);
  }
  if (buf0) *buf0 = m->buf[0];
  if (buf1) *buf1 = m->buf[1];
  if (sync) *sync = m->d_peer_sync;
  if (nv) *nv = m->hm.nv;
  return TSG_OK;
}

tsg_status tsg_mesh_slots(tsg_mesh* m, const int64_t* ids, int64_t n, int64_t* slots_out) {
  TSG_LOCK_MESH(m);
  if (!m || n < 0 || (n > 0 && (!ids || !slots_out))) return fail(TSG_ERR_INVALID, "bad arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if (tsg_status st = ensure_host_rows(m)) return st;
  for (int64_t i = 0; i < n; ++i) {
    if (ids[i] < 0 || ids[i] >= m->hm.nv) return fail(TSG_ERR_INVALID, "vertex id out of range");
    slots_out[i] = m->hm.rank[ids[i]];
  }
  return TSG_OK;
}

tsg_status tsg_peer_setup(tsg_mesh* m, int32_t rank, int32_t world, void* const* peer_buf0, void* const* peer_buf1,
                          void* const* peer_sync, const int64_t* peer_nv, int64_t n_push, const int32_t* push_peer,
                          const int64_t* push_src_ids, const int64_t* push_dst_slots) {
  TSG_LOCK_MESH(m);
  if (!m || world < 2 || world > tsg::kMaxPeers || rank < 0 || rank >= world || !peer_buf0 || !peer_buf1 ||
      !peer_sync || !peer_nv || n_push < 0 || (n_push > 0 && (!push_peer || !push_src_ids || !push_dst_slots)))
    return fail(TSG_ERR_INVALID, "bad peer setup arguments");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  tsg_status st = tsg_peer_local(m, nullptr, nullptr, nullptr, nullptr);
  if (st) return st;
  if ((st = ensure_host_rows(m))) return st;
  if (peer_sync[rank] != m->d_peer_sync || peer_buf0[rank] != m->buf[0] || peer_buf1[rank] != m->buf[1])
    return fail(TSG_ERR_INVALID, "the rank's own entry must be its tsg_peer_local pointers");
  std::vector<tsg::PeerEntry> tab(world);
  for (int r = 0; r < world; ++r) {
    if (!peer_buf0[r] || !peer_buf1[r] || !peer_sync[r] || peer_nv[r] < 0)
      return fail(TSG_ERR_INVALID, "missing peer mapping");
    tab[r] = tsg::PeerEntry{static_cast<tsg::PeerSync*>(peer_sync[r]), peer_buf0[r], peer_buf1[r], peer_nv[r]};
  }
  // Split the plan: tile rows (valence 1..31) are pushed by tile_update itself right after their
  // local store (per-slot CSR + bitmask); longer rows by peer_push after the side kernels;
  // pinned vertices never change, so their halo copies stay as set_coords left them.
  const int64_t nv = m->hm.nv;
  std::vector<int32_t> pp;
  std::vector<uint32_t> src, dst;
  std::vector<uint32_t> fcnt(nv + 1, 0), fmask((nv + 31) / 32, 0);
  std::vector<std::pair<uint32_t, uint32_t>> fent(n_push);  // (slot, entry index) of tile rows
  int64_t nf = 0;
  for (int64_t i = 0; i < n_push; ++i) {
    const int32_t q = push_peer[i];
    if (q < 0 || q >= world || q == rank) return fail(TSG_ERR_INVALID, "push peer out of range");
    if (push_src_ids[i] < 0 || push_src_ids[i] >= nv) return fail(TSG_ERR_INVALID, "push source out of range");
    if (push_dst_slots[i] < 0 || push_dst_slots[i] >= peer_nv[q]) return fail(TSG_ERR_INVALID, "push slot out of range");
    const uint32_t sl = static_cast<uint32_t>(m->hm.rank[push_src_ids[i]]);
    const uint32_t deg = m->hm.off[sl + 1] - m->hm.off[sl];
    if (deg == 0) continue;
    if (deg <= static_cast<uint32_t>(tsg::kMaxCycleDeg)) {
      fent[nf++] = {sl, static_cast<uint32_t>(i)};
      ++fcnt[sl + 1];
      fmask[sl >> 5] |= 1u << (sl & 31);
    } else {
      pp.push_back(q);
      src.push_back(sl);
      dst.push_back(static_cast<uint32_t>(push_dst_slots[i]));
    }
  }
  for (int64_t v = 0; v < nv; ++v) fcnt[v + 1] += fcnt[v];
  std::vector<uint32_t> fpeer(nf), fdst(nf), fpos(fcnt.begin(), fcnt.end() - 1);
  for (int64_t k = 0; k < nf; ++k) {
    const uint32_t sl = fent[k].first, i = fent[k].second;
    const uint32_t at = fpos[sl]++;
    fpeer[at] = static_cast<uint32_t>(push_peer[i]);
    fdst[at] = static_cast<uint32_t>(push_dst_slots[i]);
  }
  for (void* p : {static_cast<void*>(m->d_peer_tab), static_cast<void*>(m->d_push_peer),
                  static_cast<void*>(m->d_push_src), static_cast<void*>(m->d_push_dst),
                  static_cast<void*>(m->d_fpush_mask), static_cast<void*>(m->d_fpush_off),
                  static_cast<void*>(m->d_fpush_peer), static_cast<void*>(m->d_fpush_dst)})
    cudaFree(p);
  m->d_peer_tab = nullptr;
  m->d_push_peer = nullptr;
  m->d_push_src = m->d_push_dst = nullptr;
  m->d_fpush_mask = m->d_fpush_off = m->d_fpush_peer = m->d_fpush_dst = nullptr;
  int64_t b = 0;
  cudaStream_t s = m->ctx->stream;
  if ((st = upload(&m->d_peer_tab, tab, &b, s))) return st;
  if ((st = upload(&m->d_push_peer, pp, &b, s))) return st;
  if ((st = upload(&m->d_push_src, src, &b, s))) return st;
  if ((st = upload(&m->d_push_dst, dst, &b, s))) return st;
  if ((st = upload(&m->d_fpush_mask, fmask, &b, s))) return st;
  if ((st = upload(&m->d_fpush_off, fcnt, &b, s))) return st;
  if ((st = upload(&m->d_fpush_peer, fpeer, &b, s))) return st;
  if ((st = upload(&m->d_fpush_dst, fdst, &b, s))) return st;
  TSG_CUDA(cudaStreamSynchronize(s));
  m->n_push = static_cast<int64_t>(pp.size());
  m->peer_rank = rank;
  m->peer_world = world;
  m->gc.reset();
  return TSG_OK;
}

tsg_status tsg_peer_prepare(tsg_mesh* m, const tsg_smooth_cfg* c) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  tsg_status st = validate_cfg(c);
  if (st) return st;
  if (m->peer_world < 2) return fail(TSG_ERR_INVALID, "tsg_peer_setup first");
  if (c->form != TSG_FORM_A) return fail(TSG_ERR_INVALID, "the peer-memory partitioned driver runs Form A");
  TSG_CUDA(cudaSetDevice(m->ctx->device));
  if ((st = peer_graph(m, c))) return st;
  TSG_CUDA(cudaStreamSynchronize(m->ctx->stream));
  return TSG_OK;
}

tsg_status tsg_peer_clear(tsg_mesh* m) {
  TSG_LOCK_MESH(m);
  if (!m) return fail(TSG_ERR_INVALID, "null mesh");
  m->peer_world = 0;
  m->n_push = 0;
  m->gc.reset();
  return TSG_OK;
}

tsg_status tsg_ipc_handle(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return fail(TSG_ERR_INVALID, "null argument");
  cudaIpcMemHandle_t h;
  TSG_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof h == TSG_IPC_HANDLE_BYTES, "cudaIpcMemHandle_t size");
  std::memcpy(handle_out, &h, sizeof h);
  return TSG_OK;
}

tsg_status tsg_ipc_open(tsg_context* ctx, const void* handle, void** dev_ptr_out) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || !handle || !dev_ptr_out) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(ctx->device));
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof h);
  TSG_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return TSG_OK;
}

tsg_status tsg_ipc_close(tsg_context* ctx, void* dev_ptr) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || !dev_ptr) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(ctx->device));
  TSG_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return TSG_OK;
}

// Test hook: builds the layout both ways and names the first HostMesh array that differs.
tsg_status tsg_debug_layout_check(tsg_context* ctx, const tsg_mesh_desc* d, char* mismatch, int32_t cap) {
  TSG_LOCK_CTX(ctx);
  if (!ctx || !d || !mismatch || cap < 1) return fail(TSG_ERR_INVALID, "null argument");
  TSG_CUDA(cudaSetDevice(ctx->device));
  tsg::HostMesh H, D;
  int num_sms = 0;
  TSG_CUDA(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, ctx->device));
  const int32_t tile = choose_tile(d->nv, num_sms, d->precision == TSG_F64 ? 8 : 4);
  if (tile < 0) return fail(TSG_ERR_INVALID, "TSG_TILE must be one of 768, 1024, 1280");
  std::string err = tsg::build_host_mesh(*d, kTiers, H, tile);
  if (!err.empty()) return fail(TSG_ERR_INVALID, "host: " + err);
  tsg::DeviceLayout L;
  err = tsg::build_device_layout(ctx->stream, *d, kTiers, D, L, tile);
  if (err.empty()) err = tsg::download_layout(ctx->stream, L, D);
  tsg::free_layout(L);
  if (!err.empty()) return fail(TSG_ERR_CUDA, "device: " + err);
  std::string bad;
  auto cmp = [&](const char* name, const auto& a, const auto& b2) {
    if (bad.empty() && a != b2) bad = name;
  };
  cmp("order", H.order, D.order);
  cmp("rank", H.rank, D.rank);
  cmp("tri_order", H.tri_order, D.tri_order);
  cmp("off", H.off, D.off);
  cmp("nbr", H.nbr, D.nbr);
  cmp("fan", H.fan, D.fan);
  cmp("fan16", H.fan16, D.fan16);
  cmp("vinc_off", H.vinc_off, D.vinc_off);
  cmp("vinc", H.vinc, D.vinc);
  cmp("tri", H.tri, D.tri);
  cmp("medium", H.medium, D.medium);
  cmp("hubs", H.hubs, D.hubs);
  cmp("large", H.large, D.large);
  cmp("tmeta", H.tmeta, D.tmeta);
  cmp("tile_rec", H.tile_rec, D.tile_rec);
  cmp("ext_off", H.ext_off, D.ext_off);
  cmp("ext", H.ext, D.ext);
  cmp("trec", H.trec, D.trec);
  if (bad.empty() && H.tile != D.tile) bad = "tile";
  if (bad.empty() && (H.max_ext != D.max_ext || H.max_rec_words != D.max_rec_words || H.max_deg != D.max_deg))
    bad = "scalars";
  std::snprintf(mismatch, static_cast<size_t>(cap), "%s", bad.c_str());
  return TSG_OK;
}

}  // extern "C"

// Timeline instrumentation readout (TSG_TRACE builds only; see tsg_kernels.cuh).
extern "C" tsg_status tsg_debug_trace(void* out, int64_t bytes) {
#ifdef TSG_TRACE
  if (!out || bytes < 0 || static_cast<size_t>(bytes) > sizeof(tsg::g_trace)) return fail(TSG_ERR_INVALID, "bad trace buffer");
  TSG_CUDA(cudaMemcpyFromSymbol(out, tsg::g_trace, static_cast<size_t>(bytes)));
  return TSG_OK;
#else
  (void)out;
  (void)bytes;
  return fail(TSG_ERR_INVALID, "built without TSG_TRACE");
#endif
}
