// sm_100a kernels of one Smart Laplacian pass.
//
//   node_update  thread per vertex (deg <= kMaxDeg): gather the one-ring into a per-thread
//                shared-memory slice (entry-major, conflict-free), ordered neighbour sum,
//                pass-start threshold and hypothetical min α over the fan, strict accept,
//                write, block-reduced {accepted, max displacement}.
//                Reference: smooth_range / neighbor_mean / min_alpha_at
//                (proj/include/trismooth/smoothing.hpp:70-109, quality.hpp:54-64).
//   hub_update   CTA per high-valence vertex (the paper's CDP child launches, PAPER.md:334-341,
//                replaced by cooperative threads): shared-memory staged one-ring, one thread
//                does the ordered sum while the CTA evaluates the fan, block min-reduction.
//   tri_alpha    thread per triangle (refresh_tri_alphas, quality.hpp:68-74): the TwoPhase
//                field and the final write-back.
//   vertex_min   thread per vertex (reduce_vertex_minima, quality.hpp:78-89).
//   finalize     1 thread: the stop rule in the reference's order (smoothing.cpp:132-141),
//                sets the WHILE-graph condition.
#pragma once

#include <type_traits>

#include "tsg_device.cuh"

namespace tsg {

// Timeline instrumentation (build with EXTRA_NVFLAGS=-DTSG_TRACE; tools/trace_cfg3.py): per
// CTA / warp start time, duration and SM of the tile and side kernels in pass kTracePass.
#ifdef TSG_TRACE
constexpr int kTracePass = 20;
constexpr int kTraceMax = 65536;
__device__ unsigned long long g_trace[3][kTraceMax][2];
__device__ __forceinline__ unsigned long long trace_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned trace_smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}
#define TSG_TRACE_BEGIN(pass, id) \
  const unsigned long long trace_t0 = trace_now(); \
  const bool trace_on = (pass) == kTracePass && (id) < kTraceMax;
#define TSG_TRACE_END(k, id, leader)                                                   \
  if (trace_on && (leader)) {                                                          \
    g_trace[k][id][0] = trace_t0;                                                      \
    g_trace[k][id][1] = ((trace_now() - trace_t0) << 8) | trace_smid();                \
  }
#define TSG_TRACE_SYNC() __syncthreads()
#else
#define TSG_TRACE_BEGIN(pass, id)
#define TSG_TRACE_END(k, id, leader)
#define TSG_TRACE_SYNC()
#endif

constexpr int kNodeBlock = 128;
constexpr int kHubBlock = 256;
#ifndef TSG_HUB_FAST_BLOCK
#define TSG_HUB_FAST_BLOCK 128
#endif
constexpr int kHubFastBlock = TSG_HUB_FAST_BLOCK;  // hub_fast_update CTA size (128: -0.8 % pass time vs 256, measured)

enum { kStopMaxIters = 0, kStopDisplacement = 1, kStopNoMoves = 2 };
enum { kSwapPingPong = 0, kSwapCopy = 1 };

template <typename R, bool kSoA>
struct PassArgs {
  Coords<R, kSoA> buf0, buf1;   // ping-pong pair; copy mode: buf0 = live, buf1 = snapshot
  int32_t swap;
  const uint32_t* off;          // nv+1, compact CSR over slots (rows only for movable vertices)
  const uint32_t* nbr;          // slots, ascending ORIGINAL id (| kFreshBit for Form B)
  const uint32_t* fan;          // hub fan records (i1, i2, k), same offsets as nbr
  const uint16_t* fan16;        // small-vertex fan records (p1, p2, p3 ring positions)
  const uint32_t* vinc_off;     // TwoPhase: incident-triangle CSR over slots
  const uint32_t* vinc;
  const R* alpha;               // TwoPhase: pass-start α field (device triangle order)
  const int32_t* list;          // phase node list (nullptr = slots [0, count))
  int64_t count;
  PassState* st;
  int32_t* slot_acc;            // [pass][kStatSlots] partial accepted counts
  unsigned long long* slot_md;  // [pass][kStatSlots] partial max displacement bits
                                // (non-negative doubles order as u64)
  int8_t* decision;             // optional: 1 accept / 0 reject per slot
  unsigned long long* rare;     // optional diagnostics: [16] |hyp-thr| histogram, [16 + pass] near-ties
  const unsigned long long* maxabs;  // bits of max |coordinate| (set_coords / halo_unpack); at or
                                     // above kExactOnlyAbove every decision is taken exactly
};

template <typename R, bool kSoA>
__device__ __forceinline__ void select_buffers(const PassArgs<R, kSoA>& a, int pass,
                                               Coords<R, kSoA>& P, Coords<R, kSoA>& N) {
  if (a.swap == kSwapCopy || (pass & 1)) {
    P = a.buf1;
    N = a.buf0;
  } else {
    P = a.buf0;
    N = a.buf1;
  }
}

// A block-uniform value every thread reads from device memory (the pass state), broadcast from
// lane 0 so that the compiler sees a warp-uniform branch: an early return it must treat as
// divergent leaves the block barriers after it reached by divergent warps (undefined for the
// .aligned barrier of __syncthreads; compute-sanitizer synccheck).  All lanes active.
__device__ __forceinline__ int warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }

__device__ __forceinline__ bool exact_only(const unsigned long long* maxabs) {
  return *maxabs >= static_cast<unsigned long long>(__double_as_longlong(kExactOnlyAbove));
}

// Per-pass statistics are accumulated into kStatSlots spread slots (one pair per warp, slot
// chosen by the warp's global index) so that no block barrier and no single hot address sits
// on the critical path; finalize_pass folds the slots into the per-pass totals.
constexpr int kStatSlots = 32;

__device__ __forceinline__ void commit_stats_warp(int accepted, double disp, int32_t* acc_slots,
                                                  unsigned long long* md_slots) {
  const int lane = threadIdx.x & 31;
  accepted = __reduce_add_sync(0xffffffffu, accepted);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) disp = fmax(disp, __shfl_xor_sync(0xffffffffu, disp, o));
  if (lane == 0 && (accepted || disp > 0.0)) {
    const unsigned slot = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) & (kStatSlots - 1);
    if (accepted) atomicAdd(acc_slots + slot, accepted);
    if (disp > 0.0) atomicMax(md_slots + slot, static_cast<unsigned long long>(__double_as_longlong(disp)));
  }
}

// Thread-per-vertex node update.  Shared memory: (kMaxDeg + 1) x kNodeBlock coordinate pairs,
// entry-major so that lane t of every warp hits bank group t regardless of the entry it reads
// (the fan indexes entries at random).  Entry kMaxDeg is v itself: the pass-start position for
// the threshold, the candidate for the hypothetical.  A small-vertex fan record holds the ring
// positions of (p1, p2, p3) of the triangle (5 bits each), so every α is the literal
// triangle_alpha(p1, p2, p3) with no per-triangle branching.
//
// fp64 decisions are exact but division-light: α is first evaluated with a refined
// reciprocal (|error| < 2^-50 on |α| <= 1); the strict test hyp > thr is settled from those
// values whenever they are more than kGuard apart, and otherwise (rare: near-ties) every α of
// the vertex is re-evaluated with IEEE division, exactly as the reference (quality.hpp:15-23).
template <typename R, bool kSoA, bool kFormB, bool kTwoPhase, int kMaxDeg, int kBlock>
__global__ void __launch_bounds__(kBlock, kBlock == 128 ? 8 : 4) node_update(PassArgs<R, kSoA> a) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr int kSelf = kMaxDeg;
  constexpr bool kExact = sizeof(R) == 8;
  __shared__ R2 ring[(kMaxDeg + 1) * kBlock];
  __shared__ uint16_t fan_s[kMaxDeg * kBlock];
  const int tid = threadIdx.x;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kBlock + tid;

  // Topology loads do not depend on the pass state: issue them before waiting for it.
  int64_t s = 0;
  uint32_t o0 = 0;
  int deg = 0;
  if (i < a.count) {
    s = a.list ? static_cast<int64_t>(a.list[i]) : i;
    o0 = a.off[s];
    deg = static_cast<int>(a.off[s + 1] - o0);
    if (deg > kMaxDeg) deg = 0;  // hub: handled by hub_update
  }
  const PassState* st = a.st;
  const int2 state = *reinterpret_cast<const int2*>(st);  // {pass, done}
  const uint32_t* nb = a.nbr + o0;
  const uint16_t* fan = a.fan16 + o0;

  int accepted = 0;
  double disp = 0.0;
  R2 pv{}, cand{};
  R sx = R(0), sy = R(0);
  uint32_t fresh = 0;
  Coords<R, kSoA> P, N;
  // Gather in batches of 8 (ids + fan records, then coordinates: independent loads in
  // flight), ordered accumulation of the neighbour sum (Form A).
#pragma unroll
  for (int base = 0; base < kMaxDeg; base += 8) {
    if (base < deg) {
      uint32_t u[8];
      uint16_t f[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        u[j] = (base + j < deg) ? __ldg(nb + base + j) : 0u;
        f[j] = (base + j < deg) ? __ldg(fan + base + j) : uint16_t{0};
      }
      if (base == 0) {
        if (state.y) return;  // stop rule fired (stream driver); uniform across the block
        select_buffers(a, state.x, P, N);
        pv = P.load(s);
      }
      R2 c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (base + j < deg) c[j] = P.load(u[j] & ~kFreshBit);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (base + j < deg) {
          ring[(base + j) * kBlock + tid] = c[j];
          fan_s[(base + j) * kBlock + tid] = f[j];
          if constexpr (kFormB) {
            if (u[j] & kFreshBit) fresh |= 1u << (base + j);
          } else {
            sx = O::add(sx, c[j].x);
            sy = O::add(sy, c[j].y);
          }
        }
      }
    }
  }
  if (deg == 0) {
    if (state.y) return;
    select_buffers(a, state.x, P, N);
  }
  const int pass = state.x;
  if (deg > 0) {
    auto at = [&](uint32_t idx) -> R2 { return ring[idx * kBlock + tid]; };
    auto fan_at = [&](int j) -> uint32_t { return fan_s[j * kBlock + tid]; };
    // Fast α of fan triangle j.  fp64: NaN / inf (degenerate triangle) poisons `nan_acc` and
    // the decision falls back to exact evaluation; fp32: degenerate gives 0 as the reference.
    auto fast = [&](int j) -> R {
      const uint32_t f = fan_at(j);
      const R2 q1 = at(fan_p(f, 0)), q2 = at(fan_p(f, 1)), q3 = at(fan_p(f, 2));
      return alpha_fast<R>(q1.x, q1.y, q2.x, q2.y, q3.x, q3.y);
    };
    R nan_acc = R(0);

    // Threshold: pass-start minimum incident α (TwoPhase: the stored field, already exact).
    ring[kSelf * kBlock + tid] = pv;
    R thr = R(INFINITY);
    if constexpr (kTwoPhase) {
      const uint32_t t0 = a.vinc_off[s], t1 = a.vinc_off[s + 1];
      for (uint32_t t = t0; t < t1; ++t) thr = min_ref(thr, a.alpha[a.vinc[t]]);
    } else if constexpr (kFormB) {
      // (Form A fused evaluates the threshold inside the hypothetical sweep below.)
#pragma unroll 4
      for (int j = 0; j < deg; ++j) {
        R q = fast(j);
        if constexpr (!kExact) q = isfinite(q) ? q : R(0);
        nan_acc = O::add(nan_acc, q);
        thr = fmin(thr, q);
      }
    }
    bool view_moved = false;  // Form B: some fresh neighbour differs from its pass-start value
    if constexpr (kFormB) {
      // ChunkView (quality.hpp:40-50): in-chunk lower-id neighbours read this pass's values.
      uint32_t m = fresh;
      while (m) {
        const int j = __ffs(m) - 1;
        m &= m - 1;
        const R2 now = N.load_mut(nb[j] & ~kFreshBit);
        const R2 was = at(j);
        view_moved |= (now.x != was.x) || (now.y != was.y);
        ring[j * kBlock + tid] = now;
      }
      for (int j = 0; j < deg; ++j) {
        const R2 c = at(j);
        sx = O::add(sx, c.x);
        sy = O::add(sy, c.y);
      }
    }
    const R inv = O::div(R(1), static_cast<R>(deg));  // 1.0 / deg (smoothing.hpp:78)
    cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
    // Exact tie: candidate == current position and every neighbour read is the pass-start
    // value, so each hypothetical α equals its threshold α bit for bit and the strict test
    // fails.  Common once a region has converged; skips the whole hypothetical evaluation.
    const bool tie = !view_moved && cand.x == pv.x && cand.y == pv.y;
    R hyp = R(INFINITY);
    if constexpr (!kFormB && !kTwoPhase) {
      // Form A, fused: one sweep over the fan evaluates each triangle at the pass-start
      // position and at the candidate.  The ring entries are read from shared memory once and
      // v is swapped for the candidate in registers, halving the shared-memory traffic that
      // bounds this kernel (L1 data-pipe wavefronts, profiles/).  A tie needs neither.
      const int sweep = tie ? 0 : deg;
#pragma unroll 4
      for (int j = 0; j < sweep; ++j) {
        const uint32_t f = fan_at(j);
        const uint32_t i0 = fan_p(f, 0), i1 = fan_p(f, 1), i2 = fan_p(f, 2);
        const R2 q1 = at(i0), q2 = at(i1), q3 = at(i2);
        const R2 c1 = i0 == kSelf ? cand : q1, c2 = i1 == kSelf ? cand : q2, c3 = i2 == kSelf ? cand : q3;
        R t = alpha_fast<R>(q1.x, q1.y, q2.x, q2.y, q3.x, q3.y);
        R h = alpha_fast<R>(c1.x, c1.y, c2.x, c2.y, c3.x, c3.y);
        if constexpr (!kExact) {
          t = isfinite(t) ? t : R(0);
          h = isfinite(h) ? h : R(0);
        }
        nan_acc = O::add(nan_acc, O::add(t, h));
        thr = fmin(thr, t);
        hyp = fmin(hyp, h);
      }
    } else if (!tie) {
      ring[kSelf * kBlock + tid] = cand;
#pragma unroll 4
      for (int j = 0; j < deg; ++j) {
        R q = fast(j);
        if constexpr (!kExact) q = isfinite(q) ? q : R(0);
        nan_acc = O::add(nan_acc, q);
        hyp = fmin(hyp, q);
      }
    }
    const bool bad = exact_only(a.maxabs) || !(fabs(nan_acc) < R(1e30));
    bool acc;
    if (tie) {
      acc = false;
    } else if constexpr (!kExact) {
      acc = hyp > thr;  // fp32: decisions are compared in lockstep with a margin
    } else if (!bad && hyp > thr + R(kGuard)) {
      acc = true;
    } else if (!bad && hyp < thr - R(kGuard)) {
      acc = false;
    } else {
      // Near-tie: the reference's exact values (IEEE division, same operand order), needed only
      // for triangles whose fast value lies within kGuard of the fast minimum: any other
      // triangle is provably above the exact minimum (kGuard >= 2x the fast-path error).  With
      // a non-finite fast value (degenerate triangle) every triangle is evaluated exactly.
      R thr_e = thr;
      if constexpr (!kTwoPhase) {
        thr_e = R(INFINITY);
        for (int j = 0; j < deg; ++j) {
          const uint32_t f = fan_at(j);
          R2 q[3];
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const uint32_t idx = fan_p(f, c);
            q[c] = idx == kSelf ? pv
                   : (kFormB && ((fresh >> idx) & 1u)) ? P.load(nb[idx] & ~kFreshBit) : at(idx);
          }
          if (bad || alpha_fast<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y) <= thr + R(kGuard))
            thr_e = min_ref(thr_e, alpha_plain<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y));
        }
      }
      R hyp_e = R(INFINITY);
      for (int j = 0; j < deg; ++j) {
        const uint32_t f = fan_at(j);
        R2 q[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const uint32_t idx = fan_p(f, c);
          q[c] = idx == kSelf ? cand : at(idx);
        }
        if (bad || alpha_fast<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y) <= hyp + R(kGuard))
          hyp_e = min_ref(hyp_e, alpha_plain<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y));
      }
      acc = hyp_e > thr_e;
    }
    N.store(s, acc ? cand : pv);
    if (acc) {
      accepted = 1;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      disp = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
    }
    if (a.decision) a.decision[s] = acc ? 1 : 0;
  }
  commit_stats_warp(accepted, disp, a.slot_acc + pass * kStatSlots, a.slot_md + pass * kStatSlots);
}

// 1 / deg, the reference's reciprocal (smoothing.hpp:78), folded at compile time (IEEE, same
// value as the run-time division) so the node kernels skip a division subroutine.
struct InvDeg {
  double d[kMaxInvDeg + 1];
  float f[kMaxInvDeg + 1];
};
__constant__ constexpr InvDeg c_inv = [] {
  InvDeg t{};
  for (int i = 1; i <= kMaxInvDeg; ++i) {
    t.d[i] = 1.0 / static_cast<double>(i);
    t.f[i] = 1.0f / static_cast<float>(i);
  }
  return t;
}();
template <typename R>
__device__ __forceinline__ R inv_deg(int deg) {
  if constexpr (sizeof(R) == 8) {
    return c_inv.d[deg];
  } else {
    return c_inv.f[deg];
  }
}

// Per-neighbour quantities of the cycle sweep: q - v at the pass-start position and at the
// candidate, and their squared lengths.  (The outer edge b - a of a triangle is formed from
// the pass-start offsets; its rounding error is covered by kGuardCycle, tsg_device.cuh.)
template <typename R>
struct RingEdge {
  R px, py, cx, cy, lp, lc;
};

// Fast α/K of the triangle (v, a, b) at the pass-start position (first) and at the candidate
// (second) from the two neighbours' ring edges.
template <typename R>
__device__ __forceinline__ void ring_pair(const RingEdge<R>& x, const RingEdge<R>& y, R& tp, R& tc) {
  const R ex = y.px - x.px, ey = y.py - x.py;
  const R lab = fma(ex, ex, ey * ey);
  const R cp = fma(x.px, y.py, -(x.py * y.px));
  const R cc = fma(x.cx, y.cy, -(x.cy * y.cx));
  tp = cp * rcp_cubic(x.lp + y.lp + lab);
  tc = cc * rcp_cubic(x.lc + y.lc + lab);
}

template <typename R>
__device__ __forceinline__ RingEdge<R> ring_edge(typename Arith<R>::R2 q, typename Arith<R>::R2 pv,
                                                 typename Arith<R>::R2 cand) {
  RingEdge<R> e;
  e.px = q.x - pv.x;
  e.py = q.y - pv.y;
  e.cx = q.x - cand.x;
  e.cy = q.y - cand.y;
  e.lp = fma(e.px, e.px, e.py * e.py);
  e.lc = fma(e.cx, e.cx, e.cy * e.cy);
  return e;
}

// Tile arrays (tsg_prep.hpp build_tiles).
#ifndef TSG_TILE_MIN_BLOCKS
#define TSG_TILE_MIN_BLOCKS 3
#endif
constexpr int kTileMinBlocks = TSG_TILE_MIN_BLOCKS;  // 256-thread CTAs per SM the register budget is sized for

// Peer-memory partitions (tsg_peer.cuh): one rank's view of another (mapped pointers).
struct PeerSync;
struct PeerEntry {
  PeerSync* sync;
  void* buf0;
  void* buf1;
  int64_t nv;
};

// The (tile, pass) dataflow launch of tile_flow: items i = (pass p0 + i / ntiles, tile
// i % ntiles) are taken in order from a global counter; done[t] = passes of this launch that
// tile t has completed (st.release.gpu after its stores).
struct TileFlow {
  uint32_t* done;   // ntiles, zeroed before the launch
  uint32_t* next;   // item counter, zeroed before the launch
  int32_t p0, np;
  int64_t ntiles;
};

// Acquire load of a done counter: a value >= need synchronizes-with the producer's release, so
// this thread's later loads of that tile's coordinates see its stores (no separate fence).
__device__ __forceinline__ uint32_t tf_ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long tf_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until *p >= need; a dependency that never arrives (a bug, not a schedule: every CTA is
// co-resident and items are taken in order) traps after ~10 s instead of hanging the device.
__device__ __forceinline__ void tf_wait(const uint32_t* p, uint32_t need) {
  if (tf_ld_acquire(p) >= need) return;
  const unsigned long long t0 = tf_globaltimer();
  for (int k = 1;; ++k) {
    __nanosleep(64);
    if (tf_ld_acquire(p) >= need) return;
    if ((k & 1023) == 0 && tf_globaltimer() - t0 > 10000000000ull) __trap();
  }
}

// Halo stores fused into the tile kernel (peer-memory driver; all null otherwise): right after
// a tile row's new value is stored locally it is stored into every peer whose halo holds the
// vertex, so the exchange overlaps the pass tile by tile instead of following it.
struct TilePush {
  const uint32_t* mask;   // bit (s & 31) of word s >> 5: slot s is in some peer's halo
  const uint32_t* off;    // destinations of slot s: entries off[s] .. off[s+1]-1
  const uint32_t* peer;   // destination rank
  const uint32_t* dst;    // destination slot in that rank's mesh
  const PeerEntry* tab;   // the world's mapped buffers
};

template <typename R, bool kSoA>
__device__ __forceinline__ bool push_to_peers(const TilePush& p, int pass, int64_t s, typename Arith<R>::R2 v) {
  if (!p.mask || !((__ldg(p.mask + (s >> 5)) >> (s & 31)) & 1u)) return false;
  const uint32_t k1 = __ldg(p.off + s + 1);
  for (uint32_t k = __ldg(p.off + s); k < k1; ++k) {
    const PeerEntry e = p.tab[__ldg(p.peer + k)];
    const Coords<R, kSoA> D{static_cast<R*>((pass & 1) ? e.buf0 : e.buf1), e.nv};
    D.store(__ldg(p.dst + k), v);
  }
  return true;
}

struct TileArgs {
  TilePush push;
  const uint32_t* meta;      // per slot: first word | deg << 16 | group stride << 20
  const uint32_t* rec;       // words: row[j] | cycle[j] << 16 (local indices)
  const uint32_t* tile_rec;  // ntiles + 1 (first word of each tile, multiples of 4)
  const uint32_t* ext_off;   // ntiles + 1
  const uint32_t* ext;       // external slots
  int32_t ext_cap;           // external coordinates staged in shared memory per tile
  int32_t rec_cap;           // words staged in shared memory per tile (multiple of 4)
  int32_t small_max;         // rows with deg <= small_max have v at fan16 position small_max,
  int32_t medium_max;        // the others at medium_max (tsg_prep.cpp)
  int32_t tile;              // slots per tile (HostMesh::tile, <= kTileMax)
  int64_t nv;
  TileFlow flow;             // tile_flow only
};

template <typename R>
__host__ __device__ constexpr size_t tile_smem_bytes(int tile, int ext_cap, int rec_cap) {
  return sizeof(typename Arith<R>::R2) * (tile + ext_cap) + 4 * static_cast<size_t>(rec_cap) +
         4 * static_cast<size_t>(tile);
}

// ---- bulk-copy (TMA) staging helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}
// Global -> shared bulk copy (16-byte aligned, size a multiple of 16), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
// 16-byte (8-byte) asynchronous global -> shared copy (LDGSTS), completed by cp_async_wait_all.
template <int kBytes>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  if constexpr (kBytes == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_addr(dst)), "l"(src), "n"(kBytes) : "memory");
  }
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Shared-memory view of one staged tile.
template <typename R, bool kSoA, bool kStaged>
struct TileView {
  using R2 = typename Arith<R>::R2;
  const R2* pts;
  const uint32_t* words;
  Coords<R, kSoA> P;
  const uint32_t* ext;    // this tile's external slots (global)
  const uint32_t* recg;   // this tile's words (global)
  int32_t ext_cap, rec_cap, tile;
  __device__ __forceinline__ R2 get(uint32_t l) const {
    if constexpr (kStaged) {
      return pts[l];
    } else {
      return l < static_cast<uint32_t>(tile + ext_cap) ? pts[l] : P.load(__ldg(ext + l - tile));
    }
  }
  __device__ __forceinline__ uint32_t word(uint32_t w) const {
    if constexpr (kStaged) {
      return words[w];
    } else {
      return w < static_cast<uint32_t>(rec_cap) ? words[w] : __ldg(recg + w);
    }
  }
};

// Rare paths of tile_update, kept out of line so that their register needs do not shape the
// main loop: the fan-record sweep of rows without a single link cycle (need_fast) and the
// exact near-tie decision (quality.hpp:15-23 literal evaluation of the triangles whose fast
// value lies within kGuard of the fast minimum; all of them when a fast value is not finite).
template <typename R, bool kSoA, bool kStaged>
__device__ __noinline__ bool tile_decide_rare(const TileView<R, kSoA, kStaged>& tv, const uint16_t* fan, uint32_t kSelf,
                                              uint32_t w0, uint32_t stride, int deg, typename Arith<R>::R2 pv,
                                              typename Arith<R>::R2 cand, R thr, R hyp, bool bad, bool need_fast) {
  using R2 = typename Arith<R>::R2;
  constexpr bool kExact = sizeof(R) == 8;
  constexpr R kInvK = R(1) / Arith<R>::kAlpha;
  auto corners = [&](uint32_t f, R2* q, R2* c) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const uint32_t p = fan_p(f, k);
      q[k] = p == kSelf ? pv : tv.get(tv.word(w0 + p * stride) & kLocalMask);
      c[k] = p == kSelf ? cand : q[k];
    }
  };
  if (need_fast) {
    R nan_acc = R(0);
    thr = hyp = R(INFINITY);
    for (int j = 0; j < deg; ++j) {
      R2 q[3], c[3];
      corners(__ldg(fan + j), q, c);
      R tq = alpha_fast<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y) * kInvK;
      R th = alpha_fast<R>(c[0].x, c[0].y, c[1].x, c[1].y, c[2].x, c[2].y) * kInvK;
      if constexpr (!kExact) {
        tq = isfinite(tq) ? tq : R(0);
        th = isfinite(th) ? th : R(0);
      }
      nan_acc = fma(tq, th, nan_acc);
      thr = min_ref(thr, tq);
      hyp = min_ref(hyp, th);
    }
    bad = bad || !(fabs(nan_acc) < R(1e30));
    if constexpr (!kExact) return hyp > thr;
    if (!bad && hyp > thr + R(kGuard)) return true;
    if (!bad && hyp < thr - R(kGuard)) return false;
  }
  R thr_e = R(INFINITY), hyp_e = R(INFINITY);
  for (int j = 0; j < deg; ++j) {
    R2 q[3], c[3];
    corners(__ldg(fan + j), q, c);
    if (bad || alpha_fast<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y) * kInvK <= thr + R(kGuard))
      thr_e = min_ref(thr_e, alpha_plain<R>(q[0].x, q[0].y, q[1].x, q[1].y, q[2].x, q[2].y));
    if (bad || alpha_fast<R>(c[0].x, c[0].y, c[1].x, c[1].y, c[2].x, c[2].y) * kInvK <= hyp + R(kGuard))
      hyp_e = min_ref(hyp_e, alpha_plain<R>(c[0].x, c[0].y, c[1].x, c[1].y, c[2].x, c[2].y));
  }
  return hyp_e > thr_e;
}

#ifndef TSG_SUM_UNROLL
#define TSG_SUM_UNROLL 4
#endif
#ifndef TSG_CYC_UNROLL
#define TSG_CYC_UNROLL 1
#endif
constexpr int kSumUnroll = TSG_SUM_UNROLL;
constexpr int kCycUnroll = TSG_CYC_UNROLL;

// Tile-staged thread-per-vertex Form A fused update (small tier, deg <= kMaxDeg).
//
// One CTA owns kSlots consecutive slots (a Hilbert-compact patch, degree-sorted inside).  It
// stages in shared memory the patch's pass-start coordinates, the rows' words and the per-slot
// meta words with bulk copies (TMA, one mbarrier), and the coordinates of the external slots
// its rows reference with asynchronous 16-byte copies; after one barrier every gather is a
// shared-memory read.  Word j of a row = (row[j], cycle[j]) local indices: row[] in ascending
// ORIGINAL id (the summation order of neighbor_mean, smoothing.hpp:72-80), cycle[] the directed
// link cycle (every incident triangle is a rotation of (v, cycle[j], cycle[j+1])).  Rows of one
// valence are stored entry-major, so the lanes of a (degree-uniform) warp read word j of
// consecutive rows without bank conflicts.
//
// Decisions: every incident triangle of an interior manifold vertex is a rotation of (v, a, b)
// for consecutive entries a -> b of its link cycle, so one sweep around the cycle visits each
// triangle once and computes each neighbour's offsets from v (pass-start and candidate) and
// their squared lengths once: α/K = ((a-v) x (b-v)) / (|a-v|^2 + |b-v|^2 + |b-a|^2) for both
// positions of v (the reference's triangle_alpha, quality.hpp:15-23, is rotation invariant in
// exact arithmetic).  This fast filter settles hyp > thr whenever the two minima are more than
// kGuardCycle apart (error analysis in tsg_device.cuh); near-ties are collected per tile and
// decided afterwards with the reference's literal arithmetic, one warp per vertex; rows without
// a single link cycle take tile_decide_rare (fan records).
// kStaged: every tile's external coordinates and words fit the shared-memory caps.
// kSlots: slots per tile (= t.tile; a compile-time constant, measured 3% faster than a runtime
// tile size on cfg3).
// kFlow: one item of tile_flow (tile `tile`, pass `pass`): waits for the pass-1 results of the
// tiles it reads, loads coordinates through L2 (ld.cg) and publishes done[tile] at the end;
// otherwise the tile is blockIdx.x and the pass comes from the device pass state.
template <typename R, bool kSoA, int kThreads, int kMaxDeg, bool kStaged, int kSlots, bool kFlow>
__device__ __forceinline__ void tile_item(const PassArgs<R, kSoA>& a, const TileArgs& t, const int tile, int pass,
                                          const int it) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  static_assert(!kFlow || kStaged, "the dataflow launch stages every tile");
  static_assert(kSlots % kThreads == 0 && kSlots <= kTileMax, "whole vertices per thread");
  extern __shared__ __align__(16) unsigned char tile_smem[];
  __shared__ uint64_t bar;
  __shared__ int16_t q_s[kSlots];  // this tile's near-tie vertices (tile-local index)
  __shared__ int qn_s;
  constexpr int kT = kSlots;
  R2* pts = reinterpret_cast<R2*>(tile_smem);
  uint32_t* words = reinterpret_cast<uint32_t*>(pts + kT + t.ext_cap);
  uint32_t* meta_s = words + t.rec_cap;

  const int tid = threadIdx.x;
  const int64_t base = static_cast<int64_t>(tile) * kT;
  const int n_in = static_cast<int>(t.nv - base < kT ? t.nv - base : kT);
  // The pass state (which coordinate buffer is current) is read in parallel with the tile's
  // parity-independent records; only the coordinate copies wait for it.
  int2 state;
  if constexpr (kFlow)
    state = make_int2(pass, 0);
  else
    state = *reinterpret_cast<const int2*>(a.st);
  const uint32_t e0 = __ldg(t.ext_off + tile), ne = __ldg(t.ext_off + tile + 1) - e0;
  const uint32_t r0 = __ldg(t.tile_rec + tile), nr = __ldg(t.tile_rec + tile + 1) - r0;
  const int n_ext = static_cast<int>(kStaged || ne < static_cast<uint32_t>(t.ext_cap) ? ne : t.ext_cap);
  const int n_rec = static_cast<int>(kStaged || nr < static_cast<uint32_t>(t.rec_cap) ? nr : t.rec_cap);
  // Bulk copies: full AoS tiles (coordinates and meta are then 16-byte multiples); the rest
  // (SoA, the partial last tile) goes through the load/store units.
  const bool bulk = !kSoA && n_in == kT;
  if (tid == 0) {
    qn_s = 0;
    if (kFlow && it > 0)  // the previous item's barrier completed (and was waited on) before its end
      asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_addr(&bar)) : "memory");
    mbar_init(&bar, 1);
    if (bulk) {
      mbar_expect_tx(&bar, kT * sizeof(R2) + kT * 4u + 4u * n_rec);
      bulk_g2s(meta_s, t.meta + base, kT * 4u, &bar);
      if (n_rec > 0) bulk_g2s(words, t.rec + r0, 4u * n_rec, &bar);
    }
  }
  // External slot indices (up to kExtRegs per thread; larger rings take a second loop).
  constexpr int kExtRegs = 2;
  uint32_t eidx[kExtRegs];
#pragma unroll
  for (int j = 0; j < kExtRegs; ++j) {
    const int k = tid + j * kThreads;
    eidx[j] = k < n_ext ? __ldg(t.ext + e0 + k) : 0u;
  }
  Coords<R, kSoA> P, N;
  select_buffers(a, state.x, P, N);
  pass = state.x;
  auto load = [&](int64_t i) {
    if constexpr (kFlow)
      return P.load_cg(i);
    else
      return P.load(i);
  };
  const uint32_t need = static_cast<uint32_t>(pass - t.flow.p0);  // (kFlow)
  if constexpr (kFlow) {
    // Pass `pass` reads the pass-1 results of this tile and of the tiles owning its external
    // slots (and overwrites the buffer their pass-1 reads used): each thread waits, with acquire
    // loads, for the producers of what it copies.
    if (need > 0) {
      tf_wait(t.flow.done + tile, need);
#pragma unroll
      for (int j = 0; j < kExtRegs; ++j)
        if (tid + j * kThreads < n_ext) tf_wait(t.flow.done + eidx[j] / kSlots, need);
      for (int k = tid + kExtRegs * kThreads; k < n_ext; k += kThreads)
        tf_wait(t.flow.done + __ldg(t.ext + e0 + k) / kSlots, need);
    }
    if (tid == 0) asm volatile("fence.proxy.async.global;" ::: "memory");  // generic stores -> bulk reads
  }
  TSG_TRACE_BEGIN(pass, blockIdx.x)
  if (bulk && tid == 0) bulk_g2s(pts, P.base + 2 * base, kT * sizeof(R2), &bar);
  if (!bulk) {
    for (int i = tid; i < n_in; i += kThreads) {
      pts[i] = load(base + i);
      meta_s[i] = __ldg(t.meta + base + i);
    }
    const uint4* src = reinterpret_cast<const uint4*>(t.rec + r0);
    uint4* dst = reinterpret_cast<uint4*>(words);
    for (int k = tid; k < n_rec / 4; k += kThreads) dst[k] = __ldg(src + k);
  }
#pragma unroll
  for (int j = 0; j < kExtRegs; ++j) {
    const int k = tid + j * kThreads;
    if (k < n_ext) {
      if constexpr (kSoA)
        pts[kT + k] = load(eidx[j]);
      else
        cp_async<sizeof(R2)>(pts + kT + k, reinterpret_cast<const R2*>(P.base) + eidx[j]);
    }
  }
  for (int k = tid + kExtRegs * kThreads; k < n_ext; k += kThreads) {
    if constexpr (kSoA)
      pts[kT + k] = load(__ldg(t.ext + e0 + k));
    else
      cp_async<sizeof(R2)>(pts + kT + k, reinterpret_cast<const R2*>(P.base) + __ldg(t.ext + e0 + k));
  }
  if constexpr (!kSoA) cp_async_wait_all();
  __syncthreads();  // also publishes the mbarrier initialisation
  if (bulk) mbar_wait(&bar, 0);
  if constexpr (!kFlow) {
    if (state.y) return;  // (after the copies into this CTA's shared memory have landed)
  }

  const TileView<R, kSoA, kStaged> tv{pts, words, P, t.ext + e0, t.rec + r0, t.ext_cap, t.rec_cap, kT};
  const bool xonly = exact_only(a.maxabs);
  int8_t* const decision = a.decision;
  int accepted = 0;
  double disp = 0.0;
  bool pushed = false;

  // One vertex of the tile (local index i).
  auto vertex = [&](int i, uint32_t meta) {
    const int deg = static_cast<int>((meta >> kMetaDegShift) & kMetaDegMask);
    const uint32_t w0 = meta & kMetaBaseMask, stride = meta >> kMetaStrideShift;
    const R2 pv = pts[i];
    // neighbor_mean (smoothing.hpp:72-80): ordered chain over row[] (ascending original id).
    R sx = R(0), sy = R(0);
    {
      uint32_t w = w0;
#pragma unroll kSumUnroll
      for (int j = 0; j < deg; ++j, w += stride) {
        const R2 c = tv.get(tv.word(w) & kLocalMask);
        sx = O::add(sx, c.x);
        sy = O::add(sy, c.y);
      }
    }
    const R inv = inv_deg<R>(deg);
    const R2 cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
    const int64_t s = base + i;
    bool acc = false;
    // Exact tie (candidate == position; Form A reads only pass-start values): every
    // hypothetical α equals its threshold α bit for bit, the strict test fails.
    if (!(cand.x == pv.x && cand.y == pv.y)) {
      const uint32_t l0 = (tv.word(w0) >> kWordCycleShift) & kLocalMask;
      R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
      const bool cyc = l0 != kNoLocal;
      if (cyc) {
        auto tri = [&](const RingEdge<R>& x, const RingEdge<R>& y) {
          R tp, tc;
          ring_pair<R>(x, y, tp, tc);
          if constexpr (!kExact) {
            tp = isfinite(tp) ? tp : R(0);
            tc = isfinite(tc) ? tc : R(0);
          }
          nan_acc = fma(tp, tc, nan_acc);  // any non-finite value poisons the accumulator
          thr = min_ref(thr, tp);
          hyp = min_ref(hyp, tc);
        };
        auto edge_at = [&](uint32_t w) {
          return ring_edge<R>(tv.get((tv.word(w) >> kWordCycleShift) & kLocalMask), pv, cand);
        };
        // Around the cycle two triangles per iteration with the two edge variables swapping
        // roles (no loop-carried register copies); the closing triangle recomputes the first
        // edge instead of keeping it live.
        RingEdge<R> ea = ring_edge<R>(tv.get(l0), pv, cand);
        uint32_t w = w0 + stride;
        int j = 1;
#pragma unroll kCycUnroll
        for (; j + 2 <= deg; j += 2, w += 2 * stride) {
          const RingEdge<R> eb = edge_at(w);
          tri(ea, eb);
          ea = edge_at(w + stride);
          tri(eb, ea);
        }
        if (j < deg) {
          const RingEdge<R> eb = edge_at(w);
          tri(ea, eb);
          tri(eb, ring_edge<R>(tv.get(l0), pv, cand));
        } else {
          tri(ea, ring_edge<R>(tv.get(l0), pv, cand));
        }
      }
      const bool bad = xonly || !(fabs(nan_acc) < R(1e30));
      if (cyc && !kExact) {
        acc = hyp > thr;  // fp32: decisions are compared in lockstep with a margin
      } else if (cyc && !bad && hyp > thr + R(kGuardCycle)) {
        acc = true;
      } else if (cyc && !bad && hyp < thr - R(kGuardCycle)) {
        acc = false;
      } else if (cyc) {
        // Near-tie (or a degenerate triangle): decided exactly after the sweep of the whole
        // tile, by full warps instead of one divergent lane here.
        q_s[atomicAdd(&qn_s, 1)] = static_cast<int16_t>(i);
        if (a.rare) {  // diagnostics: histogram of log2 |hyp - thr| (bins 0..15 = 2^-60..2^-45)
          const double dd = fabs(static_cast<double>(hyp - thr));
          int b = dd > 0.0 ? ilogb(dd) + 60 : 0;
          b = b < 0 ? 0 : b > 15 ? 15 : b;
          atomicAdd(a.rare + b, 1ull);
        }
        return;
      } else {
        const uint32_t self = static_cast<uint32_t>(deg <= t.small_max ? t.small_max : t.medium_max);
        acc = tile_decide_rare<R, kSoA, kStaged>(tv, a.fan16 + __ldg(a.off + s), self, w0, stride, deg, pv, cand, thr,
                                                 hyp, bad, true);
      }
    }
    N.store(s, acc ? cand : pv);
    pushed |= push_to_peers<R, kSoA>(t.push, pass, s, acc ? cand : pv);
    if (acc) {
      ++accepted;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      disp = d > disp ? d : disp;
    }
    if (decision) decision[s] = acc ? 1 : 0;
  };

  // (Fully unrolled per-valence variants of `vertex` were measured slower: their code size
  // thrashes the instruction cache — stall_no_inst became the top stall.)
#pragma unroll 1
  for (int i = tid; i < n_in; i += kThreads) {
    const uint32_t meta = meta_s[i];
    if (((meta >> kMetaDegShift) & kMetaDegMask) == 0) continue;  // pinned, or a row of another tier
    vertex(i, meta);
  }
  // Exact decisions of the tile's near-ties, from the staged tile, one warp per vertex (lane j
  // evaluates triangle j): the reference's arithmetic throughout — ordered neighbour sum,
  // literal triangle_alpha with IEEE division for every incident triangle at the pass-start
  // position and at the candidate (quality.hpp:15-23, :54-64, through alpha_at with the
  // triangle's rotation k from the row words), strict test.  The minimum of finite values is
  // order-free, so the shuffle reduction equals the reference's sequential std::min.
  __syncthreads();
  const int qn = qn_s;
  if (qn > 0 && tid == 0 && a.rare) atomicAdd(a.rare + 16 + pass, static_cast<unsigned long long>(qn));
  const int lane = tid & 31;
#pragma unroll 1
  for (int e = tid >> 5; e < qn; e += kThreads / 32) {
    const int i = q_s[e];
    const uint32_t meta = meta_s[i];
    const int deg = static_cast<int>((meta >> kMetaDegShift) & kMetaDegMask);
    const uint32_t w0 = meta & kMetaBaseMask, stride = meta >> kMetaStrideShift;
    const R2 pv = pts[i];
    R sx = R(0), sy = R(0);
    for (int j = 0; j < deg; ++j) {
      const R2 c = tv.get(tv.word(w0 + j * stride) & kLocalMask);
      sx = O::add(sx, c.x);
      sy = O::add(sy, c.y);
    }
    const R inv = inv_deg<R>(deg);
    const R2 cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
    R thr = R(INFINITY), hyp = R(INFINITY);
    if (lane < deg) {
      const uint32_t wa = tv.word(w0 + lane * stride);
      const uint32_t wb = tv.word(w0 + (lane + 1 < deg ? lane + 1 : 0) * stride);
      const R2 qa = tv.get((wa >> kWordCycleShift) & kLocalMask), qb = tv.get((wb >> kWordCycleShift) & kLocalMask);
      const int k = static_cast<int>(wa >> kWordRotShift);
      const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
      const R sabx = O::mul(dabx, dabx), saby = O::mul(daby, daby);
      thr = alpha_at<R>(k, pv.x, pv.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby);
      hyp = alpha_at<R>(k, cand.x, cand.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      thr = min_ref(thr, __shfl_xor_sync(0xffffffffu, thr, o));
      hyp = min_ref(hyp, __shfl_xor_sync(0xffffffffu, hyp, o));
    }
    if (lane == 0) {
      const bool acc = hyp > thr;
      const int64_t s = base + i;
      N.store(s, acc ? cand : pv);
      pushed |= push_to_peers<R, kSoA>(t.push, pass, s, acc ? cand : pv);
      if (acc) {
        ++accepted;
        const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
        const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
        disp = d > disp ? d : disp;
      }
      if (a.decision) a.decision[s] = acc ? 1 : 0;
    }
  }
  commit_stats_warp(accepted, disp, a.slot_acc + pass * kStatSlots, a.slot_md + pass * kStatSlots);
  if (pushed) __threadfence_system();  // peer stores before the pass barrier's release (peer_sync)
  TSG_TRACE_SYNC();
  TSG_TRACE_END(0, blockIdx.x, tid == 0)
  if constexpr (kFlow) {
    __syncthreads();  // every store of the item (and every shared-memory read) is done
    if (tid == 0) {
      // Release by one thread after the barrier: cumulative over the CTA's stores (they happen
      // before it through bar.sync), so no full fence is needed (measured: cfg2 +3 %, fp32 +6 %).
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(t.flow.done + tile), "r"(need + 1) : "memory");
    }
  }
}

template <typename R, bool kSoA, int kThreads, int kMaxDeg, bool kStaged, int kSlots>
__global__ void __launch_bounds__(kThreads, kTileMinBlocks) tile_update(PassArgs<R, kSoA> a, TileArgs t) {
  tile_item<R, kSoA, kThreads, kMaxDeg, kStaged, kSlots, false>(a, t, static_cast<int>(blockIdx.x), 0, 0);
}

// Form A passes [p0, p0 + np) as a dataflow over (tile, pass) items in one cooperative launch:
// a CTA takes the next item from a global counter, so pass p + 1 starts on the tiles whose
// neighbourhood has finished pass p while the last tiles of pass p are still running — no wave
// tail and no launch per pass.  Progress: every CTA is co-resident and items are taken in
// (pass, tile) order, so the earliest unfinished item only depends on finished ones.  Each
// vertex still reads pass-start values only (same arithmetic as tile_update, bit-identical).
template <typename R, bool kSoA, int kThreads, int kMaxDeg, int kSlots>
__global__ void __launch_bounds__(kThreads, kTileMinBlocks) tile_flow(PassArgs<R, kSoA> a, TileArgs t) {
  __shared__ int next_s[2];
  const int64_t total = static_cast<int64_t>(t.flow.np) * t.flow.ntiles;
  int64_t item = blockIdx.x;
  for (int it = 0; item < total; ++it) {
    if (threadIdx.x == 0) next_s[it & 1] = static_cast<int>(atomicAdd(t.flow.next, 1u) + gridDim.x);
    const int pass = t.flow.p0 + static_cast<int>(item / t.flow.ntiles);
    const int tile = static_cast<int>(item % t.flow.ntiles);
    tile_item<R, kSoA, kThreads, kMaxDeg, true, kSlots, true>(a, t, tile, pass, it);  // ends with a barrier
    item = next_s[it & 1];
  }
}

// Warp per vertex, Form A fused, for rows above the cycle tiers (valence 16 .. any): the
// paper's CDP child launch for high-valence nodes becomes the 32 lanes of
// one warp.  Lanes gather the row (ascending original id) into the warp's shared-memory slice
// (entries beyond kCap are re-read from global memory / L2), every lane then forms the ordered
// neighbour sum from the slice (broadcast reads, uniform control flow), lanes sweep the fan
// records with the fast α/K filter for both positions of v, and a shuffle reduction gives the
// warp-uniform decision.  Near-ties are settled with the reference's exact α (alpha_at).
template <typename R, bool kSoA, int kCap>
__device__ __forceinline__ void warp_row(const PassArgs<R, kSoA>& a, const Coords<R, kSoA>& P,
                                         const Coords<R, kSoA>& N, int pass, int64_t s,
                                         typename Arith<R>::R2* ring) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  const int lane = threadIdx.x & 31;
  const uint32_t o0 = __ldg(a.off + s);
  const int deg = static_cast<int>(__ldg(a.off + s + 1) - o0);
  const uint32_t* nb = a.nbr + o0;
  const uint32_t* fan = a.fan + o0;
  const R2 pv = P.load(s);

  // neighbor_mean (smoothing.hpp:72-80): one ordered chain, computed redundantly by all lanes
  // from the shared-memory slice.  Rows longer than kCap are summed chunk by chunk (each chunk
  // gathered in parallel); the first chunk stays resident for the fan sweep, entries beyond
  // it are re-read from global memory there (parallel across lanes).
  R sx = R(0), sy = R(0);
  for (int c0 = 0; c0 < deg; c0 += kCap) {
    const int n = deg - c0 < kCap ? deg - c0 : kCap;
    if (c0 > 0) __syncwarp();
#pragma unroll 4
    for (int j = lane; j < n; j += 32) ring[j] = P.load(__ldg(nb + c0 + j));
    __syncwarp();
#pragma unroll 8
    for (int j = 0; j < n; ++j) {
      const R2 c = ring[j];
      sx = O::add(sx, c.x);
      sy = O::add(sy, c.y);
    }
  }
  if (deg > kCap) {  // restore the first chunk for the sweep
    __syncwarp();
#pragma unroll 4
    for (int j = lane; j < kCap; j += 32) ring[j] = P.load(__ldg(nb + j));
    __syncwarp();
  }
  auto get = [&](int j) -> R2 { return j < kCap ? ring[j] : P.load(__ldg(nb + j)); };
  const R inv = deg <= kMaxInvDeg ? inv_deg<R>(deg) : O::div(R(1), static_cast<R>(deg));
  const R2 cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
  const bool tie = cand.x == pv.x && cand.y == pv.y;  // warp-uniform

  bool acc = false;
  if (!tie) {
    R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
#pragma unroll 2
    for (int j = lane; j < deg; j += 32) {
      const uint32_t f = __ldg(fan + j);
      const R2 qa = get(fan_i1(f)), qb = get(fan_i2(f));
      const R ex = qb.x - qa.x, ey = qb.y - qa.y;
      const R lab = fma(ex, ex, ey * ey);
      const R pax = qa.x - pv.x, pay = qa.y - pv.y, pbx = qb.x - pv.x, pby = qb.y - pv.y;
      const R cax = qa.x - cand.x, cay = qa.y - cand.y, cbx = qb.x - cand.x, cby = qb.y - cand.y;
      const R ep = fma(pax, pax, pay * pay) + fma(pbx, pbx, pby * pby) + lab;
      const R ec = fma(cax, cax, cay * cay) + fma(cbx, cbx, cby * cby) + lab;
      R tp = fma(pax, pby, -(pay * pbx)) * rcp_cubic(ep);
      R tc = fma(cax, cby, -(cay * cbx)) * rcp_cubic(ec);
      if constexpr (!kExact) {
        tp = isfinite(tp) ? tp : R(0);
        tc = isfinite(tc) ? tc : R(0);
      }
      nan_acc = nan_acc + (tp + tc);
      thr = fmin(thr, tp);
      hyp = fmin(hyp, tc);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      thr = fmin(thr, __shfl_xor_sync(0xffffffffu, thr, o));
      hyp = fmin(hyp, __shfl_xor_sync(0xffffffffu, hyp, o));
    }
    const bool bad = exact_only(a.maxabs) || __any_sync(0xffffffffu, !(fabs(nan_acc) < R(1e30)));
    if constexpr (!kExact) {
      acc = hyp > thr;
    } else if (!bad && hyp > thr + R(kGuardCycle)) {
      acc = true;
    } else if (!bad && hyp < thr - R(kGuardCycle)) {
      acc = false;
    } else {
      // Near-tie: exact α of every triangle (alpha_at = triangle_alpha in the literal
      // operand order; the minimum of finite values is order-free).
      R thr_e = R(INFINITY), hyp_e = R(INFINITY);
      for (int j = lane; j < deg; j += 32) {
        const uint32_t f = __ldg(fan + j);
        const R2 qa = get(fan_i1(f)), qb = get(fan_i2(f));
        const int k = fan_k(f);
        const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
        const R sabx = O::mul(dabx, dabx), saby = O::mul(daby, daby);
        const R ep = alpha_at<R>(k, pv.x, pv.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby);
        const R ec = alpha_at<R>(k, cand.x, cand.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby);
        thr_e = min_ref(thr_e, ep);
        hyp_e = min_ref(hyp_e, ec);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        thr_e = min_ref(thr_e, __shfl_xor_sync(0xffffffffu, thr_e, o));
        hyp_e = min_ref(hyp_e, __shfl_xor_sync(0xffffffffu, hyp_e, o));
      }
      acc = hyp_e > thr_e;
    }
  }
  int accepted = 0;
  double disp = 0.0;
  if (lane == 0) {
    N.store(s, acc ? cand : pv);
    if (a.decision) a.decision[s] = acc ? 1 : 0;
    if (acc) {
      accepted = 1;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      disp = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
    }
  }
  commit_stats_warp(accepted, disp, a.slot_acc + pass * kStatSlots, a.slot_md + pass * kStatSlots);
}

template <typename R, bool kSoA, int kWarps, int kCap>
__global__ void __launch_bounds__(kWarps * 32) warp_update(PassArgs<R, kSoA> a) {
  using R2 = typename Arith<R>::R2;
  __shared__ R2 ring_s[kWarps * kCap];
  const int w = threadIdx.x >> 5;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * kWarps + w;
  if (idx >= a.count) return;  // warp-uniform
  const int2 state = *reinterpret_cast<const int2*>(a.st);
  if (state.y) return;
  Coords<R, kSoA> P, N;
  select_buffers(a, state.x, P, N);
  TSG_TRACE_BEGIN(state.x, idx)
  warp_row<R, kSoA, kCap>(a, P, N, state.x, a.list[idx], ring_s + w * kCap);
  TSG_TRACE_END(2, idx, (threadIdx.x & 31) == 0)
}

// Rows above the cycle tiers (valence >= 32) as a small persistent kernel that runs BESIDE the
// tile grid for the whole pass: one CTA of kWarps warps per SM at kRegs registers, sized so that
// each SM sub-partition (16 K registers) holds one side warp next to its six tile_update warps
// (6 x 80 x 32 + 32 x 32 = 16 K) — with the maximum shared-memory carveout on both kernels, the
// tile grid keeps its 3 CTAs per SM.  Warps take rows (degree-descending, the longest first)
// from a ticket counter; the last warp to leave resets the counter pair, so a launch leaves it
// zeroed for the next pass.  The 32-register cap spills a little (latency-bound code anyway).
template <typename R, bool kSoA, int kWarps, int kCap, int kRegs>
__global__ void __maxnreg__(kRegs) side_rows(PassArgs<R, kSoA> a, uint32_t* ctr) {
  using R2 = typename Arith<R>::R2;
  __shared__ R2 ring_s[kWarps * kCap];
  const int2 state = *reinterpret_cast<const int2*>(a.st);
  if (state.y) return;
  Coords<R, kSoA> P, N;
  select_buffers(a, state.x, P, N);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll 1
  for (;;) {
    uint32_t row = 0;
    if (lane == 0) row = atomicAdd(ctr, 1u);
    row = __shfl_sync(0xffffffffu, row, 0);
    if (row >= static_cast<uint64_t>(a.count)) break;
    TSG_TRACE_BEGIN(state.x, row)
    warp_row<R, kSoA, kCap>(a, P, N, state.x, a.list[row], ring_s + w * kCap);
    TSG_TRACE_END(2, row, lane == 0)
    __syncwarp();
  }
  if (lane == 0 && atomicAdd(ctr + 1, 1u) == gridDim.x * kWarps - 1) {
    ctr[0] = 0;
    ctr[1] = 0;
  }
}

// Fast α/K of the triangle (v, a, b) for one position of v: the rotation formula of the cycle
// sweep (ring_edge / ring_pair, same operation sequence, same error bound).
template <typename R>
__device__ __forceinline__ R rot_fast(typename Arith<R>::R2 qa, typename Arith<R>::R2 qb, typename Arith<R>::R2 v) {
  const R ax = qa.x - v.x, ay = qa.y - v.y, bx = qb.x - v.x, by = qb.y - v.y;
  const R ex = bx - ax, ey = by - ay;
  const R lab = fma(ex, ex, ey * ey);
  const R la = fma(ax, ax, ay * ay), lb = fma(bx, bx, by * by);
  return fma(ax, by, -(ay * bx)) * rcp_cubic(la + lb + lab);
}

// Form B decision of one vertex from staged coordinates (formb_chunk_update, formb_flow):
// sp[j * bs] / sv[j * bs] = pass-start / view value of row entry j, fan records (i1, i2, k).
// Ordered neighbour sum through the view (smoothing.hpp:72-80), threshold at the pass-start
// positions and hypothetical at the candidate with the rotation filter (rot_fast,
// kGuardCycle), near-ties / degenerate triangles with the literal alpha_at (quality.hpp:15-23).
template <typename R>
__device__ __forceinline__ bool formb_decide_staged(typename Arith<R>::R2 pv, int deg, const typename Arith<R>::R2* sp,
                                                    const typename Arith<R>::R2* sv, int bs, const uint32_t* fan,
                                                    bool xonly, typename Arith<R>::R2& cand) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  R sx = R(0), sy = R(0);
  for (int j = 0; j < deg; ++j) {
    const R2 c = sv[j * bs];
    sx = O::add(sx, c.x);
    sy = O::add(sy, c.y);
  }
  const R inv = inv_deg<R>(deg);
  cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
  R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
  for (int j = 0; j < deg; ++j) {
    const uint32_t f = fan[j];
    const int ia = static_cast<int>(fan_i1(f)) * bs, ib = static_cast<int>(fan_i2(f)) * bs;
    R tp = rot_fast<R>(sp[ia], sp[ib], pv), tc = rot_fast<R>(sv[ia], sv[ib], cand);
    if constexpr (!kExact) {
      tp = isfinite(tp) ? tp : R(0);
      tc = isfinite(tc) ? tc : R(0);
    }
    nan_acc = fma(tp, tc, nan_acc);
    thr = min_ref(thr, tp);
    hyp = min_ref(hyp, tc);
  }
  const bool bad = xonly || !(fabs(nan_acc) < R(1e30));
  if constexpr (!kExact) {
    return hyp > thr;
  } else {
    if (!bad && hyp > thr + R(kGuardCycle)) return true;
    if (!bad && hyp < thr - R(kGuardCycle)) return false;
    R thr_e = R(INFINITY), hyp_e = R(INFINITY);
    for (int j = 0; j < deg; ++j) {
      const uint32_t f = fan[j];
      const int ia = static_cast<int>(fan_i1(f)) * bs, ib = static_cast<int>(fan_i2(f)) * bs;
      const int k = fan_k(f);
      {
        const R2 qa = sp[ia], qb = sp[ib];
        const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
        thr_e = min_ref(thr_e, alpha_at<R>(k, pv.x, pv.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, O::mul(dabx, dabx),
                                           O::mul(daby, daby)));
      }
      {
        const R2 qa = sv[ia], qb = sv[ib];
        const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
        hyp_e = min_ref(hyp_e, alpha_at<R>(k, cand.x, cand.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, O::mul(dabx, dabx),
                                           O::mul(daby, daby)));
      }
    }
    return hyp_e > thr_e;
  }
}

// Form B (ChunkView, quality.hpp:40-50; worker_chunk, parallel.hpp:19-24) with one CTA per
// chunk: the CTA walks its chunk's dependency levels in order with a barrier between levels, so a
// whole pass is ONE launch (the level-set schedule needs a launch per level: 195 per pass on the
// 100x100 grid in serial Form B).  Thread per vertex, any valence: neighbour reads through the
// view (in-chunk lower-id neighbours — kFreshBit — from N, written by earlier levels of this
// CTA, the rest from the pass-start buffer P); the threshold at pass-start positions and the
// hypothetical with the rotation filter (rot_fast, kGuardCycle), near-ties / degenerate
// triangles with the reference's literal arithmetic (alpha_at).  Fused and TwoPhase give the same
// thresholds, so both strategies use this kernel.
template <typename R, bool kSoA>
__global__ void __launch_bounds__(256) formb_chunk_update(PassArgs<R, kSoA> a, const int32_t* __restrict__ order,
                                                          const int32_t* __restrict__ lvl_off,
                                                          const int32_t* __restrict__ chunk_lvl,
                                                          const uint32_t* __restrict__ rec) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  constexpr int kRecMaxDeg = 15, kRecWords = 32;
  extern __shared__ __align__(16) uint32_t rbuf[];  // [2][blockDim.x][kRecWords], then the rings
  R2* ring = reinterpret_cast<R2*>(rbuf + 2 * blockDim.x * kRecWords);  // [2 * kRecMaxDeg][blockDim.x]
  const int2 state = *reinterpret_cast<const int2*>(a.st);
  if (warp_uniform(state.y)) return;
  Coords<R, kSoA> P, N;
  select_buffers(a, state.x, P, N);
  const int pass = state.x;
  const bool xonly = exact_only(a.maxabs);
  int accepted = 0;
  double disp = 0.0;
  const int tid = threadIdx.x;

  // One vertex: row / fan entries through the accessors (staged record or global rows).
  auto update = [&](int64_t s, int deg, auto nbr_at, auto fan_at) {
    auto view = [&](uint32_t u) -> R2 { return (u & kFreshBit) ? N.load_mut(u & ~kFreshBit) : P.load(u); };
    const R2 pv = P.load(s);
    R sx = R(0), sy = R(0);
    for (int j = 0; j < deg; ++j) {  // neighbor_mean through the view (smoothing.hpp:72-80)
      const R2 c = view(nbr_at(j));
      sx = O::add(sx, c.x);
      sy = O::add(sy, c.y);
    }
    const R inv = deg <= kMaxInvDeg ? inv_deg<R>(deg) : O::div(R(1), static_cast<R>(deg));
    const R2 cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
    R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
    for (int j = 0; j < deg; ++j) {
      const uint32_t f = fan_at(j);
      const uint32_t ua = nbr_at(fan_i1(f)), ub = nbr_at(fan_i2(f));
      const R2 pa = P.load(ua & ~kFreshBit), pb = P.load(ub & ~kFreshBit);
      const R2 va = (ua & kFreshBit) ? N.load_mut(ua & ~kFreshBit) : pa;
      const R2 vb = (ub & kFreshBit) ? N.load_mut(ub & ~kFreshBit) : pb;
      R tp = rot_fast<R>(pa, pb, pv), tc = rot_fast<R>(va, vb, cand);
      if constexpr (!kExact) {
        tp = isfinite(tp) ? tp : R(0);
        tc = isfinite(tc) ? tc : R(0);
      }
      nan_acc = fma(tp, tc, nan_acc);
      thr = min_ref(thr, tp);
      hyp = min_ref(hyp, tc);
    }
    const bool bad = xonly || !(fabs(nan_acc) < R(1e30));
    bool acc;
    if constexpr (!kExact) {
      acc = hyp > thr;
    } else if (!bad && hyp > thr + R(kGuardCycle)) {
      acc = true;
    } else if (!bad && hyp < thr - R(kGuardCycle)) {
      acc = false;
    } else {
      R thr_e = R(INFINITY), hyp_e = R(INFINITY);
      for (int j = 0; j < deg; ++j) {
        const uint32_t f = fan_at(j);
        const uint32_t ua = nbr_at(fan_i1(f)), ub = nbr_at(fan_i2(f));
        const int k = fan_k(f);
        {
          const R2 qa = P.load(ua & ~kFreshBit), qb = P.load(ub & ~kFreshBit);
          const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
          thr_e = min_ref(thr_e, alpha_at<R>(k, pv.x, pv.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, O::mul(dabx, dabx),
                                             O::mul(daby, daby)));
        }
        {
          const R2 qa = view(ua), qb = view(ub);
          const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
          hyp_e = min_ref(hyp_e, alpha_at<R>(k, cand.x, cand.y, qa.x, qa.y, qb.x, qb.y, dabx, daby,
                                             O::mul(dabx, dabx), O::mul(daby, daby)));
        }
      }
      acc = hyp_e > thr_e;
    }
    N.store(s, acc ? cand : pv);
    if (acc) {
      ++accepted;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      disp = d > disp ? d : disp;
    }
    if (a.decision) a.decision[s] = acc ? 1 : 0;
  };
  // The same decision from staged coordinates: sp / sv = pass-start / view value of row entry j
  // at [j * blockDim.x], fan records from the record.
  auto update_staged = [&](int64_t s, int deg, const R2* sp, const R2* sv, const uint32_t* fan) {
    const R2 pv = P.load(s);
    R2 cand;
    const bool acc = formb_decide_staged<R>(pv, deg, sp, sv, static_cast<int>(blockDim.x), fan, xonly, cand);
    N.store(s, acc ? cand : pv);
    if (acc) {
      ++accepted;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      disp = d > disp ? d : disp;
    }
    if (a.decision) a.decision[s] = acc ? 1 : 0;
  };
  auto update_global = [&](int64_t s) {
    const uint32_t o0 = __ldg(a.off + s);
    const int deg = static_cast<int>(__ldg(a.off + s + 1) - o0);
    const uint32_t* nb = a.nbr + o0;
    const uint32_t* fan = a.fan + o0;
    update(s, deg, [&](int j) { return __ldg(nb + j); }, [&](int j) { return __ldg(fan + j); });
  };

  // The record of the first vertex of each level this thread handles is prefetched one level
  // ahead (asynchronous copies into a double buffer), so only the coordinate reads of a level
  // sit on the level's critical path (narrow levels: serial Form B on small meshes).
  const int l0 = chunk_lvl[blockIdx.x], l1 = chunk_lvl[blockIdx.x + 1];
  auto prefetch = [&](int L) {
    if (L < l1) {
      const int idx = lvl_off[L] + tid;
      if (idx < lvl_off[L + 1]) {
        uint32_t* dst = rbuf + ((L & 1) * blockDim.x + tid) * kRecWords;
        const uint32_t* src = rec + static_cast<int64_t>(idx) * kRecWords;
#pragma unroll
        for (int q = 0; q < kRecWords / 4; ++q) cp_async<16>(dst + 4 * q, src + 4 * q);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  prefetch(l0);
#pragma unroll 1
  for (int L = l0; L < l1; ++L) {
    prefetch(L + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // this level's record has landed
    const int b = lvl_off[L], e = lvl_off[L + 1];
    if (b + tid < e) {
      const uint32_t* r = rbuf + ((L & 1) * blockDim.x + tid) * kRecWords;
      const int deg = static_cast<int>(r[1]);
      if (deg <= kRecMaxDeg) {
        // All neighbour coordinates of the vertex in one batch of independent loads (pass-start
        // and view values) into this thread's slices, then the arithmetic from shared memory.
        R2* sp = ring + tid;                    // entry j at sp[j * blockDim.x]
        R2* sv = ring + kRecMaxDeg * blockDim.x + tid;
#pragma unroll
        for (int base = 0; base < kRecMaxDeg; base += 8) {
          if (base < deg) {
            R2 cp[8], cv[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (base + j < deg) {
                const uint32_t u = r[2 + base + j];
                cp[j] = P.load(u & ~kFreshBit);
                cv[j] = (u & kFreshBit) ? N.load_mut(u & ~kFreshBit) : cp[j];
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
              if (base + j < deg) {
                sp[(base + j) * blockDim.x] = cp[j];
                sv[(base + j) * blockDim.x] = cv[j];
              }
          }
        }
        update_staged(static_cast<int64_t>(r[0]), deg, sp, sv, r + 2 + kRecMaxDeg);
      } else {
        update_global(static_cast<int64_t>(r[0]));
      }
    }
#pragma unroll 1
    for (int idx = b + tid + static_cast<int>(blockDim.x); idx < e; idx += blockDim.x) update_global(order[idx]);
    __syncthreads();  // this level's N writes are read by the next levels of the chunk
  }
  commit_stats_warp(accepted, disp, a.slot_acc + pass * kStatSlots, a.slot_md + pass * kStatSlots);
}

// CTA per hub (Form A fused, valence above the warp tier's staging cap): the paper's CDP child
// launch becomes one CTA.  The row is staged in dynamic shared memory (up to
// `cap` entries, the rest re-read from global memory); warp 0 forms the ordered neighbour sum
// (smoothing.hpp:72-80) while warps 1.. sweep the fan at the pass-start position; then every
// warp sweeps the fan at the candidate; block min-reductions give the decision, near-ties are
// re-evaluated exactly (alpha_at) by the whole CTA.
template <typename R>
struct HubShared {
  typename Arith<R>::R2 cand;
  R min[2][kHubFastBlock / 32];
  int bad;
};

template <typename R, bool kSoA>
__device__ __forceinline__ void hub_row(const PassArgs<R, kSoA>& a, const Coords<R, kSoA>& P,
                                        const Coords<R, kSoA>& N, int pass, int64_t s, int cap,
                                        unsigned slot_key, typename Arith<R>::R2* ring, HubShared<R>& hs) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  constexpr int kWarps = kHubFastBlock / 32;
  R2& s_cand = hs.cand;
  R(&s_min)[2][kWarps] = hs.min;
  int& s_bad = hs.bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t o0 = __ldg(a.off + s);
  const int deg = static_cast<int>(__ldg(a.off + s + 1) - o0);
  const uint32_t* nb = a.nbr + o0;
  const uint32_t* fan = a.fan + o0;
  const int staged = deg < cap ? deg : cap;
  if (tid == 0) s_bad = 0;
#pragma unroll 4
  for (int j = tid; j < staged; j += kHubFastBlock) ring[j] = P.load(__ldg(nb + j));
  __syncthreads();
  auto get = [&](int j) -> R2 { return j < cap ? ring[j] : P.load(__ldg(nb + j)); };
  const R2 pv = P.load(s);

  R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
  if (warp == 0) {
    if (lane == 0) {
      R sx = R(0), sy = R(0);
#pragma unroll 8
      for (int j = 0; j < staged; ++j) {
        const R2 c = ring[j];
        sx = O::add(sx, c.x);
        sy = O::add(sy, c.y);
      }
      for (int j = staged; j < deg; ++j) {
        const R2 c = P.load(__ldg(nb + j));
        sx = O::add(sx, c.x);
        sy = O::add(sy, c.y);
      }
      const R inv = deg <= kMaxInvDeg ? inv_deg<R>(deg) : O::div(R(1), static_cast<R>(deg));
      s_cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
    }
  } else {
    for (int j = tid - 32; j < deg; j += kHubFastBlock - 32) {
      const uint32_t f = __ldg(fan + j);
      R tp = rot_fast<R>(get(fan_i1(f)), get(fan_i2(f)), pv);
      if constexpr (!kExact) tp = isfinite(tp) ? tp : R(0);
      nan_acc = fma(tp, tp, nan_acc);
      thr = min_ref(thr, tp);
    }
  }
  __syncthreads();
  const R2 cand = s_cand;
  const bool tie = cand.x == pv.x && cand.y == pv.y;
  if (!tie) {
    for (int j = tid; j < deg; j += kHubFastBlock) {
      const uint32_t f = __ldg(fan + j);
      R tc = rot_fast<R>(get(fan_i1(f)), get(fan_i2(f)), cand);
      if constexpr (!kExact) tc = isfinite(tc) ? tc : R(0);
      nan_acc = fma(tc, tc, nan_acc);
      hyp = min_ref(hyp, tc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    thr = min_ref(thr, __shfl_xor_sync(0xffffffffu, thr, o));
    hyp = min_ref(hyp, __shfl_xor_sync(0xffffffffu, hyp, o));
  }
  if (__any_sync(0xffffffffu, !(fabs(nan_acc) < R(1e30))) && lane == 0) s_bad = 1;
  if (lane == 0) {
    s_min[0][warp] = thr;
    s_min[1][warp] = hyp;
  }
  __syncthreads();
  thr = s_min[0][0];
  hyp = s_min[1][0];
#pragma unroll
  for (int w = 1; w < kWarps; ++w) {
    thr = min_ref(thr, s_min[0][w]);
    hyp = min_ref(hyp, s_min[1][w]);
  }
  const bool bad = exact_only(a.maxabs) || s_bad != 0;
  bool acc;
  if (tie) {
    acc = false;
  } else if constexpr (!kExact) {
    acc = hyp > thr;
  } else if (!bad && hyp > thr + R(kGuardCycle)) {
    acc = true;
  } else if (!bad && hyp < thr - R(kGuardCycle)) {
    acc = false;
  } else {
    // Near-tie: the reference's literal α of every triangle (alpha_at), CTA-wide minima.
    __syncthreads();  // s_min is reused
    R thr_e = R(INFINITY), hyp_e = R(INFINITY);
    for (int j = tid; j < deg; j += kHubFastBlock) {
      const uint32_t f = __ldg(fan + j);
      const R2 qa = get(fan_i1(f)), qb = get(fan_i2(f));
      const int k = fan_k(f);
      const R dabx = O::sub(qb.x, qa.x), daby = O::sub(qb.y, qa.y);
      const R sabx = O::mul(dabx, dabx), saby = O::mul(daby, daby);
      thr_e = min_ref(thr_e, alpha_at<R>(k, pv.x, pv.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby));
      hyp_e = min_ref(hyp_e, alpha_at<R>(k, cand.x, cand.y, qa.x, qa.y, qb.x, qb.y, dabx, daby, sabx, saby));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      thr_e = min_ref(thr_e, __shfl_xor_sync(0xffffffffu, thr_e, o));
      hyp_e = min_ref(hyp_e, __shfl_xor_sync(0xffffffffu, hyp_e, o));
    }
    if (lane == 0) {
      s_min[0][warp] = thr_e;
      s_min[1][warp] = hyp_e;
    }
    __syncthreads();
    thr_e = s_min[0][0];
    hyp_e = s_min[1][0];
#pragma unroll
    for (int w = 1; w < kWarps; ++w) {
      thr_e = min_ref(thr_e, s_min[0][w]);
      hyp_e = min_ref(hyp_e, s_min[1][w]);
    }
    acc = hyp_e > thr_e;
  }
  if (tid == 0) {
    N.store(s, acc ? cand : pv);
    if (a.decision) a.decision[s] = acc ? 1 : 0;
    if (acc) {
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      const unsigned slot = pass * kStatSlots + (slot_key & (kStatSlots - 1));
      atomicAdd(a.slot_acc + slot, 1);
      if (d > 0.0) atomicMax(a.slot_md + slot, static_cast<unsigned long long>(__double_as_longlong(d)));
    }
  }
}

template <typename R, bool kSoA>
__global__ void __launch_bounds__(kHubFastBlock) hub_fast_update(PassArgs<R, kSoA> a, int cap) {
  using R2 = typename Arith<R>::R2;
  extern __shared__ __align__(16) unsigned char hub_smem[];
  __shared__ HubShared<R> hs;
  const int2 state = *reinterpret_cast<const int2*>(a.st);
  if (warp_uniform(state.y)) return;
  Coords<R, kSoA> P, N;
  select_buffers(a, state.x, P, N);
  TSG_TRACE_BEGIN(state.x, blockIdx.x)
  hub_row<R, kSoA>(a, P, N, state.x, a.list[blockIdx.x], cap, blockIdx.x, reinterpret_cast<R2*>(hub_smem), hs);
  TSG_TRACE_SYNC();
  TSG_TRACE_END(1, blockIdx.x, threadIdx.x == 0)
}

// CTA per high-valence vertex.  Dynamic shared memory: `cap` pass-start pairs followed (Form B)
// by `cap` view pairs; entries beyond cap are read from global memory.
template <typename R, bool kSoA, bool kFormB, bool kTwoPhase>
__global__ void __launch_bounds__(kHubBlock) hub_update(PassArgs<R, kSoA> a, int cap) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  extern __shared__ __align__(16) unsigned char hub_smem[];
  R2* pring = reinterpret_cast<R2*>(hub_smem);
  R2* vring = pring + cap;
  __shared__ R2 s_cand;
  __shared__ R s_thr[kHubBlock / 32], s_hyp[kHubBlock / 32];

  const PassState* st = a.st;
  if (warp_uniform(st->done)) return;
  const int pass = st->pass;
  Coords<R, kSoA> P, N;
  select_buffers(a, pass, P, N);
  const int tid = threadIdx.x;
  const int64_t s = a.list[blockIdx.x];
  const uint32_t o0 = a.off[s];
  const int deg = static_cast<int>(a.off[s + 1] - o0);
  const uint32_t* nb = a.nbr + o0;
  const uint32_t* fan = a.fan + o0;
  const int staged = deg < cap ? deg : cap;

  for (int j = tid; j < staged; j += kHubBlock) {
    const uint32_t u = nb[j];
    const R2 c = P.load(u & ~kFreshBit);
    pring[j] = c;
    if constexpr (kFormB) vring[j] = (u & kFreshBit) ? N.load_mut(u & ~kFreshBit) : c;
  }
  __syncthreads();
  auto pget = [&](int j) -> R2 { return j < cap ? pring[j] : P.load(nb[j] & ~kFreshBit); };
  auto vget = [&](int j) -> R2 {
    if constexpr (kFormB) {
      if (j < cap) return vring[j];
      const uint32_t u = nb[j];
      return (u & kFreshBit) ? N.load_mut(u & ~kFreshBit) : P.load(u);
    } else {
      return pget(j);
    }
  };
  const R2 pv = P.load(s);
  if (tid == 0) {
    // neighbor_mean: ordered, single chain (smoothing.hpp:72-80).
    R sx = R(0), sy = R(0);
#pragma unroll 8
    for (int j = 0; j < deg; ++j) {
      const R2 c = vget(j);
      sx = O::add(sx, c.x);
      sy = O::add(sy, c.y);
    }
    const R inv = O::div(R(1), static_cast<R>(deg));
    s_cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
  }
  R thr = R(INFINITY);
  if constexpr (kTwoPhase) {
    const uint32_t t0 = a.vinc_off[s], t1 = a.vinc_off[s + 1];
    for (uint32_t t = t0 + tid; t < t1; t += kHubBlock) thr = min_ref(thr, a.alpha[a.vinc[t]]);
  } else {
    for (int j = tid; j < deg; j += kHubBlock) {
      const uint32_t f = fan[j];
      const R2 pa = pget(fan_i1(f)), pb = pget(fan_i2(f));
      const R dabx = O::sub(pb.x, pa.x), daby = O::sub(pb.y, pa.y);
      thr = min_ref(thr, alpha_at<R>(fan_k(f), pv.x, pv.y, pa.x, pa.y, pb.x, pb.y, dabx, daby,
                                     O::mul(dabx, dabx), O::mul(daby, daby)));
    }
  }
  __syncthreads();
  const R2 cand = s_cand;
  R hyp = R(INFINITY);
  for (int j = tid; j < deg; j += kHubBlock) {
    const uint32_t f = fan[j];
    const R2 pa = vget(fan_i1(f)), pb = vget(fan_i2(f));
    const R dabx = O::sub(pb.x, pa.x), daby = O::sub(pb.y, pa.y);
    hyp = min_ref(hyp, alpha_at<R>(fan_k(f), cand.x, cand.y, pa.x, pa.y, pb.x, pb.y, dabx, daby,
                                   O::mul(dabx, dabx), O::mul(daby, daby)));
  }
  // Exact min in any order (no NaN on finite input).
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    thr = min_ref(thr, __shfl_xor_sync(0xffffffffu, thr, o));
    hyp = min_ref(hyp, __shfl_xor_sync(0xffffffffu, hyp, o));
  }
  if ((tid & 31) == 0) {
    s_thr[tid >> 5] = thr;
    s_hyp[tid >> 5] = hyp;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kHubBlock / 32; ++w) {
      thr = min_ref(thr, s_thr[w]);
      hyp = min_ref(hyp, s_hyp[w]);
    }
    const bool acc = hyp > thr;
    N.store(s, acc ? cand : pv);
    if (a.decision) a.decision[s] = acc ? 1 : 0;
    if (acc) {
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      const unsigned slot = pass * kStatSlots + (blockIdx.x & (kStatSlots - 1));
      atomicAdd(a.slot_acc + slot, 1);
      if (d > 0.0) atomicMax(a.slot_md + slot, static_cast<unsigned long long>(__double_as_longlong(d)));
    }
  }
}

// α per triangle from the pass-start buffer (or buf0 when st == nullptr).
template <typename R, bool kSoA>
__global__ void __launch_bounds__(256) tri_alpha(Coords<R, kSoA> buf0, Coords<R, kSoA> buf1,
                                                 int32_t swap, const PassState* st,
                                                 const int32_t* __restrict__ tri, int64_t nt,
                                                 R* __restrict__ alpha) {
  Coords<R, kSoA> P = buf0;
  if (st) {
    if (st->done) return;
    if (swap == kSwapCopy || (st->pass & 1)) P = buf1;
  }
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int32_t v0 = __ldg(tri + 3 * t), v1 = __ldg(tri + 3 * t + 1), v2 = __ldg(tri + 3 * t + 2);
    const auto p0 = P.load(v0), p1 = P.load(v1), p2 = P.load(v2);
    alpha[t] = alpha_plain<R>(p0.x, p0.y, p1.x, p1.y, p2.x, p2.y);
  }
}

template <typename R>
__global__ void __launch_bounds__(256) vertex_min(const uint32_t* __restrict__ vinc_off,
                                                  const uint32_t* __restrict__ vinc,
                                                  const R* __restrict__ alpha, int64_t nv,
                                                  double* __restrict__ out) {
  for (int64_t s = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; s < nv;
       s += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint32_t t0 = vinc_off[s], t1 = vinc_off[s + 1];
    if (t0 == t1) {
      out[s] = __longlong_as_double(0x7ff8000000000000LL);  // kUnsetQuality (quiet NaN)
      continue;
    }
    R best = R(INFINITY);
    for (uint32_t t = t0; t < t1; ++t) best = min_ref(best, alpha[vinc[t]]);
    out[s] = static_cast<double>(best);
  }
}

// Order-preserving map double -> u64 for atomic min / max.
__device__ __forceinline__ unsigned long long ordered_key(double d) {
  const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(d));
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

template <typename R>
__global__ void __launch_bounds__(256) alpha_extrema(const R* __restrict__ alpha, int64_t nt,
                                                     unsigned long long* mn, unsigned long long* mx,
                                                     unsigned long long* nonpos) {
  unsigned long long lo = ~0ULL, hi = 0ULL, np = 0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nt;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double q = static_cast<double>(alpha[t]);
    const unsigned long long k = ordered_key(q);
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
    np += q <= 0.0 ? 1 : 0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
    np += __shfl_xor_sync(0xffffffffu, np, o);
  }
  if ((threadIdx.x & 31) != 0) return;
  atomicMin(mn, lo);
  atomicMax(mx, hi);
  if (np) atomicAdd(nonpos, np);
}

// One warp: folds the pass's stat slots into pass_acc / pass_md, then lane 0 applies the
// reference's stop rule and sets the WHILE condition.
__global__ void finalize_pass(PassState* st, const int32_t* slot_acc, const unsigned long long* slot_md,
                              int32_t* pass_acc, unsigned long long* pass_md, double tol_abs,
                              int32_t max_iters, cudaGraphConditionalHandle handle, int32_t use_handle) {
  const int lane = threadIdx.x;
  const int q = st->pass;
  const bool done = st->done != 0;
  int32_t acc = 0;
  unsigned long long mdb = 0;
  if (!done) {
    acc = slot_acc[q * kStatSlots + lane];
    mdb = slot_md[q * kStatSlots + lane];
  }
  acc = __reduce_add_sync(0xffffffffu, acc);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, mdb, o);
    mdb = other > mdb ? other : mdb;
  }
  if (lane != 0) return;
  if (!done) {
    pass_acc[q] = acc;
    pass_md[q] = mdb;
    const double md = __longlong_as_double(static_cast<long long>(mdb));
    st->pass = q + 1;
    if (acc == 0) {
      st->done = 1;
      st->stop = kStopNoMoves;
    } else if (md < tol_abs) {
      st->done = 1;
      st->stop = kStopDisplacement;
    } else if (q + 1 >= max_iters) {
      st->done = 1;
      st->stop = kStopMaxIters;
    }
  }
  if (use_handle) cudaGraphSetConditional(handle, st->done ? 0u : 1u);
}

}  // namespace tsg
