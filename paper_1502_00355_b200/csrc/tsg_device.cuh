// Device-side building blocks of the Smart Laplacian node update (sm_100a).
//
// Bit-exactness contract (fp64): every floating-point operation below is an explicit
// round-to-nearest intrinsic (__dadd_rn / __dsub_rn / __dmul_rn / __ddiv_rn / __dsqrt_rn),
// which nvcc never contracts into FMA, in the operand order of the reference
// (proj/include/trismooth/quality.hpp:15-23, smoothing.hpp:70-81, :103-105).  The
// reference binary contains no FMA (x86-64 baseline), so this reproduces its
// results bit for bit.  The fp32 instantiation uses the same formulas in float.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "tsg_layout.hpp"

namespace tsg {

template <typename R>
struct Arith;

template <>
struct Arith<double> {
  using R2 = double2;
  static constexpr double kAlpha = 3.4641016151377544;  // 2 * 1.7320508075688772935, exact
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double mul(double a, double b) { return __dmul_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ __forceinline__ static double sqrt(double a) { return __dsqrt_rn(a); }
  __device__ __forceinline__ static double2 make(double x, double y) { return make_double2(x, y); }
};

template <>
struct Arith<float> {
  using R2 = float2;
  static constexpr float kAlpha = 3.4641016151377544f;
  __device__ __forceinline__ static float add(float a, float b) { return __fadd_rn(a, b); }
  __device__ __forceinline__ static float sub(float a, float b) { return __fsub_rn(a, b); }
  __device__ __forceinline__ static float mul(float a, float b) { return __fmul_rn(a, b); }
  __device__ __forceinline__ static float div(float a, float b) { return __fdiv_rn(a, b); }
  __device__ __forceinline__ static float sqrt(float a) { return __fsqrt_rn(a); }
  __device__ __forceinline__ static float2 make(float x, float y) { return make_float2(x, y); }
};

// Coordinates of one buffer.  AoS: interleaved (x, y) pairs, one 8/16-byte vector load per
// vertex.  SoA: x[] then y[] in one allocation (y at base + nv).
template <typename R, bool kSoA>
struct Coords {
  using R2 = typename Arith<R>::R2;
  R* base;
  int64_t nv;
  __device__ __forceinline__ R2 load(int64_t i) const {
    if constexpr (kSoA) {
      return Arith<R>::make(__ldg(base + i), __ldg(base + nv + i));
    } else {
      return __ldg(reinterpret_cast<const R2*>(base) + i);
    }
  }
  // L2-coherent read (ld.global.cg) of a value another CTA of the same launch published.
  __device__ __forceinline__ R2 load_cg(int64_t i) const {
    if constexpr (kSoA) {
      return Arith<R>::make(__ldcg(base + i), __ldcg(base + nv + i));
    } else {
      return __ldcg(reinterpret_cast<const R2*>(base) + i);
    }
  }
  // Read of a buffer that other CTAs of the same launch may be writing (Form B fresh reads
  // happen only across launches, so plain loads are enough; no __ldg on mutable data).
  __device__ __forceinline__ R2 load_mut(int64_t i) const {
    if constexpr (kSoA) {
      return Arith<R>::make(base[i], base[nv + i]);
    } else {
      return reinterpret_cast<const R2*>(base)[i];
    }
  }
  __device__ __forceinline__ void store(int64_t i, R2 v) const {
    if constexpr (kSoA) {
      base[i] = v.x;
      base[nv + i] = v.y;
    } else {
      reinterpret_cast<R2*>(base)[i] = v;
    }
  }
};

// α of the triangle that has vertex v at position k (0..2) and the other two vertices
// a = t[(k+1)%3], b = t[(k+2)%3].  dab = b - a and its squares are shared between the
// pass-start and hypothetical evaluations.  Differences are re-signed exactly
// (RN(x - y) = -RN(y - x)), so the (ax, ay, bx, by, cx, cy) of triangle_alpha is a signed
// permutation of (a - v, b - v, b - a):
//   k = 0: (p1,p2,p3) = (v,a,b): A =  a-v, B =  b-v, C =  b-a
//   k = 1: (p1,p2,p3) = (b,v,a): A = -(b-v), B = -(b-a), C = a-v
//   k = 2: (p1,p2,p3) = (a,b,v): A =  b-a, B = -(a-v), C = -(b-v)
// and the edge-square sum keeps the reference's left-to-right order A, B, C.
template <typename R>
__device__ __forceinline__ R alpha_at(int k, R vx, R vy, R ax, R ay, R bx, R by, R dabx, R daby,
                                      R sabx, R saby) {
  using O = Arith<R>;
  const R dax = O::sub(ax, vx), day = O::sub(ay, vy);
  const R dbx = O::sub(bx, vx), dby = O::sub(by, vy);
  const R sax = O::mul(dax, dax), say = O::mul(day, day);
  const R sbx = O::mul(dbx, dbx), sby = O::mul(dby, dby);
  R ta, es;
  if (k == 0) {
    ta = O::sub(O::mul(dax, dby), O::mul(day, dbx));
    es = O::add(O::add(O::add(O::add(O::add(sax, say), sbx), sby), sabx), saby);
  } else if (k == 1) {
    ta = O::sub(O::mul(dbx, daby), O::mul(dby, dabx));
    es = O::add(O::add(O::add(O::add(O::add(sbx, sby), sabx), saby), sax), say);
  } else {
    ta = O::sub(O::mul(daby, dax), O::mul(dabx, day));
    es = O::add(O::add(O::add(O::add(O::add(sabx, saby), sax), say), sbx), sby);
  }
  if (es == R(0)) return R(0);
  return O::div(O::mul(Arith<R>::kAlpha, ta), es);
}

// triangle_alpha(p1, p2, p3) literally (quality.hpp:15-23).
template <typename R>
__device__ __forceinline__ R alpha_plain(R x1, R y1, R x2, R y2, R x3, R y3) {
  using O = Arith<R>;
  const R ax = O::sub(x2, x1), ay = O::sub(y2, y1);
  const R bx = O::sub(x3, x1), by = O::sub(y3, y1);
  const R cx = O::sub(x3, x2), cy = O::sub(y3, y2);
  const R ta = O::sub(O::mul(ax, by), O::mul(ay, bx));
  const R es = O::add(O::add(O::add(O::add(O::add(O::mul(ax, ax), O::mul(ay, ay)), O::mul(bx, bx)),
                                    O::mul(by, by)),
                             O::mul(cx, cx)),
                      O::mul(cy, cy));
  if (es == R(0)) return R(0);
  return O::div(O::mul(Arith<R>::kAlpha, ta), es);
}

// Reciprocal for the fast α path: the SFU estimate refined by two Newton steps
// (relative error ~2^-52; FMA is fine here, the value is only compared against a guard band).
template <int kSteps>
__device__ __forceinline__ double rcp_refined(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
#pragma unroll
  for (int i = 0; i < kSteps; ++i) {
    const double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
  }
  return r;
}
template <int kSteps>
__device__ __forceinline__ float rcp_refined(float x) {
  return __frcp_rn(x);
}

// Reciprocal for the rotation fast path: the SFU estimate (relative error e0 ~ 2^-22) refined by
// one cubic step r' = r + r(e + e^2), e = 1 - x r  (error ~e0^3 plus a few roundings; 3 FMA
// instead of the 4 of two Newton steps).  tsg_selftest_alpha_cycle measures the result.
__device__ __forceinline__ double rcp_cubic(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}
__device__ __forceinline__ float rcp_cubic(float x) { return __frcp_rn(x); }

// Decisions whose fast-path margin is within kGuard (absolute; |α| <= 1) are settled exactly.
constexpr double kGuard = 0x1p-45;
// Guard of the rotation (cycle) fast path, in α/K units (u = 2^-53).  With A = a - v, B = b - v,
// C = b - a (real), X = A x B, S = |A|^2 + |B|^2 + |C|^2, τ = X / S (|τ| <= 1/K = 0.2887):
//  * fast value t = RN(cp * rcp(es)): the numerator cp = fma(pAx, pBy, -RN(pAy pBx)) of the rounded
//    offsets is within 3u|A||B| + u|X| <= 2uS of X; the denominator es = (lp_a + lp_b) + lab is
//    within 7uS of S (4u per squared offset length, u(6|C|^2 + |A|^2 + |B|^2) for |b-a|^2 formed
//    from the offsets, two additions); rcp_cubic is within 1.01u; one final product:
//    |t - τ| <= 2u + |τ| (7u + 1.01u + u) <= 4.6u;
//  * the reference's α/K = RN(RN(K ta) / es_r) / K (quality.hpp:15-23): ta within 2uS, es_r within
//    8uS (six squares of rounded differences, five additions), two roundings:
//    |α_ref/K - τ| <= 2u + 10u |τ| <= 4.9u;
//  * minima are 1-Lipschitz, so each of thr and hyp is known to 9.5u and hyp - thr to 19u (plus
//    0.3u for forming thr ± guard).  kGuardCycle = 2^-48 = 32u leaves a factor 1.66;
//    tsg_selftest_alpha_cycle measures the per-triangle |t - α_ref/K| on the device (max 1.95u
//    over 2^24 random and near-degenerate triangles at 2^-30..2^30 scales, bound 9.5u).
constexpr double kGuardCycle = 0x1p-48;
constexpr double kExactOnlyAbove = 0x1p500;

// triangle_alpha with the division replaced by the refined reciprocal; everything before the
// division is the reference's exact operation sequence.  A degenerate triangle (es == 0 or a
// denormal es flushed to zero) yields NaN / inf, which callers detect and settle exactly.
template <typename R, int kSteps = 2>
__device__ __forceinline__ R alpha_fast(R x1, R y1, R x2, R y2, R x3, R y3) {
  using O = Arith<R>;
  const R ax = O::sub(x2, x1), ay = O::sub(y2, y1);
  const R bx = O::sub(x3, x1), by = O::sub(y3, y1);
  const R cx = O::sub(x3, x2), cy = O::sub(y3, y2);
  const R ta = O::sub(O::mul(ax, by), O::mul(ay, bx));
  const R es = O::add(O::add(O::add(O::add(O::add(O::mul(ax, ax), O::mul(ay, ay)), O::mul(bx, bx)),
                                    O::mul(by, by)),
                             O::mul(cx, cx)),
                      O::mul(cy, cy));
  return O::mul(O::mul(Arith<R>::kAlpha, ta), rcp_refined<kSteps>(es));
}

// std::min(best, x) (== x < best ? x : best), NaN-compatible with the reference.
template <typename R>
__device__ __forceinline__ R min_ref(R best, R x) {
  return x < best ? x : best;
}

// Fan record: neighbour-list positions of a and b, and v's position k in the triangle.
__host__ __device__ __forceinline__ uint32_t fan_pack(uint32_t i1, uint32_t i2, uint32_t k) {
  return i1 | (i2 << 15) | (k << 30);
}
__device__ __forceinline__ uint32_t fan_i1(uint32_t f) { return f & 0x7fffu; }
__device__ __forceinline__ uint32_t fan_i2(uint32_t f) { return (f >> 15) & 0x7fffu; }
__device__ __forceinline__ int fan_k(uint32_t f) { return static_cast<int>(f >> 30); }
// Small-vertex fan record: ring positions of p1, p2, p3 (5 bits each; kMaxDeg = v itself).
__device__ __forceinline__ uint32_t fan_p(uint32_t f, int c) { return (f >> (5 * c)) & 31u; }

constexpr int kMaxInvDeg = 32;
  // 1/deg table (thread-per-vertex tiers)

constexpr uint32_t kFreshBit = 0x80000000u;  // Form B: read this neighbour from N (live)

// Pass-loop state shared by the node kernels and the finalize kernel.
struct PassState {
  int32_t pass;  // index of the pass being executed
  int32_t done;  // 1 once a stop rule fired
  int32_t stop;  // TSG_STOP_*
  int32_t pad;
};

}  // namespace tsg
