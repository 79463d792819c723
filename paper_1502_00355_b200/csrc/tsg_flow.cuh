// Form B as a dataflow over (vertex, pass): one persistent launch runs many passes with no
// barrier between levels or passes.
//
// The reference's Form B (proj/src/smoothing.cpp:98-120 with the ChunkView of
// proj/include/trismooth/quality.hpp:40-50) is a Gauss-Seidel sweep: inside a chunk, vertex
// v reads this pass's value of every lower-id neighbour.  A level schedule runs that sweep
// pass by pass — serial Form B on the 100 x 100 grid (cfg1) is 195 dependent levels per pass,
// 19,500 per 100 passes.  But pass q+1 of v only needs pass q of its one-ring, not of the whole
// mesh, so passes pipeline like a wavefront: pass q+1 starts in the first rows while pass q is
// still sweeping the last ones.  The critical path of 100 passes on cfg1 is ~500 vertex
// updates instead of 19,500.
//
// Execution.  Every movable vertex has a counter done[s] = passes it has completed in this
// launch (pinned vertices: ~0u).  Vertex s may run pass q (0-based) when
//   done[u] >= q     for every neighbour u   (pass-start values X_q: threshold and view), and
//   done[u] >= q+1   for fresh neighbours    (in-chunk, lower id: X_{q+1} through the view).
// X_k of a vertex lives in buffer (p0 + k) & 1.  Writing X_{q+1}[s] overwrites X_{q-1}[s],
// which no neighbour still needs (they all have done >= q); a neighbour's X_q is not overwritten
// before s finishes pass q (that neighbour's pass q+1 waits for done[s] >= q+1).  So two
// buffers suffice and every read sees exactly the value the reference's sweep reads.
//
// Progress.  Entries are sorted by (level) and dealt round-robin to the threads; a thread runs
// its entries in (pass, level) order.  Every dependency has a strictly smaller (pass, level)
// key (fresh reads: same pass, lower level; pass-start reads: previous pass), so the head entry
// with the smallest key is always ready: no deadlock as long as all threads are resident
// (the launch is sized from the occupancy calculator and made cooperative, which guarantees
// co-residency).  Warps never spin inside a lane: a lane whose head is not ready skips the
// iteration, so the warp stays converged.
//
// Memory ordering.  Coordinates written in the launch are read with L2-coherent loads
// (ld.global.cg); a finished update publishes done[s] with st.release.gpu after its store, a
// reader polls with ld.relaxed.gpu and issues fence.acq_rel.gpu once all its dependencies are
// satisfied, before reading coordinates (PTX memory model: release / observe / fence).
//
// Arithmetic: the decision of formb_chunk_update (tsg_kernels.cuh) — ordered neighbour sum,
// rotation fast filter with the proven kGuardCycle band, literal alpha_at for near-ties — so
// results are bit-identical to the reference (and to the level schedules).
#pragma once

#include "tsg_kernels.cuh"
#include "tsg_prep.hpp"  // record format: kChunkRecWords, kChunkRecMaxDeg

namespace tsg {

constexpr int kFlowBlock = 128;

__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Coordinates of one buffer through L2-coherent accesses (other SMs write them in-launch).
template <typename R, bool kSoA>
struct CoordsCG {
  using R2 = typename Arith<R>::R2;
  R* base;
  int64_t nv;
  __device__ __forceinline__ R2 load(int64_t i) const {
    if constexpr (kSoA) {
      return Arith<R>::make(__ldcg(base + i), __ldcg(base + nv + i));
    } else {
      return __ldcg(reinterpret_cast<const R2*>(base) + i);
    }
  }
  __device__ __forceinline__ void store(int64_t i, R2 v) const {
    if constexpr (kSoA) {
      __stcg(base + i, v.x);
      __stcg(base + nv + i, v.y);
    } else {
      __stcg(reinterpret_cast<R2*>(base) + i, v);
    }
  }
};

template <typename R>
struct FlowArgs {
  R* buf0;
  R* buf1;
  int64_t nv;
  const uint32_t* rec;   // flow-ordered records: slot, valence, then (valence <= kChunkRecMaxDeg)
                         // neighbour slots (| kFreshBit) and fan records; kChunkRecWords words each
  const uint32_t* off;   // rows of larger valence: compact CSR over slots
  const uint32_t* nbr;   // (| kFreshBit)
  const uint32_t* fan;
  uint32_t* done;        // per slot: passes completed in this launch (pinned: ~0u)
  int64_t n;             // movable entries
  int32_t p0;            // global index of the launch's first pass (buffer parity, stat rows)
  int32_t np;            // passes in this launch
  int32_t* slot_acc;     // [pass][kStatSlots]
  unsigned long long* slot_md;
  const unsigned long long* maxabs;
};

// Decision of a row too long for a record (valence > kChunkRecMaxDeg): rows and fan records
// from global memory, coordinates through L2-coherent loads (same arithmetic as
// formb_decide_staged).
template <typename R, bool kSoA>
__device__ __noinline__ bool flow_decide_global(const FlowArgs<R>& f, int64_t s, int deg, typename Arith<R>::R2 pv,
                                                const CoordsCG<R, kSoA>& P, const CoordsCG<R, kSoA>& N, bool xonly,
                                                typename Arith<R>::R2& cand) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  constexpr bool kExact = sizeof(R) == 8;
  const uint32_t o0 = __ldg(f.off + s);
  const uint32_t* nb = f.nbr + o0;
  const uint32_t* fn = f.fan + o0;
  auto view = [&](uint32_t u) -> R2 { return (u & kFreshBit) ? N.load(u & ~kFreshBit) : P.load(u); };
  R sx = R(0), sy = R(0);
  for (int j = 0; j < deg; ++j) {
    const R2 c = view(__ldg(nb + j));
    sx = O::add(sx, c.x);
    sy = O::add(sy, c.y);
  }
  const R inv = deg <= kMaxInvDeg ? inv_deg<R>(deg) : O::div(R(1), static_cast<R>(deg));
  cand = O::make(O::mul(sx, inv), O::mul(sy, inv));
  R thr = R(INFINITY), hyp = R(INFINITY), nan_acc = R(0);
  for (int j = 0; j < deg; ++j) {
    const uint32_t fr = __ldg(fn + j);
    const uint32_t ua = __ldg(nb + fan_i1(fr)), ub = __ldg(nb + fan_i2(fr));
    const R2 pa = P.load(ua & ~kFreshBit), pb = P.load(ub & ~kFreshBit);
    const R2 va = (ua & kFreshBit) ? N.load(ua & ~kFreshBit) : pa;
    const R2 vb = (ub & kFreshBit) ? N.load(ub & ~kFreshBit) : pb;
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
  if constexpr (!kExact) {
    return hyp > thr;
  } else {
    if (!bad && hyp > thr + R(kGuardCycle)) return true;
    if (!bad && hyp < thr - R(kGuardCycle)) return false;
    R thr_e = R(INFINITY), hyp_e = R(INFINITY);
    for (int j = 0; j < deg; ++j) {
      const uint32_t fr = __ldg(fn + j);
      const uint32_t ua = __ldg(nb + fan_i1(fr)), ub = __ldg(nb + fan_i2(fr));
      const int k = fan_k(fr);
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
    return hyp_e > thr_e;
  }
}

// Dynamic shared memory of formb_flow: per thread its current entry's record (kChunkRecWords
// words) and the staged pass-start / view coordinates of a row (entry-major slices).
template <typename R>
constexpr size_t flow_smem_bytes() {
  return static_cast<size_t>(kFlowBlock) * (kChunkRecWords * sizeof(uint32_t) +
                                            2 * kChunkRecMaxDeg * sizeof(typename Arith<R>::R2));
}

template <typename R, bool kSoA>
__global__ void __launch_bounds__(kFlowBlock) formb_flow(FlowArgs<R> f) {
  using O = Arith<R>;
  using R2 = typename O::R2;
  extern __shared__ __align__(16) unsigned char flow_smem[];
  const int tid = threadIdx.x;
  uint32_t* rec_s = reinterpret_cast<uint32_t*>(flow_smem) + tid * kChunkRecWords;
  R2* sp = reinterpret_cast<R2*>(flow_smem + kFlowBlock * kChunkRecWords * sizeof(uint32_t)) + tid;
  R2* sv = sp + kChunkRecMaxDeg * kFlowBlock;
  const int64_t T = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t first = static_cast<int64_t>(blockIdx.x) * blockDim.x + tid;
  const bool xonly = exact_only(f.maxabs);
  const unsigned stat_slot = static_cast<unsigned>(first >> 5) & (kStatSlots - 1);
  int64_t e = first;
  int q = e < f.n ? 0 : f.np;
  int accepted = 0;
  double disp = 0.0;
  bool staged = false;  // rec_s holds entry e's record
  int resume = 0;       // large rows: first entry to re-check

  while (q < f.np) {
    if (!staged) {  // the record of this thread's next entry, 8 x 16 B
      const uint4* src = reinterpret_cast<const uint4*>(f.rec + e * kChunkRecWords);
#pragma unroll
      for (int k = 0; k < kChunkRecWords / 4; ++k) reinterpret_cast<uint4*>(rec_s)[k] = __ldg(src + k);
      staged = true;
    }
    const int64_t s = rec_s[0];
    const int deg = static_cast<int>(rec_s[1]);
    const bool small = deg <= kChunkRecMaxDeg;

    // Dependencies: pass-start values of the whole ring, this pass's values of fresh ones.
    bool ready = true;
    if (small) {
      uint32_t have[kChunkRecMaxDeg];
#pragma unroll
      for (int j = 0; j < kChunkRecMaxDeg; ++j)  // all counters in flight at once
        have[j] = j < deg ? ld_relaxed_gpu(f.done + (rec_s[2 + j] & ~kFreshBit)) : ~0u;
#pragma unroll
      for (int j = 0; j < kChunkRecMaxDeg; ++j) {
        const uint32_t need = (j < deg && (rec_s[2 + j] & kFreshBit)) ? static_cast<uint32_t>(q + 1)
                                                                       : static_cast<uint32_t>(q);
        ready = ready && have[j] >= need;
      }
    } else {
      const uint32_t* nb = f.nbr + __ldg(f.off + s);
      for (int c = 0; c < deg; ++c) {
        const int j = resume + c < deg ? resume + c : resume + c - deg;
        const uint32_t u = __ldg(nb + j);
        const uint32_t need = (u & kFreshBit) ? static_cast<uint32_t>(q + 1) : static_cast<uint32_t>(q);
        if (ld_relaxed_gpu(f.done + (u & ~kFreshBit)) < need) {
          ready = false;
          resume = j;
          break;
        }
      }
    }
    if (!ready) continue;
    resume = 0;
    fence_acq_rel_gpu();

    const int gp = f.p0 + q;
    const CoordsCG<R, kSoA> P{(gp & 1) ? f.buf1 : f.buf0, f.nv}, N{(gp & 1) ? f.buf0 : f.buf1, f.nv};
    const R2 pv = P.load(s);
    R2 cand;
    bool acc;
    if (small) {
      // the whole row in one batch of independent loads, then the decision from shared memory
#pragma unroll
      for (int j = 0; j < kChunkRecMaxDeg; ++j) {
        if (j < deg) {
          const uint32_t u = rec_s[2 + j];
          const R2 c = P.load(u & ~kFreshBit);
          sp[j * kFlowBlock] = c;
          sv[j * kFlowBlock] = (u & kFreshBit) ? N.load(u & ~kFreshBit) : c;
        }
      }
      acc = formb_decide_staged<R>(pv, deg, sp, sv, kFlowBlock, rec_s + 2 + kChunkRecMaxDeg, xonly, cand);
    } else {
      acc = flow_decide_global<R, kSoA>(f, s, deg, pv, P, N, xonly, cand);
    }
    N.store(s, acc ? cand : pv);
    st_release_gpu(f.done + s, static_cast<uint32_t>(q + 1));
    if (acc) {
      ++accepted;
      const R dx = O::sub(cand.x, pv.x), dy = O::sub(cand.y, pv.y);
      const double d = static_cast<double>(O::sqrt(O::add(O::mul(dx, dx), O::mul(dy, dy))));
      disp = d > disp ? d : disp;
    }
    staged = false;
    e += T;
    if (e >= f.n) {  // this thread's entries of pass q are done: commit its statistics
      if (accepted) atomicAdd(f.slot_acc + gp * kStatSlots + stat_slot, accepted);
      if (disp > 0.0)
        atomicMax(f.slot_md + gp * kStatSlots + stat_slot, static_cast<unsigned long long>(__double_as_longlong(disp)));
      accepted = 0;
      disp = 0.0;
      e = first;
      ++q;
      staged = T >= f.n;  // a thread with a single entry keeps its record
    }
  }
}

// done[] for a launch: movable entries start at 0 passes, pinned slots were set to ~0u once.
__global__ void __launch_bounds__(256) flow_reset(const uint32_t* __restrict__ rec, int64_t n, uint32_t* done) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    done[rec[i * kChunkRecWords]] = 0u;
}

}  // namespace tsg
