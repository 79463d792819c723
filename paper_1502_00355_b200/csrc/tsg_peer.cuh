// Partitioned Form A over peer memory (one process per GPU, NVLink / NVSwitch): the halo
// exchange and the global stop statistics of each pass go through direct stores into the peers'
// device memory, with a flag barrier, all inside the conditional-WHILE graph of tsg_smooth —
// one graph launch per smooth() on every rank, no host round trip and no collective library
// call per pass (the NCCL all-to-all driver, distributed.DeviceLoop, is the fallback).
//
// Per pass on rank r (reference loop proj/src/smoothing.cpp:98-141):
//   1. the node kernels update r's owned vertices (N buffer);
//   2. every owned vertex that lies in peer q's halo is stored straight into q's N buffer at q's
//      slot for it (P2P stores over NVLink; same-device pointers in tests): by tile_update right
//      after it stores the vertex locally (TilePush: the exchange overlaps the pass tile by
//      tile), by peer_push after the side kernels for rows of valence > 31;
//   3. peer_sync (one warp): r's {accepted, max displacement} of the pass is written into every
//      rank's stats table, then r publishes tick t = tick0 + pass + 1 into flag[r] of every
//      peer (st.release.sys after a system fence) and waits until every peer's flag in its own
//      sync block reached t (ld.acquire.sys); then every rank folds the same table in rank
//      order (sum / max: exact) and applies the reference's stop rule — identical on all ranks,
//      so all stop at the same pass.
// Safety: q pushes pass-p values into r's buffer (p+1)&1, which r reads only in pass p+1, after
// the pass-p barrier; q's next push (pass p+1) targets buffer p&1, which r stopped reading when it
// signalled pass p.  Copy-swap mode maps to ping-pong (identical results).  A start barrier
// (tick0) orders every rank's pre-run host work (set_coords / restore) before any push of the
// run.  Ticks are monotonic across runs (never reset), so no flag ever needs clearing.
// A barrier that waits longer than kPeerTimeoutNs sets `error` and lets the graph finish
// (tsg_smooth then fails loudly) instead of hanging the device.
#pragma once

#include "tsg_kernels.cuh"

namespace tsg {

constexpr int kMaxPeers = 64;
constexpr unsigned long long kPeerTimeoutNs = 20ull * 1000 * 1000 * 1000;

struct PeerSync {  // one per mesh; peers map it
  uint32_t flag[kMaxPeers];             // flag[q] = last tick rank q signalled to this rank
  double stats[2][kMaxPeers][2];        // [tick parity][rank] {accepted, max displacement}
  int32_t error;
  uint32_t tick0;                       // this run's start tick (written by the host)
};

// PeerEntry (one per rank, as mapped in this process) and TilePush: tsg_kernels.cuh.

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Pass-p values of this rank's send vertices into the peers' N buffers.
template <typename R, bool kSoA>
__global__ void __launch_bounds__(256) peer_push(const PassState* st, Coords<R, kSoA> b0, Coords<R, kSoA> b1,
                                                 const int32_t* __restrict__ peer, const uint32_t* __restrict__ src,
                                                 const uint32_t* __restrict__ dst, int64_t n,
                                                 const PeerEntry* __restrict__ tab) {
  if (st->done) return;
  const int pass = st->pass;
  const Coords<R, kSoA> N = (pass & 1) ? b0 : b1;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const PeerEntry e = tab[peer[i]];
    const Coords<R, kSoA> D{static_cast<R*>((pass & 1) ? e.buf0 : e.buf1), e.nv};
    D.store(dst[i], N.load_mut(src[i]));
  }
  __threadfence_system();  // this thread's peer stores before the barrier's release (next kernel)
}

// One warp.  start != 0: the run's start barrier only.  Otherwise the pass's statistics
// exchange, barrier and global stop rule; sets the WHILE condition.
__global__ void peer_sync(PassState* st, const int32_t* slot_acc, const unsigned long long* slot_md,
                          PeerSync* self, const PeerEntry* __restrict__ tab, int32_t rank, int32_t world,
                          int32_t* pass_acc, unsigned long long* pass_md, double tol_abs, int32_t max_iters,
                          cudaGraphConditionalHandle handle, int32_t start) {
  const int lane = threadIdx.x;
  const int q = st->pass;
  int32_t acc = 0;
  unsigned long long mdb = 0;
  if (!start) {
    acc = slot_acc[q * kStatSlots + lane];
    mdb = slot_md[q * kStatSlots + lane];
    acc = __reduce_add_sync(0xffffffffu, acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, mdb, o);
      mdb = other > mdb ? other : mdb;
    }
  }
  if (lane != 0) return;
  const uint32_t tick = self->tick0 + (start ? 0u : static_cast<uint32_t>(q + 1));
  const int par = tick & 1;
  if (!start)
    for (int r = 0; r < world; ++r) {
      double* slot = tab[r].sync->stats[par][rank];
      slot[0] = static_cast<double>(acc);
      slot[1] = __longlong_as_double(static_cast<long long>(mdb));
    }
  __threadfence_system();
  for (int r = 0; r < world; ++r)
    if (r != rank) st_release_sys(&tab[r].sync->flag[rank], tick);
  const unsigned long long t0 = global_ns();
  for (int r = 0; r < world; ++r) {
    if (r == rank) continue;
    while (static_cast<int32_t>(ld_acquire_sys(&self->flag[r]) - tick) < 0) {
      if (global_ns() - t0 > kPeerTimeoutNs) {
        self->error = 1;
        break;
      }
      __nanosleep(100);
    }
  }
  if (start) return;
  long long total = 0;
  double md = 0.0;
  for (int r = 0; r < world; ++r) {
    const double* slot = self->stats[par][r];
    total += static_cast<long long>(slot[0]);
    md = slot[1] > md ? slot[1] : md;
  }
  pass_acc[q] = static_cast<int32_t>(total);
  pass_md[q] = static_cast<unsigned long long>(__double_as_longlong(md));
  st->pass = q + 1;
  if (self->error) {
    st->done = 1;
    st->stop = kStopMaxIters;
  } else if (total == 0) {
    st->done = 1;
    st->stop = kStopNoMoves;
  } else if (md < tol_abs) {
    st->done = 1;
    st->stop = kStopDisplacement;
  } else if (q + 1 >= max_iters) {
    st->done = 1;
    st->stop = kStopMaxIters;
  }
  cudaGraphSetConditional(handle, st->done ? 0u : 1u);
}

}  // namespace tsg
