// Internal to libtsg.so: the context object behind the opaque tsg_context handle, the
// thread-local error message of tsg_last_error(), and the helpers every C-ABI translation
// unit (tsg_engine.cu, tsg_quality.cu) shares.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "tsg.h"

namespace tsg_abi {

inline thread_local std::string g_err;

inline tsg_status fail(tsg_status code, const std::string& msg) {
  g_err = msg;
  return code;
}

}  // namespace tsg_abi

#define TSG_CUDA(call)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return tsg_abi::fail(e_ == cudaErrorMemoryAllocation ? TSG_ERR_NOMEM : TSG_ERR_CUDA,    \
                           std::string(#call) + ": " + cudaGetErrorString(e_));               \
  } while (0)

// After a kernel launch: the launch error with the source line that made it.
#define TSG_LAUNCHED()                                                                         \
  do {                                                                                         \
    cudaError_t e_ = cudaGetLastError();                                                       \
    if (e_ != cudaSuccess)                                                                     \
      return tsg_abi::fail(TSG_ERR_CUDA, std::string("kernel launch at " __FILE__ ":") +       \
                                             std::to_string(__LINE__) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct tsg_context {
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  std::vector<cudaEvent_t> pass_events;  // stream-timed driver
  // Side stream for the medium / hub tiers, forked from and joined back into `stream` so
  // the tiers of one pass (or one Form B level) run concurrently (also inside graphs).
  cudaStream_t side = nullptr;
  cudaStream_t copy_in = nullptr, copy_out = nullptr;  // tsg_smooth_host_batch
  cudaEvent_t ev_in_ready[2] = {}, ev_in_free[2] = {}, ev_out_ready[2] = {}, ev_out_free[2] = {};
  std::vector<cudaEvent_t> fork_events;
  size_t fork_next = 0;
  // Serialises the C-ABI calls on this context: the drop-in smooth() shares one process-wide
  // context between host threads (the reference's smooth() may be called concurrently on
  // distinct meshes), and every call issues work on `stream` and reuses the events above.
  std::recursive_mutex mu;
};

namespace tsg_abi {

// One C-ABI call at a time per context (see tsg_context::mu).
struct CtxLock {
  std::unique_lock<std::recursive_mutex> lk;
  explicit CtxLock(tsg_context* c) {
    if (c) lk = std::unique_lock<std::recursive_mutex>(c->mu);
  }
};

}  // namespace tsg_abi

#define TSG_LOCK_CTX(c) tsg_abi::CtxLock tsg_ctx_lock_(c)

namespace tsg {
struct DeviceInputs;
}
namespace tsg_internal {
// tsg_mesh_upload with the topology either from the desc (din == nullptr) or already on the
// device (tsg_mesh_upload_triangles); caller holds the context lock.
tsg_status mesh_upload_impl(tsg_context* ctx, const tsg_mesh_desc* d, const tsg::DeviceInputs* din, tsg_mesh** out);
}  // namespace tsg_internal
