// Device-side layout preparation (tsg_layout_dev.cu): the device arrays of a tsg_mesh built on
// the GPU, identical to what build_host_mesh (tsg_prep.cpp) computes on the host.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>

#include "tsg_prep.hpp"

namespace tsg {

// Device arrays owned by the caller after a successful build (free_layout releases them).
// order / tri_order stay null for the identity order (no locality order given).
struct DeviceLayout {
  uint32_t *off = nullptr, *nbr = nullptr, *fan = nullptr, *tmeta = nullptr, *tile_rec = nullptr;
  uint32_t *ext_off = nullptr, *ext = nullptr, *trec = nullptr, *vinc_off = nullptr, *vinc = nullptr;
  uint16_t* fan16 = nullptr;
  int32_t* tri = nullptr;
  int64_t *order = nullptr, *tri_order = nullptr;
};

// Builds the layout on `s` from the host description (validated by the caller).  Fills the
// host mirror's nv, nt, order, rank, off, nbr, fan, tri_order, medium, hubs, large, max_deg,
// max_ext, max_rec_words.  Returns "" or an error (arrays allocated so far stay in `L`).
// Topology already on the device (tsg_mesh_upload_triangles): used instead of the desc's host
// nbr_off / nbr / inc_off / inc / boundary / tri arrays.
struct DeviceInputs {
  const int64_t* nbr_off = nullptr;  // nv + 1
  const int32_t* nbr = nullptr;
  const int64_t* inc_off = nullptr;  // nv + 1
  const int32_t* inc = nullptr;
  const int32_t* tri = nullptr;      // 3 nt
  const uint8_t* boundary = nullptr;
  int64_t nnb = 0, ninc = 0;
};

// host_rows: also download order / rank / nbr / fan / tri_order into hm (tests); otherwise hm
// holds off, the tier lists and the tile sizes, and the rest stays on the device
// (tsg_engine.cu ensure_host_rows downloads it when a host-side builder needs it).
std::string build_device_layout(cudaStream_t s, const tsg_mesh_desc& d, const Tiers& tiers, HostMesh& hm,
                                DeviceLayout& L, int32_t tile = kTile, bool host_rows = true,
                                const DeviceInputs* din = nullptr);
// The remaining HostMesh arrays from the device (fan16, tri, vinc_off, vinc, tmeta, tile_rec,
// ext_off, ext, trec): for tests that compare with build_host_mesh.
std::string download_layout(cudaStream_t s, const DeviceLayout& L, HostMesh& hm);
void free_layout(DeviceLayout& L);

}  // namespace tsg
