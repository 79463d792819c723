// Host-side preparation of the device mesh (libtsg.so, C++20, no CUDA).
//
// Converts the reference's topology (unique-neighbour CSR, incident CSR, boundary flags —
// proj/src/topology.cpp:12-95) into the compact slot-ordered arrays the node kernels read:
//   off[s]..off[s+1]  one row per MOVABLE vertex (pinned rows are empty, so "pinned" costs
//                     no flag array: the kernel skips deg == 0)
//   nbr[]             neighbour slots in ascending ORIGINAL id (the summation order of
//                     neighbor_mean, smoothing.hpp:72-80, survives any locality order)
//   fan[]             per incident triangle: positions of its two other vertices in the row
//                     and v's position k in the triangle (α operand order preserved)
// plus the Form B level schedule for W chunks (worker_chunk, parallel.hpp:19-24).
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "tsg.h"

namespace tsg {

struct HostMesh {
  int64_t nv = 0, nt = 0;
  std::vector<int64_t> order;     // slot -> original vertex
  std::vector<int64_t> rank;      // original vertex -> slot
  std::vector<int64_t> tri_order; // device triangle -> original triangle
  std::vector<uint32_t> off;      // nv+1
  std::vector<uint32_t> nbr;      // slots
  std::vector<uint32_t> fan;
  std::vector<uint32_t> vinc_off; // nv+1, all vertices
  std::vector<uint32_t> vinc;     // device triangle ids
  std::vector<int32_t> tri;       // 3*nt device slots, device triangle order
  std::vector<int32_t> hubs;      // slots with deg > max_small_deg
  int32_t max_deg = 0;
};

struct Phase {
  int64_t small_begin = 0, small_count = 0;  // range in the level node list
  int64_t hub_begin = 0, hub_count = 0;      // range in the level hub list
};

struct FormBSchedule {
  int32_t chunks = 0;
  std::vector<uint32_t> nbr_fresh;  // nbr with kFreshBit on in-chunk lower-id neighbours
  std::vector<int32_t> nodes;       // small-degree slots grouped by level
  std::vector<int32_t> hubs;        // hub slots grouped by level
  std::vector<Phase> levels;
};

// Returns "" on success, else an error message.
std::string build_host_mesh(const tsg_mesh_desc& d, int32_t max_small_deg, HostMesh& out);
std::string build_form_b(const HostMesh& hm, int32_t chunks, int32_t max_small_deg,
                         FormBSchedule& out);
void hilbert_order(int64_t nv, const double* xy, int64_t* order_out);

}  // namespace tsg
