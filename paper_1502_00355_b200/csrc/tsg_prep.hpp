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
#include "tsg_layout.hpp"

namespace tsg {

// Valence tiers of movable vertices: thread-per-vertex kernels for small (<= small_max) and
// medium (<= medium_max, a separate list) rows, CTA-per-vertex for hubs.  A small / medium fan
// record stores ring positions with v itself at position small_max / medium_max, which must
// fit 5 bits.
#ifdef __CUDACC__
#define TSG_HD __host__ __device__
#else
#define TSG_HD
#endif

struct Tiers {
  int32_t small_max = 12;
  int32_t medium_max = 31;
  TSG_HD int tier(uint32_t deg) const {
    return deg <= static_cast<uint32_t>(small_max) ? 0 : deg <= static_cast<uint32_t>(medium_max) ? 1 : 2;
  }
};

struct HostMesh {
  int64_t nv = 0, nt = 0;
  std::vector<int64_t> order;     // slot -> original vertex
  std::vector<int64_t> rank;      // original vertex -> slot
  std::vector<int64_t> tri_order; // device triangle -> original triangle
  std::vector<uint32_t> off;      // nv+1
  std::vector<uint32_t> nbr;      // slots
  std::vector<uint32_t> fan;      // every row: (i1, i2, k) records
  std::vector<uint16_t> fan16;    // small rows: ring positions of (p1, p2, p3), 5 bits each
  // Rows with deg <= kMaxCycleDeg: the one-ring as a directed cycle — cycpos[off[s] + j] is the
  // row position of the j-th cycle entry (every incident triangle is a rotation of (v,
  // row[cycpos[j]], row[cycpos[j+1]])), cycrot[...] the position k of v in that literal
  // triangle; has_cycle[s] = 0 when the link of v is not a single directed cycle (bow-tie /
  // inconsistent orientation): those rows use the fan records.  cycpos / cycrot are released
  // once the tiles are built.
  std::vector<uint8_t> cycpos, cycrot, has_cycle;
  std::vector<uint32_t> vinc_off; // nv+1, all vertices
  std::vector<uint32_t> vinc;     // device triangle ids
  std::vector<int32_t> tri;       // 3*nt device slots, device triangle order
  std::vector<int32_t> medium;    // slots of the medium tier
  std::vector<int32_t> hubs;      // slots of the hub tier
  // Form A fused: rows with deg > kMaxCycleDeg (warp per vertex; longest first).
  std::vector<int32_t> large;
  // Tiles (rows with 1 <= deg <= kMaxCycleDeg; other rows have tmeta == 0):
  //   tmeta[s]     word offset of row s's first word inside its tile's words (bits 0-15) |
  //                deg << kMetaDegShift | stride << kMetaStrideShift (word j at offset + j*stride)
  //   tile_rec[t]  first word of tile t (ntiles + 1; multiples of 4)
  //   trec         u32 words: row[j] local index | cycle[j] local index << 16 | k[j] << 30
  //                (v's position in the literal triangle (v, cycle[j], cycle[j+1]) rotated;
  //                local indices < 2^14); cycle[j] = kNoLocal when the row has no link cycle
  //   ext_off/ext  per tile: sorted external slots (ntiles + 1 offsets)
  std::vector<uint32_t> tmeta, tile_rec, ext_off, ext, trec;
  int32_t max_ext = 0, max_rec_words = 0;
  int32_t max_deg = 0;
  int32_t tile = kTile;  // slots per tile (multiple of 256, <= kTileMax; chosen per mesh)
};

struct Phase {
  int64_t small_begin = 0, small_count = 0;    // range in the level node list
  int64_t medium_begin = 0, medium_count = 0;  // range in the level medium list
  int64_t hub_begin = 0, hub_count = 0;        // range in the level hub list
};

struct FormBSchedule {
  int32_t chunks = 0;
  std::vector<uint32_t> nbr_fresh;  // nbr with kFreshBit on in-chunk lower-id neighbours
  std::vector<int32_t> nodes;       // small-degree slots grouped by level
  std::vector<int32_t> medium;      // medium-tier slots grouped by level
  std::vector<int32_t> hubs;        // hub slots grouped by level
  std::vector<Phase> levels;
  // Chunk schedule (one CTA per chunk, levels in order inside the CTA): the movable slots
  // sorted by (chunk, level, slot); chunk c owns levels chunk_lvl[c] .. chunk_lvl[c+1]-1 of
  // lvl_off, level entries lvl_off[i] .. lvl_off[i+1]-1 of cb_order.
  std::vector<int32_t> cb_order;
  std::vector<int32_t> lvl_off;
  std::vector<int32_t> chunk_lvl;
  int64_t max_chunk_work = 0;  // most movable vertices in one chunk
  // Per entry of cb_order a kChunkRecWords-word record: slot, valence, then (valence <=
  // kChunkRecMaxDeg) the row's neighbour slots (with kFreshBit) and its fan records.
  std::vector<uint32_t> cb_rec;
  // Dataflow schedule (tsg_flow.cuh): the movable slots sorted by (level, slot), one
  // kChunkRecWords record each (same format as cb_rec).
  std::vector<uint32_t> flow_rec;
};
constexpr int kChunkRecWords = 32;
constexpr int kChunkRecMaxDeg = 15;

// Structural checks of a caller's description (corner ids, CSR offsets / entries, the order
// permutation); "" when valid.  build_host_mesh runs them first.
// topology = false: the desc's CSR arrays are not used (built on the device); only the order
// permutation is checked.
std::string validate_desc(const tsg_mesh_desc& d, bool topology = true);
// Returns "" on success, else an error message.
std::string build_host_mesh(const tsg_mesh_desc& d, const Tiers& tiers, HostMesh& out, int32_t tile = kTile);
std::string build_form_b(const HostMesh& hm, int32_t chunks, const Tiers& tiers, FormBSchedule& out);
void hilbert_order(int64_t nv, const double* xy, int64_t* order_out);
std::string build_tiles(HostMesh& hm, const std::vector<uint32_t>& deg, int32_t max_deg);

}  // namespace tsg
