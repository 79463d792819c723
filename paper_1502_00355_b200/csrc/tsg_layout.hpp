// Layout constants shared by the host preparation (tsg_prep.cpp) and the kernels.
#pragma once

#include <cstdint>

namespace tsg {

constexpr int kMaxCycleDeg = 31;  // tile (thread-per-vertex) rows: valence <= 31
// Tiles of tile_update: kTile consecutive slots (the degree-sort windows of the locality
// order).  A tile's small rows address their neighbours by LOCAL index: slot - tile base for
// in-tile slots, kTile + position in the tile's sorted external-slot list otherwise.
#ifndef TSG_TILE
#define TSG_TILE 1024
#endif
constexpr int kTile = TSG_TILE;  // default slots per tile (a mesh may use up to kTileMax)
constexpr int kTileMax = 1536;  // group stride (11 bits) < 2048; meta word offsets 15 bits
constexpr uint32_t kNoLocal = 0x3fffu;  // cycle entry of a row without a single link cycle
// Tile row word: row[j] (bits 0-13) | cycle[j] (bits 16-29) | k[j] (bits 30-31).
constexpr uint32_t kLocalMask = 0x3fffu;
constexpr int kWordCycleShift = 16;
constexpr int kWordRotShift = 30;
// Tile meta word: first-word offset (15 bits: <= kTile * kMaxCycleDeg words) | valence (5
// bits) | group stride (11 bits, <= kTile) (tsg_prep.hpp HostMesh::tmeta).
constexpr uint32_t kMetaBaseMask = 0x7fffu;
constexpr int kMetaDegShift = 15;
constexpr uint32_t kMetaDegMask = 31u;
constexpr int kMetaStrideShift = 20;

}  // namespace tsg
