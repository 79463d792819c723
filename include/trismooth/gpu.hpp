// B200 extensions of the trismooth API (not in the reference).
//
//   Topology64 / build_topology   host mesh prep with 64-bit offsets: the reference's Csr is
//                                 int-indexed and its raw list overflows at 6*nt > 2^31-1
//                                 (SURVEY K6); this builds the unique-neighbour and incident
//                                 rows directly, in parallel, identical to find_neighbors'.
//   DeviceMesh                    a mesh resident on one GPU (RAII over tsg_mesh) for callers
//                                 that smooth repeatedly without re-running host prep.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "trismooth/mesh.hpp"
#include "trismooth/smoothing.hpp"

struct tsg_context;
struct tsg_mesh;

namespace trismooth::gpu {

struct Topology64 {
  std::vector<int64_t> nbr_off;   // nv+1
  std::vector<int32_t> nbr;       // ascending per row
  std::vector<int64_t> inc_off;   // nv+1
  std::vector<int32_t> inc;       // ascending per row
  std::vector<uint8_t> boundary;  // 1 = pinned (isolated or any multiplicity != 2)
};

Topology64 build_topology(int64_t nv, const int32_t* tri, int64_t nt);

/// The same topology built on the device (tsg_topology: radix sorts, no int32 raw list).
Topology64 device_topology(int64_t nv, const int32_t* tri, int64_t nt, tsg_context* ctx = nullptr);

/// The process-wide device context (device = $TSG_DEVICE, else $LOCAL_RANK, else 0).
/// Throws Error when no CUDA device is usable: there is no CPU fallback.
tsg_context* default_context();

/// bbox diagonal exactly as the reference computes it (proj/src/smoothing.cpp:62-74).
double bbox_diagonal(const double* xy, int64_t nv);

class DeviceMesh {
 public:
  /// xy: 2*nv interleaved; tri: 3*nt.  order: Hilbert locality order when `reorder`.
  DeviceMesh(const double* xy, int64_t nv, const int32_t* tri, int64_t nt, const Topology64& topo,
             Layout layout, Precision precision, bool reorder, tsg_context* ctx = nullptr);
  ~DeviceMesh();
  DeviceMesh(const DeviceMesh&) = delete;
  DeviceMesh& operator=(const DeviceMesh&) = delete;

  tsg_mesh* handle() const { return mesh_; }
  int64_t vertex_count() const { return nv_; }
  int64_t triangle_count() const { return nt_; }
  bool reordered() const { return reordered_; }
  int64_t device_bytes() const;

  void set_coords(const double* xy);
  void get_coords(double* xy) const;
  void tri_alpha(double* out) const;
  void vertex_minima(double* out) const;

  /// Passes on the device; fills iterations / stop / per-pass vectors / device_ms /
  /// kernel_launches of the returned stats (timers of host phases stay zero).
  RunStats run(const SmoothConfig& cfg, double bbox_diag);

 private:
  tsg_mesh* mesh_ = nullptr;
  int64_t nv_ = 0, nt_ = 0;
  bool reordered_ = false;
};

/// Throws Error with the libtsg message when status != 0.
void check(int status, const char* what);

}  // namespace trismooth::gpu
