// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" face over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled out-of-tree by oracle/Makefile into
// oracle/_ref/libtsref.so).  Only tests/, __graft_entry__.smoke() and bench.py's
// reference / cpu_baseline legs load it.  Every function forwards to a public
// reference entry point; nothing here re-implements reference behaviour.
//
//   tsref_perturbed_grid   -> trismooth::perturbed_grid      (proj/src/meshgen.cpp:226-260)
//   tsref_generate_points  -> trismooth::generate_points     (proj/src/meshgen.cpp:9-47)
//   tsref_triangulate      -> trismooth::delaunay_triangulate (proj/src/meshgen.cpp:221-224)
//   tsref_smooth           -> trismooth::smooth              (proj/src/smoothing.cpp:146-182)
//   tsref_topology         -> find_neighbors + determine_constraints (proj/src/topology.cpp:69-95)
//   tsref_triangle_alpha   -> trismooth::triangle_alpha      (proj/include/trismooth/quality.hpp:15-23)
//   tsref_text_hashes      -> write_triangle_format          (proj/src/io.cpp:173-206), FNV-1a-64

#include <cstdint>
#include <cstring>
#include <string>
#include <thread>

#include "trismooth/io.hpp"
#include "trismooth/meshgen.hpp"
#include "trismooth/quality.hpp"
#include "trismooth/smoothing.hpp"
#include "trismooth/topology.hpp"

using namespace trismooth;

namespace {

thread_local std::string g_err;

std::vector<Point> points_from(const double* xy, int64_t n) {
  std::vector<Point> p(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) p[i] = {xy[2 * i], xy[2 * i + 1]};
  return p;
}

std::vector<std::array<int, 3>> tris_from(const int32_t* t, int64_t nt) {
  std::vector<std::array<int, 3>> out(static_cast<size_t>(nt));
  for (int64_t i = 0; i < nt; ++i) out[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
  return out;
}

uint64_t fnv1a(const std::string& s) {
  uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

}  // namespace

extern "C" {

const char* tsref_last_error() { return g_err.c_str(); }

unsigned tsref_hardware_concurrency() { return std::thread::hardware_concurrency(); }

double tsref_triangle_alpha(double x1, double y1, double x2, double y2, double x3, double y3) {
  return triangle_alpha({x1, y1}, {x2, y2}, {x3, y3});
}

uint64_t tsref_splitmix_stream(uint64_t seed, int count, uint64_t* out) {
  SplitMix64 rng(seed);
  for (int i = 0; i < count; ++i) out[i] = rng.next();
  return count;
}

int tsref_perturbed_grid(int rows, int cols, double pert, uint64_t seed, double* xy,
                         int32_t* tri) {
  try {
    const MeshSource s = perturbed_grid(rows, cols, pert, seed);
    for (size_t i = 0; i < s.points.size(); ++i) {
      xy[2 * i] = s.points[i].x;
      xy[2 * i + 1] = s.points[i].y;
    }
    for (size_t t = 0; t < s.triangles.size(); ++t)
      for (int k = 0; k < 3; ++k) tri[3 * t + k] = s.triangles[t][k];
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int tsref_generate_points(int n, uint64_t seed, double* xy) {
  try {
    GenSpec spec;
    spec.kind = GenKind::DelaunayRandom;
    spec.n_points = n;
    spec.seed = seed;
    const auto pts = generate_points(spec);
    for (size_t i = 0; i < pts.size(); ++i) {
      xy[2 * i] = pts[i].x;
      xy[2 * i + 1] = pts[i].y;
    }
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Returns the triangle count (≤ cap) or -1.
int64_t tsref_triangulate(const double* xy, int64_t n, int32_t* tri_out, int64_t cap) {
  try {
    const auto tris = delaunay_triangulate(points_from(xy, n));
    if (static_cast<int64_t>(tris.size()) > cap) {
      g_err = "triangle buffer too small";
      return -1;
    }
    for (size_t t = 0; t < tris.size(); ++t)
      for (int k = 0; k < 3; ++k) tri_out[3 * t + k] = tris[t][k];
    return static_cast<int64_t>(tris.size());
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

// FNV-1a-64 over the reference's own .node / .ele text.
int tsref_text_hashes(const double* xy, int64_t nv, const int32_t* tri, int64_t nt,
                      uint64_t* node_fnv, uint64_t* ele_fnv) {
  try {
    const Mesh m = build_mesh(points_from(xy, nv), tris_from(tri, nt), Layout::AoS);
    const auto [node, ele] = write_triangle_format(m);
    *node_fnv = fnv1a(node);
    *ele_fnv = fnv1a(ele);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// Unique-neighbour CSR (ascending), multiplicities, incident CSR, boundary flags.
// Offsets arrays hold nv+1 entries; value arrays must hold 6*nt entries.
int tsref_topology(const double* xy, int64_t nv, const int32_t* tri, int64_t nt,
                   int64_t* nbr_off, int32_t* nbr, int32_t* mult, int64_t* inc_off, int32_t* inc,
                   uint8_t* boundary) {
  try {
    Mesh m = build_mesh(points_from(xy, nv), tris_from(tri, nt), Layout::SoA);
    init_flags(m);
    const Adjacency adj = find_neighbors(m);
    determine_constraints(m, adj);
    for (int64_t v = 0; v <= nv; ++v) {
      nbr_off[v] = adj.unique.offsets[v];
      inc_off[v] = adj.incident.offsets[v];
    }
    std::memcpy(nbr, adj.unique.values.data(), adj.unique.values.size() * sizeof(int32_t));
    std::memcpy(mult, adj.multiplicity.data(), adj.multiplicity.size() * sizeof(int32_t));
    std::memcpy(inc, adj.incident.values.data(), adj.incident.values.size() * sizeof(int32_t));
    m.visit([&](const auto& s) {
      for (int64_t v = 0; v < nv; ++v) boundary[v] = s.is_boundary(static_cast<int>(v)) ? 1 : 0;
    });
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

// cfg = {layout(0 aos,1 soa), form(0 A,1 B), strategy(0 fused,1 twophase),
//        backend(0 serial,1 parallel), workers, max_iters}
// stats = {iterations, stop(0 max_iters,1 displacement,2 no_moves), init_ms, topo_ms,
//          constr_ms, iter_ms, total_ms, min_before, min_after, mean_before, mean_after}
int tsref_smooth(const double* xy, int64_t nv, const int32_t* tri, int64_t nt, const int32_t* cfg,
                 double move_tol, double* xy_out, uint8_t* boundary_out, int32_t* accepted_out,
                 double* max_disp_out, int32_t cap_passes, double* stats, double* tri_alpha_out,
                 double* vmin_out) {
  try {
    Mesh m = build_mesh(points_from(xy, nv), tris_from(tri, nt),
                        cfg[0] == 0 ? Layout::AoS : Layout::SoA);
    SmoothConfig c;
    c.form = cfg[1] == 0 ? IterationForm::A : IterationForm::B;
    c.strategy = cfg[2] == 0 ? UpdateStrategy::Fused : UpdateStrategy::TwoPhase;
    c.backend = cfg[3] == 0 ? Backend::Serial : Backend::Parallel;
    c.workers = cfg[4];
    c.max_iters = cfg[5];
    c.move_tol = move_tol;
    const RunStats s = smooth(m, c);
    m.visit([&](const auto& st) {
      for (int64_t v = 0; v < nv; ++v) {
        const Point p = st.position(static_cast<int>(v));
        if (xy_out) {
          xy_out[2 * v] = p.x;
          xy_out[2 * v + 1] = p.y;
        }
        if (boundary_out) boundary_out[v] = st.is_boundary(static_cast<int>(v)) ? 1 : 0;
        if (vmin_out) vmin_out[v] = st.vertex_min_quality(static_cast<int>(v));
      }
      if (tri_alpha_out)
        for (int64_t t = 0; t < nt; ++t) tri_alpha_out[t] = st.tri_quality(static_cast<int>(t));
    });
    const int n = std::min<int>(cap_passes, s.iterations);
    for (int i = 0; i < n; ++i) {
      if (accepted_out) accepted_out[i] = s.accepted_per_pass[i];
      if (max_disp_out) max_disp_out[i] = s.max_disp_per_pass[i];
    }
    stats[0] = s.iterations;
    stats[1] = s.stop == StopReason::MaxIters ? 0 : s.stop == StopReason::Displacement ? 1 : 2;
    stats[2] = s.init_ms;
    stats[3] = s.topo_ms;
    stats[4] = s.constr_ms;
    stats[5] = s.iter_ms;
    stats[6] = s.total_ms;
    stats[7] = s.min_alpha_before;
    stats[8] = s.min_alpha_after;
    stats[9] = s.mean_alpha_before;
    stats[10] = s.mean_alpha_after;
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

}  // extern "C"
