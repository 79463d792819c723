// Mesh storage (include/trismooth/mesh.hpp).  Behaviour follows proj/src/mesh.cpp:
// validation messages and order (:68-82), pre-topology state (:7-18, :32-42), layout
// conversion (:117-176) and logical equality (:178-203).
#include "trismooth/mesh.hpp"

#include <algorithm>

namespace trismooth {

const char* to_string(Layout layout) { return layout == Layout::SoA ? "soa" : "aos"; }

void AosMesh::reset_topology_state() {
  for (VertexRec& r : verts_) {
    const double x = r.x, y = r.y;
    r = VertexRec{};
    r.x = x;
    r.y = y;
  }
  neighbor_ids_.clear();
  incident_ids_.clear();
}

void AosMesh::assign_adjacency(const Csr& nb, const Csr& inc) {
  neighbor_ids_ = nb.values;
  incident_ids_ = inc.values;
  const int n = vertex_count();
  for (int v = 0; v < n; ++v) {
    VertexRec& r = verts_[v];
    r.neighbor_offset = nb.offsets[v];
    r.neighbor_count = nb.offsets[v + 1] - nb.offsets[v];
    r.incident_offset = inc.offsets[v];
    r.incident_count = inc.offsets[v + 1] - inc.offsets[v];
  }
}

void SoaMesh::resize_vertices(int n) {
  x_.resize(n);
  y_.resize(n);
  reset_topology_state();
}

void SoaMesh::reset_topology_state() {
  const size_t n = x_.size();
  for (auto* v : {&neighbor_count_, &incident_count_, &neighbor_offset_, &incident_offset_})
    v->assign(n, 0);
  boundary_.assign(n, 0);
  min_quality_.assign(n, kUnsetQuality);
  neighbor_ids_.clear();
  incident_ids_.clear();
}

void SoaMesh::assign_adjacency(const Csr& nb, const Csr& inc) {
  neighbor_ids_ = nb.values;
  incident_ids_ = inc.values;
  const int n = vertex_count();
  for (int v = 0; v < n; ++v) {
    neighbor_offset_[v] = nb.offsets[v];
    neighbor_count_[v] = nb.offsets[v + 1] - nb.offsets[v];
    incident_offset_[v] = inc.offsets[v];
    incident_count_[v] = inc.offsets[v + 1] - inc.offsets[v];
  }
}

namespace {

void check_connectivity(size_t n_points, const std::vector<std::array<int, 3>>& tris) {
  if (tris.empty()) throw StructuralError("mesh must contain at least one triangle");
  const long long n = static_cast<long long>(n_points);
  for (size_t t = 0; t < tris.size(); ++t) {
    const auto& c = tris[t];
    for (const int v : c)
      if (v < 0 || v >= n)
        throw StructuralError("triangle " + std::to_string(t) + " references vertex " +
                              std::to_string(v) + " outside [0, " + std::to_string(n) + ")");
    if (c[0] == c[1] || c[1] == c[2] || c[0] == c[2])
      throw StructuralError("triangle " + std::to_string(t) + " repeats a vertex");
  }
}

// Copies every logical field from one storage into another of equal sizes.
template <class Src, class Dst>
void transfer(const Src& src, Dst& dst) {
  const int nv = src.vertex_count();
  Csr nb, inc;
  nb.offsets.assign(nv + 1, 0);
  inc.offsets.assign(nv + 1, 0);
  for (int v = 0; v < nv; ++v) {
    dst.set_position(v, src.position(v));
    dst.set_boundary(v, src.is_boundary(v));
    dst.set_vertex_min_quality(v, src.vertex_min_quality(v));
    const auto a = src.neighbors(v);
    const auto b = src.incident(v);
    nb.values.insert(nb.values.end(), a.begin(), a.end());
    inc.values.insert(inc.values.end(), b.begin(), b.end());
    nb.offsets[v + 1] = static_cast<int>(nb.values.size());
    inc.offsets[v + 1] = static_cast<int>(inc.values.size());
  }
  dst.assign_adjacency(nb, inc);
  for (int t = 0; t < src.triangle_count(); ++t) dst.set_tri_quality(t, src.tri_quality(t));
}

bool same_quality(double a, double b) { return (std::isnan(a) && std::isnan(b)) || a == b; }

}  // namespace

Mesh build_mesh(const std::vector<Point>& points,
                const std::vector<std::array<int, 3>>& triangles, Layout layout) {
  check_connectivity(points.size(), triangles);
  if (layout == Layout::SoA) {
    SoaMesh s;
    s.resize_vertices(static_cast<int>(points.size()));
    for (size_t i = 0; i < points.size(); ++i) s.set_position(static_cast<int>(i), points[i]);
    auto& tv = s.tri_verts();
    tv.reserve(3 * triangles.size());
    for (const auto& c : triangles) tv.insert(tv.end(), c.begin(), c.end());
    s.tri_qualities().assign(triangles.size(), kUnsetQuality);
    return Mesh(std::move(s));
  }
  AosMesh a;
  a.verts().resize(points.size());
  for (size_t i = 0; i < points.size(); ++i) a.set_position(static_cast<int>(i), points[i]);
  a.tris().resize(triangles.size());
  for (size_t t = 0; t < triangles.size(); ++t) a.tris()[t].v = triangles[t];
  return Mesh(std::move(a));
}

void init_flags(Mesh& mesh) {
  mesh.visit([](auto& m) { m.reset_topology_state(); });
}

Mesh convert_layout(const Mesh& mesh, Layout target) {
  return mesh.visit([target](const auto& src) -> Mesh {
    const int nv = src.vertex_count(), nt = src.triangle_count();
    if (target == Layout::SoA) {
      SoaMesh dst;
      dst.resize_vertices(nv);
      dst.tri_verts().resize(3 * static_cast<size_t>(nt));
      dst.tri_qualities().resize(nt);
      for (int t = 0; t < nt; ++t) {
        const auto c = src.tri(t);
        std::copy(c.begin(), c.end(), dst.tri_verts().begin() + 3 * static_cast<size_t>(t));
      }
      transfer(src, dst);
      return Mesh(std::move(dst));
    }
    AosMesh dst;
    dst.verts().resize(nv);
    dst.tris().resize(nt);
    for (int t = 0; t < nt; ++t) dst.tris()[t].v = src.tri(t);
    transfer(src, dst);
    return Mesh(std::move(dst));
  });
}

bool logically_equal(const Mesh& a, const Mesh& b) {
  return a.visit([&](const auto& x) {
    return b.visit([&](const auto& y) {
      if (x.vertex_count() != y.vertex_count() || x.triangle_count() != y.triangle_count())
        return false;
      for (int v = 0; v < x.vertex_count(); ++v) {
        if (!(x.position(v) == y.position(v)) || x.is_boundary(v) != y.is_boundary(v) ||
            !same_quality(x.vertex_min_quality(v), y.vertex_min_quality(v)))
          return false;
        const auto n1 = x.neighbors(v), n2 = y.neighbors(v);
        const auto i1 = x.incident(v), i2 = y.incident(v);
        if (!std::equal(n1.begin(), n1.end(), n2.begin(), n2.end()) ||
            !std::equal(i1.begin(), i1.end(), i2.begin(), i2.end()))
          return false;
      }
      for (int t = 0; t < x.triangle_count(); ++t)
        if (x.tri(t) != y.tri(t) || !same_quality(x.tri_quality(t), y.tri_quality(t))) return false;
      return true;
    });
  });
}

}  // namespace trismooth
