// Synthetic fixtures (include/trismooth/meshgen.hpp).
//
// Output contract of proj/src/meshgen.cpp: SplitMix64 points with the 1e-12 redraw rule
// (:9-47), Bowyer-Watson over the points plus a 1e4-span super triangle with the same
// orientation / in-circle expressions, insertion in generation order, cavity = the
// in-circle-connected component of the located triangle, new triangles (a, b, p) per rim edge
// (:73-217), canonical smallest-first CCW output sorted lexicographically (:94-108), and the
// perturbed lattice (:226-260).
//
// What is different is only the cost: point location starts from a triangle incident to the
// nearest already-inserted point found through a bucket grid (O(1) expected walk instead of a
// walk from the last triangle, which made the reference ~n^1.9), dead triangle slots are
// recycled, and the final sort is a counting sort on the first corner.
#include <algorithm>
#include <cmath>
#include <numbers>
#include <numeric>
#include <thread>
#include <unordered_map>

#include "trismooth/meshgen.hpp"

namespace trismooth {

namespace {

constexpr double kPi = std::numbers::pi;

inline double orient2(Point a, Point b, Point c) {
  const double abx = b.x - a.x, acy = c.y - a.y, aby = b.y - a.y, acx = c.x - a.x;
  return abx * acy - aby * acx;
}

// > 0 iff d is strictly inside the circumcircle of CCW (a, b, c); same expression tree as the
// reference predicate so near-degenerate decisions agree.
inline double incircle(Point a, Point b, Point c, Point d) {
  const double ax = a.x - d.x, ay = a.y - d.y;
  const double bx = b.x - d.x, by = b.y - d.y;
  const double cx = c.x - d.x, cy = c.y - d.y;
  const double a2 = ax * ax + ay * ay;
  const double b2 = bx * bx + by * by;
  const double c2 = cx * cx + cy * cy;
  const double t1 = ax * (by * c2 - b2 * cy);
  const double t2 = ay * (bx * c2 - b2 * cx);
  const double t3 = a2 * (bx * cy - by * cx);
  return t1 - t2 + t3;
}

class Triangulator {
 public:
  explicit Triangulator(const std::vector<Point>& pts) : n_(static_cast<int>(pts.size())) {
    P_.reserve(pts.size() + 3);
    P_ = pts;
    double x0 = P_[0].x, x1 = x0, y0 = P_[0].y, y1 = y0;
    for (const Point& p : P_) {
      x0 = std::min(x0, p.x);
      x1 = std::max(x1, p.x);
      y0 = std::min(y0, p.y);
      y1 = std::max(y1, p.y);
    }
    const double mx = 0.5 * (x0 + x1), my = 0.5 * (y0 + y1);
    const double span = std::max({x1 - x0, y1 - y0, 1e-8});
    const double big = 1e4 * span;
    P_.push_back({mx - 3.0 * big, my - big});
    P_.push_back({mx + 3.0 * big, my - big});
    P_.push_back({mx, my + 3.0 * big});
    const size_t cap = 2 * pts.size() + 16;
    V_.reserve(3 * cap);
    A_.reserve(3 * cap);
    new_tri(n_, n_ + 1, n_ + 2);
    last_ = 0;
    // bucket grid over the input bounding box, ~2 points per cell when full
    G_ = std::max(1, static_cast<int>(std::sqrt(static_cast<double>(n_) / 2.0)));
    gx0_ = x0;
    gy0_ = y0;
    gsx_ = x1 > x0 ? G_ / (x1 - x0) : 0.0;
    gsy_ = y1 > y0 ? G_ / (y1 - y0) : 0.0;
    cell_.assign(static_cast<size_t>(G_) * G_, -1);
    vtri_.assign(P_.size(), -1);
    vmark_.assign(P_.size(), -1);
    vstart_.assign(P_.size(), -1);
    vend_.assign(P_.size(), -1);
  }

  // Inserts in generation order (the reference's), or along a Hilbert curve when `spatial`:
  // the triangulation is the same (unique for points in general position; cross-checked in
  // tests/test_host_api.py), but consecutive insertions then touch neighbouring triangles,
  // which removes the cache misses that dominate at 10^7 points.
  std::vector<std::array<int, 3>> run(bool spatial) {
    if (spatial) {
      for (const int p : hilbert_sequence()) insert(p);
    } else {
      for (int p = 0; p < n_; ++p) insert(p);
    }
    // canonical output: real triangles, smallest corner first (rotation keeps orientation)
    std::vector<std::array<int, 3>> tris;
    tris.reserve(2 * static_cast<size_t>(n_));
    const int nt = static_cast<int>(alive_.size());
    for (int t = 0; t < nt; ++t) {
      if (!alive_[t]) continue;
      const int* v = &V_[3 * t];
      if (v[0] >= n_ || v[1] >= n_ || v[2] >= n_) continue;
      const int r = (v[1] < v[0]) ? (v[2] < v[1] ? 2 : 1) : (v[2] < v[0] ? 2 : 0);
      tris.push_back({v[r], v[(r + 1) % 3], v[(r + 2) % 3]});
    }
    if (tris.empty()) throw Error("triangulation failed: all points are collinear");
    // counting sort on the first corner, then sort each (tiny) bucket
    std::vector<int> start(n_ + 1, 0);
    for (const auto& t : tris) ++start[t[0] + 1];
    for (int i = 0; i < n_; ++i) start[i + 1] += start[i];
    std::vector<std::array<int, 3>> out(tris.size());
    std::vector<int> pos(start.begin(), start.end() - 1);
    for (const auto& t : tris) out[pos[t[0]]++] = t;
    for (int i = 0; i < n_; ++i)
      if (start[i + 1] - start[i] > 1) std::sort(out.begin() + start[i], out.begin() + start[i + 1]);
    return out;
  }

 private:
  int n_;
  std::vector<Point> P_;
  std::vector<int> V_;        // 3 corners per triangle slot (CCW)
  std::vector<int> A_;        // A_[3t+k]: triangle across edge (V[k], V[k+1]), -1 none
  std::vector<uint8_t> alive_;
  std::vector<int> free_;
  std::vector<int> mark_;     // per slot: epoch of last visit
  std::vector<int> incav_;    // per slot: epoch if in cavity
  int epoch_ = 0;
  int last_ = 0;
  // point location hints
  int G_ = 1;
  double gx0_ = 0, gy0_ = 0, gsx_ = 0, gsy_ = 0;
  std::vector<int> cell_;     // last inserted point per cell
  std::vector<int> vtri_;     // a live triangle incident to each vertex
  // rim linking scratch
  std::vector<int> vmark_, vstart_, vend_;
  std::vector<int> cavity_;
  struct RimEdge {
    int a, b, out;
  };
  std::vector<RimEdge> rim_;

  std::vector<int> hilbert_sequence() const {
    const double x0 = gx0_, y0 = gy0_;
    const double sx = gsx_ > 0 ? gsx_ * 65535.0 / G_ : 0.0, sy = gsy_ > 0 ? gsy_ * 65535.0 / G_ : 0.0;
    std::vector<uint64_t> key(n_);
    for (int i = 0; i < n_; ++i) {
      uint32_t x = static_cast<uint32_t>(std::clamp((P_[i].x - x0) * sx, 0.0, 65535.0));
      uint32_t y = static_cast<uint32_t>(std::clamp((P_[i].y - y0) * sy, 0.0, 65535.0));
      uint64_t d = 0;
      for (uint32_t s = 1u << 15; s > 0; s >>= 1) {
        const uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
        d += static_cast<uint64_t>(s) * s * ((3u * rx) ^ ry);
        if (ry == 0) {
          if (rx == 1) {
            x = 0xffffu - x;
            y = 0xffffu - y;
          }
          std::swap(x, y);
        }
      }
      key[i] = (d << 32) | static_cast<uint32_t>(i);
    }
    std::sort(key.begin(), key.end());
    std::vector<int> seq(n_);
    for (int i = 0; i < n_; ++i) seq[i] = static_cast<int>(key[i] & 0xffffffffu);
    return seq;
  }

  int new_tri(int a, int b, int c) {
    int t;
    if (!free_.empty()) {
      t = free_.back();
      free_.pop_back();
      V_[3 * t] = a, V_[3 * t + 1] = b, V_[3 * t + 2] = c;
      A_[3 * t] = A_[3 * t + 1] = A_[3 * t + 2] = -1;
      alive_[t] = 1;
    } else {
      t = static_cast<int>(alive_.size());
      V_.insert(V_.end(), {a, b, c});
      A_.insert(A_.end(), {-1, -1, -1});
      alive_.push_back(1);
      mark_.push_back(0);
      incav_.push_back(0);
    }
    return t;
  }

  int cell_of(Point p) const {
    int cx = static_cast<int>((p.x - gx0_) * gsx_), cy = static_cast<int>((p.y - gy0_) * gsy_);
    cx = std::clamp(cx, 0, G_ - 1);
    cy = std::clamp(cy, 0, G_ - 1);
    return cy * G_ + cx;
  }

  int hint_for(Point p) const {
    const int c = cell_of(p), cx = c % G_, cy = c / G_;
    for (int r = 0; r <= 3; ++r) {
      for (int dy = -r; dy <= r; ++dy)
        for (int dx = -r; dx <= r; ++dx) {
          if (std::max(std::abs(dx), std::abs(dy)) != r) continue;
          const int x = cx + dx, y = cy + dy;
          if (x < 0 || y < 0 || x >= G_ || y >= G_) continue;
          const int u = cell_[static_cast<size_t>(y) * G_ + x];
          if (u >= 0) return vtri_[u];
        }
    }
    return last_;
  }

  bool inside(int t, Point p) const {
    const int* v = &V_[3 * t];
    for (int k = 0; k < 3; ++k)
      if (orient2(P_[v[k]], P_[v[(k + 1) % 3]], p) < 0.0) return false;
    return true;
  }

  int locate(Point p) const {
    int cur = hint_for(p);
    const long long cap = static_cast<long long>(alive_.size()) * 4 + 16;
    for (long long step = 0; step < cap; ++step) {
      const int* v = &V_[3 * cur];
      int next = -1;
      for (int k = 0; k < 3; ++k) {
        const int nb = A_[3 * cur + k];
        if (nb != -1 && orient2(P_[v[k]], P_[v[(k + 1) % 3]], p) < 0.0) {
          next = nb;
          break;
        }
      }
      if (next == -1) return cur;
      cur = next;
    }
    const int nt = static_cast<int>(alive_.size());
    for (int t = 0; t < nt; ++t)
      if (alive_[t] && inside(t, p)) return t;
    for (int t = 0; t < nt; ++t)
      if (alive_[t] && incircle(P_[V_[3 * t]], P_[V_[3 * t + 1]], P_[V_[3 * t + 2]], p) > 0.0) return t;
    throw Error("triangulation failed: point location stalled");
  }

  void insert(int pid) {
    const Point p = P_[pid];
    const int start = locate(p);
    ++epoch_;
    cavity_.clear();
    cavity_.push_back(start);
    mark_[start] = incav_[start] = epoch_;
    for (size_t i = 0; i < cavity_.size(); ++i) {
      const int t = cavity_[i];
      for (int k = 0; k < 3; ++k) {
        const int nb = A_[3 * t + k];
        if (nb == -1 || mark_[nb] == epoch_) continue;
        mark_[nb] = epoch_;
        if (incircle(P_[V_[3 * nb]], P_[V_[3 * nb + 1]], P_[V_[3 * nb + 2]], p) > 0.0) {
          incav_[nb] = epoch_;
          cavity_.push_back(nb);
        }
      }
    }
    rim_.clear();
    for (const int t : cavity_)
      for (int k = 0; k < 3; ++k) {
        const int nb = A_[3 * t + k];
        if (nb == -1 || incav_[nb] != epoch_) rim_.push_back({V_[3 * t + k], V_[3 * t + (k + 1) % 3], nb});
      }
    for (const int t : cavity_) {
      alive_[t] = 0;
      free_.push_back(t);
    }
    // one triangle (a, b, p) per rim edge; the rim must be a simple cycle
    std::vector<int> ids(rim_.size());
    for (size_t i = 0; i < rim_.size(); ++i) {
      const RimEdge& e = rim_[i];
      if (vmark_[e.a] == pid && vstart_[e.a] != -1) throw Error("triangulation failed: cavity rim is not a simple cycle");
      if (vmark_[e.a] != pid) {
        vmark_[e.a] = pid;
        vstart_[e.a] = vend_[e.a] = -1;
      }
      if (vmark_[e.b] != pid) {
        vmark_[e.b] = pid;
        vstart_[e.b] = vend_[e.b] = -1;
      }
      if (vend_[e.b] != -1) throw Error("triangulation failed: cavity rim is not a simple cycle");
      const int id = new_tri(e.a, e.b, pid);
      ids[i] = id;
      vstart_[e.a] = id;
      vend_[e.b] = id;
      A_[3 * id] = e.out;
      if (e.out != -1) {
        int* ov = &V_[3 * e.out];
        for (int k = 0; k < 3; ++k)
          if (ov[k] == e.b && ov[(k + 1) % 3] == e.a) A_[3 * e.out + k] = id;
      }
      vtri_[e.a] = vtri_[e.b] = id;
    }
    for (size_t i = 0; i < rim_.size(); ++i) {
      const int id = ids[i];
      const int sb = vstart_[rim_[i].b], ea = vend_[rim_[i].a];
      if (sb == -1 || ea == -1) throw Error("triangulation failed: cavity rim is not a simple cycle");
      A_[3 * id + 1] = sb;  // edge (b, p) <-> sibling starting at b
      A_[3 * id + 2] = ea;  // edge (p, a) <-> sibling ending at a
    }
    if (!ids.empty()) {
      last_ = ids[0];
      vtri_[pid] = ids[0];
    }
    cell_[cell_of(p)] = pid;
  }
};

// The reference's sequential redraw rule, used only if a near-duplicate actually occurs.
std::vector<Point> points_sequential(const GenSpec& spec) {
  constexpr double kSep = 1e-12;
  SplitMix64 rng(spec.seed);
  std::vector<Point> pts;
  pts.reserve(spec.n_points);
  std::unordered_map<uint64_t, std::vector<int>> grid;
  auto cell = [](double v) { return static_cast<int64_t>(std::floor(v / kSep)); };
  auto key = [](int64_t ix, int64_t iy) {
    return static_cast<uint64_t>(ix) * 0x9E3779B97F4A7C15ULL ^ static_cast<uint64_t>(iy) * 0xC2B2AE3D27D4EB4FULL;
  };
  while (static_cast<int>(pts.size()) < spec.n_points) {
    const double x = rng.uniform01();
    const double y = rng.uniform01();
    const Point p{x, y};
    const int64_t ix = cell(p.x), iy = cell(p.y);
    bool clash = false;
    for (int64_t dx = -1; dx <= 1 && !clash; ++dx)
      for (int64_t dy = -1; dy <= 1 && !clash; ++dy) {
        const auto it = grid.find(key(ix + dx, iy + dy));
        if (it == grid.end()) continue;
        for (const int id : it->second)
          if (std::abs(pts[id].x - p.x) <= kSep && std::abs(pts[id].y - p.y) <= kSep) {
            clash = true;
            break;
          }
      }
    if (clash) continue;
    grid[key(ix, iy)].push_back(static_cast<int>(pts.size()));
    pts.push_back(p);
  }
  return pts;
}

}  // namespace

std::vector<Point> generate_points(const GenSpec& spec) {
  if (spec.n_points < 3) throw Error("point generation needs n >= 3");
  // Fast path: draw n points, then prove no pair is within 1e-12 (L-inf).  If the proof
  // fails, replay the reference's sequential redraw rule, which then differs.
  SplitMix64 rng(spec.seed);
  std::vector<Point> pts(spec.n_points);
  for (Point& p : pts) {
    p.x = rng.uniform01();
    p.y = rng.uniform01();
  }
  std::vector<int> idx(pts.size());
  std::iota(idx.begin(), idx.end(), 0);
  std::sort(idx.begin(), idx.end(), [&](int a, int b) { return pts[a].x < pts[b].x; });
  for (size_t i = 0; i < idx.size(); ++i)
    for (size_t j = i + 1; j < idx.size() && pts[idx[j]].x - pts[idx[i]].x <= 1e-12; ++j)
      if (std::abs(pts[idx[j]].y - pts[idx[i]].y) <= 1e-12) return points_sequential(spec);
  return pts;
}

std::vector<std::array<int, 3>> delaunay_triangulate(const std::vector<Point>& points) {
  if (points.size() < 3) throw Error("triangulation needs at least 3 points");
  return Triangulator(points).run(false);
}

std::vector<std::array<int, 3>> delaunay_triangulate_spatial(const std::vector<Point>& points) {
  if (points.size() < 3) throw Error("triangulation needs at least 3 points");
  return Triangulator(points).run(true);
}

MeshSource perturbed_grid(int rows, int cols, double perturbation, uint64_t seed) {
  if (rows < 2 || cols < 2) throw Error("grid needs rows and cols >= 2");
  if (!(perturbation >= 0.0 && perturbation <= 0.49)) throw Error("perturbation must be in [0, 0.49]");
  SplitMix64 rng(seed);
  const double hx = 1.0 / (cols - 1), hy = 1.0 / (rows - 1);
  MeshSource src;
  src.points.resize(static_cast<size_t>(rows) * cols);
  for (int r = 0; r < rows; ++r) {
    const bool inner_row = r > 0 && r < rows - 1;
    for (int c = 0; c < cols; ++c) {
      Point q{c * hx, r * hy};
      if (inner_row && c > 0 && c < cols - 1) {
        // x draw first, then y (the stream order is part of the fixture)
        q.x += (2.0 * rng.uniform01() - 1.0) * perturbation * hx;
        q.y += (2.0 * rng.uniform01() - 1.0) * perturbation * hy;
      }
      src.points[static_cast<size_t>(r) * cols + c] = q;
    }
  }
  src.triangles.reserve(2 * static_cast<size_t>(rows - 1) * (cols - 1));
  for (int r = 0; r + 1 < rows; ++r)
    for (int c = 0; c + 1 < cols; ++c) {
      const int a = r * cols + c, b = a + 1, d = a + cols, e = d + 1;
      src.triangles.push_back({a, b, e});
      src.triangles.push_back({a, e, d});
    }
  return src;
}

MeshSource generate(const GenSpec& spec) {
  if (spec.kind == GenKind::PerturbedGrid)
    return perturbed_grid(spec.rows, spec.cols, spec.perturbation, spec.seed);
  MeshSource src;
  src.points = generate_points(spec);
  // Up to 2M points keep the reference's insertion order verbatim; beyond (sizes the
  // reference cannot triangulate in reasonable time) insert along a Hilbert curve.
  src.triangles = spec.n_points <= (1 << 21) ? delaunay_triangulate(src.points)
                                             : delaunay_triangulate_spatial(src.points);
  return src;
}

MeshSource graded_mesh(int n_points, uint64_t seed, double hub_fraction, int max_valence) {
  if (n_points < 64) throw Error("graded_mesh needs n >= 64");
  if (!(hub_fraction >= 0.0 && hub_fraction < 0.05)) throw Error("hub_fraction must be in [0, 0.05)");
  if (max_valence < 32) throw Error("max_valence must be >= 32");
  SplitMix64 rng(seed);
  // Density 1 + 3x on [0,1]^2: x by inverse CDF of (x + 1.5 x^2) / 2.5.
  auto draw_x = [&](double u) { return (-1.0 + std::sqrt(1.0 + 6.0 * 2.5 * u)) / 3.0; };
  const double mean_h = 1.0 / std::sqrt(static_cast<double>(n_points));
  auto local_h = [&](double x) { return mean_h * std::sqrt(2.5 / (1.0 + 3.0 * x)); };

  // Hubs: valence classes 32, 64, ... max_valence; each doubling halves the count.
  struct Hub {
    double x, y, r;
    int m;
  };
  std::vector<Hub> hubs;
  const int n_hubs = static_cast<int>(hub_fraction * n_points);
  {
    std::vector<int> valences;
    for (int m = 32; m <= max_valence; m *= 2) valences.push_back(m);
    double wsum = 0.0;
    for (size_t i = 0; i < valences.size(); ++i) wsum += std::ldexp(1.0, -static_cast<int>(i));
    // grid of candidate sites keeps hubs disjoint
    const int side = std::max(1, static_cast<int>(std::ceil(std::sqrt(2.0 * n_hubs + 1))));
    std::vector<int> sites(static_cast<size_t>(side) * side);
    std::iota(sites.begin(), sites.end(), 0);
    for (size_t i = sites.size(); i > 1; --i) std::swap(sites[i - 1], sites[rng.next() % i]);
    int placed = 0;
    for (size_t cls = 0; cls < valences.size() && placed < n_hubs; ++cls) {
      int cnt = static_cast<int>(std::llround(n_hubs * std::ldexp(1.0, -static_cast<int>(cls)) / wsum));
      if (cls + 1 == valences.size()) cnt = n_hubs - placed;
      cnt = std::max(cnt, 1);
      for (int j = 0; j < cnt && placed < n_hubs; ++j, ++placed) {
        const int site = sites[placed];
        const double cx = (site % side + 0.5) / side, cy = (site / side + 0.5) / side;
        const int m = valences[cls];
        // rim spacing about half the local spacing, capped so hubs stay inside their site
        const double r = std::min(0.5 * m * local_h(cx) / (2.0 * kPi), 0.45 / side);
        hubs.push_back({cx, cy, r, m});
      }
    }
  }
  // Background points outside every hub disk, then hub centres and rims.
  std::vector<Point> pts;
  pts.reserve(static_cast<size_t>(n_points) + 64);
  const int side = std::max(1, static_cast<int>(std::ceil(std::sqrt(2.0 * n_hubs + 1))));
  std::vector<std::vector<int>> site_hub(static_cast<size_t>(side) * side);
  for (size_t h = 0; h < hubs.size(); ++h) {
    const int sx = std::min(side - 1, static_cast<int>(hubs[h].x * side));
    const int sy = std::min(side - 1, static_cast<int>(hubs[h].y * side));
    site_hub[static_cast<size_t>(sy) * side + sx].push_back(static_cast<int>(h));
  }
  int64_t rim_total = 0;
  for (const Hub& h : hubs) rim_total += h.m + 1;
  const int64_t background = std::max<int64_t>(16, n_points - rim_total);
  while (static_cast<int64_t>(pts.size()) < background) {
    const double x = draw_x(rng.uniform01()), y = rng.uniform01();
    const int sx = std::min(side - 1, static_cast<int>(x * side)), sy = std::min(side - 1, static_cast<int>(y * side));
    bool in_hub = false;
    for (const int h : site_hub[static_cast<size_t>(sy) * side + sx]) {
      const double dx = x - hubs[h].x, dy = y - hubs[h].y;
      if (dx * dx + dy * dy <= (1.05 * hubs[h].r) * (1.05 * hubs[h].r)) in_hub = true;
    }
    if (!in_hub) pts.push_back({x, y});
  }
  for (const Hub& h : hubs) {
    pts.push_back({h.x, h.y});
    const double phase = rng.uniform01() * 2.0 * kPi / h.m;
    for (int k = 0; k < h.m; ++k) {
      const double a = phase + 2.0 * kPi * k / h.m;
      pts.push_back({h.x + h.r * std::cos(a), h.y + h.r * std::sin(a)});
    }
  }
  MeshSource src;
  src.triangles = delaunay_triangulate_spatial(pts);
  src.points = std::move(pts);
  return src;
}

}  // namespace trismooth
