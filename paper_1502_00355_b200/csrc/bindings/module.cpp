// _trismooth: pybind11 module with the reference's Python surface
// (proj/bindings/module.cpp:45-205: Mesh, triangle_alpha, build_mesh, generate_delaunay,
// generate_grid, smooth, quality_summary, read_mesh, write_mesh, convert_layout — same
// argument names, defaults, return keys and exception mapping), whose smooth() runs on the
// B200 through libtsg.so.  B200 additions are trailing keyword arguments and the numpy-level
// helpers at the bottom (topology, *_arrays, DeviceMesh) used by the benchmark and tests.
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <csignal>
#include <cstdlib>
#include <cstring>

#include <execinfo.h>
#include <unistd.h>

#include "trismooth/gpu.hpp"
#include "trismooth/io.hpp"
#include "trismooth/meshgen.hpp"
#include "trismooth/quality.hpp"
#include "trismooth/smoothing.hpp"
#include "trismooth/topology.hpp"
#include "tsg.h"

namespace py = pybind11;
using namespace trismooth;

namespace {

Layout parse_layout(const std::string& s) {
  if (s == "aos") return Layout::AoS;
  if (s == "soa") return Layout::SoA;
  throw std::invalid_argument("layout must be 'aos' or 'soa'");
}
IterationForm parse_form(const std::string& s) {
  if (s == "a") return IterationForm::A;
  if (s == "b") return IterationForm::B;
  throw std::invalid_argument("form must be 'a' or 'b'");
}
UpdateStrategy parse_strategy(const std::string& s) {
  if (s == "fused") return UpdateStrategy::Fused;
  if (s == "twophase") return UpdateStrategy::TwoPhase;
  throw std::invalid_argument("strategy must be 'fused' or 'twophase'");
}
Backend parse_backend(const std::string& s) {
  if (s == "serial") return Backend::Serial;
  if (s == "parallel") return Backend::Parallel;
  throw std::invalid_argument("backend must be 'serial' or 'parallel'");
}
Precision parse_precision(const std::string& s) {
  if (s == "f64") return Precision::F64;
  if (s == "f32") return Precision::F32;
  throw std::invalid_argument("precision must be 'f64' or 'f32'");
}
Reorder parse_reorder(const std::string& s) {
  if (s == "auto") return Reorder::Auto;
  if (s == "none") return Reorder::None;
  if (s == "hilbert") return Reorder::Hilbert;
  throw std::invalid_argument("reorder must be 'auto', 'none' or 'hilbert'");
}
SwapMode parse_swap(const std::string& s) {
  if (s == "pingpong") return SwapMode::PingPong;
  if (s == "copy") return SwapMode::Copy;
  throw std::invalid_argument("swap must be 'pingpong' or 'copy'");
}

SmoothConfig make_config(const std::string& form, const std::string& strategy,
                         const std::string& backend, int workers, int max_iters, double move_tol,
                         const std::string& precision, const std::string& reorder,
                         const std::string& swap, bool use_graph) {
  SmoothConfig c;
  c.form = parse_form(form);
  c.strategy = parse_strategy(strategy);
  c.backend = parse_backend(backend);
  c.workers = workers;
  c.max_iters = max_iters;
  c.move_tol = move_tol;
  c.precision = parse_precision(precision);
  c.reorder = parse_reorder(reorder);
  c.swap = parse_swap(swap);
  c.use_graph = use_graph;
  return c;
}

using F64Array = py::array_t<double, py::array::c_style | py::array::forcecast>;
using I32Array = py::array_t<int32_t, py::array::c_style | py::array::forcecast>;

template <class T>
py::array_t<T> to_numpy(std::vector<T>&& v, std::vector<py::ssize_t> shape) {
  auto* heap = new std::vector<T>(std::move(v));
  py::capsule owner(heap, [](void* p) { delete static_cast<std::vector<T>*>(p); });
  return py::array_t<T>(shape, heap->data(), owner);
}

py::tuple source_arrays(MeshSource&& src) {
  const py::ssize_t nv = static_cast<py::ssize_t>(src.points.size());
  const py::ssize_t nt = static_cast<py::ssize_t>(src.triangles.size());
  std::vector<double> xy(2 * nv);
  std::memcpy(xy.data(), src.points.data(), sizeof(double) * 2 * nv);
  std::vector<int32_t> tri(3 * nt);
  std::memcpy(tri.data(), src.triangles.data(), sizeof(int32_t) * 3 * nt);
  return py::make_tuple(to_numpy(std::move(xy), {nv, 2}), to_numpy(std::move(tri), {nt, 3}));
}

py::dict stats_dict(const RunStats& s, bool detailed) {
  py::dict d;
  d["iterations"] = s.iterations;
  d["stop"] = std::string(to_string(s.stop));
  d["init_ms"] = s.init_ms;
  d["topo_ms"] = s.topo_ms;
  d["constr_ms"] = s.constr_ms;
  d["iter_ms"] = s.iter_ms;
  d["total_ms"] = s.total_ms;
  d["min_alpha_before"] = s.min_alpha_before;
  d["min_alpha_after"] = s.min_alpha_after;
  d["mean_alpha_before"] = s.mean_alpha_before;
  d["mean_alpha_after"] = s.mean_alpha_after;
  d["accepted_per_pass"] = s.accepted_per_pass;
  if (detailed) {
    d["max_disp_per_pass"] = s.max_disp_per_pass;
    d["device_ms"] = s.device_ms;
    d["upload_ms"] = s.upload_ms;
    d["kernel_launches"] = s.kernel_launches;
  }
  return d;
}

gpu::Topology64 topology_from_dict(const py::dict& t) {
  gpu::Topology64 T;
  auto grab64 = [&](const char* k, std::vector<int64_t>& out) {
    auto a = py::array_t<int64_t, py::array::c_style | py::array::forcecast>::ensure(t[k]);
    out.assign(a.data(), a.data() + a.size());
  };
  auto grab32 = [&](const char* k, std::vector<int32_t>& out) {
    auto a = I32Array::ensure(t[k]);
    out.assign(a.data(), a.data() + a.size());
  };
  grab64("nbr_off", T.nbr_off);
  grab64("inc_off", T.inc_off);
  grab32("nbr", T.nbr);
  grab32("inc", T.inc);
  auto b = py::array_t<uint8_t, py::array::c_style | py::array::forcecast>::ensure(t["boundary"]);
  T.boundary.assign(b.data(), b.data() + b.size());
  return T;
}

}  // namespace

namespace {
// TSG_SEGV_TRACE=1: print the native stack of a crashing thread (debug aid; glibc backtrace).
void segv_trace(int sig) {
  void* frames[64];
  const int n = backtrace(frames, 64);
  backtrace_symbols_fd(frames, n, 2);
  std::signal(sig, SIG_DFL);
  std::raise(sig);
}
}  // namespace

PYBIND11_MODULE(_trismooth, m) {
  m.doc() = "Smart Laplacian smoothing of planar triangular meshes (B200 engine)";
  if (std::getenv("TSG_SEGV_TRACE")) std::signal(SIGSEGV, segv_trace);

  py::class_<Mesh>(m, "Mesh")
      .def_property_readonly("vertex_count", &Mesh::vertex_count)
      .def_property_readonly("triangle_count", &Mesh::triangle_count)
      .def_property_readonly("layout", [](const Mesh& x) { return std::string(to_string(x.layout())); })
      .def("points",
           [](const Mesh& x) {
             std::vector<std::pair<double, double>> out(x.vertex_count());
             x.visit([&](const auto& s) {
               for (int v = 0; v < s.vertex_count(); ++v) out[v] = {s.position(v).x, s.position(v).y};
             });
             return out;
           })
      .def("triangles",
           [](const Mesh& x) {
             std::vector<std::array<int, 3>> out(x.triangle_count());
             x.visit([&](const auto& s) {
               for (int t = 0; t < s.triangle_count(); ++t) out[t] = s.tri(t);
             });
             return out;
           })
      .def("boundary",
           [](const Mesh& x) {
             std::vector<bool> out(x.vertex_count());
             x.visit([&](const auto& s) {
               for (int v = 0; v < s.vertex_count(); ++v) out[v] = s.is_boundary(v);
             });
             return out;
           })
      // --- B200 additions: numpy views of the same data ---
      .def("points_array",
           [](const Mesh& x) {
             std::vector<double> xy(2 * static_cast<size_t>(x.vertex_count()));
             x.visit([&](const auto& s) {
               for (int v = 0; v < s.vertex_count(); ++v) {
                 xy[2 * v] = s.position(v).x;
                 xy[2 * v + 1] = s.position(v).y;
               }
             });
             return to_numpy(std::move(xy), {x.vertex_count(), 2});
           })
      .def("triangles_array",
           [](const Mesh& x) {
             std::vector<int32_t> t3(3 * static_cast<size_t>(x.triangle_count()));
             x.visit([&](const auto& s) {
               for (int t = 0; t < s.triangle_count(); ++t) {
                 const auto c = s.tri(t);
                 t3[3 * t] = c[0], t3[3 * t + 1] = c[1], t3[3 * t + 2] = c[2];
               }
             });
             return to_numpy(std::move(t3), {x.triangle_count(), 3});
           })
      .def("tri_alphas",
           [](const Mesh& x) {
             std::vector<double> q(x.triangle_count());
             x.visit([&](const auto& s) {
               for (int t = 0; t < s.triangle_count(); ++t) q[t] = s.tri_quality(t);
             });
             return to_numpy(std::move(q), {x.triangle_count()});
           })
      .def("vertex_minima",
           [](const Mesh& x) {
             std::vector<double> q(x.vertex_count());
             x.visit([&](const auto& s) {
               for (int v = 0; v < s.vertex_count(); ++v) q[v] = s.vertex_min_quality(v);
             });
             return to_numpy(std::move(q), {x.vertex_count()});
           })
      .def("__repr__", [](const Mesh& x) {
        return "Mesh(" + std::to_string(x.vertex_count()) + " vertices, " +
               std::to_string(x.triangle_count()) + " triangles, " + to_string(x.layout()) + ")";
      });

  m.def(
      "triangle_alpha",
      [](std::pair<double, double> p1, std::pair<double, double> p2, std::pair<double, double> p3) {
        return triangle_alpha({p1.first, p1.second}, {p2.first, p2.second}, {p3.first, p3.second});
      },
      py::arg("p1"), py::arg("p2"), py::arg("p3"),
      "Normalized shape quality: 1 equilateral, 0 degenerate, < 0 inverted.");

  m.def(
      "build_mesh",
      [](const std::vector<std::pair<double, double>>& points,
         const std::vector<std::array<int, 3>>& triangles, const std::string& layout) {
        std::vector<Point> pts(points.size());
        for (size_t i = 0; i < points.size(); ++i) pts[i] = {points[i].first, points[i].second};
        return build_mesh(pts, triangles, parse_layout(layout));
      },
      py::arg("points"), py::arg("triangles"), py::arg("layout") = "aos");

  m.def(
      "generate_delaunay",
      [](int n, uint64_t seed, const std::string& layout) {
        const Layout l = parse_layout(layout);
        GenSpec spec;
        spec.kind = GenKind::DelaunayRandom;
        spec.n_points = n;
        spec.seed = seed;
        const MeshSource src = generate(spec);
        return build_mesh(src.points, src.triangles, l);
      },
      py::arg("n"), py::arg("seed") = 1, py::arg("layout") = "aos",
      "Seeded uniform points in the unit square, Delaunay-triangulated.");

  m.def(
      "generate_grid",
      [](int rows, int cols, double perturbation, uint64_t seed, const std::string& layout) {
        const Layout l = parse_layout(layout);
        const MeshSource src = perturbed_grid(rows, cols, perturbation, seed);
        return build_mesh(src.points, src.triangles, l);
      },
      py::arg("rows"), py::arg("cols"), py::arg("perturbation") = 0.3, py::arg("seed") = 1,
      py::arg("layout") = "aos");

  m.def(
      "smooth",
      [](Mesh& mesh, const std::string& form, const std::string& strategy, const std::string& backend,
         int workers, int max_iters, double move_tol, const std::string& precision,
         const std::string& reorder, const std::string& swap, bool use_graph, bool detailed) {
        const SmoothConfig cfg = make_config(form, strategy, backend, workers, max_iters, move_tol,
                                             precision, reorder, swap, use_graph);
        RunStats rs;
        {
          // the passes take the device for a while: let other Python threads run (calls on
          // the shared device context are serialised inside libtsg)
          py::gil_scoped_release nogil;
          rs = smooth(mesh, cfg);
        }
        return stats_dict(rs, detailed);
      },
      py::arg("mesh"), py::arg("form") = "b", py::arg("strategy") = "twophase",
      py::arg("backend") = "serial", py::arg("workers") = 1, py::arg("max_iters") = 100,
      py::arg("move_tol") = 1e-6, py::arg("precision") = "f64", py::arg("reorder") = "auto",
      py::arg("swap") = "pingpong", py::arg("use_graph") = true, py::arg("detailed") = false,
      "Smooth in place on the GPU; returns run statistics.");

  // quality_summary (proj/bindings/module.cpp:157-185): same keys and values; the α field and
  // its min / max / non-positive count come from the device audit (csrc/tsg_quality.cu), the
  // mean is the sequential sum in triangle order, the flags from the host topology.
  m.def(
      "quality_summary",
      [](Mesh& mesh) {
        init_flags(mesh);
        const QualityReport q = audit_tri_alphas(mesh);
        const Adjacency adj = find_neighbors(mesh);
        determine_constraints(mesh, adj);
        int pinned = 0;
        mesh.visit([&](const auto& s) {
          for (int v = 0; v < s.vertex_count(); ++v) pinned += s.is_boundary(v) ? 1 : 0;
        });
        py::dict d;
        d["min_alpha"] = q.min_alpha;
        d["mean_alpha"] = q.mean_alpha;
        d["max_alpha"] = q.max_alpha;
        d["non_positive"] = q.non_positive;
        d["boundary_vertices"] = pinned;
        d["interior_vertices"] = mesh.vertex_count() - pinned;
        return d;
      },
      py::arg("mesh"));

  // B200 addition: the `trismooth quality` report (proj/tools/main.cpp:151-208) without the
  // CLI: quality_summary's keys plus the 20-bin histogram, on the device.
  m.def(
      "quality_report",
      [](Mesh& mesh) {
        const QualityReport q = audit_tri_alphas(mesh);
        py::dict d;
        d["triangles"] = mesh.triangle_count();
        d["vertices"] = mesh.vertex_count();
        d["min_alpha"] = q.min_alpha;
        d["mean_alpha"] = q.mean_alpha;
        d["max_alpha"] = q.max_alpha;
        d["non_positive"] = q.non_positive;
        d["histogram_bins"] = q.histogram;
        return d;
      },
      py::arg("mesh"));

  m.def(
      "compute_all_qualities", [](Mesh& mesh) { compute_all_qualities(mesh); }, py::arg("mesh"),
      "α of every triangle into the mesh (device audit kernel).");
  m.def(
      "reduce_vertex_minima", [](Mesh& mesh) { reduce_vertex_minima(mesh); }, py::arg("mesh"),
      "Per-vertex minimum of the stored incident α (device audit kernel); needs adjacency.");
  m.def(
      "update_two_phase", [](Mesh& mesh) { update_two_phase(mesh); }, py::arg("mesh"));

  m.def(
      "read_mesh",
      [](const std::string& node, const std::string& ele, const std::string& layout) {
        return read_mesh_files(node, ele, parse_layout(layout));
      },
      py::arg("node"), py::arg("ele"), py::arg("layout") = "aos");

  m.def(
      "write_binary",
      [](const std::string& path, F64Array xy, I32Array tri) {
        write_mesh_binary(path, xy.data(), xy.size() / 2, tri.data(), tri.size() / 3);
      },
      py::arg("path"), py::arg("xy"), py::arg("tri"),
      "Binary mesh file (TSGMESH1: sizes, float64 xy, int32 corners) — the fast path beside .node/.ele.");
  m.def(
      "read_binary",
      [](const std::string& path) {
        BinaryMesh b;
        {
          py::gil_scoped_release nogil;
          b = read_mesh_binary(path);
        }
        const int64_t nv = b.nv, nt = b.nt;
        return py::make_tuple(to_numpy(std::move(b.xy), {static_cast<py::ssize_t>(nv), 2}),
                              to_numpy(std::move(b.tri), {static_cast<py::ssize_t>(nt), 3}));
      },
      py::arg("path"));

  m.def(
      "write_mesh", [](const Mesh& mesh, const std::string& prefix) { write_mesh_files(mesh, prefix); },
      py::arg("mesh"), py::arg("prefix"), "Writes <prefix>.node and <prefix>.ele.");

  m.def(
      "convert_layout",
      [](const Mesh& mesh, const std::string& layout) { return convert_layout(mesh, parse_layout(layout)); },
      py::arg("mesh"), py::arg("layout"));

  // ------------------------------------------------------------------ B200 additions
  m.def(
      "delaunay_arrays",
      [](int n, uint64_t seed) {
        GenSpec spec;
        spec.kind = GenKind::DelaunayRandom;
        spec.n_points = n;
        spec.seed = seed;
        MeshSource src;
        {
          py::gil_scoped_release nogil;
          src = generate(spec);
        }
        return source_arrays(std::move(src));
      },
      py::arg("n"), py::arg("seed") = 1, "(xy float64 (n,2), tri int32 (nt,3)) of generate_delaunay.");
  m.def(
      "grid_arrays",
      [](int rows, int cols, double perturbation, uint64_t seed) {
        return source_arrays(perturbed_grid(rows, cols, perturbation, seed));
      },
      py::arg("rows"), py::arg("cols"), py::arg("perturbation") = 0.3, py::arg("seed") = 1);
  m.def(
      "graded_arrays",
      [](int n, uint64_t seed, double hub_fraction, int max_valence) {
        MeshSource src;
        {
          py::gil_scoped_release nogil;
          src = graded_mesh(n, seed, hub_fraction, max_valence);
        }
        return source_arrays(std::move(src));
      },
      py::arg("n"), py::arg("seed") = 1, py::arg("hub_fraction") = 1e-3, py::arg("max_valence") = 1024);
  m.def(
      "triangulate",
      [](F64Array xy, bool spatial) {
        std::vector<Point> pts(xy.size() / 2);
        std::memcpy(static_cast<void*>(pts.data()), xy.data(), sizeof(double) * 2 * pts.size());
        std::vector<std::array<int, 3>> tris;
        {
          py::gil_scoped_release nogil;
          tris = spatial ? delaunay_triangulate_spatial(pts) : delaunay_triangulate(pts);
        }
        std::vector<int32_t> t3(3 * tris.size());
        std::memcpy(t3.data(), tris.data(), sizeof(int32_t) * t3.size());
        return to_numpy(std::move(t3), {static_cast<py::ssize_t>(tris.size()), 3});
      },
      py::arg("xy"), py::arg("spatial") = false);
  m.def(
      "topology",
      [](int64_t nv, I32Array tri) {
        gpu::Topology64 T;
        {
          py::gil_scoped_release nogil;
          T = gpu::build_topology(nv, tri.data(), tri.size() / 3);
        }
        py::dict d;
        const py::ssize_t n1 = static_cast<py::ssize_t>(T.nbr_off.size());
        const py::ssize_t nn = static_cast<py::ssize_t>(T.nbr.size());
        const py::ssize_t ni = static_cast<py::ssize_t>(T.inc.size());
        d["nbr_off"] = to_numpy(std::move(T.nbr_off), {n1});
        d["nbr"] = to_numpy(std::move(T.nbr), {nn});
        d["inc_off"] = to_numpy(std::move(T.inc_off), {n1});
        d["inc"] = to_numpy(std::move(T.inc), {ni});
        d["boundary"] = to_numpy(std::move(T.boundary), {static_cast<py::ssize_t>(nv)});
        return d;
      },
      py::arg("nv"), py::arg("tri"), "Unique-neighbour / incident CSR (int64 offsets) and pins.");
  m.def("bbox_diagonal", [](F64Array xy) { return gpu::bbox_diagonal(xy.data(), xy.size() / 2); });
  m.def("device_count", []() { return tsg_device_count(); });

  py::class_<gpu::DeviceMesh>(m, "DeviceMesh")
      .def(py::init([](F64Array xy, I32Array tri, const py::dict& topo, const std::string& layout,
                       const std::string& precision, bool reorder) {
             const gpu::Topology64 T = topology_from_dict(topo);
             return std::make_unique<gpu::DeviceMesh>(xy.data(), static_cast<int64_t>(xy.size() / 2),
                                                      tri.data(), static_cast<int64_t>(tri.size() / 3), T,
                                                      parse_layout(layout), parse_precision(precision), reorder);
           }),
           py::arg("xy"), py::arg("tri"), py::arg("topology"), py::arg("layout") = "aos",
           py::arg("precision") = "f64", py::arg("reorder") = false)
      .def_property_readonly("vertex_count", &gpu::DeviceMesh::vertex_count)
      .def_property_readonly("triangle_count", &gpu::DeviceMesh::triangle_count)
      .def_property_readonly("device_bytes", &gpu::DeviceMesh::device_bytes)
      .def_property_readonly("reordered", &gpu::DeviceMesh::reordered)
      .def_property_readonly("handle", [](const gpu::DeviceMesh& d) { return reinterpret_cast<uintptr_t>(d.handle()); })
      .def("set_coords", [](gpu::DeviceMesh& d, F64Array xy) { d.set_coords(xy.data()); })
      .def("get_coords",
           [](const gpu::DeviceMesh& d) {
             std::vector<double> xy(2 * d.vertex_count());
             d.get_coords(xy.data());
             return to_numpy(std::move(xy), {static_cast<py::ssize_t>(d.vertex_count()), 2});
           })
      .def("tri_alpha",
           [](const gpu::DeviceMesh& d) {
             std::vector<double> q(d.triangle_count());
             d.tri_alpha(q.data());
             return to_numpy(std::move(q), {static_cast<py::ssize_t>(d.triangle_count())});
           })
      .def("vertex_minima",
           [](const gpu::DeviceMesh& d) {
             std::vector<double> q(d.vertex_count());
             d.vertex_minima(q.data());
             return to_numpy(std::move(q), {static_cast<py::ssize_t>(d.vertex_count())});
           })
      .def(
          "run",
          [](gpu::DeviceMesh& d, double bbox_diag, const std::string& form, const std::string& strategy,
             const std::string& backend, int workers, int max_iters, double move_tol,
             const std::string& swap, bool use_graph) {
            const SmoothConfig cfg = make_config(form, strategy, backend, workers, max_iters, move_tol,
                                                 "f64", "none", swap, use_graph);
            RunStats s;
            {
              py::gil_scoped_release nogil;
              s = d.run(cfg, bbox_diag);
            }
            return stats_dict(s, true);
          },
          py::arg("bbox_diag"), py::arg("form") = "a", py::arg("strategy") = "fused",
          py::arg("backend") = "serial", py::arg("workers") = 1, py::arg("max_iters") = 100,
          py::arg("move_tol") = 0.0, py::arg("swap") = "pingpong", py::arg("use_graph") = true);
}
