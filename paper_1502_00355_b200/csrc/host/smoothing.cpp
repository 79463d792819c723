// smooth() on the B200 (include/trismooth/smoothing.hpp) and the device-mesh plumbing of
// include/trismooth/gpu.hpp.
//
// Pipeline and statistics follow proj/src/smoothing.cpp:146-182; the pass loop
// (:76-142) runs in libtsg.so as one CUDA-graph launch.  Host prep (adjacency,
// constraints, locality order) stays in C++ on the host, as in the reference.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <string>

#include "trismooth/gpu.hpp"
#include "trismooth/smoothing.hpp"
#include "trismooth/topology.hpp"
#include "tsg.h"

namespace trismooth {

const char* to_string(IterationForm form) { return form == IterationForm::B ? "b" : "a"; }
const char* to_string(UpdateStrategy s) { return s == UpdateStrategy::TwoPhase ? "twophase" : "fused"; }
const char* to_string(Backend b) { return b == Backend::Parallel ? "parallel" : "serial"; }
const char* to_string(Precision p) { return p == Precision::F32 ? "f32" : "f64"; }
const char* to_string(StopReason r) {
  switch (r) {
    case StopReason::NoMoves: return "no_moves";
    case StopReason::Displacement: return "displacement";
    case StopReason::MaxIters: return "max_iters";
  }
  return "?";
}

void validate(const SmoothConfig& c) {
  if (c.workers < 1) throw Error("workers must be >= 1");
  if (c.max_iters < 1) throw Error("max_iters must be >= 1");
  if (!(c.move_tol >= 0.0)) throw Error("move_tol must be >= 0");
}

namespace gpu {

void check(int status, const char* what) {
  if (status != TSG_OK) throw Error(std::string(what) + ": " + tsg_last_error());
}

tsg_context* default_context() {
  static std::mutex mu;
  static tsg_context* ctx = nullptr;
  std::lock_guard<std::mutex> lk(mu);
  if (!ctx) {
    int dev = 0;
    if (const char* e = std::getenv("TSG_DEVICE")) dev = std::atoi(e);
    else if (const char* r = std::getenv("LOCAL_RANK")) dev = std::atoi(r);
    const int n = tsg_device_count();
    if (n <= 0) throw Error("trismooth: no CUDA device available (the B200 engine has no CPU fallback)");
    check(tsg_context_create(dev % n, &ctx), "tsg_context_create");
  }
  return ctx;
}

double bbox_diagonal(const double* xy, int64_t nv) {
  double xmin = std::numeric_limits<double>::infinity(), xmax = -xmin, ymin = xmin, ymax = -xmin;
  for (int64_t v = 0; v < nv; ++v) {
    xmin = std::min(xmin, xy[2 * v]);
    xmax = std::max(xmax, xy[2 * v]);
    ymin = std::min(ymin, xy[2 * v + 1]);
    ymax = std::max(ymax, xy[2 * v + 1]);
  }
  return std::hypot(xmax - xmin, ymax - ymin);
}

DeviceMesh::DeviceMesh(const double* xy, int64_t nv, const int32_t* tri, int64_t nt,
                       const Topology64& topo, Layout layout, Precision precision, bool reorder,
                       tsg_context* ctx)
    : nv_(nv), nt_(nt), reordered_(reorder) {
  if (!ctx) ctx = default_context();
  std::vector<int64_t> order;
  if (reorder) {
    order.resize(nv);
    check(tsg_hilbert_order(nv, xy, order.data()), "tsg_hilbert_order");
  }
  tsg_mesh_desc d{};
  d.nv = nv;
  d.nt = nt;
  d.xy = xy;
  d.tri = tri;
  d.nbr_off = topo.nbr_off.data();
  d.nbr = topo.nbr.data();
  d.inc_off = topo.inc_off.data();
  d.inc = topo.inc.data();
  d.boundary = topo.boundary.data();
  d.order = reorder ? order.data() : nullptr;
  d.layout = layout == Layout::SoA ? TSG_LAYOUT_SOA : TSG_LAYOUT_AOS;
  d.precision = precision == Precision::F32 ? TSG_F32 : TSG_F64;
  check(tsg_mesh_upload(ctx, &d, &mesh_), "tsg_mesh_upload");
}

DeviceMesh::~DeviceMesh() { tsg_mesh_free(mesh_); }

int64_t DeviceMesh::device_bytes() const { return tsg_mesh_device_bytes(mesh_); }
void DeviceMesh::set_coords(const double* xy) { check(tsg_mesh_set_coords(mesh_, xy), "tsg_mesh_set_coords"); }
void DeviceMesh::get_coords(double* xy) const { check(tsg_mesh_get_coords(mesh_, xy), "tsg_mesh_get_coords"); }
void DeviceMesh::tri_alpha(double* out) const { check(tsg_tri_alpha(mesh_, out), "tsg_tri_alpha"); }
void DeviceMesh::vertex_minima(double* out) const {
  check(tsg_vertex_minima(mesh_, out), "tsg_vertex_minima");
}

RunStats DeviceMesh::run(const SmoothConfig& cfg, double diag) {
  validate(cfg);
  tsg_smooth_cfg c{};
  c.form = cfg.form == IterationForm::B ? TSG_FORM_B : TSG_FORM_A;
  c.strategy = cfg.strategy == UpdateStrategy::TwoPhase ? TSG_STRATEGY_TWOPHASE : TSG_STRATEGY_FUSED;
  c.chunks = cfg.backend == Backend::Parallel ? cfg.workers : 1;  // smoothing.cpp:81
  c.swap = cfg.swap == SwapMode::Copy ? TSG_SWAP_COPY : TSG_SWAP_PINGPONG;
  c.max_iters = cfg.max_iters;
  c.driver = cfg.use_graph ? TSG_DRIVER_GRAPH : TSG_DRIVER_STREAM;
  c.move_tol = cfg.move_tol;
  c.bbox_diag = diag;
  RunStats rs;
  rs.accepted_per_pass.resize(cfg.max_iters);
  rs.max_disp_per_pass.resize(cfg.max_iters);
  tsg_smooth_stats st{};
  check(tsg_smooth(mesh_, &c, &st, rs.accepted_per_pass.data(), rs.max_disp_per_pass.data(),
                   cfg.max_iters),
        "tsg_smooth");
  rs.iterations = st.iterations;
  rs.accepted_per_pass.resize(st.iterations);
  rs.max_disp_per_pass.resize(st.iterations);
  rs.stop = st.stop == TSG_STOP_NO_MOVES      ? StopReason::NoMoves
            : st.stop == TSG_STOP_DISPLACEMENT ? StopReason::Displacement
                                                : StopReason::MaxIters;
  rs.device_ms = st.device_ms;
  rs.kernel_launches = st.launches;
  return rs;
}

}  // namespace gpu

namespace {

using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

// min and sequential-sum mean over the stored triangle α (smoothing.cpp:49-60).
void summarize(const std::vector<double>& alpha, double& lo, double& mean) {
  lo = std::numeric_limits<double>::infinity();
  double sum = 0.0;
  for (const double q : alpha) {
    lo = std::min(lo, q);
    sum += q;
  }
  mean = sum / static_cast<double>(alpha.size());
}

}  // namespace

RunStats smooth(Mesh& mesh, const SmoothConfig& config) {
  validate(config);
  const auto t_total = Clock::now();
  tsg_context* ctx = gpu::default_context();

  auto t0 = Clock::now();
  init_flags(mesh);
  const double init_flags_ms = ms_since(t0);

  t0 = Clock::now();
  const Adjacency adj = find_neighbors(mesh);
  const double topo_ms = ms_since(t0);

  t0 = Clock::now();
  determine_constraints(mesh, adj);
  const double constr_host_ms = ms_since(t0);

  const int64_t nv = mesh.vertex_count(), nt = mesh.triangle_count();
  std::vector<double> xy(2 * nv);
  std::vector<int32_t> tri(3 * nt);
  gpu::Topology64 topo;
  topo.boundary.resize(nv);
  mesh.visit([&](const auto& m) {
    for (int64_t v = 0; v < nv; ++v) {
      const Point p = m.position(static_cast<int>(v));
      xy[2 * v] = p.x;
      xy[2 * v + 1] = p.y;
      topo.boundary[v] = m.is_boundary(static_cast<int>(v)) ? 1 : 0;
    }
    for (int64_t t = 0; t < nt; ++t) {
      const auto c = m.tri(static_cast<int>(t));
      tri[3 * t] = c[0], tri[3 * t + 1] = c[1], tri[3 * t + 2] = c[2];
    }
  });
  topo.nbr_off.assign(adj.unique.offsets.begin(), adj.unique.offsets.end());
  topo.inc_off.assign(adj.incident.offsets.begin(), adj.incident.offsets.end());
  topo.nbr.assign(adj.unique.values.begin(), adj.unique.values.end());
  topo.inc.assign(adj.incident.values.begin(), adj.incident.values.end());

  // Locality order only where it cannot change results: Form A reads every neighbour from the
  // previous pass and the device keeps each neighbour row in original-id order (K10).
  const bool reorder = config.form == IterationForm::A &&
                       (config.reorder == Reorder::Hilbert ||
                        (config.reorder == Reorder::Auto && nv > 65536));
  t0 = Clock::now();
  gpu::DeviceMesh dm(xy.data(), nv, tri.data(), nt, topo, mesh.layout(), config.precision, reorder, ctx);
  const double upload_ms = ms_since(t0);

  // compute_all_qualities + reduce_vertex_minima on the device (quality.cpp:27-32, :60-65).
  t0 = Clock::now();
  std::vector<double> alpha(nt), vmin(nv);
  dm.tri_alpha(alpha.data());
  const double alpha_ms = ms_since(t0);
  t0 = Clock::now();
  dm.vertex_minima(vmin.data());
  const double vmin_ms = ms_since(t0);

  RunStats stats;
  summarize(alpha, stats.min_alpha_before, stats.mean_alpha_before);
  const double diag = gpu::bbox_diagonal(xy.data(), nv);

  t0 = Clock::now();
  RunStats run = dm.run(config, diag);
  stats.iter_ms = ms_since(t0);
  stats.iterations = run.iterations;
  stats.stop = run.stop;
  stats.accepted_per_pass = std::move(run.accepted_per_pass);
  stats.max_disp_per_pass = std::move(run.max_disp_per_pass);
  stats.device_ms = run.device_ms;
  stats.kernel_launches = run.kernel_launches;

  // Write-back: coordinates, triangle α and vertex minima synced to the final coordinates.
  dm.get_coords(xy.data());
  dm.tri_alpha(alpha.data());
  dm.vertex_minima(vmin.data());
  mesh.visit([&](auto& m) {
    for (int64_t v = 0; v < nv; ++v) {
      m.set_position(static_cast<int>(v), Point{xy[2 * v], xy[2 * v + 1]});
      m.set_vertex_min_quality(static_cast<int>(v), vmin[v]);
    }
    for (int64_t t = 0; t < nt; ++t) m.set_tri_quality(static_cast<int>(t), alpha[t]);
  });
  summarize(alpha, stats.min_alpha_after, stats.mean_alpha_after);

  stats.init_ms = init_flags_ms + alpha_ms;
  stats.topo_ms = topo_ms;
  stats.constr_ms = constr_host_ms + vmin_ms;
  stats.upload_ms = upload_ms;
  stats.total_ms = ms_since(t_total);
  return stats;
}

}  // namespace trismooth
