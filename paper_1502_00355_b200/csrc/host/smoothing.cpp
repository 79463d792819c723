// smooth() on the B200 (include/trismooth/smoothing.hpp) and the device-mesh plumbing of
// include/trismooth/gpu.hpp.
//
// Pipeline and statistics follow proj/src/smoothing.cpp:146-182; the pass loop (:76-142) runs
// in libtsg.so as one CUDA-graph launch, the adjacency and constraints (find_neighbors /
// determine_constraints) are built on the device (tsg_topology) and installed into the mesh;
// the device layout (locality order, tiles) is prepared on the host (tsg_prep.cpp).
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

Topology64 device_topology(int64_t nv, const int32_t* tri, int64_t nt, tsg_context* ctx) {
  if (!ctx) ctx = default_context();
  Topology64 T;
  T.nbr_off.resize(nv + 1);
  T.inc_off.resize(nv + 1);
  T.nbr.resize(static_cast<size_t>(std::max<int64_t>(1, 6 * nt)));
  T.inc.resize(static_cast<size_t>(std::max<int64_t>(1, 3 * nt)));
  T.boundary.resize(nv);
  int64_t n = 0;
  check(tsg_topology(ctx, nv, nt, tri, T.nbr_off.data(), T.nbr.data(), static_cast<int64_t>(T.nbr.size()),
                     T.inc_off.data(), T.inc.data(), T.boundary.data(), &n),
        "tsg_topology");
  T.nbr.resize(n);
  T.nbr.shrink_to_fit();
  T.inc.resize(3 * nt);
  return T;
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

  // Host arrays the device path reads: coordinates and corners in original numbering.
  const int64_t nv = mesh.vertex_count(), nt = mesh.triangle_count();
  std::vector<double> xy(2 * nv);
  std::vector<int32_t> tri(3 * nt);
  mesh.visit([&](const auto& m) {
    for (int64_t v = 0; v < nv; ++v) {
      const Point p = m.position(static_cast<int>(v));
      xy[2 * v] = p.x;
      xy[2 * v + 1] = p.y;
    }
    for (int64_t t = 0; t < nt; ++t) {
      const auto c = m.tri(static_cast<int>(t));
      tri[3 * t] = c[0], tri[3 * t + 1] = c[1], tri[3 * t + 2] = c[2];
    }
  });

  // find_neighbors + determine_constraints (proj/src/topology.cpp:12-95) on the device: the
  // same unique / incident rows and flags, with int64 offsets (no int32 raw list).
  t0 = Clock::now();
  gpu::Topology64 topo = gpu::device_topology(nv, tri.data(), nt, ctx);
  const double topo_ms = ms_since(t0);

  // Install the adjacency and the constraint flags into the mesh as the reference does
  // (tests read them after smooth()).  The reference's Csr is int-indexed: beyond 2^31 entries
  // the rows stay device-side only.
  t0 = Clock::now();
  const bool fits = topo.nbr_off[nv] < (int64_t{1} << 31) && topo.inc_off[nv] < (int64_t{1} << 31);
  mesh.visit([&](auto& m) {
    if (fits) {
      Csr unique, incident;
      unique.offsets.assign(topo.nbr_off.begin(), topo.nbr_off.end());
      unique.values.assign(topo.nbr.begin(), topo.nbr.end());
      incident.offsets.assign(topo.inc_off.begin(), topo.inc_off.end());
      incident.values.assign(topo.inc.begin(), topo.inc.end());
      m.assign_adjacency(unique, incident);
    }
    for (int64_t v = 0; v < nv; ++v) m.set_boundary(static_cast<int>(v), topo.boundary[v] != 0);
  });
  const double constr_host_ms = ms_since(t0);

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
