/*
 * tsg.h — C ABI of the B200 Smart Laplacian engine (libtsg.so).
 *
 * This is the drop-in boundary between host code (the trismooth C++ API in
 * include/trismooth/, the pybind11 module _trismooth, or any FFI: ctypes, cgo, JNI)
 * and the sm_100a kernels.  Plain C: explicit int64 counts, caller-owned host
 * buffers, library-owned device buffers behind opaque handles, integer status
 * (TSG_OK = 0) plus a thread-local message (tsg_last_error).  No exceptions and no
 * torch types cross this boundary.  Calls on one context are serialised by a per-context
 * lock, so host threads may share a context (the drop-in smooth() does); each call is still
 * single-orchestrator (proj/include/trismooth/parallel.hpp:26-28).
 *
 * Reference interfaces each entry point replaces (paths under /root/reference/proj):
 *   tsg_mesh_upload        the in-memory Mesh + Adjacency after find_neighbors /
 *                          determine_constraints (src/topology.cpp:69-95, src/mesh.cpp:20-53)
 *   tsg_tri_alpha          compute_all_qualities        (src/quality.cpp:27-32)
 *   tsg_vertex_minima      reduce_vertex_minima         (src/quality.cpp:60-65)
 *   tsg_smooth             run_passes                   (src/smoothing.cpp:76-142), i.e.
 *                          smooth_range / neighbor_mean / min_alpha_at per vertex
 *                          (include/trismooth/smoothing.hpp:70-109, quality.hpp:54-64)
 *   tsg_mesh_set_coords /  the coordinate fields of AosMesh / SoaMesh
 *   tsg_mesh_get_coords    (include/trismooth/mesh.hpp:61-70, :203-212)
 *   tsg_smooth_host        smooth() minus host topology prep (src/smoothing.cpp:146-182):
 *                          host coords in -> passes -> host coords + stats out
 *   tsg_quality_tri_alpha  compute_all_qualities on a bare (xy, tri) pair plus the reductions
 *                          of quality_summary / `trismooth quality` (src/quality.cpp:27-32,
 *                          bindings/module.cpp:157-185, tools/main.cpp:151-208)
 *   tsg_quality_vertex_minima  reduce_vertex_minima over a caller's incident CSR and stored
 *                          α field (src/quality.cpp:60-65, include/trismooth/quality.hpp:78-89)
 */
#ifndef TSG_H_
#define TSG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSG_ABI_VERSION 1

typedef int32_t tsg_status;
enum {
  TSG_OK = 0,
  TSG_ERR_INVALID = 1, /* bad argument / unsupported combination */
  TSG_ERR_CUDA = 2,    /* CUDA runtime or driver error (message has the detail) */
  TSG_ERR_NOMEM = 3,   /* device or host allocation failed */
  TSG_ERR_NODEVICE = 4 /* no CUDA device / extension cannot run here */
};

enum { TSG_LAYOUT_AOS = 0, TSG_LAYOUT_SOA = 1 };          /* mesh.hpp:24 Layout */
enum { TSG_F64 = 0, TSG_F32 = 1 };                        /* coordinate + arithmetic type */
enum { TSG_FORM_A = 0, TSG_FORM_B = 1 };                  /* smoothing.hpp:14 IterationForm */
enum { TSG_STRATEGY_FUSED = 0, TSG_STRATEGY_TWOPHASE = 1 }; /* smoothing.hpp:20 UpdateStrategy */
enum { TSG_SWAP_PINGPONG = 0, TSG_SWAP_COPY = 1 };        /* no-copy pointer swap / explicit copy */
enum { TSG_STOP_MAX_ITERS = 0, TSG_STOP_DISPLACEMENT = 1, TSG_STOP_NO_MOVES = 2 };
enum { TSG_DRIVER_GRAPH = 0, TSG_DRIVER_STREAM = 1 };     /* WHILE-graph loop / plain launches */

typedef struct tsg_context tsg_context;
typedef struct tsg_mesh tsg_mesh;

/*
 * Host description of a prepared mesh.  All arrays are in ORIGINAL vertex / triangle
 * numbering and are read only during tsg_mesh_upload.
 *   nbr_off/nbr   unique-neighbour CSR, each row ascending (Adjacency::unique)
 *   inc_off/inc   incident-triangle CSR, each row ascending (Adjacency::incident)
 *   boundary      1 = pinned (determine_constraints)
 *   order         optional locality order: order[s] = original id stored at device
 *                 slot s (a permutation of 0..nv-1); NULL = identity.  Results are
 *                 unaffected: neighbour sums keep ascending ORIGINAL-id order and
 *                 Form B chunks / lower-id tests use original ids.
 */
typedef struct {
  int64_t nv;
  int64_t nt;
  const double* xy;      /* 2*nv interleaved x,y */
  const int32_t* tri;    /* 3*nt */
  const int64_t* nbr_off;
  const int32_t* nbr;
  const int64_t* inc_off;
  const int32_t* inc;
  const uint8_t* boundary;
  const int64_t* order;
  int32_t layout;    /* TSG_LAYOUT_* : device coordinate layout */
  int32_t precision; /* TSG_F64 | TSG_F32 */
} tsg_mesh_desc;

typedef struct {
  int32_t form;      /* TSG_FORM_* */
  int32_t strategy;  /* TSG_STRATEGY_* (identical results; schedule differs) */
  int32_t chunks;    /* Form B chunk count W (Backend::Parallel workers); 1 = serial */
  int32_t swap;      /* TSG_SWAP_* */
  int32_t max_iters; /* >= 1 */
  int32_t driver;    /* TSG_DRIVER_* */
  double move_tol;   /* >= 0; 0 disables the displacement stop */
  double bbox_diag;  /* std::hypot of the bbox extents, computed by the caller */
} tsg_smooth_cfg;

typedef struct {
  int32_t iterations;
  int32_t stop;          /* TSG_STOP_* */
  int64_t node_updates;  /* nv * iterations (pinned vertices counted, as the reference) */
  double device_ms;      /* CUDA-event time of the pass loop */
  double node_kernel_ms; /* CUDA-event time summed over node-update launches (stream driver) */
  int64_t launches;      /* kernels launched by this call */
  int32_t schedule;      /* TSG_SCHEDULE_*: how the passes ran */
  int32_t reserved;
} tsg_smooth_stats;

/* tsg_smooth_stats.schedule */
#define TSG_SCHEDULE_GRAPH 0   /* per-pass kernels in a conditional-WHILE CUDA graph */
#define TSG_SCHEDULE_STREAM 1  /* per-pass plain launches (TSG_DRIVER_STREAM) */
#define TSG_SCHEDULE_PEER 2    /* peer-memory partitioned graph */
#define TSG_SCHEDULE_FLOW 3    /* dataflow launch: tile_flow (Form A) / formb_flow (Form B) */

/* Reductions of the quality audit (folds as the reference writes them: min / max start
 * at 2.0 / -2.0, NaN never replaces, ties keep the first triangle; histogram bins of width
 * 0.1 over [-1, 1], bin = (int)((alpha + 1) * 10) clamped to [0, 19]). */
#define TSG_QUALITY_BINS 20
typedef struct {
  double min_alpha;
  double max_alpha;
  int64_t non_positive;               /* alpha <= 0 */
  int64_t histogram[TSG_QUALITY_BINS];
} tsg_quality_report;

/* ---- context ---- */
int32_t tsg_abi_version(void);
const char* tsg_last_error(void);
int32_t tsg_device_count(void);
tsg_status tsg_context_create(int32_t device, tsg_context** out);
tsg_status tsg_context_destroy(tsg_context* ctx);
/* Returns the cudaStream_t the context launches on (for callers that sync / time). */
void* tsg_context_stream(tsg_context* ctx);

/* ---- mesh ---- */
tsg_status tsg_mesh_upload(tsg_context* ctx, const tsg_mesh_desc* desc, tsg_mesh** out);
tsg_status tsg_mesh_free(tsg_mesh* mesh);
/* bytes of device memory held by the mesh */
int64_t tsg_mesh_device_bytes(const tsg_mesh* mesh);
/* Coordinates in ORIGINAL numbering (2*nv doubles; f32 meshes round on upload). */
tsg_status tsg_mesh_set_coords(tsg_mesh* mesh, const double* xy);
tsg_status tsg_mesh_get_coords(tsg_mesh* mesh, double* xy_out);
/* Device-side reset to the coordinates of the last upload / set_coords (no host traffic;
 * asynchronous on the context stream).  Benchmarks restart every step from the same mesh. */
tsg_status tsg_mesh_restore_coords(tsg_mesh* mesh);

/* ---- quality (device) ---- */
/* alpha_out: nt doubles in original triangle order (compute_all_qualities). */
tsg_status tsg_tri_alpha(tsg_mesh* mesh, double* alpha_out);
/* vmin_out: nv doubles, NaN for vertices without incident triangles (reduce_vertex_minima). */
tsg_status tsg_vertex_minima(tsg_mesh* mesh, double* vmin_out);
/* {min alpha, max alpha, count alpha <= 0}; exact (order-free) reductions. */
tsg_status tsg_alpha_extrema(tsg_mesh* mesh, double* min_out, double* max_out, int64_t* nonpos_out);

/* ---- the hot path ---- */
/*
 * Upload from points and triangles only: the adjacency, constraints and device layout are built
 * on the device without a host round trip (tsg_topology + the device layout of
 * tsg_mesh_upload).  The desc's nbr_off / nbr / inc_off / inc / boundary are ignored (may be
 * NULL); xy, tri, nv, nt, layout, precision and order are read.  Same mesh as tsg_mesh_upload
 * with tsg_topology's arrays.
 */
tsg_status tsg_mesh_upload_triangles(tsg_context* ctx, const tsg_mesh_desc* desc, tsg_mesh** out);

/*
 * Runs passes until max_iters, accepted == 0 (NoMoves) or max_disp < move_tol*bbox_diag
 * (Displacement), in the reference's order (src/smoothing.cpp:132-141).  Coordinates stay
 * on the device.  accepted_per_pass / max_disp_per_pass receive min(capacity, iterations)
 * entries (either may be NULL).
 */
tsg_status tsg_smooth(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, tsg_smooth_stats* stats,
                      int32_t* accepted_per_pass, double* max_disp_per_pass, int32_t capacity);

/* Host-buffer variant: H2D of xy_in, tsg_smooth, D2H into xy_out (both original order). */
tsg_status tsg_smooth_host(tsg_mesh* mesh, const double* xy_in, const tsg_smooth_cfg* cfg,
                           double* xy_out, tsg_smooth_stats* stats, int32_t* accepted_per_pass,
                           double* max_disp_per_pass, int32_t capacity);
/* Smooths n coordinate sets of the same mesh end to end: xy_in[k] (host, original order; pinned
 * memory for asynchronous copies) -> cfg passes -> xy_out[k], with the host->device copy of item
 * k+1 and the device->host copy of item k-1 overlapping the passes of item k (copy engines on
 * their own streams, two device staging slots).  Graph driver only; per-item passes executed and
 * TSG_STOP_* in iterations_out / stop_out (may be NULL).  Leaves the device coordinates of the
 * last item current (the restore point of tsg_mesh_restore_coords is unchanged). */
tsg_status tsg_smooth_host_batch(tsg_mesh* mesh, int32_t n, const double* const* xy_in, const tsg_smooth_cfg* cfg,
                                 double* const* xy_out, int32_t* iterations_out, int32_t* stop_out);

/*
 * One pass in lockstep from the current device state, without the stop rule; writes the
 * per-vertex decision (1 accept, 0 reject, -1 pinned; original order) and advances the
 * coordinates.  Used for the fp32 lockstep parity contract.
 */
tsg_status tsg_pass_lockstep(tsg_mesh* mesh, int32_t form, int32_t chunks, int8_t* decision_out,
                             int32_t* accepted_out, double* max_disp_out);

/* ---- multi-GPU partitions (one process per GPU; see paper_1502_00355_b200/distributed.py) ---- */
/*
 * One pass of `cfg` (form, strategy, chunks, swap; max_iters / driver / move_tol ignored) from
 * the current device state, without the stop rule; returns this mesh's accepted count and max
 * displacement.  The caller combines them across partitions and applies the stop rule.
 */
tsg_status tsg_pass(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, int32_t* accepted_out, double* max_disp_out);
/* Halo plan in ORIGINAL (local) vertex numbering: send_ids are owned vertices other partitions
 * read, recv_ids the locally pinned halo copies of other partitions' vertices (peer order). */
tsg_status tsg_halo_plan(tsg_mesh* mesh, const int64_t* send_ids, int64_t n_send,
                         const int64_t* recv_ids, int64_t n_recv);
/* Packs the current coordinates of the send vertices into 2*n_send doubles, or writes 2*n_recv
 * doubles into the halo vertices (both buffers).  *_is_host: 0 = device pointer (e.g. a buffer an
 * NCCL all-to-all reads / writes), 1 = host pointer.  Synchronous on the context stream. */
tsg_status tsg_halo_pack(tsg_mesh* mesh, double* out, int32_t out_is_host);
tsg_status tsg_halo_unpack(tsg_mesh* mesh, const double* in, int32_t in_is_host);

/* Device-resident partitioned pass loop (Form A): every call below only ENQUEUES work on the
 * context stream (no host synchronisation), so a driver can chain, per pass,
 *   tsg_dist_pass -> tsg_dist_halo_pack -> all-to-all -> tsg_dist_halo_unpack
 *                 -> all-gather of the stats pairs -> tsg_dist_finalize
 * with NCCL collectives ordered on the same stream, and poll tsg_dist_status every few passes.
 * Kernels of passes enqueued after the global stop fired exit immediately.
 *   begin:    resets the device pass state for a run of cfg->max_iters passes
 *   pass:     one pass's node kernels; writes this partition's {accepted count, max
 *             displacement} of the pass as two doubles to the DEVICE buffer stats_dev
 *   halo_*:   halo copies through DEVICE buffers, current buffer chosen on the device
 *   finalize: the reference's stop rule (smoothing.cpp:132-141) on the n_parts all-gathered
 *             DEVICE pairs (sum of accepted, max of displacement)
 *   status:   synchronises; passes executed, done flag, TSG_STOP_*
 *   end:      synchronises; per-pass totals (as tsg_smooth), the final state and the number of
 *             kernels the dist calls enqueued since begin */
tsg_status tsg_dist_begin(tsg_mesh* mesh, const tsg_smooth_cfg* cfg);
tsg_status tsg_dist_pass(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, double* stats_dev);
tsg_status tsg_dist_halo_pack(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, double* out_dev);
tsg_status tsg_dist_halo_unpack(tsg_mesh* mesh, const double* in_dev);
tsg_status tsg_dist_finalize(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, const double* gathered_dev, int32_t n_parts);
tsg_status tsg_dist_status(tsg_mesh* mesh, int32_t* iterations, int32_t* done, int32_t* stop);
tsg_status tsg_dist_end(tsg_mesh* mesh, const tsg_smooth_cfg* cfg, int32_t* accepted_per_pass,
                        double* max_disp_per_pass, int32_t capacity, int32_t* iterations_out, int32_t* stop_out,
                        int64_t* launches_out);

/* Form B schedule (identical results; tsg_smooth only — the batch and partitioned entry points
 * use LEVELS / CHUNKS):
 *   LEVELS  one set of tier kernels per dependency level of each pass;
 *   CHUNKS  one CTA per chunk walking its levels, one launch per pass;
 *   FLOW    one persistent launch for many passes: (vertex, pass) dataflow with per-vertex
 *           pass counters, so pass q+1 pipelines behind pass q (tsg_flow.cuh);
 *   AUTO    (default) FLOW for tsg_smooth, else CHUNKS or LEVELS by the per-level cost model. */
enum { TSG_FORMB_AUTO = 0, TSG_FORMB_LEVELS = 1, TSG_FORMB_CHUNKS = 2, TSG_FORMB_FLOW = 3 };
tsg_status tsg_mesh_formb_schedule(tsg_mesh* mesh, int32_t mode);

/* Form A fused, rows of valence >= 32 (the paper's high-valence nodes): AUTO (default) runs them
 * in a small persistent kernel beside the tile grid (one 4-warp CTA per SM, warps taking rows
 * longest-first) when their estimated time fits inside the tile grid's, else as per-tier grids
 * (CTA per hub, warp per row) after it; KERNELS / PERSIST force one of the two (identical
 * results). */
enum { TSG_SIDE_AUTO = 0, TSG_SIDE_KERNELS = 1, TSG_SIDE_PERSIST = 2 };
tsg_status tsg_mesh_side_schedule(tsg_mesh* mesh, int32_t mode);

/* ---- diagnostics ---- */
/* Evaluates n seeded random triangles (unit scale, tiny, huge, near-degenerate) with the
 * kernels' fast alpha (refined reciprocal) and with the reference's IEEE division; returns the
 * maximum |fast - exact| over triangles with |exact| <= 1 and the count of non-finite fast
 * values.  newton_steps (1 or 2) selects the reciprocal refinement under test; the kernels'
 * fast path is only trusted outside a 2^-45 guard band (tsg_device.cuh). */
tsg_status tsg_selftest_alpha(tsg_context* ctx, int64_t n, uint64_t seed, int32_t newton_steps,
                              double* max_abs_err_out, int64_t* nonfinite_out);
/* The same for the rotation (cycle) fast path of the Form A fused kernels: the maximum
 * |t - alpha_ref / K| in alpha/K units, K = 2*sqrt(3) as the reference rounds it.  Its guard
 * band is 2^-48 in those units (derivation in tsg_device.cuh, kGuardCycle). */
tsg_status tsg_selftest_alpha_cycle(tsg_context* ctx, int64_t n, uint64_t seed, double* max_abs_err_out,
                                    int64_t* nonfinite_out);

/* Timeline instrumentation readout: copies the per-CTA / per-warp (start ns, duration ns << 8 |
 * SM id) records of one pass into out.  Only builds made with -DTSG_TRACE record them
 * (tools/trace_cfg3.py); other builds return TSG_ERR_INVALID. */
tsg_status tsg_debug_trace(void* out, int64_t bytes);

/* ---- locality ordering (host prep helper) ---- */
/* order_out[s] = original id for slot s: vertices sorted along a Hilbert curve over the
 * bounding box (ties by original id).  Pure host code, deterministic. */
tsg_status tsg_hilbert_order(int64_t nv, const double* xy, int64_t* order_out);
/* The same order computed on the device (radix sort of the same keys). */
tsg_status tsg_hilbert_order_device(tsg_context* ctx, int64_t nv, const double* xy, int64_t* order_out);

/* ---- quality audit on the device (no tsg_mesh needed) ----
 * tsg_quality_tri_alpha: alpha_out[t] = triangle_alpha of triangle t (bit-exact), plus the
 * report (may be NULL).  xy: 2*nv interleaved, tri: 3*nt.  Corner ids are range-checked.
 * tsg_quality_vertex_minima: vmin_out[v] = min of alpha[inc[j]] over v's row of the
 * incident CSR (inc_off: nv+1 entries from 0), NaN for an empty row. */
tsg_status tsg_quality_tri_alpha(tsg_context* ctx, int64_t nv, const double* xy, int64_t nt,
                                 const int32_t* tri, double* alpha_out, tsg_quality_report* report);
tsg_status tsg_quality_vertex_minima(tsg_context* ctx, int64_t nv, const int64_t* inc_off,
                                     const int32_t* inc, int64_t nt, const double* alpha,
                                     double* vmin_out);

/* ---- partitioned Form A over peer memory (one process per GPU, NVLink / NVSwitch) ----
 * Each rank uploads its partition (owned vertices + one-ring halo, halo pinned) as usual, then:
 *   tsg_peer_local   its own coordinate buffers and sync block (allocated on first use), to be
 *                    shared with the peers: raw pointers in one process, or CUDA IPC handles
 *                    (tsg_ipc_handle / tsg_ipc_open) across processes;
 *   tsg_mesh_slots   device slot of local vertex ids (the peers' push destinations);
 *   tsg_peer_setup   the world's mapped pointers (entry `rank` = its own tsg_peer_local values)
 *                    and this rank's push plan: for each owned vertex in peer q's halo, the
 *                    local id and q's slot for it.
 * From then on tsg_smooth on the mesh (Form A) runs the partitioned loop: per pass the node
 * kernels, direct stores of the send vertices into the peers' buffers and a flag barrier with
 * the global stop statistics, all inside one conditional-WHILE graph per rank (tsg_peer.cuh).
 * Every rank must run the same sequence of tsg_smooth calls with the same configuration;
 * results are bit-identical to one GPU.  tsg_peer_clear returns to single-mesh runs. */
#define TSG_IPC_HANDLE_BYTES 64
tsg_status tsg_peer_local(tsg_mesh* mesh, void** buf0, void** buf1, void** sync, int64_t* nv);
tsg_status tsg_mesh_slots(tsg_mesh* mesh, const int64_t* ids, int64_t n, int64_t* slots_out);
tsg_status tsg_peer_setup(tsg_mesh* mesh, int32_t rank, int32_t world, void* const* peer_buf0,
                          void* const* peer_buf1, void* const* peer_sync, const int64_t* peer_nv,
                          int64_t n_push, const int32_t* push_peer, const int64_t* push_src_ids,
                          const int64_t* push_dst_slots);
/* Allocations, capture and instantiation of the peer graph for `cfg` (they may synchronise the
 * device): call on every rank before the first tsg_smooth with that configuration whenever
 * several ranks share a device or a process. */
tsg_status tsg_peer_prepare(tsg_mesh* mesh, const tsg_smooth_cfg* cfg);
tsg_status tsg_peer_clear(tsg_mesh* mesh);
tsg_status tsg_ipc_handle(const void* dev_ptr, void* handle_out);
tsg_status tsg_ipc_open(tsg_context* ctx, const void* handle, void** dev_ptr_out);
tsg_status tsg_ipc_close(tsg_context* ctx, void* dev_ptr);

/* ---- mesh topology on the device (find_neighbors + determine_constraints,
 * proj/src/topology.cpp:12-95, without the int32 raw list) ----
 * nbr_off / inc_off: nv+1 int64; nbr: unique neighbours, each row ascending (capacity nbr_cap,
 * 6*nt always suffices; the count is returned in n_nbr_out); inc: 3*nt incident triangles,
 * each row ascending; boundary: 1 = isolated or some neighbour multiplicity != 2. */
tsg_status tsg_topology(tsg_context* ctx, int64_t nv, int64_t nt, const int32_t* tri, int64_t* nbr_off,
                        int32_t* nbr, int64_t nbr_cap, int64_t* inc_off, int32_t* inc, uint8_t* boundary,
                        int64_t* n_nbr_out);

/* Test hook: builds the device layout of `desc` on the GPU (tsg_layout_dev.cu) and on the host
 * (build_host_mesh) and writes the name of the first array that differs into `mismatch`
 * ("" when identical). */
tsg_status tsg_debug_layout_check(tsg_context* ctx, const tsg_mesh_desc* desc, char* mismatch, int32_t cap);

#ifdef __cplusplus
}
#endif
#endif /* TSG_H_ */
