/*
 * lemgpu.h -- C-ABI of the B200-native D8 landscape-evolution step.
 *
 * This is the ONLY seam between host code and the sm_100a kernels.  Plain C
 * types, caller-owned host buffers, an opaque device context.  It replaces
 * the body of one reference execution strategy:
 *
 *   lem::strategy_step(Raster<double>& elev, const GridGraph&, const SimParams&,
 *                      const StepSetup&, const Strategy&, SimWorkspace&,
 *                      const StepInstrumentation*)        proj/include/lem/scheduler.hpp:38-41
 *     -> dispatch switch                                   proj/src/scheduler.cpp:425-462
 *   lem::run_simulation(Raster<double>, const RunConfig&,
 *                       const StepCallback&)               proj/include/lem/scheduler.hpp:61-62
 *     -> stepping loop                                     proj/src/scheduler.cpp:490-498
 *
 * A maintainer adds StrategyKind::kRbGpu ("rb_gpu", proj/include/lem/strategy.hpp:12-56)
 * and routes it here; see INTEGRATION.md for the C++ shim and the ctypes
 * binding the Python tests use.
 *
 * Status codes mirror the reference's exception classes
 * (proj/include/lem/error.hpp:10-43) the way ErrorCollector::rethrow does
 * (proj/src/scheduler.cpp:45-49):
 *   0 ok, 1 ConfigError, 2 StructureError (cycle), 3 ConvergenceError(cell),
 *   4 CUDA error (lem::Error), 5 other lem::Error.
 *
 * Threading: calls on one context are serialised on that context's CUDA
 * stream and are not thread-safe; distinct contexts are independent.
 */
#ifndef LEMGPU_H
#define LEMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LEMGPU_ABI_VERSION 3
#define LEMGPU_NOFLOW 0xFFFFFFFFu /* kNoFlow, proj/include/lem/raster.hpp:16 */

enum {
  LEMGPU_OK = 0,
  LEMGPU_ECONFIG = 1,
  LEMGPU_ESTRUCTURE = 2,
  LEMGPU_ECONVERGENCE = 3,
  LEMGPU_ECUDA = 4,
  LEMGPU_EOTHER = 5
};

/* Phase slots, same order as lem::Phase (proj/include/lem/simulation.hpp:19-22). */
enum {
  LEMGPU_PHASE_RECEIVERS = 0,
  LEMGPU_PHASE_DONORS = 1,
  LEMGPU_PHASE_ORDER = 2,
  LEMGPU_PHASE_ACCUM = 3,
  LEMGPU_PHASE_UPLIFT = 4,
  LEMGPU_PHASE_EROSION = 5
};

/* POD mirror of lem::SimParams (proj/include/lem/erosion.hpp:15-25) plus the
 * neighbourhood connectivity of RunConfig (proj/include/lem/config.hpp:63). */
typedef struct lemgpu_params {
  double K;           /* erodibility                        (erosion.hpp:16) */
  double m_exp;       /* drainage-area exponent             (erosion.hpp:17) */
  double n_exp;       /* slope exponent, > 0                (erosion.hpp:18) */
  double uplift_rate; /* interior uplift per unit time      (erosion.hpp:19) */
  double dt;          /* implicit timestep                  (erosion.hpp:20) */
  double epsilon;     /* Newton step-difference tolerance   (erosion.hpp:21) */
  double dx, dy;      /* cell spacing                       (erosion.hpp:22-23) */
  int32_t max_newton_iters; /*                              (erosion.hpp:24) */
  int32_t connectivity;     /* 4 or 8                       (config.hpp:63) */
} lemgpu_params;

/* Per-realisation overrides for an ensemble context (paper future work,
 * PAPER.md:749): each member runs with its own K and m. */
typedef struct lemgpu_member {
  double K;
  double m_exp;
} lemgpu_member;

/* Mirror of lem::StepDiagnostics + PhaseTimings
 * (proj/include/lem/simulation.hpp:25-40), plus device-side facts. */
typedef struct lemgpu_diag {
  /* PhaseTimings::seconds, lem::Phase order.  The step's device time (first
   * kernel start to the end of the step, %globaltimer) split in proportion to
   * the SM cycles every CTA spent in each phase: the kernels fuse phases
   * (receivers + donors; order + accumulation + uplift + erosion) and overlap,
   * so the six slots add up to the step's device time. */
  double seconds[6];
  uint64_t newton_iters;    /* sum of Newton iterations over eroded cells (erosion.cpp:76-77) */
  uint32_t interior_noflow; /* interior cells with rec == kNoFlow (simulation.cpp:42-44) */
  uint32_t nlevels;         /* TraversalPlan::nlevels() (traversal.hpp:34) */
  uint32_t lut_misses;      /* cells whose pow(A,m) was computed on the device, not read from the
                               host-libm table (bit-identical either way: glibc_pow.cuh) */
  uint32_t status;          /* LEMGPU_* for this step */
  uint32_t err_cell;        /* ConvergenceError::cell() when status == 3 */
  uint32_t escaped_trees;   /* trees finished by the escape path (tile path), else source chunks */
  /* Kernel spans of the step (device %globaltimer, first CTA start to last CTA
   * end; the receiver and tile passes overlap when pipelined):
   * [0] receiver pass (k_recv), [1] tile pass (k_tiles), [2] escape path's
   * level expansion, [3] escape path's accumulation + uplift + erosion. */
  double kernel_s[4];
  uint32_t escaped_cells;   /* cells of the escaped trees */
  uint32_t mfd_passes;      /* routing = kMfd: tile passes of the MFD accumulation (k_mfd_tiles); else 0 */
} lemgpu_diag;

/* Schedule / tuning / test knobs of a context (no reference counterpart).
 * Zero-initialised = the production defaults; the library reads no
 * environment variables.  Every knob gives the same bits (the schedules are
 * dependency-respecting orders of identical per-cell arithmetic); the tests
 * use them to force every code path. */
typedef struct lemgpu_options {
  int32_t global_path;     /* 1: every tree through the global level path (no tile pass) */
  int32_t force_escape;    /* 1: every tile tree escapes; 2: trees with an odd root cell escape */
  int32_t force_deep;      /* 1: per-level sweeps even for shallow plans */
  int32_t eager;           /* 1: the step's kernels launched one by one, not as a CUDA graph (ncu) */
  int32_t no_tma;          /* 1: plain loads instead of TMA boxes */
  int32_t no_narrow;       /* 1: every escape level grid-wide (no narrow runs on one CTA) */
  int32_t no_esc_small;    /* 1: escaped trees always through the cooperative kernels */
  int32_t pipe;            /* receiver / tile pipeline bands: 0 default (24 for >= 256 tile rows), -1 off */
  int32_t pipe_unchained;  /* 1: receiver bands independent (default: chained) */
  uint32_t tile_grid;      /* CTAs of k_tiles (0: occupancy x SMs) */
  uint32_t esc_grid;       /* CTAs of the cooperative escape expansion (0: one per SM) */
  uint32_t esc_small_grid; /* CTAs of k_esc_small (0: one per SM) */
  uint32_t pipe_tile_grid; /* k_tiles CTAs per pipeline band (0: 4 per SM) */
  uint32_t lut_entries;    /* size of the host-libm F table per member and class (0: min(W*H + 1, 65537));
                              raised to cover every tile-tree cell count */
  uint32_t host_bands;     /* banded host step: bands (0: one per ~25 MB, <= 32; 1..3: unbanded) */
  uint32_t patch_cap;      /* banded host step: escaped-cell patch capacity (0: max(2^20, N/16)) */
  int32_t host_profile;    /* 1: banded host step prints its timing to stderr */
  int32_t esc_forest;      /* escaped trees by k_esc_forest (exact-area steps): 0 auto (>= 1/4 of the cells
                              escape), 1 always, -1 never (level path) */
  int32_t mfd_levels;      /* 1: routing = kMfd through the level-synchronous plan + accumulation and the
                              global level path (default: MFD area by tile passes, D8 part on the tile path) */
  int32_t phase_clocks;    /* 1: lemgpu_diag.seconds holds lem::Phase seconds (per-CTA phase clocks in the
                              tile pass, ~1.5 % of a 10000^2 step); 0: the seconds are 0 (kernel_s still
                              holds the kernel spans).  The C++ shim and the Python drop-in turn it on. */
} lemgpu_options;

typedef struct lemgpu_ctx lemgpu_ctx;

/* ---- lifetime ---------------------------------------------------------- */

/* One DEM of width x height on CUDA device `device`.  Validates params the
 * way SimParams::validate does (proj/src/erosion.cpp:10-17) and the grid
 * bounds of RunConfig::validate (proj/src/config.cpp:155-173).
 * Replaces: SimWorkspace construction (proj/include/lem/simulation.hpp:43-52). */
int lemgpu_create(int device, uint32_t width, uint32_t height, const lemgpu_params* params,
                  lemgpu_ctx** out);

/* `members` independent realisations of width x height, batched into the
 * same launches (stacked row-major, member-major).  per_member may be NULL
 * (all members use params->K / params->m_exp). */
int lemgpu_create_ensemble(int device, uint32_t width, uint32_t height, uint32_t members,
                           const lemgpu_params* params, const lemgpu_member* per_member,
                           lemgpu_ctx** out);

/* lemgpu_create_ensemble with explicit options (NULL: defaults). */
int lemgpu_create_ex(int device, uint32_t width, uint32_t height, uint32_t members, const lemgpu_params* params,
                     const lemgpu_member* per_member, const lemgpu_options* options, lemgpu_ctx** out);

void lemgpu_destroy(lemgpu_ctx* ctx);

/* ---- state ------------------------------------------------------------- */

/* Copy all members' elevations in / out (member-major, row-major, f64).
 * Upload rejects non-finite values like run_simulation does
 * (proj/src/scheduler.cpp:474-477) -> LEMGPU_ECONFIG. */
int lemgpu_upload_elev(lemgpu_ctx* ctx, const double* host);
int lemgpu_download_elev(lemgpu_ctx* ctx, double* host);

/* Device-side lem::generate_terrain (proj/src/terrain.cpp:19-31), bit-exact;
 * seeds[m] for member m (seeds may be NULL -> seed 42 for every member). */
int lemgpu_generate_terrain(lemgpu_ctx* ctx, const uint64_t* seeds);

/* Priority-Flood depression filling of the device elevation, in place
 * (every member): lem::priority_flood_fill (proj/src/depressions.cpp:26-68),
 * bit-identical.  mode: LEMGPU_FILL_OFF (no-op), LEMGPU_FILL_EXACT (raise to
 * the spill elevation), LEMGPU_FILL_EPSILON (spill + epsilon; epsilon must be
 * > 0, config.cpp:164-165 -> LEMGPU_ECONFIG).  Replaces the fill that
 * run_simulation applies to the generated terrain (proj/src/scheduler.cpp:505). */
enum { LEMGPU_FILL_OFF = 0, LEMGPU_FILL_EXACT = 1, LEMGPU_FILL_EPSILON = 2 };
int lemgpu_fill(lemgpu_ctx* ctx, int mode, double epsilon);

/* StepSetup::routing / mfd_exponent (proj/include/lem/simulation.hpp:55-60,
 * config.hpp:14-32): routing 0 = d8/d4 (the receiver of the neighbourhood),
 * 1 = kMfd -- the drainage area that feeds the erosion is the slope-weighted
 * multiple-flow accumulation (compute_mfd / generate_mfd_order /
 * accumulate_mfd, proj/src/mfd.cpp:33-132) while the erosion still follows
 * the D8 receiver.  mfd_exponent must be > 0 (config.cpp:166) -> ECONFIG.
 * Replaces: the Routing::kMfd branch of simulate_front (simulation.cpp:53-60)
 * and step_rb_par_all (scheduler.cpp:248-254). */
int lemgpu_set_routing(lemgpu_ctx* ctx, int routing, double mfd_exponent);

/* The MFD drainage area and plan of the last step (routing = 1): A[N] =
 * ws.accum, order[N] / levels[nlevels + 1] = ws.mfd_plan (level-major,
 * ascending within a level, mfd.cpp:66-104).  Any pointer may be NULL. */
int lemgpu_download_mfd(lemgpu_ctx* ctx, double* A, uint32_t* order, uint32_t* levels, uint32_t* nlevels);

/* ---- stepping ---------------------------------------------------------- */

/* Run nsteps timesteps with the elevation device-resident, then synchronise.
 * per_step (nullable) receives nsteps diagnostics.  On a failing step the
 * call stops there and returns its status; later steps are not run.
 * Replaces: the run_simulation loop (proj/src/scheduler.cpp:490-498). */
int lemgpu_step(lemgpu_ctx* ctx, uint32_t nsteps, lemgpu_diag* per_step);

/* Enqueue nsteps without synchronising (diagnostics stay on the device
 * until lemgpu_sync).  For timing loops. */
int lemgpu_step_async(lemgpu_ctx* ctx, uint32_t nsteps);

/* Synchronise; copies out up to `cap` diagnostics of the steps enqueued
 * since the last sync (oldest first) and returns the first failing status. */
int lemgpu_sync(lemgpu_ctx* ctx, lemgpu_diag* out, uint32_t cap, uint32_t* count);

/* Asynchronous snapshot: after lemgpu_step_async, copy the elevation the last
 * enqueued step produced (and that step's diagnostics; diag_host nullable)
 * into host memory on a side stream, returning at once.  The next step runs
 * beside the copy (it only reads that state); the step after, which writes
 * the same buffer, waits for the copy on the device.  lemgpu_snapshot_wait
 * blocks until the copy has landed.  One snapshot in flight per context; pin
 * the host memory (lemgpu_host_register) for the copy to overlap.  Used by the
 * C++ shim's run_simulation (StepCallback / `lem run` snapshots,
 * proj/tools/lem.cpp:143-147). */
int lemgpu_snapshot_async(lemgpu_ctx* ctx, double* host, lemgpu_diag* diag_host);
int lemgpu_snapshot_wait(lemgpu_ctx* ctx);

/* One lem::strategy_step on a HOST raster: upload elev, one step, download
 * elev (the drop-in semantics of strategy_step(Raster<double>&, ...)).
 * Replaces: proj/src/scheduler.cpp:408-464 for StrategyKind::kRbGpu. */
int lemgpu_step_host(lemgpu_ctx* ctx, double* elev_inout, lemgpu_diag* diag);

/* ---- inspection (parity / debug) -------------------------------------- */

/* Graph of the LAST step, in the reference's formats:
 *   rec[N]            FlowGraph::rec            (flow_graph.hpp:23)
 *   dnum[N]           FlowGraph::dnum           (flow_graph.hpp:25)
 *   donor[N*conn]     FlowGraph::donor slots, kNoFlow-padded (flow_graph.hpp:24)
 *   order[N]          TraversalPlan::order      (traversal.hpp:21)
 *   levels[nlevels+1] TraversalPlan::levels     (traversal.hpp:22)
 *   A[N]              AccumField::values        (accumulation.hpp:13-16)
 * Any pointer may be NULL.  `levels` must hold N+2 entries when non-NULL. */
int lemgpu_download_graph(lemgpu_ctx* ctx, uint32_t* rec, uint8_t* dnum, uint32_t* donor,
                          uint32_t* order, uint32_t* levels, uint32_t* nlevels, double* A);

/* ---- ensemble ------------------------- */

/* Members [first, first + count) of `members_total` owned by `rank` of
 * `nranks`: contiguous balanced ranges, the reference's partition_sources
 * rule (proj/src/scheduler.cpp:396-406). */
int lemgpu_shard_members(uint32_t members_total, int nranks, int rank, uint32_t* first, uint32_t* count);

/* The context of one rank of a sharded ensemble: its member range of
 * per_member_all[members_total] (NULL: params' K and m for all), batched into
 * one context, with the per-member statistics enabled at its table rows every
 * stats_interval-th step.  Add the communicator with lemgpu_stats_comm_init. */
int lemgpu_create_ensemble_shard(int device, uint32_t width, uint32_t height, uint32_t members_total, int nranks,
                                 int rank, const lemgpu_params* params, const lemgpu_member* per_member_all,
                                 uint32_t stats_interval, const lemgpu_options* options, lemgpu_ctx** out);

/* Per-member statistics every `interval`-th step (0 or 1: every step): table
 * row (member_offset + m) of [members_total][4] = {mean, max, min, sum} of the
 * elevation that step STARTS from (the state the previous step left), by a
 * bandwidth-bound pass (8 B/cell) that runs beside the step's kernels in its
 * graph, in a fixed summation order (deterministic).  With interval > 1 those
 * steps launch a second pair of step graphs.  The statistics of the final
 * state: lemgpu_member_stats_device. */
int lemgpu_stats_enable(lemgpu_ctx* ctx, uint32_t member_offset, uint32_t members_total, uint32_t interval);
/* NCCL: rank 0 makes the id (ncclGetUniqueId, 128 bytes), the caller
 * broadcasts it (torch.distributed, MPI, ...), every rank joins.  From then
 * on each step's graph ends with ONE ncclAllReduce of the table (every row is
 * non-zero on exactly one rank, so the SUM is an exact gather).  NCCL is
 * loaded at run time (libnccl.so.2). */
int lemgpu_nccl_unique_id(void* id_out, uint32_t bytes);
int lemgpu_stats_comm_init(lemgpu_ctx* ctx, const void* id, uint32_t bytes, int nranks, int rank);
/* The table of the last step that computed it (host copy after a sync) / its device address. */
int lemgpu_stats_table(lemgpu_ctx* ctx, double* host_out);
const double* lemgpu_stats_table_device(const lemgpu_ctx* ctx);

/* Per-member statistics of the current elevation: out[4*m + {0,1,2,3}] =
 * {mean h, max h, min h, sum h}.  Deterministic (fixed reduction order).
 * `device_out` is a DEVICE pointer written on the context's stream. */
int lemgpu_member_stats_device(lemgpu_ctx* ctx, double* device_out);

/* ---- errors ------------------------------------------------------------ */
const char* lemgpu_error_message(const lemgpu_ctx* ctx);
uint32_t lemgpu_error_cell(const lemgpu_ctx* ctx);

/* ---- plumbing ---------------------------------------------------------- */
uint32_t lemgpu_abi_version(void);
uint64_t lemgpu_num_cells(const lemgpu_ctx* ctx);     /* members * width * height */
void* lemgpu_stream(lemgpu_ctx* ctx);                 /* the context's cudaStream_t */
int lemgpu_device_bytes(const lemgpu_ctx* ctx, uint64_t* bytes);
/* Kernel nodes of one step's CUDA graph (the pipelined tile path runs the
 * receiver pass and k_tiles in bands).  Top-level nodes only: the bodies of
 * the global level path's conditional WHILE nodes (k_expand, k_deep_accum,
 * k_deep_erode; LEMGPU_PATH=global only) run a data-dependent number of times
 * and are not counted. */
uint32_t lemgpu_kernels_per_step(const lemgpu_ctx* ctx);
/* Bands of the receiver / tile pipeline of the step graph (0: not pipelined;
 * rasters of >= 256 tile rows are). */
uint32_t lemgpu_pipeline_bands(const lemgpu_ctx* ctx);

/* Device time accumulated over the steps synced since timing was enabled,
 * `ms` holds 5: [0] whole step (CUDA events around each graph launch on the
 * context stream), then the summed lemgpu_diag::kernel_s spans: [1] receiver
 * pass, [2] escape-path level expansion, [3] escape-path accumulation +
 * uplift + erosion, [4] tile pass. */
int lemgpu_kernel_timing(lemgpu_ctx* ctx, int enable);
int lemgpu_kernel_times(lemgpu_ctx* ctx, double* ms, uint32_t* launches);

/* Debug: %globaltimer stamps (ns) of the last completed step: k_recv_donor
 * begin/end, then the end of k_level0, of every k_expand level and of the
 * accumulation/erosion sweeps. */
int lemgpu_debug_timeline(lemgpu_ctx* ctx, uint64_t* ns, uint32_t cap, uint32_t* count);
/* Debug / test hook (no reference counterpart): copy `bytes` of a device
 * scratch array of the last step to host memory.  which: 0 = queue (order),
 * 1 = escape-path level bounds, 2 = control block, 3 = the tile pass's
 * per-cell level (u8, 0xFF: cell of an escaped tree) and 4 = its per-cell
 * drainage area (f64) -- 3 and 4 need lemgpu_debug_tile_capture.  Not used by
 * the step. */
int lemgpu_debug_copy(lemgpu_ctx* ctx, int which, void* host, uint64_t bytes);
/* Debug / test hook: when enabled, every step's tile pass (k_tiles) also
 * writes the TraversalPlan level and the drainage area of each cell it
 * finishes, straight from its shared-memory level lists and counts, so the
 * tests can pin those phases directly (not through the export path).  Costs
 * 9 B/cell of extra writes per step while on. */
int lemgpu_debug_tile_capture(lemgpu_ctx* ctx, int enable);

/* Which glibc pow the device reproduces (glibc_pow.cuh): 1 = __pow_fma,
 * 0 = __pow_sse2 -- the variant the HOST libm's ifunc selected, found at
 * context creation by probing ::pow -- or -1 when neither restatement matches
 * the host libm (pow(A,m) beyond the table and n != 1 are then not
 * bit-identical with the reference on this host).  ctx may be NULL. */
int lemgpu_pow_variant(const lemgpu_ctx* ctx);
/* Test hook (no reference counterpart): out[i] = pow(x[i], y[i]) computed by
 * the device restatement of glibc pow (variant as above) on `device` -- for
 * y = 2 through the n = 2 Newton fast path; host arrays of n doubles.  Lets
 * the tests compare it with the host libm. */
int lemgpu_debug_pow(int device, int variant, const double* x, const double* y, double* out, uint64_t n);

/* Pin / unpin caller host memory (cudaHostRegister) for fast H2D/D2H. */
int lemgpu_host_register(void* ptr, size_t bytes);
int lemgpu_host_unregister(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* LEMGPU_H */
