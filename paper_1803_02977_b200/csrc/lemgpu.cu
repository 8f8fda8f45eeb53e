// lemgpu.cu -- host side of the C-ABI declared in include/lemgpu.h.
//
// Owns one device context per DEM (or per batch of ensemble members):
// device buffers laid out for HBM (SoA: cell-major state, queue-position-major
// scratch), one CUDA stream, and ONE instantiated CUDA graph per context that
// is a whole timestep (see common.cuh): the level loops are graph WHILE nodes
// driven from the device, so a step is a single cudaGraphLaunch.
// No phase ever runs on the CPU.  The host computes only what must come from
// the host libm to be bit-identical with the reference: the stencil
// distances (neighborhood.hpp:17-23), pow(dist, n) and the pow(A, m) table.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "lemgpu.h"
#include "common.cuh"
#include "k_order.cuh"
#include "k_physics.cuh"
#include "k_recv_donor.cuh"
#include "k_fill.cuh"
#include "k_tiles.cuh"
#include "k_forest.cuh"
#include "k_mfd.cuh"
#include "k_mfd_tiles.cuh"
#include "k_util.cuh"

using namespace lemgpu;

struct lemgpu_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  StepArgs a{};
  lemgpu_params params{};
  std::vector<lemgpu_member> members;
  int scan_grid = 0, chunk_grid = 0, deep_grid = 0, tile_grid = 0;
  int tile_grid_mfd = 0;  // CTAs of the FP-area k_tiles that MFD routing runs
  int esc_grid = 0;  // CTAs of the level expansion of the escaped trees (a small workload)
  int deep_coop_grid = 0;  // CTAs of k_deep_coop (kDeepTPB threads, co-resident)
  int forest_grid = 0;     // CTAs of k_esc_forest (kFTPB threads, co-resident)
  int mfd_grid = 0;        // CTAs of k_mfd_levels (co-resident)
  int use_tiles = 1;  // k_tiles + escape path (else the global level path for every tree)
  bool opt_global = false;  // lemgpu_options::global_path (the tile path stays off after routing = d8 again)
  int routing = 0;          // 0 d8 / d4 (StepSetup::routing kD8), 1 kMfd (lemgpu_set_routing)
  bool opt_mfd_levels = false;  // lemgpu_options::mfd_levels (MFD through the level-synchronous global path)
  int mfd_tiles_grid = 0;       // CTAs of k_mfd_tiles (persistent)
  uint32_t mfd_src = 0;         // buffer the last step read (the MFD plan export rebuilds from it)
  // ping-pong elevation buffers: a step reads hbuf[p] and writes hbuf[p ^ 1];
  // graph[p] / exec[p] is the step that reads hbuf[p]
  double* hbuf[2] = {nullptr, nullptr};
  uint32_t cur = 0;         // buffer holding the elevation after every enqueued step
  uint32_t cur_synced = 0;  // ... before the pending steps
  cudaGraph_t graph[2] = {nullptr, nullptr};
  cudaGraphExec_t exec[2] = {nullptr, nullptr};
  CUtensorMap hmap[2]{};  // TMA descriptors of hbuf[p]: k_recv_donor box
  CUtensorMap tmap[2]{};  // ... k_tiles box
  uint32_t* d_levels_esc = nullptr;
  bool esc_small = true;  // k_esc_small ahead of the cooperative escape path
  int esc_small_grid = 1;  // its CTAs (kEscSmallPerSM per SM)
  int pipe = 0, pipe_tile_grid = 0;  // pipelined receivers / tiles (bands), k_tiles CTAs per band
  int pipe_chain = 1;                // receiver bands chained (else independent)
  int pow_variant = -1;              // host_pow_variant(): the glibc pow the device reproduces
  uint32_t pipe_bands = 0;           // bands of the pipelined graph (0: not pipelined)
  uint32_t opt_patch_cap = 0;        // lemgpu_options::patch_cap
  // ensemble statistics (lemgpu_stats_enable) and their NCCL all-reduce
  double* st_part = nullptr;   // receiver-block partials
  double* st_local = nullptr;  // [members_total][4]: this rank's rows, zeros elsewhere (all-reduce input)
  double* st_all = nullptr;    // [members_total][4]: every member (all-reduce output; == st_local without a comm)
  uint32_t st_total = 0, st_member0 = 0;
  uint32_t st_interval = 1;  // statistics every st_interval-th step (the graphs stat_exec[p])
  uint64_t st_steps = 0;     // steps enqueued since the statistics were enabled
  bool st_on = false;
  cudaGraph_t st_graph[2] = {nullptr, nullptr};
  cudaGraphExec_t st_exec[2] = {nullptr, nullptr};
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  // asynchronous snapshots (lemgpu_snapshot_async): side stream, events, the buffer being copied
  cudaStream_t s_snap = nullptr;
  cudaEvent_t ev_snap_step = nullptr, ev_snap_done = nullptr;
  bool snap_pending = false;
  uint32_t snap_buf = 0;
  bool host_profile = false;         // lemgpu_options::host_profile
  // banded host steps (lemgpu_step_host): copy streams, per-band events, patch count
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  std::vector<cudaEvent_t> band_ev;
  uint32_t* h_patch = nullptr;  // mapped pinned: count, then cells[patch_cap], then vals[patch_cap]
  uint32_t patch_cap = 0;
  int bands = 0;  // 0: one band per ~25 MB of raster, at most 32 (fewer than 4: no banding)
  // device allocations
  double* d_kdt = nullptr;
  double* d_mexp = nullptr;
  double* d_lut = nullptr;
  double* d_lut2 = nullptr;  // interleaved {F, RN(1 / RN(1 + F))} (n = 1 Newton without IEEE divisions)
  lemgpu_diag* d_diag = nullptr;
  uint32_t diag_cap = 4096;
  uint32_t pending = 0;  // steps enqueued since the last sync
  uint32_t last_nlevels = 0;
  bool have_graph = false;
  uint64_t device_bytes = 0;
  // timing: CUDA events around each graph launch + device phase stamps
  bool timing = false;
  std::vector<cudaEvent_t> ev;  // 2 per pending step
  double kernel_ms[5] = {0, 0, 0, 0, 0};  // step, recv_donor, order (escape), physics (escape), k_tiles
  uint32_t kernel_launches = 0;
  // errors
  std::string msg;
  uint32_t err_cell = LEMGPU_NOFLOW;
};

namespace {

thread_local std::string g_create_error;

int fail(lemgpu_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (ctx)
    ctx->msg = buf;
  else
    g_create_error = buf;
  return code;
}

#define CU(ctx, call)                                                                         \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail((ctx), LEMGPU_ECUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_),    \
                  __FILE__, __LINE__, cudaGetErrorString(e_));                                \
  } while (0)

// include/lem/neighborhood.hpp:17-23, compiled with -ffp-contract=off.
double offset_length(int dx, int dy, double sx, double sy) {
  const double ox = dx * sx;
  const double oy = dy * sy;
  if (dy == 0) return std::fabs(ox);
  if (dx == 0) return std::fabs(oy);
  return std::sqrt(ox * ox + oy * oy);
}

// SimParams::validate (proj/src/erosion.cpp:10-17).
int validate(const lemgpu_params* p, std::string& why) {
  if (!(p->dt > 0)) return why = "dt must be > 0", 1;
  if (!(p->epsilon > 0)) return why = "epsilon must be > 0", 1;
  if (!(p->K >= 0)) return why = "K must be >= 0", 1;
  if (!(p->n_exp > 0)) return why = "n_exp must be > 0", 1;
  if (!(p->dx > 0) || !(p->dy > 0)) return why = "cell spacing must be > 0", 1;
  if (p->max_newton_iters < 1) return why = "max_newton_iters must be >= 1", 1;
  if (p->connectivity == 6) return why = "hexagonal (6-connected) grids are not implemented", 1;
  if (p->connectivity != 4 && p->connectivity != 8)
    return why = "connectivity must be 4 or 8, got " + std::to_string(p->connectivity), 1;
  return 0;
}

// Which glibc pow the host libm runs (its ifunc picks __pow_fma on CPUs with
// FMA + AVX2, else __pow_sse2): the restatement (glibc_pow.cuh) that agrees
// with ::pow on a probe set spanning the regimes the step uses -- drainage
// areas to m, Newton differences to n and n - 1, random bit patterns.  The
// two variants disagree on ~0.04 % of such inputs, so 20000 probes separate
// them.  -1: neither matches (the device pow is then not the host's).
int host_pow_variant() {
  static int v = -2;
  if (v != -2) return v;
  double (*volatile libm_pow)(double, double) = &::pow;  // no constant folding
  uint64_t st = 0x243F6A8885A308D3ull;
  auto nx = [&st]() {
    uint64_t z = (st += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  };
  auto u01 = [&]() { return (double)(nx() >> 11) * 0x1p-53; };
  bool fma_ok = true, sse_ok = true;
  for (int i = 0; i < 20000 && (fma_ok || sse_ok); ++i) {
    double x, y;
    switch (i % 4) {
      case 0: x = (double)(1 + nx() % 8000000); y = 0.25 + 0.6 * u01(); break;
      case 1: x = std::ldexp(u01() + 0.5, -(int)(nx() % 60)); y = 2.0; break;
      case 2: x = std::ldexp(u01() + 0.5, -(int)(nx() % 60)); y = -0.9 + 2.8 * u01(); break;
      default: {
        uint64_t a = nx(), b = nx();
        std::memcpy(&x, &a, 8);
        std::memcpy(&y, &b, 8);
      }
    }
    const double w = libm_pow(x, y);
    auto same = [&](double g) {
      uint64_t ga, wa;
      std::memcpy(&ga, &g, 8);
      std::memcpy(&wa, &w, 8);
      return ga == wa || (std::isnan(g) && std::isnan(w));
    };
    fma_ok = fma_ok && same(glibc_pow<true>(x, y));
    sse_ok = sse_ok && same(glibc_pow<false>(x, y));
  }
  v = fma_ok ? 1 : sse_ok ? 0 : -1;
  return v;
}

__global__ void k_debug_pow(int variant, const double* x, const double* y, double* out, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = y[i] == 2.0 ? glibc_pow_sq_dev(variant, x[i]) : glibc_pow_dev(variant, x[i], y[i]);  // y = 2: the Newton fast path
}

// True when every sum of k <= nmax copies of w is exactly k*w, i.e. w's
// significand leaves room for log2(nmax) more bits.  Then A is a function
// of the integer donor count and pow(A, m) can come from a host table.
bool area_sums_exact(double w, uint64_t nmax) {
  int e;
  double m = std::frexp(w, &e);  // w = m * 2^e, m in [0.5,1)
  uint64_t sig = (uint64_t)std::ldexp(m, 53);
  int tz = 0;
  while (tz < 53 && !(sig & 1)) {
    sig >>= 1;
    ++tz;
  }
  const int sig_bits = 53 - tz;
  int need = 0;
  while (need < 64 && (1ull << need) <= nmax) ++need;
  return sig_bits + need <= 53;
}

template <typename T>
int dmalloc(lemgpu_ctx* ctx, T** p, size_t count) {
  const size_t bytes = count * sizeof(T);
  CU(ctx, cudaMalloc((void**)p, bytes ? bytes : 16));
  ctx->device_bytes += bytes;
  return 0;
}

// One timestep as a CUDA graph (see common.cuh).  StepArgs is captured by
// value in every kernel node; everything that changes from step to step lives
// in the device control block.
int add_kernel(lemgpu_ctx* ctx, cudaGraph_t g, cudaGraphNode_t* prev, const void* fn, dim3 grid,
               dim3 block, size_t smem, StepArgs* sa, CUtensorMap* map, bool cooperative = false) {
  cudaKernelNodeParams kp{};
  void* args[] = {sa, map};  // copied into the node
  kp.func = const_cast<void*>(fn);
  kp.gridDim = grid;
  kp.blockDim = block;
  kp.sharedMemBytes = (unsigned)smem;
  kp.kernelParams = args;
  cudaGraphNode_t n;
  CU(ctx, cudaGraphAddKernelNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &kp));
  if (cooperative) {  // all CTAs co-resident: the kernel's grid barrier is safe
    cudaKernelNodeAttrValue v{};
    v.cooperative = 1;
    CU(ctx, cudaGraphKernelNodeSetAttribute(n, cudaKernelNodeAttributeCooperative, &v));
  }
  *prev = n;
  return 0;
}

// A kernel node with an explicit dependency list (pipelined tile path).
int add_kernel_deps(lemgpu_ctx* ctx, cudaGraph_t g, const std::vector<cudaGraphNode_t>& deps, cudaGraphNode_t* out,
                    const void* fn, dim3 grid, dim3 block, size_t smem, StepArgs* sa, CUtensorMap* map) {
  cudaKernelNodeParams kp{};
  void* args[] = {sa, map};
  kp.func = const_cast<void*>(fn);
  kp.gridDim = grid;
  kp.blockDim = block;
  kp.sharedMemBytes = (unsigned)smem;
  kp.kernelParams = args;
  CU(ctx, cudaGraphAddKernelNode(out, g, deps.empty() ? nullptr : deps.data(), deps.size(), &kp));
  return 0;
}

// NCCL, loaded on first use (dlopen): the library itself does not depend on
// it, and a process that already holds torch's libnccl.so.2 shares that copy.
struct NcclApi {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  const char* (*errStr)(ncclResult_t) = nullptr;
  bool load() {
    if (tried) return ok;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return false;
    }
    getUniqueId = reinterpret_cast<decltype(getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    commInitRank = reinterpret_cast<decltype(commInitRank)>(dlsym(h, "ncclCommInitRank"));
    allReduce = reinterpret_cast<decltype(allReduce)>(dlsym(h, "ncclAllReduce"));
    commDestroy = reinterpret_cast<decltype(commDestroy)>(dlsym(h, "ncclCommDestroy"));
    errStr = reinterpret_cast<decltype(errStr)>(dlsym(h, "ncclGetErrorString"));
    ok = getUniqueId && commInitRank && allReduce && commDestroy && errStr;
    if (!ok) why = "libnccl.so.2 lacks a needed symbol";
    return ok;
  }
};
NcclApi& nccl() {
  static NcclApi api;
  return api;
}

// The statistics nodes of a step: the per-member fold of the receiver pass's
// partials (or, for short members, a separate pass), then ONE all-reduce of
// the whole table over NCCL (SUM: every member's row is non-zero on exactly
// one rank, so the sum is an exact copy), captured into the step graph.
int add_stats_nodes(lemgpu_ctx* ctx, cudaGraph_t g, cudaGraphNode_t* prev, StepArgs* a) {
  // the pass reads the step's INPUT elevation, which nothing writes during the
  // step: a root node, running beside the step's kernels; the fold joins it
  cudaGraphNode_t pass, fold;
  int rc = add_kernel_deps(ctx, g, {}, &pass, (const void*)k_stats_pass, dim3(a->st_chunks, a->M), dim3(kTPB), 0, a,
                           nullptr);
  if (!rc) {
    std::vector<cudaGraphNode_t> d{pass};
    if (*prev) d.push_back(*prev);
    rc = add_kernel_deps(ctx, g, d, &fold, (const void*)k_stats_fold, dim3((a->M + 31) / 32), dim3(32), 0, a, nullptr);
  }
  if (rc) return rc;
  *prev = fold;
  if (!ctx->comm) return 0;
  cudaStream_t cs;
  CU(ctx, cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  cudaGraph_t child = nullptr;
  CU(ctx, cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const ncclResult_t nr = nccl().allReduce(ctx->st_local, ctx->st_all, (size_t)ctx->st_total * 4, ncclDouble, ncclSum,
                                           ctx->comm, cs);
  const cudaError_t ce = cudaStreamEndCapture(cs, &child);
  cudaStreamDestroy(cs);
  if (nr != ncclSuccess) return fail(ctx, LEMGPU_ECUDA, "ncclAllReduce capture: %s", nccl().errStr(nr));
  if (ce != cudaSuccess) return fail(ctx, LEMGPU_ECUDA, "stream capture: %s", cudaGetErrorString(ce));
  cudaGraphNode_t n;
  CU(ctx, cudaGraphAddChildGraphNode(&n, g, prev, 1, child));
  cudaGraphDestroy(child);
  *prev = n;
  return 0;
}

// The step being enqueued ends with the statistics.
bool stats_due(const lemgpu_ctx* ctx) { return ctx->st_on && (ctx->st_steps + 1) % ctx->st_interval == 0; }

// Eager form of the statistics pass, at the start of the step (it reads the input).
void enqueue_stats_pass(lemgpu_ctx* ctx, StepArgs& a, cudaStream_t st) {
  if (ctx->st_on && stats_due(ctx)) k_stats_pass<<<dim3(a.st_chunks, a.M), kTPB, 0, st>>>(a);
}

// Eager form of add_stats_nodes (eager steps, banded host steps).
int enqueue_stats(lemgpu_ctx* ctx, StepArgs& a, cudaStream_t st) {
  if (!ctx->st_on || !stats_due(ctx)) return 0;
  k_stats_fold<<<(a.M + 31) / 32, 32, 0, st>>>(a);  // (k_stats_pass ran at the step's start: enqueue_stats_pass)
  if (ctx->comm) {
    const ncclResult_t nr = nccl().allReduce(ctx->st_local, ctx->st_all, (size_t)ctx->st_total * 4, ncclDouble,
                                             ncclSum, ctx->comm, st);
    if (nr != ncclSuccess) return fail(ctx, LEMGPU_ECUDA, "ncclAllReduce: %s", nccl().errStr(nr));
  }
  return 0;
}

int add_while(lemgpu_ctx* ctx, cudaGraph_t g, cudaGraphNode_t* prev, cudaGraphConditionalHandle h,
              const void* fn, dim3 grid, size_t smem, StepArgs* sa) {
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t n;
  CU(ctx, cudaGraphAddNode(&n, g, *prev ? prev : nullptr, *prev ? 1 : 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  cudaGraphNode_t inner = nullptr;
  const int rc = add_kernel(ctx, body, &inner, fn, grid, dim3(kTPB), smem, sa, nullptr);
  if (rc) return rc;
  *prev = n;
  return 0;
}

// The StepArgs of the step that reads hbuf[p].
StepArgs step_args(const lemgpu_ctx* ctx, uint32_t p) {
  StepArgs a = ctx->a;
  a.h = ctx->hbuf[p];
  a.hout = ctx->hbuf[p ^ 1u];
  a.tiles = ctx->use_tiles;
  a.levels = ctx->use_tiles ? ctx->d_levels_esc : ctx->a.levels;
  a.expect_cells = ctx->use_tiles ? 0u : a.N;
  if (ctx->use_tiles) a.scan_grid = (uint32_t)ctx->esc_grid;
  if (!ctx->use_tiles) a.planes = nullptr;  // only k_tiles reads the code bit planes
  a.dmask_valid = ctx->use_tiles ? 0 : 1;   // the tile path derives donor masks from the codes where needed
  if (a.mfd_A) a.esc_forest = 0;  // k_esc_forest carries integer counts; the MFD area is read by the other kernels
  return a;
}

template <int CONN, bool EX, bool MF = false, bool PH = true>
const void* tiles_fn_nk(int nk) {
  return nk == 1 ? (const void*)k_tiles<CONN, 1, EX, MF, PH> : nk == 2 ? (const void*)k_tiles<CONN, 2, EX, MF, PH>
                                                                        : (const void*)k_tiles<CONN, 0, EX, MF, PH>;
}
// (routing = kMfd: the MF instantiation reads the MFD area from global
// memory; the count layout serves for its escape marks whatever the cell area)
const void* tiles_fn(const StepArgs& a) {
  if (a.mfd_A) return a.conn == 8 ? tiles_fn_nk<8, true, true>(a.nkind) : tiles_fn_nk<4, true, true>(a.nkind);
  if (a.lut_exact && !a.phclk)  // the production instantiation: no phase clocks
    return a.conn == 8 ? tiles_fn_nk<8, true, false, false>(a.nkind) : tiles_fn_nk<4, true, false, false>(a.nkind);
  if (a.lut_exact) return a.conn == 8 ? tiles_fn_nk<8, true>(a.nkind) : tiles_fn_nk<4, true>(a.nkind);
  return a.conn == 8 ? tiles_fn_nk<8, false>(a.nkind) : tiles_fn_nk<4, false>(a.nkind);
}
// the tile path's receiver pass (k_recv): division-free selection for D8 with unit cardinal spacing
const void* recv_fn(const StepArgs& a) {
  if (a.conn == 4) return (const void*)k_recv<4, false>;
  return a.unit_card ? (const void*)k_recv<8, true> : (const void*)k_recv<8, false>;
}
const void* forest_fn(int nk) {
  return nk == 1 ? (const void*)k_esc_forest<1> : nk == 2 ? (const void*)k_esc_forest<2> : (const void*)k_esc_forest<0>;
}
size_t tiles_smem(const StepArgs& a) {
  return a.lut_exact || a.mfd_A ? tiles_smem_bytes<true>() : tiles_smem_bytes<false>();
}

// The step graph that reads hbuf[p]; with_stats: ending with the ensemble
// statistics and their all-reduce.
int build_graph(lemgpu_ctx* ctx, uint32_t p, bool with_stats = false) {
  StepArgs a = step_args(ctx, p);
  cudaGraph_t g;
  CU(ctx, cudaGraphCreate(&g, 0));
  (with_stats && ctx->st_interval > 1 ? ctx->st_graph[p] : ctx->graph[p]) = g;
  if (!ctx->use_tiles)  // the tile path expands the escaped trees inside one cooperative kernel
    CU(ctx, cudaGraphConditionalHandleCreate(&a.h_expand, g, 1, cudaGraphCondAssignDefault));
  if (!ctx->use_tiles) {  // the tile path sweeps deep plans inside one cooperative kernel
    CU(ctx, cudaGraphConditionalHandleCreate(&a.h_dacc, g, 0, cudaGraphCondAssignDefault));
    CU(ctx, cudaGraphConditionalHandleCreate(&a.h_deros, g, 0, cudaGraphCondAssignDefault));
  }
  // tile path with k_esc_small: the cooperative escape kernels behind an IF
  // node that k_esc_small's last CTA clears when it finished every escaped tree
  // (their launches are most of a small raster's step)
  a.esc_if = ctx->use_tiles && ctx->esc_small ? 1 : 0;
  if (a.esc_if) CU(ctx, cudaGraphConditionalHandleCreate(&a.h_esc, g, 1, cudaGraphCondAssignDefault));
  const int nk = a.nkind;
  const void* fdc = nk == 1 ? (const void*)k_deep_coop<1> : nk == 2 ? (const void*)k_deep_coop<2> : (const void*)k_deep_coop<0>;
  const void* fk1 = ctx->use_tiles ? recv_fn(a)
                                   : (a.conn == 8 ? (const void*)k_recv_donor<8> : (const void*)k_recv_donor<4>);
  const void* fes = nk == 1 ? (const void*)k_esc_small<1> : nk == 2 ? (const void*)k_esc_small<2> : (const void*)k_esc_small<0>;
  const void* fch = nk == 1 ? (const void*)k_chunks<1> : nk == 2 ? (const void*)k_chunks<2> : (const void*)k_chunks<0>;
  const void* fde = nk == 1 ? (const void*)k_deep_erode<1> : nk == 2 ? (const void*)k_deep_erode<2> : (const void*)k_deep_erode<0>;
  cudaGraphNode_t prev = nullptr;
  int rc;
  const dim3 g1((a.W + kBX - 1) / kBX, (a.Htot + kBY - 1) / kBY);
  // the tile path's escape kernels after k_esc_small (in the IF node's body, or inline)
  auto add_escape = [&](cudaGraph_t gg, cudaGraphNode_t* pv) -> int {
    int r;
    if ((a.esc_forest && (r = add_kernel(ctx, gg, pv, forest_fn(nk), dim3(ctx->forest_grid), dim3(kFTPB),
                                         kForestSmemBytes, &a, nullptr, true))) ||
        (r = add_kernel(ctx, gg, pv, (const void*)k_esc_bfs, dim3(a.scan_grid), dim3(kTPB), 0, &a, nullptr, true)) ||
        (r = add_kernel(ctx, gg, pv, fch, dim3(ctx->chunk_grid), dim3(kChunkTPB), kChunksSmemBytes, &a, nullptr)) ||
        (r = add_kernel(ctx, gg, pv, fdc, dim3(ctx->deep_coop_grid), dim3(kDeepTPB), kDeepSmemBytes, &a, nullptr,
                        true)))
      return r;
    return 0;
  };
  auto add_escape_path = [&]() -> int {
    if (!a.esc_if) return add_escape(g, &prev);
    cudaGraphNodeParams cp{};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = a.h_esc;
    cp.conditional.type = cudaGraphCondTypeIf;
    cp.conditional.size = 1;
    cudaGraphNode_t n;
    CU(ctx, cudaGraphAddNode(&n, g, prev ? &prev : nullptr, prev ? 1 : 0, &cp));
    cudaGraphNode_t inner = nullptr;
    const int r = add_escape(cp.conditional.phGraph_out[0], &inner);
    prev = n;
    return r;
  };
  if (ctx->use_tiles && a.mfd_A) {
    // routing = kMfd: the MFD drainage area first (pass 0 over every tile,
    // then the queued tiles until a pass queues none), then the D8 tile path
    CU(ctx, cudaGraphConditionalHandleCreate(&a.h_mfd, g, 0, cudaGraphCondAssignDefault));
    StepArgs a0 = a;
    a0.mfd_all = 1;
    a.mfd_all = 0;
    if ((rc = add_kernel(ctx, g, &prev, (const void*)k_mfd_tiles, dim3(ctx->mfd_tiles_grid), dim3(kMTPB),
                         kMfdTileSmemBytes, &a0, nullptr)) ||
        (rc = add_kernel(ctx, g, &prev, (const void*)k_mfd_tiles, dim3(ctx->mfd_tiles_grid), dim3(kMTPB),
                         kMfdTileSmemBytes, &a, nullptr)) ||
        (rc = add_while(ctx, g, &prev, a.h_mfd, (const void*)k_mfd_tail, dim3(ctx->scan_grid), 0, &a)))
      return rc;
  }
  if (ctx->use_tiles && ctx->pipe > 1 && !a.mfd_A) {
    // pipelined: the receiver pass in bands of tile rows (a chain), k_tiles of
    // band b after the receivers of band b+1; k_tiles limited to 4 CTAs per
    // SM so the next receiver band's CTAs run beside it
    const uint32_t W = a.W, Ht = a.Htot, ntx = (W + kTX - 1) / kTX, nty = (Ht + kTY - 1) / kTY;
    // tile rows per band, a multiple of kRq so every band starts on a k_recv
    // row block (kBY rows) as well as on a tile row (kTY rows)
    constexpr uint32_t kRq = (uint32_t)(kBY / std::gcd(kBY, kTY));
    const uint32_t R = ((nty + (uint32_t)ctx->pipe - 1) / (uint32_t)ctx->pipe + kRq - 1) / kRq * kRq;
    const uint32_t nb = (nty + R - 1) / R;
    ctx->pipe_bands = nb;
    std::vector<cudaGraphNode_t> rn(nb), tn(nb);
    for (uint32_t b = 0; b < nb; ++b) {
      StepArgs ab = a;
      const uint32_t y0 = b * R * (uint32_t)kTY, y1 = std::min((b + 1) * R * (uint32_t)kTY, Ht);  // raster rows
      ab.by0 = y0 / (uint32_t)kBY;
      const uint32_t nby = (y1 - y0 + (uint32_t)kBY - 1) / (uint32_t)kBY;
      std::vector<cudaGraphNode_t> d;
      if (b && ctx->pipe_chain) d.push_back(rn[b - 1]);
      if ((rc = add_kernel_deps(ctx, g, d, &rn[b], fk1, dim3(g1.x, nby), dim3(kTPB), 0, &ab, &ctx->hmap[p])))
        return rc;
    }
    for (uint32_t b = 0; b < nb; ++b) {
      StepArgs ab = a;
      ab.t_lo = b * R * ntx;
      ab.t_hi = std::min((b + 1) * R, nty) * ntx;
      std::vector<cudaGraphNode_t> d{rn[std::min(b + 1, nb - 1)]};
      if (!ctx->pipe_chain) {  // the receiver bands are independent: depend on the three this band reads
        if (b + 1 < nb) d.push_back(rn[b]);
        if (b >= 1) d.push_back(rn[b - 1]);
      }
      const uint32_t grid = std::min<uint32_t>((uint32_t)ctx->pipe_tile_grid, ab.t_hi - ab.t_lo);
      if ((rc = add_kernel_deps(ctx, g, d, &tn[b], tiles_fn(a), dim3(grid), dim3(kTTPB), tiles_smem(a), &ab,
                                &ctx->tmap[p])))
        return rc;
    }
    cudaGraphNode_t join;
    CU(ctx, cudaGraphAddEmptyNode(&join, g, tn.data(), tn.size()));
    prev = join;
    if ((ctx->esc_small &&
         (rc = add_kernel(ctx, g, &prev, fes, dim3(ctx->esc_small_grid), dim3(kTPB), kEscSmallSmemBytes, &a, nullptr))) ||
        (rc = add_escape_path()))
      return rc;
  } else if (ctx->use_tiles) {
    if ((rc = add_kernel(ctx, g, &prev, fk1, g1, dim3(kTPB), 0, &a, &ctx->hmap[p])) ||
        (rc = add_kernel(ctx, g, &prev, tiles_fn(a), dim3(a.mfd_A ? ctx->tile_grid_mfd : ctx->tile_grid), dim3(kTTPB),
                         tiles_smem(a), &a,
                         &ctx->tmap[p])) ||
        (ctx->esc_small &&
         (rc = add_kernel(ctx, g, &prev, fes, dim3(ctx->esc_small_grid), dim3(kTPB), kEscSmallSmemBytes, &a, nullptr))) ||
        (rc = add_escape_path()))
      return rc;
  } else {
    if ((a.mfd_A &&  // routing = kMfd: the MFD graph, plan and drainage area first (they read only h)
         ((rc = add_kernel(ctx, g, &prev, (const void*)k_mfd_graph, dim3(ctx->deep_grid), dim3(kTPB), 0, &a, nullptr)) ||
          (rc = add_kernel(ctx, g, &prev, (const void*)k_mfd_levels, dim3(ctx->mfd_grid), dim3(kTPB), 0, &a, nullptr,
                           true)))) ||
        (rc = add_kernel(ctx, g, &prev, fk1, g1, dim3(kTPB), 0, &a, &ctx->hmap[p])) ||
        (rc = add_kernel(ctx, g, &prev, (const void*)k_l0_count, dim3(ctx->scan_grid), dim3(kTPB), 0, &a, nullptr)) ||
        (rc = add_kernel(ctx, g, &prev, (const void*)k_l0_write, dim3(ctx->scan_grid), dim3(kTPB), 0, &a, nullptr)))
      return rc;
  }
  if ((!ctx->use_tiles && (rc = add_while(ctx, g, &prev, a.h_expand, (const void*)k_expand, dim3(a.scan_grid), 0, &a))) ||
      (!ctx->use_tiles &&
       (rc = add_kernel(ctx, g, &prev, fch, dim3(ctx->chunk_grid), dim3(kChunkTPB), kChunksSmemBytes, &a, nullptr))) ||
      (!ctx->use_tiles &&
       ((rc = add_kernel(ctx, g, &prev, (const void*)k_deep_prep, dim3(ctx->deep_grid), dim3(kTPB), 0, &a, nullptr)) ||
        (rc = add_while(ctx, g, &prev, a.h_dacc, (const void*)k_deep_accum, dim3(ctx->deep_grid), 0, &a)) ||
        (rc = add_while(ctx, g, &prev, a.h_deros, fde, dim3(ctx->deep_grid), 0, &a)) ||
        (rc = add_kernel(ctx, g, &prev, (const void*)k_deep_final, dim3(ctx->deep_grid), dim3(kTPB), 0, &a, nullptr)))) ||
      (with_stats && (rc = add_stats_nodes(ctx, g, &prev, &a))) ||
      (rc = add_kernel(ctx, g, &prev, (const void*)k_finalize, dim3(1), dim3(32), 0, &a, nullptr)))
    return rc;
  CU(ctx, cudaGraphInstantiate(with_stats && ctx->st_interval > 1 ? &ctx->st_exec[p] : &ctx->exec[p], g, 0));
  return 0;
}

// StepArgs is captured by value in the graph nodes: rebuild both step graphs
// after a change of the context's configuration.
void destroy_graphs(lemgpu_ctx* ctx) {
  for (uint32_t p = 0; p < 2; ++p) {
    if (ctx->exec[p]) cudaGraphExecDestroy(ctx->exec[p]);
    if (ctx->graph[p]) cudaGraphDestroy(ctx->graph[p]);
    if (ctx->st_exec[p]) cudaGraphExecDestroy(ctx->st_exec[p]);
    if (ctx->st_graph[p]) cudaGraphDestroy(ctx->st_graph[p]);
    ctx->exec[p] = ctx->st_exec[p] = nullptr;
    ctx->graph[p] = ctx->st_graph[p] = nullptr;
  }
}

// Statistics every step: they are part of the step graphs; every k-th step:
// a second pair of graphs with them, launched on those steps.
int rebuild_graphs(lemgpu_ctx* ctx) {
  destroy_graphs(ctx);
  for (uint32_t p = 0; p < 2; ++p) {
    int rc = build_graph(ctx, p, ctx->st_on && ctx->st_interval == 1);
    if (!rc && ctx->st_on && ctx->st_interval > 1) rc = build_graph(ctx, p, true);
    if (rc) return rc;
  }
  return 0;
}


int create_impl(int device, uint32_t W, uint32_t H, uint32_t M, const lemgpu_params* p,
                const lemgpu_member* per_member, const lemgpu_options* opts, lemgpu_ctx** out) {
  *out = nullptr;
  const lemgpu_options o = opts ? *opts : lemgpu_options{};
  if (!p) return fail(nullptr, LEMGPU_ECONFIG, "params must not be NULL");
  std::string why;
  if (validate(p, why)) return fail(nullptr, LEMGPU_ECONFIG, "%s", why.c_str());
  if (W < 3 || H < 3) return fail(nullptr, LEMGPU_ECONFIG, "raster must be at least 3x3");
  if (M < 1) return fail(nullptr, LEMGPU_ECONFIG, "members must be >= 1");
  const uint64_t N64 = (uint64_t)W * H * M;
  if (N64 >= 0xFFFFFFFFull)  // config.cpp:159-161 caps the grid at 2^32-1 cells
    return fail(nullptr, LEMGPU_ECONFIG, "grid of %llu cells exceeds 2^32-1", (unsigned long long)N64);

  lemgpu_ctx* ctx = new (std::nothrow) lemgpu_ctx();
  if (!ctx) return fail(nullptr, LEMGPU_EOTHER, "out of host memory");
  ctx->device = device;
  ctx->params = *p;
  ctx->members.resize(M);
  for (uint32_t m = 0; m < M; ++m)
    ctx->members[m] = per_member ? per_member[m] : lemgpu_member{p->K, p->m_exp};
  for (uint32_t m = 0; m < M; ++m) {
    if (!(ctx->members[m].K >= 0)) {
      delete ctx;
      return fail(nullptr, LEMGPU_ECONFIG, "K must be >= 0 (member %u)", m);
    }
  }

  auto bail = [&](int rc) {
    g_create_error = ctx->msg;
    lemgpu_destroy(ctx);
    return rc;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, LEMGPU_ECUDA, "cannot select CUDA device %d", device);
  }
  int coop = 0, nsm = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
  if (!coop) {
    delete ctx;
    return fail(nullptr, LEMGPU_ECUDA, "device %d lacks cooperative launch", device);
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return fail(nullptr, LEMGPU_ECUDA, "cudaStreamCreate failed");
  }

  StepArgs& a = ctx->a;
  const uint32_t N = (uint32_t)N64;
  a.W = W;
  a.H = H;
  a.M = M;
  a.N = N;
  a.MN = W * H;
  a.Htot = H * M;
  a.perim = M * (2 * W + 2 * H - 4);
  a.conn = p->connectivity;
  a.nkind = p->n_exp == 1.0 ? 1 : p->n_exp == 2.0 ? 2 : 0;
  a.maxit = p->max_newton_iters;
  a.du = p->uplift_rate * p->dt;
  a.w0 = p->dx * p->dy;  // SimParams::cell_area (erosion.hpp:26)
  a.w0_is_one = a.w0 == 1.0;
  a.n_exp = p->n_exp;
  a.eps = p->epsilon;
  a.dist_one = 0;
  for (int k = 0; k < 8; ++k) {
    a.dist[k] = offset_length(dir_ox(k), dir_oy(k), p->dx, p->dy);
    if (a.dist[k] == 1.0) a.dist_one |= 1u << k;
  }
  a.unit_card = (a.dist[1] == 1.0 && a.dist[3] == 1.0) ? 1 : 0;
  a.rinv_diag = 1.0 / a.dist[0];
  a.dist_recip = 0;
  for (int k = 0; k < 8; ++k) {
    a.rdist[k] = 1.0 / a.dist[k];
    if (a.dist[k] >= 1.0 && a.dist[k] < 0x1p500) a.dist_recip |= 1u << k;
  }
  a.powdist_h = std::pow(a.dist[3], p->n_exp);
  a.powdist_v = std::pow(a.dist[1], p->n_exp);
  a.powdist_d = std::pow(a.dist[0], p->n_exp);
  a.lut_exact = area_sums_exact(a.w0, (uint64_t)a.MN) ? 1 : 0;
  ctx->pow_variant = host_pow_variant();
  a.pow_fma = ctx->pow_variant != 0 ? 1 : 0;
  uint32_t lut_entries = a.MN < 65536u ? a.MN + 1 : 65537u;
  if (o.lut_entries) {
    // the tile pass indexes the table with tile-tree cell counts unchecked (k_tiles EX path)
    const uint32_t need = std::min<uint32_t>(a.MN, (uint32_t)(kDW * kDH)) + 1u;
    lut_entries = std::max(o.lut_entries, need);
  }
  if (lut_entries < 2) lut_entries = 2;
  a.lut_entries = lut_entries;

  // host-libm tables (bit-identical with the reference's pow on this host):
  // F(a, class) = ((K*dt) * pow(a*w0, m)) / pow(dist_class, n), the exact
  // rounding sequence of erode_one_cell (erosion.cpp:38-39)
  std::vector<double> kdt(M), mexp(M), lut((size_t)M * 3 * lut_entries);
  const double pdc[3] = {a.powdist_h, a.powdist_v, a.powdist_d};
  for (uint32_t m = 0; m < M; ++m) {
    kdt[m] = ctx->members[m].K * p->dt;  // erosion.cpp:38: K * dt first
    mexp[m] = ctx->members[m].m_exp;
    for (uint32_t i = 0; i < lut_entries; ++i) {
      const double kp = kdt[m] * std::pow((double)i * a.w0, mexp[m]);
      for (int c = 0; c < 3; ++c) lut[((size_t)m * 3 + c) * lut_entries + i] = kp / pdc[c];
    }
  }

  int rc;
  if ((rc = dmalloc(ctx, &ctx->d_kdt, M)) || (rc = dmalloc(ctx, &ctx->d_mexp, M)) ||
      (rc = dmalloc(ctx, &ctx->d_lut, lut.size())) || (rc = dmalloc(ctx, &ctx->d_lut2, 2 * lut.size())) || (rc = dmalloc(ctx, &ctx->hbuf[0], N)) ||
      (rc = dmalloc(ctx, &ctx->hbuf[1], N)) || (rc = dmalloc(ctx, &ctx->d_levels_esc, (size_t)N + 2)) ||
      (rc = dmalloc(ctx, &a.rcode, (size_t)N + 16)) ||
      (rc = dmalloc(ctx, &a.planes, (size_t)4 * H * M * ((W + 31) / 32))) || (rc = dmalloc(ctx, &a.dmask, (size_t)N + 16)) ||
      (rc = dmalloc(ctx, &a.order, (size_t)N + kFChunk)) || (rc = dmalloc(ctx, &a.ppos, (size_t)N + kFChunk)) ||
      (rc = dmalloc(ctx, &a.cdir, N)) || (rc = dmalloc(ctx, &a.hx, (size_t)N + kFChunk)) ||
      (rc = dmalloc(ctx, &a.fc, (size_t)N + 1)) ||
      (rc = dmalloc(ctx, &a.cbound, ((size_t)N / kChunkRoots + 2) * kCBS)) ||
      (rc = dmalloc(ctx, &a.Aq, (size_t)N + kFChunk)) || (rc = dmalloc(ctx, &a.hq, (size_t)N + kFChunk)) ||
      (rc = dmalloc(ctx, &a.levels, (size_t)N + 2)) ||
      (rc = dmalloc(ctx, &a.pdm, N)) || (rc = dmalloc(ctx, &a.part, 4096)) ||
      (rc = dmalloc(ctx, &a.bins, 3 * 4096)) || (rc = dmalloc(ctx, &a.ctl, 1)) ||
      (rc = dmalloc(ctx, &ctx->d_diag, ctx->diag_cap)))
    return bail(rc);
  a.h = ctx->hbuf[0];
  a.hout = ctx->hbuf[1];
  a.W32 = (W + 31) / 32;
  a.dmask_valid = 1;
  a.kdt = ctx->d_kdt;
  a.mexp = ctx->d_mexp;
  a.ftab = ctx->d_lut;
  a.ftab2 = ctx->d_lut2;
  a.cb_stride = N / kChunkRoots + 2;
  a.cb_cap = (uint32_t)std::min<uint64_t>(0xFFFFFFFFull, ((uint64_t)N / kChunkRoots + 2) * kCBS);
  a.fbins = a.levels;  // the global path's level array: unused by the tile path's steps
  a.diag = ctx->d_diag;
#define CUB(call)                          \
  do {                                     \
    if ((call) != cudaSuccess) {           \
      fail(ctx, LEMGPU_ECUDA, "%s", #call); \
      return bail(LEMGPU_ECUDA);           \
    }                                      \
  } while (0)
  CUB(cudaMemcpy(ctx->d_kdt, kdt.data(), M * sizeof(double), cudaMemcpyHostToDevice));
  CUB(cudaMemcpy(ctx->d_mexp, mexp.data(), M * sizeof(double), cudaMemcpyHostToDevice));
  CUB(cudaMemcpy(ctx->d_lut, lut.data(), lut.size() * sizeof(double), cudaMemcpyHostToDevice));
  {
    // slope = 1.0 + (F * n) * pow(diff, n - 1) = 1.0 + F for n = 1 (erosion.cpp:26; pow(x, 0) == 1);
    // its correctly rounded reciprocal (host IEEE division) for the device's
    // Markstein-corrected quotients (newton_n1_tab, k_tiles.cuh)
    std::vector<double> lut2(2 * lut.size());
    a.tab_ok = 1;
    for (size_t i = 0; i < lut.size(); ++i) {
      if (!(lut[i] < 0x1p500)) a.tab_ok = 0;
      lut2[2 * i] = lut[i];
      lut2[2 * i + 1] = 1.0 / (1.0 + lut[i]);
    }
    CUB(cudaMemcpy(ctx->d_lut2, lut2.data(), lut2.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  CUB(cudaMemset(ctx->hbuf[0], 0, (size_t)N * sizeof(double)));
  CUB(cudaMemset(ctx->hbuf[1], 0, (size_t)N * sizeof(double)));
  CUB(cudaMemset(a.rcode, 0, (size_t)N + 16));
  CUB(cudaMemset(a.dmask, 0, (size_t)N + 16));
  CUB(cudaMemset(a.bins, 0, 3 * 4096 * sizeof(uint32_t)));
  Ctl c0{};
  c0.err_cell = LEMGPU_NOFLOW;
  c0.t_k1_begin = ~0ull;
  c0.t_k1_end = 0;
  c0.t_t_begin = ~0ull;
  c0.t_t_end = 0;
  c0.t_mfd_begin = ~0ull;
  CUB(cudaMemcpy(a.ctl, &c0, sizeof c0, cudaMemcpyHostToDevice));

  // launch geometry
  int occ = 0;
  CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_expand, kTPB, 0));
  ctx->scan_grid = (occ > 0 ? occ : 1) * nsm;
  if (ctx->scan_grid > 4096) ctx->scan_grid = 4096;  // part/bins capacity
  ctx->use_tiles = 1;
  ctx->esc_grid = nsm;
  if (o.esc_grid) ctx->esc_grid = (int)o.esc_grid;
  if (ctx->esc_grid < 1 || ctx->esc_grid > ctx->scan_grid) ctx->esc_grid = ctx->scan_grid;
  if (o.global_path) ctx->use_tiles = 0;
  ctx->opt_global = o.global_path != 0;
  ctx->opt_mfd_levels = o.mfd_levels != 0;
  a.force_escape = 0;
  a.force_escape = o.force_escape;
  a.phclk = o.phase_clocks ? 1 : 0;
  {
    const void* ft = tiles_fn(a);
    CUB(cudaFuncSetAttribute(ft, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiles_smem(a)));
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ft, kTTPB, tiles_smem(a)));
    const uint32_t ntiles = ((W + kTX - 1) / kTX) * ((H * M + kTY - 1) / kTY);
    uint32_t tg = (uint32_t)(occ > 0 ? occ : 1) * (uint32_t)nsm;
    if (o.tile_grid) tg = o.tile_grid;  // testing: few CTAs, many tiles each
    if (tg < 1) tg = 1;
    ctx->tile_grid = (int)(tg < ntiles ? tg : ntiles);
    // MFD routing: the instantiation may differ (tiles_fn)
    StepArgs am = a;
    am.mfd_A = reinterpret_cast<double*>(16);  // only selects the instantiation
    const void* fm = tiles_fn(am);
    CUB(cudaFuncSetAttribute(fm, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tiles_smem(am)));
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fm, kTTPB, tiles_smem(am)));
    tg = o.tile_grid ? o.tile_grid : (uint32_t)(occ > 0 ? occ : 1) * (uint32_t)nsm;
    ctx->tile_grid_mfd = (int)(tg < ntiles ? tg : ntiles);
  }
  a.eager = 0;
  a.force_deep = o.force_deep ? 1 : 0;
  if (o.no_esc_small) ctx->esc_small = false;
  ctx->esc_small_grid = kEscSmallPerSM * nsm;
  {  // pipelined receivers / tiles for tall rasters: 24 bands (measured best at 10000^2: 2.127 -> 2.061 ms)
    const uint32_t nty = (H * M + kTY - 1) / kTY;
    ctx->pipe = nty >= 256 ? 24 : 0;  // (5000^2: 157 tile rows, banding costs more than it overlaps)
  }
  if (o.pipe) ctx->pipe = o.pipe < 0 ? 0 : o.pipe;
  ctx->pipe_tile_grid = 4 * nsm;
  if (o.pipe_unchained) ctx->pipe_chain = 0;
  if (o.pipe_tile_grid) ctx->pipe_tile_grid = (int)o.pipe_tile_grid;
  if (o.esc_small_grid) ctx->esc_small_grid = (int)o.esc_small_grid;
  ctx->bands = (int)o.host_bands;
  ctx->opt_patch_cap = o.patch_cap;
  ctx->host_profile = o.host_profile != 0;
  if (ctx->bands <= 0) {  // measured on 10000^2 (tools/e2e_probe.py): 32 bands of 25 MB beat 16 and 64
    const uint64_t nbands = N64 * 8 / (25ull << 20);
    ctx->bands = (int)std::min<uint64_t>(32, nbands < 4 ? 1 : nbands);
  }
  if (a.force_deep) ctx->esc_small = false;  // testing the deep sweeps of the escape path
  // k_esc_forest for exact-area steps (integer drainage counts): auto / always / never
  a.esc_forest = !a.lut_exact || o.esc_forest < 0 || a.force_deep ? 0 : o.esc_forest > 0 ? 2 : 1;
  a.no_narrow = o.no_narrow ? 1 : 0;  // testing: grid-wide sweeps for every level
  a.eager = o.eager ? 1 : 0;
  for (const void* f : {(const void*)k_esc_small<0>, (const void*)k_esc_small<1>, (const void*)k_esc_small<2>})
    CUB(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kEscSmallSmemBytes));
  for (const void* f : {(const void*)k_deep_coop<0>, (const void*)k_deep_coop<1>, (const void*)k_deep_coop<2>})
    CUB(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDeepSmemBytes));
  for (const void* f : {(const void*)k_esc_forest<0>, (const void*)k_esc_forest<1>, (const void*)k_esc_forest<2>})
    CUB(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kForestSmemBytes));
  {
    int occf = 0;
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, forest_fn(a.nkind), kFTPB, kForestSmemBytes));
    ctx->forest_grid = (occf > 0 ? occf : 1) * nsm;
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, k_mfd_levels, kTPB, 0));
    ctx->mfd_grid = std::min(ctx->scan_grid, (occf > 0 ? occf : 1) * nsm);
    CUB(cudaFuncSetAttribute((const void*)k_mfd_tiles, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kMfdTileSmemBytes));
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occf, k_mfd_tiles, kMTPB, kMfdTileSmemBytes));
    ctx->mfd_tiles_grid = (occf > 0 ? occf : 1) * nsm;
  }
  {
    const void* fdc = a.nkind == 1 ? (const void*)k_deep_coop<1> : a.nkind == 2 ? (const void*)k_deep_coop<2>
                                                                              : (const void*)k_deep_coop<0>;
    int occd = 0;
    CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occd, fdc, kDeepTPB, kDeepSmemBytes));
    ctx->deep_coop_grid = (occd > 0 ? occd : 1) * nsm;
  }
  const void* fchunks = a.nkind == 1 ? (const void*)k_chunks<1> : a.nkind == 2 ? (const void*)k_chunks<2> : (const void*)k_chunks<0>;
  CUB(cudaFuncSetAttribute(fchunks, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kChunksSmemBytes));
  CUB(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fchunks, kChunkTPB, kChunksSmemBytes));
  ctx->chunk_grid = (occ > 0 ? occ : 1) * nsm;
  ctx->deep_grid = 8 * nsm;
  a.scan_grid = ctx->scan_grid;
  // TMA descriptors of both elevation buffers: rows of W doubles; boxes = one
  // k_recv_donor halo tile and one k_tiles window.  The row pitch must be a
  // multiple of 16 bytes (even W); otherwise the kernels stage h with plain loads.
  a.use_tma = 0;
  if ((W % 2) == 0 && !o.no_tma) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess && fn) {
      auto encode = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill)>(fn);
      const cuuint64_t gdim[2] = {W, (cuuint64_t)H * M};
      const cuuint64_t gstride[1] = {(cuuint64_t)W * sizeof(double)};
      const cuuint32_t box_r[2] = {kBX + 4, kBY + 4};
      const cuuint32_t box_t[2] = {kWP, kDH};
      const cuuint32_t estr[2] = {1, 1};
      bool ok = true;
      for (int p = 0; p < 2; ++p) {
        ok = ok && encode(&ctx->hmap[p], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ctx->hbuf[p], gdim, gstride, box_r, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
        ok = ok && encode(&ctx->tmap[p], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, ctx->hbuf[p], gdim, gstride, box_t, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
      }
      a.use_tma = ok ? 1 : 0;
    }
  }
  for (uint32_t p = 0; p < 2; ++p) {
    const int rcg = build_graph(ctx, p);
    if (rcg) return bail(rcg);
  }
  *out = ctx;
  return LEMGPU_OK;
#undef CUB
}

// Eager (profiling) mode: the same kernels launched one by one; the loop
// conditions come back through the control block, one small D2H per level.
// ncu cannot profile kernel nodes of graphs with conditional nodes.
int run_levels_eager(lemgpu_ctx* ctx, const StepArgs& a) {
  cudaStream_t st = ctx->stream;
  const int nk = a.nkind;
  const size_t co = offsetof(Ctl, cond);
  char* cbase = reinterpret_cast<char*>(a.ctl) + co;
  unsigned cond[3] = {a.tiles ? 0u : 1u, 0, 0};  // the tile path expands inside k_esc_bfs
  while (cond[0]) {
    k_expand<<<a.scan_grid, kTPB, 0, st>>>(a);
    CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
    CU(ctx, cudaStreamSynchronize(st));
  }
  if (nk == 1)
    k_chunks<1><<<ctx->chunk_grid, kChunkTPB, kChunksSmemBytes, st>>>(a);
  else if (nk == 2)
    k_chunks<2><<<ctx->chunk_grid, kChunkTPB, kChunksSmemBytes, st>>>(a);
  else
    k_chunks<0><<<ctx->chunk_grid, kChunkTPB, kChunksSmemBytes, st>>>(a);
  if (a.tiles) {
    void* dargs[] = {const_cast<StepArgs*>(&a)};
    const void* fdc = nk == 1 ? (const void*)k_deep_coop<1> : nk == 2 ? (const void*)k_deep_coop<2> : (const void*)k_deep_coop<0>;
    CU(ctx, cudaLaunchCooperativeKernel(fdc, dim3(ctx->deep_coop_grid), dim3(kDeepTPB), dargs, kDeepSmemBytes, st));
    return LEMGPU_OK;
  }
  k_deep_prep<<<ctx->deep_grid, kTPB, 0, st>>>(a);
  CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
  CU(ctx, cudaStreamSynchronize(st));
  while (cond[1]) {
    k_deep_accum<<<ctx->deep_grid, kTPB, 0, st>>>(a);
    CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
    CU(ctx, cudaStreamSynchronize(st));
  }
  while (cond[2]) {
    if (nk == 1)
      k_deep_erode<1><<<ctx->deep_grid, kTPB, 0, st>>>(a);
    else if (nk == 2)
      k_deep_erode<2><<<ctx->deep_grid, kTPB, 0, st>>>(a);
    else
      k_deep_erode<0><<<ctx->deep_grid, kTPB, 0, st>>>(a);
    CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
    CU(ctx, cudaStreamSynchronize(st));
  }
  k_deep_final<<<ctx->deep_grid, kTPB, 0, st>>>(a);
  return LEMGPU_OK;
}

void set_eager_conds(const StepArgs& a, cudaStream_t st) {
  static const unsigned init[3] = {1, 0, 0};
  char* cbase = reinterpret_cast<char*>(a.ctl) + offsetof(Ctl, cond);
  cudaMemcpyAsync(cbase, init, sizeof init, cudaMemcpyHostToDevice, st);
  cudaStreamSynchronize(st);  // init is host memory
}

// The tile path after k_tiles, launched eagerly: k_esc_small, the cooperative
// level expansion of the escaped trees, their physics.
int enqueue_escape_eager(lemgpu_ctx* ctx, StepArgs& a, cudaStream_t st) {
  if (ctx->esc_small) {
    if (a.nkind == 1)
      k_esc_small<1><<<ctx->esc_small_grid, kTPB, kEscSmallSmemBytes, st>>>(a);
    else if (a.nkind == 2)
      k_esc_small<2><<<ctx->esc_small_grid, kTPB, kEscSmallSmemBytes, st>>>(a);
    else
      k_esc_small<0><<<ctx->esc_small_grid, kTPB, kEscSmallSmemBytes, st>>>(a);
  }
  void* eargs[] = {&a};
  if (a.esc_forest)
    CU(ctx, cudaLaunchCooperativeKernel(forest_fn(a.nkind), dim3(ctx->forest_grid), dim3(kFTPB), eargs,
                                        kForestSmemBytes, st));
  CU(ctx, cudaLaunchCooperativeKernel((const void*)k_esc_bfs, dim3(a.scan_grid), dim3(kTPB), eargs, 0, st));
  return run_levels_eager(ctx, a);
}

int enqueue_step_eager(lemgpu_ctx* ctx, uint32_t p) {
  StepArgs a = step_args(ctx, p);
  a.eager = 1;
  cudaStream_t st = ctx->stream;
  set_eager_conds(a, st);
  enqueue_stats_pass(ctx, a, st);
  if (ctx->use_tiles && a.mfd_A) {  // the MFD tile passes, the loop condition through the control block
    StepArgs a0 = a;
    a0.mfd_all = 1;
    a.mfd_all = 0;
    k_mfd_tiles<<<ctx->mfd_tiles_grid, kMTPB, kMfdTileSmemBytes, st>>>(a0);
    k_mfd_tiles<<<ctx->mfd_tiles_grid, kMTPB, kMfdTileSmemBytes, st>>>(a);
    unsigned cond[4];
    const char* cbase = reinterpret_cast<const char*>(a.ctl) + offsetof(Ctl, cond);
    for (;;) {
      CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
      CU(ctx, cudaStreamSynchronize(st));
      if (!cond[3]) break;
      k_mfd_tail<<<ctx->scan_grid, kTPB, 0, st>>>(a);
    }
  }
  if (ctx->use_tiles) {
    const dim3 g1((a.W + kBX - 1) / kBX, (a.Htot + kBY - 1) / kBY);
    {
      void* rargs[] = {&a, &ctx->hmap[p]};
      CU(ctx, cudaLaunchKernel(recv_fn(a), g1, dim3(kTPB), rargs, 0, st));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(a.mfd_A ? ctx->tile_grid_mfd : ctx->tile_grid);
    cfg.blockDim = dim3(kTTPB);
    cfg.dynamicSmemBytes = tiles_smem(a);
    cfg.stream = st;
    void* args[] = {&a, &ctx->tmap[p]};
    CU(ctx, cudaLaunchKernelExC(&cfg, tiles_fn(a), args));
    const int rc = enqueue_escape_eager(ctx, a, st);
    if (rc) return rc;
  } else {
    const dim3 g1((a.W + kBX - 1) / kBX, (a.Htot + kBY - 1) / kBY);
    if (a.mfd_A) {
      k_mfd_graph<<<ctx->deep_grid, kTPB, 0, st>>>(a);
      void* margs[] = {&a};
      CU(ctx, cudaLaunchCooperativeKernel((const void*)k_mfd_levels, dim3(ctx->mfd_grid), dim3(kTPB), margs, 0, st));
    }
    if (a.conn == 8)
      k_recv_donor<8><<<g1, kTPB, 0, st>>>(a, ctx->hmap[p]);
    else
      k_recv_donor<4><<<g1, kTPB, 0, st>>>(a, ctx->hmap[p]);
    k_l0_count<<<ctx->scan_grid, kTPB, 0, st>>>(a);
    k_l0_write<<<ctx->scan_grid, kTPB, 0, st>>>(a);
    const int rc = run_levels_eager(ctx, a);
    if (rc) return rc;
  }
  if (const int rcs = enqueue_stats(ctx, a, st)) return rcs;
  k_finalize<<<1, 32, 0, st>>>(a);
  CU(ctx, cudaGetLastError());
  return LEMGPU_OK;
}

// One step on a HOST raster with the copies overlapped: the raster is cut into
// bands of tile rows; band b goes up on one stream while the compute stream
// runs k_recv on band b-1 and k_tiles on band b-2, and a third stream copies
// band b-3's new elevations down as soon as no tile tree can still write them
// (the tiles of the band below have run).  The escaped trees are finished
// after the last band; their cells' final values are gathered and patched
// into the host raster.  A PCIe-bound step then costs about one raster copy
// instead of two.  Requires pinned host memory (else the copies would not
// overlap) and the tile path.
int step_host_banded(lemgpu_ctx* ctx, double* elev, lemgpu_diag* diag) {
  const auto tb0 = std::chrono::steady_clock::now();
  if (ctx->pending) {
    const int rc0 = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc0) return rc0;
  }
  const uint32_t p = ctx->cur;
  StepArgs a = step_args(ctx, p);
  a.eager = 1;
  cudaStream_t st = ctx->stream;
  set_eager_conds(a, st);
  if (!ctx->s_h2d) {
    CU(ctx, cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
    CU(ctx, cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
    // room for the escaped trees of a typical step (a few % of the cells);
    // more than that and the whole raster is copied down again
    ctx->patch_cap = std::max<uint32_t>(1u << 20, a.N / 16);
    if (ctx->opt_patch_cap) ctx->patch_cap = ctx->opt_patch_cap;  // testing
    ctx->patch_cap = (ctx->patch_cap + 63u) & ~63u;  // the vals after the cells stay 8-byte aligned
    CU(ctx, cudaHostAlloc(&ctx->h_patch, 16 + (size_t)ctx->patch_cap * 12, cudaHostAllocMapped));
  }
  const uint32_t W = a.W, Ht = a.Htot;
  const uint32_t ntx = (W + kTX - 1) / kTX, nty = (Ht + kTY - 1) / kTY;
  // tile rows per band: bands start on k_recv row blocks too
  constexpr uint32_t kRq = (uint32_t)(kBY / std::gcd(kBY, kTY));  // lcm(kBY, kTY) / kTY
  const uint32_t R = ((nty + (uint32_t)ctx->bands - 1) / (uint32_t)ctx->bands + kRq - 1) / kRq * kRq;
  const uint32_t nb = (nty + R - 1) / R;
  while (ctx->band_ev.size() < 3 * (size_t)nb + 2) {
    cudaEvent_t e;  // timed only for host_profile's band timeline
    CU(ctx, cudaEventCreateWithFlags(&e, ctx->host_profile ? cudaEventDefault : cudaEventDisableTiming));
    ctx->band_ev.push_back(e);
  }
  cudaEvent_t* eh = ctx->band_ev.data();  // band b uploaded
  cudaEvent_t* et = eh + nb;              // band b's tiles done
  cudaEvent_t e0 = eh[2 * nb];
  cudaEvent_t* ed = eh + 2 * nb + 1;      // band b's copies down done
  cudaEvent_t eg = eh[3 * nb + 1];        // the escaped cells' values gathered
  cudaEvent_t* tev = nullptr;
  if (ctx->timing) {  // step events as enqueue_step records them
    while (ctx->ev.size() < 2) {
      cudaEvent_t e;
      CU(ctx, cudaEventCreate(&e));
      ctx->ev.push_back(e);
    }
    tev = &ctx->ev[0];
    CU(ctx, cudaEventRecord(tev[0], st));
  }
  CU(ctx, cudaEventRecord(e0, st));  // earlier work on the context stream
  CU(ctx, cudaStreamWaitEvent(ctx->s_h2d, e0, 0));
  CU(ctx, cudaStreamWaitEvent(ctx->s_d2h, e0, 0));
  auto rows = [&](uint32_t b, uint32_t& r0, uint32_t& r1) {
    r0 = b * R * (uint32_t)kTY;
    r1 = std::min((b + 1) * R * (uint32_t)kTY, Ht);
  };
  // band b goes up with the first kBY + 2 rows of band b+1: k_recv of band b
  // also computes the codes of band b+1's first row block (k_tiles of band b
  // reads them, kLY + 1 rows deep), so k_recv(b) and k_tiles(b) wait only for
  // band b's own upload, and band b's copy down trails its upload by one band
  constexpr uint32_t kHead = kBY + 2;
  auto up = [&](uint32_t r0, uint32_t r1) -> int {
    if (r1 > r0)
      CU(ctx, cudaMemcpyAsync(ctx->hbuf[p] + (size_t)r0 * W, elev + (size_t)r0 * W, (size_t)(r1 - r0) * W * sizeof(double),
                              cudaMemcpyHostToDevice, ctx->s_h2d));
    return LEMGPU_OK;
  };
  uint32_t up_to = 0;  // rows [0, up_to) are on their way up
  for (uint32_t b = 0; b < nb; ++b) {
    uint32_t r0, r1;
    rows(b, r0, r1);
    const uint32_t want = b + 1 < nb ? std::min(r1 + kHead, Ht) : Ht;
    int rcu;
    if ((rcu = up(std::max(up_to, r0), want))) return rcu;
    up_to = std::max(up_to, want);
    CU(ctx, cudaEventRecord(eh[b], ctx->s_h2d));
  }
  auto recv = [&](uint32_t b) -> int {  // row blocks [r0 (+ kBY after band 0), r1 + kBY)
    CU(ctx, cudaStreamWaitEvent(st, eh[b], 0));
    uint32_t r0, r1;
    rows(b, r0, r1);
    const uint32_t q0 = b ? r0 + (uint32_t)kBY : r0, q1 = std::min(r1 + (uint32_t)kBY, Ht);
    if (q1 <= q0) return LEMGPU_OK;
    StepArgs ab = a;
    ab.by0 = q0 / kBY;
    const dim3 g((W + kBX - 1) / kBX, (q1 - q0 + kBY - 1) / kBY);
    void* rargs[] = {&ab, &ctx->hmap[p]};
    CU(ctx, cudaLaunchKernel(recv_fn(a), g, dim3(kTPB), rargs, 0, st));
    return LEMGPU_OK;
  };
  int rc;
  for (uint32_t b = 0; b < nb; ++b) {
    if ((rc = recv(b))) return rc;
    StepArgs ab = a;
    ab.t_lo = b * R * ntx;
    ab.t_hi = std::min((b + 1) * R, nty) * ntx;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(std::min<uint32_t>((uint32_t)ctx->tile_grid, ab.t_hi - ab.t_lo));
    cfg.blockDim = dim3(kTTPB);
    cfg.dynamicSmemBytes = tiles_smem(a);
    cfg.stream = st;
    void* args[] = {&ab, &ctx->tmap[p]};
    CU(ctx, cudaLaunchKernelExC(&cfg, tiles_fn(a), args));
    CU(ctx, cudaEventRecord(et[b], st));
    // once band b's tiles have run, band b is final (escaped trees aside)
    // except its last kHalo rows, which trees of band b+1 may still reach,
    // and band b-1's last kHalo rows are final
    auto down = [&](uint32_t r0, uint32_t r1) -> int {
      if (r1 > r0)
        CU(ctx, cudaMemcpyAsync(elev + (size_t)r0 * W, ctx->hbuf[p ^ 1u] + (size_t)r0 * W,
                                (size_t)(r1 - r0) * W * sizeof(double), cudaMemcpyDeviceToHost, ctx->s_d2h));
      return LEMGPU_OK;
    };
    uint32_t r0, r1;
    rows(b, r0, r1);
    CU(ctx, cudaStreamWaitEvent(ctx->s_d2h, et[b], 0));
    if (b >= 1) {
      uint32_t q0, q1;
      rows(b - 1, q0, q1);
      if ((rc = down(q1 - std::min<uint32_t>(kHalo, q1 - q0), q1))) return rc;
    }
    const uint32_t body_end = b + 1 < nb ? r1 - std::min<uint32_t>(kHalo, r1 - r0) : r1;
    if ((rc = down(r0, body_end))) return rc;
    CU(ctx, cudaEventRecord(ed[b], ctx->s_d2h));
  }
  if ((rc = enqueue_escape_eager(ctx, a, st))) return rc;
  {
    char* hp = nullptr;
    CU(ctx, cudaHostGetDevicePointer(reinterpret_cast<void**>(&hp), ctx->h_patch, 0));
    k_esc_gather<<<ctx->scan_grid, kTPB, 0, st>>>(a, reinterpret_cast<uint32_t*>(hp + 16),
                                                 reinterpret_cast<double*>(hp + 16 + (size_t)ctx->patch_cap * 4),
                                                 reinterpret_cast<uint32_t*>(hp), ctx->patch_cap);
    CU(ctx, cudaEventRecord(eg, st));
  }
  enqueue_stats_pass(ctx, a, st);  // the input buffer is complete and unchanged by now
  if ((rc = enqueue_stats(ctx, a, st))) return rc;
  k_finalize<<<1, 32, 0, st>>>(a);
  CU(ctx, cudaGetLastError());
  if (tev) CU(ctx, cudaEventRecord(tev[1], st));
  ctx->mfd_src = p;
  ctx->cur = p ^ 1u;
  ++ctx->pending;
  ++ctx->st_steps;
  ctx->have_graph = true;
  using clk = std::chrono::steady_clock;
  const auto tq0 = clk::now();
  // the escaped cells' values are gathered while the last bands are still on
  // their way down: patch the cells of the bands already down now (rows above
  // the first band whose copies are pending, less its predecessor's last
  // kHalo rows, which travel with it), the rest after the copies
  const uint32_t* pcells = ctx->h_patch + 4;
  const double* pvals = reinterpret_cast<const double*>(reinterpret_cast<const char*>(ctx->h_patch) + 16 +
                                                        (size_t)ctx->patch_cap * 4);
  auto patch = [&](uint32_t n, uint32_t row_lo, uint32_t row_hi) {
    // random writes into the raster: latency-bound, spread over a few threads
    const uint32_t nt = n < 65536u ? 1u : std::min(8u, std::max(1u, std::thread::hardware_concurrency()));
    const uint64_t lo = (uint64_t)row_lo * W, hi = (uint64_t)row_hi * W;
    auto part = [&](uint32_t t) {
      const uint32_t i0 = (uint32_t)((uint64_t)n * t / nt), i1 = (uint32_t)((uint64_t)n * (t + 1) / nt);
      for (uint32_t i = i0; i < i1; ++i)
        if (pcells[i] >= lo && pcells[i] < hi) elev[pcells[i]] = pvals[i];
    };
    std::vector<std::thread> pool;
    for (uint32_t t = 1; t < nt; ++t) pool.emplace_back(part, t);
    part(0);
    for (auto& th : pool) th.join();
  };
  uint32_t early_rows = 0;
  CU(ctx, cudaEventSynchronize(eg));
  const uint32_t n_early = *reinterpret_cast<volatile uint32_t*>(ctx->h_patch);
  if (n_early <= ctx->patch_cap) {
    uint32_t bd = 0;  // first band whose copies down are pending
    while (bd < nb && cudaEventQuery(ed[bd]) == cudaSuccess) ++bd;
    if (bd == nb) {
      early_rows = Ht;
    } else if (bd > 0) {
      uint32_t r0, r1;
      rows(bd, r0, r1);
      early_rows = r0 > kHalo ? r0 - kHalo : 0u;
    }
    if (early_rows) patch(n_early, 0, early_rows);
  }
  const auto tqe = clk::now();
  CU(ctx, cudaStreamSynchronize(ctx->s_d2h));
  const auto tq1 = clk::now();
  lemgpu_diag d{};
  uint32_t cnt = 0;
  rc = lemgpu_sync(ctx, &d, 1, &cnt);
  const auto tq2 = clk::now();
  if (diag) *diag = d;
  if (rc) {  // the failed step leaves the elevation as it was: its input buffer
    if (rc != LEMGPU_ECUDA)
      cudaMemcpy(elev, ctx->hbuf[ctx->cur], (size_t)a.N * sizeof(double), cudaMemcpyDeviceToHost);
    return rc;
  }
  // patch the cells of the escaped trees (those of the bands that were still
  // on their way down)
  const uint32_t n = *reinterpret_cast<volatile uint32_t*>(ctx->h_patch);
  if (n > ctx->patch_cap) {
    CU(ctx, cudaMemcpy(elev, ctx->hbuf[ctx->cur], (size_t)a.N * sizeof(double), cudaMemcpyDeviceToHost));
  } else if (early_rows < Ht) {
    patch(n, early_rows, Ht);
  }
  if (ctx->host_profile) {
    const auto tq3 = clk::now();
    auto ms = [](clk::duration x) { return std::chrono::duration<double, std::milli>(x).count(); };
    std::fprintf(stderr, "step_host_banded: enqueue %.3f ms, gather + early patch (rows < %u) %.3f ms, then d2h done "
                 "%.3f ms, sync %.3f ms, patch of %u cells %.3f ms\n",
                 ms(tq0 - tb0), early_rows, ms(tqe - tq0), ms(tq1 - tqe), ms(tq2 - tq1), n, ms(tq3 - tq2));
    // device timeline from e0 (ms): band uploaded / tiles done / copies down done, and the gather
    auto el = [&](cudaEvent_t e) {
      float t = -1.f;
      cudaEventElapsedTime(&t, e0, e);
      return t;
    };
    std::fprintf(stderr, "  bands %u:", nb);
    for (uint32_t b = 0; b < nb; ++b) std::fprintf(stderr, " [%.2f %.2f %.2f]", el(eh[b]), el(et[b]), el(ed[b]));
    std::fprintf(stderr, " gather %.2f\n", el(eg));
  }
  return LEMGPU_OK;
}

int enqueue_step(lemgpu_ctx* ctx) {
  if (ctx->pending >= ctx->diag_cap) return fail(ctx, LEMGPU_EOTHER, "too many steps pending");
  cudaEvent_t* ev = nullptr;
  if (ctx->timing) {
    while (ctx->ev.size() < 2 * (size_t)(ctx->pending + 1)) {
      cudaEvent_t e;
      CU(ctx, cudaEventCreate(&e));
      ctx->ev.push_back(e);
    }
    ev = &ctx->ev[2 * ctx->pending];
    CU(ctx, cudaEventRecord(ev[0], ctx->stream));
  }
  const uint32_t p = ctx->cur;
  // a snapshot still copying the buffer this step writes: wait for it (on the device)
  if (ctx->snap_pending && ctx->snap_buf == (p ^ 1u)) CU(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_snap_done, 0));
  if (ctx->a.dbg_level) {  // debug capture: every step starts from "not finished by the tile pass"
    CU(ctx, cudaMemsetAsync(ctx->a.dbg_level, 0xFF, ctx->a.N, ctx->stream));
    CU(ctx, cudaMemsetAsync(ctx->a.dbg_A, 0xFF, (size_t)ctx->a.N * sizeof(double), ctx->stream));
  }
  if (ctx->a.eager) {
    const int rc = enqueue_step_eager(ctx, p);
    if (rc) return rc;
  } else {
    CU(ctx, cudaGraphLaunch(ctx->st_interval > 1 && stats_due(ctx) ? ctx->st_exec[p] : ctx->exec[p], ctx->stream));
  }
  ++ctx->st_steps;
  if (ev) CU(ctx, cudaEventRecord(ev[1], ctx->stream));
  ctx->mfd_src = p;
  ctx->cur = p ^ 1u;
  ++ctx->pending;
  ctx->have_graph = true;
  return LEMGPU_OK;
}

}  // namespace

extern "C" {

uint32_t lemgpu_abi_version(void) { return LEMGPU_ABI_VERSION; }

int lemgpu_create(int device, uint32_t width, uint32_t height, const lemgpu_params* params,
                  lemgpu_ctx** out) {
  return create_impl(device, width, height, 1, params, nullptr, nullptr, out);
}

int lemgpu_create_ensemble(int device, uint32_t width, uint32_t height, uint32_t members,
                           const lemgpu_params* params, const lemgpu_member* per_member,
                           lemgpu_ctx** out) {
  return create_impl(device, width, height, members, params, per_member, nullptr, out);
}

int lemgpu_create_ex(int device, uint32_t width, uint32_t height, uint32_t members, const lemgpu_params* params,
                     const lemgpu_member* per_member, const lemgpu_options* options, lemgpu_ctx** out) {
  return create_impl(device, width, height, members, params, per_member, options, out);
}

void lemgpu_destroy(lemgpu_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  StepArgs& a = ctx->a;
  void* ptrs[] = {ctx->d_kdt, ctx->d_mexp, ctx->d_lut, ctx->d_lut2, ctx->hbuf[0], ctx->hbuf[1], ctx->d_levels_esc, a.rcode, a.planes,  a.dmask, a.order,
                  a.ppos,     a.cdir,      a.fc,        a.cbound,     a.Aq,  a.hq,     a.levels, a.pdm, a.part, a.bins,
                  a.ctl,      ctx->d_diag, a.hx};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (a.dbg_level) cudaFree(a.dbg_level);
  if (a.dbg_A) cudaFree(a.dbg_A);
  for (void* q : {(void*)a.mfd_A, (void*)a.mfd_wsum, (void*)a.mfd_lm, (void*)a.mfd_rem, (void*)a.mfd_ord,
                  (void*)a.mfd_lv, (void*)a.mfd_lev, (void*)a.mfd_wl, (void*)a.mfd_stamp})
    if (q) cudaFree(q);
  if (ctx->st_local) cudaFree(ctx->st_local);
  if (ctx->st_part) cudaFree(ctx->st_part);
  if (ctx->comm) nccl().commDestroy(ctx->comm);
  for (cudaEvent_t e : ctx->ev) cudaEventDestroy(e);
  destroy_graphs(ctx);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
  if (ctx->s_snap) cudaStreamDestroy(ctx->s_snap);
  if (ctx->ev_snap_step) cudaEventDestroy(ctx->ev_snap_step);
  if (ctx->ev_snap_done) cudaEventDestroy(ctx->ev_snap_done);
  if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
  for (cudaEvent_t e : ctx->band_ev) cudaEventDestroy(e);
  if (ctx->h_patch) cudaFreeHost(ctx->h_patch);
  delete ctx;
}

const char* lemgpu_error_message(const lemgpu_ctx* ctx) {
  return ctx ? ctx->msg.c_str() : g_create_error.c_str();
}
uint32_t lemgpu_error_cell(const lemgpu_ctx* ctx) { return ctx ? ctx->err_cell : LEMGPU_NOFLOW; }
uint64_t lemgpu_num_cells(const lemgpu_ctx* ctx) { return ctx ? ctx->a.N : 0; }
void* lemgpu_stream(lemgpu_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }
uint32_t lemgpu_kernels_per_step(const lemgpu_ctx* ctx) {
  if (!ctx || !ctx->graph[0]) return 0;
  size_t n = 0;
  if (cudaGraphGetNodes(ctx->graph[0], nullptr, &n) != cudaSuccess) return 0;
  std::vector<cudaGraphNode_t> nodes(n);
  if (cudaGraphGetNodes(ctx->graph[0], nodes.data(), &n) != cudaSuccess) return 0;
  uint32_t k = 0;
  for (cudaGraphNode_t v : nodes) {
    cudaGraphNodeType t;
    if (cudaGraphNodeGetType(v, &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
  }
  return k;
}

uint32_t lemgpu_pipeline_bands(const lemgpu_ctx* ctx) { return ctx ? ctx->pipe_bands : 0; }

int lemgpu_device_bytes(const lemgpu_ctx* ctx, uint64_t* bytes) {
  if (!ctx || !bytes) return LEMGPU_ECONFIG;
  *bytes = ctx->device_bytes;
  return LEMGPU_OK;
}

int lemgpu_upload_elev(lemgpu_ctx* ctx, const double* host) {
  if (!ctx || !host) return fail(ctx, LEMGPU_ECONFIG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  const StepArgs& a = ctx->a;
  double* hc = ctx->hbuf[ctx->cur];
  CU(ctx, cudaMemcpyAsync(hc, host, (size_t)a.N * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  // reject non-finite input (scheduler.cpp:474-477); reuse fc[N] as scratch
  uint32_t* bad = a.fc + a.N;
  CU(ctx, cudaMemsetAsync(bad, 0xFF, sizeof(uint32_t), ctx->stream));
  k_check_finite<<<1184, kTPB, 0, ctx->stream>>>(hc, a.N, bad);
  uint32_t first = 0;
  CU(ctx, cudaMemcpyAsync(&first, bad, sizeof first, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (first != LEMGPU_NOFLOW)
    return fail(ctx, LEMGPU_ECONFIG, "input terrain has a non-finite value at cell %u", first);
  ctx->have_graph = false;
  return LEMGPU_OK;
}

int lemgpu_download_elev(lemgpu_ctx* ctx, double* host) {
  if (!ctx || !host) return fail(ctx, LEMGPU_ECONFIG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaMemcpyAsync(host, ctx->hbuf[ctx->cur], (size_t)ctx->a.N * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return LEMGPU_OK;
}

int lemgpu_fill(lemgpu_ctx* ctx, int mode, double epsilon) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  if (mode < LEMGPU_FILL_OFF || mode > LEMGPU_FILL_EPSILON) return fail(ctx, LEMGPU_ECONFIG, "unknown fill mode %d", mode);
  if (mode == LEMGPU_FILL_EPSILON && !(epsilon > 0.0))  // config.cpp:164-165
    return fail(ctx, LEMGPU_ECONFIG, "fill_epsilon must be > 0 for epsilon_ascending fill");
  if (mode == LEMGPU_FILL_OFF) return LEMGPU_OK;
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc0 = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc0) return rc0;
  }
  const StepArgs& a = ctx->a;
  cudaStream_t st = ctx->stream;
  FillArgs fa{};
  fa.h = ctx->hbuf[ctx->cur];
  fa.f = ctx->hbuf[ctx->cur ^ 1u];
  fa.W = a.W;
  fa.H = a.H;
  fa.Htot = a.Htot;
  fa.ntx = (a.W + kFX - 1) / kFX;
  fa.nty = (a.Htot + kFY - 1) / kFY;
  fa.mode = mode;
  fa.eps = epsilon;
  const uint32_t nt = fa.ntx * fa.nty;
  uint32_t* d = nullptr;  // dirty[2][nt], any
  CU(ctx, cudaMalloc(&d, ((size_t)2 * nt + 1) * sizeof(uint32_t)));
  k_fill_init<<<2368, kTPB, 0, st>>>(fa.h, fa.f, a.W, a.H, a.Htot);
  int rc = LEMGPU_OK;
  for (uint32_t pass = 0;; ++pass) {
    uint32_t* cur = d + (pass & 1u) * nt;
    fa.dirty_prev = pass ? d + ((pass + 1) & 1u) * nt : nullptr;
    fa.dirty_cur = cur;
    fa.any = d + 2 * nt;
    cudaMemsetAsync(cur, 0, (size_t)nt * sizeof(uint32_t), st);
    cudaMemsetAsync(fa.any, 0, sizeof(uint32_t), st);
    k_fill_pass<<<nt, kTPB, 0, st>>>(fa);
    uint32_t any = 0;
    if (cudaMemcpyAsync(&any, fa.any, sizeof any, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
      rc = fail(ctx, LEMGPU_ECUDA, "fill: %s", cudaGetErrorString(cudaGetLastError()));
      break;
    }
    if (!any) break;
  }
  cudaFree(d);
  if (rc) return rc;
  ctx->cur ^= 1u;
  ctx->cur_synced = ctx->cur;
  ctx->have_graph = false;
  return LEMGPU_OK;
}

int lemgpu_generate_terrain(lemgpu_ctx* ctx, const uint64_t* seeds) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  const StepArgs& a = ctx->a;
  std::vector<unsigned long long> s(a.M, 42ull);
  if (seeds)
    for (uint32_t m = 0; m < a.M; ++m) s[m] = seeds[m];
  unsigned long long* d_seeds = nullptr;
  CU(ctx, cudaMalloc(&d_seeds, a.M * sizeof(unsigned long long)));
  CU(ctx, cudaMemcpy(d_seeds, s.data(), a.M * sizeof(unsigned long long), cudaMemcpyHostToDevice));
  k_terrain<<<2368, kTPB, 0, ctx->stream>>>(ctx->hbuf[ctx->cur], a.N, a.MN, d_seeds);
  CU(ctx, cudaGetLastError());
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  cudaFree(d_seeds);
  ctx->have_graph = false;
  return LEMGPU_OK;
}

int lemgpu_step_async(lemgpu_ctx* ctx, uint32_t nsteps) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  for (uint32_t s = 0; s < nsteps; ++s) {
    if (ctx->pending >= ctx->diag_cap) {
      uint32_t cnt = 0;
      const int rc = lemgpu_sync(ctx, nullptr, 0, &cnt);
      if (rc) return rc;
    }
    const int rc = enqueue_step(ctx);
    if (rc) return rc;
  }
  return LEMGPU_OK;
}

int lemgpu_sync(lemgpu_ctx* ctx, lemgpu_diag* out, uint32_t cap, uint32_t* count) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (ctx->snap_pending) {  // the diagnostics ring is reused after a sync: the snapshot copy must be done
    CU(ctx, cudaEventSynchronize(ctx->ev_snap_done));
    ctx->snap_pending = false;
  }
  const uint32_t n = ctx->pending;
  std::vector<lemgpu_diag> d(n);
  if (n) CU(ctx, cudaMemcpy(d.data(), ctx->d_diag, n * sizeof(lemgpu_diag), cudaMemcpyDeviceToHost));
  if (ctx->timing && n) {
    for (uint32_t s = 0; s < n; ++s) {
      float t = 0;
      cudaEventElapsedTime(&t, ctx->ev[2 * s], ctx->ev[2 * s + 1]);
      ctx->kernel_ms[0] += t;
      ctx->kernel_ms[1] += d[s].kernel_s[0] * 1e3;
      ctx->kernel_ms[2] += d[s].kernel_s[2] * 1e3;
      ctx->kernel_ms[3] += d[s].kernel_s[3] * 1e3;
      ctx->kernel_ms[4] += d[s].kernel_s[1] * 1e3;
    }
    ctx->kernel_launches += n;
  }
  ctx->pending = 0;
  const uint32_t c0buf = ctx->cur_synced;
  ctx->cur_synced = ctx->cur;
  if (n) CU(ctx, cudaMemset(reinterpret_cast<char*>(ctx->a.ctl) + offsetof(Ctl, slot), 0, sizeof(uint32_t)));
  int status = LEMGPU_OK;
  for (uint32_t s = 0; s < n; ++s) {
    if (d[s].status != 0) {
      status = d[s].status == 0xFFFFFFFFu ? LEMGPU_EOTHER : (int)d[s].status;
      ctx->err_cell = d[s].err_cell;
      if (status == LEMGPU_ECONVERGENCE)
        fail(ctx, status, "Newton iteration did not converge at cell %u after %d iterations",
             d[s].err_cell, ctx->params.max_newton_iters);
      else if (status == LEMGPU_ESTRUCTURE)
        fail(ctx, status, "receiver graph has a cycle: only %u of %u cells reachable from sources",
             d[s].err_cell, ctx->a.N);
      else
        fail(ctx, status, "step %u failed with status %u", s, d[s].status);
      // clear the sticky device flag so the context can be reused
      Ctl cb{};
      CU(ctx, cudaMemcpy(&cb, ctx->a.ctl, sizeof cb, cudaMemcpyDeviceToHost));
      cb.err_flag = 0;
      cb.err_cell = LEMGPU_NOFLOW;
      cb.slot = 0;
      CU(ctx, cudaMemcpy(ctx->a.ctl, &cb, sizeof cb, cudaMemcpyHostToDevice));
      // a failed step leaves the elevation as it was before that step: its
      // input buffer (steps never write the buffer they read; later steps
      // of the batch did not run)
      ctx->cur = ctx->cur_synced = (c0buf + s) & 1u;
      ctx->mfd_src = ctx->cur;  // the failed step read this buffer
      break;
    }
    ctx->last_nlevels = d[s].nlevels;
  }
  if (out)
    for (uint32_t s = 0; s < n && s < cap; ++s) out[s] = d[s];
  if (count) *count = n;
  return status;
}

int lemgpu_step(lemgpu_ctx* ctx, uint32_t nsteps, lemgpu_diag* per_step) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  uint32_t done = 0;
  while (done < nsteps) {
    const uint32_t chunk = (nsteps - done) < ctx->diag_cap ? (nsteps - done) : ctx->diag_cap;
    if (ctx->pending) {
      const int rc0 = lemgpu_sync(ctx, nullptr, 0, nullptr);
      if (rc0) return rc0;
    }
    int rc = lemgpu_step_async(ctx, chunk);
    if (rc) return rc;
    uint32_t cnt = 0;
    rc = lemgpu_sync(ctx, per_step ? per_step + done : nullptr, chunk, &cnt);
    if (rc) return rc;
    done += chunk;
  }
  return LEMGPU_OK;
}

int lemgpu_snapshot_async(lemgpu_ctx* ctx, double* host, lemgpu_diag* diag_host) {
  if (!ctx || !host) return fail(ctx, LEMGPU_ECONFIG, "null argument");
  if (!ctx->pending) return fail(ctx, LEMGPU_ECONFIG, "no step enqueued since the last sync");
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->snap_pending) {
    CU(ctx, cudaEventSynchronize(ctx->ev_snap_done));
    ctx->snap_pending = false;
  }
  if (!ctx->s_snap) {
    CU(ctx, cudaStreamCreateWithFlags(&ctx->s_snap, cudaStreamNonBlocking));
    CU(ctx, cudaEventCreateWithFlags(&ctx->ev_snap_step, cudaEventDisableTiming));
    CU(ctx, cudaEventCreateWithFlags(&ctx->ev_snap_done, cudaEventDisableTiming));
  }
  // the state after the last enqueued step, and that step's diagnostics slot
  CU(ctx, cudaEventRecord(ctx->ev_snap_step, ctx->stream));
  CU(ctx, cudaStreamWaitEvent(ctx->s_snap, ctx->ev_snap_step, 0));
  CU(ctx, cudaMemcpyAsync(host, ctx->hbuf[ctx->cur], (size_t)ctx->a.N * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->s_snap));
  if (diag_host)
    CU(ctx, cudaMemcpyAsync(diag_host, ctx->d_diag + (ctx->pending - 1), sizeof(lemgpu_diag), cudaMemcpyDeviceToHost,
                            ctx->s_snap));
  CU(ctx, cudaEventRecord(ctx->ev_snap_done, ctx->s_snap));
  ctx->snap_buf = ctx->cur;
  ctx->snap_pending = true;
  return LEMGPU_OK;
}

int lemgpu_snapshot_wait(lemgpu_ctx* ctx) {
  if (!ctx) return LEMGPU_ECONFIG;
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->snap_pending) {
    CU(ctx, cudaEventSynchronize(ctx->ev_snap_done));
    ctx->snap_pending = false;
  }
  return LEMGPU_OK;
}

int lemgpu_step_host(lemgpu_ctx* ctx, double* elev_inout, lemgpu_diag* diag) {
  if (!ctx || !elev_inout) return fail(ctx, LEMGPU_ECONFIG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  const StepArgs& a = ctx->a;
  if (ctx->use_tiles && ctx->bands > 1 && !a.eager && !a.mfd_A) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, elev_inout) == cudaSuccess && pa.type == cudaMemoryTypeHost)
      return step_host_banded(ctx, elev_inout, diag);
    cudaGetLastError();  // pageable memory: the copies would not overlap
  }
  CU(ctx, cudaMemcpyAsync(ctx->hbuf[ctx->cur], elev_inout, (size_t)a.N * sizeof(double), cudaMemcpyHostToDevice,
                          ctx->stream));
  int rc = lemgpu_step_async(ctx, 1);
  if (rc) return rc;
  CU(ctx, cudaMemcpyAsync(elev_inout, ctx->hbuf[ctx->cur], (size_t)a.N * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  lemgpu_diag d{};
  uint32_t cnt = 0;
  rc = lemgpu_sync(ctx, &d, 1, &cnt);
  if (diag) *diag = d;
  if (rc && rc != LEMGPU_ECUDA)  // the failed step left the elevation unchanged
    cudaMemcpy(elev_inout, ctx->hbuf[ctx->cur], (size_t)a.N * sizeof(double), cudaMemcpyDeviceToHost);
  return rc;
}

int lemgpu_download_graph(lemgpu_ctx* ctx, uint32_t* rec, uint8_t* dnum, uint32_t* donor,
                          uint32_t* order, uint32_t* levels, uint32_t* nlevels, double* A) {
  if (!ctx) return fail(ctx, LEMGPU_ECONFIG, "null context");
  if (!ctx->have_graph) return fail(ctx, LEMGPU_ECONFIG, "no step has run since the last upload");
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  // The TraversalPlan and the accumulation of the last step, rebuilt from
  // its flow graph (rcode / dmask, written by the step) with the global
  // level path: level 0 = all NoFlow cells ascending, one expansion per
  // level, then A swept deepest level first in slot order -- the reference's
  // generate_queue + accumulate (traversal.cpp:19-48, accumulation.cpp:7-17).
  StepArgs a = ctx->a;
  a.tiles = 0;
  a.eager = 1;
  a.expect_cells = a.N;
  {
    cudaStream_t st = ctx->stream;
    if (ctx->use_tiles) k_fill_dmask<<<2368, kTPB, 0, st>>>(a);
    set_eager_conds(a, st);
    k_l0_count<<<ctx->scan_grid, kTPB, 0, st>>>(a);
    k_l0_write<<<ctx->scan_grid, kTPB, 0, st>>>(a);
    const size_t co = offsetof(Ctl, cond);
    char* cbase = reinterpret_cast<char*>(a.ctl) + co;
    unsigned cond[3] = {1, 0, 0};
    while (cond[0]) {
      k_expand<<<ctx->scan_grid, kTPB, 0, st>>>(a);
      CU(ctx, cudaMemcpyAsync(cond, cbase, sizeof cond, cudaMemcpyDeviceToHost, st));
      CU(ctx, cudaStreamSynchronize(st));
    }
    Ctl c{};
    CU(ctx, cudaMemcpy(&c, a.ctl, sizeof c, cudaMemcpyDeviceToHost));
    if (c.err_flag) return fail(ctx, LEMGPU_ESTRUCTURE, "receiver graph has a cycle");
    ctx->last_nlevels = c.nlev;
    for (int L = (int)c.nlev - 1; L >= 0; --L) k_acc_level<<<ctx->deep_grid, kTPB, 0, st>>>(a, (uint32_t)L);
    // leave the per-step control state as a step expects it
    c.lvl = 0;
    c.done = 0;
    c.mode = kModeShallow;
    c.cond[0] = c.cond[1] = c.cond[2] = 0;
    CU(ctx, cudaMemcpyAsync(a.ctl, &c, sizeof c, cudaMemcpyHostToDevice, st));
    CU(ctx, cudaStreamSynchronize(st));
  }
  const size_t N = a.N;
  uint32_t* d_rec = nullptr;
  uint8_t* d_dnum = nullptr;
  uint32_t* d_donor = nullptr;
  double* d_A = nullptr;
  if (rec) CU(ctx, cudaMalloc(&d_rec, N * 4));
  if (dnum) CU(ctx, cudaMalloc(&d_dnum, N));
  if (donor) CU(ctx, cudaMalloc(&d_donor, N * a.conn * 4));
  if (A) CU(ctx, cudaMalloc(&d_A, N * 8));
  if (rec || dnum || donor) k_export_graph<<<2368, kTPB, 0, ctx->stream>>>(a, d_rec, d_dnum, d_donor);
  if (A) k_export_accum<<<2368, kTPB, 0, ctx->stream>>>(a, d_A);
  CU(ctx, cudaGetLastError());
  if (rec) CU(ctx, cudaMemcpyAsync(rec, d_rec, N * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (dnum) CU(ctx, cudaMemcpyAsync(dnum, d_dnum, N, cudaMemcpyDeviceToHost, ctx->stream));
  if (donor) CU(ctx, cudaMemcpyAsync(donor, d_donor, N * a.conn * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (A) CU(ctx, cudaMemcpyAsync(A, d_A, N * 8, cudaMemcpyDeviceToHost, ctx->stream));
  if (order) CU(ctx, cudaMemcpyAsync(order, a.order, N * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (levels) CU(ctx, cudaMemcpyAsync(levels, a.levels, ((size_t)ctx->last_nlevels + 1) * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  if (nlevels) *nlevels = ctx->last_nlevels;
  cudaFree(d_rec);
  cudaFree(d_dnum);
  cudaFree(d_donor);
  cudaFree(d_A);
  return LEMGPU_OK;
}

int lemgpu_member_stats_device(lemgpu_ctx* ctx, double* device_out) {
  if (!ctx || !device_out) return fail(ctx, LEMGPU_ECONFIG, "null argument");
  CU(ctx, cudaSetDevice(ctx->device));
  const StepArgs& a = ctx->a;
  const uint32_t chunks = 64;
  // partials live in the accumulation scratch (Aq), which is per-step scratch
  double* part = a.Aq;
  if ((size_t)a.M * chunks * 3 > a.N) return fail(ctx, LEMGPU_ECONFIG, "members too small for stats scratch");
  k_stats_partial<<<dim3(chunks, a.M), kTPB, 0, ctx->stream>>>(ctx->hbuf[ctx->cur], a.MN, chunks, part);
  k_stats_final<<<(a.M + 127) / 128, 128, 0, ctx->stream>>>(part, a.M, chunks, a.MN, device_out);
  CU(ctx, cudaGetLastError());
  ctx->have_graph = false;  // Aq was clobbered
  return LEMGPU_OK;
}

int lemgpu_kernel_timing(lemgpu_ctx* ctx, int enable) {
  if (!ctx) return LEMGPU_ECONFIG;
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  ctx->timing = enable != 0;
  for (double& v : ctx->kernel_ms) v = 0;
  ctx->kernel_launches = 0;
  return LEMGPU_OK;
}

int lemgpu_kernel_times(lemgpu_ctx* ctx, double* ms, uint32_t* launches) {
  if (!ctx || !ms) return LEMGPU_ECONFIG;
  for (int i = 0; i < 5; ++i) ms[i] = ctx->kernel_ms[i];
  if (launches) *launches = ctx->kernel_launches;
  return LEMGPU_OK;
}

int lemgpu_debug_timeline(lemgpu_ctx* ctx, uint64_t* ns, uint32_t cap, uint32_t* count) {
  if (!ctx || !ns) return LEMGPU_ECONFIG;
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  Ctl c{};
  CU(ctx, cudaMemcpy(&c, ctx->a.ctl, sizeof c, cudaMemcpyDeviceToHost));
  const uint32_t n = c.nltl < cap ? c.nltl : cap;
  for (uint32_t i = 0; i < n; ++i) ns[i] = c.ltl[i];
  if (count) *count = n;
  return LEMGPU_OK;
}

int lemgpu_debug_copy(lemgpu_ctx* ctx, int which, void* host, uint64_t bytes) {
  if (!ctx || !host) return LEMGPU_ECONFIG;
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  const void* src = which == 0 ? (const void*)ctx->a.order : which == 1 ? (const void*)ctx->d_levels_esc
                    : which == 2 ? (const void*)ctx->a.ctl : which == 3 ? (const void*)ctx->a.dbg_level
                    : which == 4 ? (const void*)ctx->a.dbg_A : (const void*)ctx->a.bins;
  const uint64_t cap = which == 0 ? (uint64_t)ctx->a.N * 4 : which == 1 ? ((uint64_t)ctx->a.N + 2) * 4
                       : which == 2 ? sizeof(Ctl) : which == 3 ? (uint64_t)ctx->a.N : which == 4 ? (uint64_t)ctx->a.N * 8
                       : 3 * 4096 * 4;
  if (!src) return fail(ctx, LEMGPU_ECONFIG, "debug capture is off");
  CU(ctx, cudaMemcpy(host, src, bytes < cap ? bytes : cap, cudaMemcpyDeviceToHost));
  return LEMGPU_OK;
}

int lemgpu_debug_tile_capture(lemgpu_ctx* ctx, int enable) {
  if (!ctx) return LEMGPU_ECONFIG;
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  StepArgs& a = ctx->a;
  if (enable && !a.dbg_level) {
    CU(ctx, cudaMalloc(&a.dbg_level, a.N));
    CU(ctx, cudaMalloc(&a.dbg_A, (size_t)a.N * sizeof(double)));
  } else if (!enable && a.dbg_level) {
    cudaFree(a.dbg_level);
    cudaFree(a.dbg_A);
    a.dbg_level = nullptr;
    a.dbg_A = nullptr;
  } else {
    return LEMGPU_OK;
  }
  if (const int rc = rebuild_graphs(ctx)) return rc;
  if (a.dbg_level) {
    CU(ctx, cudaMemset(a.dbg_level, 0xFF, a.N));
    CU(ctx, cudaMemset(a.dbg_A, 0xFF, (size_t)a.N * sizeof(double)));
  }
  return LEMGPU_OK;
}

int lemgpu_set_routing(lemgpu_ctx* ctx, int routing, double mfd_exponent) {
  if (!ctx) return LEMGPU_ECONFIG;
  if (routing != 0 && routing != 1) return fail(ctx, LEMGPU_ECONFIG, "routing must be 0 (d8) or 1 (mfd)");
  if (!(mfd_exponent > 0.0) || !std::isfinite(mfd_exponent))
    return fail(ctx, LEMGPU_ECONFIG, "mfd_exponent must be > 0");  // config.cpp:166
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  StepArgs& a = ctx->a;
  const size_t N = a.N;
  const size_t ntm = 2 * (size_t)mfd_cap(a.W, a.Htot);  // k_mfd_tiles: tiles of both grids
  if (routing == 1 && !a.mfd_A) {
    if ((dmalloc(ctx, &a.mfd_A, N)) || (dmalloc(ctx, &a.mfd_wsum, N)) || (dmalloc(ctx, &a.mfd_lm, N)) ||
        (dmalloc(ctx, &a.mfd_rem, N)) || (dmalloc(ctx, &a.mfd_ord, N)) || (dmalloc(ctx, &a.mfd_lv, N + 2)) ||
        (dmalloc(ctx, &a.mfd_lev, N)) || (dmalloc(ctx, &a.mfd_wl, ntm)) || (dmalloc(ctx, &a.mfd_stamp, ntm)))
      return LEMGPU_ECUDA;
    CU(ctx, cudaMemset(a.mfd_stamp, 0, ntm * sizeof(uint32_t)));
    CU(ctx, cudaMemset(a.mfd_A, 0, N * sizeof(double)));
  } else if (routing == 0 && a.mfd_A) {
    for (void* q : {(void*)a.mfd_A, (void*)a.mfd_wsum, (void*)a.mfd_lm, (void*)a.mfd_rem, (void*)a.mfd_ord,
                    (void*)a.mfd_lv, (void*)a.mfd_lev, (void*)a.mfd_wl, (void*)a.mfd_stamp})
      cudaFree(q);
    a.mfd_A = a.mfd_wsum = nullptr;
    a.mfd_lm = nullptr;
    a.mfd_rem = a.mfd_ord = a.mfd_lv = a.mfd_lev = a.mfd_wl = a.mfd_stamp = nullptr;
  }
  a.mfd_exp = mfd_exponent;
  ctx->routing = routing;
  // MFD: the area by tile passes ahead of the D8 tile path (option
  // mfd_levels: the level-synchronous plan + the global level path)
  ctx->use_tiles = ctx->opt_global || (routing == 1 && ctx->opt_mfd_levels) ? 0 : 1;
  return rebuild_graphs(ctx);
}

int lemgpu_download_mfd(lemgpu_ctx* ctx, double* A, uint32_t* order, uint32_t* levels, uint32_t* nlevels) {
  if (!ctx) return LEMGPU_ECONFIG;
  if (!ctx->a.mfd_A) return fail(ctx, LEMGPU_ECONFIG, "routing is not mfd (lemgpu_set_routing)");
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  const StepArgs& a = ctx->a;
  const size_t N = a.N;
  if (A) CU(ctx, cudaMemcpy(A, a.mfd_A, N * sizeof(double), cudaMemcpyDeviceToHost));
  if ((order || levels || nlevels) && ctx->use_tiles) {
    // the tile passes need no plan: rebuild the step's (generate_mfd_order)
    // from the elevation that step read -- k_mfd_levels also re-evaluates A
    // level by level, to the same bits
    StepArgs b = step_args(ctx, ctx->mfd_src);
    b.eager = 1;
    k_mfd_graph<<<ctx->deep_grid, kTPB, 0, ctx->stream>>>(b);
    void* margs[] = {&b};
    CU(ctx, cudaLaunchCooperativeKernel((const void*)k_mfd_levels, dim3(ctx->mfd_grid), dim3(kTPB), margs, 0,
                                        ctx->stream));
    CU(ctx, cudaStreamSynchronize(ctx->stream));
  }
  if (order || levels || nlevels) {
    // the reference's TraversalPlan (mfd.cpp:66-104): level-major, ascending
    // within a level -- a counting sort of the cell-major levels
    Ctl c{};
    CU(ctx, cudaMemcpy(&c, a.ctl, sizeof c, cudaMemcpyDeviceToHost));
    const uint32_t nl = c.mfd_nlev;
    std::vector<uint32_t> lev(N), start(nl + 1, 0);
    CU(ctx, cudaMemcpy(lev.data(), a.mfd_lev, N * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < N; ++i) {
      if (lev[i] >= nl) return fail(ctx, LEMGPU_ESTRUCTURE, "MFD plan incomplete (cell %zu)", i);
      ++start[lev[i] + 1];
    }
    for (uint32_t l = 0; l < nl; ++l) start[l + 1] += start[l];
    if (levels)
      for (uint32_t l = 0; l <= nl; ++l) levels[l] = start[l];
    if (order)
      for (size_t i = 0; i < N; ++i) order[start[lev[i]]++] = (uint32_t)i;
    if (nlevels) *nlevels = nl;
  }
  return LEMGPU_OK;
}

int lemgpu_stats_enable(lemgpu_ctx* ctx, uint32_t member_offset, uint32_t members_total, uint32_t interval) {
  if (!ctx) return LEMGPU_ECONFIG;
  StepArgs& a = ctx->a;
  if (members_total < member_offset + a.M)
    return fail(ctx, LEMGPU_ECONFIG, "members_total %u < member_offset %u + %u local members", members_total,
                member_offset, a.M);
  if (ctx->st_on) return fail(ctx, LEMGPU_ECONFIG, "statistics already enabled");
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  const size_t tb = (size_t)members_total * 4 * sizeof(double);
  CU(ctx, cudaMalloc(&ctx->st_local, 2 * tb));
  CU(ctx, cudaMemset(ctx->st_local, 0, 2 * tb));
  ctx->st_all = ctx->st_local;  // no communicator: the local table is the table
  ctx->st_total = members_total;
  ctx->st_member0 = member_offset;
  // chunks per member: ~4 CTAs per SM over the whole ensemble, >= 1
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  a.st_chunks = std::max<uint32_t>(1u, std::min<uint32_t>(4u * (uint32_t)nsm / a.M + 1u, (a.MN + 4095u) / 4096u));
  CU(ctx, cudaMalloc(&ctx->st_part, (size_t)a.M * a.st_chunks * 3 * sizeof(double)));
  a.st_part = ctx->st_part;
  ctx->st_interval = interval ? interval : 1u;
  a.st_table = ctx->st_local;
  a.st_member0 = member_offset;
  ctx->st_on = true;
  return rebuild_graphs(ctx);
}

int lemgpu_nccl_unique_id(void* id_out, uint32_t bytes) {
  if (!id_out || bytes < sizeof(ncclUniqueId)) return LEMGPU_ECONFIG;
  if (!nccl().load()) return fail(nullptr, LEMGPU_EOTHER, "%s", nccl().why.c_str());
  ncclUniqueId id;
  const ncclResult_t r = nccl().getUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, LEMGPU_ECUDA, "ncclGetUniqueId: %s", nccl().errStr(r));
  std::memcpy(id_out, &id, sizeof id);
  return LEMGPU_OK;
}

int lemgpu_stats_comm_init(lemgpu_ctx* ctx, const void* id, uint32_t bytes, int nranks, int rank) {
  if (!ctx || !id || bytes < sizeof(ncclUniqueId) || nranks < 1 || rank < 0 || rank >= nranks)
    return fail(ctx, LEMGPU_ECONFIG, "bad communicator arguments");
  if (!ctx->st_on) return fail(ctx, LEMGPU_ECONFIG, "enable the statistics first (lemgpu_stats_enable)");
  if (ctx->comm) return fail(ctx, LEMGPU_ECONFIG, "communicator already set");
  if (!nccl().load()) return fail(ctx, LEMGPU_EOTHER, "%s", nccl().why.c_str());
  CU(ctx, cudaSetDevice(ctx->device));
  if (ctx->pending) {
    const int rc = lemgpu_sync(ctx, nullptr, 0, nullptr);
    if (rc) return rc;
  }
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof uid);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = nccl().commInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) return fail(ctx, LEMGPU_ECUDA, "ncclCommInitRank: %s", nccl().errStr(r));
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->st_all = ctx->st_local + (size_t)ctx->st_total * 4;  // out-of-place all-reduce
  return rebuild_graphs(ctx);
}

int lemgpu_stats_table(lemgpu_ctx* ctx, double* host_out) {
  if (!ctx || !host_out) return LEMGPU_ECONFIG;
  if (!ctx->st_on) return fail(ctx, LEMGPU_ECONFIG, "statistics are not enabled");
  CU(ctx, cudaSetDevice(ctx->device));
  CU(ctx, cudaMemcpyAsync(host_out, ctx->st_all, (size_t)ctx->st_total * 4 * sizeof(double), cudaMemcpyDeviceToHost,
                          ctx->stream));
  CU(ctx, cudaStreamSynchronize(ctx->stream));
  return LEMGPU_OK;
}

const double* lemgpu_stats_table_device(const lemgpu_ctx* ctx) { return ctx && ctx->st_on ? ctx->st_all : nullptr; }

int lemgpu_shard_members(uint32_t members_total, int nranks, int rank, uint32_t* first, uint32_t* count) {
  if (nranks < 1 || rank < 0 || rank >= nranks || !first || !count) return LEMGPU_ECONFIG;
  // partition_sources (scheduler.cpp:396-406): bounds[w] = total * w / workers
  const uint64_t b0 = (uint64_t)members_total * (uint64_t)rank / (uint64_t)nranks;
  const uint64_t b1 = (uint64_t)members_total * (uint64_t)(rank + 1) / (uint64_t)nranks;
  *first = (uint32_t)b0;
  *count = (uint32_t)(b1 - b0);
  return LEMGPU_OK;
}

int lemgpu_create_ensemble_shard(int device, uint32_t width, uint32_t height, uint32_t members_total, int nranks,
                                 int rank, const lemgpu_params* params, const lemgpu_member* per_member_all,
                                 uint32_t stats_interval, const lemgpu_options* options, lemgpu_ctx** out) {
  if (!out) return LEMGPU_ECONFIG;
  *out = nullptr;
  uint32_t first = 0, count = 0;
  if (lemgpu_shard_members(members_total, nranks, rank, &first, &count) != LEMGPU_OK || count == 0)
    return fail(nullptr, LEMGPU_ECONFIG, "rank %d of %d owns no member of %u", rank, nranks, members_total);
  const int rc = create_impl(device, width, height, count, params, per_member_all ? per_member_all + first : nullptr,
                             options, out);
  if (rc) return rc;
  const int rs = lemgpu_stats_enable(*out, first, members_total, stats_interval);
  if (rs) {
    g_create_error = (*out)->msg;
    lemgpu_destroy(*out);
    *out = nullptr;
  }
  return rs;
}

int lemgpu_pow_variant(const lemgpu_ctx* ctx) { return ctx ? ctx->pow_variant : host_pow_variant(); }

int lemgpu_debug_pow(int device, int variant, const double* x, const double* y, double* out, uint64_t n) {
  if (!x || !y || !out) return LEMGPU_ECONFIG;
  if (cudaSetDevice(device) != cudaSuccess) return LEMGPU_ECUDA;
  double* d = nullptr;
  if (cudaMalloc(&d, 3 * n * sizeof(double) + 8) != cudaSuccess) return LEMGPU_ECUDA;
  int rc = LEMGPU_OK;
  if (cudaMemcpy(d, x, n * 8, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(d + n, y, n * 8, cudaMemcpyHostToDevice) != cudaSuccess)
    rc = LEMGPU_ECUDA;
  if (!rc && n) {
    k_debug_pow<<<1184, kTPB>>>(variant != 0, d, d + n, d + 2 * n, n);
    if (cudaGetLastError() != cudaSuccess || cudaMemcpy(out, d + 2 * n, n * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = LEMGPU_ECUDA;
  }
  cudaFree(d);
  return rc;
}

int lemgpu_host_register(void* ptr, size_t bytes) {
  return cudaHostRegister(ptr, bytes, cudaHostRegisterDefault) == cudaSuccess ? LEMGPU_OK : LEMGPU_ECUDA;
}
int lemgpu_host_unregister(void* ptr) {
  return cudaHostUnregister(ptr) == cudaSuccess ? LEMGPU_OK : LEMGPU_ECUDA;
}

}  // extern "C"
