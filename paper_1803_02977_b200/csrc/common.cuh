// common.cuh -- shared definitions of the sm_100a D8 landscape-evolution step.
//
// One timestep is a CUDA graph of these kernels:
//
//   k_recv              receiver codes + code bit planes                  (k_recv_donor.cuh)
//   k_tiles             level order, accumulation, uplift and erosion of
//                       every drainage tree rooted in a 64x32 tile whose
//                       cells stay within 3 cells of it                  (k_tiles.cuh)
//   then, for the trees that escape their tile:
//   k_esc_small         a small escape set in one CTA's shared memory      (k_tiles.cuh)
//   k_esc_forest        cooperative: most of the raster escaped (filled DEMs): levels by
//                       pointer jumping, trees split between CTAs, swept with block
//                       barriers only                                     (k_forest.cuh)
//   k_esc_bfs           cooperative: every level of the escaped trees      (k_order.cuh)
//   k_chunks            accumulation + uplift + erosion per source chunk  (k_physics.cuh)
//   k_deep_coop         cooperative: the same sweeps level by level for
//                       deep plans                                        (k_physics.cuh)
//   k_finalize          per-step diagnostics                              (k_physics.cuh)
//
// The global level path (LEMGPU_PATH=global, and the parity export) runs
// k_recv_donor (receivers + donor masks), k_l0_count/_write (level 0) and
// WHILE { k_expand } / WHILE { k_deep_* } graph loops instead.  The number of
// levels is data dependent and discovered on the device (cooperative loops
// or graph WHILE nodes set with cudaGraphSetConditional), so a step is one
// cudaGraphLaunch with no host round trip.
//
// Arithmetic is FP64 and never contracted: compiled with --fmad=false and
// every rounding-relevant operation is an explicit __d*_rn intrinsic, so the
// results are bit-identical to the reference built with -ffp-contract=off
// (proj/CMakeLists.txt:14).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "glibc_pow.cuh"
#include "lemgpu.h"

namespace lemgpu {

constexpr int kTPB = 256;           // threads per CTA (all kernels)
constexpr int kNW = kTPB / 32;      // warps per CTA
constexpr uint8_t kNoFlowCode = 8;  // rcode value for kNoFlow

// k_tiles: owned tile, BFS halo (see k_tiles.cuh)
#ifndef LEMGPU_TILE_Y
// measured best of {16,24,32,40,48} rows x {128..384} threads x {3..7} CTAs/SM
// (tools/variants_check.sh): 64x32 tiles, 6 warps, 5 CTAs/SM (45 KB smem each)
#define LEMGPU_TILE_Y 32
#define LEMGPU_TILE_TPB 192
#define LEMGPU_TILE_MINB 5
#endif
constexpr int kTX = 64, kTY = LEMGPU_TILE_Y, kHalo = 3;
constexpr int kTTPB = LEMGPU_TILE_TPB;

// k_recv / k_recv_donor tile (output cells): halo of 2 for h, 1 for the receiver codes.
constexpr int kBX = 128;
constexpr int kBY = 32;
// scan tiles
constexpr int kL0IPT = 16;              // level-0 cells per thread (one uint4 of rcodes)
constexpr int kL0Tile = kTPB * kL0IPT;  // 4096 cells
constexpr int kExIPT = 2;               // frontier items per thread
constexpr int kExTile = kTPB * kExIPT;  // 512 frontier cells
// source chunks of the physics sweeps
#ifndef LEMGPU_CHUNK_ROOTS
#define LEMGPU_CHUNK_ROOTS 16  // measured best of {16,24,32,40,48} at 10000^2 (occupancy-bound)
#define LEMGPU_CHUNK_CAP 256
#define LEMGPU_CHUNK_MINB 8
#endif
constexpr int kChunkRoots = LEMGPU_CHUNK_ROOTS;  // level-0 sources per chunk (one warp each)
constexpr int kChunkCap = LEMGPU_CHUNK_CAP;      // cells per chunk held in shared memory
constexpr int kChunkSlots = kChunkCap / 32;  // cells per lane
constexpr int kChunkTPB = 128;        // k_chunks CTA: 4 warps, 4 chunks in flight
constexpr int kChunkMaxLevels = 24;   // shallow (chunked) plans: nlevels <= this
constexpr int kCBS = kChunkMaxLevels + 1;

enum : uint32_t { kModeShallow = 0, kModeDeep = 1, kModeFailed = 2, kModeDone = 3 };

// Frozen D8 stencil (src/neighborhood.cpp:12): k -> (ox, oy).  The opposite
// direction of k is 7-k.  D4 is the cardinal subsequence {1,3,4,6}
// (neighborhood.cpp:20-29), kept at its D8 slot so stencil order and the
// opposite-direction rule are shared.
__host__ __device__ constexpr int dir_ox(int k) {
  return (k == 0 || k == 3 || k == 5) ? -1 : (k == 1 || k == 6) ? 0 : 1;
}
__host__ __device__ constexpr int dir_oy(int k) { return k < 3 ? -1 : k < 5 ? 0 : 1; }
// Branch-free runtime form: linear offset of direction k in a raster of width W.
__device__ __forceinline__ int dir_off(uint32_t k, int W) {
  const int ox = (int)((0x9224u >> (2 * k)) & 3u) - 1;
  const int oy = (int)((0xA940u >> (2 * k)) & 3u) - 1;
  return ox + oy * W;
}
__host__ __device__ constexpr bool dir_in(int conn, int k) {
  return conn == 8 || k == 1 || k == 3 || k == 4 || k == 6;
}

// IEEE round-to-nearest arithmetic usable on host and device (host code is
// compiled with -ffp-contract=off, so plain operators do not fuse).
#ifdef __CUDA_ARCH__
#define LG_ADD(x, y) __dadd_rn((x), (y))
#define LG_SUB(x, y) __dsub_rn((x), (y))
#define LG_MUL(x, y) __dmul_rn((x), (y))
#define LG_DIV(x, y) __ddiv_rn((x), (y))
#else
#define LG_ADD(x, y) ((x) + (y))
#define LG_SUB(x, y) ((x) - (y))
#define LG_MUL(x, y) ((x) * (y))
#define LG_DIV(x, y) ((x) / (y))
#endif

#ifdef __CUDA_ARCH__
#define LG_FMA(x, y, z) __fma_rn((x), (y), (z))
#else
#define LG_FMA(x, y, z) std::fma((x), (y), (z))
#endif
// pow(x, y) bit-identical with the host glibc (glibc_pow.cuh).  Out of line:
// its ~60 FP64 operations and two table lookups stay out of the register
// budget of the kernels that call it on rare paths.
__device__ __noinline__ double glibc_pow_dev(int pow_fma, double x, double y) {
  return pow_fma ? glibc_pow<true>(x, y) : glibc_pow<false>(x, y);
}

// pow(x, 2) bit-identical with the host glibc: RN(x*x) unless x^2 is within
// 1/64 ulp of a rounding midpoint or outside [2^-128, 2^128) (glibc_pow_sq),
// else the full restatement.
__device__ __forceinline__ double glibc_pow_sq_dev(int pow_fma, double x) {
  if (x == 0.0) return 0.0;
  const double hi = __dmul_rn(x, x);
  const double lo = __fma_rn(x, x, -hi);
  const unsigned long long b = (unsigned long long)__double_as_longlong(hi);
  const uint32_t e = (uint32_t)(b >> 52) & 0x7ffu;
  if (e - (1023u - 128u) < 256u) {  // x^2 in [2^-128, 2^128): the 1/64-ulp bound of glibc_pow_sq holds
    const double ulp = __longlong_as_double((long long)(e - 52u) << 52);
    const double lim = (b & 0x000fffffffffffffull) ? __dmul_rn(ulp, 0.484375) : __dmul_rn(ulp, 0.234375);
    if (fabs(lo) < lim) return hi;
  }
  return glibc_pow_dev(pow_fma, x, 2.0);
}

// High 32 bits of a double (sign, exponent, top 20 mantissa bits).
__host__ __device__ __forceinline__ int hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  unsigned long long b;
  __builtin_memcpy(&b, &x, 8);
  return (int)(b >> 32);
#endif
}

// Device control block (one per context).
struct Ctl {
  // persistent
  uint32_t err_flag;  // sticky LEMGPU_* of the first failing step
  uint32_t err_cell;  // failing cell (any failing cell is acceptable)
  uint32_t err_slot;  // diagnostics slot of the step that failed
  uint32_t slot;      // diagnostics slot of the running step
  uint32_t cond[5];   // loop conditions when the step runs eagerly (no graph)
  // per step (reset by k_finalize)
  uint32_t lvl;          // level being expanded
  uint32_t done;         // finished CTAs of the running kernel
  uint32_t n0, nch, nlev, mode;
  uint32_t dlvl;  // level of the deep sweeps
  uint32_t misses;
  unsigned long long newton;
  // tile path (k_tiles): escaped roots, cells finished in tiles, interior pits, deepest level + 1
  uint32_t nesc, tile_cells, n0i, tile_nlev;
  uint32_t gbar_count, gbar_gen;  // grid barrier of the cooperative escape-path kernel
  uint32_t esc_small;             // 1: k_esc_small finished the escaped trees this step
  uint32_t esc_fail, esc_cells, esc_nlev, esc_misses, esc_done;  // k_esc_small's CTAs: overflow count, totals
  unsigned long long esc_iters;
  uint32_t nr_l, nr_lo, nr_hi, nr_done;  // k_esc_bfs: where a narrow run handed back to the grid
  uint32_t fr_flag[3], fr_maxd;          // k_esc_forest: pointer-jumping round flags, deepest escaped level
  uint32_t fr_rounds, fr_maxcells;       // ... rounds taken, most cells of one CTA
  uint32_t mfd_cnt[3], mfd_nlev;         // k_mfd_levels: per-level append counters, MFD plan levels
  uint32_t mfd_pass, mfd_wl_n[2];        // k_mfd_tiles: pass id (monotonic), queued tiles per pass parity
  uint32_t mfd_passes;                   // ... passes of this step
  uint32_t mfd_done;                     // ... cells finalised in the running pass / round
  uint32_t mfd_tail_n[2], mfd_tail_cur;  // k_mfd_tail: listed cells per list, the list being read
  unsigned long long t_mfd_begin;        // ... first pass start (the step's device time starts there)
  unsigned long long fr_t[3];            // ... latest end over the CTAs of the counts, F and erosion sweeps
  unsigned long long t_k1_begin, t_k1_end, t_order_end, t_phys_end;
  unsigned long long t_t_begin, t_t_end;  // k_tiles
  unsigned long long ph_cyc[32][6];  // SM cycles per lem::Phase charged by the CTAs this step (PhClk), 32 spread slots
  uint32_t ntl, nltl;
  unsigned long long tl[96];   // debug timeline of the running step (finisher stamps)
  unsigned long long ltl[98];  // ... and of the last completed step
};

struct StepArgs {
  // geometry (stacked members: rows [m*H, (m+1)*H) belong to member m)
  uint32_t W, H, M;
  uint32_t N;     // W*H*M  (< 2^32, RunConfig::validate, config.cpp:159-161)
  uint32_t MN;    // W*H
  uint32_t Htot;  // H*M
  uint32_t perim;  // perimeter cells over all members
  int conn;
  int maxit;
  int nkind;      // 1: n == 1, 2: n == 2, 0: general n
  int lut_exact;  // A is always an exact integer multiple of w0
  int w0_is_one;
  uint32_t lut_entries;
  uint32_t dist_one;  // bit k set when dist[k] == 1.0 (division is the identity)
  int unit_card;      // dx == dy == 1: cardinal slopes are the drops themselves
  double rinv_diag;   // RN(1 / dist_diag): pre-decides far-from-tie comparisons only
  double rdist[8];    // RN(1 / dist[k]) (host): correctly rounded quotients by dist (div_rn_recip)
  uint32_t dist_recip;  // bit k: 1 <= dist[k] < 2^500, the reciprocal path applies
  double dist[8];     // offset_length of direction k (neighborhood.hpp:17-23)
  double powdist_h, powdist_v, powdist_d;  // host-libm pow(dist, n) per offset class
  double du, w0, n_exp, eps;
  const double* kdt;   // per member K*dt
  const double* mexp;  // per member m
  const double* ftab;  // per member and offset class: F(a) = (K*dt * pow(a*w0, m)) / pow(dist, n), host libm
  const double* ftab2;  // same index: {F, RN(1 / RN(1 + F))} pairs
  // state / scratch.  h is the elevation the step reads (never written during
  // the step), hout the elevation it writes (ping-pong buffers; the step's
  // receivers always see the complete previous surface)
  double* h;
  double* hout;
  uint8_t* rcode;
  uint8_t* dmask;
  int dmask_valid;   // dmask holds this step's donor masks (else derived from rcode where needed)
  uint32_t* planes;  // 4 bit planes of rcode, [plane][row][W32] words (k_recv -> k_tiles)
  uint32_t W32;      // words per plane row
  uint32_t* order;
  uint32_t* ppos;     // position-major: queue position of the receiver (levels >= 1)
  uint8_t* cdir;      // position-major: stencil direction receiver -> cell (levels >= 1)
  uint32_t* fc;
  uint32_t* cbound;  // [level][chunk]: first position of a source chunk at each level
  uint32_t cb_stride;
  double* Aq;
  double* hq;
  uint32_t* levels;
  uint8_t* pdm;       // donor mask of the cell at each queue position
  uint32_t* part;     // level-0 per-segment NoFlow counts
  uint32_t* bins;     // 3 x scan_grid per-segment child counts (rotating)
  uint32_t scan_grid;  // CTAs of the scan kernels (segments per level)
  int eager;          // 1: no graph; loop conditions go through ctl->cond
  int use_tma;        // k_recv / k_recv_donor / k_tiles stage h with one TMA box per tile
  int force_deep;     // testing: use the per-level sweeps even for shallow plans
  int force_escape;   // testing: 1 = every tree of k_tiles escapes, 2 = trees of odd root cells escape
  int tiles;          // 1: the step runs k_tiles + the escape path (else the global level path)
  uint32_t by0;       // k_recv: first row block of the launch (banded host steps; else 0)
  uint32_t t_lo, t_hi;  // k_tiles: tile range of the launch (t_hi 0: every tile)
  int no_narrow;      // testing: escape expansion / deep sweeps without narrow runs
  int tab_ok;         // every F of the table is < 2^500: div_rn_recip applies (k_physics.cuh)
  int pow_fma;        // the host glibc's pow variant the device reproduces: 1 __pow_fma, 0 __pow_sse2
  uint32_t expect_cells;  // cells the level expansion must place (cycle check); 0 = no check
  // ensemble statistics (lemgpu_stats_enable): k_stats_pass reduces {sum,
  // max, min} of the step's new elevation over st_chunks fixed chunks per
  // member into st_part[(m * st_chunks + chunk) * 3]; k_stats_fold folds them
  // into st_table rows [st_member0, st_member0 + M) of 4 doubles
  double* st_part;
  double* st_table;
  uint32_t st_chunks;
  uint32_t st_member0;
  // k_esc_forest (k_forest.cuh): 0 off, 1 when >= 1/4 of the cells escape, 2 always (EX only)
  int esc_forest;
  int phclk;         // lemgpu_options::phase_clocks: lem::Phase seconds (the tile pass's phase clocks)
  uint32_t* fbins;   // [owner CTA][depth] counts / cursors (the global path's levels array, N + 2)
  uint32_t cb_cap;   // entries of cbound (k_esc_forest: level starts)
  double* hx;        // position-major elevations (k_esc_forest)
  // MFD routing (k_mfd.cuh; mfd_A != nullptr: the erosion reads this drainage area)
  double* mfd_A;      // cell-major MFD drainage area
  double* mfd_wsum;   // cell-major sum of the receiver weights
  uint8_t* mfd_lm;    // cell-major mask of strictly lower neighbours (the MFD receivers)
  uint32_t* mfd_rem;  // receiver countdown of the dependency-counting plan
  uint32_t* mfd_ord;  // the MFD plan, level-major (any order within a level)
  uint32_t* mfd_lv;   // its level starts
  uint32_t* mfd_lev;  // cell-major level (for the export)
  double mfd_exp;     // StepSetup::mfd_exponent
  uint32_t* mfd_wl;     // k_mfd_tiles: two work lists of tiles (pass parity), ntiles each
  uint32_t* mfd_stamp;  // ... per tile: the pass it is queued for
  int mfd_all;          // ... 1: this launch is pass 0 (every tile)
  uint8_t* dbg_level;  // debug capture (nullptr: off): level of every cell k_tiles finishes (escaped: untouched)
  double* dbg_A;       // ... and its drainage area
  Ctl* ctl;
  lemgpu_diag* diag;  // ring of per-step diagnostics (slot = ctl->slot)
  cudaGraphConditionalHandle h_expand, h_dacc, h_deros, h_mfd, h_esc;
  int esc_if;  // 1: the escape kernels after k_esc_small sit in a graph IF node on h_esc
};

// ---------------------------------------------------------------- helpers

__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

__device__ __forceinline__ void timeline(Ctl* ctl) {
  const uint32_t i = ctl->ntl;
  if (i < 96) {
    ctl->tl[i] = globaltimer();
    ctl->ntl = i + 1;
  }
}

// ---------------------------------------------------------------- phase clocks
// lem::Phase busy time (PhaseTimings, simulation.hpp:19-32).  The kernels fuse
// phases (k_recv: receivers + donors; k_tiles / k_esc_small: order,
// accumulation, uplift, erosion) and overlap (receiver bands beside tile
// bands), so the phases are not kernel spans: thread 0 of every CTA charges
// the SM cycles between its phase boundaries (taken where a block barrier
// closes a phase) to that phase, in shared memory, and adds them to the
// step's totals when the CTA ends.  k_finalize splits the step's device time
// (first kernel start to k_finalize) in these proportions: the six slots add
// up to the step and say where the SMs spent it.
struct PhClk {
  uint32_t last;  // 32-bit SM clock (%clock): deltas between marks are far below 2^32 cycles
  uint32_t pad;
  unsigned long long acc[6];
};
#ifdef LEMGPU_NO_PHCLK
#define LEMGPU_PHCLK_ON 0
#else
#define LEMGPU_PHCLK_ON 1
#endif
__device__ __forceinline__ void phclk_begin(PhClk& c) {
  if (LEMGPU_PHCLK_ON && threadIdx.x == 0) {
    c.last = (uint32_t)clock();
#pragma unroll
    for (int i = 0; i < 6; ++i) c.acc[i] = 0;
  }
}
__device__ __forceinline__ void phclk_mark(PhClk& c, int ended) {
  if (LEMGPU_PHCLK_ON && threadIdx.x == 0) {
    const uint32_t n = (uint32_t)clock();
    c.acc[ended] += n - c.last;
    c.last = n;
  }
}
__device__ __forceinline__ void phclk_end(PhClk& c, int ended, Ctl* ctl) {
  if (LEMGPU_PHCLK_ON && threadIdx.x == 0) {
    phclk_mark(c, ended);
    // spread over 32 slots: tens of thousands of CTAs (k_recv) would
    // otherwise serialise on six addresses
    unsigned long long* slot = ctl->ph_cyc[(blockIdx.x + blockIdx.y * 7u) & 31u];
#pragma unroll
    for (int i = 0; i < 6; ++i)
      if (c.acc[i]) atomicAdd(slot + i, c.acc[i]);
  }
}

// A kernel that is one phase: thread 0's cycles from construction to scope exit.
struct PhWhole {
  Ctl* ctl;
  int ph;
  unsigned long long t0;
  __device__ __forceinline__ PhWhole(Ctl* c, int p) : ctl(c), ph(p), t0(0) {
    if (threadIdx.x == 0) t0 = (unsigned long long)clock64();
  }
  __device__ __forceinline__ ~PhWhole() {
    if (threadIdx.x == 0) atomicAdd(&ctl->ph_cyc[blockIdx.x & 31u][ph], (unsigned long long)clock64() - t0);
  }
};

// True in every thread of exactly one CTA: the last CTA of the grid to get
// here (all others have finished their work and fenced it).  The caller's
// finisher code then sees every CTA's global writes.  Resets the counter.
__device__ __forceinline__ bool last_block_done(Ctl* ctl) {
  __shared__ uint32_t s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const uint32_t nb = gridDim.x * gridDim.y * gridDim.z;
    const uint32_t prev = atomicAdd(&ctl->done, 1u);
    s_last = (prev == nb - 1) ? 1u : 0u;
    if (s_last) {
      ctl->done = 0;
      __threadfence();
    }
  }
  __syncthreads();
  return s_last != 0;
}

// Exclusive block scan of one u32 per thread; *total gets the block sum.
// scratch: kNW+1 u32 of shared memory; contains the barriers it needs.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, uint32_t* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) scratch[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < kNW ? scratch[lane] : 0u;
#pragma unroll
    for (int o = 1; o < kNW; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < kNW) scratch[lane] = w;
  }
  __syncthreads();
  const uint32_t warp_excl = warp ? scratch[warp - 1] : 0u;
  *total = scratch[kNW - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// Loop condition of the step graph (0: level expansion, 1: deep
// accumulation, 2: deep erosion, 3: MFD tail rounds, 4: escape kernels after k_esc_small): a graph conditional when the step is a
// CUDA graph, a control-block word when it runs eagerly (profiling).
__device__ __forceinline__ void set_cond(const StepArgs& a, int which, unsigned v) {
  if (a.eager) {
    a.ctl->cond[which] = v;
  } else {
    const cudaGraphConditionalHandle h = which == 0 ? a.h_expand : which == 1 ? a.h_dacc : which == 2 ? a.h_deros
                                         : which == 3 ? a.h_mfd : a.h_esc;
    cudaGraphSetConditional(h, v);
  }
}

// donors_of (flow_graph.hpp:64-72) as a stencil bitmask: neighbour k drains
// here when its receiver code is 7-k.  From the materialised mask, or from the
// receiver codes of the neighbours (off-raster neighbours are skipped, and the
// perimeter rows separating stacked members never drain anywhere).
__device__ __forceinline__ uint32_t donor_mask_at(const StepArgs& a, uint32_t c) {
  if (a.dmask_valid) return __ldg(a.dmask + c);
  const uint32_t y = c / a.W, x = c - y * a.W;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!dir_in(a.conn, k)) continue;
    const uint32_t nx = x + dir_ox(k), ny = y + dir_oy(k);
    if (nx >= a.W || ny >= a.Htot) continue;
    if (__ldg(a.rcode + (size_t)ny * a.W + nx) == (uint8_t)(7 - k)) m |= 1u << k;
  }
  return m;
}

// donor_mask_at for a cell below level 0: it has a receiver, so it is interior
// and all 8 neighbours exist -- the 8 code loads go out together, no bounds
// tests (the global level path's dmask when it is materialised).
__device__ __forceinline__ uint32_t donor_mask_interior(const StepArgs& a, uint32_t c) {
  if (a.dmask_valid) return __ldg(a.dmask + c);
  const uint8_t* r = a.rcode + c;
  const int W = (int)a.W;
  uint32_t v[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) v[k] = dir_in(a.conn, k) ? (uint32_t)__ldg(r + dir_ox(k) + dir_oy(k) * W) : 0xFFu;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) m |= (v[k] == (uint32_t)(7 - k) ? 1u : 0u) << k;
  return m;
}

// Barrier of a grid whose CTAs are all resident (cooperative launch): the
// last CTA to arrive releases the others by bumping the generation.
__device__ __forceinline__ void grid_barrier(Ctl* ctl) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t nb = gridDim.x * gridDim.y * gridDim.z;
    const uint32_t gen = ld_volatile_u32(&ctl->gbar_gen);
    __threadfence();
    if (atomicAdd(&ctl->gbar_count, 1u) == nb - 1) {
      ctl->gbar_count = 0;
      __threadfence();
      atomicAdd(&ctl->gbar_gen, 1u);
    } else {
      while (ld_volatile_u32(&ctl->gbar_gen) == gen) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ bool is_interior(const StepArgs& a, uint32_t c) {
  const uint32_t y = c / a.W, x = c - y * a.W, yl = y % a.H;
  return x > 0 && x < a.W - 1 && yl > 0 && yl < a.H - 1;
}

}  // namespace lemgpu
