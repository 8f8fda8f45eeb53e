// k_tiles.cuh -- one whole timestep per raster tile: the fast path.
//
//   steepest_receiver  proj/include/lem/flow_graph.hpp:44-59
//   donors_of          proj/include/lem/flow_graph.hpp:64-72
//   generate_queue     proj/src/traversal.cpp:19-48 (per private queue, as in
//                      step_private_queues, proj/src/scheduler.cpp:269-392)
//   accumulate_into    proj/src/accumulation.cpp:7-17, accumulation.hpp:21-28
//   uplift             proj/src/erosion.cpp:52-57
//   erode_one_cell     proj/src/erosion.cpp:36-50 (+ newton_erode_cell :19-34)
//
// Every cell drains along its receivers to exactly one level-0 cell (a pit or
// a perimeter cell), so the raster is a forest and the trees are independent:
// a step only needs, per tree, its cells grouped by level (the paper's
// breadth-first level ordering) to accumulate
// upstream->downstream and to erode downstream->upstream.  The reference's
// fastest strategy (rb_private_queues) exploits exactly this with one private
// queue per worker over a slice of the sources; here the private queue
// belongs to a CTA and the sources are the level-0 cells of a 64x32 tile.
//
// k_recv has already written, for every cell, the receiver code and the four
// bit planes of the code (donor masks are derived from the codes where
// needed).  A CTA (persistent, looping over tiles) does, for its tile T:
//   1. one TMA box brings h for the BFS domain (T grown by kHalo cells); the
//      codes of the domain and the ring around it are loaded, and the code
//      bit planes are shifted to the window's word grid;
//   2. bitmaps: domain cells with a receiver, T's level-0 cells (code 8), and
//      the border cells that have a donor in the ring (outside the domain);
//   3. breadth first from T's level-0 cells: level l+1 = the domain cells
//      whose receiver is in level l, one bitmap pass per level (shift + and
//      per direction), listed level-major (block prefix of the word counts):
//      the level structure of the reference's TraversalPlan for T's sources;
//   4. drainage area: exact cell counts (every cell adds 1 to each ancestor;
//      integer adds commute) or, for a cell area that is not exact, the
//      reference's FP pull in slot order level by level;
//   5. uplift + implicit erosion level by level (block barrier per level),
//      each cell reading its receiver's already updated elevation; the new
//      elevations go to hout.
// A tree with a cell whose donor lies outside the domain (its cells reach
// more than 3 cells beyond T; 0.3 % of the cells of a fresh random-noise DEM, ~2.5 % after some steps) or
// deeper than kTMaxLev ESCAPES: none of its cells is written, its root is
// appended to a list, and the level-synchronous global path (k_order.cuh +
// k_physics.cuh) finishes it after this kernel.  h is read-only during the
// step (hout is the other ping-pong buffer), so the stencil of any CTA sees
// the complete previous surface no matter which trees other CTAs finished.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "k_order.cuh"
#include "k_physics.cuh"
#include "k_recv_donor.cuh"

namespace lemgpu {

// Window coordinates: column x, row y; q = y * kWP + x; global cell =
// (wx0 + x, wy0 + y).  The tile T is columns [kLX, kLX+kTX) x rows [kLY,
// kLY+kTY); the BFS domain is T grown by kHalo; the receiver codes of the
// ring around the domain tell which domain cells have donors outside it.
constexpr int kWP = 72;             // window pitch = TMA box width (doubles): the ring columns exactly
constexpr int kLX = kHalo + 1;      // first tile column in the window
constexpr int kLY = kHalo + 2;      // first tile row in the window
constexpr int kWY = kTY + 2 * kLY;  // window rows
constexpr int kDX0 = kLX - kHalo, kDX1 = kLX + kTX + kHalo;  // domain columns [kDX0, kDX1)
constexpr int kDY0 = kLY - kHalo, kDY1 = kLY + kTY + kHalo;  // domain rows
constexpr int kDW = kDX1 - kDX0, kDH = kDY1 - kDY0;
constexpr int kQ0 = kDY0 * kWP;          // q of the first domain row
constexpr int kDN = kDH * kWP;           // per-cell arrays: the domain rows
constexpr int kRN = (kDH + 2) * kWP;     // receiver codes: the domain rows and the ring rows
constexpr int kCap = kDW * kDH;          // queue: every domain cell at most once
constexpr int kTMaxLev = 64;             // deeper trees escape
// measured (round 2, after the counts overlap; 10000^2 ms/step): BFS 32 / 48 /
// 64 with ERO 0: 2.032 / 2.026 / 2.028; ERO 8 / 16 / 32 with BFS 32: 2.044 /
// 2.046 / 2.048 -- the one-warp erosion tail no longer pays
#ifndef LEMGPU_SMALL_BFS
#define LEMGPU_SMALL_BFS 48
#endif
#ifndef LEMGPU_SMALL_ERO
#define LEMGPU_SMALL_ERO 0
#endif
constexpr int kSmallLevel = LEMGPU_SMALL_BFS;  // levels this small are expanded by one warp
constexpr int kSmallEro = LEMGPU_SMALL_ERO;    // erosion levels this small (in total) run on one warp
static_assert(kLX % 4 == 0 && kWP % 4 == 0 && kDX1 + 1 <= kWP, "window geometry");
static_assert(kWY * kWP < 65535, "16-bit window indices");
static_assert(kDN % 4 == 0, "vector fills of the per-cell arrays");

// Bitmaps of the window: row y, 32-column word w (columns 32w .. 32w+31).
constexpr int kBW = 3;            // words per row (96 >= kWP columns)
constexpr int kBN = kWY * kBW;    // words per bitmap
constexpr int kBPairs = kDH * kBW;  // (row, word) pairs of the domain rows
constexpr int kBWarps = (kBPairs + 31) / 32;  // warps holding them
static_assert(kBW * 32 >= kWP && kBPairs <= kTTPB && (kDH + 2) * kBW <= kTTPB, "bitmap geometry");

// EX: the drainage area is an exact multiple of the cell area (lut_exact), so
// it is carried as an integer cell count and indexes the host-libm F table
// directly; otherwise it is the reference's FP sum (f64).
template <bool EX>
struct TileSmem {
  double hw[kDN];  // h of the domain rows (TMA destination), updated in place by the erosion
  alignas(16) typename std::conditional<EX, uint32_t, double>::type acc[kDN];  // drainage area: cell count (EX) or FP sum
  uint16_t list[kCap];         // the tile's queue, level-major
  uint8_t rc[kRN];             // receiver codes of the domain and ring rows
  alignas(16) uint8_t esc[EX ? 16 : kDN];  // the cell's tree escapes (FP path; EX: bit 31 of acc) (set on roots, inherited downstream -> upstream)
  uint8_t rowint[kWY];         // window row holds interior cells
  uint32_t pl[3][kBN];         // bit planes 0-2 of the receiver codes, aligned to the window
  uint32_t vr[kBN];            // domain cells with a receiver (code < 8)
  uint32_t lk[kBN];            // domain cells with a donor outside the domain
  uint32_t wsum[2][kTTPB / 32];  // per-warp level counts (double-buffered by level parity)
  uint32_t lv[2][kBN];         // current / next level
  uint32_t lvs[kTMaxLev + 1];  // first queue position of each level
  uint64_t bar;
};
template <bool EX>
constexpr size_t tiles_smem_bytes() { return sizeof(TileSmem<EX>); }

// Window-index offset of direction k (0..7, stencil order): one byte permute
// of the packed table (offset + 128 per byte).
constexpr uint32_t woff_b(int k) { return (uint32_t)(128 + dir_ox(k) + dir_oy(k) * kWP); }
constexpr uint32_t kWOffLo = woff_b(0) | woff_b(1) << 8 | woff_b(2) << 16 | woff_b(3) << 24;
constexpr uint32_t kWOffHi = woff_b(4) | woff_b(5) << 8 | woff_b(6) << 16 | woff_b(7) << 24;
__device__ __forceinline__ int woff(uint32_t k) { return (int)(__byte_perm(kWOffLo, kWOffHi, k) & 0xFFu) - 128; }

// F = ((K*dt) * pow(A, m)) / pow(dist, n) (erosion.cpp:38-39) from the host
// libm table when A is an exact multiple of the cell area, else with the
// device restatement of the host glibc pow (identical bits).
__device__ __forceinline__ double tile_F(const StepArgs& a, uint32_t mem, uint32_t cls, double A,
                                         uint32_t& misses) {
  const double q = a.w0_is_one ? A : __ddiv_rn(A, a.w0);
  if (a.lut_exact && q < (double)a.lut_entries && q == floor(q) && (!a.mfd_A || a.w0_is_one))
    return __ldg(a.ftab + ((size_t)mem * 3 + cls) * a.lut_entries + (uint32_t)q);
  ++misses;
  const double pd = cls == 0 ? a.powdist_h : cls == 1 ? a.powdist_v : a.powdist_d;
  return __ddiv_rn(__dmul_rn(__ldg(a.kdt + mem), glibc_pow_dev(a.pow_fma, A, __ldg(a.mexp + mem))), pd);
}

// Drainage area of a tile cell for the debug capture: count (escape mark in
// bit 31 dropped) x cell area, or the FP sum itself.
template <bool EX, typename T>
__device__ __forceinline__ double dbg_area(T v, double w0) {
  if constexpr (EX)
    return __dmul_rn((double)(v & 0x7FFFFFFFu), w0);
  else
    return (double)v;
}

// MF (routing = kMfd, with EX's layout): the erosion reads the MFD drainage
// area from global memory (final before this kernel: k_mfd_tiles); no counts.
// PH: lem::Phase clocks (lemgpu_options::phase_clocks); their marks sit on the
// barrier-separated critical paths (measured 1.4 % of a 10000^2 step).
template <int CONN, int NK, bool EX, bool MF = false, bool PH = true>
__global__ void __launch_bounds__(kTTPB, EX ? LEMGPU_TILE_MINB : 2) k_tiles(StepArgs a, const __grid_constant__ CUtensorMap hmap) {
  extern __shared__ __align__(128) unsigned char smraw[];
  TileSmem<EX>& s = *reinterpret_cast<TileSmem<EX>*>(smraw);
  __shared__ PhClk s_pc;
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->err_flag)) return;  // an earlier step failed (uniform)
  if constexpr (PH) phclk_begin(s_pc);
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const int W = (int)a.W, Ht = (int)a.Htot;
  const uint32_t ntx = (a.W + kTX - 1) / kTX, nty = (a.Htot + kTY - 1) / kTY;
  const uint32_t ntiles = ntx * nty;
  const uint32_t E = a.lut_entries;
  const bool tab = EX && NK == 1 && a.tab_ok && !MF;
  if (tid == 0) {
    atomicMin(&ctl->t_t_begin, globaltimer());
    if (a.use_tma) mbar_init(&s.bar, 1);
  }
  // the escape path's level-0 and level-1 bins start at zero
  for (uint32_t i = blockIdx.x * kTTPB + tid; i < 2 * a.scan_grid; i += gridDim.x * kTTPB) a.bins[i] = 0;

#define HW(q) s.hw[(q) - kQ0]
#define ACC(q) s.acc[(q) - kQ0]
// escape mark of a cell: bit 31 of its cell count (EX), else its own byte
#define ESC_GET(q) (EX ? ((uint32_t)s.acc[(q) - kQ0] >> 31) : (uint32_t)s.esc[(q) - kQ0])
#define ESC_SET(q)                                                    \
  do {                                                                \
    if (EX)                                                           \
      reinterpret_cast<uint32_t*>(s.acc)[(q) - kQ0] |= 0x80000000u;   \
    else                                                              \
      s.esc[(q) - kQ0] = 1;                                           \
  } while (0)
#define RC(q) s.rc[(q) - (kDY0 - 1) * kWP]
  uint32_t iters = 0;               // per thread and tile (cells of the tile x max_newton_iters < 2^32)
  unsigned long long iters64 = 0;  // per thread
  uint32_t misses = 0, cells = 0, n0i = 0, maxl = 0;
  uint32_t phase = 0;
  const uint32_t t_end = a.t_hi ? a.t_hi : ntiles;  // banded host steps launch one band of tile rows at a time
  for (uint32_t t = a.t_lo + blockIdx.x; t < t_end; t += gridDim.x, phase ^= 1u) {
    const int tx0 = (int)(t % ntx) * kTX, ty0 = (int)(t / ntx) * kTY;
    const int wx0 = tx0 - kLX, wy0 = ty0 - kLY;
    const uint32_t gbase = (uint32_t)wy0 * a.W + (uint32_t)wx0;  // global index of window (0, 0), mod 2^32
    // global cell of window index q (mod 2^32 arithmetic)
    auto gcell = [&](uint32_t q) {
      const uint32_t y = q / kWP;
      return gbase + q + y * (a.W - (uint32_t)kWP);
    };
    iters64 += iters;
    iters = 0;
    __syncthreads();  // the previous tile is finished with every shared array
    if (tid == 0 && a.use_tma) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes of hw before the TMA overwrite
      mbar_expect_tx(&s.bar, (uint32_t)sizeof(s.hw));
      tma_load_2d(s.hw, &hmap, wx0, wy0 + kDY0, &s.bar);  // out-of-raster cells arrive as 0
    }
    if (!a.use_tma) {
      for (int i = (int)tid; i < kDN; i += kTTPB) {
        const int y = kDY0 + i / kWP, x = i % kWP;
        const int gx = wx0 + x, gy = wy0 + y;
        s.hw[i] = (gx >= 0 && gx < W && gy >= 0 && gy < Ht) ? __ldg(a.h + (size_t)gy * W + gx) : 0.0;
      }
    }
    // receiver codes of rows kDY0-1 .. kDY1 from k_recv's output
    // (asynchronous 4-byte copies, cp.async); cells outside the raster read as NoFlow
    for (int i = (int)tid; i < kRN / 4; i += kTTPB) {
      const int y = kDY0 - 1 + (4 * i) / kWP, x = (4 * i) % kWP;
      const int gx = wx0 + x, gy = wy0 + y;
      uint32_t* dst = reinterpret_cast<uint32_t*>(s.rc) + i;
      if (gy >= 0 && gy < Ht && gx >= 0 && gx + 3 < W && (a.W & 3u) == 0) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)),
                     "l"(a.rcode + (size_t)gy * a.W + gx)
                     : "memory");
      } else {
        uint32_t v = 0x08080808u;
        if (gy >= 0 && gy < Ht) {
          const size_t g = (size_t)gy * a.W + gx;
          v = 0;
          for (int j = 0; j < 4; ++j) {
            const bool in = gx + j >= 0 && gx + j < W;
            v |= (in ? (uint32_t)a.rcode[g + j] : 8u) << (8 * j);
          }
        }
        *dst = v;
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // escape marks 0, cell counts 1 (EX) for the whole domain
    if (!EX)
      for (int i = (int)tid; i < kDN / 4; i += kTTPB) reinterpret_cast<uint32_t*>(s.esc)[i] = 0u;
    if (EX)
      for (int i = (int)tid; i < kDN / 4; i += kTTPB)
        reinterpret_cast<uint4*>(&s.acc[0])[i] = make_uint4(1u, 1u, 1u, 1u);
    // bit planes 0-2 of the codes, shifted to the window's columns (rows kDY0-1 .. kDY1);
    // outside the raster every plane reads 1 (code 15)
    if (tid < (uint32_t)((kDH + 2) * kBW)) {
      const int yy = (int)tid / kBW, w = (int)tid % kBW, y = kDY0 - 1 + yy;
      const int gy = wy0 + y, gx = wx0 + 32 * w;
      const int j = gx >> 5, sh = gx & 31;
      uint32_t pw[4];
#pragma unroll
      for (int pl = 0; pl < 4; ++pl) {
        const uint32_t* row = a.planes + ((size_t)pl * a.Htot + (gy >= 0 && gy < Ht ? gy : 0)) * a.W32;
        const bool rin = gy >= 0 && gy < Ht;
        const uint32_t lo = (rin && j >= 0 && j < (int)a.W32) ? __ldg(row + j) : ~0u;
        const uint32_t hi = (rin && j + 1 >= 0 && j + 1 < (int)a.W32) ? __ldg(row + j + 1) : ~0u;
        pw[pl] = sh ? __funnelshift_r(lo, hi, sh) : lo;
      }
      const int o = y * kBW + w;
      s.pl[0][o] = pw[0];
      s.pl[1][o] = pw[1];
      s.pl[2][o] = pw[2];
      // domain cells with a receiver, and the tile's level-0 cells (code 8)
      const uint32_t dom = (y >= kDY0 && y < kDY1) ? (w == 0 ? (~0u << kDX0) : w == 1 ? ~0u : ((1u << (kDX1 - 64)) - 1u)) : 0u;
      const uint32_t til = (y >= kLY && y < kLY + kTY) ? (w == 0 ? (~0u << kLX) : w == 1 ? ~0u : ((1u << (kLX + kTX - 64)) - 1u)) : 0u;
      s.vr[o] = ~pw[3] & dom;
      s.lv[0][o] = pw[3] & ~pw[0] & ~pw[1] & ~pw[2] & til;
      s.lv[1][o] = 0u;  // rows outside the domain stay empty in both level buffers
      s.lk[o] = 0u;
    }
    if (tid < (uint32_t)kWY) {
      const int gy = wy0 + (int)tid;
      uint8_t ok = 0;
      if (gy >= 0 && gy < Ht) {
        const uint32_t yl = (uint32_t)gy % a.H;
        ok = yl > 0 && yl < a.H - 1;
      }
      s.rowint[tid] = ok;
    }
    if (tid < (uint32_t)(2 * kBW)) {  // rows 0 and kWY-1: never part of a level
      const int o = (tid < kBW ? 0 : (kWY - 1) * kBW) + (int)(tid % kBW);
      s.lv[0][o] = s.lv[1][o] = 0u;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");  // this thread's code copies have landed
    __syncthreads();
    // domain cells on the border with a donor in the ring outside the domain:
    // one thread per border cell, checking only its ring neighbours
    for (uint32_t bi = tid; bi < (uint32_t)(2 * kDW + 2 * (kDH - 2)); bi += kTTPB) {
      int x, y;
      uint32_t ring;  // directions whose neighbour lies in the ring
      if (bi < (uint32_t)kDW) {
        x = kDX0 + (int)bi, y = kDY0, ring = 0x07u;
      } else if (bi < (uint32_t)(2 * kDW)) {
        x = kDX0 + (int)bi - kDW, y = kDY1 - 1, ring = 0xE0u;
      } else if (bi < (uint32_t)(2 * kDW + kDH - 2)) {
        x = kDX0, y = kDY0 + 1 + (int)bi - 2 * kDW, ring = 0x29u;
      } else {
        x = kDX1 - 1, y = kDY0 + 1 + (int)bi - 2 * kDW - (kDH - 2), ring = 0x94u;
      }
      if (x == kDX0) ring |= 0x29u;
      if (x == kDX1 - 1) ring |= 0x94u;
      if (CONN == 4) ring &= 0x5Au;
      const int q = y * kWP + x;
      bool leak = false;
      for (uint32_t m = ring; m; m &= m - 1) {
        const uint32_t k = __ffs(m) - 1;
        leak |= RC(q + woff(k)) == (uint8_t)(7 - k);
      }
      if (leak) atomicOr(&s.lk[y * kBW + (x >> 5)], 1u << (x & 31));
    }
    if (a.use_tma) mbar_wait(&s.bar, phase);
    __syncthreads();
    // ---- 5. the levels, breadth first from the tile's roots: level l+1 =
    // the domain cells whose receiver is in level l (one bitmap pass per
    // level: shift + and per direction), listed level-major (block prefix of
    // the word counts); a tree reaching a cell with a leaking donor escapes
    // (its root is marked)
    // Once a level has at most kSmallLevel cells, warp 0 continues alone from
    // the queue (children = neighbours whose code points back), with warp
    // barriers only.
    uint32_t nl = 0, qpos = 0;
    bool warp_mode = false;
    for (uint32_t l = 0;; ++l) {
      const uint32_t* cur = s.lv[(l + 1) & 1];  // level l-1 (level 0: the roots, in lv[0])
      uint32_t* nxt = s.lv[l & 1];              // level l
      uint32_t word = 0, y = 0, w = 0, incl = 0, cnt = 0;
      uint32_t* ws = s.wsum[l & 1];
      if (tid < (uint32_t)kBWarps * 32) {
        if (tid < (uint32_t)kBPairs) {
          y = kDY0 + tid / kBW;
          w = tid - (y - kDY0) * kBW;
          const uint32_t o = y * kBW + w;
          if (l == 0) {
            word = nxt[o];
          } else {
            // S_k(cur): bit x of row y = bit x + ox_k of row y + oy_k
            uint32_t sh[3][3];  // [oy+1][ox+1]
            uint32_t any = 0;
#pragma unroll
            for (int oy = -1; oy <= 1; ++oy) {
              const uint32_t* row = cur + (y + oy) * kBW;
              const uint32_t c = row[w], lo = w > 0 ? row[w - 1] : 0u, hi = w + 1 < (uint32_t)kBW ? row[w + 1] : 0u;
              sh[oy + 1][0] = (c << 1) | (lo >> 31);
              sh[oy + 1][1] = c;
              sh[oy + 1][2] = (c >> 1) | (hi << 31);
              any |= c | lo | hi;
            }
            if (any) {
              const uint32_t p0 = s.pl[0][o], p1 = s.pl[1][o], p2 = s.pl[2][o];
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                if (!dir_in(CONN, k)) continue;
                const uint32_t rk = ((k & 1) ? p0 : ~p0) & ((k & 2) ? p1 : ~p1) & ((k & 4) ? p2 : ~p2);
                word |= rk & sh[dir_oy(k) + 1][dir_ox(k) + 1];
              }
              word &= s.vr[o];
            }
          }
        }
        cnt = __popc(word);
        incl = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t yv = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= (uint32_t)o) incl += yv;
        }
        if (lane == 31) ws[tid >> 5] = incl;
        if (l > 0 && tid < (uint32_t)kBPairs) nxt[y * kBW + w] = word;
      }
      __syncthreads();
      uint32_t wbase = 0, tot = 0;
#pragma unroll
      for (int i = 0; i < kBWarps; ++i) {
        const uint32_t v = ws[i];
        wbase += i < (int)(tid >> 5) ? v : 0u;
        tot += v;
      }
      if (tot == 0) break;
      if (tid == 0) s.lvs[l] = qpos;
      if (tid < (uint32_t)kBPairs) {
        uint32_t pos = qpos + wbase + incl - cnt;
        const uint32_t leaks = word & s.lk[y * kBW + w];
        const uint32_t qw = y * kWP + 32 * w;
        while (word) {
          const uint32_t b = __ffs(word) - 1;
          word &= word - 1;
          s.list[pos++] = (uint16_t)(qw + b);
        }
        for (uint32_t lb = leaks; lb; lb &= lb - 1) {  // a donor outside the domain: the tree escapes
          uint32_t r = qw + __ffs(lb) - 1, code = RC(r);
          while (code != kNoFlowCode) {
            r = (uint32_t)((int)r + woff(code));
            code = RC(r);
          }
          ESC_SET(r);
        }
      }
      qpos += tot;
      nl = l + 1;
      if (l + 1 == (uint32_t)kTMaxLev) break;
      if (tot <= (uint32_t)kSmallLevel && kSmallLevel > 0) {
        warp_mode = true;
        break;
      }
    }
    // EX: the cell counts of the levels listed so far need only the receiver
    // codes, so while warp 0 lists the deep levels alone the other warps
    // already walk those cells' ancestors (cnt_from: where the counts go on)
    uint32_t cnt_from = 0;
    if (warp_mode) {
      __syncthreads();  // the last block level is listed
      if (EX && !MF && tid >= 32) {
        const uint32_t lv1 = nl > 1 ? s.lvs[1] : qpos;
        for (uint32_t i = lv1 + tid - 32; i < qpos; i += kTTPB - 32) {
          uint32_t p = s.list[i], code = RC(p);
          do {
            p = (uint32_t)((int)p + woff(code));
            atomicAdd(reinterpret_cast<uint32_t*>(&ACC(p)), 1u);
            code = RC(p);
          } while (code != kNoFlowCode);
        }
      }
      cnt_from = qpos;
      if (tid < 32) {
        uint32_t fs = s.lvs[nl - 1];  // frontier: level nl-1
        for (;;) {
          const uint32_t fe = qpos;
          uint32_t run = 0;
          for (uint32_t j0 = fs; j0 < fe; j0 += 32) {
            const uint32_t i = j0 + lane;
            uint32_t f = 0, kids = 0;
            if (i < fe) {
              f = s.list[i];
              const uint32_t fy = f / kWP, fx = f - fy * kWP;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                if (!dir_in(CONN, k)) continue;
                const uint32_t nx = fx + dir_ox(k), ny = fy + dir_oy(k);
                if (nx - kDX0 >= (uint32_t)kDW || ny - kDY0 >= (uint32_t)kDH) continue;
                if (RC(f + woff(k)) == (uint8_t)(7 - k)) kids |= 1u << k;
              }
            }
            const uint32_t c = __popc(kids);
            uint32_t inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const uint32_t yv = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= (uint32_t)o) inc += yv;
            }
            uint32_t pos = qpos + run + inc - c;
            while (kids) {
              const uint32_t k = __ffs(kids) - 1;
              kids &= kids - 1;
              const uint32_t q = (uint32_t)((int)f + woff(k));
              s.list[pos++] = (uint16_t)q;
              const uint32_t qy = q / kWP, qx = q - qy * kWP;
              if ((s.lk[qy * kBW + (qx >> 5)] >> (qx & 31)) & 1u) {
                uint32_t r = q, code = RC(q);
                while (code != kNoFlowCode) {
                  r = (uint32_t)((int)r + woff(code));
                  code = RC(r);
                }
                if (EX)  // atomically: the other warps' count adds may hit the same word
                  atomicOr(reinterpret_cast<uint32_t*>(s.acc) + (r - kQ0), 0x80000000u);
                else
                  ESC_SET(r);
              }
            }
            run += __shfl_sync(0xffffffffu, inc, 31);
          }
          if (run == 0) break;
          if (lane == 0) s.lvs[nl] = qpos;
          fs = qpos;
          qpos += run;
          ++nl;
          __syncwarp();
          if (nl == (uint32_t)kTMaxLev) break;
        }
        if (lane == 0) {
          s.lvs[nl] = qpos;
          s.wsum[0][0] = nl;
        }
      }
      __syncthreads();
      nl = s.wsum[0][0];
    } else {
      if (tid == 0) s.lvs[nl] = qpos;
      __syncthreads();
    }
    if (nl == (uint32_t)kTMaxLev) {
      // level kTMaxLev would not be empty: every tree reaching it escapes
      for (uint32_t i = s.lvs[nl - 1] + tid; i < s.lvs[nl]; i += kTTPB) {
        uint32_t r = s.list[i];
        bool kids = false;  // donors inside the domain (a donor outside already escaped the tree)
#pragma unroll
        for (int k = 0; k < 8; ++k) kids |= dir_in(CONN, k) && RC(r + woff(k)) == (uint8_t)(7 - k);
        if (!kids) continue;
        uint32_t code = RC(r);
        while (code != kNoFlowCode) {
          r = (uint32_t)((int)r + woff(code));
          code = RC(r);
        }
        ESC_SET(r);
      }
      __syncthreads();
    }
    if (a.force_escape) {
      for (uint32_t i = s.lvs[0] + tid; i < s.lvs[nl > 0 ? 1 : 0]; i += kTTPB) {
        const uint32_t q = s.list[i];
        if (a.force_escape == 1 || (gcell(q) & 1u)) ESC_SET(q);
      }
      __syncthreads();
    }
    // ---- 6. drainage area
    if constexpr (PH) phclk_mark(s_pc, LEMGPU_PHASE_ORDER);  // staging + the levels
    if (EX) {
      // cell counts: every cell adds 1 to each ancestor (integer adds commute)
      // (MF: the erosion reads the MFD drainage area, simulation.cpp:55-60)
      const uint32_t c0 = cnt_from ? cnt_from : s.lvs[1];
      for (uint32_t i = (nl > 1 && !MF ? c0 : 0u) + tid; i < (nl > 1 && !MF ? s.lvs[nl] : 0u); i += kTTPB) {
        uint32_t p = s.list[i], code = RC(p);
        do {
          p = (uint32_t)((int)p + woff(code));
          atomicAdd(reinterpret_cast<uint32_t*>(&ACC(p)), 1u);
          code = RC(p);
        } while (code != kNoFlowCode);
      }
      __syncthreads();
    } else {
      // deepest level first: A = w + the children's A in slot order (the
      // reference's FP summation order, accumulation.hpp:21-28)
      for (int l = (int)nl - 1; l >= 0; --l) {
        for (uint32_t i = s.lvs[l] + tid; i < s.lvs[l + 1]; i += kTTPB) {
          const uint32_t q = s.list[i];
          uint32_t m = 0;  // donors (slot order = stencil order), all inside the domain for a kept tree
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t n = (uint32_t)((int)q + woff(k)), ny = n / kWP, nx = n - ny * kWP;
            if (dir_in(CONN, k) && nx - kDX0 < (uint32_t)kDW && ny - kDY0 < (uint32_t)kDH && RC(n) == (uint8_t)(7 - k))
              m |= 1u << k;
          }
          double A = a.w0;
          while (m) {
            const uint32_t k = __ffs(m) - 1;
            m &= m - 1;
            A = __dadd_rn(A, (double)ACC((int)q + woff(k)));
          }
          ACC(q) = A;
        }
        __syncthreads();
      }
    }
    if constexpr (PH) phclk_mark(s_pc, LEMGPU_PHASE_ACCUM);
    // ---- 7. level 0: uplift interior sources (never eroded)
    // escaped roots -> the global level path (level 0 of its queue)
    for (uint32_t i0 = 0; i0 < (nl ? s.lvs[1] : 0u); i0 += kTTPB) {
      const uint32_t i = i0 + tid;
      bool e = false;
      uint32_t q = 0, gc = 0;
      if (i < s.lvs[1]) {
        q = s.list[i];
        gc = gcell(q);
        const uint32_t y = q / kWP, x = q - y * kWP;
        const int gx = wx0 + (int)x;
        const bool inter = s.rowint[y] && gx > 0 && gx < W - 1;  // interior NoFlow cell (simulation.cpp:42-44)
        n0i += inter ? 1u : 0u;
        e = ESC_GET(q) != 0;
        if (!e) {
          double hv = HW(q);
          if (inter) {
            hv = __dadd_rn(hv, a.du);
            HW(q) = hv;
          }
          a.hout[gc] = hv;
          ++cells;
        }
      }
      const uint32_t eb = __ballot_sync(0xffffffffu, e);
      if (eb) {
        const int ld = __ffs(eb) - 1;
        uint32_t p = 0;
        if (lane == (uint32_t)ld) p = atomicAdd(&ctl->nesc, (uint32_t)__popc(eb));
        p = __shfl_sync(0xffffffffu, p, ld);
        if (e) a.order[p + __popc(eb & ((1u << lane) - 1u))] = gc;
      }
    }
    __syncthreads();
    if constexpr (PH) phclk_mark(s_pc, LEMGPU_PHASE_UPLIFT);
    // erosion, downstream -> upstream, with the receiver's updated elevation
    auto erode = [&](uint32_t i) -> bool {
      const uint32_t q = s.list[i];
      const uint32_t code = RC(q);
      const uint32_t p = (uint32_t)((int)q + woff(code));
      if (ESC_GET(p)) {  // the tree escapes: inherit the mark, leave the cell to the level path
        ESC_SET(q);
        return false;
      }
      ++cells;
      uint32_t mem = 0;
      if (a.M > 1) mem = (uint32_t)(wy0 + (int)(q / kWP)) / a.H;
      const uint32_t cls = dir_class(code);  // class of dist(c, rec[c])
      const double h0 = __dadd_rn(HW(q), a.du);  // uplift (every cell below level 0 is interior)
      const double hn = HW(p);
      int itn;
      bool ok;
      double hnew;
      if (tab) {
        const double2 fy = __ldg(reinterpret_cast<const double2*>(a.ftab2) + (mem * 3 + cls) * E + (uint32_t)ACC(q));
        hnew = newton_n1_tab(h0, hn, fy.x, fy.y, a.eps, a.maxit, itn, ok);
      } else {
        double F;
        if (EX)
          F = MF ? tile_F(a, mem, cls, __ldg(a.mfd_A + gcell(q)), misses)
                 : __ldg(a.ftab + (mem * 3 + cls) * E + (uint32_t)ACC(q));
        else
          F = tile_F(a, mem, cls, (double)ACC(q), misses);
        if (NK == 1)
          hnew = newton_n1(h0, hn, F, a.eps, a.maxit, itn, ok);
        else
          hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, a.pow_fma, itn, ok);
      }
      const uint32_t gc = gcell(q);
      if (ok) {
        iters += (uint32_t)itn;
      } else {
        atomicMin(&ctl->err_cell, gc);
        ctl->err_slot = ctl->slot;
        atomicMax(&ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
      }
      HW(q) = hnew;
      a.hout[gc] = hnew;
      return true;
    };
    // the last levels, once at most kSmallLevel cells remain, by warp 0 alone
    uint32_t lw = nl;
    while (lw > 1 && s.lvs[nl] - s.lvs[lw - 1] <= (uint32_t)kSmallEro) --lw;
    for (uint32_t l = 1; l < lw; ++l) {
      bool any = false;
      for (uint32_t i = s.lvs[l] + tid; i < s.lvs[l + 1]; i += kTTPB) any |= erode(i);
      if (__syncthreads_or(any)) maxl = max(maxl, l + 1);
    }
    if (tid < 32) {
      for (uint32_t l = lw; l < nl; ++l) {
        bool any = false;
        for (uint32_t i = s.lvs[l] + lane; i < s.lvs[l + 1]; i += 32) any |= erode(i);
        if (__any_sync(0xffffffffu, any)) maxl = max(maxl, l + 1);
        __syncwarp();
      }
    }
    if (nl) maxl = max(maxl, 1u);
    if (a.dbg_level) {  // debug capture (lemgpu_debug_tile_capture): level and drainage area of the finished cells
      __syncthreads();  // escape marks are final (inherited during the erosion)
      for (uint32_t l = 0; l < nl; ++l)
        for (uint32_t i = s.lvs[l] + tid; i < s.lvs[l + 1]; i += kTTPB) {
          const uint32_t q = s.list[i];
          if (ESC_GET(q)) continue;
          a.dbg_level[gcell(q)] = (uint8_t)l;
          a.dbg_A[gcell(q)] = MF ? a.mfd_A[gcell(q)] : dbg_area<EX>(ACC(q), a.w0);
        }
    }
    if constexpr (PH) phclk_mark(s_pc, LEMGPU_PHASE_EROSION);
  }

  // ---- counters: one atomic per warp for the whole kernel
  iters64 += iters;
  for (int o = 16; o; o >>= 1) {
    iters64 += __shfl_down_sync(0xffffffffu, iters64, o);
    misses += __shfl_down_sync(0xffffffffu, misses, o);
    n0i += __shfl_down_sync(0xffffffffu, n0i, o);
    cells += __shfl_down_sync(0xffffffffu, cells, o);
  }
  if (lane == 0) {
    if (iters64) atomicAdd(&ctl->newton, iters64);
    if (misses) atomicAdd(&ctl->misses, misses);
    if (n0i) atomicAdd(&ctl->n0i, n0i);
    if (cells) atomicAdd(&ctl->tile_cells, cells);
  }
  if (tid == 0) atomicMax(&ctl->tile_nlev, maxl);
  __syncthreads();
  if constexpr (PH) phclk_end(s_pc, LEMGPU_PHASE_EROSION, ctl);
  if (tid == 0) atomicMax(&ctl->t_t_end, globaltimer());
}

#undef HW
#undef ACC
#undef RC
#undef ESC_GET
#undef ESC_SET

// Banded host steps: the final elevation of every cell of the escaped trees
// (the escape path wrote them after the bands were copied out), for the host
// to patch in.  count = cells placed by the escape path's level expansion.
// cells / vals / count are mapped pinned host memory (written over PCIe);
// more than cap cells: only the count is written.
__global__ void __launch_bounds__(kTPB) k_esc_gather(StepArgs a, uint32_t* cells, double* vals, uint32_t* count,
                                                     uint32_t cap) {
  const Ctl* ctl = a.ctl;
  // k_esc_small: the compact list of its cells in ppos; else the level path's queue
  const bool small = ctl->esc_small != 0;
  const uint32_t n = ctl->nesc && !ctl->err_flag ? (small ? ctl->esc_cells : a.levels[ctl->nlev]) : 0u;
  if (blockIdx.x == 0 && threadIdx.x == 0) *count = n;
  if (n > cap) return;
  for (uint32_t i = blockIdx.x * kTPB + threadIdx.x; i < n; i += gridDim.x * kTPB) {
    const uint32_t c = small ? a.ppos[i] : a.order[i];
    cells[i] = c;
    vals[i] = a.hout[c];
  }
}

// ---------------------------------------------------------------------------
// The escaped trees in shared memory: the roots are split evenly over the
// CTAs (kEscSmallPerSM per SM) and each CTA finishes its share of trees alone -- the
// same breadth-first levels (donor masks from the receiver codes), the
// reference's FP accumulation in slot order, uplift and erosion level by level
// -- with block barriers only, instead of the cooperative global path whose
// grid barrier per level dominates a small escape set.  A CTA whose share has
// more than kEscSmallRoots roots, kEscSmallCap cells or kEscSmallLev levels
// counts a failure; then the cooperative path runs for every escaped tree (the
// trees already written get the same bits again) and this kernel's counters
// are dropped.  Otherwise the last CTA marks the escape work done.
constexpr int kEscSmallRoots = 1024;
// cells per CTA share, CTAs per SM: measured (round 2) 6144 x 1 / 2048 x 3 /
// 1536 x 4 / 1024 x 6: 10000^2 2.033 / 2.020 / 2.020 / 2.037 ms/step, ens64
// 5.617 / 5.587 / 5.586 / 5.60 (a share beyond the capacity fails over to the
// cooperative path, exactly as before)
#ifndef LEMGPU_ESC_SMALL_CAP
#define LEMGPU_ESC_SMALL_CAP 2048
#define LEMGPU_ESC_SMALL_PER_SM 3
#endif
#ifndef LEMGPU_ESC_SMALL_PER_SM
#define LEMGPU_ESC_SMALL_PER_SM 1
#endif
constexpr int kEscSmallCap = LEMGPU_ESC_SMALL_CAP;
constexpr int kEscSmallPerSM = LEMGPU_ESC_SMALL_PER_SM;
constexpr int kEscSmallLev = 64;  // deeper shares fail early (deep plans belong to the cooperative path)
struct EscSmallSmem {
  double h[kEscSmallCap];  // the step's input elevation (staged at discovery), then the new one
  double A[kEscSmallCap];  // drainage area, then F
  double y[kEscSmallCap];  // n = 1: RN(1 / RN(1 + F)) for newton_n1_tab
  uint32_t cell[kEscSmallCap];
  uint16_t par[kEscSmallCap];  // parent slot (roots: 0xFFFF)
  uint16_t fc[kEscSmallCap];   // first child slot
  uint8_t kd[kEscSmallCap];    // direction parent -> cell
  uint8_t nk[kEscSmallCap];    // number of children
  uint32_t lvl[kEscSmallLev + 1];
  uint32_t scan[kNW + 1];
  uint32_t base, flag;
};
constexpr size_t kEscSmallSmemBytes = sizeof(EscSmallSmem);

template <int NK>
__global__ void __launch_bounds__(kTPB) k_esc_small(StepArgs a) {
  extern __shared__ __align__(128) unsigned char smraw[];
  EscSmallSmem& s = *reinterpret_cast<EscSmallSmem*>(smraw);
  __shared__ PhClk s_pc;
  phclk_begin(s_pc);
  Ctl* ctl = a.ctl;
  const uint32_t tid = threadIdx.x, G = gridDim.x;
  const uint32_t n = ld_volatile_u32(&ctl->nesc);  // 0 when an earlier step failed (k_tiles did not run)
  const uint32_t r0 = (uint32_t)((uint64_t)n * blockIdx.x / G), r1 = (uint32_t)((uint64_t)n * (blockIdx.x + 1) / G);
  const uint32_t nr = r1 - r0;
  bool ok = nr <= (uint32_t)kEscSmallRoots;
  uint32_t nl = 0;
  if (ok && nr > 0) {
    for (uint32_t i = tid; i < nr; i += kTPB) {
      const uint32_t c = a.order[r0 + i];
      s.cell[i] = c;
      s.par[i] = 0xFFFFu;
      // the elevation the step reads, copied asynchronously (consumed by the erosion)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&s.h[i])), "l"(a.h + c) : "memory");
    }
    if (tid == 0) {
      s.lvl[0] = 0;
      s.lvl[1] = nr;
    }
    __syncthreads();
    // breadth-first levels
    nl = 1;
    for (;;) {
      const uint32_t ls = s.lvl[nl - 1], le = s.lvl[nl];
      uint32_t carry = le;
      // the other CTAs' failure flag, loaded now so that its L2 round trip
      // overlaps this level's donor masks (published to the block below)
      const uint32_t fail_seen = tid == 0 ? ld_volatile_u32(&ctl->esc_fail) : 0u;
      for (uint32_t b0 = ls; b0 < le; b0 += kTPB) {
        const uint32_t i = b0 + tid;
        uint32_t m = 0;
        if (i < le) m = nl > 1 ? donor_mask_interior(a, s.cell[i]) : donor_mask_at(a, s.cell[i]);
        uint32_t tot;
        const uint32_t ex = block_excl_scan((uint32_t)__popc(m), &tot, s.scan);
        if (carry + tot > (uint32_t)kEscSmallCap) {
          ok = false;  // uniform: tot and carry are block-wide
          break;
        }
        if (i < le) {
          uint32_t c = carry + ex;
          s.fc[i] = (uint16_t)c;
          s.nk[i] = (uint8_t)__popc(m);
          const uint32_t cell = s.cell[i];
          while (m) {
            const uint32_t k = __ffs(m) - 1;
            m &= m - 1;
            const uint32_t cc = (uint32_t)((int)cell + dir_off(k, (int)a.W));
            s.cell[c] = cc;
            s.par[c] = (uint16_t)i;
            s.kd[c] = (uint8_t)k;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(&s.h[c])), "l"(a.h + cc)
                         : "memory");  // off every level's dependent chain
            ++c;
          }
        }
        carry += tot;
      }
      if (!ok) break;
      if (tid == 0) s.flag = fail_seen;
      __syncthreads();
      if (carry == le) break;  // the next level is empty
      if (s.flag) {  // another CTA already failed: the cooperative path will run (uniform: read after the barrier)
        ok = false;
        break;
      }
      if (nl == (uint32_t)kEscSmallLev) {
        ok = false;
        break;
      }
      if (tid == 0) s.lvl[nl + 1] = carry;
      ++nl;
      __syncthreads();
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");  // no copy in flight past here (a failed CTA exits)
  if (!ok) {
    if (tid == 0) atomicAdd(&ctl->esc_fail, 1u);
  } else if (nr > 0) {
    phclk_mark(s_pc, LEMGPU_PHASE_ORDER);
    // accumulation, deepest level first: A = w + the children's A in slot order
    for (int l = (int)nl - 1; l >= 0; --l) {
      for (uint32_t i = s.lvl[l] + tid; i < s.lvl[l + 1]; i += kTPB) {
        double A = a.w0;
        const uint32_t nk = l + 1 < (int)nl ? s.nk[i] : 0u, c0 = s.fc[i];
        for (uint32_t q = 0; q < nk; ++q) A = __dadd_rn(A, s.A[c0 + q]);
        if (a.mfd_A) A = __ldg(a.mfd_A + s.cell[i]);  // routing = kMfd: the MFD area (k_mfd_tiles)
        s.A[i] = A;
      }
      __syncthreads();
    }
    phclk_mark(s_pc, LEMGPU_PHASE_ACCUM);
    // F of every cell below level 0 at once (its table lookup or pow off the
    // level chain), in place of the area
    uint32_t iters = 0, misses = 0;
    for (uint32_t i = s.lvl[1 < nl ? 1 : 0] + tid; i < (nl > 1 ? s.lvl[nl] : 0u); i += kTPB) {
      const uint32_t mem = a.M > 1 ? s.cell[i] / a.MN : 0u;
      const double F = tile_F(a, mem, dir_class(s.kd[i]), s.A[i], misses);  // class symmetric in k <-> 7-k
      s.A[i] = F;
      if (NK == 1) s.y[i] = F < 0x1p500 ? __ddiv_rn(1.0, __dadd_rn(1.0, F)) : 0.0;  // 0: IEEE Newton
    }
    __syncthreads();  // (the staged elevations landed before the accumulation)
    // uplift (level 0: interior sources only), erosion level by level, from shared memory
    for (uint32_t l = 0; l < nl; ++l) {
      for (uint32_t i = s.lvl[l] + tid; i < s.lvl[l + 1]; i += kTPB) {
        const uint32_t c = s.cell[i];
        double hv = s.h[i];
        if (l == 0) {
          if (is_interior(a, c)) hv = __dadd_rn(hv, a.du);
        } else {
          const double h0 = __dadd_rn(hv, a.du);
          const double hn = s.h[s.par[i]];
          const double F = s.A[i];
          int itn;
          bool okn;
          if (NK == 1 && s.y[i] != 0.0)
            hv = newton_n1_tab(h0, hn, F, s.y[i], a.eps, a.maxit, itn, okn);
          else if (NK == 1)
            hv = newton_n1(h0, hn, F, a.eps, a.maxit, itn, okn);
          else
            hv = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, a.pow_fma, itn, okn);
          if (okn) {
            iters += (uint32_t)itn;
          } else {
            hv = h0;  // as chunk_in_global: the failed cell keeps its uplifted height
            atomicMin(&ctl->err_cell, c);
            ctl->err_slot = ctl->slot;
            atomicMax(&ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
          }
        }
        s.h[i] = hv;
        a.hout[c] = hv;
      }
      __syncthreads();
    }
    // counters aside (dropped if another CTA fails); this CTA's cells appended
    // to the compact list of escaped cells (a.ppos, for the host-step patch)
    for (int o = 16; o; o >>= 1) {
      iters += __shfl_down_sync(0xffffffffu, iters, o);
      misses += __shfl_down_sync(0xffffffffu, misses, o);
    }
    if ((tid & 31) == 0) {
      if (iters) atomicAdd(&ctl->esc_iters, (unsigned long long)iters);
      if (misses) atomicAdd(&ctl->esc_misses, misses);
    }
    const uint32_t cells = s.lvl[nl];
    if (tid == 0) {
      s.base = atomicAdd(&ctl->esc_cells, cells);
      atomicMax(&ctl->esc_nlev, nl);
    }
    __syncthreads();
    for (uint32_t i = tid; i < cells; i += kTPB) a.ppos[s.base + i] = s.cell[i];
  }
  // the last CTA decides
  __shared__ uint32_t s_last;
  __syncthreads();
  phclk_end(s_pc, ok ? LEMGPU_PHASE_EROSION : LEMGPU_PHASE_ORDER, ctl);
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(&ctl->esc_done, 1u) == G - 1 ? 1u : 0u;
  }
  __syncthreads();
  if (s_last && tid == 0) {
    __threadfence();
    ctl->esc_done = 0;
    // the cooperative escape kernels run only when a CTA's share did not fit
    if (a.esc_if) set_cond(a, 4, ld_volatile_u32(&ctl->esc_fail) ? 1u : 0u);
    if (ld_volatile_u32(&ctl->esc_fail) == 0) {
      ctl->nlev = ld_volatile_u32(&ctl->esc_nlev);
      ctl->n0 = n;
      ctl->mode = kModeDone;
      ctl->esc_small = 1;
      ctl->newton += *reinterpret_cast<volatile unsigned long long*>(&ctl->esc_iters);
      ctl->misses += ld_volatile_u32(&ctl->esc_misses);
      const unsigned long long t = globaltimer();
      ctl->t_order_end = t;
      ctl->t_phys_end = t;
    }
  }
}

}  // namespace lemgpu
