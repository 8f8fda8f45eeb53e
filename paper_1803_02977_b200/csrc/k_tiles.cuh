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
// a step only needs, per tree, its cells in breadth-first order (the paper's
// level ordering) to accumulate upstream->downstream and to
// erode downstream->upstream.  The reference's fastest strategy
// (rb_private_queues) exploits exactly this with one private queue per worker
// over a slice of the sources; here the private queues belong to the warps of
// a CTA and the sources are the level-0 cells of a 64x32 raster tile.
//
// A CTA (persistent, looping over tiles) does, for its tile T:
//   1. one TMA box brings h for T grown by 5 cells (kWY x kWP doubles);
//   2. receiver codes for T grown by 4 cells (register sliding 3x3 window);
//   3. donor masks for T grown by 3 cells (SWAR byte compares) = the BFS
//      domain; T's own rcode / dmask bytes go to HBM (they are the step's
//      compact FlowGraph, used by the escape path and the parity export);
//   4. each warp takes the sources in 4 rows of T and grows their trees level
//      by level inside the domain (warp scans, a shared allocator gives every
//      level of a warp one contiguous entry range), then accumulates A in
//      reverse level order (pull over each cell's children in slot order --
//      the reference's FP summation order, so A is bit-identical for any cell
//      area), uplifts and erodes in level order with the receivers' updated
//      elevations, and writes the new elevations to hout.
// A tree that reaches the edge of the domain (any cell more than 3 cells
// outside T; ~0.3% of the cells of a random-noise DEM) or grows deeper than
// kTMaxLev levels ESCAPES: none of its cells is written, its root is appended
// to a list, and the level-synchronous global path (k_order.cuh +
// k_physics.cuh) finishes it after this kernel.  h is read-only during the
// step (hout is the other ping-pong buffer), so the stencil of any CTA sees
// the complete previous surface no matter which trees other CTAs finished.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "k_physics.cuh"
#include "k_recv_donor.cuh"

namespace lemgpu {

// Window coordinates: column x, row y; global cell = (wx0 + x, wy0 + y).
constexpr int kWP = 80;             // window pitch = TMA box width (doubles)
constexpr int kLX = 8;              // first tile column in the window
constexpr int kLY = kHalo + 2;      // first tile row in the window
constexpr int kWY = kTY + 2 * kLY;  // window rows
constexpr int kDX0 = kLX - kHalo, kDX1 = kLX + kTX + kHalo;  // BFS domain columns [kDX0, kDX1)
constexpr int kDY0 = kLY - kHalo, kDY1 = kLY + kTY + kHalo;  // BFS domain rows
constexpr int kRX0 = kDX0 - 1, kRX1 = kDX1 + 1;              // receiver-code columns
constexpr int kRY0 = kDY0 - 1, kRY1 = kDY1 + 1;              // receiver-code rows
constexpr int kRP = 84;          // rc pitch; the code of window column x is stored at byte x + 1
constexpr int kCap = (kDX1 - kDX0) * (kDY1 - kDY0);  // entries: every domain cell at most once
constexpr int kTWarps = kTTPB / 32;
constexpr int kTMaxLev = 32;  // levels per warp forest (deeper trees escape)
constexpr int kRCols = kRX1 - kRX0;  // 72
constexpr int kRSegs = kTTPB / kRCols;  // row segments of the receiver sweep (3)
constexpr int kDGroups = (kRX1 - kRX0) / 4;  // 4-cell donor-mask groups per row (18)
static_assert(kRX0 % 4 == 0 && (kRX1 - kRX0) % 4 == 0, "donor groups must be word aligned");
static_assert(kLX % 4 == 0 && kTX % 4 == 0, "tile groups must be word aligned");
static_assert(kRX1 + 1 <= kWP && kRY1 + 1 == kWY, "h window covers the receiver stencils");
static_assert(kRX1 + 4 <= kRP, "rc pitch");
static_assert(kTY == 4 * kTWarps, "each warp owns 4 tile rows");
static_assert(kCap < 4096 && kWY * kWP < 65536, "16-bit entry fields");

// Entry fields.  ep = (parent entry << 3) | direction parent -> cell; a root
// has parent field kRootPar and bit 0 = "interior cell" (uplifted); bit 15
// marks an entry whose tree escapes (set on roots during the BFS, inherited
// top-down during the erosion sweep).
constexpr uint32_t kRootTag = 0x7FF8u;
constexpr uint32_t kEscBit = 0x8000u;
__device__ __forceinline__ bool ep_is_root(uint32_t pk) { return (pk & kRootTag) == kRootTag; }

// EX: the drainage area is an exact multiple of the cell area (lut_exact), so
// it is carried as an integer cell count and indexes the host-libm F table
// directly; otherwise it is the reference's FP sum (f64).
template <bool EX>
struct TileSmem {
  double hw[kWY * kWP];  // h window (TMA destination), updated in place by the erosion
  typename std::conditional<EX, uint32_t, double>::type eA[kCap];  // drainage area of each entry
  uint16_t ew[kCap];     // window index y*kWP + x of each entry
  uint16_t ep[kCap];     // see above
  uint16_t efc[kCap];    // first child entry (children are contiguous, slot order)
  uint8_t dm[kWY * kWP];   // donor masks restricted to the BFS domain
  uint8_t own[kWY * kWP];  // bit 1: some donor lies outside the domain; bit 0: cell finished here
  uint8_t rc[kWY * kRP];   // receiver codes
  uint8_t rowint[kWY];     // window row holds interior cells
  uint16_t lvs[kTWarps][kTMaxLev];  // per warp: first entry of each level
  uint16_t lvn[kTWarps][kTMaxLev];  // per warp: entries of each level
  uint32_t ecount;                  // entry allocator
  uint64_t bar;
};
template <bool EX>
constexpr size_t tiles_smem_bytes() { return sizeof(TileSmem<EX>); }

// D8, unit cardinal spacing: receiver code without divisions.  t_k = d_k
// (cardinal, exact) or RN(d_k * RN(1/sqrt2)) (diagonal, within 2^-51 relative
// of the reference slope RN(d_k / sqrt2)).  The high words of positive
// doubles order them; when exactly one t_k has a high word within 1 of the
// largest, every other t_j is below it by more than 2^-22 relative, so it is
// the unique strict maximum of the reference slopes as well.  Ties, near
// ties, subnormal or non-finite maxima take the reference loop.
template <int CONN>
__device__ __forceinline__ uint8_t receiver_code_hi(const double (&d)[8], const StepArgs& a) {
  if (CONN == 8 && a.unit_card) {
    int hi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool diag = (k == 0 || k == 2 || k == 5 || k == 7);
      hi[k] = __double2hiint(diag ? __dmul_rn(d[k], a.rinv_diag) : d[k]);
    }
    const int mx = max(max(max(hi[0], hi[1]), max(hi[2], hi[3])), max(max(hi[4], hi[5]), max(hi[6], hi[7])));
    if (mx < 0) return kNoFlowCode;  // every drop negative or -0: no downhill neighbour
    if (mx < 0x00100000) {           // no normal positive slope: +0 drops (flats) or subnormal ones
      bool pos = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) pos |= d[k] > 0.0;
      return pos ? receiver_code_ref<CONN>(d, a) : kNoFlowCode;
    }
    if (mx >= 0x7FF00000) return receiver_code_ref<CONN>(d, a);
    const int thr = mx - 1;
    int ncand = 0, idx = 0;
#pragma unroll
    for (int k = 7; k >= 0; --k) {
      ncand += hi[k] >= thr ? 1 : 0;
      idx = hi[k] == mx ? k : idx;
    }
    if (ncand == 1) return (uint8_t)idx;
    return receiver_code_ref<CONN>(d, a);
  }
  return receiver_code_ref<CONN>(d, a);
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, uint32_t lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (uint32_t)o) v += y;
  }
  return v;
}

// Directions k whose neighbour of window cell (x, y) lies inside the BFS domain.
__device__ __forceinline__ uint32_t domain_dirs(uint32_t x, uint32_t y) {
  uint32_t m = 0xFFu;
  if (x == (uint32_t)kDX0) m &= ~0x29u;      // ox = -1: k = 0, 3, 5
  if (x == (uint32_t)kDX1 - 1) m &= ~0x94u;  // ox = +1: k = 2, 4, 7
  if (y == (uint32_t)kDY0) m &= ~0x07u;      // oy = -1: k = 0, 1, 2
  if (y == (uint32_t)kDY1 - 1) m &= ~0xE0u;  // oy = +1: k = 5, 6, 7
  return m;
}

// F = ((K*dt) * pow(A, m)) / pow(dist, n) (erosion.cpp:38-39) from the host
// libm table when A is an exact multiple of the cell area.
__device__ __forceinline__ double tile_F(const StepArgs& a, uint32_t mem, uint32_t cls, double A,
                                         uint32_t& misses) {
  const double q = a.w0_is_one ? A : __ddiv_rn(A, a.w0);
  if (a.lut_exact && q < (double)a.lut_entries && q == floor(q))
    return __ldg(a.ftab + ((size_t)mem * 3 + cls) * a.lut_entries + (uint32_t)q);
  ++misses;
  const double pd = cls == 0 ? a.powdist_h : cls == 1 ? a.powdist_v : a.powdist_d;
  return __ddiv_rn(__dmul_rn(__ldg(a.kdt + mem), pow(A, __ldg(a.mexp + mem))), pd);
}

template <int CONN, int NK, bool EX>
__global__ void __launch_bounds__(kTTPB, EX ? 3 : 2) k_tiles(StepArgs a, const __grid_constant__ CUtensorMap hmap) {
  extern __shared__ __align__(128) unsigned char smraw[];
  TileSmem<EX>& s = *reinterpret_cast<TileSmem<EX>*>(smraw);
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->err_flag)) return;  // an earlier step failed (uniform)
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int W = (int)a.W, Ht = (int)a.Htot;
  const uint32_t ntx = (a.W + kTX - 1) / kTX, nty = (a.Htot + kTY - 1) / kTY;
  const uint32_t ntiles = ntx * nty;
  const uint32_t E = a.lut_entries;
  if (tid == 0) {
    atomicMin(&ctl->t_k1_begin, globaltimer());
    if (a.use_tma) mbar_init(&s.bar, 1);
  }
  // the escape path's level-0 and level-1 bins start at zero
  for (uint32_t i = blockIdx.x * kTTPB + tid; i < 2 * a.scan_grid; i += gridDim.x * kTTPB) a.bins[i] = 0;

  unsigned long long iters = 0;  // per lane
  uint32_t misses = 0, cells = 0, n0i = 0, maxl = 0;
  uint32_t phase = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, phase ^= 1u) {
    const int tx0 = (int)(t % ntx) * kTX, ty0 = (int)(t / ntx) * kTY;
    const int wx0 = tx0 - kLX, wy0 = ty0 - kLY;
    __syncthreads();  // the previous tile is finished with every shared array
    if (tid == 0) {
      s.ecount = 0;
      if (a.use_tma) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes of hw before the TMA overwrite
        mbar_expect_tx(&s.bar, (uint32_t)sizeof(s.hw));
        tma_load_2d(s.hw, &hmap, wx0, wy0, &s.bar);  // out-of-raster cells arrive as 0
      }
    }
    if (!a.use_tma) {
      for (int i = (int)tid; i < kWY * kWP; i += kTTPB) {
        const int y = i / kWP, x = i - y * kWP;
        const int gx = wx0 + x, gy = wy0 + y;
        s.hw[i] = (gx >= 0 && gx < W && gy >= 0 && gy < Ht) ? __ldg(a.h + (size_t)gy * W + gx) : 0.0;
      }
    }
    for (int i = (int)tid; i < kWY * kRP / 4; i += kTTPB) reinterpret_cast<uint32_t*>(s.rc)[i] = 0x08080808u;
    if (tid < (uint32_t)kWY) {
      const int gy = wy0 + (int)tid;
      uint8_t ok = 0;
      if (gy >= 0 && gy < Ht) {
        const uint32_t yl = (uint32_t)gy % a.H;
        ok = yl > 0 && yl < a.H - 1;
      }
      s.rowint[tid] = ok;
    }
    __syncthreads();
    if (a.use_tma) mbar_wait(&s.bar, phase);

    // ---- 2. receiver codes: one column per thread, 3x3 register window sliding down
    if (tid < (uint32_t)(kRCols * kRSegs)) {
      const int x = kRX0 + (int)(tid % kRCols), seg = (int)(tid / kRCols);
      const int nrow = kRY1 - kRY0;
      const int yb = kRY0 + seg * nrow / kRSegs, ye = kRY0 + (seg + 1) * nrow / kRSegs;
      const int gx = wx0 + x;
      const bool colint = gx > 0 && gx < W - 1;
      const double* col = s.hw + x - 1;
      double w0[3], w1[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        w0[q] = col[(yb - 1) * kWP + q];
        w1[q] = col[yb * kWP + q];
      }
      for (int y = yb; y < ye; ++y) {
        double w2[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) w2[q] = col[(y + 1) * kWP + q];
        uint8_t code = kNoFlowCode;
        if (colint && s.rowint[y]) {
          const double ec = w1[1];
          double d[8];
          d[0] = __dsub_rn(ec, w0[0]);
          d[1] = __dsub_rn(ec, w0[1]);
          d[2] = __dsub_rn(ec, w0[2]);
          d[3] = __dsub_rn(ec, w1[0]);
          d[4] = __dsub_rn(ec, w1[2]);
          d[5] = __dsub_rn(ec, w2[0]);
          d[6] = __dsub_rn(ec, w2[1]);
          d[7] = __dsub_rn(ec, w2[2]);
          if (CONN == 4) d[0] = d[2] = d[5] = d[7] = 0.0;
          code = receiver_code_hi<CONN>(d, a);
        }
        s.rc[y * kRP + x + 1] = code;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          w0[q] = w1[q];
          w1[q] = w2[q];
        }
      }
    }
    __syncthreads();

    // ---- 3. donor masks of the domain (4 cells per item), restricted to the
    // domain, with a per-cell flag for donors outside it; the tile's own
    // receiver codes and (complete) donor masks go to HBM
    for (int it = (int)tid; it < (kDY1 - kDY0) * kDGroups; it += kTTPB) {
      const int y = kDY0 + it / kDGroups, x = kRX0 + 4 * (it % kDGroups);
      uint32_t lo[3], hi[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        lo[q] = *reinterpret_cast<const uint32_t*>(s.rc + (y - 1 + q) * kRP + x);
        hi[q] = *reinterpret_cast<const uint32_t*>(s.rc + (y - 1 + q) * kRP + x + 4);
      }
      uint32_t pm = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!dir_in(CONN, k)) continue;
        const int q = 1 + dir_oy(k);
        const uint32_t sel = dir_ox(k) < 0 ? 0x3210u : dir_ox(k) == 0 ? 0x4321u : 0x5432u;
        pm |= zero_bytes(__byte_perm(lo[q], hi[q], sel) ^ (0x01010101u * (uint32_t)(7 - k))) << k;
      }
      // directions that stay inside the domain, per byte
      uint32_t dd = 0xFFFFFFFFu;
      if (x == kRX0) dd &= ~(0x29u << 8);                 // cell x+1 = kDX0: no ox = -1
      if (x + 4 == kRX1) dd &= ~(0x94u << 16);            // cell x+2 = kDX1-1: no ox = +1
      if (y == kDY0) dd &= ~0x07070707u;                  // no oy = -1
      if (y == kDY1 - 1) dd &= ~0xE0E0E0E0u;              // no oy = +1
      const uint32_t vm = pm & dd;
      const uint32_t leak = (~zero_bytes(pm & ~dd) & 0x01010101u) << 1;
      *reinterpret_cast<uint32_t*>(s.dm + y * kWP + x) = vm;
      *reinterpret_cast<uint32_t*>(s.own + y * kWP + x) = leak;
      if (y >= kLY && y < kLY + kTY && x >= kLX && x < kLX + kTX) {
        const int gy = wy0 + y, gx = wx0 + x;
        if (gy < Ht && gx < W) {
          const uint32_t pc = __byte_perm(lo[1], hi[1], 0x4321u);
          const size_t base = (size_t)gy * a.W + gx;
          if (gx + 3 < W && (a.W & 3u) == 0) {
            *reinterpret_cast<uint32_t*>(a.rcode + base) = pc;
            *reinterpret_cast<uint32_t*>(a.dmask + base) = pm;
          } else {
            for (int j = 0; j < 4 && gx + j < W; ++j) {
              a.rcode[base + j] = (uint8_t)(pc >> (8 * j));
              a.dmask[base + j] = (uint8_t)(pm >> (8 * j));
            }
          }
        }
      }
    }
    __syncthreads();

    // ---- 4. per warp: the trees rooted in tile rows 4w..4w+3
    uint16_t* lvs = s.lvs[warp];
    uint16_t* lvn = s.lvn[warp];
    {
      // level 0: the NoFlow cells of the rows, ascending
      uint32_t bal[8], nr = 0, intm = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int y = kLY + 4 * (int)warp + (j >> 1), x = kLX + 32 * (j & 1) + (int)lane;
        const int gx = wx0 + x, gy = wy0 + y;
        const bool root = gx < W && gy < Ht && s.rc[y * kRP + x + 1] == kNoFlowCode;
        bal[j] = __ballot_sync(0xffffffffu, root);
        nr += __popc(bal[j]);
        const bool in = root && s.rowint[y] && gx > 0 && gx < W - 1;  // interior NoFlow cell
        intm |= (in ? 1u : 0u) << j;
        n0i += in ? 1u : 0u;
      }
      uint32_t base = 0;
      if (lane == 0 && nr) base = atomicAdd(&s.ecount, nr);
      base = __shfl_sync(0xffffffffu, base, 0);
      uint32_t pos = base;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int y = kLY + 4 * (int)warp + (j >> 1), x = kLX + 32 * (j & 1) + (int)lane;
        if ((bal[j] >> lane) & 1u) {
          const uint32_t i = pos + __popc(bal[j] & ((1u << lane) - 1u));
          s.ew[i] = (uint16_t)(y * kWP + x);
          uint32_t pk = kRootTag | ((intm >> j) & 1u);
          if (a.force_escape == 1 || (a.force_escape == 2 && (((wy0 + y) * W + wx0 + x) & 1))) pk |= kEscBit;
          s.ep[i] = (uint16_t)pk;
        }
        pos += __popc(bal[j]);
      }
      if (lane == 0) {
        lvs[0] = (uint16_t)base;
        lvn[0] = (uint16_t)nr;
      }
    }
    __syncwarp();
    // levels 1, 2, ...: two passes per level (count, then write into one range)
    uint32_t nl = 1;
    for (uint32_t l = 0;; ++l) {
      const uint32_t fs = lvs[l], fn = lvn[l];
      uint32_t run = 0;
      for (uint32_t j0 = 0; j0 < fn; j0 += 32) {
        const uint32_t j = j0 + lane, i = fs + j;
        uint32_t cnt = 0;
        if (j < fn) {
          const uint32_t wi = s.ew[i];
          cnt = __popc((uint32_t)s.dm[wi]);
          if (s.own[wi] & 2u) {  // a donor outside the domain: the whole tree escapes
            uint32_t r = i, pk = s.ep[r];
            while (!ep_is_root(pk)) {
              r = (pk & 0x7FFFu) >> 3;
              pk = s.ep[r];
            }
            s.ep[r] = (uint16_t)(pk | kEscBit);
          }
        }
        const uint32_t incl = warp_incl_scan(cnt, lane);
        if (j < fn) s.efc[i] = (uint16_t)(run + incl - cnt);
        run += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (run == 0) break;
      if (l + 1 >= (uint32_t)kTMaxLev) {  // too deep for the per-warp level table: escape
        for (uint32_t j = lane; j < fn; j += 32) {
          uint32_t r = fs + j, pk = s.ep[r];
          while (!ep_is_root(pk)) {
            r = (pk & 0x7FFFu) >> 3;
            pk = s.ep[r];
          }
          s.ep[r] = (uint16_t)(pk | kEscBit);
        }
        break;
      }
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&s.ecount, run);
      base = __shfl_sync(0xffffffffu, base, 0);
      for (uint32_t j = lane; j < fn; j += 32) {
        const uint32_t i = fs + j;
        const uint32_t wi = s.ew[i];
        uint32_t vm = s.dm[wi];
        uint32_t c = base + s.efc[i];
        s.efc[i] = (uint16_t)c;
        while (vm) {
          const uint32_t k = __ffs(vm) - 1;
          vm &= vm - 1;
          s.ew[c] = (uint16_t)((int)wi + dir_off(k, kWP));
          s.ep[c] = (uint16_t)((i << 3) | k);
          ++c;
        }
      }
      if (lane == 0) {
        lvs[l + 1] = (uint16_t)base;
        lvn[l + 1] = (uint16_t)run;
      }
      nl = l + 2;
      __syncwarp();
    }
    __syncwarp();

    // accumulation, deepest level first: A = w + the children's A in slot
    // order (escaped trees are accumulated too, harmlessly, and never used)
    for (int l = (int)nl - 1; l >= 0; --l) {
      const uint32_t fs = lvs[l], fn = lvn[l];
      for (uint32_t j = lane; j < fn; j += 32) {
        const uint32_t i = fs + j;
        const uint32_t nch = __popc((uint32_t)s.dm[s.ew[i]]);
        const uint32_t c0 = s.efc[i];
        if (EX) {
          uint32_t A = 1u;
          for (uint32_t q = 0; q < nch; ++q) A += (uint32_t)s.eA[c0 + q];
          s.eA[i] = A;
        } else {
          double A = a.w0;
          for (uint32_t q = 0; q < nch; ++q) A = __dadd_rn(A, (double)s.eA[c0 + q]);
          s.eA[i] = A;
        }
      }
      __syncwarp();
    }
    // level 0: uplift interior sources (never eroded); escaped roots -> the
    // global level path (level 0 of its queue)
    {
      const uint32_t fn = lvn[0], fs = lvs[0];
      for (uint32_t j0 = 0; j0 < fn; j0 += 32) {
        const uint32_t j = j0 + lane, i = fs + j;
        uint32_t pk = 0, wi = 0;
        if (j < fn) {
          pk = s.ep[i];
          wi = s.ew[i];
        }
        const bool e = j < fn && (pk & kEscBit);
        if (j < fn && !e) {
          if (pk & 1u) s.hw[wi] = __dadd_rn(s.hw[wi], a.du);
          s.own[wi] = 1u;
          ++cells;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, e);
        if (!b) continue;
        uint32_t p = 0;
        if (lane == 0) p = atomicAdd(&ctl->nesc, __popc(b));
        p = __shfl_sync(0xffffffffu, p, 0);
        if (e) {
          const uint32_t y = wi / kWP, x = wi - y * kWP;
          a.order[p + __popc(b & ((1u << lane) - 1u))] = (uint32_t)(wy0 + (int)y) * a.W + (uint32_t)(wx0 + (int)x);
        }
      }
    }
    __syncwarp();
    // erosion, downstream -> upstream, with the receiver's updated elevation
    for (uint32_t l = 1; l < nl; ++l) {
      const uint32_t fs = lvs[l], fn = lvn[l];
      bool any = false;
      for (uint32_t j = lane; j < fn; j += 32) {
        const uint32_t i = fs + j;
        const uint32_t pk = s.ep[i], p = pk >> 3;
        const uint32_t pp = s.ep[p];
        if (pp & kEscBit) {  // the tree escapes: inherit the mark, leave the cell to the level path
          s.ep[i] = (uint16_t)(pk | kEscBit);
          continue;
        }
        any = true;
        const uint32_t wi = s.ew[i];
        uint32_t mem = 0;
        if (a.M > 1) mem = (uint32_t)(wy0 + (int)(wi / kWP)) / a.H;
        const uint32_t cls = dir_class(pk & 7u);
        double F;
        if (EX)
          F = __ldg(a.ftab + (mem * 3 + cls) * E + (uint32_t)s.eA[i]);
        else
          F = tile_F(a, mem, cls, (double)s.eA[i], misses);
        const double h0 = __dadd_rn(s.hw[wi], a.du);  // uplift (every cell below level 0 is interior)
        const double hn = s.hw[s.ew[p]];
        int it;
        bool ok;
        double hnew;
        if (NK == 1)
          hnew = newton_n1(h0, hn, F, a.eps, a.maxit, it, ok);
        else
          hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, it, ok);
        if (ok) {
          iters += (unsigned long long)it;
        } else {
          const uint32_t y = wi / kWP, x = wi - y * kWP;
          atomicMin(&ctl->err_cell, (uint32_t)(wy0 + (int)y) * a.W + (uint32_t)(wx0 + (int)x));
          ctl->err_slot = ctl->slot;
          atomicMax(&ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
        }
        s.hw[wi] = hnew;
        s.own[wi] = 1u;
        ++cells;
      }
      if (__any_sync(0xffffffffu, any)) maxl = max(maxl, l);
      __syncwarp();
    }
    __syncthreads();
    // ---- 5. write back every cell finished here, row by row (coalesced)
    for (int y = kDY0 + (int)warp; y < kDY1; y += kTWarps) {
      const int gy = wy0 + y;
#pragma unroll
      for (int x0 = kDX0 & ~31; x0 < kDX1; x0 += 32) {
        const int x = x0 + (int)lane;
        if (x >= kDX0 && x < kDX1 && (s.own[y * kWP + x] & 1u))
          a.hout[(size_t)gy * a.W + (wx0 + x)] = s.hw[y * kWP + x];
      }
    }
  }

  // ---- counters: one atomic per warp for the whole kernel
  for (int o = 16; o; o >>= 1) {
    iters += __shfl_down_sync(0xffffffffu, iters, o);
    misses += __shfl_down_sync(0xffffffffu, misses, o);
    cells += __shfl_down_sync(0xffffffffu, cells, o);
    n0i += __shfl_down_sync(0xffffffffu, n0i, o);
  }
  if (lane == 0) {
    if (iters) atomicAdd(&ctl->newton, iters);
    if (misses) atomicAdd(&ctl->misses, misses);
    if (cells) atomicAdd(&ctl->tile_cells, cells);
    if (n0i) atomicAdd(&ctl->n0i, n0i);
    atomicMax(&ctl->tile_nlev, maxl + 1);
  }
  __syncthreads();
  if (tid == 0) atomicMax(&ctl->t_k1_end, globaltimer());
}

// Level 0 of the escape path: the escaped roots (listed by k_tiles in
// order[0, nesc)), their donor masks and the per-segment child counts of
// the first expansion.  Order of the list is irrelevant to the results (every
// schedule of the per-cell arithmetic is bit-identical).
__global__ void __launch_bounds__(kTPB) k_esc_l0(StepArgs a) {
  Ctl* ctl = a.ctl;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t n = ld_volatile_u32(&ctl->nesc);
  const uint32_t Sb = seg_size(n, G);
  if (!ld_volatile_u32(&ctl->err_flag)) {
    const uint32_t s0 = min(b * Sb, n), s1 = min(s0 + Sb, n);
    pdm_and_bins<false>(a, nullptr, nullptr, 0u, s0, s1, 0u, Sb, a.bins);
  }
  if (last_block_done(ctl) && threadIdx.x == 0) {
    a.levels[0] = 0;
    a.levels[1] = n;
    ctl->n0 = n;
    ctl->nch = (n + kChunkRoots - 1) / kChunkRoots;
    ctl->lvl = 0;
    ctl->t_k1_end = max(ctl->t_k1_end, globaltimer());
    timeline(ctl);
  }
}

}  // namespace lemgpu
