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
// A CTA (persistent, looping over tiles) does, for its tile T:
//   1. one TMA box brings h for T grown by 5 cells (kWY x kWP doubles);
//   2. receiver codes for T grown by 4 cells (register sliding 3x3 window);
//   3. donor masks for T grown by 3 cells (SWAR byte compares) = the domain;
//      T's own rcode / dmask bytes go to HBM (they are the step's compact
//      FlowGraph, used by the escape path and the parity export);
//   4. bitmaps of the domain: cells by receiver direction, cells with a
//      donor outside the domain, T's level-0 cells (one ballot per word);
//   5. breadth first from T's level-0 cells: level l+1 = the domain cells
//      whose receiver is in level l, one bitmap pass per level (shift + and
//      per direction), listed level-major (block prefix of the word counts):
//      the level structure of the reference's TraversalPlan for T's sources;
//   6. drainage area: exact cell counts (every cell adds 1 to each ancestor;
//      integer adds commute) or, for a cell area that is not exact, the
//      reference's FP pull in slot order level by level;
//   7. uplift + implicit erosion level by level (block barrier per level),
//      each cell reading its receiver's already updated elevation; the new
//      elevations go to hout.
// A tree with a cell whose donor lies outside the domain (its cells reach
// more than 3 cells beyond T; ~0.3% of the cells of a random-noise DEM) or
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
// (wx0 + x, wy0 + y).
constexpr int kWP = 84;             // window pitch = TMA box width (doubles)
constexpr int kLX = 8;              // first tile column in the window
constexpr int kLY = kHalo + 2;      // first tile row in the window
constexpr int kWY = kTY + 2 * kLY;  // window rows
constexpr int kWN = kWY * kWP;      // window cells
constexpr int kDX0 = kLX - kHalo, kDX1 = kLX + kTX + kHalo;  // domain columns [kDX0, kDX1)
constexpr int kDY0 = kLY - kHalo, kDY1 = kLY + kTY + kHalo;  // domain rows
constexpr int kDW = kDX1 - kDX0, kDH = kDY1 - kDY0;
constexpr int kRX0 = kDX0 - 1, kRX1 = kDX1 + 1;  // receiver-code columns
constexpr int kRY0 = kDY0 - 1, kRY1 = kDY1 + 1;  // receiver-code rows
constexpr int kCap = kDW * kDH;                  // queue: every domain cell at most once
constexpr int kTMaxLev = 64;                     // deeper trees escape
constexpr int kRCols = kRX1 - kRX0;              // 72
constexpr int kRSegs = kTTPB / kRCols;           // row segments of the receiver sweep (3)
constexpr int kDGroups = (kRX1 - kRX0) / 4;      // 4-cell donor-mask groups per row (18)
static_assert(kRX0 % 4 == 0 && (kRX1 - kRX0) % 4 == 0 && kWP % 4 == 0, "donor groups must be word aligned");
static_assert(kLX % 4 == 0 && kTX % 4 == 0, "tile groups must be word aligned");
static_assert(kRX1 + 1 <= kWP && kRY1 + 1 == kWY, "h window covers the receiver stencils");
static_assert(kWN < 65535, "16-bit window indices");

// Bitmaps of the window: row y, 32-column word w (columns 32w .. 32w+31).
constexpr int kBW = 3;            // words per row (96 >= kWP columns)
constexpr int kBN = kWY * kBW;    // words per bitmap
constexpr int kBPairs = kDH * kBW;  // (row, word) pairs of the domain rows
constexpr int kBWarps = (kBPairs + 31) / 32;  // warps holding them
static_assert(kBW * 32 >= kWP && kBPairs <= kTTPB, "bitmap geometry");

// EX: the drainage area is an exact multiple of the cell area (lut_exact), so
// it is carried as an integer cell count and indexes the host-libm F table
// directly; otherwise it is the reference's FP sum (f64).
template <bool EX>
struct TileSmem {
  double hw[kWN];  // h window (TMA destination), updated in place by the erosion
  typename std::conditional<EX, uint32_t, double>::type acc[kWN];  // drainage area: cell count (EX) or FP sum
  uint16_t list[kCap];         // the tile's queue, level-major
  uint8_t rc[kWN + 8];         // receiver codes; the code of q is at q + 1
  uint8_t dm[kWN];             // donor masks restricted to the domain
  uint8_t fl[kWN];             // 1: some donor of the cell lies outside the domain
  uint8_t esc[kWN];            // the cell's tree escapes (set on roots, inherited downstream -> upstream)
  uint8_t rowint[kWY];         // window row holds interior cells
  uint32_t pl[4][kBN];         // bit planes 0-2 of the receiver code, and "code < 8"
  uint32_t lk[kBN];            // domain cells with a donor outside the domain
  uint32_t wsum[2][kTTPB / 32];  // per-warp level counts (double-buffered by level parity)
  uint32_t lv[2][kBN];         // current / next level
  uint32_t lvs[kTMaxLev + 1];  // first queue position of each level
  uint32_t nlev;
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
// ties, subnormal or non-finite maxima take the reference loop
// (tests/native/test_receiver_code.cu checks this against the loop).
template <int CONN>
__host__ __device__ __forceinline__ uint8_t receiver_code_hi(const double (&d)[8], const StepArgs& a) {
  if (CONN == 8 && a.unit_card) {
    int hi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool diag = (k == 0 || k == 2 || k == 5 || k == 7);
      hi[k] = hi_word(diag ? LG_MUL(d[k], a.rinv_diag) : d[k]);
    }
    auto mx2 = [](int u, int v) { return u > v ? u : v; };
    const int mx = mx2(mx2(mx2(hi[0], hi[1]), mx2(hi[2], hi[3])), mx2(mx2(hi[4], hi[5]), mx2(hi[6], hi[7])));
    if (mx < 0) return kNoFlowCode;  // every drop negative or -0: no downhill neighbour
    if (mx < 0x00100000) {           // no normal positive slope: +0 drops (flats) or subnormal ones
      bool pos = false;
#pragma unroll
      for (int k = 0; k < 8; ++k) pos |= d[k] > 0.0;
      return pos ? receiver_code_ref<CONN>(d, a) : kNoFlowCode;
    }
    if (mx >= 0x7FF00000) return receiver_code_ref<CONN>(d, a);
    const int thr = mx - 1;
    uint32_t cand = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) cand |= (hi[k] >= thr ? 1u : 0u) << k;
    if ((cand & (cand - 1u)) == 0) {  // a single candidate: the maximum
#ifdef __CUDA_ARCH__
      return (uint8_t)(__ffs(cand) - 1);
#else
      return (uint8_t)__builtin_ctz(cand);
#endif
    }
    return receiver_code_ref<CONN>(d, a);
  }
  return receiver_code_ref<CONN>(d, a);
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
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const int W = (int)a.W, Ht = (int)a.Htot;
  const uint32_t ntx = (a.W + kTX - 1) / kTX, nty = (a.Htot + kTY - 1) / kTY;
  const uint32_t ntiles = ntx * nty;
  const uint32_t E = a.lut_entries;
  const bool tab = EX && NK == 1 && a.tab_ok;
  if (tid == 0) {
    atomicMin(&ctl->t_k1_begin, globaltimer());
    if (a.use_tma) mbar_init(&s.bar, 1);
  }
  // the escape path's level-0 and level-1 bins start at zero
  for (uint32_t i = blockIdx.x * kTTPB + tid; i < 2 * a.scan_grid; i += gridDim.x * kTTPB) a.bins[i] = 0;

  unsigned long long iters = 0;  // per thread
  uint32_t misses = 0, cells = 0, n0i = 0, maxl = 0;
  uint32_t phase = 0;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x, phase ^= 1u) {
    const int tx0 = (int)(t % ntx) * kTX, ty0 = (int)(t / ntx) * kTY;
    const int wx0 = tx0 - kLX, wy0 = ty0 - kLY;
    const uint32_t gbase = (uint32_t)wy0 * a.W + (uint32_t)wx0;  // global index of window (0, 0), mod 2^32
    // global cell of window index q (mod 2^32 arithmetic)
    auto gcell = [&](uint32_t q) {
      const uint32_t y = q / kWP;
      return gbase + q + y * (a.W - (uint32_t)kWP);
    };
    __syncthreads();  // the previous tile is finished with every shared array
    if (tid == 0 && a.use_tma) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes of hw before the TMA overwrite
      mbar_expect_tx(&s.bar, (uint32_t)sizeof(s.hw));
      tma_load_2d(s.hw, &hmap, wx0, wy0, &s.bar);  // out-of-raster cells arrive as 0
    }
    if (!a.use_tma) {
      for (int i = (int)tid; i < kWN; i += kTTPB) {
        const int y = i / kWP, x = i - y * kWP;
        const int gx = wx0 + x, gy = wy0 + y;
        s.hw[i] = (gx >= 0 && gx < W && gy >= 0 && gy < Ht) ? __ldg(a.h + (size_t)gy * W + gx) : 0.0;
      }
    }
    for (int i = (int)tid; i < (kWN + 8) / 4; i += kTTPB) reinterpret_cast<uint32_t*>(s.rc)[i] = 0x08080808u;
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

    // ---- 2. receiver codes: one column per thread, 3x3 register window
    // sliding down (unrolled by three rows so the window never moves registers)
    if (tid < (uint32_t)(kRCols * kRSegs)) {
      const int x = kRX0 + (int)(tid % kRCols), seg = (int)(tid / kRCols);
      const int nrow = kRY1 - kRY0;
      const int yb = kRY0 + seg * nrow / kRSegs, ye = kRY0 + (seg + 1) * nrow / kRSegs;
      const int gx = wx0 + x;
      const bool colint = gx > 0 && gx < W - 1;
      const double* col = s.hw + x - 1;
      uint8_t* rcol = s.rc + x + 1;
      auto emit = [&](int y, const double (&u)[3], const double (&m)[3], const double (&v)[3]) {
        uint8_t code = kNoFlowCode;
        if (colint && s.rowint[y]) {
          const double ec = m[1];
          double d[8];
          d[0] = __dsub_rn(ec, u[0]);
          d[1] = __dsub_rn(ec, u[1]);
          d[2] = __dsub_rn(ec, u[2]);
          d[3] = __dsub_rn(ec, m[0]);
          d[4] = __dsub_rn(ec, m[2]);
          d[5] = __dsub_rn(ec, v[0]);
          d[6] = __dsub_rn(ec, v[1]);
          d[7] = __dsub_rn(ec, v[2]);
          if (CONN == 4) d[0] = d[2] = d[5] = d[7] = 0.0;
          code = receiver_code_hi<CONN>(d, a);
        }
        rcol[y * kWP] = code;
      };
      auto load = [&](double (&r)[3], int y) {
#pragma unroll
        for (int q = 0; q < 3; ++q) r[q] = col[y * kWP + q];
      };
      double r0[3], r1[3], r2[3];
      load(r0, yb - 1);
      load(r1, yb);
      int y = yb;
      for (; y + 3 <= ye; y += 3) {
        load(r2, y + 1);
        emit(y, r0, r1, r2);
        load(r0, y + 2);
        emit(y + 1, r1, r2, r0);
        load(r1, y + 3);
        emit(y + 2, r2, r0, r1);
      }
      if (y < ye) {
        load(r2, y + 1);
        emit(y, r0, r1, r2);
        if (y + 1 < ye) {
          load(r0, y + 2);
          emit(y + 1, r1, r2, r0);
        }
      }
    }
    __syncthreads();

    // ---- 3. donor masks of the domain (4 cells per item), restricted to the
    // domain, with a per-cell flag for donors outside it; the tile's own
    // receiver codes and (complete) donor masks go to HBM
    for (int it = (int)tid; it < kDH * kDGroups; it += kTTPB) {
      const int y = kDY0 + it / kDGroups, x = kRX0 + 4 * (it % kDGroups);
      uint32_t lo[3], hi[3];
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        lo[q] = *reinterpret_cast<const uint32_t*>(s.rc + (y - 1 + q) * kWP + x);
        hi[q] = *reinterpret_cast<const uint32_t*>(s.rc + (y - 1 + q) * kWP + x + 4);
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
      if (x == kRX0) dd &= ~(0x29u << 8);       // cell x+1 = kDX0: no ox = -1
      if (x + 4 == kRX1) dd &= ~(0x94u << 16);  // cell x+2 = kDX1-1: no ox = +1
      if (y == kDY0) dd &= ~0x07070707u;        // no oy = -1
      if (y == kDY1 - 1) dd &= ~0xE0E0E0E0u;    // no oy = +1
      *reinterpret_cast<uint32_t*>(s.dm + y * kWP + x) = pm & dd;
      *reinterpret_cast<uint32_t*>(s.fl + y * kWP + x) = ~zero_bytes(pm & ~dd) & 0x01010101u;
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
    // ---- 4. bitmaps of the domain: the four bit planes of the receiver code
    // (code 15 outside the domain), cells with leaking donors, and the
    // tile's roots (level 0); one ballot per (row, word) and bitmap
    for (uint32_t pr = tid >> 5; pr < (uint32_t)kBN; pr += kTTPB / 32) {
      const uint32_t y = pr / kBW, w = pr - y * kBW, x = 32 * w + lane;
      const uint32_t q = y * kWP + x;
      const bool dom = y - kDY0 < (uint32_t)kDH && x - kDX0 < (uint32_t)kDW;
      const uint32_t code = dom ? (uint32_t)s.rc[q + 1] : 0xFu;
      const int gx = wx0 + (int)x, gy = wy0 + (int)y;
      const bool root = code == kNoFlowCode && x - kLX < (uint32_t)kTX && y - kLY < (uint32_t)kTY && gx < W && gy < Ht;
      const uint32_t b0 = __ballot_sync(0xffffffffu, code & 1u), b1 = __ballot_sync(0xffffffffu, code & 2u);
      const uint32_t b2 = __ballot_sync(0xffffffffu, code & 4u), b3 = __ballot_sync(0xffffffffu, code & 8u);
      const uint32_t bl = __ballot_sync(0xffffffffu, dom && s.fl[q]);
      const uint32_t br = __ballot_sync(0xffffffffu, root);
      if (lane == 0) {
        s.pl[0][pr] = b0;
        s.pl[1][pr] = b1;
        s.pl[2][pr] = b2;
        s.pl[3][pr] = ~b3;  // cells with a receiver direction 0..7
        s.lk[pr] = bl;
        s.lv[0][pr] = br;
        s.lv[1][pr] = 0u;  // rows outside the domain stay empty in both level buffers
      }
    }
    __syncthreads();
    // ---- 5. the levels, breadth first from the tile's roots: level l+1 =
    // the domain cells whose receiver is in level l (one bitmap pass per
    // level: shift + and per direction), listed level-major (block prefix of
    // the word counts); a tree reaching a cell with a leaking donor escapes
    // (its root is marked)
    uint32_t nl = 0, qpos = 0;
    for (uint32_t l = 0;; ++l) {
      const uint32_t* cur = s.lv[(l + 1) & 1];  // level l-1 (level 0: the roots, in lv[0])
      uint32_t* nxt = s.lv[l & 1];              // level l
      uint32_t word = 0, y = 0, w = 0;
      if (tid < (uint32_t)kBPairs) {
        y = kDY0 + tid / kBW;
        w = tid - (y - kDY0) * kBW;
        const uint32_t o = y * kBW + w;
        if (l == 0) {
          word = nxt[o];
        } else {
          // S_k(cur): bit x of row y = bit x + ox_k of row y + oy_k
          uint32_t sh[3][3];  // [oy+1][ox+1]
#pragma unroll
          for (int oy = -1; oy <= 1; ++oy) {
            const uint32_t* row = cur + (y + oy) * kBW;
            const uint32_t c = row[w], lo = w > 0 ? row[w - 1] : 0u, hi = w + 1 < (uint32_t)kBW ? row[w + 1] : 0u;
            sh[oy + 1][0] = (c << 1) | (lo >> 31);
            sh[oy + 1][1] = c;
            sh[oy + 1][2] = (c >> 1) | (hi << 31);
          }
          const uint32_t p0 = s.pl[0][o], p1 = s.pl[1][o], p2 = s.pl[2][o];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (!dir_in(CONN, k)) continue;
            const uint32_t rk = ((k & 1) ? p0 : ~p0) & ((k & 2) ? p1 : ~p1) & ((k & 4) ? p2 : ~p2);
            word |= rk & sh[dir_oy(k) + 1][dir_ox(k) + 1];
          }
          word &= s.pl[3][o];
        }
      }
      const uint32_t cnt = __popc(word);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t yv = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += yv;
      }
      uint32_t* ws = s.wsum[l & 1];
      if (lane == 31 && tid < (uint32_t)kBPairs + 31) ws[tid >> 5] = incl;
      if (l > 0 && tid < (uint32_t)kBPairs) nxt[y * kBW + w] = word;
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
        while (word) {
          const uint32_t b = __ffs(word) - 1;
          word &= word - 1;
          const uint32_t q = y * kWP + 32 * w + b;
          s.list[pos++] = (uint16_t)q;
          s.esc[q] = 0;
          if (EX) s.acc[q] = 1u;
          if ((leaks >> b) & 1u) {  // a donor outside the domain: the tree escapes
            uint32_t r = q, code = s.rc[q + 1];
            while (code != kNoFlowCode) {
              r = (uint32_t)((int)r + dir_off(code, kWP));
              code = s.rc[r + 1];
            }
            s.esc[r] = 1;
          }
        }
      }
      qpos += tot;
      nl = l + 1;
      if (l + 1 == (uint32_t)kTMaxLev) break;
    }
    if (tid == 0) s.lvs[nl] = qpos;
    __syncthreads();
    if (nl == (uint32_t)kTMaxLev) {
      // level kTMaxLev would not be empty: every tree reaching it escapes
      for (uint32_t i = s.lvs[nl - 1] + tid; i < s.lvs[nl]; i += kTTPB) {
        uint32_t r = s.list[i];
        if (!s.dm[r]) continue;
        uint32_t code = s.rc[r + 1];
        while (code != kNoFlowCode) {
          r = (uint32_t)((int)r + dir_off(code, kWP));
          code = s.rc[r + 1];
        }
        s.esc[r] = 1;
      }
      __syncthreads();
    }
    if (a.force_escape) {
      for (uint32_t i = s.lvs[0] + tid; i < s.lvs[nl > 0 ? 1 : 0]; i += kTTPB) {
        const uint32_t q = s.list[i];
        if (a.force_escape == 1 || (gcell(q) & 1u)) s.esc[q] = 1;
      }
      __syncthreads();
    }
    // ---- 6. drainage area
    if (EX) {
      // cell counts: every cell adds 1 to each ancestor (integer adds commute)
      for (uint32_t i = (nl > 1 ? s.lvs[1] : 0u) + tid; i < (nl > 1 ? s.lvs[nl] : 0u); i += kTTPB) {
        uint32_t p = s.list[i], code = s.rc[p + 1];
        do {
          p = (uint32_t)((int)p + dir_off(code, kWP));
          atomicAdd(reinterpret_cast<uint32_t*>(&s.acc[p]), 1u);
          code = s.rc[p + 1];
        } while (code != kNoFlowCode);
      }
      __syncthreads();
    } else {
      // deepest level first: A = w + the children's A in slot order (the
      // reference's FP summation order, accumulation.hpp:21-28)
      for (int l = (int)nl - 1; l >= 0; --l) {
        for (uint32_t i = s.lvs[l] + tid; i < s.lvs[l + 1]; i += kTTPB) {
          const uint32_t q = s.list[i];
          uint32_t m = s.dm[q];
          double A = a.w0;
          while (m) {
            const uint32_t k = __ffs(m) - 1;
            m &= m - 1;
            A = __dadd_rn(A, (double)s.acc[(int)q + dir_off(k, kWP)]);
          }
          s.acc[q] = A;
        }
        __syncthreads();
      }
    }
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
        e = s.esc[q] != 0;
        if (!e) {
          double hv = s.hw[q];
          if (inter) {
            hv = __dadd_rn(hv, a.du);
            s.hw[q] = hv;
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
    // erosion, downstream -> upstream, with the receiver's updated elevation
    for (uint32_t l = 1; l < nl; ++l) {
      bool any = false;
      for (uint32_t i = s.lvs[l] + tid; i < s.lvs[l + 1]; i += kTTPB) {
        const uint32_t q = s.list[i];
        const uint32_t code = s.rc[q + 1];
        const uint32_t p = (uint32_t)((int)q + dir_off(code, kWP));
        if (s.esc[p]) {  // the tree escapes: inherit the mark, leave the cell to the level path
          s.esc[q] = 1;
          continue;
        }
        any = true;
        ++cells;
        uint32_t mem = 0;
        if (a.M > 1) mem = (uint32_t)(wy0 + (int)(q / kWP)) / a.H;
        const uint32_t cls = dir_class(code);  // class of dist(c, rec[c])
        const double h0 = __dadd_rn(s.hw[q], a.du);  // uplift (every cell below level 0 is interior)
        const double hn = s.hw[p];
        int itn;
        bool ok;
        double hnew;
        if (tab) {
          const double2 fy = __ldg(reinterpret_cast<const double2*>(a.ftab2) + (mem * 3 + cls) * E + (uint32_t)s.acc[q]);
          hnew = newton_n1_tab(h0, hn, fy.x, fy.y, a.eps, a.maxit, itn, ok);
        } else {
          double F;
          if (EX)
            F = __ldg(a.ftab + (mem * 3 + cls) * E + (uint32_t)s.acc[q]);
          else
            F = tile_F(a, mem, cls, (double)s.acc[q], misses);
          if (NK == 1)
            hnew = newton_n1(h0, hn, F, a.eps, a.maxit, itn, ok);
          else
            hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, itn, ok);
        }
        const uint32_t gc = gcell(q);
        if (ok) {
          iters += (unsigned long long)itn;
        } else {
          atomicMin(&ctl->err_cell, gc);
          ctl->err_slot = ctl->slot;
          atomicMax(&ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
        }
        s.hw[q] = hnew;
        a.hout[gc] = hnew;
      }
      if (__syncthreads_or(any)) maxl = max(maxl, l + 1);
    }
    if (nl) maxl = max(maxl, 1u);
  }

  // ---- counters: one atomic per warp for the whole kernel
  for (int o = 16; o; o >>= 1) {
    iters += __shfl_down_sync(0xffffffffu, iters, o);
    misses += __shfl_down_sync(0xffffffffu, misses, o);
    n0i += __shfl_down_sync(0xffffffffu, n0i, o);
    cells += __shfl_down_sync(0xffffffffu, cells, o);
  }
  if (lane == 0) {
    if (iters) atomicAdd(&ctl->newton, iters);
    if (misses) atomicAdd(&ctl->misses, misses);
    if (n0i) atomicAdd(&ctl->n0i, n0i);
    if (cells) atomicAdd(&ctl->tile_cells, cells);
  }
  if (tid == 0) atomicMax(&ctl->tile_nlev, maxl);
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
