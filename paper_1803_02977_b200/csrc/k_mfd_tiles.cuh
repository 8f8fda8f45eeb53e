// k_mfd_tiles.cuh -- the MFD drainage area tile by tile (StepSetup::routing =
// kMfd, the accumulation that feeds the D8 erosion):
//
//   compute_mfd            proj/src/mfd.cpp:33-64  (lower mask + weight sum per cell)
//   build_mfd_donor_table  proj/src/mfd.cpp:8-31   (donor slots: ascending index = stencil order)
//   accumulate_mfd         proj/src/mfd.cpp:106-132, add_mfd_donor_flow mfd.hpp:66-73
//
// A[c] = w + sum over the donors n of c, in slot order, of alpha(n, c) * A[n]
// (alpha = RN(pow(slope, e) / wsum[n])): once every donor of c has its final
// value, evaluating this expression gives c the reference's bits, whatever
// order the cells are finalised in.  The reference orders the whole raster by
// dependency levels (generate_mfd_order) and sweeps them; a level-synchronous
// device sweep reads every level's cells scattered over the raster (~1.4 KB
// of DRAM traffic per cell at 10000^2).  Here a CTA owns a 64x32 tile: it
// stages the elevations of the tile and two rings, derives the lower masks
// and weight sums of the tile and its first ring, and finalises the tile's
// cells by in-tile dependency counting (a cell is ready when all its donors
// are final), level by level in shared memory.  A cell stays unfinished while
// a donor in another tile is unfinished; unfinished cells hold a NaN
// sentinel in the global A, so a donor's 8-byte value is either its final
// value or the sentinel.  Pass 0 runs every tile, reads no other tile and
// stores the lower masks and weight sums; pass 1 runs the tiles of a grid
// shifted by half a tile (chains that zig-zag along a pass-0 tile edge land
// inside one tile) that hold unfinished cells, reading the ring from
// the global A, and lists the cells still unfinished (~1 % of a random-noise
// DEM).  Those are finished by k_mfd_tail rounds (graph WHILE node): a listed
// cell whose donors are all final is evaluated, the others are listed again,
// until the list is empty.  Each cell is evaluated once, from final donors: A
// is exactly the reference's accumulation.
//
// The MFD plan itself (generate_mfd_order) is needed only by the export
// (lemgpu_download_mfd), which rebuilds it with k_mfd_graph + k_mfd_levels
// from the elevation the step read.
#pragma once

#include "common.cuh"
#include "k_mfd.cuh"

namespace lemgpu {

#ifndef LEMGPU_MFD_TY
#define LEMGPU_MFD_TY 28  // 64x28: 55 KB of shared memory, 4 CTAs per SM (measured best of 16/24/28/32/48/64)
#endif
#ifndef LEMGPU_MFD_TPB
#define LEMGPU_MFD_TPB 256
#endif
constexpr int kMX = 64, kMY = LEMGPU_MFD_TY;  // tile
constexpr int kMP = kMX + 2;            // window pitch: the tile and one ring
constexpr int kMWY = kMY + 2;           // window rows
constexpr int kMN = kMP * kMWY;         // window cells
constexpr int kMT = kMX * kMY;          // tile cells
constexpr int kMTPB = LEMGPU_MFD_TPB;
constexpr unsigned long long kMfdUnset = 0x7FF4DEAD00000000ull;  // NaN payload: not final yet

// Tiles of grid g (0: origin (0, 0); 1: shifted by (-kMX/2, -kMY/2)).
__host__ __device__ __forceinline__ uint32_t mfd_ntx(uint32_t W, int g) { return (W + (g ? kMX / 2 : 0) + kMX - 1) / kMX; }
__host__ __device__ __forceinline__ uint32_t mfd_nty(uint32_t H, int g) { return (H + (g ? kMY / 2 : 0) + kMY - 1) / kMY; }
// work-list / stamp capacity per grid
__host__ __device__ __forceinline__ uint32_t mfd_cap(uint32_t W, uint32_t H) {
  const uint32_t a = mfd_ntx(W, 0) * mfd_nty(H, 0), b = mfd_ntx(W, 1) * mfd_nty(H, 1);
  return a > b ? a : b;
}

struct MfdTileSmem {
  double h[kMN];        // window elevations (0 off the raster: never read for an existing neighbour)
  double ws[kMN];       // weight sums (tile; pass 1: and ring)
  double A[kMN];        // drainage area: final value or the kMfdUnset bits
  alignas(4) uint8_t rem[kMT];  // unfinished donors of an unfinished tile cell (byte countdowns, word atomics)
  uint16_t list[kMT];   // cells finalised in this visit, level-major
  uint8_t lm[kMN];      // mask of strictly lower neighbours (0: boundary / off raster); ring cells in
                        // pass 0: only the bits towards the window
  uint32_t cnt[3];      // per-level append counters (rotating)
  uint32_t mark;        // next-grid tiles to queue: bit dy*2 + dx
  uint32_t pass, n, g;  // pass id, work items and grid of this pass
};
constexpr size_t kMfdTileSmemBytes = sizeof(MfdTileSmem);

__device__ __forceinline__ int mwoff(int k) { return dir_ox(k) + dir_oy(k) * kMP; }
__device__ __forceinline__ bool m_in_tile(int q) {
  const int y = q / kMP, x = q - y * kMP;
  return (unsigned)(x - 1) < (unsigned)kMX && (unsigned)(y - 1) < (unsigned)kMY;
}
__device__ __forceinline__ bool m_unset(double v) { return (unsigned long long)__double_as_longlong(v) == kMfdUnset; }

// Pass 0 (a.mfd_all: every tile of grid 0) or pass 1 (the queued tiles of grid 1).
__global__ void __launch_bounds__(kMTPB) k_mfd_tiles(StepArgs a) {
  extern __shared__ __align__(16) unsigned char mraw[];
  MfdTileSmem& s = *reinterpret_cast<MfdTileSmem*>(mraw);
  Ctl* ctl = a.ctl;
  const int all = a.mfd_all;
  const uint32_t tid = threadIdx.x;
  PhWhole ph(ctl, LEMGPU_PHASE_ACCUM);
  if (tid == 0) {
    if (all) atomicMin(&ctl->t_mfd_begin, globaltimer());
    const uint32_t P = ld_volatile_u32(&ctl->mfd_pass);
    const uint32_t g = all ? 0u : 1u;
    s.pass = P;
    s.g = g;
    s.n = ld_volatile_u32(&ctl->err_flag) ? 0u
          : all ? mfd_ntx(a.W, 0) * mfd_nty(a.Htot, 0) : ld_volatile_u32(&ctl->mfd_wl_n[P & 1u]);
  }
  __syncthreads();
  const uint32_t P = s.pass, nitems = s.n;
  const int g = (int)s.g;
  const uint32_t ntx = mfd_ntx(a.W, g);
  const uint32_t ntx1 = mfd_ntx(a.W, g ^ 1), nty1 = mfd_nty(a.Htot, g ^ 1);
  const uint32_t cap = mfd_cap(a.W, a.Htot);
  const uint32_t* wl = a.mfd_wl + (size_t)(P & 1u) * cap;
  uint32_t* wl_next = a.mfd_wl + (size_t)((P + 1u) & 1u) * cap;
  const int W = (int)a.W, Ht = (int)a.Htot;
  const int sx = g ? kMX / 2 : 0, sy = g ? kMY / 2 : 0;          // this grid's shift
  const int nsx = g ? 0 : kMX / 2, nsy = g ? 0 : kMY / 2;        // the next grid's
  uint32_t done = 0;                                             // cells this CTA finalised
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint32_t t = all ? it : __ldcg(wl + it);
    const int tx = (int)(t % ntx), ty = (int)(t / ntx);
    const int x0 = tx * kMX - sx, y0 = ty * kMY - sy;  // first tile cell
    const int wx0 = x0 - 1, wy0 = y0 - 1;
    __syncthreads();  // the previous tile is done with shared memory
    // ---- stage: window elevations; A of the tile and the ring (pass 0:
    // nothing is final yet -- other tiles' values may be a previous step's)
    uint32_t unf = 0;
    for (int i = (int)tid; i < kMN; i += kMTPB) {
      const int y = i / kMP, x = i - y * kMP, gx = wx0 + x, gy = wy0 + y;
      const bool in = gx >= 0 && gx < W && gy >= 0 && gy < Ht;
      const size_t g0 = (size_t)gy * a.W + gx;
      s.h[i] = in ? __ldg(a.h + g0) : 0.0;
      const double v = in && !all ? __ldcg(a.mfd_A + g0) : __longlong_as_double((long long)kMfdUnset);
      s.A[i] = v;
      unf += in && m_in_tile(i) && m_unset(v) ? 1u : 0u;
    }
    if (tid < 3) s.cnt[tid] = 0;
    if (tid == 0) s.mark = 0;
    if (__syncthreads_count(unf != 0) == 0) continue;  // every cell of this tile is final
    // ---- compute_mfd for the tile: lower mask, weight sum; for a ring cell
    // only its lower mask towards the window (pass 0 reads no other tile's
    // values, so a ring donor only blocks its receivers).  Pass 1: the tile
    // and the ring as pass 0 stored them.
    if (!all) {
      for (int i = (int)tid; i < kMN; i += kMTPB) {
        const int y = i / kMP, x = i - y * kMP, gx = wx0 + x, gy = wy0 + y;
        const bool in = gx >= 0 && gx < W && gy >= 0 && gy < Ht;
        const size_t g0 = (size_t)gy * a.W + gx;
        s.lm[i] = in ? __ldcg(a.mfd_lm + g0) : (uint8_t)0;
        s.ws[i] = in ? __ldcg(a.mfd_wsum + g0) : 0.0;
      }
    } else
    for (int i = (int)tid; i < kMN; i += kMTPB) {
      const int y = i / kMP, x = i - y * kMP, gx = wx0 + x, gy = wy0 + y;
      uint32_t m = 0;
      double wsum = 0.0;
      const bool tc = m_in_tile(i);
      if (gx > 0 && gx < W - 1 && gy > 0 && gy < Ht) {
        const uint32_t yl = (uint32_t)gy % a.H;
        if (yl > 0 && yl < a.H - 1) {  // interior (boundary cells have no receivers, mfd.cpp:43)
          const double hc = s.h[i];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (!dir_in(a.conn, k)) continue;
            if (!tc && (unsigned)(x + dir_ox(k)) >= (unsigned)kMP) continue;  // ring cell: in-window bits only
            if (!tc && (unsigned)(y + dir_oy(k)) >= (unsigned)kMWY) continue;
            const double hn = s.h[i + mwoff(k)];
            if (hn >= hc) continue;  // receivers must be strictly lower (mfd.cpp:48)
            if (tc) wsum = __dadd_rn(wsum, mfd_weight(a, mfd_slope(a, hc, hn, k)));
            m |= 1u << k;
          }
        }
      }
      s.lm[i] = (uint8_t)m;
      s.ws[i] = wsum;
      if (m_in_tile(i) && gx >= 0 && gx < W && gy >= 0 && gy < Ht) {  // for pass 1 and the tail rounds
        const size_t g0 = (size_t)gy * a.W + gx;
        __stcg(a.mfd_lm + g0, (uint8_t)m);
        __stcg(a.mfd_wsum + g0, wsum);
      }
    }
    __syncthreads();
    // ---- unfinished tile cells: count their unfinished donors; level 0 = none
    for (int j = (int)tid; j < kMT; j += kMTPB) {
      const int q = (j / kMX + 1) * kMP + (j % kMX) + 1;
      if (!m_unset(s.A[q]) || x0 + j % kMX >= W || y0 + j / kMX >= Ht || x0 + j % kMX < 0 || y0 + j / kMX < 0)
        continue;
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int n = q + mwoff(k);
        r += (((s.lm[n] >> (7 - k)) & 1u) && m_unset(s.A[n])) ? 1u : 0u;
      }
      s.rem[j] = (uint8_t)r;
      if (r == 0) s.list[atomicAdd(&s.cnt[0], 1u)] = (uint16_t)q;
    }
    __syncthreads();
    // ---- levels: evaluate A (every donor final), release the in-tile receivers
    uint32_t qs = 0, qe = s.cnt[0];
    for (uint32_t l = 0; qs < qe; ++l) {
      uint32_t* nc = &s.cnt[(l + 1) % 3];
      if (tid == 0) s.cnt[(l + 2) % 3] = 0;  // last read before the previous barrier
      for (uint32_t i = qs + tid; i < qe; i += kMTPB) {
        const int q = s.list[i];
        const double hc = s.h[q];
        // the donors' terms first, then their sum in slot order (ascending
        // index = stencil order).  All eight directions are evaluated without
        // branches (a non-donor gets harmless operands and is masked out of the
        // sum): the lanes of a warp stay converged and the eight division
        // chains overlap.
        double tk[8];
        uint32_t dm = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int n = q + mwoff(k);
          const bool don = dir_in(a.conn, k) && ((s.lm[n] >> (7 - k)) & 1u);
          dm |= don ? 1u << k : 0u;
          // n's weight towards q: its slope in direction 7-k (same length as k)
          const double d = don ? __dsub_rn(s.h[n], hc) : 1.0;
          const double sl = ((a.dist_one >> k) & 1u) ? d
                            : ((a.dist_recip >> k) & 1u) ? div_rn_recip(d, a.dist[k], a.rdist[k])
                                                         : __ddiv_rn(d, a.dist[k]);
          const double w = mfd_weight(a, sl);
          tk[k] = __dmul_rn(__ddiv_rn(w, don ? s.ws[n] : 1.0), don ? s.A[n] : 0.0);
        }
        double acc = a.w0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if ((dm >> k) & 1u) acc = __dadd_rn(acc, tk[k]);
        s.A[q] = acc;
        for (uint32_t m = s.lm[q]; m; m &= m - 1) {
          const int r = q + mwoff(__ffs(m) - 1);
          if (!m_in_tile(r)) continue;
          const int j = (r / kMP - 1) * kMX + (r % kMP) - 1;
          const uint32_t sh = 8u * (uint32_t)(j & 3);
          if (((atomicSub(reinterpret_cast<uint32_t*>(s.rem) + (j >> 2), 1u << sh) >> sh) & 0xFFu) == 1u)
            s.list[qe + atomicAdd(nc, 1u)] = (uint16_t)r;
        }
      }
      __syncthreads();
      qs = qe;
      qe += *reinterpret_cast<volatile uint32_t*>(nc);
    }
    done += tid == 0 ? qe : 0u;
    // ---- write the finalised cells (pass 0: every tile cell, final or the
    // sentinel); the next grid's tiles holding cells still unfinished are queued
    for (int j = (int)tid; j < kMT; j += kMTPB) {
      const int y = j / kMX, x = j - y * kMX, gx = x0 + x, gy = y0 + y;
      if (gx < 0 || gx >= W || gy < 0 || gy >= Ht) continue;
      const int q = (y + 1) * kMP + x + 1;
      const double v = s.A[q];
      if (m_unset(v)) {
        if (all) {  // pass 0: the pass-1 tile holding the cell is queued
          const int ix = (gx + nsx) / kMX - (x0 + nsx) / kMX, iy = (gy + nsy) / kMY - (y0 + nsy) / kMY;
          atomicOr(&s.mark, 1u << (iy * 2 + ix));
          __stcg(a.mfd_A + (size_t)gy * a.W + gx, v);
        } else {  // pass 1: listed for the tail rounds
          a.mfd_ord[atomicAdd(&ctl->mfd_tail_n[0], 1u)] = (uint32_t)gy * a.W + (uint32_t)gx;
        }
      } else {
        __stcg(a.mfd_A + (size_t)gy * a.W + gx, v);
      }
    }
    __syncthreads();
    if (tid < 4 && ((s.mark >> tid) & 1u)) {
      const uint32_t nx = (uint32_t)((x0 + nsx) / kMX + (int)(tid & 1u));
      const uint32_t ny = (uint32_t)((y0 + nsy) / kMY + (int)(tid >> 1));
      if (nx < ntx1 && ny < nty1) {
        const uint32_t tn = ny * ntx1 + nx;
        if (atomicExch(a.mfd_stamp + (size_t)(g ^ 1) * cap + tn, P + 1u) != P + 1u)
          wl_next[atomicAdd(&ctl->mfd_wl_n[(P + 1u) & 1u], 1u)] = tn;
      }
    }
  }
  if (tid == 0 && done) atomicAdd(&ctl->mfd_done, done);
  // ---- the last CTA closes the pass; after pass 1 the tail rounds run if
  // cells are left (list 0)
  if (last_block_done(ctl) && tid == 0) {
    ctl->mfd_done = 0;
    ctl->mfd_wl_n[P & 1u] = 0;
    ctl->mfd_pass = P + 1u;
    ctl->mfd_passes += 1u;
    if (!all) {
      ctl->mfd_tail_cur = 0;
      set_cond(a, 3, ld_volatile_u32(&ctl->mfd_tail_n[0]) ? 1u : 0u);
    }
  }
}

// One tail round: every listed cell whose donors are all final is evaluated
// (add_mfd_donor_flow, mfd.hpp:66-73); the others are listed for the next
// round.  A donor finalised by another thread during the round may or may not
// be seen: either way a cell is only evaluated from final donors.
__global__ void __launch_bounds__(kTPB) k_mfd_tail(StepArgs a) {
  Ctl* ctl = a.ctl;
  const uint32_t cur = ld_volatile_u32(&ctl->mfd_tail_cur), nxt = cur ^ 1u;
  const uint32_t n = ld_volatile_u32(&ctl->err_flag) ? 0u : ld_volatile_u32(&ctl->mfd_tail_n[cur]);
  const uint32_t* lst = cur ? a.mfd_lev : a.mfd_ord;
  uint32_t* lnx = cur ? a.mfd_ord : a.mfd_lev;
  const uint32_t lane = threadIdx.x & 31u;
  const int W = (int)a.W;
  uint32_t done = 0;
  for (uint32_t i0 = blockIdx.x * kTPB; i0 < n; i0 += gridDim.x * kTPB) {  // warp-uniform trip count
    const uint32_t i = i0 + threadIdx.x;
    bool left = false;
    if (i < n) {
      const uint32_t c = __ldcg(lst + i);
      const uint32_t y = c / a.W, x = c - y * a.W;
      const double hc = __ldg(a.h + c);
      double tk[8];
      uint32_t dm = 0;
      bool ready = true;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        tk[k] = 0.0;
        const uint32_t nx = x + dir_ox(k), ny = y + dir_oy(k);
        if (!dir_in(a.conn, k) || nx >= a.W || ny >= a.Htot) continue;
        const uint32_t nb = (uint32_t)((int)c + dir_ox(k) + dir_oy(k) * W);
        if (!((__ldcg(a.mfd_lm + nb) >> (7 - k)) & 1u)) continue;
        const double An = __ldcg(a.mfd_A + nb);
        if (m_unset(An)) {
          ready = false;
          continue;
        }
        dm |= 1u << k;
        const double w = mfd_weight(a, mfd_slope(a, __ldg(a.h + nb), hc, 7 - k));
        tk[k] = __dmul_rn(__ddiv_rn(w, __ldcg(a.mfd_wsum + nb)), An);
      }
      if (ready) {
        double acc = a.w0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if ((dm >> k) & 1u) acc = __dadd_rn(acc, tk[k]);
        __stcg(a.mfd_A + c, acc);
        ++done;
      } else {
        left = true;
      }
      if (left) {
        const uint32_t b = __activemask(), bl = __ballot_sync(b, true);  // lanes still unfinished
        const int ld = __ffs(bl) - 1;
        uint32_t p = 0;
        if ((int)lane == ld) p = atomicAdd(&ctl->mfd_tail_n[nxt], (uint32_t)__popc(bl));
        p = __shfl_sync(bl, p, ld);
        lnx[p + __popc(bl & ((1u << lane) - 1u))] = c;
      }
    }
  }
  for (int o = 16; o; o >>= 1) done += __shfl_xor_sync(0xffffffffu, done, o);
  if (lane == 0 && done) atomicAdd(&ctl->mfd_done, done);
  if (last_block_done(ctl) && threadIdx.x == 0) {
    const uint32_t nn = ld_volatile_u32(&ctl->mfd_tail_n[nxt]);
    const uint32_t fin = ld_volatile_u32(&ctl->mfd_done);
    ctl->mfd_done = 0;
    ctl->mfd_tail_n[cur] = 0;
    ctl->mfd_tail_cur = nxt;
    ctl->mfd_passes += 1u;
    bool more = nn != 0;
    if (more && fin == 0 && n) {  // no progress: a cycle (impossible with strict descent), reported
      more = false;
      ctl->mfd_tail_n[nxt] = 0;
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_cell = 0;
      ctl->err_slot = ctl->slot;
    }
    set_cond(a, 3, more ? 1u : 0u);
  }
}

}  // namespace lemgpu
