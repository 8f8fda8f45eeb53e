// k_mfd_tiles.cuh -- the MFD drainage area tile by tile (StepSetup::routing =
// kMfd, the accumulation that feeds the D8 erosion):
//
//   compute_mfd            proj/src/mfd.cpp:33-64  (lower mask + weight sum per cell)
//   build_mfd_donor_table  proj/src/mfd.cpp:8-31   (donor slots: ascending index = stencil order)
//   accumulate_mfd         proj/src/mfd.cpp:106-132, add_mfd_donor_flow mfd.hpp:66-73
//
// A[c] = w + sum over the donors n of c, in slot order, of alpha(n, c) * A[n]
// (alpha = RN(pow(slope, e) / wsum[n])): every cell's value is one fixed
// function of its donors' values, and the donors are strictly higher, so the
// system has exactly one solution -- the reference's bits -- and any
// evaluation order that reads final donor values reproduces them.  The
// reference orders the whole raster by dependency levels (generate_mfd_order)
// and sweeps them; a level-synchronous sweep on the device reads every
// level's cells scattered over the raster (~1.4 KB of DRAM traffic per cell at
// 10000^2).  Here a CTA owns a 64x32 tile: it stages the tile's elevations
// with two rings, derives the lower masks and weight sums of the tile and its
// first ring, orders the tile's cells by in-tile dependency counting (a cell
// is ready when its donors inside the tile are done) and evaluates A level by
// level in shared memory; donors in the ring contribute the values currently
// in the global A.  A tile whose border cells changed the value that a
// neighbouring tile reads (a cell with a receiver across the tile edge)
// queues that neighbour for the next pass.  Pass 0 runs every tile; the
// passes repeat (graph WHILE node) until a pass queues nothing.  Then every
// tile was last evaluated on inputs equal to the current values: the global
// A is the fixed point, i.e. exactly the reference's accumulation.  (The
// number of passes is bounded by how often a dependency chain crosses tile
// edges, ~12 at 1000^2 random noise; the late passes touch a few tiles.)
//
// The MFD plan itself (generate_mfd_order) is needed only by the export
// (lemgpu_download_mfd), which rebuilds it with k_mfd_graph + k_mfd_levels
// from the elevation the step read.
#pragma once

#include "common.cuh"
#include "k_mfd.cuh"

namespace lemgpu {

constexpr int kMX = 64, kMY = 32;       // tile
constexpr int kMP = kMX + 4;            // window pitch: the tile and two rings
constexpr int kMWY = kMY + 4;           // window rows
constexpr int kMN = kMP * kMWY;         // window cells
constexpr int kMT = kMX * kMY;          // tile cells
constexpr int kMTPB = 256;
constexpr uint32_t kMfdMaxPasses = 1u << 20;  // safety bound (a DAG converges far earlier)

struct MfdTileSmem {
  double h[kMN];        // window elevations (0 off the raster: never read for an existing neighbour)
  double ws[kMN];       // weight sums (tile + first ring; interior cells)
  double A[kMN];        // drainage area: first ring from the global A, tile evaluated here
  uint32_t rem[kMT];    // in-tile donors not yet evaluated
  uint16_t list[kMT];   // the tile's cells, dependency-level-major
  uint8_t lm[kMN];      // mask of strictly lower neighbours (0: boundary / off raster / outer ring)
  uint32_t cnt[3];      // per-level append counters (rotating)
  uint32_t mark;        // neighbour tiles to queue: bit (dy+1)*3 + (dx+1)
  uint32_t pass, n;     // pass id, work items of this pass
};
constexpr size_t kMfdTileSmemBytes = sizeof(MfdTileSmem);

__device__ __forceinline__ int mwoff(int k) { return dir_ox(k) + dir_oy(k) * kMP; }
__device__ __forceinline__ bool m_in_tile(int q) {
  const int y = q / kMP, x = q - y * kMP;
  return (unsigned)(x - 2) < (unsigned)kMX && (unsigned)(y - 2) < (unsigned)kMY;
}

// One pass over the queued tiles (a.mfd_all: every tile, pass 0 of the step).
__global__ void __launch_bounds__(kMTPB) k_mfd_tiles(StepArgs a) {
  extern __shared__ __align__(16) unsigned char mraw[];
  MfdTileSmem& s = *reinterpret_cast<MfdTileSmem*>(mraw);
  Ctl* ctl = a.ctl;
  const int all = a.mfd_all;
  const uint32_t tid = threadIdx.x;
  const uint32_t ntx = (a.W + kMX - 1) / kMX, nty = (a.Htot + kMY - 1) / kMY, ntiles = ntx * nty;
  PhWhole ph(ctl, LEMGPU_PHASE_ACCUM);
  if (tid == 0) {
    if (all) atomicMin(&ctl->t_mfd_begin, globaltimer());
    const uint32_t P = ld_volatile_u32(&ctl->mfd_pass);
    s.pass = P;
    s.n = ld_volatile_u32(&ctl->err_flag) ? 0u : all ? ntiles : ld_volatile_u32(&ctl->mfd_wl_n[P & 1u]);
  }
  __syncthreads();
  const uint32_t P = s.pass, nitems = s.n;
  const uint32_t* wl = a.mfd_wl + (size_t)(P & 1u) * ntiles;
  uint32_t* wl_next = a.mfd_wl + (size_t)((P + 1u) & 1u) * ntiles;
  const int W = (int)a.W, Ht = (int)a.Htot;
  for (uint32_t it = blockIdx.x; it < nitems; it += gridDim.x) {
    const uint32_t t = all ? it : __ldcg(wl + it);
    const int tx = (int)(t % ntx), ty = (int)(t / ntx);
    const int wx0 = tx * kMX - 2, wy0 = ty * kMY - 2;
    __syncthreads();  // the previous tile is done with shared memory
    // ---- stage: elevations of the window, the global A of the first ring
    for (int i = (int)tid; i < kMN; i += kMTPB) {
      const int y = i / kMP, x = i - y * kMP, gx = wx0 + x, gy = wy0 + y;
      const bool in = gx >= 0 && gx < W && gy >= 0 && gy < Ht;
      const size_t g = (size_t)gy * a.W + gx;
      s.h[i] = in ? __ldg(a.h + g) : 0.0;
      const bool ring1 = x >= 1 && x < kMP - 1 && y >= 1 && y < kMWY - 1 && !m_in_tile(i);
      if (ring1) s.A[i] = in ? __ldcg(a.mfd_A + g) : 0.0;
    }
    if (tid < 3) s.cnt[tid] = 0;
    if (tid == 0) s.mark = 0;
    __syncthreads();
    // ---- compute_mfd for the tile and its first ring: lower mask, weight sum
    for (int i = (int)tid; i < kMN; i += kMTPB) {
      const int y = i / kMP, x = i - y * kMP, gx = wx0 + x, gy = wy0 + y;
      uint32_t m = 0;
      double wsum = 0.0;
      if (x >= 1 && x < kMP - 1 && y >= 1 && y < kMWY - 1 && gx > 0 && gx < W - 1 && gy > 0 && gy < Ht) {
        const uint32_t yl = (uint32_t)gy % a.H;
        if (yl > 0 && yl < a.H - 1) {  // interior (boundary cells have no receivers, mfd.cpp:43)
          const double hc = s.h[i];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (!dir_in(a.conn, k)) continue;
            const double hn = s.h[i + mwoff(k)];
            if (hn >= hc) continue;  // receivers must be strictly lower (mfd.cpp:48)
            wsum = __dadd_rn(wsum, mfd_weight(a, mfd_slope(a, hc, hn, k)));
            m |= 1u << k;
          }
        }
      }
      s.lm[i] = (uint8_t)m;
      s.ws[i] = wsum;
    }
    __syncthreads();
    // ---- in-tile dependency counts; level 0 = cells without donors in the tile
    for (int j = (int)tid; j < kMT; j += kMTPB) {
      const int q = (j / kMX + 2) * kMP + (j % kMX) + 2;
      uint32_t r = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int n = q + mwoff(k);
        r += (m_in_tile(n) && ((s.lm[n] >> (7 - k)) & 1u)) ? 1u : 0u;
      }
      s.rem[j] = r;
      if (r == 0) s.list[atomicAdd(&s.cnt[0], 1u)] = (uint16_t)q;
    }
    __syncthreads();
    // ---- levels: evaluate A, release the in-tile receivers
    uint32_t qs = 0, qe = s.cnt[0];
    for (uint32_t l = 0; qs < qe; ++l) {
      uint32_t* nc = &s.cnt[(l + 1) % 3];
      if (tid == 0) s.cnt[(l + 2) % 3] = 0;  // last read before the previous barrier
      for (uint32_t i = qs + tid; i < qe; i += kMTPB) {
        const int q = s.list[i];
        const double hc = s.h[q];
        double acc = a.w0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {  // donors in slot order (ascending index = stencil order)
          const int n = q + mwoff(k);
          if (!dir_in(a.conn, k) || !((s.lm[n] >> (7 - k)) & 1u)) continue;
          // n's weight towards q: its slope in direction 7-k (same length as k)
          const double w = mfd_weight(a, mfd_slope(a, s.h[n], hc, 7 - k));
          acc = __dadd_rn(acc, __dmul_rn(__ddiv_rn(w, s.ws[n]), s.A[n]));
        }
        s.A[q] = acc;
        for (uint32_t m = s.lm[q]; m; m &= m - 1) {
          const int r = q + mwoff(__ffs(m) - 1);
          if (!m_in_tile(r)) continue;
          const int j = (r / kMP - 2) * kMX + (r % kMP) - 2;
          if (atomicSub(&s.rem[j], 1u) == 1u) s.list[qe + atomicAdd(nc, 1u)] = (uint16_t)r;
        }
      }
      __syncthreads();
      qs = qe;
      qe += *reinterpret_cast<volatile uint32_t*>(nc);
    }
    // ---- write the tile; a changed value that a neighbouring tile reads
    // (a receiver across the tile edge) queues that tile
    for (int j = (int)tid; j < kMT; j += kMTPB) {
      const int y = j / kMX, x = j - y * kMX, gx = tx * kMX + x, gy = ty * kMY + y;
      if (gx >= W || gy >= Ht) continue;
      const int q = (y + 2) * kMP + x + 2;
      const size_t g = (size_t)gy * a.W + gx;
      const double v = s.A[q];
      uint32_t out = 0;  // receivers in other tiles
      if (x == 0 || x == kMX - 1 || y == 0 || y == kMY - 1)
        for (uint32_t m = s.lm[q]; m; m &= m - 1) {
          const int k = __ffs(m) - 1;
          const int rx = x + dir_ox(k), ry = y + dir_oy(k);
          const int dx = rx < 0 ? -1 : rx >= kMX ? 1 : 0, dy = ry < 0 ? -1 : ry >= kMY ? 1 : 0;
          if (dx || dy) out |= 1u << ((dy + 1) * 3 + dx + 1);
        }
      if (out && __double_as_longlong(__ldcg(a.mfd_A + g)) != __double_as_longlong(v)) atomicOr(&s.mark, out);
      __stcg(a.mfd_A + g, v);
    }
    __syncthreads();
    if (tid < 9 && ((s.mark >> tid) & 1u)) {
      const int nx = tx + (int)(tid % 3) - 1, ny = ty + (int)(tid / 3) - 1;
      if (nx >= 0 && nx < (int)ntx && ny >= 0 && ny < (int)nty) {
        const uint32_t tn = (uint32_t)ny * ntx + (uint32_t)nx;
        __threadfence();  // the tile's new values before the queue entry
        if (atomicExch(a.mfd_stamp + tn, P + 1u) != P + 1u)
          wl_next[atomicAdd(&ctl->mfd_wl_n[(P + 1u) & 1u], 1u)] = tn;
      }
    }
  }
  // ---- the last CTA closes the pass: the next pass runs if it has work
  if (last_block_done(ctl) && tid == 0) {
    const uint32_t nn = ld_volatile_u32(&ctl->mfd_wl_n[(P + 1u) & 1u]);
    ctl->mfd_wl_n[P & 1u] = 0;
    ctl->mfd_pass = P + 1u;
    ctl->mfd_passes += 1u;
    bool more = nn != 0;
    if (more && ctl->mfd_passes >= kMfdMaxPasses) {  // cannot happen on a DAG; reported, never looped forever
      more = false;
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_slot = ctl->slot;
    }
    set_cond(a, 3, more ? 1u : 0u);
  }
}

}  // namespace lemgpu
