// k_mfd.cuh -- multiple-flow-direction accumulation (StepSetup::routing =
// kMfd): the drainage area that feeds the erosion, which still follows the
// D8 receiver (proj/include/lem/config.hpp:18-19, simulation.cpp:53-60).
//
//   compute_mfd            proj/src/mfd.cpp:33-64
//   build_mfd_donor_table  proj/src/mfd.cpp:8-31   (donor slots = ascending index = stencil order)
//   generate_mfd_order     proj/src/mfd.cpp:66-104 (dependency counting)
//   accumulate_mfd         proj/src/mfd.cpp:106-132, add_mfd_donor_flow mfd.hpp:62-69
//
// The reference materialises an 8-slot receiver table, its inverse donor
// table and per-slot weights (~150 B per cell).  Here a cell keeps only its
// lower-neighbour mask (1 B) and the sum of its weights (8 B): a donor n of c
// is a neighbour whose mask has c's direction, and its weight
// pow((h[n] - h[c]) / dist, e) is recomputed from the elevations with the
// reference's operations, so alpha(n, c) = RN(w / wsum[n]) has the reference's
// bits.  The plan is the reference's dependency counting, level by level in
// one cooperative kernel: level 0 = cells without lower neighbours; a cell
// joins level l+1 when the last of its receivers is placed (atomic countdown
// -- the level a cell lands in does not depend on the order of the
// decrements).  The accumulation pulls each cell's donors in slot order,
// highest level first, so every donor is final when read: A has the
// reference's bits.  Within a level the cells sit in any order; the export
// (lemgpu_download_mfd) sorts them the reference's way.
#pragma once

#include "common.cuh"
#include "k_physics.cuh"

namespace lemgpu {

// Whether cell c (stacked rows: member perimeters included) is a boundary cell.
__device__ __forceinline__ bool mfd_boundary(const StepArgs& a, uint32_t c) { return !is_interior(a, c); }

// w = pow(slope, e) with the host glibc's bits (e == 1: the identity, exactly).
__device__ __forceinline__ double mfd_weight(const StepArgs& a, double slope) {
  return a.mfd_exp == 1.0 ? slope : glibc_pow_dev(a.pow_fma, slope, a.mfd_exp);
}

// slope = (h[c] - h[nb]) / dist[k]: exact for dist == 1, else the correctly
// rounded quotient from the host reciprocal (div_rn_recip) or by IEEE division.
__device__ __forceinline__ double mfd_slope(const StepArgs& a, double hc, double hn, int k) {
  const double d = __dsub_rn(hc, hn);
  if ((a.dist_one >> k) & 1u) return d;
  return ((a.dist_recip >> k) & 1u) ? div_rn_recip(d, a.dist[k], a.rdist[k]) : __ddiv_rn(d, a.dist[k]);
}

// compute_mfd per cell: the mask of strictly lower neighbours (stencil
// order) and the sum of their weights, accumulated in stencil order; the
// receiver countdown of the plan starts at the number of receivers.
__global__ void __launch_bounds__(kTPB) k_mfd_graph(StepArgs a) {
  const uint32_t N = a.N;
  const int W = (int)a.W;
  for (uint32_t c = blockIdx.x * kTPB + threadIdx.x; c < N; c += gridDim.x * kTPB) {
    uint32_t m = 0;
    double ws = 0.0;
    if (!mfd_boundary(a, c)) {
      const double hc = __ldg(a.h + c);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!dir_in(a.conn, k)) continue;
        const double hn = __ldg(a.h + (uint32_t)((int)c + dir_ox(k) + dir_oy(k) * W));
        if (hn >= hc) continue;  // receivers must be strictly lower (mfd.cpp:48)
        ws = __dadd_rn(ws, mfd_weight(a, mfd_slope(a, hc, hn, k)));
        m |= 1u << k;
      }
    }
    a.mfd_lm[c] = (uint8_t)m;
    a.mfd_wsum[c] = ws;
    a.mfd_rem[c] = (uint32_t)__popc(m);
  }
}

// Donor mask of c: neighbour k is a donor when c is one of its receivers
// (its lower mask has the opposite direction 7-k).  Off-raster neighbours
// are skipped; boundary cells have an empty mask, so they are never donors.
__device__ __forceinline__ uint32_t mfd_donors(const StepArgs& a, uint32_t c) {
  const uint32_t y = c / a.W, x = c - y * a.W;
  uint32_t m = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!dir_in(a.conn, k)) continue;
    const uint32_t nx = x + dir_ox(k), ny = y + dir_oy(k);
    if (nx >= a.W || ny >= a.Htot) continue;
    if ((__ldcg(a.mfd_lm + ny * a.W + nx) >> (7 - k)) & 1u) m |= 1u << k;
  }
  return m;
}

// The MFD plan and the accumulation in one cooperative kernel (grid
// barriers between levels).
__global__ void __launch_bounds__(kTPB) k_mfd_levels(StepArgs a) {
  __shared__ uint32_t scan[kNW + 1];
  __shared__ uint32_t s_base;
  Ctl* ctl = a.ctl;
  const uint32_t N = a.N, G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const uint32_t gstride = G * kTPB;
  const int W = (int)a.W;
  PhWhole ph(ctl, LEMGPU_PHASE_ACCUM);
  // ---- level 0: the cells without receivers, ascending (one segment per CTA)
  const uint32_t S = (N + G - 1) / G, c0 = min(b * S, N), c1 = min(c0 + S, N);
  {
    uint32_t cnt = 0;
    for (uint32_t c = c0 + tid; c < c1; c += kTPB) cnt += __ldcg(a.mfd_rem + c) == 0u ? 1u : 0u;
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) scan[tid >> 5] = cnt;
    __syncthreads();
    if (tid == 0) {
      uint32_t t = 0;
      for (int j = 0; j < kNW; ++j) t += scan[j];
      a.part[b] = t;
    }
  }
  if (b == 0 && tid < 3) ctl->mfd_cnt[tid] = 0;
  grid_barrier(ctl);
  {
    if (tid == 0) {
      uint32_t base = 0, tot = 0;
      for (uint32_t j = 0; j < G; ++j) {
        const uint32_t v = __ldcg(a.part + j);
        base += j < b ? v : 0u;
        tot += v;
      }
      s_base = base;
      if (b == 0) {
        a.mfd_lv[0] = 0;
        a.mfd_lv[1] = tot;
      }
    }
    __syncthreads();
    uint32_t carry = s_base;
    for (uint32_t t0 = c0; t0 < c1; t0 += kTPB) {
      const uint32_t c = t0 + tid;
      const bool z = c < c1 && __ldcg(a.mfd_rem + c) == 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan(z ? 1u : 0u, &tot, scan);
      if (z) {
        a.mfd_ord[carry + ex] = c;
        a.mfd_lev[c] = 0;
      }
      carry += tot;
    }
  }
  grid_barrier(ctl);
  // ---- level l+1: donors of level l whose countdown reaches zero, appended
  // after level l (per-level counters, three in rotation: the one cleared
  // during level l was last read two barriers ago)
  uint32_t lo = 0, hi = __ldcg(a.mfd_lv + 1), nl = 1;
  while (hi > lo) {
    uint32_t* cnt = &ctl->mfd_cnt[nl % 3];
    if (b == 0 && tid == 0) ctl->mfd_cnt[(nl + 1) % 3] = 0;
    for (uint32_t i0 = lo + b * kTPB; i0 < hi; i0 += gstride) {  // warp-uniform trip count
      const uint32_t i = i0 + tid;
      uint32_t kids[8], nk = 0;
      if (i < hi) {
        const uint32_t c = __ldcg(a.mfd_ord + i);
        uint32_t m = mfd_donors(a, c);
        while (m) {
          const uint32_t k = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t n = (uint32_t)((int)c + dir_ox(k) + dir_oy(k) * W);
          if (atomicSub(a.mfd_rem + n, 1u) == 1u) kids[nk++] = n;
        }
      }
      uint32_t inc = nk;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
      }
      const uint32_t wt = __shfl_sync(0xffffffffu, inc, 31);
      uint32_t p0 = 0;
      if (lane == 31 && wt) p0 = atomicAdd(cnt, wt);
      p0 = hi + __shfl_sync(0xffffffffu, p0, 31) + inc - nk;
      for (uint32_t j = 0; j < nk; ++j) {
        a.mfd_ord[p0 + j] = kids[j];
        a.mfd_lev[kids[j]] = nl;
      }
    }
    grid_barrier(ctl);
    lo = hi;
    hi += ld_volatile_u32(cnt);
    if (hi > lo) {
      if (b == 0 && tid == 0) a.mfd_lv[nl + 1] = hi;
      ++nl;
    }
  }
  if (b == 0 && tid == 0) {
    ctl->mfd_nlev = nl;
    if (hi != N) {  // a cycle (mfd.cpp:98-101): cannot happen with strict descent; reported like the reference
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_cell = hi;
      ctl->err_slot = ctl->slot;
    }
  }
  // ---- accumulation, last level first: A = w + sum over donors (slot order) of alpha * A[donor]
  for (uint32_t l = nl; l-- > 0;) {
    const uint32_t s0 = __ldcg(a.mfd_lv + l), e0 = __ldcg(a.mfd_lv + l + 1);
    for (uint32_t i = s0 + b * kTPB + tid; i < e0; i += gstride) {
      const uint32_t c = __ldcg(a.mfd_ord + i);
      uint32_t m = mfd_donors(a, c);
      double acc = a.w0;
      if (m) {
        const double hc = __ldg(a.h + c);
        while (m) {
          const uint32_t k = __ffs(m) - 1;
          m &= m - 1;
          const uint32_t n = (uint32_t)((int)c + dir_ox(k) + dir_oy(k) * W);
          // n's weight for c: its slope towards c (direction 7-k, same length as k)
          const double w = mfd_weight(a, mfd_slope(a, __ldg(a.h + n), hc, (int)(7 - k)));
          const double alpha = __ddiv_rn(w, __ldcg(a.mfd_wsum + n));
          acc = __dadd_rn(acc, __dmul_rn(alpha, __ldcg(a.mfd_A + n)));
        }
      }
      a.mfd_A[c] = acc;
    }
    grid_barrier(ctl);
  }
}

}  // namespace lemgpu
