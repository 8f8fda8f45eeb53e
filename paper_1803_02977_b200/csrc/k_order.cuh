// k_order.cuh -- the breadth-first level order (phase 3), the paper's key
// restructuring.
//
//   generate_queue   proj/src/traversal.cpp:19-48
//
// Level 0 is the ascending list of cells with rec == kNoFlow (traversal.cpp:
// 27-29); level l+1 is, for each level-l cell in order, its donors in slot
// (= stencil = bit) order (traversal.cpp:35-44).  Every level is a stream
// compaction over a static partition of its position range into one segment
// per CTA (reduce-then-scan, no serial look-back chain):
//
//   * the per-segment item counts of level l are accumulated into bins by
//     the kernel that WRITES level l (warp-aggregated integer atomics), so each
//     level needs a single kernel: CTA b sums the bins of segments < b for its
//     base, then scans its segment tile by tile (warp shuffles + smem, carry
//     between tiles) and writes the children and fc[pos], the queue position
//     of the first child;
//   * each queue entry carries its cell's donor mask (pdm, written when the
//     entry is created), so counting and expanding a level read it coalesced
//     instead of gathering dmask by cell index.
//
// The level loop is a graph WHILE node; the last CTA of each level clears its
// condition when the next level is empty.
#pragma once

#include "common.cuh"

namespace lemgpu {

constexpr int kKidCap = 8 * kExTile;  // children of one expansion tile, staged in smem (any fan-out)

struct ScanSmem {
  uint32_t scan[kNW + 1];
  uint32_t base;
  uint32_t ord[kExTile];
  uint8_t dm[kExTile];
  uint32_t kids[kKidCap];   // child cells of the tile, in queue order
  uint16_t kpk[kKidCap];    // (tile-local parent index << 3) | direction parent -> child
};

// Sum of v over the first `upto` entries of bins[] (one CTA, all threads);
// also the sum of all `nb` entries.
template <bool COOP = false>
__device__ __forceinline__ void bins_prefix(const uint32_t* bins, uint32_t upto, uint32_t nb,
                                            uint32_t* scratch, uint32_t& pre, uint32_t& total) {
  uint32_t p = 0, t = 0;
  for (uint32_t i = threadIdx.x; i < nb; i += kTPB) {
    const uint32_t v = COOP ? __ldcg(bins + i) : bins[i];
    t += v;
    if (i < upto) p += v;
  }
  p = __reduce_add_sync(0xffffffffu, p);
  t = __reduce_add_sync(0xffffffffu, t);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __shared__ uint32_t sp[kNW], st[kNW];
  if (lane == 0) {
    sp[warp] = p;
    st[warp] = t;
  }
  __syncthreads();
  p = 0;
  t = 0;
#pragma unroll
  for (int w = 0; w < kNW; ++w) {
    p += sp[w];
    t += st[w];
  }
  pre = p;
  total = t;
  __syncthreads();
  (void)scratch;
}

// Add v to bins[bin] with one atomic per distinct bin of the warp.
__device__ __forceinline__ void bin_add(uint32_t* bins, uint32_t bin, uint32_t v, bool active) {
  const uint32_t key = active ? bin : 0xFFFFFFFFu;
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const uint32_t sum = __reduce_add_sync(peers, v);
  if (active && (threadIdx.x & 31) == (uint32_t)(__ffs(peers) - 1) && sum) atomicAdd(bins + bin, sum);
}

// Second pass over the queue positions [p0, p1) just written by this CTA:
// each entry's donor mask (coalesced pdm store, gathered dmask with several
// loads in flight per thread) and the per-segment child counts of the next
// sweep (segments of Sn positions starting at `base`).
template <bool KIDS>
__device__ __forceinline__ void pdm_and_bins(const StepArgs& a, const uint32_t* kids, const uint16_t* kpk,
                                             uint32_t tb, uint32_t p0, uint32_t p1, uint32_t base, uint32_t Sn,
                                             uint32_t* bins) {
  uint32_t cur_bin = 0xFFFFFFFFu, cur_end = 0, sum = 0;
  for (uint32_t pb = p0 + threadIdx.x; pb < p1; pb += 4 * kTPB) {
    uint32_t cm[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t p = pb + u * kTPB;
      if (p < p1) {
        uint32_t child;
        if (KIDS) {
          child = kids[p - p0];
          const uint32_t pk = kpk[p - p0];
          a.order[p] = child;
          a.ppos[p] = tb + (pk >> 3);
          a.cdir[p] = (uint8_t)(pk & 7u);
        } else {
          child = a.order[p];
        }
        cm[u] = KIDS ? donor_mask_interior(a, child) : donor_mask_at(a, child);
      } else {
        cm[u] = 0u;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t p = pb + u * kTPB;
      if (p < p1) {
        a.pdm[p] = (uint8_t)cm[u];
        if (p >= cur_end) {
          if (sum) atomicAdd(bins + cur_bin, sum);
          cur_bin = (p - base) / Sn;
          cur_end = base + (cur_bin + 1) * Sn;
          sum = 0;
        }
        sum += __popc(cm[u]);
      }
    }
  }
  bin_add(bins, cur_bin, sum, cur_bin != 0xFFFFFFFFu);
}

// segment size of a level of n items over G CTAs
__device__ __forceinline__ uint32_t seg_size(uint32_t n, uint32_t G) { return n ? (n + G - 1) / G : 1u; }

// --------------------------------------------------------------- level 0
// pass 1: NoFlow count per segment of the cell range
__global__ void __launch_bounds__(kTPB) k_l0_count(StepArgs a) {
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->err_flag)) return;  // sticky failure of an earlier step (uniform)
  PhWhole ph(ctl, LEMGPU_PHASE_ORDER);
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t S = ((a.N + G - 1) / G + 15u) & ~15u;
  const uint32_t s0 = b * S, s1 = min(a.N, s0 + S);
  uint32_t cnt = 0;
  for (uint32_t c = s0 + threadIdx.x * 16; c < s1; c += kTPB * 16) {
    if (c + 16 <= s1) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.rcode + c));
      cnt += (__popc(__vcmpeq4(v.x, 0x08080808u)) + __popc(__vcmpeq4(v.y, 0x08080808u)) +
              __popc(__vcmpeq4(v.z, 0x08080808u)) + __popc(__vcmpeq4(v.w, 0x08080808u))) >> 3;
    } else {
      for (uint32_t j = c; j < s1; ++j) cnt += a.rcode[j] == kNoFlowCode;
    }
  }
  cnt = __reduce_add_sync(0xffffffffu, cnt);
  __shared__ uint32_t sw[kNW];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int w = 0; w < kNW; ++w) t += sw[w];
    a.part[b] = t;
  }
  for (uint32_t i = b * kTPB + threadIdx.x; i < G; i += G * kTPB) a.bins[i] = 0;  // bins of level 0
}

// pass 2: write level 0 (ascending cells), its donor masks and the bins of
// its child counts
__global__ void __launch_bounds__(kTPB) k_l0_write(StepArgs a) {
  __shared__ ScanSmem sm;
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->err_flag)) return;
  PhWhole ph(ctl, LEMGPU_PHASE_ORDER);
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t S = ((a.N + G - 1) / G + 15u) & ~15u;
  const uint32_t s0 = b * S, s1 = min(a.N, s0 + S);
  uint32_t pre, n0;
  bins_prefix(a.part, b, G, sm.scan, pre, n0);
  const uint32_t Sb = seg_size(n0, G);  // level-0 segment size for k_expand(0)
  for (uint32_t i = b * kTPB + threadIdx.x; i < G; i += G * kTPB) a.bins[G + i] = 0;  // bins of level 1
  uint32_t carry = pre;
  for (uint32_t t0 = s0; t0 < s1; t0 += kL0Tile) {
    const uint32_t c0 = t0 + threadIdx.x * kL0IPT;
    uint32_t w[4] = {0, 0, 0, 0};
    if (c0 + kL0IPT <= s1) {
      const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.rcode + c0));
      w[0] = v.x;
      w[1] = v.y;
      w[2] = v.z;
      w[3] = v.w;
    } else {
      for (uint32_t j = 0; j < (uint32_t)kL0IPT; ++j)
        if (c0 + j < s1) w[j >> 2] |= (uint32_t)a.rcode[c0 + j] << (8 * (j & 3));
    }
    uint32_t eq[4], cnt = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      eq[q] = __vcmpeq4(w[q], 0x08080808u);
      cnt += __popc(eq[q]) >> 3;
    }
    uint32_t tot;
    const uint32_t first = carry;
    uint32_t out = carry + block_excl_scan(cnt, &tot, sm.scan);
    carry += tot;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t e = eq[q];
      while (e) {
        const int bit = __ffs(e) - 1;
        e &= ~(0xFFu << (bit & ~7));
        a.order[out++] = c0 + q * 4 + (bit >> 3);
      }
    }
    __syncthreads();  // this tile's queue entries are visible to the whole CTA
    pdm_and_bins<false>(a, nullptr, nullptr, 0u, first, first + tot, 0u, Sb, a.bins);
  }
  if (last_block_done(ctl) && threadIdx.x == 0) {
    a.levels[0] = 0;
    a.levels[1] = n0;
    a.fc[a.N] = a.N;
    ctl->n0 = n0;
    ctl->nch = (n0 + kChunkRoots - 1) / kChunkRoots;
    ctl->lvl = 0;
    timeline(ctl);
  }
}

// --------------------------------------------------------- level l -> l+1
// One level of the while loop.  Also derives the per-chunk position ranges
// of this level from fc[] of the previous one: a chunk of consecutive sources
// owns ONE contiguous range per level, P_l(k) = fc[P_{l-1}(k)] (the end of a
// level maps to the end of the next).
// One frontier expansion: level l = positions [lo, hi) -> level l+1 written
// from position hi; returns the size of level l+1 (every CTA computes it).
// COOP: called inside one persistent (cooperative) kernel, so data written by
// other CTAs in earlier levels is read past L1 (__ldcg).
template <bool COOP>
__device__ __forceinline__ uint32_t ld_x(const uint32_t* p) { return COOP ? __ldcg(p) : *p; }
template <bool COOP>
__device__ __forceinline__ uint32_t ld_x(const uint8_t* p) { return COOP ? (uint32_t)__ldcg(p) : (uint32_t)*p; }

template <bool COOP>
__device__ __forceinline__ uint32_t expand_level(const StepArgs& a, ScanSmem& sm, uint32_t l, uint32_t lo,
                                                 uint32_t hi, bool err) {
  Ctl* ctl = a.ctl;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  uint32_t total = 0;
  if (!err) {
    const uint32_t* bins_in = a.bins + (size_t)(l % 3) * G;
    uint32_t* bins_out = a.bins + (size_t)((l + 1) % 3) * G;
    uint32_t* bins_clr = a.bins + (size_t)((l + 2) % 3) * G;
    for (uint32_t i = b * kTPB + threadIdx.x; i < G; i += G * kTPB) bins_clr[i] = 0;
    if (l <= (uint32_t)kChunkMaxLevels) {
      const uint32_t nch = ctl->nch;
      uint32_t* cb = a.cbound + (size_t)l * a.cb_stride;
      const uint32_t* cbp = a.cbound + (size_t)(l ? l - 1 : 0) * a.cb_stride;
      for (uint32_t k = b * kTPB + threadIdx.x; k <= nch; k += G * kTPB) {
        uint32_t v;
        if (l == 0) {
          v = min(k * (uint32_t)kChunkRoots, hi);
        } else {
          const uint32_t p = ld_x<COOP>(cbp + k);
          v = p >= lo ? hi : ld_x<COOP>(a.fc + p);
        }
        cb[k] = v;
      }
    }
    uint32_t pre;
    bins_prefix<COOP>(bins_in, b, G, sm.scan, pre, total);
    const uint32_t S = seg_size(hi - lo, G);
    const uint32_t Sn = seg_size(total, G);  // segment size of the next level
    const uint32_t s0 = lo + min(b * S, hi - lo), s1 = lo + min((b + 1) * S, hi - lo);
    uint32_t carry = hi + pre;
    const uint32_t W = a.W;
    // register double buffer: the next tile's cells and masks are in flight
    // while the current tile is scanned and expanded
    uint32_t nc[kExIPT], nm[kExIPT];
#pragma unroll
    for (int j = 0; j < kExIPT; ++j) {
      const uint32_t p = s0 + j * kTPB + threadIdx.x;
      nc[j] = p < s1 ? ld_x<COOP>(a.order + p) : 0u;
      nm[j] = p < s1 ? ld_x<COOP>(a.pdm + p) : 0u;
    }
    for (uint32_t tb = s0; tb < s1; tb += kExTile) {
      // coalesced staging of the tile's cells and donor masks
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) {
        sm.ord[j * kTPB + threadIdx.x] = nc[j];
        sm.dm[j * kTPB + threadIdx.x] = (uint8_t)nm[j];
      }
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) {
        const uint32_t p = tb + kExTile + j * kTPB + threadIdx.x;
        nc[j] = p < s1 ? ld_x<COOP>(a.order + p) : 0u;
        nm[j] = p < s1 ? ld_x<COOP>(a.pdm + p) : 0u;
      }
      __syncthreads();
      uint32_t c[kExIPT], m[kExIPT], cnt = 0;
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) {
        c[j] = sm.ord[threadIdx.x * kExIPT + j];
        m[j] = sm.dm[threadIdx.x * kExIPT + j];
        cnt += __popc(m[j]);
      }
      uint32_t tot;
      uint32_t out = carry + block_excl_scan(cnt, &tot, sm.scan);
      carry += tot;
      const uint32_t first = carry - tot;
      uint32_t fcv[kExIPT];
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) {
        fcv[j] = out;
        uint32_t mm = m[j];
        while (mm) {
          const uint32_t k = __ffs(mm) - 1;
          mm &= mm - 1;
          const uint32_t child = (uint32_t)((int)c[j] + dir_off(k, (int)W));
          sm.kids[out - first] = child;
          sm.kpk[out - first] = (uint16_t)(((threadIdx.x * kExIPT + j) << 3) | k);
          ++out;
        }
      }
      __syncthreads();  // sm.ord reused to transpose fc for coalesced stores
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) sm.ord[threadIdx.x * kExIPT + j] = fcv[j];
      __syncthreads();
#pragma unroll
      for (int j = 0; j < kExIPT; ++j) {
        const uint32_t p = tb + j * kTPB + threadIdx.x;
        if (p < s1) a.fc[p] = sm.ord[j * kTPB + threadIdx.x];
      }
      pdm_and_bins<true>(a, sm.kids, sm.kpk, tb, first, first + tot, hi, Sn, bins_out);
      __syncthreads();
    }
  }
  return total;
}

// Bookkeeping after level l is expanded (one thread): the next level's bound,
// or the plan's completion (nlevels, cycle check, schedule of the physics).
__device__ __forceinline__ void expand_finish(const StepArgs& a, uint32_t l, uint32_t hi, uint32_t total, bool err,
                                              bool coop = false) {
  Ctl* ctl = a.ctl;

  if (total > 0) {
    a.levels[l + 2] = hi + total;
    ctl->lvl = l + 1;
    if (!coop) set_cond(a, 0, 1);
  } else {
    // plan complete: nlevels = l + 1 (traversal.cpp:45); cycle check (:46)
    ctl->nlev = l + 1;
    uint32_t mode = (l + 1 <= (uint32_t)kChunkMaxLevels && !a.force_deep) ? kModeShallow : kModeDeep;
    a.fc[hi] = hi;  // end sentinel of the last level's child ranges
    if (!err && a.expect_cells && hi != a.expect_cells) {
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_cell = hi;  // cells placed
      ctl->err_slot = ctl->slot;
      mode = kModeFailed;
    }
    if (err) mode = kModeFailed;
    ctl->mode = mode;
    if (mode == kModeDeep) {
      ctl->dlvl = l;  // deepest level first
      if (!coop) set_cond(a, 1, 1);  // the tile path sweeps deep plans in k_deep_coop
    }
    ctl->t_order_end = globaltimer();
    if (!coop) set_cond(a, 0, 0);
  }
  timeline(ctl);
}

__global__ void __launch_bounds__(kTPB) k_expand(StepArgs a) {
  __shared__ ScanSmem sm;
  Ctl* ctl = a.ctl;
  PhWhole ph(ctl, LEMGPU_PHASE_ORDER);
  const uint32_t l = ld_volatile_u32(&ctl->lvl);
  const bool err = ld_volatile_u32(&ctl->err_flag) != 0;
  const uint32_t lo = a.levels[l], hi = a.levels[l + 1];
  const uint32_t total = expand_level<false>(a, sm, l, lo, hi, err);
  if (last_block_done(ctl) && threadIdx.x == 0) expand_finish(a, l, hi, total, err);
}

// Narrow levels of the escape expansion (filled DEMs: thousands of levels of
// a few hundred cells): CTA 0 expands a run of them alone, the frontier in
// shared memory, block barriers between levels, while the other CTAs wait at
// one grid barrier for the whole run.  Per level: counts, a block scan, the
// children (order / ppos / cdir / fc as the grid expansion writes them), their
// donor masks.  Only past level kChunkMaxLevels (the plan is then deep, so the
// chunk bounds of the shallow physics are not needed).  Leaves the narrow run
// when a level is wider than kNX (then its per-segment child counts are
// rebuilt for the grid) or the plan is complete; the hand-back point goes to
// ctl->nr_*.
constexpr uint32_t kNX = 2048;
struct NarrowSmem {
  uint32_t cell[2][kNX];  // frontier / next frontier cells
  uint8_t mask[2][kNX];   // their donor masks
  uint16_t par[kNX];      // next frontier: parent index in the frontier
  uint16_t fco[kNX];      // frontier: offset of its first child in the next frontier
  uint8_t dir[kNX];       // next frontier: direction parent -> child
  uint32_t scan[kNW + 1];
};

__device__ __forceinline__ void expand_narrow_run(const StepArgs& a, NarrowSmem& ns, uint32_t l, uint32_t lo, uint32_t hi) {
  Ctl* ctl = a.ctl;
  const uint32_t tid = threadIdx.x, G = gridDim.x, W = a.W;
  for (uint32_t i = tid; i < hi - lo; i += kTPB) {
    ns.cell[0][i] = __ldcg(a.order + lo + i);
    ns.mask[0][i] = (uint8_t)__ldcg(a.pdm + lo + i);
  }
  __syncthreads();
  uint32_t cur = 0;
  bool done = false;
  for (;;) {
    const uint32_t n = hi - lo;
    // this thread's parents: a contiguous chunk, so children stay in queue order
    const uint32_t per = (n + kTPB - 1) / kTPB, i0 = min(tid * per, n), i1 = min(i0 + per, n);
    uint32_t cnt = 0;
    for (uint32_t i = i0; i < i1; ++i) cnt += __popc(ns.mask[cur][i]);
    uint32_t total;
    uint32_t out = block_excl_scan(cnt, &total, ns.scan);
    if (total > kNX) {
      // the next frontier does not fit: written straight to the queue, and
      // the run ends after this level
      for (uint32_t i = i0; i < i1; ++i) {
        a.fc[lo + i] = hi + out;
        uint32_t m = ns.mask[cur][i];
        const uint32_t c = ns.cell[cur][i];
        while (m) {
          const uint32_t k = __ffs(m) - 1;
          m &= m - 1;
          a.order[hi + out] = (uint32_t)((int)c + dir_off(k, (int)W));
          a.ppos[hi + out] = lo + i;
          a.cdir[hi + out] = (uint8_t)k;
          ++out;
        }
      }
      __syncthreads();
      for (uint32_t q = tid; q < total; q += kTPB) a.pdm[hi + q] = (uint8_t)donor_mask_interior(a, __ldcg(a.order + hi + q));
    } else {
      // children into shared memory only; the queue entries go out coalesced
      // below, overlapping the donor-mask loads
      for (uint32_t i = i0; i < i1; ++i) {
        ns.fco[i] = (uint16_t)out;
        uint32_t m = ns.mask[cur][i];
        const uint32_t c = ns.cell[cur][i];
        while (m) {
          const uint32_t k = __ffs(m) - 1;
          m &= m - 1;
          ns.cell[cur ^ 1u][out] = (uint32_t)((int)c + dir_off(k, (int)W));
          ns.par[out] = (uint16_t)i;
          ns.dir[out] = (uint8_t)k;
          ++out;
        }
      }
      __syncthreads();
      for (uint32_t i = tid; i < n; i += kTPB) a.fc[lo + i] = hi + ns.fco[i];
      // donor masks of the children: 4 per thread in flight at once
      for (uint32_t q0 = tid; q0 < total; q0 += 4 * kTPB) {
        uint32_t ch[4], mk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ch[u] = q0 + u * kTPB < total ? ns.cell[cur ^ 1u][q0 + u * kTPB] : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) mk[u] = q0 + u * kTPB < total ? donor_mask_interior(a, ch[u]) : 0u;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = q0 + u * kTPB;
          if (q < total) {
            a.order[hi + q] = ch[u];
            a.ppos[hi + q] = lo + ns.par[q];
            a.cdir[hi + q] = ns.dir[q];
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t q = q0 + u * kTPB;
          if (q < total) {
            a.pdm[hi + q] = (uint8_t)mk[u];
            ns.mask[cur ^ 1u][q] = (uint8_t)mk[u];
          }
        }
      }
    }
    __syncthreads();
    if (tid == 0) expand_finish(a, l, hi, total, false, true);
    if (total == 0) {
      done = true;
      break;
    }
    lo = hi;
    hi += total;
    ++l;
    cur ^= 1u;
    if (total > kNX) {
      // back to the grid: per-segment child counts of level l for G CTAs,
      // and the next level's count slot cleared
      uint32_t* bins_in = a.bins + (size_t)(l % 3) * G;
      uint32_t* bins_nx = a.bins + (size_t)((l + 1) % 3) * G;
      for (uint32_t i = tid; i < G; i += kTPB) {
        bins_in[i] = 0;
        bins_nx[i] = 0;
      }
      __syncthreads();
      const uint32_t S = seg_size(total, G);
      for (uint32_t p = lo + tid; p < hi; p += kTPB) {
        const uint32_t v = __popc(__ldcg(a.pdm + p));
        if (v) atomicAdd(bins_in + (p - lo) / S, v);
      }
      break;
    }
  }
  __syncthreads();
  if (tid == 0) {
    ctl->nr_l = l;
    ctl->nr_lo = lo;
    ctl->nr_hi = hi;
    ctl->nr_done = done ? 1u : 0u;
  }
}

// The whole level expansion of the escaped trees in ONE cooperative kernel
// (the tile path's small residual workload): level 0 = the roots listed by
// k_tiles (their donor masks and the bins of the first expansion), then one
// expand_level per level separated by
// grid barriers instead of one graph WHILE iteration (kernel launch) each.
__global__ void __launch_bounds__(kTPB) k_esc_bfs(StepArgs a) {
  __shared__ union {
    ScanSmem sm;
    NarrowSmem ns;
  } u;
  ScanSmem& sm = u.sm;
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->esc_small) || ld_volatile_u32(&ctl->mode) == kModeDone)
    return;  // k_esc_small or k_esc_forest finished the escaped trees (uniform)
  PhWhole ph(ctl, LEMGPU_PHASE_ORDER);
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const bool err = ld_volatile_u32(&ctl->err_flag) != 0;
  const uint32_t n = ld_volatile_u32(&ctl->nesc);
  const uint32_t Sb = seg_size(n, G);
  if (!err) {
    const uint32_t s0 = min(b * Sb, n), s1 = min(s0 + Sb, n);
    pdm_and_bins<false>(a, nullptr, nullptr, 0u, s0, s1, 0u, Sb, a.bins);
  }
  if (b == 0 && threadIdx.x == 0) {
    a.levels[0] = 0;
    a.levels[1] = n;
    ctl->n0 = n;
    ctl->nch = (n + kChunkRoots - 1) / kChunkRoots;
    ctl->lvl = 0;
    ctl->t_t_end = max(ctl->t_t_end, globaltimer());
  }
  grid_barrier(ctl);
  // every CTA derives the next level's bounds itself (the size of level l+1
  // is the sum of the bins every CTA reads), so one barrier per level suffices
  uint32_t lo = 0, hi = n;
  for (uint32_t l = 0;;) {
    if (!err && !a.no_narrow && l >= (uint32_t)kChunkMaxLevels && hi - lo <= kNX) {
      if (b == 0) expand_narrow_run(a, u.ns, l, lo, hi);
      grid_barrier(ctl);
      if (ld_volatile_u32(&ctl->nr_done)) break;
      l = ld_volatile_u32(&ctl->nr_l);
      lo = ld_volatile_u32(&ctl->nr_lo);
      hi = ld_volatile_u32(&ctl->nr_hi);
      continue;
    }
    const uint32_t total = expand_level<true>(a, sm, l, lo, hi, err);
    grid_barrier(ctl);
    if (b == 0 && threadIdx.x == 0) expand_finish(a, l, hi, total, err, true);
    if (total == 0) break;
    lo = hi;
    hi += total;
    ++l;
  }
}

}  // namespace lemgpu
