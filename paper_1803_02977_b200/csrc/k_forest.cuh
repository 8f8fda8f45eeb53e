// k_forest.cuh -- the escaped trees when they are most of the raster (the
// deep-level regime of filled DEMs: thousands of levels).
//
//   generate_queue     proj/src/traversal.cpp:19-48   (levels = depth below the root)
//   accumulate_into    proj/src/accumulation.cpp:7-17, accumulation.hpp:21-28
//   uplift             proj/src/erosion.cpp:52-57
//   erode / newton_erode_cell  proj/src/erosion.cpp:19-81
//
// The level-synchronous escape path (k_esc_bfs + k_deep_coop) pays one grid
// or block barrier plus dependent global round trips per level for each of
// three sweeps (expansion, accumulation, erosion): ~3 us per level and sweep,
// 10 ms / 92 ms per step on the epsilon-filled 1000^2 / 4000^2 DEMs.  Here:
//
//   1. levels without a sweep: the level of a cell is its depth below its
//      root, found for every cell at once by pointer jumping on the receiver
//      forest (J[c] = {distance, target}, target <- target's target, about
//      log2(depth) + 1 grid-wide rounds);
//   2. the forest is split between the CTAs by TREE (owner = hash of the
//      root): trees are independent, so from here on a CTA never waits for
//      another.  One counting sort by (owner, depth) lays every CTA's cells
//      out level-major in its own position range;
//   3. each CTA sweeps its levels alone with block barriers only: drainage
//      counts pushed to the receiver's slot (integer adds commute: exact
//      whatever the order -- EX, every partial sum an exact multiple of the
//      cell area), F = K*dt*pow(A,m)/pow(dist,n) and the Newton reciprocal
//      for all its cells in one throughput pass (off the dependent chain),
//      then uplift + Newton level by level, the previous level's counts / new
//      elevations in shared-memory rings.
//
// Within a level the cells may sit in any order (each cell's arithmetic reads
// only its receiver's final h and its own count), so h and the diagnostics
// are the reference's bit for bit.  The reference's own order (TraversalPlan)
// is still produced by the parity export (lemgpu_download_graph).
#pragma once

#include "common.cuh"
#include "k_physics.cuh"
#include "k_recv_donor.cuh"

namespace lemgpu {

constexpr int kFTPB = 1024;              // one CTA per SM
constexpr uint32_t kFNW = kFTPB / 32;    // warps per CTA
constexpr uint32_t kFRing = 4096;        // cells of one level of a CTA held in a shared-memory ring slot
constexpr uint32_t kFLv = 8192;          // level starts of a CTA kept in shared memory (deeper: global)
constexpr uint32_t kFTop = 0x80000000u;  // escaped-root mark in the distance word of J
constexpr int kFMaxRounds = 40;          // 2^40 > any depth: a receiver cycle stops here (StructureError)

constexpr uint32_t kFChunk = 1024;  // positions per bulk-copied chunk (chunks start at multiples of it)
constexpr uint32_t kFSlotsA = 16;   // chunks of receiver positions in flight (counts sweep)
constexpr uint32_t kFSlotsE = 4;    // chunks of {receiver position, F, reciprocal, h0} in flight (erosion)

struct ForestSmem {
  union {
    struct {
      uint32_t cnt[3][kFRing];           // counts of levels d, d-1 (receiving) and d-2 (being reset)
      uint32_t pp[kFSlotsA][kFChunk];    // staged receiver positions
    } a;
    struct {
      double h[2][kFRing];               // new elevations of levels d-1 and d
      double f[kFSlotsE][kFChunk];       // staged F
      double y[kFSlotsE][kFChunk];       // staged RN(1 / RN(1 + F))
      double h0[kFSlotsE][kFChunk];      // staged uplifted elevations
      uint32_t pp[kFSlotsE][kFChunk];    // staged receiver positions
    } e;
  } u;
  uint32_t lv[kFLv + 1];  // this CTA's level starts (absolute positions), lv[D] = end
  uint32_t red[32];
  uint64_t bar[kFSlotsA + kFSlotsE];
};
constexpr size_t kForestSmemBytes = sizeof(ForestSmem);

// Barrier of the first n threads of the CTA (named barrier 1; n a multiple of 32).
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// One bulk asynchronous copy global -> shared (16-byte aligned, multiple of 16
// bytes), completing on the mbarrier's transaction count.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ uint32_t forest_owner(uint32_t root, uint32_t G) {
  return (uint32_t)(((unsigned long long)(root * 2654435761u) * G) >> 32);
}

// Block-wide sum of one u32 per thread (kFTPB threads), result in every thread.
__device__ __forceinline__ uint32_t forest_block_sum(uint32_t v, uint32_t* red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t t = threadIdx.x < kFNW ? red[threadIdx.x] : 0u;
  if (threadIdx.x < 32)
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  __syncthreads();
  if (threadIdx.x == 0) red[0] = t;
  __syncthreads();
  const uint32_t r = red[0];
  __syncthreads();
  return r;
}

template <int NK>
__global__ void __launch_bounds__(kFTPB, 1) k_esc_forest(StepArgs a) {
  extern __shared__ __align__(16) unsigned char fsm_raw[];
  ForestSmem& s = *reinterpret_cast<ForestSmem*>(fsm_raw);
  Ctl* ctl = a.ctl;
  // uniform exits: an earlier failure, k_esc_small finished the escaped trees,
  // nothing escaped, or the escape set is small (the level path is cheaper
  // than a pass over every cell)
  if (!a.esc_forest || ld_volatile_u32(&ctl->err_flag) || ld_volatile_u32(&ctl->esc_small)) return;
  const uint32_t nesc = ld_volatile_u32(&ctl->nesc);
  if (nesc == 0) return;
  const uint32_t N = a.N;
  if (a.esc_forest == 1 && (unsigned long long)(N - ld_volatile_u32(&ctl->tile_cells)) * 4ull < N) return;
  __shared__ PhClk s_pc;
  phclk_begin(s_pc);
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const uint32_t gstride = G * kFTPB, wbase = b * kFTPB + (tid & ~31u);  // warp-uniform loop bases
  const int W = (int)a.W;
  unsigned long long* J = reinterpret_cast<unsigned long long*>(a.Aq);  // cell-major {distance | target}
  uint32_t* key = a.fc;    // cell-major: owner * D + depth of an escaped cell, else ~0 (phases 3-5)
  uint32_t* cur = a.fbins;  // [owner][depth]: cell counts, then scatter cursors
  uint32_t* fst = a.cbound;  // [owner][depth]: first position (absolute)

  // ---- 1. J: distance 1 to the receiver; roots point at themselves
  for (uint32_t c = b * kFTPB + tid; c < N; c += gstride) {
    const uint32_t code = a.rcode[c];
    J[c] = code >= 8u ? (unsigned long long)c : ((1ull << 32) | (uint32_t)((int)c + dir_off(code, W)));
  }
  if (b == 0 && tid < 3) {
    ctl->fr_flag[tid] = 0;
    ctl->fr_t[tid] = 0;
  }
  if (b == 0 && tid == 0) {
    ctl->fr_maxd = 0;
    ctl->fr_maxcells = 0;
    timeline(ctl);
  }
  grid_barrier(ctl);
  // the escaped roots (k_tiles' list) get the mark
  for (uint32_t i = b * kFTPB + tid; i < nesc; i += gstride) {
    const uint32_t r = __ldcg(a.order + i);
    J[r] = ((unsigned long long)kFTop << 32) | r;
  }
  grid_barrier(ctl);
  // ---- pointer jumping (in place: a 64-bit word is always a consistent pair)
  for (int rd = 0;; ++rd) {
    if (b == 0 && tid == 0) ctl->fr_flag[(rd + 1) % 3] = 0;  // read by every CTA two barriers ago
    bool ch = false;
    for (uint32_t c = b * kFTPB + tid; c < N; c += gstride) {
      const unsigned long long j = __ldcg(J + c);
      const uint32_t n1 = (uint32_t)j;
      if (n1 == c) continue;  // a root
      const unsigned long long j2 = __ldcg(J + n1);
      const uint32_t n2 = (uint32_t)j2;
      if (n2 == n1) continue;  // n1 is a root: final
      __stcg(J + c, (((j >> 32) + (j2 >> 32)) << 32) | n2);
      ch = true;
    }
    if (__syncthreads_or(ch) && tid == 0) atomicOr(&ctl->fr_flag[rd % 3], 1u);
    grid_barrier(ctl);
    if (!ld_volatile_u32(&ctl->fr_flag[rd % 3]) || rd + 1 == kFMaxRounds) {
      if (b == 0 && tid == 0) {
        ctl->fr_rounds = rd + 1;
        timeline(ctl);
      }
      break;
    }
  }
  // ---- 2. escaped cells (root marked and reached: a cycle never reaches a
  // root -> missing cells -> StructureError in k_finalize), deepest level
  uint32_t md = 0;
  for (uint32_t c = b * kFTPB + tid; c < N; c += gstride) {
    const unsigned long long j = __ldcg(J + c);
    const uint32_t n = (uint32_t)j;
    bool esc;
    uint32_t d;
    if (n == c) {
      esc = (j >> 32) & kFTop;
      d = 0;
    } else {
      const unsigned long long jr = __ldcg(J + n);
      esc = (uint32_t)jr == n && ((jr >> 32) & kFTop);
      d = (uint32_t)(j >> 32);
    }
    if (esc) md = max(md, d);
  }
  for (int o = 16; o; o >>= 1) md = max(md, __shfl_xor_sync(0xffffffffu, md, o));
  if (lane == 0 && md) atomicMax(&ctl->fr_maxd, md);
  grid_barrier(ctl);
  const uint32_t D = ld_volatile_u32(&ctl->fr_maxd) + 1;  // levels of the escaped plan
  // bins of (owner, depth): fit the scratch, else leave the step to the level path (uniform)
  if ((unsigned long long)G * D + 1 > (unsigned long long)N + 1 || (unsigned long long)G * D + 1 > a.cb_cap) {
    if (b == 0 && tid == 0) ctl->fr_flag[0] = ctl->fr_flag[1] = ctl->fr_flag[2] = 0;
    return;
  }
  for (uint32_t i = b * kFTPB + tid; i < G * D; i += gstride) cur[i] = 0;
  grid_barrier(ctl);
  // ---- 3. counts per (owner, depth), warp-aggregated
  for (uint32_t c0 = wbase; c0 < N; c0 += gstride) {
    const uint32_t c = c0 + lane;
    uint32_t k = ~0u;
    if (c < N) {
      const unsigned long long j = __ldcg(J + c);
      const uint32_t n = (uint32_t)j;
      if (n == c) {
        if ((j >> 32) & kFTop) k = forest_owner(c, G) * D;
      } else {
        const unsigned long long jr = __ldcg(J + n);
        if ((uint32_t)jr == n && ((jr >> 32) & kFTop)) k = forest_owner(n, G) * D + (uint32_t)(j >> 32);
      }
      key[c] = k;
    }
    const uint32_t am = __ballot_sync(0xffffffffu, k != ~0u);
    if (k != ~0u) {
      const uint32_t peers = __match_any_sync(am, k);
      if (lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(cur + k, (uint32_t)__popc(peers));
    }
  }
  grid_barrier(ctl);
  if (b == 0 && tid == 0) timeline(ctl);
  // ---- 4. positions: CTA b owns one contiguous range, level-major
  {
    uint32_t t = 0;
    for (uint32_t d = tid; d < D; d += kFTPB) t += __ldcg(cur + b * D + d);
    t = forest_block_sum(t, s.red);
    if (tid == 0) a.bins[b] = t;
  }
  grid_barrier(ctl);
  uint32_t base = 0, total_all = 0;
  {
    uint32_t t = 0, u = 0;
    for (uint32_t j = tid; j < G; j += kFTPB) {
      const uint32_t v = __ldcg(a.bins + j);
      t += j < b ? v : 0u;
      u += v;
    }
    base = forest_block_sum(t, s.red);
    total_all = forest_block_sum(u, s.red);
  }
  // exclusive scan of this CTA's D counts (tiles of kFTPB, carry between tiles)
  {
    uint32_t carry = base;
    for (uint32_t d0 = 0; d0 < D; d0 += kFTPB) {
      const uint32_t d = d0 + tid;
      const uint32_t v = d < D ? __ldcg(cur + b * D + d) : 0u;
      uint32_t x = v;
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) s.red[tid >> 5] = x;
      __syncthreads();
      if (tid < 32) {
        uint32_t w = tid < kFNW ? s.red[tid] : 0u;
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= (uint32_t)o) w += y;
        }
        if (tid < kFNW) s.red[tid] = w;
      }
      __syncthreads();
      const uint32_t ex = carry + (tid >= 32 ? s.red[(tid >> 5) - 1] : 0u) + x - v;
      if (d < D) {
        fst[b * D + d] = ex;
        cur[b * D + d] = ex;
        if (d < kFLv) s.lv[d] = ex;
      }
      carry += s.red[kFNW - 1];
      __syncthreads();
    }
    if (tid == 0) {
      fst[b * D + D] = carry;  // (the next CTA's first start, or the total for the last CTA)
      if (D <= kFLv) s.lv[D] = carry;
    }
  }
  if (b == G - 1 && tid == 0) {
    a.levels[0] = 0;
    a.levels[D] = total_all;  // escaped cells (k_finalize's cycle check, k_esc_gather)
  }
  grid_barrier(ctl);
  // ---- 5. scatter: order[pos] = cell, J[c].target = pos (the receiver's position is looked up below)
  for (uint32_t c0 = wbase; c0 < N; c0 += gstride) {
    const uint32_t c = c0 + lane;
    const uint32_t k = c < N ? __ldcg(key + c) : ~0u;
    const uint32_t am = __ballot_sync(0xffffffffu, k != ~0u);
    if (k != ~0u) {
      const uint32_t peers = __match_any_sync(am, k);
      const uint32_t ld = (uint32_t)(__ffs(peers) - 1);
      uint32_t p0 = 0;
      if (lane == ld) p0 = atomicAdd(cur + k, (uint32_t)__popc(peers));
      p0 = __shfl_sync(peers, p0, ld);
      const uint32_t pos = p0 + __popc(peers & ((1u << lane) - 1u));
      a.order[pos] = c;
      const unsigned long long j = __ldcg(J + c);
      __stcg(J + c, (j & 0xFFFFFFFF00000000ull) | pos);
    }
  }
  grid_barrier(ctl);
  if (b == 0 && tid == 0) {
    ctl->t_order_end = globaltimer();
    timeline(ctl);
  }
  // ---- this CTA's positions [P0, P1); level d = [lv(d), lv(d+1))
  auto lvl = [&](uint32_t d) -> uint32_t { return d < kFLv ? s.lv[d] : __ldcg(fst + b * D + d); };
  const uint32_t P0 = lvl(0), P1 = D < kFLv ? s.lv[D] : __ldcg(fst + b * D + D);
  // receiver position and direction; counts start at 1 (the cell itself)
  uint32_t* cnt = a.fc;  // position-major counts (the keys are dead)
  for (uint32_t i = b * kFTPB + tid; i < total_all; i += gstride) {
    const uint32_t c = __ldcg(a.order + i);
    const uint32_t code = a.rcode[c];
    uint32_t pp = ~0u;
    if (code < 8u) pp = (uint32_t)__ldcg(J + (uint32_t)((int)c + dir_off(code, W)));
    a.ppos[i] = pp;
    a.cdir[i] = (uint8_t)code;
    cnt[i] = 1u;
  }
  grid_barrier(ctl);  // J (a.Aq) is read above by every CTA; from here on a.Aq holds reciprocals
  phclk_mark(s_pc, LEMGPU_PHASE_ORDER);
  // levels of this CTA's trees: 1 + its deepest non-empty level
  uint32_t Dl = 0;
  for (uint32_t d = tid; d < D; d += kFTPB)
    if (lvl(d) < P1) Dl = d + 1;
  for (int o = 16; o; o >>= 1) Dl = max(Dl, __shfl_xor_sync(0xffffffffu, Dl, o));
  if (lane == 0) s.red[tid >> 5] = Dl;
  __syncthreads();
  Dl = 0;
  for (uint32_t j = 0; j < kFNW; ++j) Dl = max(Dl, s.red[j]);
  __syncthreads();
  // the warps that sweep the counts: about half a cell per thread of an
  // average level (measured: one warp per 16 cells of an average level beats
  // one per 64 -- dem1000fill's counts 0.69 -> 0.56 ms -- and one per 8 or 32);
  // the others skip the sweep
  const uint32_t avgw = (P1 - P0) / max(Dl, 1u);
  uint32_t nact = 32u * min(kFNW, max(2u, (avgw + 15u) / 16u));
  bool act = tid < nact;
  // ---- 6. drainage counts, deepest level first: each cell adds its final
  // count to its receiver's slot (shared-memory ring; global for wide levels).
  // The receiver positions of the coming levels stream into shared memory
  // ahead of the sweep (bulk async copies).  One helper thread (the CTA's
  // last, idle on levels narrower than the CTA) issues the copies and waits
  // for the next level's chunks, and the ring slot of level d-2 is reset by
  // the top threads, so a level costs the busy warps one shared-memory round
  // trip and a block barrier.
  uint32_t HT = nact - 1;
  const uint32_t rtid = nact - 1 - tid;
  auto ring_reset = [&](uint32_t d, uint32_t s0, uint32_t e0) {  // level d = [s0, e0) -> counts 1
    if (e0 - s0 > kFRing) return;
    uint32_t* rb = s.u.a.cnt[d % 3];
    for (uint32_t i = rtid; i < e0 - s0; i += nact) rb[i] = 1u;
  };
  if (tid < kFSlotsA) mbar_init(&s.bar[tid], 1);
  // chunk k of the descending sweep = positions [(qa - k) * kFChunk, +kFChunk)
  const uint32_t qa = P1 > P0 ? (P1 - 1) / kFChunk : 0u;
  const uint32_t ka_last = Dl > 1 ? qa - lvl(1) / kFChunk : 0u;
  uint32_t ka_next = 0;
  uint32_t ka_done = 0;  // helper: chunks [0, ka_done) have landed (waited once each: mbarrier waits are not free)
  auto issue_a = [&](uint32_t limit) {  // helper thread: chunks up to index `limit` of the sweep
    for (; ka_next <= limit && ka_next <= ka_last; ++ka_next) {
      const uint32_t sl = ka_next % kFSlotsA;
      if (ka_next >= kFSlotsA && ka_next - kFSlotsA >= ka_done) mbar_wait(&s.bar[sl], ((ka_next - kFSlotsA) / kFSlotsA) & 1u);
      mbar_expect_tx(&s.bar[sl], kFChunk * 4);
      bulk_g2s(s.u.a.pp[sl], a.ppos + (size_t)(qa - ka_next) * kFChunk, kFChunk * 4, &s.bar[sl]);
    }
  };
  auto wait_a = [&](uint32_t kl, uint32_t kh) {
    for (uint32_t k = ka_done; k <= kh; ++k) mbar_wait(&s.bar[k % kFSlotsA], (k / kFSlotsA) & 1u);
    ka_done = max(ka_done, kh + 1);
  };
  const long long ck0 = clock64();
  {
  // carried level bounds: level d = [s0, e0), level d-1 starts at ps
  uint32_t e0 = P1, s0 = Dl > 0 ? lvl(Dl - 1) : P1;
  bool staged = false;
  __syncthreads();  // barriers initialised
  if (Dl > 1) {
    ring_reset(Dl - 1, s0, e0);
    const uint32_t ps = lvl(Dl - 2);
    ring_reset(Dl - 2, ps, s0);
    staged = qa - s0 / kFChunk <= kFSlotsA - 1;
    if (tid == HT) {
      issue_a(kFSlotsA - 1);
      if (staged) wait_a(0, qa - s0 / kFChunk);
    }
  }
  __syncthreads();
  if (act) {
    uint32_t* rc = s.u.a.cnt[(Dl - 1) % 3];  // ring slots of levels d, d-1, d-2 (rotating)
    uint32_t* rp = s.u.a.cnt[(Dl + 1) % 3];
    uint32_t* rq = s.u.a.cnt[Dl % 3];
    for (uint32_t d = Dl; d-- > 1;) {
      const uint32_t ps = lvl(d - 1);
      const uint32_t pps = d >= 2 ? lvl(d - 2) : 0u;
      const bool wide = e0 - s0 > kFRing, pwide = s0 - ps > kFRing;
      // two cells per iteration: both loads in flight before the atomics
      for (uint32_t i = s0 + tid; i < e0; i += 2 * nact) {
        const uint32_t i2 = i + nact;
        const bool two = i2 < e0;
        uint32_t p, p2 = 0, v, v2 = 0;
        if (staged) {
          p = s.u.a.pp[(qa - i / kFChunk) % kFSlotsA][i % kFChunk];
          if (two) p2 = s.u.a.pp[(qa - i2 / kFChunk) % kFSlotsA][i2 % kFChunk];
        } else {
          p = __ldcg(a.ppos + i);
          if (two) p2 = __ldcg(a.ppos + i2);
        }
        if (wide) {
          v = __ldcg(cnt + i);
          if (two) v2 = __ldcg(cnt + i2);
        } else {
          v = rc[i - s0];
          if (two) v2 = rc[i2 - s0];
#ifndef LEMGPU_FOREST_EXP
          cnt[i] = v;
          if (two) cnt[i2] = v2;
#endif
        }
        if (pwide) {
          atomicAdd(cnt + p, v);
          if (two) atomicAdd(cnt + p2, v2);
        } else {
          atomicAdd(rp + (p - ps), v);
          if (two) atomicAdd(rp + (p2 - ps), v2);
        }
      }
      // level d-2 takes the slot level d+1 used
      if (d >= 2 && ps - pps <= kFRing)
        for (uint32_t i = rtid; i < ps - pps; i += nact) rq[i] = 1u;
      // the next level (d-1) is staged when its chunks fit behind this level's first one
      const uint32_t kl = qa - (e0 - 1) / kFChunk, khn = qa - ps / kFChunk;
      const bool staged_n = khn <= kl + kFSlotsA - 1;
      if (tid == HT && d > 1) {
        issue_a(kl + kFSlotsA - 1);  // slots of chunks before this level's are free
        if (staged_n) wait_a(qa - (s0 - 1) / kFChunk, khn);
      }
      named_bar_sync(1, nact);
      e0 = s0;
      s0 = ps;
      staged = staged_n;
      uint32_t* t = rc;
      rc = rp;
      rp = rq;
      rq = t;
    }
  }
  __syncthreads();
  if (Dl > 0) {  // level 0: the roots' final counts
    const uint32_t w = lvl(1) - P0;
    if (w <= kFRing)
      for (uint32_t i = tid; i < w; i += kFTPB) cnt[P0 + i] = s.u.a.cnt[0][i];
  }
  if (tid == HT)  // every issued copy has landed before the space is reused
    for (uint32_t k = max(ka_done, ka_next > kFSlotsA ? ka_next - kFSlotsA : 0u); k < ka_next; ++k)
      mbar_wait(&s.bar[k % kFSlotsA], (k / kFSlotsA) & 1u);
  __syncthreads();
  }
  phclk_mark(s_pc, LEMGPU_PHASE_ACCUM);
  if (tid == 0) {
    atomicMax(&ctl->fr_t[0], globaltimer());
    atomicMax(&ctl->fr_maxcells, P1 - P0);
    uint32_t* sb = a.bins + 4096 + 8 * b;  // per-CTA sweep statistics (debug copy 5)
    sb[0] = Dl;
    sb[1] = P1 - P0;
    sb[4] = (uint32_t)((clock64() - ck0) >> 10);
    sb[2] = nact;
  }
  grid_barrier(ctl);  // every CTA's counts are final: F for all positions, grid-wide
  // ---- 7. F and the Newton reciprocal of every cell below level 0, the
  // uplifted elevation of every cell (position-major), grid-wide
  const bool tab = NK == 1 && a.tab_ok;
  uint32_t misses = 0;
  double* Fq = a.hq;
  double* Yq = a.Aq;
  double* Hq = a.hx;
  const uint32_t E = a.lut_entries;
  {
    const uint32_t total = __ldcg(a.levels + D);
    for (uint32_t i = b * kFTPB + tid; i < total; i += gstride) {
      const uint32_t c = __ldcg(a.order + i);
      double hv = a.h[c];
      if (__ldcg(a.ppos + i) == ~0u) {  // level 0: uplift of the interior sources, never eroded
        if (is_interior(a, c)) hv = __dadd_rn(hv, a.du);
        Hq[i] = hv;
        continue;
      }
      Hq[i] = __dadd_rn(hv, a.du);  // every cell below level 0 is interior
      const uint32_t k = __ldcg(cnt + i);
      const uint32_t mem = a.M > 1 ? c / a.MN : 0u;
      const uint32_t cls = dir_class(__ldcg(a.cdir + i));
      double F, y = 0.0;
      if (k < E) {
        if (tab) {
          const double2 fy = __ldg(reinterpret_cast<const double2*>(a.ftab2) + ((size_t)mem * 3 + cls) * E + k);
          F = fy.x;
          y = fy.y;
        } else {
          F = __ldg(a.ftab + ((size_t)mem * 3 + cls) * E + k);
        }
      } else {
        F = erode_F(a, mem, cls, __dmul_rn((double)k, a.w0), misses);
        if (tab) y = __ddiv_rn(1.0, __dadd_rn(1.0, F));
      }
      Fq[i] = F;
      Yq[i] = y;
    }
  }
  grid_barrier(ctl);
  phclk_mark(s_pc, LEMGPU_PHASE_UPLIFT);
  if (tid == 0) atomicMax(&ctl->fr_t[1], globaltimer());
  // erosion: every warp (measured faster than a subset sized to the average
  // level: the widest levels dominate and the Newton solves are latency-bound)
  nact = kFTPB;
  act = tid < nact;
  HT = nact - 1;
  // ---- 8. erosion, level 1 upwards, each cell against its receiver's new h;
  // receiver positions, F, reciprocal and uplifted h of the coming levels
  // stream into shared memory ahead of the sweep (same helper thread)
  unsigned long long iters = 0;
  if (tid < kFSlotsE) mbar_init(&s.bar[kFSlotsA + tid], 1);
  {
    const uint32_t w0n = (Dl > 1 ? lvl(1) : P1) - P0;
    if (w0n <= kFRing)
      for (uint32_t i = tid; i < w0n; i += kFTPB) s.u.e.h[0][i] = __ldcg(Hq + P0 + i);
  }
  uint64_t* bare = s.bar + kFSlotsA;
  const uint32_t qe = Dl > 1 ? lvl(1) / kFChunk : 0u, ke_last = Dl > 1 ? (P1 - 1) / kFChunk - qe : 0u;
  uint32_t ke_next = 0;
  uint32_t ke_done = 0;
  auto issue_e = [&](uint32_t limit) {
    for (; ke_next <= limit && ke_next <= ke_last; ++ke_next) {
      const uint32_t sl = ke_next % kFSlotsE;
      if (ke_next >= kFSlotsE && ke_next - kFSlotsE >= ke_done) mbar_wait(&bare[sl], ((ke_next - kFSlotsE) / kFSlotsE) & 1u);
      const size_t p0 = (size_t)(qe + ke_next) * kFChunk;
      mbar_expect_tx(&bare[sl], kFChunk * 28);
      bulk_g2s(s.u.e.pp[sl], a.ppos + p0, kFChunk * 4, &bare[sl]);
      bulk_g2s(s.u.e.f[sl], Fq + p0, kFChunk * 8, &bare[sl]);
      bulk_g2s(s.u.e.y[sl], Yq + p0, kFChunk * 8, &bare[sl]);
      bulk_g2s(s.u.e.h0[sl], Hq + p0, kFChunk * 8, &bare[sl]);
    }
  };
  auto wait_e = [&](uint32_t kl, uint32_t kh) {
    for (uint32_t k = ke_done; k <= kh; ++k) mbar_wait(&bare[k % kFSlotsE], (k / kFSlotsE) & 1u);
    ke_done = max(ke_done, kh + 1);
  };
  const long long ck1 = clock64();
  // carried level bounds: level d = [s0, e0), level d-1 = [ps, s0)
  uint32_t ps = P0, s0 = Dl > 1 ? lvl(1) : P1, e0 = Dl > 1 ? lvl(2 < Dl ? 2 : Dl) : P1;
  bool staged = false;
  __syncthreads();  // barriers initialised, ring slot of level 0 filled
  if (Dl > 1) {
    staged = (e0 - 1) / kFChunk - qe <= kFSlotsE - 1;
    if (tid == HT) {
      issue_e(kFSlotsE - 1);
      if (staged) wait_e(0, (e0 - 1) / kFChunk - qe);
    }
  }
  __syncthreads();
  if (act) {
    for (uint32_t d = 1; d < Dl; ++d) {
      const uint32_t en = d + 1 < Dl ? lvl(d + 2 < Dl ? d + 2 : Dl) : e0;  // end of level d+1
      const bool wide = e0 - s0 > kFRing, pwide = s0 - ps > kFRing;
      const double* rp = s.u.e.h[(d - 1) & 1];
      double* rc = s.u.e.h[d & 1];
      for (uint32_t i = s0 + tid; i < e0; i += nact) {
        uint32_t p;
        double F, y, h0;
        if (staged) {
          const uint32_t sl = (i / kFChunk - qe) % kFSlotsE, o = i % kFChunk;
          p = s.u.e.pp[sl][o];
          F = s.u.e.f[sl][o];
          y = s.u.e.y[sl][o];
          h0 = s.u.e.h0[sl][o];
        } else {
          p = __ldcg(a.ppos + i);
          F = __ldcg(Fq + i);
          y = __ldcg(Yq + i);
          h0 = __ldcg(Hq + i);
        }
        const double hn = pwide ? __ldcg(Hq + p) : rp[p - ps];
        int itn;
        bool ok;
        double hnew;
        if (tab && F < 0x1p500)
          hnew = newton_n1_tab(h0, hn, F, y, a.eps, a.maxit, itn, ok);
        else if (NK == 1)
          hnew = newton_n1(h0, hn, F, a.eps, a.maxit, itn, ok);
        else
          hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, a.pow_fma, itn, ok);
        if (ok) {
          iters += (unsigned long long)itn;
        } else {
          hnew = h0;
          atomicMin(&ctl->err_cell, __ldcg(a.order + i));
          ctl->err_slot = ctl->slot;
          atomicMax(&ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
        }
        __stcg(Hq + i, hnew);
        if (!wide) rc[i - s0] = hnew;
      }
      // the next level (d+1) is staged when its chunks fit behind this level's first one
      const uint32_t kl = s0 / kFChunk - qe, khn = (en - 1) / kFChunk - qe;
      const bool staged_n = khn <= kl + kFSlotsE - 1;
      if (tid == HT && d + 1 < Dl) {
        issue_e(kl + kFSlotsE - 1);
        if (staged_n) wait_e(e0 / kFChunk - qe, khn);
      }
      named_bar_sync(1, nact);
      ps = s0;
      s0 = e0;
      e0 = en;
      staged = staged_n;
    }
  }
  __syncthreads();
  if (tid == HT)
    for (uint32_t k = max(ke_done, ke_next > kFSlotsE ? ke_next - kFSlotsE : 0u); k < ke_next; ++k)
      mbar_wait(&bare[k % kFSlotsE], (k / kFSlotsE) & 1u);
  flush_counters(ctl, iters, misses);
  if (tid == 0) {
    atomicMax(&ctl->fr_t[2], globaltimer());
    a.bins[4096 + 8 * b + 7] = (uint32_t)((clock64() - ck1) >> 10);
  }
  grid_barrier(ctl);
  // ---- write-back of every escaped cell, grid-wide
  {
    const uint32_t total = __ldcg(a.levels + D);
    for (uint32_t i = b * kFTPB + tid; i < total; i += gstride) a.hout[__ldcg(a.order + i)] = __ldcg(Hq + i);
  }
  phclk_end(s_pc, LEMGPU_PHASE_EROSION, ctl);
  if (last_block_done(ctl) && tid == 0) {
    for (int i = 0; i < 3; ++i) {  // debug timeline: the per-CTA sweeps' latest ends
      if (ctl->ntl < 96) ctl->tl[ctl->ntl++] = ctl->fr_t[i];
    }
    ctl->n0 = nesc;
    ctl->nlev = D;
    ctl->mode = kModeDone;
    ctl->t_phys_end = globaltimer();
    timeline(ctl);
  }
}

}  // namespace lemgpu
