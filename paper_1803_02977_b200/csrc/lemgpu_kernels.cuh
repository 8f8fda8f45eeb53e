// lemgpu_kernels.cuh -- sm_100a kernels of the D8 landscape-evolution step.
//
// Hot path (one timestep):
//   k_recv_donor : receivers (flow_graph.hpp:44-59) + donor bitmask
//                  (flow_graph.hpp:64-72), one smem-staged 3x3-of-3x3 stencil.
//   k_flow       : persistent cooperative kernel.  Breadth-first level order
//                  (traversal.cpp:19-48) by decoupled-look-back frontier
//                  expansion, reverse-level accumulation (accumulation.cpp:7-17),
//                  forward-level uplift + implicit stream-power erosion
//                  (erosion.cpp:19-81), one grid barrier per level.
//
// Arithmetic is FP64 and never contracted: the file is compiled with
// --fmad=false AND every rounding-relevant operation is an explicit
// __d*_rn intrinsic, so results are bit-identical to the reference built
// with -ffp-contract=off (proj/CMakeLists.txt:14).
#pragma once

#include <cooperative_groups.h>
#include <cstdint>

#include "lemgpu.h"

namespace lemgpu {

namespace cg = cooperative_groups;

constexpr int kTPB = 256;             // threads per CTA, all kernels
constexpr int kNW = kTPB / 32;
constexpr uint8_t kNoFlowCode = 8;    // rcode value for kNoFlow
// k_recv_donor tile (output cells); halo of 2 for h, 1 for rcode.
constexpr int kBX = 128;
constexpr int kBY = 32;
// k_flow scan tiles.
constexpr int kL0IPT = 16;                 // level-0 cells per thread (one uint4 of rcodes)
constexpr int kL0Tile = kTPB * kL0IPT;     // 4096 cells
constexpr int kExIPT = 4;                  // frontier items per thread
constexpr int kExTile = kTPB * kExIPT;     // 1024 frontier cells

// Frozen D8 stencil (src/neighborhood.cpp:12): k -> (ox, oy).  The
// opposite direction of k is 7-k.  D4 is the cardinal subsequence
// {1,3,4,6} (neighborhood.cpp:20-29), kept at its D8 slot so stencil order
// and the opposite-direction rule are shared.
__host__ __device__ constexpr int dir_ox(int k) { return (k == 0 || k == 3 || k == 5) ? -1 : (k == 1 || k == 6) ? 0 : 1; }
__host__ __device__ constexpr int dir_oy(int k) { return k < 3 ? -1 : k < 5 ? 0 : 1; }
__host__ __device__ constexpr bool dir_in(int conn, int k) {
  return conn == 8 || k == 1 || k == 3 || k == 4 || k == 6;
}

// Device control block (one per context).
struct Ctl {
  uint32_t epoch;           // look-back status epoch (see lookback())
  uint32_t err_flag;        // sticky LEMGPU_* of the first failing step
  uint32_t err_cell;        // min failing cell (any failing cell is acceptable)
  uint32_t level_total[2];  // children produced by the level just expanded
  uint32_t pad;
  unsigned long long t_k1_begin, t_k1_end;  // globaltimer span of k_recv_donor
};

struct StepArgs {
  // geometry (stacked members: rows [m*H, (m+1)*H) belong to member m)
  uint32_t W, H, M;
  uint32_t N;         // W*H*M  (< 2^32, RunConfig::validate, config.cpp:159-161)
  uint32_t MN;        // W*H
  uint32_t Htot;      // H*M
  uint32_t perim;     // perimeter cells over all members
  int conn;
  int nkind;          // 1: n==1, 2: n==2, 0: general n
  int maxit;
  int lut_exact;      // A is always an exact integer multiple of w0
  int w0_is_one;
  uint32_t lut_entries;
  uint32_t dist_one;  // bit k set when dist[k] == 1.0 (division is the identity)
  int off[8];         // linear offset of direction k (oy*W + ox)
  double dist[8];     // offset_length of direction k (neighborhood.hpp:17-23)
  double powdist_h, powdist_v, powdist_d;  // host-libm pow(dist, n): horizontal, vertical, diagonal
  double du, w0, n_exp, eps;
  const double* kdt;  // per member K*dt
  const double* mexp; // per member m
  const double* lut;  // per member: lut[m*lut_entries + a] = pow(a*w0, m_m), host libm
  // state / scratch
  double* h;
  uint8_t* rcode;
  uint8_t* dmask;
  uint32_t* order;
  uint32_t* ppos;
  uint32_t* fc;
  uint8_t* cdir;
  double* Aq;
  double* hq;
  uint32_t* levels;
  unsigned long long* tstat;
  Ctl* ctl;
  lemgpu_diag* diag;
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

// Exclusive block scan of one u32 per thread; *total gets the block sum.
// scratch: kNW+1 u32 of shared memory.  Contains the barriers it needs and
// leaves scratch reusable on return.
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
    if (lane < kNW) scratch[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  const uint32_t warp_excl = warp ? scratch[warp - 1] : 0u;
  *total = scratch[kNW - 1];
  __syncthreads();
  return warp_excl + x - v;
}

// Decoupled look-back (single-pass chained scan).  Called by warp 0 of the
// CTA that owns tile t; returns the exclusive prefix of tile t in every
// lane.  Status word: [63:34] epoch, [33:32] flag (1 aggregate, 2 inclusive),
// [31:0] value.  A fresh epoch per scan makes stale words from earlier scans
// invalid without clearing the array.  Tiles of one scan are owned
// round-robin by co-resident CTAs that process them in increasing order, so
// the smallest unfinished tile can always make progress (no deadlock).
__device__ __forceinline__ uint32_t lookback(unsigned long long* tstat, uint32_t t, uint32_t agg,
                                             uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  const unsigned long long tag_agg = (unsigned long long)((epoch << 2) | 1u) << 32;
  const unsigned long long tag_inc = (unsigned long long)((epoch << 2) | 2u) << 32;
  if (t == 0) {
    if (lane == 0) st_relaxed_u64(tstat, tag_inc | agg);
    return 0u;
  }
  if (lane == 0) st_relaxed_u64(tstat + t, tag_agg | agg);
  uint32_t excl = 0;
  long long idx = (long long)t - 1;
  while (true) {
    const long long j = idx - lane;
    uint32_t flag = 2, val = 0;
    if (j >= 0) {
      unsigned long long s;
      do {
        s = ld_relaxed_u64(tstat + j);
        const uint32_t hi = (uint32_t)(s >> 32);
        flag = (hi >> 2) == epoch ? (hi & 3u) : 0u;
      } while (flag == 0);
      val = (uint32_t)s;
    }
    const uint32_t incmask = __ballot_sync(0xffffffffu, flag == 2);
    const int first = incmask ? __ffs(incmask) - 1 : 31;
    excl += __reduce_add_sync(0xffffffffu, lane <= first ? val : 0u);
    if (incmask) break;
    idx -= 32;
  }
  if (lane == 0) st_relaxed_u64(tstat + t, tag_inc | (excl + agg));
  return excl;
}

// ------------------------------------------------------- receivers/donors

// One CTA: a kBY x kBX tile of cells.  h is staged with a 2-cell halo, the
// receiver code with a 1-cell halo, so the donor mask of every tile cell is
// computed from receivers evaluated in the same CTA -- one HBM read of h,
// one byte written per output array, no atomics (pull-based donors).
template <int CONN>
__global__ void __launch_bounds__(kTPB) k_recv_donor(StepArgs a) {
  __shared__ double sh[kBY + 4][kBX + 4];
  __shared__ uint8_t rc[kBY + 2][kBX + 2 + 2];
  if (ld_volatile_u32(&a.ctl->err_flag)) return;
  if (threadIdx.x == 0) atomicMin(&a.ctl->t_k1_begin, globaltimer());
  const long long x0 = (long long)blockIdx.x * kBX, y0 = (long long)blockIdx.y * kBY;
  const long long W = a.W, Ht = a.Htot;

  for (int i = threadIdx.x; i < (kBY + 4) * (kBX + 4); i += kTPB) {
    const int r = i / (kBX + 4), cc = i - r * (kBX + 4);
    const long long gy = y0 - 2 + r, gx = x0 - 2 + cc;
    double v = 0.0;
    if (gy >= 0 && gy < Ht && gx >= 0 && gx < W) v = __ldg(a.h + gy * W + gx);
    sh[r][cc] = v;
  }
  __syncthreads();

  // steepest_receiver (flow_graph.hpp:44-59): s = (ec - en) / dist, strict
  // '>' against s_max starting at 0, first maximum in stencil order wins.
  // Neighbours with ec - en <= 0 give s <= 0 and can never win, so their
  // division is skipped; division by a unit distance is the identity.
  for (int i = threadIdx.x; i < (kBY + 2) * (kBX + 2); i += kTPB) {
    const int r = i / (kBX + 2), cc = i - r * (kBX + 2);
    const long long gy = y0 - 1 + r, gx = x0 - 1 + cc;
    uint8_t code = kNoFlowCode;
    if (gy >= 0 && gy < Ht && gx > 0 && gx < W - 1) {
      const uint32_t yl = (uint32_t)(gy % a.H);
      if (yl > 0 && yl < a.H - 1) {
        const double ec = sh[r + 1][cc + 1];
        double smax = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (!dir_in(CONN, k)) continue;
          const double d = __dsub_rn(ec, sh[r + 1 + dir_oy(k)][cc + 1 + dir_ox(k)]);
          if (d > 0.0) {
            const double s = ((a.dist_one >> k) & 1u) ? d : __ddiv_rn(d, a.dist[k]);
            if (s > smax) {
              smax = s;
              code = (uint8_t)k;
            }
          }
        }
      }
    }
    rc[r][cc] = code;
  }
  __syncthreads();

  // donors_of (flow_graph.hpp:64-72): neighbour n in direction k donates to
  // c iff rec[n] == c, i.e. n's code is the opposite direction 7-k.
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < kBY; r += kNW) {
    const long long gy = y0 + r;
    if (gy >= Ht) break;
    const int cc0 = lane * 4;
    uint32_t pc = 0, pm = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int cc = cc0 + j;
      uint32_t m = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!dir_in(CONN, k)) continue;
        if (rc[r + 1 + dir_oy(k)][cc + 1 + dir_ox(k)] == (uint8_t)(7 - k)) m |= 1u << k;
      }
      pm |= m << (8 * j);
      pc |= (uint32_t)rc[r + 1][cc + 1] << (8 * j);
    }
    const long long gx = x0 + cc0;
    const long long base = gy * W + gx;
    if (gx + 3 < W && (W & 3) == 0) {
      *reinterpret_cast<uint32_t*>(a.rcode + base) = pc;
      *reinterpret_cast<uint32_t*>(a.dmask + base) = pm;
    } else {
      for (int j = 0; j < 4; ++j)
        if (gx + j < W) {
          a.rcode[base + j] = (uint8_t)(pc >> (8 * j));
          a.dmask[base + j] = (uint8_t)(pm >> (8 * j));
        }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) atomicMax(&a.ctl->t_k1_end, globaltimer());
}

// ------------------------------------------------------------ flow kernel

struct FlowSmem {
  uint32_t scan[kNW + 1];
  uint32_t bcast;
  uint32_t ord[kExTile];
  unsigned long long red[kNW];
  uint32_t red32[kNW];
};

// Level 0 (traversal.cpp:27-29): every cell with rec == kNoFlow, ascending.
__device__ __forceinline__ void tile_level0(const StepArgs& a, FlowSmem& sm, uint32_t t,
                                            uint32_t ntiles, uint32_t epoch) {
  const uint32_t cell0 = t * (uint32_t)kL0Tile + threadIdx.x * kL0IPT;
  uint32_t w[4] = {0, 0, 0, 0};
  if ((unsigned long long)cell0 + kL0IPT <= a.N) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(a.rcode + cell0));
    w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
  } else {
    for (int j = 0; j < kL0IPT; ++j)
      if (cell0 + j < a.N) w[j >> 2] |= (uint32_t)a.rcode[cell0 + j] << (8 * (j & 3));
  }
  uint32_t eq[4], cnt = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    eq[q] = __vcmpeq4(w[q], 0x08080808u);
    cnt += __popc(eq[q]) >> 3;
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan(cnt, &total, sm.scan);
  if (threadIdx.x < 32) {
    const uint32_t pre = lookback(a.tstat, t, total, epoch);
    if (threadIdx.x == 0) sm.bcast = pre;
  }
  __syncthreads();
  const uint32_t pre = sm.bcast;
  uint32_t out = pre + excl;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t e = eq[q];
    while (e) {
      const int bit = __ffs(e) - 1;
      a.order[out++] = cell0 + q * 4 + (bit >> 3);
      e &= ~(0xFFu << (bit & ~7));
    }
  }
  if (t == ntiles - 1 && threadIdx.x == 0) {
    a.ctl->level_total[0] = pre + total;
    a.levels[0] = 0;
    a.levels[1] = pre + total;
  }
  __syncthreads();
}

// Expand frontier [lo, hi) into the next level (traversal.cpp:35-44): for
// each frontier cell in order, its donors in stencil (= bit) order.  The
// exclusive scan of popcount(dmask) over the frontier is the first-child
// position fc[pos]; children also record their parent position (ppos) and
// the direction parent->child (cdir) for the erosion sweep.
__device__ __forceinline__ void tile_expand(const StepArgs& a, FlowSmem& sm, uint32_t t,
                                            uint32_t ntiles, uint32_t lo, uint32_t hi,
                                            uint32_t epoch, int par) {
  const uint32_t tb = lo + t * (uint32_t)kExTile;
#pragma unroll
  for (int j = 0; j < kExIPT; ++j) {
    const uint32_t p = tb + j * kTPB + threadIdx.x;
    sm.ord[j * kTPB + threadIdx.x] = p < hi ? a.order[p] : LEMGPU_NOFLOW;
  }
  __syncthreads();
  uint32_t c[kExIPT], m[kExIPT], cnt = 0;
#pragma unroll
  for (int j = 0; j < kExIPT; ++j) {
    c[j] = sm.ord[threadIdx.x * kExIPT + j];
    m[j] = c[j] != LEMGPU_NOFLOW ? (uint32_t)__ldg(a.dmask + c[j]) : 0u;
    cnt += __popc(m[j]);
  }
  uint32_t total;
  const uint32_t excl = block_excl_scan(cnt, &total, sm.scan);
  if (threadIdx.x < 32) {
    const uint32_t pre = lookback(a.tstat, t, total, epoch);
    if (threadIdx.x == 0) sm.bcast = pre;
  }
  __syncthreads();
  const uint32_t pre = sm.bcast;
  uint32_t out = hi + pre + excl;
#pragma unroll
  for (int j = 0; j < kExIPT; ++j) {
    const uint32_t pos = tb + threadIdx.x * kExIPT + j;
    if (pos < hi) {
      a.fc[pos] = out;
      uint32_t mm = m[j];
      while (mm) {
        const int k = __ffs(mm) - 1;
        mm &= mm - 1;
        a.order[out] = (uint32_t)((long long)c[j] + dir_ox(k) + (long long)dir_oy(k) * a.W);
        a.ppos[out] = pos;
        a.cdir[out] = (uint8_t)k;
        ++out;
      }
    }
  }
  if (t == ntiles - 1 && threadIdx.x == 0) a.ctl->level_total[par] = pre + total;
  __syncthreads();
}

// newton_erode_cell (erosion.cpp:19-34) for n == 1.  glibc pow(x, 1.0) == x
// and pow(x, 0.0) == 1 exactly (SURVEY 8(c) [measured]), so residual =
// (h - h0) + F*diff and slope = 1.0 + (F*1.0)*1.0 = 1.0 + F, evaluated in
// the reference's association order.
__device__ __forceinline__ double newton_n1(double h0, double hn, double F, double eps, int maxit,
                                            int& iters, bool& ok) {
  double h = h0, hp = h0;
  const double slope = __dadd_rn(1.0, F);
  for (int it = 1; it <= maxit; ++it) {
    const double diff = __dsub_rn(h, hn);
    const double res = __dadd_rn(__dsub_rn(h, h0), __dmul_rn(F, diff));
    h = __dsub_rn(h, __ddiv_rn(res, slope));
    if (h < hn) h = hn;
    const double d = __dsub_rn(h, hp);
    hp = h;
    if (fabs(d) <= eps) {
      iters = it;
      ok = true;
      return h;
    }
  }
  iters = maxit;
  ok = false;
  return h;
}

// General n.  n == 2 uses diff*diff for pow(diff, 2) (correctly rounded;
// glibc pow differs from it in ~0.08% of inputs by <= 1 ulp, SURVEY 7 hard
// part 2) and the identity pow(diff, 1) = diff; other n use CUDA pow.  The
// elevation is then within the stated 1e-9 relative tolerance, not bitwise.
template <int NK>
__device__ __forceinline__ double newton_gen(double h0, double hn, double F, double n, double eps,
                                             int maxit, int& iters, bool& ok) {
  double h = h0, hp = h0;
  const double Fn = __dmul_rn(F, n);
  for (int it = 1; it <= maxit; ++it) {
    const double diff = __dsub_rn(h, hn);
    double pn, pn1;
    if (NK == 2) {
      pn = __dmul_rn(diff, diff);
      pn1 = diff;
    } else {
      pn = pow(diff, n);
      pn1 = pow(diff, __dsub_rn(n, 1.0));
    }
    const double res = __dadd_rn(__dsub_rn(h, h0), __dmul_rn(F, pn));
    const double slope = __dadd_rn(1.0, __dmul_rn(Fn, pn1));
    h = __dsub_rn(h, __ddiv_rn(res, slope));
    if (h < hn) h = hn;
    const double d = __dsub_rn(h, hp);
    hp = h;
    if (fabs(d) <= eps) {
      iters = it;
      ok = true;
      return h;
    }
  }
  iters = maxit;
  ok = false;
  return h;
}

template <int NK>
__device__ __forceinline__ void erode_pos(const StepArgs& a, uint32_t pos, unsigned long long& iters,
                                          uint32_t& misses) {
  const uint32_t c = a.order[pos];
  const uint32_t p = a.ppos[pos];
  const int k = a.cdir[pos];           // parent -> child; child -> receiver is 7-k
  const double A = a.Aq[pos];
  const double hn = a.hq[p];           // receiver, already updated this step
  const double h0 = __dadd_rn(a.h[c], a.du);  // uplift (erosion.cpp:52-57), one rounding
  const uint32_t mem = a.M > 1 ? c / a.MN : 0u;
  // F = K*dt*pow(A,m)/pow(dist,n) (erosion.cpp:38-39): (K*dt) first.
  double powA;
  const double q = a.w0_is_one ? A : __ddiv_rn(A, a.w0);
  if (a.lut_exact && q < (double)a.lut_entries && q == floor(q)) {
    powA = __ldg(a.lut + (size_t)mem * a.lut_entries + (uint32_t)q);
  } else {
    powA = pow(A, __ldg(a.mexp + mem));
    ++misses;
  }
  // pow(dist(c, rec[c]), n): opposite directions share a distance class.
  const double pd = (k == 1 || k == 6) ? a.powdist_v : (k == 3 || k == 4) ? a.powdist_h : a.powdist_d;
  const double F = __ddiv_rn(__dmul_rn(__ldg(a.kdt + mem), powA), pd);
  int it;
  bool ok;
  double hnew;
  if (NK == 1)
    hnew = newton_n1(h0, hn, F, a.eps, a.maxit, it, ok);
  else
    hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, it, ok);
  if (ok) {
    a.h[c] = hnew;
    a.hq[pos] = hnew;
    iters += (unsigned long long)it;
  } else {
    atomicMin(&a.ctl->err_cell, c);
    atomicMax(&a.ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
  }
}

template <int NK>
__global__ void __launch_bounds__(kTPB) k_flow(StepArgs a) {
  cg::grid_group grid = cg::this_grid();
  __shared__ FlowSmem sm;
  const uint32_t G = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  const bool lead = (b == 0 && tid == 0);
  Ctl* ctl = a.ctl;
  if (ld_volatile_u32(&ctl->err_flag)) {  // sticky failure of an earlier step: not run
    if (lead) a.diag->status = 0xFFFFFFFFu;
    return;
  }

  uint32_t E0 = ld_volatile_u32(&ctl->epoch);
  const unsigned long long t_begin = globaltimer();
  if ((unsigned long long)E0 + a.N + 4ull >= (1ull << 30)) {
    // Epoch space nearly exhausted: clear all status words and restart.
    const uint32_t ntst = a.N / kExTile + 2;
    for (uint32_t i = b * kTPB + tid; i < ntst; i += G * kTPB) a.tstat[i] = 0ull;
    E0 = 1;
    grid.sync();
  }
  if (lead) {
    a.diag->newton_iters = 0;
    a.diag->lut_misses = 0;
    a.diag->status = 0;
    a.diag->err_cell = LEMGPU_NOFLOW;
    a.fc[a.N] = a.N;
  }

  // ---- level 0
  const uint32_t nt0 = (a.N + kL0Tile - 1) / kL0Tile;
  for (uint32_t t = b; t < nt0; t += G) tile_level0(a, sm, t, nt0, E0);
  grid.sync();

  // ---- breadth-first expansion, one grid barrier per level
  uint32_t lo = 0, hi = ld_volatile_u32(&ctl->level_total[0]);
  uint32_t l = 0;
  while (true) {
    const uint32_t F = hi - lo;
    const uint32_t nt = (F + kExTile - 1) / kExTile;
    for (uint32_t t = b; t < nt; t += G) tile_expand(a, sm, t, nt, lo, hi, E0 + 1 + l, (l + 1) & 1);
    grid.sync();
    const uint32_t total = ld_volatile_u32(&ctl->level_total[(l + 1) & 1]);
    if (total == 0) break;
    if (lead) a.levels[l + 2] = hi + total;
    lo = hi;
    hi += total;
    ++l;
  }
  const uint32_t nlev = l + 1;
  const unsigned long long t_order = globaltimer();
  bool failed = false;
  if (hi != a.N) {  // cells unreachable from the sources: a receiver cycle (traversal.cpp:46)
    if (lead) {
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_cell = hi;  // cells placed
    }
    failed = true;
  }

  // ---- accumulation, deepest level first (accumulation.cpp:7-17); the
  // level-0 pass also applies uplift to the level-0 pits (erosion.cpp:52-57).
  unsigned long long t_accum = t_order;
  if (!failed) {
    for (int L = (int)nlev - 1; L >= 0; --L) {
      const uint32_t s = a.levels[L], e = a.levels[L + 1];
      for (uint32_t pos = s + b * kTPB + tid; pos < e; pos += G * kTPB) {
        double acc = a.w0;
        const uint32_t j0 = a.fc[pos], j1 = a.fc[pos + 1];
        for (uint32_t j = j0; j < j1; ++j) acc = __dadd_rn(acc, a.Aq[j]);
        a.Aq[pos] = acc;
        if (L == 0) {
          const uint32_t c = a.order[pos];
          const uint32_t x = c % a.W, yl = (c / a.W) % a.H;
          double hv = a.h[c];
          if (x > 0 && x < a.W - 1 && yl > 0 && yl < a.H - 1) {
            hv = __dadd_rn(hv, a.du);
            a.h[c] = hv;
          }
          a.hq[pos] = hv;
        }
      }
      grid.sync();
    }
    t_accum = globaltimer();

    // ---- erosion, levels 1..L-1 downstream -> upstream (erosion.cpp:66-81)
    unsigned long long iters = 0;
    uint32_t misses = 0;
    for (uint32_t L = 1; L < nlev; ++L) {
      const uint32_t s = a.levels[L], e = a.levels[L + 1];
      for (uint32_t pos = s + b * kTPB + tid; pos < e; pos += G * kTPB) erode_pos<NK>(a, pos, iters, misses);
      grid.sync();
      if (ld_volatile_u32(&ctl->err_flag)) break;
    }
    // deterministic integer reduction of the per-thread counters
    const int lane = tid & 31, warp = tid >> 5;
    for (int o = 16; o; o >>= 1) {
      iters += __shfl_down_sync(0xffffffffu, iters, o);
      misses += __shfl_down_sync(0xffffffffu, misses, o);
    }
    if (lane == 0) {
      sm.red[warp] = iters;
      sm.red32[warp] = misses;
    }
    __syncthreads();
    if (tid == 0) {
      unsigned long long s = 0;
      uint32_t mm = 0;
      for (int w = 0; w < kNW; ++w) {
        s += sm.red[w];
        mm += sm.red32[w];
      }
      if (s) atomicAdd(reinterpret_cast<unsigned long long*>(&a.diag->newton_iters), s);
      if (mm) atomicAdd(&a.diag->lut_misses, mm);
    }
  }
  grid.sync();
  if (lead) {
    const unsigned long long t_end = globaltimer();
    const uint32_t st = ctl->err_flag;
    lemgpu_diag* d = a.diag;
    d->seconds[LEMGPU_PHASE_RECEIVERS] = (double)(ctl->t_k1_end - ctl->t_k1_begin) * 1e-9;
    d->seconds[LEMGPU_PHASE_DONORS] = 0.0;  // fused into k_recv_donor
    d->seconds[LEMGPU_PHASE_ORDER] = (double)(t_order - t_begin) * 1e-9;
    d->seconds[LEMGPU_PHASE_ACCUM] = (double)(t_accum - t_order) * 1e-9;
    d->seconds[LEMGPU_PHASE_UPLIFT] = 0.0;  // fused into the accumulation / erosion sweeps
    d->seconds[LEMGPU_PHASE_EROSION] = (double)(t_end - t_accum) * 1e-9;
    d->nlevels = nlev;
    d->interior_noflow = a.levels[1] - a.perim;
    d->status = st;
    d->err_cell = st ? ctl->err_cell : LEMGPU_NOFLOW;
    ctl->epoch = E0 + 2 + l;
    ctl->t_k1_begin = ~0ull;
    ctl->t_k1_end = 0ull;
  }
}

// ------------------------------------------------------------ utilities

// lem::generate_terrain (terrain.cpp:12-31), per member seed.
__global__ void k_terrain(double* h, uint32_t N, uint32_t MN, const unsigned long long* seeds) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    const uint32_t m = i / MN, li = i - m * MN;
    unsigned long long z = seeds[m] + (unsigned long long)li * 0x9E3779B97F4A7C15ull;
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    h[i] = __dmul_rn((double)(z >> 11), 0x1.0p-53);
  }
}

// First non-finite cell (run_simulation's input check, scheduler.cpp:474-477).
__global__ void k_check_finite(const double* h, uint32_t N, uint32_t* first_bad) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x)
    if (!isfinite(h[i])) atomicMin(first_bad, i);
}

// FlowGraph export in the reference layout (flow_graph.hpp:19-38).
__global__ void k_export_graph(StepArgs a, uint32_t* rec, uint8_t* dnum, uint32_t* donor) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
    const uint8_t code = a.rcode[c];
    if (rec) rec[c] = code == kNoFlowCode ? LEMGPU_NOFLOW : (uint32_t)((long long)c + a.off[code]);
    const uint32_t m = a.dmask[c];
    if (dnum) dnum[c] = (uint8_t)__popc(m);
    if (donor) {
      uint32_t* slot = donor + (size_t)c * a.conn;
      int j = 0;
      for (int k = 0; k < 8; ++k)
        if ((m >> k) & 1u) slot[j++] = (uint32_t)((long long)c + a.off[k]);
      for (; j < a.conn; ++j) slot[j] = LEMGPU_NOFLOW;
    }
  }
}

__global__ void k_export_accum(StepArgs a, double* A) {
  for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < a.N; p += gridDim.x * blockDim.x)
    A[a.order[p]] = a.Aq[p];
}

// Per-member {sum, max, min} partials over fixed chunks (deterministic).
__global__ void k_stats_partial(const double* h, uint32_t MN, uint32_t chunks, double* part) {
  const uint32_t m = blockIdx.y, ch = blockIdx.x;
  const uint32_t per = (MN + chunks - 1) / chunks;
  const uint32_t s = ch * per, e = min(MN, s + per);
  const double* hm = h + (size_t)m * MN;
  double sum = 0.0, mx = -INFINITY, mn = INFINITY;
  for (uint32_t i = s + threadIdx.x; i < e; i += blockDim.x) {
    const double v = hm[i];
    sum = __dadd_rn(sum, v);
    mx = fmax(mx, v);
    mn = fmin(mn, v);
  }
  __shared__ double ss[kTPB], sx[kTPB], sn[kTPB];
  ss[threadIdx.x] = sum;
  sx[threadIdx.x] = mx;
  sn[threadIdx.x] = mn;
  __syncthreads();
  for (int o = kTPB / 2; o; o >>= 1) {
    if ((int)threadIdx.x < o) {
      ss[threadIdx.x] = __dadd_rn(ss[threadIdx.x], ss[threadIdx.x + o]);
      sx[threadIdx.x] = fmax(sx[threadIdx.x], sx[threadIdx.x + o]);
      sn[threadIdx.x] = fmin(sn[threadIdx.x], sn[threadIdx.x + o]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double* o = part + ((size_t)m * chunks + ch) * 3;
    o[0] = ss[0];
    o[1] = sx[0];
    o[2] = sn[0];
  }
}

__global__ void k_stats_final(const double* part, uint32_t M, uint32_t chunks, uint32_t MN, double* out) {
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < M; m += gridDim.x * blockDim.x) {
    double sum = 0.0, mx = -INFINITY, mn = INFINITY;
    for (uint32_t ch = 0; ch < chunks; ++ch) {
      const double* p = part + ((size_t)m * chunks + ch) * 3;
      sum = __dadd_rn(sum, p[0]);
      mx = fmax(mx, p[1]);
      mn = fmin(mn, p[2]);
    }
    out[4 * m + 0] = __ddiv_rn(sum, (double)MN);
    out[4 * m + 1] = mx;
    out[4 * m + 2] = mn;
    out[4 * m + 3] = sum;
  }
}

}  // namespace lemgpu
