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
constexpr int kExIPT = 8;                  // frontier items per thread
constexpr int kExTile = kTPB * kExIPT;     // 2048 frontier cells

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
  uint32_t ntl, pad2;
  unsigned long long tl[96];  // debug timeline of the last k_flow (globaltimer at each barrier)
};
#define LG_TL(lead, ctl)                                             \
  do {                                                               \
    if ((lead) && (ctl)->ntl < 96) (ctl)->tl[(ctl)->ntl++] = globaltimer(); \
  } while (0)

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
  int unit_card;      // dx == dy == 1: cardinal slopes are the drops themselves
  double rinv_diag;   // RN(1 / dist_diag), used only to pre-decide far-from-tie comparisons
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
  uint32_t* cbound;   // per source chunk: first position at each level
  double* Aq;
  double* hq;
  uint32_t* levels;
  unsigned long long* tstat;
  Ctl* ctl;
  lemgpu_diag* diag;
};

// ---------------------------------------------------------------- helpers

// IEEE round-to-nearest arithmetic usable on host and device (the host side
// is compiled with -ffp-contract=off, so plain operators do not fuse).
#ifdef __CUDA_ARCH__
#define LG_SUB(x, y) __dsub_rn((x), (y))
#define LG_MUL(x, y) __dmul_rn((x), (y))
#define LG_DIV(x, y) __ddiv_rn((x), (y))
#else
#define LG_SUB(x, y) ((x) - (y))
#define LG_MUL(x, y) ((x) * (y))
#define LG_DIV(x, y) ((x) / (y))
#endif

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

// Stencil slots are addressed relative to the centre (1,1) of a 3x3 window.
// steepest_receiver (flow_graph.hpp:44-59): s_k = (ec - en_k) / dist_k, strict
// '>' against s_max = 0, so the FIRST maximum in stencil order wins.
//
// Fast path for unit cardinal spacing (dx == dy == 1, the reference default):
// cardinal slopes are the drops themselves (x / 1.0 is exact) and the only
// rounding-sensitive quantity is the diagonal quotient RN(d / sqrt2).  RN is
// monotone, so the best diagonal is the one with the largest drop dd and the
// class comparison RN(dd/c) vs dc is decided by one multiplication by RN(1/c)
// unless the two are within 2^-40 relative (then the true IEEE division is
// taken).  Diagonal ties are resolved exactly: only drops within 2^-50 of dd
// can round to the same quotient, and those are divided for real.  The
// result is the reference's argmax bit for bit, with ~0 divisions per cell.
// The reference loop itself (with the exact skips: ec - en <= 0 can never
// beat s_max >= 0, and x / 1.0 == x).  Used directly for general spacing /
// D4, and as the exact slow path of the D8 fast path below.
template <int CONN>
__host__ __device__ __forceinline__ uint8_t receiver_code_ref(const double (&d)[8], const StepArgs& a) {
  double smax = 0.0;
  uint8_t code = kNoFlowCode;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (!dir_in(CONN, k)) continue;
    if (d[k] > 0.0) {
      const double s = ((a.dist_one >> k) & 1u) ? d[k] : LG_DIV(d[k], a.dist[k]);
      if (s > smax) {
        smax = s;
        code = (uint8_t)k;
      }
    }
  }
  return code;
}

template <int CONN>
__host__ __device__ __forceinline__ uint8_t receiver_code(const double (&d)[8], const StepArgs& a) {
  if (CONN == 8 && a.unit_card) {
    const double dc = fmax(fmax(d[1], d[3]), fmax(d[4], d[6]));
    const double dd = fmax(fmax(d[0], d[2]), fmax(d[5], d[7]));
    const bool cpos = dc > 0.0, dpos = dd > 0.0;
    if (!cpos && !dpos) return kNoFlowCode;
    bool card_ok = cpos, diag_ok = dpos;
    if (cpos && dpos) {
      // RN(dd / c) vs dc, decided by RN(dd * RN(1/c)) unless within 2^-40
      const double approx = LG_MUL(dd, a.rinv_diag);
      if (dd < 0x1p-1000 || dc < 0x1p-1000 || fabs(LG_SUB(approx, dc)) <= LG_MUL(dc, 0x1p-40))
        return receiver_code_ref<CONN>(d, a);
      diag_ok = approx > dc;
      card_ok = !diag_ok;
    }
    uint32_t mask = 0;
    if (card_ok) {
      mask = (d[1] == dc ? 0x02u : 0u) | (d[3] == dc ? 0x08u : 0u) | (d[4] == dc ? 0x10u : 0u) |
             (d[6] == dc ? 0x40u : 0u);
    } else {
      // a second diagonal within 2^-50 of dd may round to the same quotient
      const double near = LG_MUL(dd, 1.0 - 0x1p-50);
      const bool amb = (d[0] > near && d[0] != dd) || (d[2] > near && d[2] != dd) ||
                       (d[5] > near && d[5] != dd) || (d[7] > near && d[7] != dd);
      if (amb) return receiver_code_ref<CONN>(d, a);
      mask = (d[0] == dd ? 0x01u : 0u) | (d[2] == dd ? 0x04u : 0u) | (d[5] == dd ? 0x20u : 0u) |
             (d[7] == dd ? 0x80u : 0u);
    }
#ifdef __CUDA_ARCH__
    return (uint8_t)(__ffs(mask) - 1);
#else
    return (uint8_t)__builtin_ctz(mask);
#endif
  }
  return receiver_code_ref<CONN>(d, a);
}

// One CTA: a kBY x kBX tile of cells.  h is staged with a 2-cell halo, the
// receiver code with a 1-cell halo, so the donor mask of every tile cell is
// computed from receivers evaluated in the same CTA -- one HBM read of h,
// one byte written per output array, no atomics (pull-based donors).
// Warp-per-row loops keep all row arithmetic warp-uniform.
template <int CONN>
__global__ void __launch_bounds__(kTPB) k_recv_donor(StepArgs a) {
  __shared__ double sh[kBY + 4][kBX + 4];
  __shared__ uint8_t rc[kBY + 2][kBX + 4];
  if (ld_volatile_u32(&a.ctl->err_flag)) return;
  if (threadIdx.x == 0) atomicMin(&a.ctl->t_k1_begin, globaltimer());
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
  const uint32_t W = a.W, Ht = a.Htot;

  // ---- stage h: rows y0-2 .. y0+kBY+1, columns x0-2 .. x0+kBX+1
  for (int r = warp; r < kBY + 4; r += kNW) {
    const int gy = (int)y0 - 2 + r;
    const bool rowok = gy >= 0 && (uint32_t)gy < Ht;
    const double* row = a.h + (size_t)(rowok ? gy : 0) * W;
#pragma unroll
    for (int j = 0; j < kBX / 32; ++j) {
      const uint32_t gx = x0 + lane + 32 * j;
      sh[r][2 + lane + 32 * j] = (rowok && gx < W) ? __ldg(row + gx) : 0.0;
    }
    if (lane < 4) {
      const int cc = lane < 2 ? lane : kBX + lane;  // 0,1 | kBX+2,kBX+3
      const int gx = (int)x0 - 2 + cc;
      sh[r][cc] = (rowok && gx >= 0 && (uint32_t)gx < W) ? __ldg(row + gx) : 0.0;
    }
  }
  __syncthreads();

  // ---- receiver codes: rows y0-1 .. y0+kBY, columns x0-1 .. x0+kBX
  for (int r = warp; r < kBY + 2; r += kNW) {
    const int gy = (int)y0 - 1 + r;
    bool rowint = false;
    if (gy >= 0 && (uint32_t)gy < Ht) {
      const uint32_t yl = (uint32_t)gy % a.H;
      rowint = yl > 0 && yl < a.H - 1;
    }
    for (int j = 0; j <= kBX / 32; ++j) {
      int cc;  // column within rc (rc column c <-> sh column c+1 <-> gx = x0-1+c)
      if (j < kBX / 32) {
        cc = 1 + lane + 32 * j;
      } else {
        if (lane >= 2) break;
        cc = lane == 0 ? 0 : kBX + 1;
      }
      const int gx = (int)x0 - 1 + cc;
      uint8_t code = kNoFlowCode;
      if (rowint && gx > 0 && gx < (int)W - 1) {
        const double ec = sh[r + 1][cc + 1];
        double d[8];
#pragma unroll
        for (int k = 0; k < 8; ++k)
          d[k] = dir_in(CONN, k) ? __dsub_rn(ec, sh[r + 1 + dir_oy(k)][cc + 1 + dir_ox(k)]) : 0.0;
        code = receiver_code<CONN>(d, a);
      }
      rc[r][cc] = code;
    }
  }
  __syncthreads();

  // ---- donors_of (flow_graph.hpp:64-72): neighbour n in direction k donates
  // to c iff rec[n] == c, i.e. n's code is the opposite direction 7-k.
  for (int r = warp; r < kBY; r += kNW) {
    const uint32_t gy = y0 + r;
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
    const uint32_t gx = x0 + cc0;
    const size_t base = (size_t)gy * W + gx;
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
//
// Phase A (order): level 0 by a single-pass compaction of rcode == kNoFlow,
// then one frontier expansion per level -- decoupled look-back scan of
// popcount(dmask) -> first-child positions fc[] and the children themselves.
// One grid barrier per level (the only inherently level-synchronous part).
//
// Phase B (accumulation + uplift + erosion) exploits the single-receiver
// structure the way the paper's RB+PQ strategy does (scheduler.cpp:269-392):
// the sources (level 0) are cut into chunks of kChunkRoots consecutive
// sources; a chunk's upstream forest occupies ONE contiguous position range
// per level (children of consecutive parents are consecutive), so its
// per-level ranges follow from fc[] alone and chunks are fully independent.
// Each CTA takes whole chunks: the forest is staged in shared memory,
// accumulated deepest-level-first and eroded downstream->upstream with CTA
// barriers only -- no grid barrier, and every cell's h is read and written
// once, with the spatial locality of the source order.  Chunks too large for
// shared memory run the same sweeps on position-major global scratch, and
// plans deeper than kChunkMaxLevels use grid-wide level sweeps instead.
// All three schedules evaluate the identical per-cell arithmetic in a
// dependency-respecting order, so h is bit-identical among them.

constexpr int kChunkRoots = 128;
constexpr int kChunkCap = 2048;
constexpr int kChunkMaxLevels = 32;
constexpr int kCBS = kChunkMaxLevels + 1;  // chunk-boundary entries per chunk

struct ExpandSmem {
  uint32_t scan[kNW + 1];
  uint32_t bcast;
  uint32_t ord[kExTile];
};

struct ChunkSmem {
  double h[kChunkCap];
  double A[kChunkCap];
  uint32_t c[kChunkCap];
  uint16_t cs[kChunkCap];
  uint16_t par[kChunkCap];
  uint8_t cn[kChunkCap];
  uint32_t lo[kCBS + 1];
  uint32_t base[kCBS + 1];
  uint32_t nl, total;
};

struct FlowSmem {
  union {
    ExpandSmem ex;
    ChunkSmem ch;
  };
  unsigned long long red[kNW];
  uint32_t red32[kNW];
};
constexpr size_t kFlowSmemBytes = sizeof(FlowSmem);

// Level 0 (traversal.cpp:27-29): every cell with rec == kNoFlow, ascending.
__device__ __forceinline__ void tile_level0(const StepArgs& a, ExpandSmem& sm, uint32_t t,
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
// exclusive scan of popcount(dmask) over the frontier gives the first-child
// position fc[pos].
__device__ __forceinline__ void tile_expand(const StepArgs& a, ExpandSmem& sm, uint32_t t,
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
  const long long W = a.W;
#pragma unroll
  for (int j = 0; j < kExIPT; ++j) {
    const uint32_t pos = tb + threadIdx.x * kExIPT + j;
    if (pos < hi) {
      a.fc[pos] = out;
      uint32_t mm = m[j];
      while (mm) {
        const int k = __ffs(mm) - 1;
        mm &= mm - 1;
        a.order[out++] = (uint32_t)((long long)c[j] + dir_ox(k) + dir_oy(k) * W);
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

__device__ __forceinline__ bool is_interior(const StepArgs& a, uint32_t c) {
  const uint32_t y = c / a.W, x = c - y * a.W, yl = y % a.H;
  return x > 0 && x < a.W - 1 && yl > 0 && yl < a.H - 1;
}

// erode_one_cell (erosion.cpp:36-50) for cell c with receiver rc: uplifted
// start h0, already-updated receiver elevation hn, drainage area A.
template <int NK>
__device__ __forceinline__ double erode_cell(const StepArgs& a, uint32_t c, uint32_t rc, double h0,
                                             double hn, double A, unsigned long long& iters,
                                             uint32_t& misses, bool& ok) {
  const uint32_t mem = a.M > 1 ? c / a.MN : 0u;
  // F = K*dt*pow(A,m)/pow(dist,n) (erosion.cpp:38-39): (K*dt) first; pow(A,m)
  // from the host-libm table when A is an exact multiple of the cell area.
  double powA;
  const double q = a.w0_is_one ? A : __ddiv_rn(A, a.w0);
  if (a.lut_exact && q < (double)a.lut_entries && q == floor(q)) {
    powA = __ldg(a.lut + (size_t)mem * a.lut_entries + (uint32_t)q);
  } else {
    powA = pow(A, __ldg(a.mexp + mem));
    ++misses;
  }
  // pow(dist(c, rec[c]), n) by offset class (grid_graph.hpp:53-57)
  const int off = (int)(c - rc);
  const double pd = (off == 1 || off == -1) ? a.powdist_h
                    : (off == (int)a.W || off == -(int)a.W) ? a.powdist_v : a.powdist_d;
  const double F = __ddiv_rn(__dmul_rn(__ldg(a.kdt + mem), powA), pd);
  int it;
  double hnew;
  if (NK == 1)
    hnew = newton_n1(h0, hn, F, a.eps, a.maxit, it, ok);
  else
    hnew = newton_gen<NK>(h0, hn, F, a.n_exp, a.eps, a.maxit, it, ok);
  if (ok) {
    iters += (unsigned long long)it;
  } else {
    atomicMin(&a.ctl->err_cell, c);
    atomicMax(&a.ctl->err_flag, (uint32_t)LEMGPU_ECONVERGENCE);
  }
  return hnew;
}

// One chunk in shared memory.  Local index i enumerates the chunk's forest
// level by level (base[l] .. base[l+1]); parents/children are local indices.
template <int NK>
__device__ __forceinline__ void chunk_smem(const StepArgs& a, ChunkSmem& s, unsigned long long& iters,
                                           uint32_t& misses) {
  const uint32_t T = s.total, nl = s.nl, tid = threadIdx.x;
  // load, stage 1: cell and child range of every position (independent
  // loads, 4 in flight per thread)
  {
    uint32_t l = 0;
    for (uint32_t i0 = tid; i0 < T; i0 += 4 * kTPB) {
      uint32_t pos[4], lv[4], c[4], f0[4], f1[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * kTPB;
        if (i < T) {
          while (s.base[l + 1] <= i) ++l;
          lv[u] = l;
          pos[u] = s.lo[l] + (i - s.base[l]);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (i0 + u * kTPB < T) {
          c[u] = a.order[pos[u]];
          f0[u] = a.fc[pos[u]];
          f1[u] = a.fc[pos[u] + 1];
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t i = i0 + u * kTPB;
        if (i < T) {
          s.c[i] = c[u];
          s.cn[i] = (uint8_t)(f1[u] - f0[u]);
          s.cs[i] = (uint16_t)(f1[u] > f0[u] ? s.base[lv[u] + 1] + (f0[u] - s.lo[lv[u] + 1]) : 0u);
        }
      }
    }
  }
  __syncthreads();
  // load, stage 2: uplifted h (erosion.cpp:52-57: interior cells only)
  for (uint32_t i0 = tid; i0 < T; i0 += 4 * kTPB) {
    double hv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * kTPB;
      if (i < T) hv[u] = a.h[s.c[i]];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t i = i0 + u * kTPB;
      if (i < T) s.h[i] = (i >= s.base[1] || is_interior(a, s.c[i])) ? __dadd_rn(hv[u], a.du) : hv[u];
    }
  }
  for (uint32_t i = tid; i < T; i += kTPB) {
    const uint32_t n = s.cn[i], c0 = s.cs[i];
    for (uint32_t j = 0; j < n; ++j) s.par[c0 + j] = (uint16_t)i;
  }
  // accumulation, deepest level first (accumulation.hpp:21-28: fixed slot order)
  for (int l = (int)nl - 1; l >= 0; --l) {
    for (uint32_t i = s.base[l] + tid; i < s.base[l + 1]; i += kTPB) {
      double acc = a.w0;
      const uint32_t n = s.cn[i], c0 = s.cs[i];
      for (uint32_t j = 0; j < n; ++j) acc = __dadd_rn(acc, s.A[c0 + j]);
      s.A[i] = acc;
    }
    __syncthreads();
  }
  // drainage area out, position-major (AccumField::values, via the order)
  {
    uint32_t l = 0;
    for (uint32_t i = tid; i < T; i += kTPB) {
      while (s.base[l + 1] <= i) ++l;
      a.Aq[s.lo[l] + (i - s.base[l])] = s.A[i];
    }
  }
  // erosion, downstream -> upstream (erosion.cpp:66-81); level 0 never eroded
  for (uint32_t l = 1; l < nl; ++l) {
    for (uint32_t i = s.base[l] + tid; i < s.base[l + 1]; i += kTPB) {
      const uint32_t p = s.par[i];
      bool ok;
      const double hnew = erode_cell<NK>(a, s.c[i], s.c[p], s.h[i], s.h[p], s.A[i], iters, misses, ok);
      if (ok) s.h[i] = hnew;
    }
    __syncthreads();
  }
  for (uint32_t i = tid; i < T; i += kTPB) {
    const uint32_t c = s.c[i];
    if (i >= s.base[1] || is_interior(a, c)) a.h[c] = s.h[i];
  }
  __syncthreads();
}

// The same sweeps on position-major global scratch (hq, Aq, ppos), for a
// chunk that does not fit in shared memory (GRID = false: CTA barriers) or
// for the whole plan at once when it is deeper than kChunkMaxLevels (GRID =
// true: per-level ranges are the global levels, grid barriers).
template <int NK, bool GRID>
__device__ void sweep_global(const StepArgs& a, cg::grid_group& grid, const uint32_t* lo,
                             const uint32_t* hi, uint32_t nl, unsigned long long& iters,
                             uint32_t& misses) {
  const uint32_t start = GRID ? blockIdx.x * kTPB + threadIdx.x : threadIdx.x;
  const uint32_t stride = GRID ? gridDim.x * kTPB : kTPB;
  auto sync = [&]() {
    if (GRID)
      grid.sync();
    else
      __syncthreads();
  };
  for (uint32_t l = 0; l < nl; ++l) {
    for (uint32_t pos = lo[l] + start; pos < hi[l]; pos += stride) {
      const uint32_t c = a.order[pos];
      double hv = a.h[c];
      if (l > 0 || is_interior(a, c)) hv = __dadd_rn(hv, a.du);
      a.hq[pos] = hv;
      if (l + 1 < nl)
        for (uint32_t j = a.fc[pos], j1 = a.fc[pos + 1]; j < j1; ++j) a.ppos[j] = pos;
    }
  }
  sync();
  for (int l = (int)nl - 1; l >= 0; --l) {
    for (uint32_t pos = lo[l] + start; pos < hi[l]; pos += stride) {
      double acc = a.w0;
      if ((uint32_t)l + 1 < nl)
        for (uint32_t j = a.fc[pos], j1 = a.fc[pos + 1]; j < j1; ++j) acc = __dadd_rn(acc, a.Aq[j]);
      a.Aq[pos] = acc;
    }
    sync();
  }
  for (uint32_t l = 1; l < nl; ++l) {
    for (uint32_t pos = lo[l] + start; pos < hi[l]; pos += stride) {
      const uint32_t p = a.ppos[pos];
      bool ok;
      const double hnew =
          erode_cell<NK>(a, a.order[pos], a.order[p], a.hq[pos], a.hq[p], a.Aq[pos], iters, misses, ok);
      if (ok) a.hq[pos] = hnew;
    }
    sync();
    if (GRID && ld_volatile_u32(&a.ctl->err_flag)) break;
  }
  for (uint32_t l = 0; l < nl; ++l) {
    for (uint32_t pos = lo[l] + start; pos < hi[l]; pos += stride) {
      const uint32_t c = a.order[pos];
      if (l > 0 || is_interior(a, c)) a.h[c] = a.hq[pos];
    }
  }
  sync();
}

template <int NK>
__global__ void __launch_bounds__(kTPB, 3) k_flow(StepArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) unsigned char smem_raw[];
  FlowSmem& sm = *reinterpret_cast<FlowSmem*>(smem_raw);
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
    // look-back epoch space nearly exhausted: clear all status words, restart
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
    ctl->ntl = 0;
    ctl->tl[ctl->ntl++] = t_begin;
  }

  // ---- Phase A: breadth-first level order
  const uint32_t nt0 = (a.N + kL0Tile - 1) / kL0Tile;
  for (uint32_t t = b; t < nt0; t += G) tile_level0(a, sm.ex, t, nt0, E0);
  grid.sync();
  LG_TL(lead, ctl);

  uint32_t lo = 0, hi = ld_volatile_u32(&ctl->level_total[0]);
  const uint32_t n0 = hi;
  const uint32_t nch = (n0 + kChunkRoots - 1) / kChunkRoots;
  for (uint32_t k = b * kTPB + tid; k <= nch; k += G * kTPB) a.cbound[(size_t)k * kCBS] = min(k * kChunkRoots, n0);
  uint32_t l = 0;
  while (true) {
    const uint32_t F = hi - lo;
    const uint32_t nt = (F + kExTile - 1) / kExTile;
    for (uint32_t t = b; t < nt; t += G) tile_expand(a, sm.ex, t, nt, lo, hi, E0 + 1 + l, (l + 1) & 1);
    grid.sync();
    LG_TL(lead, ctl);
    const uint32_t total = ld_volatile_u32(&ctl->level_total[(l + 1) & 1]);
    // chunk boundaries one level down: P_{l+1}(k) = fc[P_l(k)] (the end of a
    // level maps to the end of the next; fc there belongs to the next sweep)
    if (l + 1 <= (uint32_t)kChunkMaxLevels) {
      for (uint32_t k = b * kTPB + tid; k <= nch; k += G * kTPB) {
        const uint32_t p = a.cbound[(size_t)k * kCBS + l];
        a.cbound[(size_t)k * kCBS + l + 1] = p >= hi ? hi + total : a.fc[p];
      }
    }
    if (total == 0) break;
    if (lead) a.levels[l + 2] = hi + total;
    lo = hi;
    hi += total;
    ++l;
  }
  const uint32_t nlev = l + 1;
  grid.sync();
  LG_TL(lead, ctl);
  const unsigned long long t_order = globaltimer();
  unsigned long long iters = 0;
  uint32_t misses = 0;
  const bool failed = hi != a.N;  // cells unreachable from the sources: a cycle (traversal.cpp:46)
  if (failed) {
    if (lead) {
      ctl->err_flag = LEMGPU_ESTRUCTURE;
      ctl->err_cell = hi;  // cells placed
    }
  } else if (nlev <= (uint32_t)kChunkMaxLevels) {
    // ---- Phase B: independent source chunks, one CTA each
    ChunkSmem& s = sm.ch;
    for (uint32_t k = b; k < nch; k += G) {
      if (tid <= nlev) {
        const uint32_t x = a.cbound[(size_t)k * kCBS + tid];
        const uint32_t y = a.cbound[(size_t)(k + 1) * kCBS + tid];
        s.lo[tid] = x;
        s.base[tid] = y - x;  // level sizes, turned into a prefix below
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t acc = 0, d = 0;
        for (uint32_t q = 0; q < nlev; ++q) {
          const uint32_t n = s.base[q];
          s.base[q] = acc;
          acc += n;
          if (n) d = q + 1;
        }
        for (uint32_t q = nlev; q <= (uint32_t)kCBS; ++q) s.base[q] = acc;
        s.nl = d;
        s.total = acc;
      }
      __syncthreads();
      if (s.total <= (uint32_t)kChunkCap) {
        chunk_smem<NK>(a, s, iters, misses);
      } else {
        // copy the chunk's per-level ranges out of the union first
        uint32_t rlo[kCBS], rhi[kCBS];
        const uint32_t nl = s.nl;
        for (uint32_t q = 0; q < nl; ++q) {
          rlo[q] = s.lo[q];
          rhi[q] = s.lo[q] + (s.base[q + 1] - s.base[q]);
        }
        __syncthreads();
        sweep_global<NK, false>(a, grid, rlo, rhi, nl, iters, misses);
      }
    }
  } else {
    // ---- deep plan: grid-wide level sweeps
    sweep_global<NK, true>(a, grid, a.levels, a.levels + 1, nlev, iters, misses);
  }
  // deterministic integer reduction of the per-thread counters
  {
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
      unsigned long long sum = 0;
      uint32_t mm = 0;
      for (int w = 0; w < kNW; ++w) {
        sum += sm.red[w];
        mm += sm.red32[w];
      }
      if (sum) atomicAdd(reinterpret_cast<unsigned long long*>(&a.diag->newton_iters), sum);
      if (mm) atomicAdd(&a.diag->lut_misses, mm);
    }
  }
  grid.sync();
  LG_TL(lead, ctl);
  if (lead) {
    const unsigned long long t_end = globaltimer();
    const uint32_t st = ctl->err_flag;
    lemgpu_diag* d = a.diag;
    d->seconds[LEMGPU_PHASE_RECEIVERS] = (double)(ctl->t_k1_end - ctl->t_k1_begin) * 1e-9;
    d->seconds[LEMGPU_PHASE_DONORS] = 0.0;  // fused into k_recv_donor
    d->seconds[LEMGPU_PHASE_ORDER] = (double)(t_order - t_begin) * 1e-9;
    d->seconds[LEMGPU_PHASE_ACCUM] = 0.0;   // fused with uplift + erosion per source chunk
    d->seconds[LEMGPU_PHASE_UPLIFT] = 0.0;
    d->seconds[LEMGPU_PHASE_EROSION] = (double)(t_end - t_order) * 1e-9;
    d->nlevels = nlev;
    d->interior_noflow = a.levels[1] - a.perim;
    d->status = st;
    d->err_cell = st ? ctl->err_cell : LEMGPU_NOFLOW;
    d->reserved = nch;
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
