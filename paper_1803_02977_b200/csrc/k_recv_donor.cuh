// k_recv_donor.cuh -- the receiver passes: k_recv (tile path: receiver codes +
// their bit planes) and k_recv_donor (global path / export: receiver codes +
// donor masks, one stencil pass).
//
//   steepest_receiver  proj/include/lem/flow_graph.hpp:44-59
//   donors_of          proj/include/lem/flow_graph.hpp:64-72
//
// k_recv_donor: one CTA owns a kBY x kBX tile.  h is staged in shared memory with a 2-cell
// halo (one coalesced HBM read of h), receiver codes are computed for the
// tile plus a 1-cell ring, and the donor bitmask of every tile cell is then
// a pull over the neighbours' codes (no atomics).  Outputs: rcode (the D8
// direction 0..7 of the receiver, 8 = kNoFlow) and dmask (bit k set when the
// neighbour in direction k drains into the cell), one byte each.
#pragma once

#include "common.cuh"

namespace lemgpu {

// The reference loop itself, with its exact skips: ec - en <= 0 never beats
// s_max >= 0 and x / 1.0 == x.  Used for general spacing / D4 and as the exact
// slow path of the D8 fast path.
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

__host__ __device__ __forceinline__ double dmax2(double x, double y) { return y > x ? y : x; }

// D8, unit cardinal spacing (the reference default): division-free argmax.
// t_k = d_k for cardinals (exact: x / 1.0 == x) and t_k = RN(d_k * RN(1/c))
// for diagonals, within 2^-51 relative of the true slope RN(d_k / c).  If a
// single direction lies within 2^-48 of max t it is the unique argmax of the
// true slopes; several cardinal candidates are exact and the first maximum
// wins; anything else (near ties involving a diagonal, subnormal drops) takes
// the reference loop.  Verified against the loop on 2M adversarial vectors
// (tests/native/test_receiver_code.cu).
template <int CONN>
__host__ __device__ __forceinline__ uint8_t receiver_code(const double (&d)[8], const StepArgs& a) {
  if (CONN == 8 && a.unit_card) {
    double t[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool diag = (k == 0 || k == 2 || k == 5 || k == 7);
      t[k] = diag ? LG_MUL(d[k], a.rinv_diag) : d[k];
    }
    const double tmax = dmax2(dmax2(dmax2(t[0], t[1]), dmax2(t[2], t[3])),
                              dmax2(dmax2(t[4], t[5]), dmax2(t[6], t[7])));
    // t_k > 0 <=> d_k > 0 (RN(x * 0.707..) of a positive x never rounds to 0),
    // so tmax <= 0 means no downhill neighbour; tiny positive maxima take the
    // reference loop
    if (!(tmax > 0x1p-1000)) return tmax > 0.0 ? receiver_code_ref<CONN>(d, a) : kNoFlowCode;
    const double thr = LG_MUL(tmax, 1.0 - 0x1p-48);
    uint32_t cand = 0;
#pragma unroll
    for (int k = 0; k < 8; ++k) cand |= (t[k] >= thr ? 1u : 0u) << k;
    if ((cand & (cand - 1)) == 0) {  // a single candidate
#ifdef __CUDA_ARCH__
      return (uint8_t)(__ffs(cand) - 1);
#else
      return (uint8_t)__builtin_ctz(cand);
#endif
    }
    if ((cand & 0xA5u) == 0) {  // only cardinals (exact values): first maximum
      uint32_t eq = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) eq |= ((cand >> k) & 1u) && t[k] == tmax ? (1u << k) : 0u;
#ifdef __CUDA_ARCH__
      return (uint8_t)(__ffs(eq) - 1);
#else
      return (uint8_t)__builtin_ctz(eq);
#endif
    }
    return receiver_code_ref<CONN>(d, a);
  }
  return receiver_code_ref<CONN>(d, a);
}

// D8, unit cardinal spacing: receiver code without divisions.  t_k = d_k
// (cardinal, exact) or RN(d_k * RN(1/sqrt2)) (diagonal, within 2^-51 relative
// of the reference slope RN(d_k / sqrt2)).  The high words of positive
// doubles order them; when exactly one t_k has a high word within 1 of the
// largest, every other t_j is below it by more than 2^-22 relative, so it is
// the unique strict maximum of the reference slopes as well.  Ties, near
// ties, subnormal or non-finite maxima take the reference loop
// (tests/native/test_receiver_code.cu checks this against the loop).
template <int CONN, bool UNIT = false>  // UNIT: the caller knows a.unit_card
__host__ __device__ __forceinline__ uint8_t receiver_code_hi(const double (&d)[8], const StepArgs& a) {
  if (CONN == 8 && (UNIT || a.unit_card)) {
    int hi[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const bool diag = (k == 0 || k == 2 || k == 5 || k == 7);
      hi[k] = hi_word(diag ? LG_MUL(d[k], a.rinv_diag) : d[k]);
    }
    auto mx2 = [](int u, int v) { return u > v ? u : v; };
    const int mx = mx2(mx2(mx2(hi[0], hi[1]), mx2(hi[2], hi[3])), mx2(mx2(hi[4], hi[5]), mx2(hi[6], hi[7])));
    // one unsigned range test for the common case, a normal finite positive maximum
    if ((uint32_t)(mx - 0x00100000) >= 0x7FE00000u) {
      if (mx < 0) return kNoFlowCode;  // every drop negative or -0: no downhill neighbour
      if (mx < 0x00100000) {           // no normal positive slope: +0 drops (flats) or subnormal ones
        bool pos = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) pos |= d[k] > 0.0;
        return pos ? receiver_code_ref<CONN>(d, a) : kNoFlowCode;
      }
      return receiver_code_ref<CONN>(d, a);  // inf / NaN
    }
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

// ---- TMA (cp.async.bulk.tensor) staging of the h tile, mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// exact per-byte equality mask: 0x01 in every byte of x that is zero
__device__ __forceinline__ uint32_t zero_bytes(uint32_t x) {
  const uint32_t t = ((x & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | x;
  return (~t & 0x80808080u) >> 7;
}

#ifndef LEMGPU_RECV_MINB
#define LEMGPU_RECV_MINB 5  // measured: 5 CTAs/SM (48 regs) beats 4 (64 regs)
#endif
// The global level path's receiver pass (LEMGPU_PATH=global and the parity
// export): receiver codes AND the donor masks of the tile, which needs the
// receiver codes of the ring around it.  (The tile path's pass is k_recv below.)
template <int CONN>
__global__ void __launch_bounds__(kTPB, LEMGPU_RECV_MINB) k_recv_donor(StepArgs a, const __grid_constant__ CUtensorMap hmap) {
  __shared__ __align__(128) double sh[kBY + 4][kBX + 4];
  __shared__ __align__(4) uint8_t rc[kBY + 2][kBX + 4];
  __shared__ uint8_t rowint[kBY + 2];
  __shared__ __align__(8) uint64_t bar;
  __shared__ PhClk s_pc;
  if (ld_volatile_u32(&a.ctl->err_flag)) return;
  phclk_begin(s_pc);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t x0 = blockIdx.x * kBX, y0 = blockIdx.y * kBY;
  const uint32_t W = a.W, Ht = a.Htot;
  if (tid == 0) {
    atomicMin(&a.ctl->t_k1_begin, globaltimer());
    if (a.use_tma) {
      // one TMA box = the whole halo tile; out-of-range cells arrive as 0
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (uint32_t)sizeof(sh));
      tma_load_2d(&sh[0][0], &hmap, (int)x0 - 2, (int)y0 - 2, &bar);
    }
  }

  // ---- stage h: rows y0-2 .. y0+kBY+1, columns x0-2 .. x0+kBX+1
  if (!a.use_tma) for (int r = warp; r < kBY + 4; r += kNW) {
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
  if (tid < kBY + 2) {  // rc row r <-> gy = y0 - 1 + r: does it hold interior cells?
    const int gy = (int)y0 - 1 + tid;
    uint8_t ok = 0;
    if (gy >= 0 && (uint32_t)gy < Ht) {
      const uint32_t yl = (uint32_t)gy % a.H;
      ok = yl > 0 && yl < a.H - 1;
    }
    rowint[tid] = ok;
  }
  __syncthreads();
  if (a.use_tma) mbar_wait(&bar, 0);

  // ---- receiver codes for rc rows 0..kBY+1 (gy = y0-1+r), rc columns
  // c = 0..kBX+1 (gx = x0-1+c).  Columns 1..kBX: one thread per column and
  // half of the rows, sliding a 3x3 register window down the column (three
  // shared loads per cell); the two ring columns are done separately.
  {
    const int c = 1 + (tid & (kBX - 1));
    const int ra = 0, rz = kBY + 2;  // receiver-code rows [ra, rz): the tile and its ring
    const int rbeg = (tid < kBX) ? ra : (ra + rz) / 2;
    const int rend = (tid < kBX) ? (ra + rz) / 2 : rz;
    const int gx = (int)x0 - 1 + c;
    const bool colint = gx > 0 && gx < (int)W - 1;
    // window rows u = sh row r, m = r+1, v = r+2 (sh columns c..c+2),
    // unrolled by three rows so the window never moves registers
    auto emit = [&](int r, const double (&u)[3], const double (&m)[3], const double (&v)[3]) {
      uint8_t code = kNoFlowCode;
      if (colint && rowint[r]) {
        const double ec = m[1];
        double d[8];
        d[0] = LG_SUB(ec, u[0]);
        d[1] = LG_SUB(ec, u[1]);
        d[2] = LG_SUB(ec, u[2]);
        d[3] = LG_SUB(ec, m[0]);
        d[4] = LG_SUB(ec, m[2]);
        d[5] = LG_SUB(ec, v[0]);
        d[6] = LG_SUB(ec, v[1]);
        d[7] = LG_SUB(ec, v[2]);
        if (CONN == 4) d[0] = d[2] = d[5] = d[7] = 0.0;
        code = receiver_code_hi<CONN>(d, a);
      }
      rc[r][c] = code;
    };
    auto load = [&](double (&w)[3], int row) {
#pragma unroll
      for (int q = 0; q < 3; ++q) w[q] = sh[row][c + q];
    };
    double r0[3], r1[3], r2[3];
    load(r0, rbeg);
    load(r1, rbeg + 1);
    int r = rbeg;
    for (; r + 3 <= rend; r += 3) {
      load(r2, r + 2);
      emit(r, r0, r1, r2);
      load(r0, r + 3);
      emit(r + 1, r1, r2, r0);
      load(r1, r + 4);
      emit(r + 2, r2, r0, r1);
    }
    if (r < rend) {
      load(r2, r + 2);
      emit(r, r0, r1, r2);
      if (r + 1 < rend) {
        load(r0, r + 3);
        emit(r + 1, r1, r2, r0);
      }
    }
  }
  if (tid < 2 * (kBY + 2)) {  // ring columns c = 0 and c = kBX+1
    const int r = tid >> 1, c = (tid & 1) ? kBX + 1 : 0;
    const int gx = (int)x0 - 1 + c;
    uint8_t code = kNoFlowCode;
    if (rowint[r] && gx > 0 && gx < (int)W - 1) {
      const double ec = sh[r + 1][c + 1];
      double d[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) d[k] = dir_in(CONN, k) ? LG_SUB(ec, sh[r + 1 + dir_oy(k)][c + 1 + dir_ox(k)]) : 0.0;
      code = receiver_code_hi<CONN>(d, a);
    }
    rc[r][c] = code;
  }
  __syncthreads();

  // ---- donors_of: neighbour in direction k donates iff its code is 7-k.
  phclk_mark(s_pc, LEMGPU_PHASE_RECEIVERS);
  // Four cells per thread in SWAR form: for each direction, the four
  // neighbour codes are one byte window of a shared row.
  for (int r = warp; r < kBY; r += kNW) {
    const uint32_t gy = y0 + r;
    if (gy >= Ht) break;
    const int c4 = lane * 4;  // tile columns c4..c4+3 <-> rc columns c4+1..c4+4
    uint32_t lo[3], hi[3];
    lo[1] = *reinterpret_cast<const uint32_t*>(&rc[r + 1][c4]);
    hi[1] = *reinterpret_cast<const uint32_t*>(&rc[r + 1][c4 + 4]);
    uint32_t pm = 0;
    {  // materialised donor masks (the global level path reads them)
      lo[0] = *reinterpret_cast<const uint32_t*>(&rc[r][c4]);
      hi[0] = *reinterpret_cast<const uint32_t*>(&rc[r][c4 + 4]);
      lo[2] = *reinterpret_cast<const uint32_t*>(&rc[r + 2][c4]);
      hi[2] = *reinterpret_cast<const uint32_t*>(&rc[r + 2][c4 + 4]);
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (!dir_in(CONN, k)) continue;
        const int q = 1 + dir_oy(k);
        const uint32_t sel = dir_ox(k) < 0 ? 0x3210u : dir_ox(k) == 0 ? 0x4321u : 0x5432u;
        const uint32_t win = __byte_perm(lo[q], hi[q], sel);
        pm |= zero_bytes(win ^ (0x01010101u * (uint32_t)(7 - k))) << k;
      }
    }
    const uint32_t pc = __byte_perm(lo[1], hi[1], 0x4321u);
    const uint32_t gx = x0 + c4;
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
  phclk_end(s_pc, LEMGPU_PHASE_DONORS, a.ctl);
  if (threadIdx.x == 0) atomicMax(&a.ctl->t_k1_end, globaltimer());
}

// ballot of (w & mask) != 0 -- one predicate-setting LOP3 per vote
__device__ __forceinline__ uint32_t ballot_bits(uint32_t w, uint32_t mask) {
  uint32_t r;
  asm volatile(
      "{ .reg .pred p; .reg .b32 t; and.b32 t, %1, %2; setp.ne.u32 p, t, 0; vote.sync.ballot.b32 %0, p, 0xffffffff; }"
      : "=r"(r)
      : "r"(w), "r"(mask));
  return r;
}

// The tile path's receiver pass: receiver codes (rcode, one byte per cell) and
// their bit planes, nothing else.  Each thread owns one column of the
// kBY x kBX tile and half of its rows (16) and slides a 3x3 register window
// down it.  Pass 1 is branch-free: the division-free selection of
// receiver_code_hi's common case for all 16 cells, codes packed as nibbles in
// two registers, undecided cells (near ties, flats, non-finite drops) flagged.
// Pass 2 settles the flagged cells with the full selection (rare).  Pass 3
// stores: 32 contiguous code bytes per warp and row, and the bit planes as
// four ballots of that warp row.  UNIT: D8 with unit cardinal spacing;
// otherwise every cell takes the reference loop in pass 2.
template <int CONN, bool UNIT>
__global__ void __launch_bounds__(kTPB, LEMGPU_RECV_MINB)
    k_recv(const __grid_constant__ StepArgs a, const __grid_constant__ CUtensorMap hmap) {
  __shared__ __align__(128) double sh[kBY + 4][kBX + 4];
  __shared__ __align__(8) uint64_t bar;
  __shared__ PhClk s_pc;
  phclk_begin(s_pc);
  // an earlier step of the batch failed: nothing to do (checked once the TMA
  // box has landed -- a CTA must not exit with a bulk copy in flight)
  const uint32_t failed = ld_volatile_u32(&a.ctl->err_flag);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t x0 = blockIdx.x * kBX, y0 = (blockIdx.y + a.by0) * kBY;
  const uint32_t W = a.W, Ht = a.Htot;
  if (tid == 0) {
    atomicMin(&a.ctl->t_k1_begin, globaltimer());
    if (a.use_tma) {
      mbar_init(&bar, 1);
      mbar_expect_tx(&bar, (uint32_t)sizeof(sh));
      tma_load_2d(&sh[0][0], &hmap, (int)x0 - 2, (int)y0 - 2, &bar);
    }
  }
  if (!a.use_tma) for (int r = warp; r < kBY + 4; r += kNW) {
    const int gy = (int)y0 - 2 + r;
    const bool rowok = gy >= 0 && (uint32_t)gy < Ht;
    const double* row = a.h + (size_t)(rowok ? gy : 0) * W;
#pragma unroll
    for (int j = 0; j < kBX / 32; ++j) {
      const uint32_t gx = x0 + lane + 32 * j;
      sh[r][2 + lane + 32 * j] = (rowok && gx < W) ? __ldg(row + gx) : 0.0;
    }
    if (lane < 4) {
      const int cc = lane < 2 ? lane : kBX + lane;
      const int gx = (int)x0 - 2 + cc;
      sh[r][cc] = (rowok && gx >= 0 && (uint32_t)gx < W) ? __ldg(row + gx) : 0.0;
    }
  }
  static_assert(kBY == 32, "16 rows per thread, codes in two nibble words");
  const int cx = tid & (kBX - 1);  // window columns sh cx+1..cx+3, centre gx
  const uint32_t gx = x0 + cx;
  const int t0 = tid < kBX ? 0 : kBY / 2;  // this thread's rows: t0 .. t0+15
  // interior rows (members are stacked; their first and last rows are base
  // level): bit i <-> tile row t0 + i
  uint32_t rows;
  {
    const uint32_t gy = y0 + (uint32_t)t0 + (uint32_t)(lane & 15);
    bool ok = gy < Ht;
    if (ok) {
      const uint32_t yl = a.M > 1 ? gy % a.H : gy;  // one member: no division
      ok = yl > 0 && yl < a.H - 1;
    }
    rows = __ballot_sync(0xffffffffu, ok) & 0xFFFFu;
  }
  if (!(gx > 0 && gx < W - 1)) rows = 0;
  __syncthreads();
  if (a.use_tma) mbar_wait(&bar, 0);
  if (failed) return;

  // ---- pass 1
  const double* col = &sh[t0][cx + 1];  // sh row t0, window column 0
  constexpr int kRow = kBX + 4;
  uint32_t cw0 = 0u, cw1 = 0u;  // code of row i in nibble i&7 of cw0 (i < 8) / cw1
  uint32_t slow = 0;
  if (CONN == 8 && UNIT) {
    const double rinv = a.rinv_diag;
    double w[3][3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      w[0][q] = col[1 * kRow + q];
      w[1][q] = col[2 * kRow + q];
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      // window rows: north (i+1)%3, centre (i+2)%3 = the row loaded last, south i%3 (new)
      double (&s)[3] = w[(i + 2) % 3];
#pragma unroll
      for (int q = 0; q < 3; ++q) s[q] = col[(i + 3) * kRow + q];
      const double (&u)[3] = w[i % 3];
      const double (&m)[3] = w[(i + 1) % 3];
      const double ec = m[1];
      const int h0 = hi_word(LG_MUL(LG_SUB(ec, u[0]), rinv)), h1 = hi_word(LG_SUB(ec, u[1]));
      const int h2 = hi_word(LG_MUL(LG_SUB(ec, u[2]), rinv)), h3 = hi_word(LG_SUB(ec, m[0]));
      const int h4 = hi_word(LG_SUB(ec, m[2])), h5 = hi_word(LG_MUL(LG_SUB(ec, s[0]), rinv));
      const int h6 = hi_word(LG_SUB(ec, s[1])), h7 = hi_word(LG_MUL(LG_SUB(ec, s[2]), rinv));
      const int mx = max(max(max(h0, h1), max(h2, h3)), max(max(h4, h5), max(h6, h7)));
      const int thr = mx - 1;
      const uint32_t cand = (h0 >= thr ? 1u : 0u) | (h1 >= thr ? 2u : 0u) | (h2 >= thr ? 4u : 0u) |
                            (h3 >= thr ? 8u : 0u) | (h4 >= thr ? 16u : 0u) | (h5 >= thr ? 32u : 0u) |
                            (h6 >= thr ? 64u : 0u) | (h7 >= thr ? 128u : 0u);
      const bool interior = (rows >> i) & 1u;
      const bool easy = (uint32_t)(mx - 0x00100000) < 0x7FE00000u && (cand & (cand - 1u)) == 0;
      const uint32_t code = interior ? (uint32_t)(__ffs(cand) - 1) : kNoFlowCode;
      if (i < 8)
        cw0 |= (code & 15u) << (4 * (i & 7));
      else
        cw1 |= (code & 15u) << (4 * (i & 7));
      slow |= (interior && !easy ? 1u : 0u) << i;
    }
  } else {
    cw0 = cw1 = 0x11111111u * kNoFlowCode;  // non-interior cells
    slow = rows;
  }
  // ---- pass 2: cells pass 1 left undecided
  while (slow) {
    const int i = __ffs(slow) - 1;
    slow &= slow - 1;
    const double* cc = col + (i + 1) * kRow;  // north row of cell i
    const double ec = cc[kRow + 1];
    double d[8];
    d[0] = LG_SUB(ec, cc[0]);
    d[1] = LG_SUB(ec, cc[1]);
    d[2] = LG_SUB(ec, cc[2]);
    d[3] = LG_SUB(ec, cc[kRow]);
    d[4] = LG_SUB(ec, cc[kRow + 2]);
    d[5] = LG_SUB(ec, cc[2 * kRow]);
    d[6] = LG_SUB(ec, cc[2 * kRow + 1]);
    d[7] = LG_SUB(ec, cc[2 * kRow + 2]);
    if (CONN == 4) d[0] = d[2] = d[5] = d[7] = 0.0;
    const uint32_t code = UNIT ? receiver_code_hi<CONN, true>(d, a) : receiver_code_ref<CONN>(d, a);
    const int sh4 = 4 * (i & 7);
    if (i < 8)
      cw0 = (cw0 & ~(15u << sh4)) | (code << sh4);
    else
      cw1 = (cw1 & ~(15u << sh4)) | (code << sh4);
  }
  // ---- pass 3: stores (codes, and the bit planes the donors are derived from)
  phclk_mark(s_pc, LEMGPU_PHASE_RECEIVERS);
  const int nr = min(kBY / 2, max(0, (int)Ht - (int)(y0 + (uint32_t)t0)));  // rows inside the raster (warp-uniform)
  const uint32_t j = x0 / 32 + (uint32_t)(cx >> 5);  // plane word of this warp's columns
  const bool xok = gx < W, pok = lane < 4 && j < a.W32;
  if (!xok) cw0 = cw1 = 0xFFFFFFFFu;  // bit planes: columns beyond W read as code 15
  uint8_t* rp = a.rcode + (size_t)(y0 + (uint32_t)t0) * W + gx;
  uint32_t* pp = a.planes + ((size_t)(lane & 3) * Ht + y0 + (uint32_t)t0) * a.W32 + j;
  const size_t W32 = a.W32;
  const bool p1 = lane & 1, p2 = lane & 2;
  auto store_row = [&](int i) {
    const uint32_t w = i < 8 ? cw0 : cw1;
    const int sh4 = 4 * (i & 7);
    if (xok) *rp = (uint8_t)((w >> sh4) & 15u);
    const uint32_t b0 = ballot_bits(w, 1u << sh4), b1 = ballot_bits(w, 2u << sh4);
    const uint32_t b2 = ballot_bits(w, 4u << sh4), b3 = ballot_bits(w, 8u << sh4);
    if (pok) *pp = p2 ? (p1 ? b3 : b2) : (p1 ? b1 : b0);
    rp += W;
    pp += W32;
  };
  if (nr == kBY / 2) {
#pragma unroll
    for (int i = 0; i < 16; ++i) store_row(i);
  } else {
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (i < nr) store_row(i);
  }
  phclk_end(s_pc, LEMGPU_PHASE_DONORS, a.ctl);
  if (threadIdx.x == 0) atomicMax(&a.ctl->t_k1_end, globaltimer());  // (no barrier: thread 0's end ~ the CTA's)
}

}  // namespace lemgpu
