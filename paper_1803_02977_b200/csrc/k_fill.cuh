// k_fill.cuh -- Priority-Flood depression filling on the device.
//
//   priority_flood_fill  proj/src/depressions.cpp:26-68 (FillMode,
//                        include/lem/depressions.hpp:8-27)
//
// The reference floods inward from the perimeter with a min-heap of (spill
// elevation, cell).  Pops come out in non-decreasing elevation (a pushed cell
// is never below the spill that raised it), so the first neighbour to pop --
// and visit a cell c -- is the neighbour of lowest filled elevation m, and
//   exact:    f[c] = max(h[c], m)
//   epsilon:  f[c] = h[c] > m ? h[c] : RN(m + eps)
// with f = h on the perimeter.  (Equal elevations tie-break by index in the
// heap but give the same m.)  The reference's result is therefore a fixed
// point of f = G(h, min_neighbours f), and the greatest one: exact mode's
// minimax spill elevation (the fixpoint oracle of acceptance.cpp:243-245), and
// for eps > 0 the only one (every raised cell needs a strictly lower
// neighbour, so chains end at the perimeter).  It is reached by relaxation
// from f = +inf inside the raster: every update only lowers f and keeps it at
// or above the fixed point, so the order of the updates -- here tile-local
// Gauss-Seidel sweeps in shared memory, and tiles reading each other's
// borders while they change -- does not matter for the result, only for the
// number of passes.  A pass skips tiles whose 3x3 tile neighbourhood did not
// change in the previous pass.
#pragma once

#include "common.cuh"

namespace lemgpu {

constexpr int kFX = 64, kFY = 32;                // tile
constexpr int kFPitch = kFX + 2;                 // shared row: tile + 1-cell halo
constexpr int kFCells = kFX * kFY / kTPB;        // cells per thread
static_assert(kFX * kFY % kTPB == 0 && kTPB % kFX == 0, "fill tile geometry");

struct FillArgs {
  const double* h;       // the terrain
  double* f;             // the filled surface (in: +inf inside, h on the perimeter)
  uint32_t W, H, Htot;   // member width / height, stacked rows
  uint32_t ntx, nty;     // tiles
  int mode;              // 1 exact, 2 epsilon ascending
  double eps;
  const uint32_t* dirty_prev;  // tiles changed in the previous pass (nullptr: first pass, all)
  uint32_t* dirty_cur;
  uint32_t* any;               // set when any tile changed
};

__device__ __forceinline__ bool fill_perimeter(uint32_t x, uint32_t y, uint32_t W, uint32_t H) {
  const uint32_t yl = y % H;
  return x == 0 || x == W - 1 || yl == 0 || yl == H - 1;
}

__global__ void __launch_bounds__(kTPB) k_fill_init(const double* h, double* f, uint32_t W, uint32_t H, uint32_t Htot) {
  const size_t n = (size_t)W * Htot;
  for (size_t i = (size_t)blockIdx.x * kTPB + threadIdx.x; i < n; i += (size_t)gridDim.x * kTPB) {
    const uint32_t y = (uint32_t)(i / W), x = (uint32_t)(i - (size_t)y * W);
    f[i] = fill_perimeter(x, y, W, H) ? h[i] : __longlong_as_double(0x7FF0000000000000ll);
  }
}

__global__ void __launch_bounds__(kTPB) k_fill_pass(FillArgs fa) {
  __shared__ double fs[kFY + 2][kFPitch];
  const uint32_t tx = blockIdx.x % fa.ntx, ty = blockIdx.x / fa.ntx;
  if (fa.dirty_prev) {  // nothing around this tile changed last pass: nothing can change here
    bool d = false;
    for (int oy = -1; oy <= 1; ++oy)
      for (int ox = -1; ox <= 1; ++ox) {
        const int nx = (int)tx + ox, ny = (int)ty + oy;
        if (nx >= 0 && ny >= 0 && nx < (int)fa.ntx && ny < (int)fa.nty) d |= fa.dirty_prev[ny * fa.ntx + nx] != 0;
      }
    if (!d) return;
  }
  const int x0 = (int)(tx * kFX), y0 = (int)(ty * kFY);
  const double inf = __longlong_as_double(0x7FF0000000000000ll);
  // stage f of the tile and its halo (off-raster: +inf, never the minimum)
  for (int i = threadIdx.x; i < (kFY + 2) * kFPitch; i += kTPB) {
    const int ly = i / kFPitch, lx = i - ly * kFPitch;
    const int gx = x0 - 1 + lx, gy = y0 - 1 + ly;
    fs[ly][lx] = (gx >= 0 && gy >= 0 && gx < (int)fa.W && gy < (int)fa.Htot) ? fa.f[(size_t)gy * fa.W + gx] : inf;
  }
  // this thread's cells: column lx, rows ly0 + k * (kTPB / kFX)
  const int lx = threadIdx.x % kFX, ly0 = threadIdx.x / kFX;
  double hv[kFCells];
  uint32_t upd = 0;  // bit k: cell k may be raised (interior, inside the raster)
#pragma unroll
  for (int k = 0; k < kFCells; ++k) {
    const int ly = ly0 + k * (kTPB / kFX);
    const uint32_t gx = (uint32_t)(x0 + lx), gy = (uint32_t)(y0 + ly);
    hv[k] = 0.0;
    if (gx < fa.W && gy < fa.Htot && !fill_perimeter(gx, gy, fa.W, fa.H)) {
      hv[k] = fa.h[(size_t)gy * fa.W + gx];
      upd |= 1u << k;
    }
  }
  __syncthreads();
  // Gauss-Seidel sweeps until the tile is stable
  bool changed_any = false;
  for (;;) {
    bool ch = false;
#pragma unroll
    for (int k = 0; k < kFCells; ++k) {
      if (!((upd >> k) & 1u)) continue;
      const int ly = ly0 + k * (kTPB / kFX) + 1, cx = lx + 1;
      double m = fmin(fmin(fmin(fs[ly - 1][cx - 1], fs[ly - 1][cx]), fmin(fs[ly - 1][cx + 1], fs[ly][cx - 1])),
                      fmin(fmin(fs[ly][cx + 1], fs[ly + 1][cx - 1]), fmin(fs[ly + 1][cx], fs[ly + 1][cx + 1])));
      const double nv = fa.mode == 1 ? fmax(hv[k], m) : (hv[k] > m ? hv[k] : __dadd_rn(m, fa.eps));
      if (nv < fs[ly][cx]) {
        fs[ly][cx] = nv;
        ch = true;
      }
    }
    if (!__syncthreads_or(ch)) break;
    changed_any = true;
  }
  if (changed_any) {
#pragma unroll
    for (int k = 0; k < kFCells; ++k) {
      if (!((upd >> k) & 1u)) continue;
      const int ly = ly0 + k * (kTPB / kFX);
      fa.f[(size_t)(y0 + ly) * fa.W + (x0 + lx)] = fs[ly + 1][lx + 1];
    }
    if (threadIdx.x == 0) {
      fa.dirty_cur[blockIdx.x] = 1u;
      *fa.any = 1u;
    }
  }
}

}  // namespace lemgpu
