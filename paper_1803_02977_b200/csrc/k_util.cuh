// k_util.cuh -- non-hot-path kernels: terrain generation, input check,
// graph/accumulation export for parity, per-member statistics.
#pragma once

#include "common.cuh"

namespace lemgpu {


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

// Donor masks of every cell from the receiver codes (the tile path does not
// materialise them in the step; the parity export and the global level path
// read them).
__global__ void k_fill_dmask(StepArgs a) {
  StepArgs b = a;
  b.dmask_valid = 0;
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x)
    a.dmask[c] = (uint8_t)donor_mask_at(b, c);
}

// FlowGraph export in the reference layout (flow_graph.hpp:19-38).
__global__ void k_export_graph(StepArgs a, uint32_t* rec, uint8_t* dnum, uint32_t* donor) {
  for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < a.N; c += gridDim.x * blockDim.x) {
    const uint8_t code = a.rcode[c];
    if (rec) rec[c] = code == kNoFlowCode ? LEMGPU_NOFLOW : (uint32_t)((long long)c + dir_ox(code) + (long long)dir_oy(code) * a.W);
    const uint32_t m = a.dmask[c];
    if (dnum) dnum[c] = (uint8_t)__popc(m);
    if (donor) {
      uint32_t* slot = donor + (size_t)c * a.conn;
      int j = 0;
      for (int k = 0; k < 8; ++k)
        if ((m >> k) & 1u) slot[j++] = (uint32_t)((long long)c + dir_ox(k) + (long long)dir_oy(k) * a.W);
      for (; j < a.conn; ++j) slot[j] = LEMGPU_NOFLOW;
    }
  }
}

// One level of the export accumulation (accumulate_into, accumulation.cpp:
// 7-17): A = w + the children's A in slot order; children of the last entry
// of a level end where the next level's children begin (fc is monotone).
__global__ void k_acc_level(StepArgs a, uint32_t L) {
  const uint32_t s = a.levels[L], e = a.levels[L + 1];
  for (uint32_t pos = s + blockIdx.x * blockDim.x + threadIdx.x; pos < e; pos += gridDim.x * blockDim.x) {
    double acc = a.w0;
    for (uint32_t j = a.fc[pos], j1 = a.fc[pos + 1]; j < j1; ++j) acc = __dadd_rn(acc, a.Aq[j]);
    a.Aq[pos] = acc;
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

// Ensemble statistics of the elevation a step starts from (the
// state the previous step left): a bandwidth-bound pass (8 B/cell) over fixed
// chunks of every member -- grid (st_chunks, M) -- that runs beside the
// step's issue- and latency-bound kernels (it reads the input buffer, which
// the step never writes), then a fold per member.  Fixed summation order:
// deterministic.  Fusing the
// reduction into k_recv or k_tiles was measured (64 x 2000^2: +0.85 ms/step,
// +15 %) -- those kernels are instruction-bound, the reduction's ~0.5
// instructions per cell cost more there than 8 B/cell of HBM traffic here.
__global__ void __launch_bounds__(kTPB) k_stats_pass(StepArgs a) {
  if (ld_volatile_u32(&a.ctl->err_flag)) return;
  const uint32_t m = blockIdx.y, ch = blockIdx.x, C = gridDim.x;
  const uint32_t per = ((a.MN + C - 1) / C + 1u) & ~1u;  // even: 16-byte aligned double2 loads when MN is even
  const uint32_t s0 = min(a.MN, ch * per), s1 = min(a.MN, s0 + per);
  const double* hm = a.h + (size_t)m * a.MN;
  double su = 0.0, mx = -INFINITY, mn = INFINITY;
  if ((a.MN & 1u) == 0) {
    const double2* v2 = reinterpret_cast<const double2*>(hm + s0);
    for (uint32_t i = threadIdx.x; i < (s1 - s0) / 2; i += kTPB) {
      const double2 v = __ldcs(v2 + i);
      su = __dadd_rn(__dadd_rn(su, v.x), v.y);
      mx = fmax(mx, fmax(v.x, v.y));
      mn = fmin(mn, fmin(v.x, v.y));
    }
  } else {
    for (uint32_t i = s0 + threadIdx.x; i < s1; i += kTPB) {
      const double v = hm[i];
      su = __dadd_rn(su, v);
      mx = fmax(mx, v);
      mn = fmin(mn, v);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    su = __dadd_rn(su, __shfl_xor_sync(0xffffffffu, su, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  __shared__ double sw[kNW][3];
  if ((threadIdx.x & 31) == 0) {
    sw[threadIdx.x >> 5][0] = su;
    sw[threadIdx.x >> 5][1] = mx;
    sw[threadIdx.x >> 5][2] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = sw[0][0], x = sw[0][1], n = sw[0][2];
    for (int w = 1; w < kNW; ++w) {
      s = __dadd_rn(s, sw[w][0]);
      x = fmax(x, sw[w][1]);
      n = fmin(n, sw[w][2]);
    }
    double* o = a.st_part + ((size_t)m * C + ch) * 3;
    o[0] = s;
    o[1] = x;
    o[2] = n;
  }
}

__global__ void __launch_bounds__(32) k_stats_fold(StepArgs a) {
  if (ld_volatile_u32(&a.ctl->err_flag)) return;
  const uint32_t m = blockIdx.x * 32 + threadIdx.x;
  if (m >= a.M) return;
  const double* p = a.st_part + (size_t)m * a.st_chunks * 3;
  double s = p[0], x = p[1], n = p[2];
  for (uint32_t c = 1; c < a.st_chunks; ++c) {
    s = __dadd_rn(s, p[3 * c]);
    x = fmax(x, p[3 * c + 1]);
    n = fmin(n, p[3 * c + 2]);
  }
  double* o = a.st_table + (size_t)(a.st_member0 + m) * 4;
  o[0] = __ddiv_rn(s, (double)a.MN);
  o[1] = x;
  o[2] = n;
  o[3] = s;
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
