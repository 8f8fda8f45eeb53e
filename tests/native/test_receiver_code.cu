// Host-side exhaustive check of the division-skipping receiver selection
// (receiver_code<8> in lemgpu_kernels.cuh) against the reference's plain
// loop, steepest_receiver (proj/include/lem/flow_graph.hpp:44-59):
//     s = (ec - en) / dist; if (s > s_max) { s_max = s; n_max = n; }
// Random drops plus adversarial ties: diagonal quotients equal to cardinal
// drops, drops one ulp apart, diagonals that round to the same quotient.
// Built by tests/test_native.py with nvcc (host code, -ffp-contract=off).
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <random>

#include "../../paper_1803_02977_b200/csrc/k_tiles.cuh"

using namespace lemgpu;

static uint8_t naive(const double (&d)[8], const double (&dist)[8]) {
  double smax = 0.0;
  uint8_t code = kNoFlowCode;
  for (int k = 0; k < 8; ++k) {
    const double s = d[k] / dist[k];
    if (s > smax) {
      smax = s;
      code = (uint8_t)k;
    }
  }
  return code;
}

int main() {
  StepArgs a{};
  for (int k = 0; k < 8; ++k) {
    const double ox = dir_ox(k), oy = dir_oy(k);
    a.dist[k] = (oy == 0) ? std::fabs(ox) : (ox == 0) ? std::fabs(oy) : std::sqrt(ox * ox + oy * oy);
    if (a.dist[k] == 1.0) a.dist_one |= 1u << k;
  }
  a.unit_card = 1;
  a.rinv_diag = 1.0 / a.dist[0];
  const double c = a.dist[0];
  std::mt19937_64 rng(12345);
  std::uniform_real_distribution<double> U(-1.0, 1.0);
  long long n = 0, bad = 0;
  auto check = [&](const double (&d)[8]) {
    ++n;
    const uint8_t want = naive(d, a.dist), got = receiver_code<8>(d, a), got2 = receiver_code_hi<8>(d, a);
    if (want != got || want != got2) {
      if (bad < 10) {
        std::printf("MISMATCH want %d got %d / %d:", want, got, got2);
        for (int k = 0; k < 8; ++k) std::printf(" %.17g", d[k]);
        std::printf("\n");
      }
      ++bad;
    }
  };
  const int diag[4] = {0, 2, 5, 7}, card[4] = {1, 3, 4, 6};
  for (int it = 0; it < 2000000; ++it) {
    double d[8];
    const double scale = std::ldexp(1.0, (int)(rng() % 40) - 30);
    for (int k = 0; k < 8; ++k) d[k] = U(rng) * scale;
    const int mode = it % 8;
    if (mode == 1) {  // a cardinal equals the diagonal quotient exactly
      const int kd = diag[rng() % 4], kc = card[rng() % 4];
      d[kd] = std::fabs(d[kd]) + scale;
      d[kc] = d[kd] / c;
    } else if (mode == 2) {  // ... and one ulp either side
      const int kd = diag[rng() % 4], kc = card[rng() % 4];
      d[kd] = std::fabs(d[kd]) + scale;
      d[kc] = std::nextafter(d[kd] / c, (rng() & 1) ? 1e300 : -1e300);
    } else if (mode == 3) {  // two diagonals one ulp apart (may round to the same quotient)
      const int i = rng() % 4, j = (i + 1 + rng() % 3) % 4;
      d[diag[i]] = std::fabs(d[diag[i]]) + scale;
      d[diag[j]] = std::nextafter(d[diag[i]], (rng() & 1) ? 1e300 : -1e300);
      for (int k : card) d[k] = -std::fabs(d[k]);
    } else if (mode == 4) {  // equal cardinals
      const int i = rng() % 4, j = (i + 1 + rng() % 3) % 4;
      d[card[i]] = std::fabs(d[card[i]]);
      d[card[j]] = d[card[i]];
    } else if (mode == 5) {  // everything uphill or flat
      for (int k = 0; k < 8; ++k) d[k] = (rng() & 1) ? -std::fabs(d[k]) : 0.0;
    } else if (mode == 6) {  // many equal diagonal drops + matching cardinal
      const double x = std::fabs(d[0]) + scale;
      for (int k : diag) d[k] = (rng() & 1) ? x : std::nextafter(x, -1e300);
      d[card[rng() % 4]] = x / c;
    } else if (mode == 7) {  // subnormal corner, or +0 drops (flats left by the erosion floor)
      if (rng() & 1)
        for (int k = 0; k < 8; ++k) d[k] = U(rng) * 1e-310;
      else
        for (int k = 0; k < 8; ++k) d[k] = (rng() % 3) ? -std::fabs(d[k]) : 0.0;
    }
    check(d);
  }
  std::printf("receiver_code: %lld cases, %lld mismatches\n", n, bad);
  return bad ? 1 : 0;
}
