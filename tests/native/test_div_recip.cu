// Host check of div_rn_recip (k_physics.cuh): RN(a / b) from the host-rounded
// reciprocal y = RN(1 / b) with one Markstein correction step, against the
// IEEE division (x86 SSE2, correctly rounded) on random, table-shaped and
// adversarial operands.  b = 1 + F >= 1 as in the n = 1 Newton slope
// (erosion.cpp:26).  Built and run by tests/test_native.py.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>

#include "../../paper_1803_02977_b200/csrc/k_physics.cuh"

using namespace lemgpu;

static uint64_t bits(double x) {
  uint64_t b;
  std::memcpy(&b, &x, 8);
  return b;
}

int main(int argc, char** argv) {
  const long long N = argc > 1 ? std::atoll(argv[1]) : 200000000LL;
  std::mt19937_64 rng(2024);
  std::uniform_real_distribution<double> U(0.0, 1.0);
  long long n = 0, bad = 0;
  auto check = [&](double a, double b) {
    const double y = 1.0 / b;
    const double want = a / b, got = div_rn_recip(a, b, y);
    ++n;
    if (bits(want) != bits(got)) {
      if (bad < 10) std::printf("MISMATCH a=%.17g b=%.17g want=%.17g got=%.17g\n", a, b, want, got);
      ++bad;
    }
  };
  // b values: the F tables (K dt pow(A, m) / pow(dist, n)) of typical runs,
  // extreme mantissas, and random
  const double specials[] = {1.0, std::nextafter(1.0, 2.0), std::nextafter(2.0, 1.0), 1.5, 1.0 + 0x1p-30,
                             1.0 + 0x1p-52 * 3, 0x1p40 - 1, 3.0, std::nextafter(3.0, 0.0), 1e6 + 0.5};
  for (long long it = 0; it < N; ++it) {
    double b;
    const int mode = (int)(it % 8);
    if (mode < 3) {
      const double K = 1e-6 * (double)(1 + rng() % 8), m = 0.35 + 0.05 * (double)(rng() % 8);
      const double A = (double)(1 + rng() % 65536);
      const double dist = (rng() & 1) ? 1.0 : std::sqrt(2.0);
      b = 1.0 + (K * 1000.0 * std::pow(A, m)) / dist;
    } else if (mode == 3) {
      b = specials[rng() % (sizeof specials / sizeof specials[0])];
    } else if (mode == 4) {  // random mantissa, b in [1, 2)
      uint64_t mb = 0x3FF0000000000000ull | (rng() & 0xFFFFFFFFFFFFFull);
      std::memcpy(&b, &mb, 8);
    } else {
      b = 1.0 + std::ldexp(U(rng), (int)(rng() % 80) - 60);
    }
    double a;
    const int am = (int)((it / 8) % 4);
    if (am == 0) {  // random magnitude and sign over the fast range and beyond
      a = std::ldexp(U(rng) + 0.5, (int)(rng() % 1900) - 950) * ((rng() & 1) ? 1.0 : -1.0);
    } else if (am == 1) {  // near-midpoint quotients: a = RN(b * (q + ulp(q)/2)) and neighbours
      const double q = std::ldexp(U(rng) + 0.5, (int)(rng() % 60) - 30);
      const double mid = q + std::ldexp(std::nextafter(q, 1e300) - q, -1);
      a = b * mid;
      const int k = (int)(rng() % 5) - 2;
      for (int j = 0; j < std::abs(k); ++j) a = std::nextafter(a, k > 0 ? 1e300 : -1e300);
    } else if (am == 2) {  // erosion-shaped: F * (h0 - hn) with h ~ 240, drops 1e-8 .. 1
      const double F = b - 1.0;
      a = F * std::ldexp(U(rng) + 0.5, -(int)(rng() % 27));
    } else {  // exact multiples (quotient representable)
      const double q = std::ldexp((double)(rng() >> 30), -(int)(rng() % 40));
      a = b * q;
    }
    if (a == 0.0 || !std::isfinite(a)) continue;
    check(a, b);
  }
  std::printf("div_rn_recip: %lld cases, %lld mismatches\n", n, bad);
  return bad ? 1 : 0;
}
