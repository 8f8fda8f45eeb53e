// Bit-exactness of the glibc pow restatement (paper_1803_02977_b200/csrc/glibc_pow.cuh)
// against the host libm's pow, on the CPU.
//
//   test_glibc_pow <fma|sse2> [count] [seed]
//
// Compares glibc_pow<variant> with ::pow on `count` inputs from every regime
// the reference hits (pow(A, m) for drainage areas, pow(diff, n) for Newton
// differences, pow(dist, n)) plus random bit patterns, integer / half-integer
// exponents, negative bases, subnormals, zeros, infinities and NaNs.  Exit 0
// when every result is identical (NaNs compared by NaN-ness).  The sse2
// restatement is checked against the libm with GLIBC_TUNABLES masking FMA and
// AVX2 (tests/test_native.py), which makes glibc's ifunc pick __pow_sse2.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "glibc_pow.cuh"

static uint64_t s_state;
static uint64_t next_u64() {  // splitmix64
  uint64_t z = (s_state += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static double u01() { return (double)(next_u64() >> 11) * 0x1p-53; }
static double asd(uint64_t u) {
  double d;
  std::memcpy(&d, &u, 8);
  return d;
}
static uint64_t asu(double d) {
  uint64_t u;
  std::memcpy(&u, &d, 8);
  return u;
}

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: %s fma|sse2 [count] [seed]\n", argv[0]);
    return 2;
  }
  const bool fma = std::strcmp(argv[1], "fma") == 0;
  const uint64_t count = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 20000000ull;
  s_state = argc > 3 ? std::strtoull(argv[3], nullptr, 10) : 12345;
  double (*volatile libm_pow)(double, double) = &::pow;

  static const double specials[] = {0.0, -0.0, 1.0, -1.0, 2.0, -2.0, 0.5, -0.5, 3.0, -3.0, 1e-310, -1e-310,
                                    4.9e-324, 1e308, -1e308, INFINITY, -INFINITY, NAN, 0x1p-1022, 0x1p1023,
                                    1.0000000000000002, 0.9999999999999999, 0x1p-65, -0x1p-65, 0x1p63, 0x1p64,
                                    1075.0, -1075.0, 0.35, 0.7, 1e-20, 1e20, 511.5, 1023.99};
  const int ns = sizeof specials / sizeof specials[0];
  uint64_t bad = 0, n = 0;
  auto check = [&](double x, double y) {
    const double want = libm_pow(x, y);
    const double got = lemgpu::glibc_pow_v(fma ? 1 : 0, x, y);
    ++n;
    const bool same = (std::isnan(want) && std::isnan(got)) || asu(want) == asu(got);
    if (!same) {
      if (bad < 10)
        std::printf("MISMATCH pow(%a, %a): libm %a  restated %a\n", x, y, want, got);
      ++bad;
    }
  };
  for (int i = 0; i < ns; ++i)
    for (int j = 0; j < ns; ++j) check(specials[i], specials[j]);
  for (uint64_t i = 0; i < count; ++i) {
    const uint32_t kind = (uint32_t)(i % 10);
    double x, y;
    switch (kind) {
      case 0:  // pow(A*w, m): integer drainage areas, stream-power exponents
        x = (double)(1 + (next_u64() % 8000000));
        y = 0.25 + 0.6 * u01();
        break;
      case 1:  // the configs' m values exactly
        x = (double)(1 + (next_u64() % 70000000));
        y = 0.35 + 0.05 * (double)(next_u64() % 8);
        break;
      case 2:  // pow(diff, 2), pow(diff, n) for Newton differences
        x = std::ldexp(u01() + 0.5, -(int)(next_u64() % 60));
        y = (next_u64() & 1) ? 2.0 : 1.0 + 2.0 * u01();
        break;
      case 3:  // pow(diff, n - 1) for n < 1 and n > 1
        x = std::ldexp(u01() + 0.5, -(int)(next_u64() % 80));
        y = -0.9 + 2.8 * u01();
        break;
      case 4:  // random bit patterns
        x = asd(next_u64());
        y = asd(next_u64());
        break;
      case 5:  // moderate x, moderate y (overflow / subnormal result scaling)
        x = std::ldexp(u01() + 0.5, (int)(next_u64() % 200) - 100);
        y = (u01() - 0.5) * 40.0;
        break;
      case 6:  // results near overflow / underflow (specialcase)
        x = 1.0 + u01();
        y = (next_u64() & 1 ? 1.0 : -1.0) * (700.0 + 400.0 * u01()) / std::log(x > 1.0 ? x : 1.5);
        break;
      case 7:  // negative x with integer y
        x = -std::ldexp(u01() + 0.5, (int)(next_u64() % 40) - 20);
        y = (double)((int)(next_u64() % 41) - 20);
        break;
      case 8:  // subnormal x
        x = asd(next_u64() & 0x000fffffffffffffull);
        y = (u01() - 0.5) * 4.0;
        break;
      default:  // x near 1 (log's table boundary), tiny / huge y
        x = 1.0 + (u01() - 0.5) * 0x1p-20;
        y = std::ldexp(u01() - 0.5, (int)(next_u64() % 140) - 70);
        break;
    }
    check(x, y);
  }
  // the n = 2 fast path: glibc_pow_sq(x) == pow(x, 2), on random x and on x
  // whose square sits near a rounding midpoint (x = sqrt of a midpoint, nudged)
  uint64_t bad_sq = 0, nsq = 0;
  uint64_t nband = 0;
  for (uint64_t i = 0; i < count / 2; ++i) {
    double x;
    if (i % 4 == 1) {
      x = std::ldexp(u01() + 0.5, (int)(next_u64() % 120) - 80);
    } else if (i % 4 == 3) {
      // x^2 between 1/64 and 1/16 ulp away from a rounding midpoint: the band
      // the fast path newly decides (it answered only beyond 1/32 before)
      for (;;) {
        x = std::ldexp(u01() + 0.5, (int)(next_u64() % 136) - 68);
        const double hi = x * x, lo = std::fma(x, x, -hi);
        const double ulp = std::ldexp(1.0, std::ilogb(hi) - 52);
        const double d = ulp / 2 - std::fabs(lo);
        if (d >= ulp / 64 && d < ulp / 16) break;
      }
      ++nband;
    } else {
      const double m = std::ldexp(1.0 + u01(), (int)(next_u64() % 100) - 70);  // a square
      const double mid = m + std::ldexp(1.0, std::ilogb(m) - 53);            // the midpoint above it
      x = std::sqrt(mid);
      const int nudge = (int)(next_u64() % 7) - 3;
      for (int k = 0; k < (nudge < 0 ? -nudge : nudge); ++k) x = std::nextafter(x, nudge < 0 ? 0.0 : 1e300);
    }
    ++nsq;
    const double want = libm_pow(x, 2.0);
    const double got = fma ? lemgpu::glibc_pow_sq<true>(x) : lemgpu::glibc_pow_sq<false>(x);
    if (asu(want) != asu(got)) {
      if (bad_sq < 5) std::printf("POW_SQ MISMATCH x = %a: libm %a fast %a\n", x, want, got);
      ++bad_sq;
    }
  }
  std::printf("glibc_pow_sq: %llu inputs (%llu within 1/16 ulp of a midpoint), %llu mismatches\n",
              (unsigned long long)nsq, (unsigned long long)nband, (unsigned long long)bad_sq);
  bad += bad_sq;
  // identities the n = 1 and n = 2 Newton paths rely on (k_physics.cuh):
  // pow(x, 1) == x and pow(x, 0) == 1 for every positive finite x (normal or not)
  uint64_t bad_id = 0;
  for (uint64_t i = 0; i < count / 4; ++i) {
    const double x = asd(next_u64() & 0x7fefffffffffffffull);  // positive finite
    if (!(x > 0)) continue;
    if (asu(libm_pow(x, 1.0)) != asu(x) || libm_pow(x, 0.0) != 1.0) {
      if (bad_id < 5) std::printf("IDENTITY FAILS for x = %a: pow(x,1) = %a\n", x, libm_pow(x, 1.0));
      ++bad_id;
    }
  }
  std::printf("identities pow(x,1)==x, pow(x,0)==1: %llu inputs, %llu failures\n", (unsigned long long)(count / 4),
              (unsigned long long)bad_id);
  bad += bad_id;
  std::printf("%s: %llu inputs, %llu mismatches\n", fma ? "glibc_pow<fma>" : "glibc_pow<sse2>", (unsigned long long)n,
              (unsigned long long)bad);
  return bad ? 1 : 0;
}
