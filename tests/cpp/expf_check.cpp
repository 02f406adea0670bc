// Compare dsb::glibc_expf (device recipe, host build) with libm expf over every
// float bit pattern with stride argv[1] (1 = exhaustive, ~30 s).
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "expf_glibc.h"

int main(int argc, char** argv) {
  const unsigned long long stride = argc > 1 ? strtoull(argv[1], nullptr, 10) : 1;
  unsigned long long bad = 0, n = 0;
  for (unsigned long long u = 0; u <= 0xffffffffull; u += stride) {
    const float x = dsb::u2f(static_cast<uint32_t>(u));
    const float a = dsb::glibc_expf(x), b = expf(x);
    if (dsb::f2u(a) != dsb::f2u(b) && !(std::isnan(a) && std::isnan(b))) {
      if (bad < 5) printf("x=%a got %a want %a\n", x, a, b);
      ++bad;
    }
    ++n;
  }
  printf("checked %llu mismatches %llu\n", n, bad);
  return bad != 0;
}
