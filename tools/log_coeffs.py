"""Coefficients and host check of the far-pair log (kernels.cuh log_tab).

1. p(t): the quartic Chebyshev fit (mpmath, 60 digits) of (log1p t - t) / t^2
   on |t| <= 2^-8 (128 buckets per octave); prints its coefficients as hex
   floats (highest first) and the bound
   |log1p t - (t + t^2 p(t))| <= err * t^2 <= err * 2^-8 |t|.
2. A host emulation of log_tab (the same table search as eval.cu log_table,
   the same operations, C fma) against 80-bit logl: max ulp over 8M points in
   [2^-20, 4] and every bucket edge of every exponent.

    python tools/log_coeffs.py
"""
import os
import subprocess
import tempfile

import mpmath as mp

mp.mp.dps = 60
a = mp.mpf(2) ** -8 * (1 + mp.mpf(2) ** -11)


def f(t):
    if abs(t) < mp.mpf(10) ** -30:
        return mp.mpf(-1) / 2
    return (mp.log1p(t) - t) / t ** 2


poly, err = mp.chebyfit(f, [-a, a], 5, error=True)
coeffs = [float(x) for x in poly]
print("p(t), highest first:", [c.hex() for c in coeffs])
print("max |f - p| =", mp.nstr(err, 5), "; relative to t: 2^%s" % mp.nstr(mp.log(err * a, 2), 5))

EMUL = r"""
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>
static const int K = 0x3FE6B000, NB = 7, N = 1 << NB, SH = 20 - NB;
static double fromhl(uint32_t h, uint32_t l) { uint64_t b = (uint64_t(h) << 32) | l; double d; memcpy(&d, &b, 8); return d; }
static uint32_t hiw(double x) { uint64_t b; memcpy(&b, &x, 8); return b >> 32; }
static uint32_t low(double x) { uint64_t b; memcpy(&b, &x, 8); return (uint32_t)b; }
static double rc[N], lc[N];
static const double C6 = %(c6)s, C5 = %(c5)s, C4 = %(c4)s, C3 = %(c3)s, C2 = %(c2)s;
static double newlog(double x) {
  int hi = (int)hiw(x), t1 = hi - K, kk = t1 >> 20, j = (t1 >> SH) & (N - 1);
  double m = fromhl(hi - (t1 & (int)0xfff00000u), low(x));
  double t = fma(m, rc[j], -1.0);
  double p = fma(t, C6, C5); p = fma(t, p, C4); p = fma(t, p, C3); p = fma(t, p, C2);
  double l1p = fma(t * t, p, t);
  return fma((double)kk, 0x1.62e42fefa39efp-1, lc[j] + l1p);
}
int main() {
  int tries = 0;
  for (int j = 0; j < N; ++j) {  // eval.cu log_table
    long double c = fromhl(K + (j << SH) + (1 << (SH - 1)), 0);
    long double r0 = 1.0L / c;
    double best_r = (double)r0, best_e = 1.0;
    for (int i = 0; i < 4096 && best_e > 1.0 / 64; ++i, ++tries) {
      long double step = 1e-9L * (long double)((i & 1) ? -((i + 1) / 2) : i / 2);
      double r = (double)(r0 * (1.0L + step));
      long double L = -logl((long double)r);
      double Ld = (double)L;
      long double u = Ld == 0.0 ? 1.0L : (long double)(nextafter(fabs(Ld), 1.0) - fabs(Ld));
      double e = (double)(fabsl(L - (long double)Ld) / u);
      if (e < best_e) best_e = e, best_r = r;
    }
    rc[j] = best_r;
    lc[j] = (double)(-logl((long double)best_r));
  }
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(std::log(std::ldexp(1.0, -20)), std::log(4.0)), V(0.7, 1.42);
  std::vector<double> xs;
  for (int i = 0; i < 4000000; ++i) xs.push_back(std::exp(U(g)));
  for (int i = 0; i < 4000000; ++i) xs.push_back(V(g));
  for (int j = 0; j < N; ++j)
    for (int k = -20; k <= 1; ++k) {
      uint32_t h = K + (j << SH) + (k << 20);
      double b = fromhl(h, 0), e = fromhl(h + (1 << SH) - 1, 0xffffffffu);
      xs.push_back(b); xs.push_back(nextafter(b, 0)); xs.push_back(e); xs.push_back(nextafter(e, 4));
    }
  double mx = 0;
  for (double x : xs) {
    if (x < std::ldexp(1.0, -20) || x > 4) continue;
    long double r = logl((long double)x);
    double rr = (double)r, sp = rr == 0 ? 4.9e-324 : std::fabs(nextafter(std::fabs(rr), INFINITY) - std::fabs(rr));
    mx = std::fmax(mx, (double)(fabsl((long double)newlog(x) - r)) / sp);
  }
  printf("table search: %%d candidates for %%d buckets; max ulp against logl over %%zu points: %%.3f; log_tab(1) = %%g\n",
         tries, N, xs.size(), mx, newlog(1.0));
}
"""
with tempfile.TemporaryDirectory() as d:
    src, exe = os.path.join(d, "emul.cpp"), os.path.join(d, "emul")
    with open(src, "w") as fh:
        fh.write(EMUL % dict(c6=coeffs[0].hex(), c5=coeffs[1].hex(), c4=coeffs[2].hex(), c3=coeffs[3].hex(),
                             c2=coeffs[4].hex()))
    subprocess.run(["g++", "-O2", "-ffp-contract=off", "-o", exe, src], check=True)
    print(subprocess.run([exe], capture_output=True, text=True, check=True).stdout.strip())
