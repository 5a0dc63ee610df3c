/*
 * oracle/expf_check.c -- host check of the expf restatement used by the
 * strict kernels (paper_2506_10315_b200/csrc/lopt_common.cuh glibc_expf).
 *
 * TEST INFRASTRUCTURE ONLY.  numba lowers np.exp on float32 to libm expf
 * (pkg/src/lopt/engine.py:537); this program evaluates the same double
 * arithmetic sequence as the device code on the host and compares it with
 * the process's libm expf over every `stride`-th float bit pattern (stride 1
 * = all 2^32 inputs).  Prints the mismatch count.
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static const uint64_t T[32] = {
    0x3ff0000000000000ULL, 0x3fefd9b0d3158574ULL, 0x3fefb5586cf9890fULL, 0x3fef9301d0125b51ULL,
    0x3fef72b83c7d517bULL, 0x3fef54873168b9aaULL, 0x3fef387a6e756238ULL, 0x3fef1e9df51fdee1ULL,
    0x3fef06fe0a31b715ULL, 0x3feef1a7373aa9cbULL, 0x3feedea64c123422ULL, 0x3feece086061892dULL,
    0x3feebfdad5362a27ULL, 0x3feeb42b569d4f82ULL, 0x3feeab07dd485429ULL, 0x3feea47eb03a5585ULL,
    0x3feea09e667f3bcdULL, 0x3fee9f75e8ec5f74ULL, 0x3feea11473eb0187ULL, 0x3feea589994cce13ULL,
    0x3feeace5422aa0dbULL, 0x3feeb737b0cdc5e5ULL, 0x3feec49182a3f090ULL, 0x3feed503b23e255dULL,
    0x3feee89f995ad3adULL, 0x3feeff76f2fb5e47ULL, 0x3fef199bdd85529cULL, 0x3fef3720dcef9069ULL,
    0x3fef5818dcfba487ULL, 0x3fef7c97337b9b5fULL, 0x3fefa4afa2a490daULL, 0x3fefd0765b6e4540ULL};

static uint32_t asu(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }

/* same sequence as lopt_common.cuh glibc_expf (fma = correctly rounded fma) */
static float restated_expf(float x) {
  const double kInvLn2N = 0x1.71547652b82fep+0 * 32, kShift = 0x1.8p+52;
  const double C0 = 0x1.c6af84b912394p-5 / 32 / 32 / 32, C1 = 0x1.ebfce50fac4f3p-3 / 32 / 32,
               C2 = 0x1.62e42ff0c52d6p-1 / 32;
  const uint32_t ux = asu(x), abstop = (ux >> 20) & 0x7ffu;
  if (abstop >= 0x42bu) {
    if (ux == 0xff800000u) return 0.0f;
    if (abstop >= 0x7f8u) return x + x;
    if (x > 0x1.62e42ep6f) return INFINITY;
    if (x < -0x1.9fe368p6f) return 0.0f;
  }
  const double xd = x, z = kInvLn2N * xd;
  double kd = z + kShift;
  uint64_t ki; memcpy(&ki, &kd, 8);
  kd -= kShift;
  const double r = fma(kInvLn2N, xd, -kd);
  uint64_t t = T[ki & 31u] + (ki << 47);
  double s; memcpy(&s, &t, 8);
  const double zz = fma(C0, r, C1), r2 = r * r;
  double y = fma(C2, r, 1.0);
  y = fma(zz, r2, y);
  return (float)(y * s);
}

int main(int argc, char **argv) {
  const long long stride = argc > 1 ? atoll(argv[1]) : 1;
  unsigned long long mism = 0, tot = 0;
#pragma omp parallel for reduction(+ : mism, tot) schedule(static)
  for (long long i = 0; i < (1LL << 32); i += stride) {
    const uint32_t u = (uint32_t)i;
    float x; memcpy(&x, &u, 4);
    if (isnan(x)) continue;
    tot++;
    if (asu(expf(x)) != asu(restated_expf(x))) mism++;
  }
  printf("%llu %llu\n", mism, tot);
  return 0;
}
