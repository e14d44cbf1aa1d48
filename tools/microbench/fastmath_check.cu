// Bitwise check of fast_sqrt_normal / fast_div_normal (csrc/common.cuh) against
// the compiler's IEEE sqrt() and / on the device: random operands across the
// exponent range the Jacobi rotations use them in, plus structured cases.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -I../../paper_2603_11953_b200/csrc
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "common.cuh"

using namespace mpsvd::dev;

__device__ unsigned long long g_bad_sqrt = 0, g_bad_div = 0, g_n = 0;
__device__ double g_ex[4];

__device__ __forceinline__ uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// random double with exponent in [elo, ehi] (unbiased exponent), random sign optional
__device__ __forceinline__ double rnd(uint64_t& st, int elo, int ehi, bool neg) {
  st = mix(st);
  const uint64_t mant = st & 0xFFFFFFFFFFFFFull;
  st = mix(st);
  const int e = elo + (int)(st % (uint64_t)(ehi - elo + 1));
  uint64_t bits = ((uint64_t)(e + 1023) << 52) | mant;
  if (neg && (st >> 40 & 1)) bits |= 1ull << 63;
  return __longlong_as_double((long long)bits);
}

__global__ void check(int iters, int mode) {
  uint64_t st = mix(((uint64_t)blockIdx.x << 32) ^ threadIdx.x ^ ((uint64_t)mode << 56));
  unsigned long long bs = 0, bd = 0;
  for (int i = 0; i < iters; ++i) {
    double a, b;
    if (mode == 0) {  // wide exponents
      a = rnd(st, -800, 800, false);
      b = rnd(st, -400, 400, true);
    } else if (mode == 1) {  // near one (c^2 in [0.5, 1], unit-scale matrices)
      a = rnd(st, -2, 1, false);
      b = rnd(st, -2, 2, true);
    } else {  // mantissas with few bits (exact / halfway cases)
      a = rnd(st, -60, 60, false);
      b = rnd(st, -60, 60, true);
      a = __longlong_as_double(__double_as_longlong(a) & ~0xFFFFFFFFFFull);
      b = __longlong_as_double(__double_as_longlong(b) & ~0xFFFFFFFFFFFull);
    }
    const double s1 = sqrt(a), s2 = fast_sqrt_normal(a);
    if (__double_as_longlong(s1) != __double_as_longlong(s2)) {
      if (!bs) { g_ex[0] = a; }
      ++bs;
    }
    // quotient kept inside the normal range, as the callers guarantee
    double num = rnd(st, -200, 200, true);
    if (mode == 1) num = rnd(st, -3, 3, true);
    const double d1 = num / b, d2 = fast_div_normal(num, b);
    if (__double_as_longlong(d1) != __double_as_longlong(d2)) {
      if (!bd) { g_ex[1] = num; g_ex[2] = b; }
      ++bd;
    }
    const double d3 = 1.0 / a, d4 = fast_div_normal(1.0, a);
    if (__double_as_longlong(d3) != __double_as_longlong(d4)) {
      if (!bd) { g_ex[1] = 1.0; g_ex[2] = a; }
      ++bd;
    }
  }
  atomicAdd(&g_bad_sqrt, bs);
  atomicAdd(&g_bad_div, bd);
  atomicAdd(&g_n, (unsigned long long)iters);
}

int main() {
  for (int mode = 0; mode < 3; ++mode) {
    check<<<148 * 8, 256>>>(4096, mode);
    cudaDeviceSynchronize();
  }
  unsigned long long bs, bd, n;
  double ex[4];
  cudaMemcpyFromSymbol(&bs, g_bad_sqrt, 8);
  cudaMemcpyFromSymbol(&bd, g_bad_div, 8);
  cudaMemcpyFromSymbol(&n, g_n, 8);
  cudaMemcpyFromSymbol(ex, g_ex, sizeof(ex));
  printf("fastmath_check: %llu operands per function: sqrt mismatches %llu, div mismatches %llu (of 2x)\n", n, bs, bd);
  if (bs) printf("  first sqrt mismatch at a = %a\n", ex[0]);
  if (bd) printf("  first div mismatch at %a / %a\n", ex[1], ex[2]);
  printf("JSON {\"operands\": %llu, \"sqrt_mismatches\": %llu, \"div_mismatches\": %llu}\n", n, bs, bd);
  return (bs || bd) ? 1 : 0;
}
