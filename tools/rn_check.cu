// Bitwise check of the branch-free div_fast / sqrt_fast / dvd_const_fast
// (ocp_common.cuh) against __ddiv_rn / __dsqrt_rn on the GPU: random operands
// over the accepted exponent range plus near-tie patterns (quotients and roots
// within a few ulps of a rounding boundary).  Any operand pair the fast version
// accepts (slow == false) must give the intrinsic's bits.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2411_00546_b200/csrc
//        -o tools/rn_check tools/rn_check.cu
#include <cstdio>
#include <cstdint>
#include "ocp_common.cuh"

using namespace ocp;

__device__ __forceinline__ uint64_t mix(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// random double with biased exponent in [elo, ehi] and random sign
__device__ __forceinline__ double rnd(uint64_t& s, int elo, int ehi, bool sign) {
  const uint64_t r = mix(s);
  const uint64_t e = elo + (mix(s) % (uint64_t)(ehi - elo + 1));
  uint64_t bits = (r & 0x000fffffffffffffull) | (e << 52);
  if (sign && (r >> 63)) bits |= 0x8000000000000000ull;
  return __longlong_as_double((long long)bits);
}

__global__ void k_check(int iters, unsigned long long* out) {
  uint64_t s = 0x1234567ull + 7919ull * (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x);
  unsigned long long bad_div = 0, bad_sqrt = 0, bad_dc = 0, skipped = 0, bad_tie = 0;
  for (int it = 0; it < iters; ++it) {
    // 1. random division, exponents 2^-480 .. 2^480
    {
      const double a = rnd(s, 1023 - 480, 1023 + 480, true), b = rnd(s, 1023 - 480, 1023 + 480, true);
      bool slow = false;
      const double q = div_fast(a, b, slow);
      if (slow) ++skipped;
      else if (__double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) ++bad_div;
    }
    // 2. near-tie division: a = RN(q b) nudged by a few ulps, q with few mantissa bits set
    {
      const double b = rnd(s, 1023 - 3, 1023 + 3, false);
      double q = rnd(s, 1023 - 3, 1023 + 3, false);
      // q = (integer + 1/2) ulp patterns: low mantissa bits random in a short window
      const long long qb = (__double_as_longlong(q) & ~0xffffll) | (long long)(mix(s) & 0xf);
      q = __longlong_as_double(qb);
      double a = __dmul_rn(q, b);
      a = __longlong_as_double(__double_as_longlong(a) + (long long)(mix(s) % 5) - 2);
      bool slow = false;
      const double r = div_fast(a, b, slow);
      if (!slow && __double_as_longlong(r) != __double_as_longlong(__ddiv_rn(a, b))) ++bad_tie;
    }
    // 3. the residual's own division shape: a / sqrt(a^2 + eps)
    {
      const double a = rnd(s, 1023 - 30, 1023 + 12, true);
      const double eps = rnd(s, 1023 - 50, 1023, false);
      const double arg = __dadd_rn(__dmul_rn(a, a), eps);
      bool slow = false;
      const double sf = sqrt_fast(arg, slow);
      const double si = __dsqrt_rn(arg);
      if (!slow && __double_as_longlong(sf) != __double_as_longlong(si)) ++bad_sqrt;
      const double qf = div_fast(a, si, slow);
      if (!slow && __double_as_longlong(qf) != __double_as_longlong(__ddiv_rn(a, si))) ++bad_div;
    }
    // 4. random sqrt over the whole accepted range, and near perfect squares
    {
      const double x = rnd(s, 60, 2040, false);
      bool slow = false;
      const double r = sqrt_fast(x, slow);
      if (slow) ++skipped;
      else if (__double_as_longlong(r) != __double_as_longlong(__dsqrt_rn(x))) ++bad_sqrt;
      const double m = rnd(s, 1023 - 8, 1023 + 8, false);
      double sq = __dmul_rn(m, m);
      sq = __longlong_as_double(__double_as_longlong(sq) + (long long)(mix(s) % 7) - 3);
      slow = false;
      const double r2 = sqrt_fast(sq, slow);
      if (!slow && __double_as_longlong(r2) != __double_as_longlong(__dsqrt_rn(sq))) ++bad_tie;
    }
    // 5. constant-divisor division incl. signed zeros
    {
      const double b = (it & 1) ? 1e-3 : 1e-2;
      const double rb = 1.0 / b;
      double a = rnd(s, 1023 - 400, 1023 + 400, true);
      if ((it & 1023) == 0) a = (it & 1024) ? 0.0 : -0.0;
      bool slow = false;
      const double q = dvd_const_fast(a, b, rb, slow);
      if (!slow && __double_as_longlong(q) != __double_as_longlong(__ddiv_rn(a, b))) ++bad_dc;
    }
  }
  atomicAdd(out + 0, bad_div);
  atomicAdd(out + 1, bad_sqrt);
  atomicAdd(out + 2, bad_dc);
  atomicAdd(out + 3, skipped);
  atomicAdd(out + 4, bad_tie);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? atoi(argv[1]) : 4096;
  unsigned long long* out;
  cudaMallocManaged(&out, 8 * 8);
  for (int i = 0; i < 8; ++i) out[i] = 0;
  const int grid = 148 * 16, block = 256;
  k_check<<<grid, block>>>(iters, out);
  cudaDeviceSynchronize();
  const double n = (double)grid * block * iters;
  printf("rn_check: %.3g iterations (7 comparisons each): mismatches div %llu, sqrt %llu, dvd_const %llu, "
         "near-tie %llu; outside the fast range %llu (%s)\n",
         n, out[0], out[1], out[2], out[4], out[3], cudaGetErrorString(cudaGetLastError()));
  return (out[0] | out[1] | out[2] | out[4]) ? 1 : 0;
}
