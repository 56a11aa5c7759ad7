// Bit-identity of the epilogue's branch-free division fast path
// (ofdmrx_fft.cuh: recip / div_fast under the in_range guards used by
// finish_points_qb) with IEEE division (__fdiv_rn, what numpy computes).
// Test infrastructure for tests/test_gpu_division.py.  Sweeps: every divisor
// mantissa at several exponents x sampled dividends (the s_hat = num / den
// guard, [2^-40, 2^40)), random dividends over the demap guard
// ([2^-90, 2^90)) against the QAM scales, and random bit patterns.
#include <cstdio>
#include <cstdint>
#include "ofdmrx_fft.cuh"

using namespace ofdmrx;

__device__ unsigned long long g_bad = 0, g_fast = 0, g_total = 0;

__device__ __forceinline__ uint32_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
  return (uint32_t)x;
}
// a / b through the fast path whenever the product's guard admits it: both
// operands in [2^-40, 2^40) (s_hat = num / den), or the dividend in
// [2^-90, 2^90) and the divisor in [2^-8, 2^8) (the demap's s_hat / scale)
__device__ void check(float a, float b, bool demap, unsigned long long& bad, unsigned long long& fast) {
  const bool admit = demap ? in_range(kPow2m90, kPow2p90, a, a, 1.0f) && in_range(kPow2m8, kPow2p8, b, 1.0f, 1.0f)
                           : in_range(kPow2m40, kPow2p40, a, a, b);
  if (!admit) return;
  ++fast;
  const float q = div_fast(a, recip(b)), want = __fdiv_rn(a, b);
  if (__float_as_uint(q) != __float_as_uint(want)) ++bad;
}

__global__ void sweep_mantissa(int exp_b, uint64_t seed) {
  unsigned long long bad = 0, fast = 0, tot = 0;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x) {
    const float b = __uint_as_float(((uint32_t)(exp_b + 127) << 23) | m);
    for (int j = 0; j < 4; ++j) {
      const uint32_t r = mix(seed * 0x9e3779b97f4a7c15ULL + m * 4ull + j);
      const float a = __uint_as_float((r & 0x807fffffu) | (((r >> 23) % 80u + 87u) << 23));  // 2^-40 .. 2^40
      check(a, b, false, bad, fast);
      ++tot;
    }
  }
  atomicAdd(&g_bad, bad); atomicAdd(&g_fast, fast); atomicAdd(&g_total, tot);
}

__global__ void sweep_demap(float scale, uint64_t seed, int per_thread) {
  unsigned long long bad = 0, fast = 0, tot = 0;
  const uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    const uint32_t r = mix(seed * 0x100000000ULL + id * per_thread + i);
    const float s = __uint_as_float((r & 0x807fffffu) | ((37u + (r >> 23) % 180u) << 23));  // 2^-90 .. 2^90
    check(s, scale, true, bad, fast);
    ++tot;
  }
  atomicAdd(&g_bad, bad); atomicAdd(&g_fast, fast); atomicAdd(&g_total, tot);
}

__global__ void sweep_random(uint64_t seed, int per_thread) {  // any bit patterns (guard decides)
  unsigned long long bad = 0, fast = 0, tot = 0;
  const uint64_t id = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (int i = 0; i < per_thread; ++i) {
    const uint64_t k = (id * per_thread + i) * 2 + seed * 0x1000000000ULL;
    const float a = __uint_as_float(mix(k)), b = __uint_as_float(mix(k + 1));
    check(a, b, false, bad, fast);
    check(a, __uint_as_float((__float_as_uint(b) & 0x807fffffu) | ((119u + (mix(k + 7) >> 28)) << 23)), true, bad, fast);
    ++tot;
  }
  atomicAdd(&g_bad, bad); atomicAdd(&g_fast, fast); atomicAdd(&g_total, tot);
}

int main() {
  for (int e = -40; e < 40; e += 7) sweep_mantissa<<<148 * 8, 256>>>(e, 17 + e + 40);
  sweep_mantissa<<<148 * 8, 256>>>(39, 3);
  const float scales[3] = {0.70710677f, 0.31622776f, 0.15430336f};  // QPSK, 16-, 64-QAM (qam_consts)
  for (int k = 0; k < 3; ++k) sweep_demap<<<148 * 8, 256>>>(scales[k], 5 + k, 64);
  sweep_random<<<148 * 8, 256>>>(1, 64);
  if (cudaDeviceSynchronize() != cudaSuccess) { printf("{\"error\": \"launch\"}\n"); return 2; }
  unsigned long long bad, fast, tot;
  cudaMemcpyFromSymbol(&bad, g_bad, 8); cudaMemcpyFromSymbol(&fast, g_fast, 8); cudaMemcpyFromSymbol(&tot, g_total, 8);
  printf("{\"checked\": %llu, \"fast_path\": %llu, \"mismatches\": %llu}\n", tot, fast, bad);
  return bad == 0 ? 0 : 1;
}
