// Device self-test of the grouped exact division (raster_math.cuh xdiv_*) that every selection-path quotient
// uses: bit-for-bit comparison with IEEE a / b on pseudo-random hard cases — significands near 1 and near 2,
// quotients near powers of two and near 1 (clamp boundaries), zero numerators, and exponents across and beyond
// the fast path's range (where the grouped path must fall back to the IEEE division).
#include <cuda_runtime.h>

#include <cstdint>

#include "raster_math.cuh"

namespace drb {

__device__ __forceinline__ uint64_t splitmix64(uint64_t& s) {
  uint64_t z = (s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ double draw(uint64_t& s, int lo, int hi) {
  const uint64_t r = splitmix64(s), m = splitmix64(s);
  const int e = lo + (int)(r % (uint64_t)(hi - lo + 1));
  uint64_t frac = m & 0xfffffffffffffull;
  switch ((r >> 20) & 7) {
    case 0: frac = 0xfffffffffffffull ^ (frac & 0xffull); break;  // 1.111..1x
    case 1: frac = frac & 0xffull; break;                           // 1.000..0x
    case 2: frac = frac & 0xfffff00000000ull; break;                // short significand
    case 3: frac = 0xfffffffffffffull ^ (frac & 0xfffffffull); break;
    default: break;
  }
  const uint64_t bits = ((r >> 63) << 63) | ((uint64_t)(e + 1023) << 52) | frac;
  return __longlong_as_double((long long)bits);
}

__global__ void k_selftest_div(uint64_t n, uint64_t seed, unsigned long long* bad, double* first_bad) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = tid; i < n; i += stride) {
    uint64_t s = seed ^ (i * 0xd1b54a32d192ed03ull);
    const int mode = (int)(splitmix64(s) % 6);
    double a[3], b;
    if (mode == 0) {  // the rasterizer's ranges (NDC coordinates, areas >= 1e-10)
      b = draw(s, -34, 4);
      for (double& x : a) x = draw(s, -40, 4);
    } else if (mode == 1) {  // everything finite, including the fast path's range limits
      b = draw(s, -1022, 1023);
      for (double& x : a) x = draw(s, -1022, 1023);
    } else if (mode == 2) {  // quotients close to powers of two
      b = draw(s, -30, 30);
      for (double& x : a) x = __longlong_as_double(__double_as_longlong(b * 0x1p+3) + (long long)(splitmix64(s) % 9) - 4);
    } else if (mode == 3) {  // quotients close to 1 (clamp boundaries)
      b = draw(s, -30, 30);
      for (double& x : a) x = __longlong_as_double(__double_as_longlong(b) + (long long)(splitmix64(s) % 65) - 32);
    } else if (mode == 4) {  // zero / tiny / subnormal numerators
      b = draw(s, -30, 30);
      a[0] = 0.0;
      a[1] = -0.0;
      a[2] = __longlong_as_double((long long)(splitmix64(s) & 0xfffffffffffffull));
    } else {  // tiny and huge divisors
      b = (splitmix64(s) & 1) ? draw(s, -1022, -960) : draw(s, 960, 1023);
      for (double& x : a) x = draw(s, -60, 60);
    }
    double q3[3];
    xdiv3(a[0], a[1], a[2], b, q3);
    double t[3];
    seg_t3_exact(a[0], b, a[1], b, a[2], b, t);
    for (int k = 0; k < 3; ++k) {
      const double want = a[k] / b;
      const double want_t = b > 0 ? clamp01(want) : 0.0;
      const bool same = __double_as_longlong(want) == __double_as_longlong(q3[k]) || (want != want && q3[k] != q3[k]);
      const bool same_t = __double_as_longlong(want_t) == __double_as_longlong(t[k]) ||
                          (want_t != want_t && t[k] != t[k]);
      if (!same || !same_t) {
        if (atomicAdd(bad, 1ull) == 0ull) {
          first_bad[0] = a[k];
          first_bad[1] = b;
        }
      }
    }
  }
}

}  // namespace drb

extern "C" int dr_selftest_division(uint64_t n, uint64_t seed, uint64_t* mismatches, double* first_bad_ab) {
  unsigned long long* d_bad = nullptr;
  double* d_first = nullptr;
  if (cudaMalloc(&d_bad, sizeof(unsigned long long)) != cudaSuccess) return 4;
  if (cudaMalloc(&d_first, 2 * sizeof(double)) != cudaSuccess) {
    cudaFree(d_bad);
    return 4;
  }
  cudaMemset(d_bad, 0, sizeof(unsigned long long));
  cudaMemset(d_first, 0, 2 * sizeof(double));
  drb::k_selftest_div<<<148 * 8, 256>>>(n, seed, d_bad, d_first);
  unsigned long long h_bad = 0;
  double h_first[2] = {0, 0};
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpy(&h_bad, d_bad, sizeof(h_bad), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(h_first, d_first, sizeof(h_first), cudaMemcpyDeviceToHost);
  cudaFree(d_bad);
  cudaFree(d_first);
  if (e != cudaSuccess) return 4;
  if (mismatches) *mismatches = (uint64_t)h_bad;
  if (first_bad_ab) {
    first_bad_ab[0] = h_first[0];
    first_bad_ab[1] = h_first[1];
  }
  return 0;
}
