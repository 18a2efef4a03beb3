// div_int_rn (sf_internal.cuh) against __ddiv_rn, bit for bit, over the operand domain the library
// uses (integer-valued 1 <= num < 2^31, 1 <= den < 2^63), sampled with a counter RNG and with
// structured edge cases.  Prints "<samples> <mismatches>".
#include <cstdio>
#include <cstdlib>
#include "../../paper_2601_12784_b200/csrc/sf_internal.cuh"

__device__ unsigned long long mix(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void k(unsigned long long n, unsigned long long *bad, unsigned long long *first) {
  for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long a = mix(2 * i), b = mix(2 * i + 1);
    long long num, den;
    switch (i & 3) {
      case 0: num = 1 + (long long)(a % 2147483647ULL); den = 1 + (long long)(b % ((1ULL << 53) - 1)); break;
      case 1: num = 1 + (long long)(a % 4096); den = 1 + (long long)(b % (1ULL << 40)); break;   // Eq 2 / 4 shapes
      case 2: num = 1 + (long long)(a % 256); den = (long long)(1ULL << (b % 53)) + (long long)((b >> 8) % 3) - 1; break;
      case 3: num = 1 + (long long)(a % 2147483647ULL); den = ((i >> 2) & 1) ? 1 + (long long)(b % 4096)
                                                                        : 1 + (long long)(b % ((1ULL << 62) - 1)); break;
    }
    if (den < 1) den = 1;
    const double x = __ll2double_rn(num), y = __ll2double_rn(den);   // den > 2^53 rounds, as in Eq 2
    const double q1 = sf::div_int_rn(x, y), q2 = __ddiv_rn(x, y);
    if (__double_as_longlong(q1) != __double_as_longlong(q2)) {
      if (atomicAdd(bad, 1ULL) == 0) { first[0] = num; first[1] = den; }
    }
  }
}

int main(int argc, char **argv) {
  const unsigned long long n = argc > 1 ? strtoull(argv[1], 0, 10) : (1ULL << 30);
  unsigned long long *d;
  cudaMalloc(&d, 3 * sizeof(unsigned long long));
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  k<<<148 * 8, 256>>>(n, d, d + 1);
  unsigned long long h[3];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  printf("%llu %llu\n", n, h[0]);
  if (h[0]) printf("first mismatch: %lld / %lld\n", (long long)h[1], (long long)h[2]);
  return cudaDeviceSynchronize() != cudaSuccess;
}
