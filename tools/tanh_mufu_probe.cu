// Probe (not product code): exhaustive error of the tensor-core sweep's
// tanh_mufu (tc_common.cuh) against tanh in FP64 over EVERY float z with
// |z| <= 16 (beyond 9 the clamp returns tanh(9) rounded: checked too), the
// input of the derived tensor-core guard.
#include <cstdio>
#include <cuda_fp16.h>
#include "../paper_2406_01939_b200/csrc/tc_common.cuh"
using namespace pcd;

__global__ void k(unsigned lo, unsigned hi, unsigned long long* mx, unsigned* arg) {
  for (unsigned long long b = lo + blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; b < hi;
       b += (unsigned long long)gridDim.x * blockDim.x) {
    for (int sgn = 0; sgn < 2; ++sgn) {
      const float z = __uint_as_float((unsigned)b | (sgn ? 0x80000000u : 0u));
      const double e = fabs((double)tanh_mufu(z) - tanh((double)z));
      const unsigned long long eb = (unsigned long long)__double_as_longlong(e);
      if (eb > *mx) {
        atomicMax(mx, eb);
        *arg = __float_as_uint(z);
      }
    }
  }
}

int main() {
  unsigned long long* mx;
  unsigned* arg;
  cudaMalloc(&mx, 8);
  cudaMalloc(&arg, 4);
  // bands of |z|: the worst absolute error in each
  const float edges[] = {0.f, 1e-30f, 1e-3f, 0.1f, 0.5f, 1.f, 2.f, 4.f, 9.f, 16.f};
  double overall = 0;
  for (int i = 0; i + 1 < (int)(sizeof edges / sizeof edges[0]); ++i) {
    cudaMemset(mx, 0, 8);
    const unsigned lo = *(const unsigned*)&edges[i], hi = *(const unsigned*)&edges[i + 1];
    k<<<148 * 16, 256>>>(lo, hi, mx, arg);
    cudaDeviceSynchronize();
    unsigned long long h;
    unsigned a;
    cudaMemcpy(&h, mx, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&a, arg, 4, cudaMemcpyDeviceToHost);
    double e;
    memcpy(&e, &h, 8);
    float z;
    memcpy(&z, &a, 4);
    overall = e > overall ? e : overall;
    printf("|z| in [%g, %g): max |tanh_mufu - tanh| = %.4e (= %.3f * 2^-24) near z = %.8g\n", edges[i], edges[i + 1], e,
           e * 16777216.0, z);
  }
  printf("overall max abs error %.6e = %.4f * 2^-24\n", overall, overall * 16777216.0);
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
