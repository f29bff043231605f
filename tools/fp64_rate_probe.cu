// DFMA / FFMA throughput probe on one B200 (not a test): 148 x 512 threads,
// 16 independent FMA chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <typename T>
__global__ void k(T* out, int iters, T s) {
  T a[16];
  for (int i = 0; i < 16; ++i) a[i] = (T)(threadIdx.x + i);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], s, (T)0.5);
  T r = 0;
  for (int i = 0; i < 16; ++i) r += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
template <typename T>
void run(const char* name) {
  T* d;
  cudaMalloc(&d, 148 * 512 * sizeof(T));
  const int iters = 20000;
  k<T><<<148, 512>>>(d, 100, (T)0.999);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<T><<<148, 512>>>(d, iters, (T)0.999);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fl = 2.0 * 16 * iters * 148.0 * 512;
  printf("%s: %.2f TFLOP/s (%.3f ms)\n", name, fl / ms / 1e9, ms);
}
int main() { run<double>("DFMA"); run<float>("FFMA"); }
