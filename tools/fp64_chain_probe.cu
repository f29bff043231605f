// Probe (not product code): latency of the exact FP64 acc = acc + w*x chain
// (the recheck's inner loop) with weights from registers / global (L2-hot).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(const double* __restrict__ W, const double* __restrict__ x, int K, int width, int reps,
                      long long* clk, double* out) {
  const int r = threadIdx.x;
  __shared__ double xs[256];
  for (int i = r; i < K; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  double acc = 0.0;
  long long t0 = clock64();
  // (a) register-only dependent chain
  double a = 1.0 + r * 1e-9;
  for (int c = 0; c < K; ++c) a = __dadd_rn(a, __dmul_rn(a, 1e-9));
  long long t1 = clock64();
  // (b) weights from global, 16 loads ahead
  for (int rep = 0; rep < reps; ++rep) {
    acc = 0.0;
    const double* w = W + r;
    for (int c = 0; c + 16 <= K; c += 16) {
      double wv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) wv[u] = __ldg(w + (size_t)(c + u) * width);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, __dmul_rn(wv[u], xs[c + u]));
    }
  }
  long long t2 = clock64();
  if (r == 0) { clk[0] = t1 - t0; clk[1] = (t2 - t1) / reps; }
  out[r] = acc + a;
}

int main() {
  const int K = 208, width = 64;
  double *W, *x, *out; long long* clk;
  cudaMalloc(&W, K * width * 8); cudaMalloc(&x, K * 8); cudaMalloc(&out, 256 * 8); cudaMalloc(&clk, 16);
  cudaMemset(W, 0, K * width * 8); cudaMemset(x, 0, K * 8);
  for (int it = 0; it < 3; ++it) {
    chain<<<1, 64>>>(W, x, K, width, 4, clk, out);
    cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, clk, 16, cudaMemcpyDeviceToHost);
    printf("K=%d: register chain %lld clk (%.1f/elem), global-weight chain %lld clk (%.1f/elem)\n", K, h[0],
           (double)h[0] / K, h[1], (double)h[1] / K);
  }
  return 0;
}
