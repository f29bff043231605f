// Probe (not product code): the fp32 accumulation behaviour of
// tcgen05.mma.kind::f16 on sm_100a, the input of the derived tensor-core guard
// (DESIGN.md §4.3a). M = 64 rows, N = 16 columns, S k-steps of K = 16 issued
// back to back into one TMEM accumulator initialised with C (accumulate = 1).
// Each row/column pair is one test: D = C + sum_k a_k b_k over K = 16 S.
//   crafted rows: alignment width and rounding mode of one k-step;
//   random rows: the error of long chains against exact (binary128) sums,
//   in units of u = 2^-24 times sum |terms| and times max |partial|.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <random>
#include <vector>
#include <cuda_fp16.h>
#include "../paper_2406_01939_b200/csrc/tc_common.cuh"
using namespace pcd;

constexpr int kM = 64, kN = 16, kMaxS = 13;

__global__ void probe(const __half* A, const __half* B, const float* Cinit, int S, float* out) {
  extern __shared__ __align__(1024) unsigned char sm[];
  unsigned char* sA = sm;                       // S chunks of 64 x 16 halves
  unsigned char* sB = sm + kMaxS * kM * 16 * 2;  // S chunks of 16 x 16 halves
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kM * 16 * S; i += blockDim.x) {
    const int r = i / (16 * S), k = i % (16 * S);
    *(__half*)(sA + (k / 16) * kM * 32 + canon_off(kM, r, k % 16)) = A[r * 16 * S + k];
  }
  for (int i = tid; i < kN * 16 * S; i += blockDim.x) {
    const int n = i / (16 * S), k = i % (16 * S);
    *(__half*)(sB + (k / 16) * kN * 32 + canon_off(kN, n, k % 16)) = B[n * 16 * S + k];
  }
  if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = tbase;
  // C -> TMEM (M = 64 accumulator: rows r live in lanes 32(r/16) + r%16, as tc_pp.cu's half 0)
  {
    // 32x32b store: thread = lane of its 32-lane subpartition, 16 columns
    const int r = (lane < 16) ? 16 * warp + lane : -1;
    uint32_t v[16];
    for (int c = 0; c < 16; ++c) v[c] = r >= 0 ? __float_as_uint(Cinit[r * kN + c]) : 0u;
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            tm + ((uint32_t)(32 * warp) << 16)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
        : "memory");
    tmem_wait_st();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    const uint32_t id = idesc_f16(kM, kN);
    for (int s = 0; s < S; ++s) {
      const uint64_t a = umma_desc(smem_u32(sA + s * kM * 32), kM * 16, 128);
      const uint64_t b = umma_desc(smem_u32(sB + s * kN * 32), kN * 16, 128);
      mma_f16(tm, a, b, id, 1);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  float v[16];
  tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
  tmem_wait_ld();
  if (lane < 16)
    for (int c = 0; c < 16; ++c) out[(16 * warp + lane) * kN + c] = v[c];
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(32));
  }
}

struct Case {
  std::vector<__half> A, B;
  std::vector<float> C;
  int S;
};

static void run(const Case& cs, std::vector<float>& D) {
  __half *dA, *dB;
  float *dC, *dD;
  cudaMalloc(&dA, cs.A.size() * 2);
  cudaMalloc(&dB, cs.B.size() * 2);
  cudaMalloc(&dC, cs.C.size() * 4);
  cudaMalloc(&dD, kM * kN * 4);
  cudaMemcpy(dA, cs.A.data(), cs.A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, cs.B.data(), cs.B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dC, cs.C.data(), cs.C.size() * 4, cudaMemcpyHostToDevice);
  const size_t smem = kMaxS * (kM + kN) * 32;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  probe<<<1, 128, smem>>>(dA, dB, dC, cs.S, dD);
  const cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
  D.resize(kM * kN);
  cudaMemcpy(D.data(), dD, kM * kN * 4, cudaMemcpyDeviceToHost);
  cudaFree(dA); cudaFree(dB); cudaFree(dC); cudaFree(dD);
}

static Case blank(int S) {
  Case c;
  c.S = S;
  c.A.assign(kM * 16 * S, __float2half(0.f));
  c.B.assign(kN * 16 * S, __float2half(0.f));
  c.C.assign(kM * kN, 0.f);
  return c;
}

int main() {
  // ---- crafted single k-step cases (column 0: b = 1 everywhere)
  {
    Case c = blank(1);
    for (int k = 0; k < 16; ++k) c.B[0 * 16 + k] = __float2half(1.f);
    // rows 0..9: 1 + 2^-e for e = 20..29 (one small product)
    for (int i = 0; i < 10; ++i) { c.A[i * 16 + 0] = __float2half(1.f); c.A[i * 16 + 1] = __float2half(ldexpf(1.f, -(20 + i))); }
    // rows 10..19: 1 + 15 * 2^-e for e = 22..31 (fifteen small products)
    for (int i = 0; i < 10; ++i) { c.A[(10 + i) * 16 + 0] = __float2half(1.f);
      for (int k = 1; k < 16; ++k) c.A[(10 + i) * 16 + k] = __float2half(ldexpf(1.f, -(22 + i))); }
    // rows 20..23: 1 + 1.5 * 2^-23 (= 1 + 2^-23 + 2^-24: RN -> 1 + 2^-22, RZ -> 1 + 2^-23)
    for (int i = 0; i < 4; ++i) { c.A[(20 + i) * 16 + 0] = __float2half(1.f);
      c.A[(20 + i) * 16 + 1] = __float2half(ldexpf(1.f, -23)); c.A[(20 + i) * 16 + 2] = __float2half(ldexpf(1.f, -24)); }
    // rows 24..27: 1 - 1.5 * 2^-24 (RN -> 1 - 2^-23, RZ -> 1 - 2^-24... in [0.5, 1) the ulp is 2^-24)
    for (int i = 0; i < 4; ++i) { c.A[(24 + i) * 16 + 0] = __float2half(1.f);
      c.A[(24 + i) * 16 + 1] = __float2half(-ldexpf(1.f, -24)); c.A[(24 + i) * 16 + 2] = __float2half(-ldexpf(1.f, -25)); }
    // rows 28..37: C = 1 (accumulator) + one product 2^-e, e = 20..29
    for (int i = 0; i < 10; ++i) { c.C[(28 + i) * kN + 0] = 1.f; c.A[(28 + i) * 16 + 1] = __float2half(ldexpf(1.f, -(20 + i))); }
    // rows 38..47: C = 1 + fifteen products 2^-e, e = 22..31
    for (int i = 0; i < 10; ++i) { c.C[(38 + i) * kN + 0] = 1.f;
      for (int k = 1; k < 16; ++k) c.A[(38 + i) * 16 + k] = __float2half(ldexpf(1.f, -(22 + i))); }
    // rows 48..51: cancellation 2^10 - (2^10 - 2^-10) style: a0 = 1024, a1 = -1023.5? (exact), plus 2^-20
    for (int i = 0; i < 4; ++i) { c.A[(48 + i) * 16 + 0] = __float2half(1024.f); c.A[(48 + i) * 16 + 1] = __float2half(-1024.f);
      c.A[(48 + i) * 16 + 2] = __float2half(ldexpf(1.f, -(14 + 4 * i))); }
    std::vector<float> D;
    run(c, D);
    auto show = [&](const char* what, int r0, int n, int e0) {
      for (int i = 0; i < n; ++i) {
        const double d = D[(r0 + i) * kN + 0];
        printf("%s e=%d: D-1 = %.9g (= %.6f * 2^-24)\n", what, e0 + i, d - 1.0, (d - 1.0) * 16777216.0);
      }
    };
    show("1 + 2^-e          ", 0, 10, 20);
    show("1 + 15*2^-e       ", 10, 10, 22);
    printf("1 + 1.5*2^-23: D-1 = %.6f * 2^-24 (RN 4, RZ 2)\n", (D[20 * kN] - 1.0) * 16777216.0);
    printf("1 - 1.5*2^-24: D-1 = %.6f * 2^-24 (RN -2, RZ -1)\n", (D[24 * kN] - 1.0) * 16777216.0);
    show("C=1, + 2^-e       ", 28, 10, 20);
    show("C=1, + 15*2^-e    ", 38, 10, 22);
    for (int i = 0; i < 4; ++i) printf("1024 - 1024 + 2^-%d: D = %.9g (exact %.9g)\n", 14 + 4 * i, D[(48 + i) * kN], ldexp(1.0, -(14 + 4 * i)));
  }
  // ---- random chains: errors against exact sums
  std::mt19937_64 g(12345);
  for (int S : {1, 4, 13}) {
    for (int dist = 0; dist < 3; ++dist) {
      double worst_sum = 0, worst_max = 0, mean_sum = 0;
      int cnt = 0;
      for (int trial = 0; trial < 8; ++trial) {
        Case c = blank(S);
        std::uniform_real_distribution<float> U(-1.f, 1.f), P(0.f, 1.f);
        for (auto& a : c.A) a = __float2half(dist == 1 ? P(g) : U(g));          // dist 1: nonnegative features
        for (auto& b : c.B) b = __float2half(0.1f * U(g));                        // weights U(-0.1, 0.1)
        for (auto& x : c.C) x = dist == 2 ? 50.f * U(g) : 0.f;                     // dist 2: large accumulator
        std::vector<float> D;
        run(c, D);
        for (int r = 0; r < kM; ++r)
          for (int n = 0; n < kN; ++n) {
            __float128 ex = c.C[r * kN + n], part = ex;
            double sabs = fabs((double)c.C[r * kN + n]), pmax = sabs;
            for (int k = 0; k < 16 * S; ++k) {
              const double p = (double)__half2float(c.A[r * 16 * S + k]) * (double)__half2float(c.B[n * 16 * S + k]);
              ex += (__float128)p;
              part += (__float128)p;
              sabs += fabs(p);
              pmax = fmax(pmax, fabs((double)part));
            }
            const double err = fabs((double)D[r * kN + n] - (double)ex);
            const double u = ldexp(1.0, -24);
            worst_sum = fmax(worst_sum, err / (u * sabs));
            worst_max = fmax(worst_max, err / (u * fmax(pmax, sabs / (16.0 * S + 1))));
            mean_sum += err / (u * sabs);
            ++cnt;
          }
      }
      printf("random S=%2d (K=%3d) dist=%d: max err / (u sum|terms|) = %.3f, mean %.4f; max err / (u max|partial|) = %.3f\n",
             S, 16 * S, dist, worst_sum, mean_sum / cnt, worst_max);
    }
  }
  return 0;
}
