// Probe (not product code): TMEM layout of two tcgen05.mma M=64 tiles at
// lane offsets 0 and 16, and the 16x32bx2 load mapping.
#include <cstdio>
#include <cuda_fp16.h>
#include "../paper_2406_01939_b200/csrc/tc_common.cuh"
using namespace pcd;

__global__ void probe(float* out, float* out2) {
  __shared__ __align__(1024) unsigned char sm[2 * 64 * 16 * 2 + 16 * 16 * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  unsigned char* A0 = sm;
  unsigned char* A1 = sm + 64 * 16 * 2;
  unsigned char* B = sm + 2 * 64 * 16 * 2;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 64 * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;
    *(__half*)(A0 + canon_off(64, r, k)) = __float2half(k == 0 ? (float)(r + 1) : 0.f);
    *(__half*)(A1 + canon_off(64, r, k)) = __float2half(k == 0 ? (float)(100 + r) : 0.f);
  }
  for (int i = tid; i < 16 * 16; i += blockDim.x) {
    const int n = i / 16, k = i % 16;
    *(__half*)(B + canon_off(16, n, k)) = __float2half(k == 0 ? (float)(n + 1) : 0.f);
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
  if (tid == 0) {
    const uint32_t id = idesc_f16(64, 16);
    const uint64_t a0 = umma_desc(smem_u32(A0), 1024, 128), a1 = umma_desc(smem_u32(A1), 1024, 128);
    const uint64_t b = umma_desc(smem_u32(B), 256, 128);
    mma_f16(tm, a0, b, id, 0);
    mma_f16(tm + (16u << 16), a1, b, id, 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  // 32x32b: thread = lane of its subpartition, 16 columns
  {
    float v[16];
    tmem_ld16(tm + ((uint32_t)(32 * warp) << 16), v);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out[(32 * warp + lane) * 16 + c] = v[c];
  }
  // 16x32bx2 at lane offset 32*warp + 16, split offset 8 columns, .x1
  {
    uint32_t r0;
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x1.b32 {%0}, [%1], 8;" : "=r"(r0)
                 : "r"(tm + ((uint32_t)(32 * warp + 16) << 16)));
    tmem_wait_ld();
    out2[warp * 32 + lane] = __uint_as_float(r0);
  }
  // 16x32bx2.x4 at lane base 32*warp, split 8: expect th0 cols 0..3, th1 cols 8..11
  {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], 8;"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(tm + ((uint32_t)(32 * warp) << 16)));
    tmem_wait_ld();
    for (int i = 0; i < 4; ++i) out2[128 + (warp * 32 + lane) * 4 + i] = __uint_as_float(r[i]);
    // store back +1000 with 16x32bx2.x4 at cols 16.., read with 32x32b
    uint32_t w[4];
    for (int i = 0; i < 4; ++i) w[i] = __float_as_uint(__uint_as_float(r[i]) + 1000.f);
    asm volatile("tcgen05.st.sync.aligned.16x32bx2.x4.b32 [%0], 8, {%1,%2,%3,%4};"
                 :: "r"(tm + ((uint32_t)(32 * warp) << 16) + 16), "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    float v[16];
    tmem_ld16(tm + ((uint32_t)(32 * warp) << 16) + 16, v);
    tmem_wait_ld();
    for (int c = 0; c < 16; ++c) out2[128 + 512 + (32 * warp + lane) * 16 + c] = v[c];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(32));
  }
}

int main() {
  float *d, *d2;
  cudaMalloc(&d, 128 * 16 * 4);
  cudaMalloc(&d2, (128 + 512 + 2048) * 4);
  cudaMemset(d, 0, 128 * 16 * 4);
  probe<<<1, 128>>>(d, d2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("err %s\n", cudaGetErrorString(e));
  float h[128 * 16], h2[128 + 512 + 2048];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2, d2, sizeof h2, cudaMemcpyDeviceToHost);
  for (int l = 0; l < 128; ++l) printf("lane %3d: %6.0f %6.0f %6.0f\n", l, h[l * 16], h[l * 16 + 1], h[l * 16 + 2]);
  for (int t = 0; t < 32; t += 7) printf("x4 warp0 thread %d: %.0f %.0f %.0f %.0f\n", t, h2[128 + t * 4], h2[128 + t * 4 + 1], h2[128 + t * 4 + 2], h2[128 + t * 4 + 3]);
  for (int l = 0; l < 32; l += 5) { printf("st lane %d:", l); for (int c = 0; c < 16; ++c) printf(" %.0f", h2[640 + l * 16 + c]); printf("\n"); }
  for (int w = 0; w < 4; ++w) {
    printf("16x32bx2 warp %d:", w);
    for (int t = 0; t < 32; ++t) printf(" %.0f", h2[w * 32 + t]);
    printf("\n");
  }
  return 0;
}
