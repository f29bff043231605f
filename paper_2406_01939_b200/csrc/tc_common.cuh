// tc_common.cuh — shared pieces of the tcgen05/TMEM tensor-core sweep
// (tc_pp.cu) for run partitions: constants, weight-image layout, PTX glue.
//
// Every step, each row (process) evaluates the dual-price MLP
// (policies.hpp:121-168) at its next own slot; the three layers run as
// tcgen05.mma.kind::f16 GEMMs over 64-row tiles
//   z1 = F[64 x 208] . W1^T[208 x 64]        (features c/c0, x/x0, t/T)
//   z2 = tanh(z1+b1)[64 x 64] . W2^T         (64 x 64)
//   q  = tanh(z2+b2)[64 x 64] . W3'^T        (64 x N3), W3' = W3[:J] + W3[J:]
// with operands split into fp16 hi + (scaled) lo parts and three products
// (hi.hi + hi.lo + lo.hi) accumulated in fp32 TMEM (two accumulators so the
// 2^-11-scaled cross terms keep full precision): ~2^-22 relative per product.
// score_j = r_j - q_j needs only the SUM of the two prices, hence W3'.
//
// Exactness: the tensor-core argmax is accepted only when its decision
// margins (best - second best >= guard, |best| >= guard_abs vs the decline
// score 0) clear guards derived a priori from the policy's weights and the
// measured tcgen05 / MUFU error behaviour (engine.cu tc_error_bound,
// DESIGN.md §4.3a); otherwise the row is re-evaluated with the exact FP64
// path (bit-identical to the reference). The state of each row is the
// run-partition closed form, identical to k_sweep_product.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>
#include <cstdint>

#include "kernels.cuh"

namespace pcd {

constexpr int kTcRows = 128;
constexpr int kTcStats = 6;  // TcArgs::stats entries
// speculation queue entry: [0] t, [1] pos, [2] first window pos, [3] end pos
// (indices into pslots), [4] process, [5] run, [6] product, [7] reward row,
// [8] order time, [9] the speculated decision
constexpr int kSpecStride = 12;
constexpr int kTcK1 = 208;     // 2J+1 <= 208 (J <= 103)
constexpr int kTcH = 64;
constexpr int kTcN3 = 112;     // J <= 112
constexpr float kLoScale = 2048.f;          // lo parts are stored * 2^11
constexpr float kLoInv = 1.f / 2048.f;

// smem image layout of the weights (bytes), canonical K-major no-swizzle:
//   off(r,k) = (k/8)*16*R + (r/8)*128 + (r%8)*16 + (k%8)*2
constexpr int kW1Bytes = kTcH * kTcK1 * 2;   // one of hi / lo
constexpr int kW2Bytes = kTcH * kTcH * 2;
constexpr int kW3Bytes = kTcN3 * kTcH * 2;
constexpr int kWImgBytes = 2 * (kW1Bytes + kW2Bytes + kW3Bytes);
constexpr int kWImgRows = kWImgBytes / 256;  // TMA view of the image: [kWImgRows][128] fp16
static_assert(kWImgBytes % 512 == 0 && kWImgRows / 2 <= 256, "two TMA boxes of <= 256 rows");

// layer-1 operand columns: capacities at [0, J), zero padding to RJ = J
// rounded up to 8 (every capacity 8-column chunk is whole, so a row's
// capacity slots can take the prefetched checkpoint row, tc_pp.cu), inventory
// features at [RJ, RJ + J), the time feature at RJ + J
__host__ __device__ constexpr int tc_rj(int J) { return (J + 7) & ~7; }
__host__ __device__ constexpr int tc_k1_needed(int J) { return tc_rj(J) + J + 1; }
// reference input index (MlpParams::forward's order: c/c0, x/x0, t/T) of a
// layer-1 operand column, or -1 for a zero column
__host__ __device__ constexpr int tc_l1_input(int k, int J) {
  return k < J ? k : k < tc_rj(J) ? -1 : k < tc_rj(J) + J ? J + (k - tc_rj(J)) : k == tc_rj(J) + J ? 2 * J : -1;
}

__host__ __device__ constexpr int canon_off(int R, int r, int k) {
  return (k >> 3) * 16 * R + (r >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2;
}

struct TcArgs {
  SweepArgs s;          // state, publish and counter pointers (as k_sweep_product)
  const int* wq;        // work list: processes with window slots, heaviest first
  int* wctl;            // {entries of wq, next entry beyond the dealt ones}
  const int* wbeg;      // [M] first window position of each process in pslots (k_window_load)
  const int* wlen;      // [M] its window slot count
  const unsigned char* wimg2; // kWImgBytes: per layer one 2N-row K-major operand [hi; lo]
  int n3;                     // layer-3 width class (tc_pp_width_class(J))
  const float* b1f;     // [64]
  const float* b2f;     // [64]
  const float* inv_c0;  // [J]
  const float* inv_x0;  // [I*J]
  const float* rtabq;   // [R*J] rewards minus the combined output bias b3[:J] + b3[J:], in fp32
  float guard;          // decision margin (best - second) below which a row is re-evaluated
  float guard_abs;      // |best| (vs the decline score 0) below which a row is re-evaluated
  const float* gnode;   // or per best node j: [j] margin and [kTcN3 + j] |best| thresholds (<= the above)
  int verify;           // debug: exact re-evaluation of every row
  // speculation: a row whose margins lie between spec_floor (1/256) of the
  // guards and the guards takes the tensor-core decision at once and is queued
  // for the post-sweep verification (tc_spec.cu); rows below are re-evaluated
  // in the sweep. spec == 0: every row within the guard is re-evaluated there.
  int spec;
  float spec_floor;     // speculate above this fraction of the guards
  int spec_flip;        // debug: publish wrong speculated decisions (the verification must catch them)
  int spec_cap;         // entries of spec_q
  int* spec_n;          // queued entries (atomic)
  int* spec_q;          // [spec_cap][kSpecStride]
  long long* prof;      // debug: per-phase clock64 totals of CTA 0 (or nullptr)
  unsigned long long* stats;  // [0] tc rows, [1] flagged, [2] flagged & tc wrong,
                              // [3] (verify) unflagged & tc wrong -- must stay 0,
                              // [4] (verify) max |score_tc - score_exact| over
                              //     feasible nodes of re-evaluated rows (float bits),
                              // [5] speculated rows
};

// tc_inc.cu: the sweep with layer 1 off the tensor cores (nodes J <= kIncMaxJ)
constexpr int kIncMaxJ = 104;
struct IncArgs {
  TcArgs t;           // everything the ping-pong sweep takes (its layer-2/3 weight image is reused)
  const float* af;    // [J][64] A_j = W1[:, j] / c0_j (capacity weights over the normaliser)
  const float* wx;    // [J][64] W1[:, J + j] (inventory weights)
  const float* wt;    // [64]    W1[:, 2J] (time weight)
  const int* tau;     // [J] death slot of every node under the frozen cache (k_tau)
  const int* bA;      // [J] first block at which node j is no longer alive-far (k_trans)
  const int* bD;      // [J] first block at which node j is dead-far (k_trans)
};
struct IncPrep {      // per-iteration G rows and node transition blocks
  const int* hck;
  const int* ev;
  const int* tau;
  const int* ckcap;
  const double* a64;  // [J][64] A_j in FP64
  const double* b1;   // [64]
  const int* wload_sorted;  // [0] = the largest window load of this rank's processes
  int lo, hi, J, nb;
  float* grow;        // [nb][64]
  int* bA;
  int* bD;
};

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity));
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// TMA: arm an mbarrier for `bytes` of transaction, then a 2-D tensor tile
// (cp.async.bulk.tensor, SASS UTMALDG) or a plain bulk copy (UBLKCP) that
// completes on it
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const void* tmap, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// 4-byte async global -> shared copy (LDGSTS), completed by this thread's wait
__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// named barrier over `count` threads that also returns how many of them passed pred
__device__ __forceinline__ int bar_red_popc(int id, int count, bool pred) {
  int r;
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %3, 0;\n\tbarrier.red.popc.u32 %0, %1, %2, p;\n\t}"
               : "=r"(r)
               : "r"(id), "r"(count), "r"((int)pred)
               : "memory");
  return r;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm_100)
  return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  // c_format=F32 (bit 4), a/b format F16 (0), K-major A/B, N>>3 @17, M>>4 @24
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float exp2f_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256)

// 256-bit read-only loads (sm_100: LDG.E.ENL2.256) of streamed checkpoint
// rows / event blocks, not allocated in L1 and streamed through L2 with evict_first priority (read ~once per iteration;
// keeps the hot small tables — FP64 weights, run inventories — resident)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void ldg256_na_ef(const void* p, uint32_t* r, uint64_t pol) {
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p), "l"(pol));
}
__device__ __forceinline__ double ldg_f64_el(const double* p, uint64_t pol) {
  double v;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
  return v;
}
// ... kept in L1 (the reward table, re-read by every step)
__device__ __forceinline__ void ldg256_el(const void* p, uint32_t* r) {
  asm volatile("ld.global.nc.L1::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "l"(p));
}

__device__ __forceinline__ void split_f16(float x, __half& hi, __half& lo) {
  hi = __float2half_rn(x);
  lo = __float2half_rn((x - __half2float(hi)) * kLoScale);
}


inline float __uint_as_float_host(uint32_t b) {
  float f;
  __builtin_memcpy(&f, &b, 4);
  return f;
}

__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 hh = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(hh);
  const __half2 l = __floats2half2_rn((x0 - hf.x) * kLoScale, (x1 - hf.y) * kLoScale);
  hi = *(const uint32_t*)&hh;
  lo = *(const uint32_t*)&l;
}
// tanh(z) = 1 - 2/(1 + e^{2z}): MUFU ex2 and rcp; max |tanh_mufu(z) - tanh(z)|
// over every float is 3.97 * 2^-24 (tools/tanh_mufu_probe.cu), the kTanhErr
// of the derived guard (engine.cu tc_error_bound). Weights are finite (the
// tensor-core path is refused otherwise), so z is finite and the clamp at
// +-9 costs < 2^-24.
__device__ __forceinline__ float tanh_mufu(float z) {
  z = fminf(fmaxf(z, -9.f), 9.f);
  const float d = 1.f + exp2f_approx(2.8853900817779268f * z);
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(d));
  return fmaf(-2.f, y, 1.f);
}

}  // namespace pcd
