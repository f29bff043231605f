// tc_inc.cu — the tcgen05 run-partition sweep with layer 1 OFF the per-step
// tensor-core path ("incremental layer 1").
//
// The dual network's first layer is affine in the features,
//   z1 = b1 + sum_j A_j c_j + sum_j W1x_j x_pj / x0_pj + w_t t / T,   A_j = W1[:, j] / c0_j,
// and the row state is the run-partition closed form
//   c_j = max(0, U_t[j] + D_j),  U_t[j] = ckcap[j] - H_t[j]  (process-independent),
//   D_j = Hown_j - F_j  (the row's own deltas, |D_j| <= L = its window load).
// Hence sum_j A_j c_j = G_t + sum_j A_j (max(0, U_t + D_j) - max(0, U_t)) with
// the process-independent G_t = sum_j A_j max(0, U_t[j]). Per iteration
// k_grows builds G_b (b1 folded in) for every 8-slot block b of the window in
// FP64 (stored fp32), and each row keeps
//   acc = sum_{j alive-far} A_j D_j + sum_j W1x_j x_pj / x0_pj      (FP64, per row, incremental)
// where node j is "alive-far" at block b while U_b[j] > V = Lmax + 7 (then the
// clamp term is exactly D_j), "dead-far" once U_b[j] <= -Lmax (term 0, c = 0)
// and "near" in between (term computed exactly from hck). One step is then:
//   F': wait for the TMA-fed G_b row + event block of the step (issued one step
//       ahead), apply the previous step's two D / one x deltas to acc, process
//       the node transitions of the new block, subtract the <= 7 partial-block
//       events from G (G_t), add the near-node terms, z1 -> tanh -> fp16 hi/lo
//   L2 / E2 / L3 on tcgen05 (fp16x3 split, fp32 TMEM accumulators) as tc_pp.cu
//   S: scores, argmax, decision margin; the guard / exact FP64 recheck as tc_pp.cu
//   U: publish, D / x deltas, next step's TMA.
// Per step the row touches 256 + 32 bytes of prefetched smem instead of the
// 416-byte prefix row, and layer 1's K = 208 MMA (26 instructions) and its
// feature build are gone. Thread / TMEM mapping as tc_pp.cu (two 64-row
// halves per CTA; a row's four threads own hidden units 8g.., 8(g+4).. and
// node chunks g, g+4, g+8, g+12).
#include <cuda.h>
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>

#include "tc_common.cuh"
#include "tc_recheck.cuh"

namespace pcd {
namespace inc {

constexpr int kBlock = 512;
constexpr int kHalfRows = 64;
constexpr int kHalfThreads = 256;
constexpr int kMaxJ = kIncMaxJ;  // 112
constexpr int kMaxCI = 4;        // node chunks per thread
constexpr uint32_t kTmemCols = 512, kColL2 = 0, kColL3 = 128;
constexpr int kAH = kHalfRows * kTcH * 2;   // one of hi / lo of a half's K = 64 operand (8 KB)
constexpr int kChunkB = kHalfRows * 8 * 2;  // bytes per k-chunk of a half's operand
constexpr int kWBytes = 2 * kW2Bytes + 2 * kW3Bytes;
constexpr int kInfo = 40;

enum {
  RI_T = 0, RI_P, RI_POS, RI_END, RI_ANY, RI_DEC, RI_FLAG, RI_RR, RI_TN, RI_XDIRTY, RI_OT, RI_EVT, RI_X, RI_M,
  RI_DRESET, RI_XUPD, RI_GPH, RI_GCNT, RI_B,
  RI_UEV, RI_UOLD, RI_UWR, RI_UREF, RI_UPN, RI_URRN, RI_UOTN, RI_UTNN, RI_UXN,
  RI_EV0  // 8 ints: the step's event block (the smem copy is refilled by the next step's TMA)
};
static_assert(RI_EV0 + 8 <= kInfo, "per-row state fits");
enum { CT_FLAG = 66, CT_DIS, CT_BAD, CT_QACT, kCtl = 80 };

struct Layout {
  static constexpr int g = 0;                                    // [128][64] fp32 G rows (TMA, 256 B each)
  static constexpr int w = g + kTcRows * kTcH * 4;               // layers 2 / 3 weight image
  static constexpr int a = w + kWBytes;                          // half h: hi at a + 2h kAH, lo + kAH
  static constexpr int af = a + 4 * kAH;                         // [kMaxJ][64] fp32 A_j
  static constexpr int wx = af + kMaxJ * kTcH * 4;               // [kMaxJ][64] fp32 W1[:, J + j]
  static constexpr int d = wx + kMaxJ * kTcH * 4;                // [128][kMaxJ] int16 D
  static constexpr int ev = d + kTcRows * kMaxJ * 2;             // [128][8] event blocks (bulk copies)
  static constexpr int ix = ev + kTcRows * 8 * 4;                // [128][4] 16-byte chunk holding 1/x0 of the last decision
  static constexpr int info = ix + kTcRows * 4 * 4;              // [128][kInfo]
  static constexpr int best = info + kTcRows * kInfo * 4;        // [128][4 groups][3]
  static constexpr int ck = best + kTcRows * 12 * 4;             // ckcap[112] tau[112] Ab Aj Db Dj [112]
  static constexpr int wt = ck + 6 * kMaxJ * 4;                  // w_t[64] b2[64]
  static constexpr int ctl = wt + 2 * kTcH * 4;                  // 2 x kCtl
  static constexpr int prof = ctl + 2 * kCtl * 4;                // debug phase clocks [20]
  static constexpr int bar = prof + 20 * 8;                      // MMA mbarrier per half, setup mbarrier
  static constexpr int rbar = bar + 4 * 8;                       // one TMA mbarrier per row
  static constexpr int tmem = rbar + kTcRows * 8;
  static constexpr int total = tmem + 16;
};
static_assert(Layout::total <= 232448, "incremental sweep shared memory budget");
static_assert(Layout::w % 1024 == 0 && Layout::a % 1024 == 0 && Layout::af % 16 == 0 && Layout::ev % 16 == 0 &&
                  Layout::info % 16 == 0 && Layout::prof % 8 == 0 && Layout::bar % 8 == 0,
              "aligned smem regions");
static_assert(rc::kRcVec * 8 <= kAH && (2 * kMaxJ + 3) * 4 <= kAH, "recheck scratch fits the half's operand");

__device__ __forceinline__ int kc64(int k) { return (k >> 3) * kChunkB + (k & 7) * 2; }
__device__ __forceinline__ int ro64(int r) { return (r >> 3) * 128 + (r & 7) * 16; }
__device__ __forceinline__ void bar_half(int h) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(kHalfThreads) : "memory");
}
__device__ __forceinline__ void ld8s(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], 8;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ bool bit128(const uint32_t* m, int j) { return (m[j >> 5] >> (j & 31)) & 1u; }

// ---------------------------------------------------------------------------
// Per-iteration prep. G rows: one CTA of 64 threads (one per hidden unit) per
// segment of 64 blocks; G at the segment's first block from its prefix row
// (FP64 GEMV), then block by block, subtracting A_j for every event that still
// finds node j stocked (slot < tau[j]).
constexpr int kGSeg = 64;
static __global__ void __launch_bounds__(64) k_grows(const int* __restrict__ hck, const int* __restrict__ ev,
                                                     const int* __restrict__ tau, const int* __restrict__ ckcap,
                                                     const double* __restrict__ a64, const double* __restrict__ b1,
                                                     int lo, int hi, int J, int nb, float* __restrict__ grow) {
  __shared__ int sev[kGSeg * kK];
  __shared__ int stau[kMaxJ];
  const int u = threadIdx.x, b0 = blockIdx.x * kGSeg, HJ = hck_stride(J), base = hck_base(lo);
  const int nblk = min(kGSeg, nb - b0);
  for (int j = u; j < J; j += 64) stau[j] = tau[j];
  for (int i = u; i < nblk * kK; i += 64) {
    const int s = base + (b0 << kLogK) + i;
    sev[i] = (s >= lo && s < hi) ? ev[s] : -1;
  }
  double g = b1[u];
  const int* hr = hck + (size_t)b0 * HJ;
  for (int j = 0; j < J; ++j) g += a64[(size_t)j * kTcH + u] * (double)max(0, ckcap[j] - hr[j]);
  __syncthreads();
  for (int r = 0; r < nblk; ++r) {
    grow[(size_t)(b0 + r) * kTcH + u] = (float)g;
    const int sb = base + ((b0 + r) << kLogK);
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const int j = sev[r * kK + k];
      if (j >= 0 && sb + k < stau[j]) g -= a64[(size_t)j * kTcH + u];
    }
  }
}

// Node transition blocks for window load bound L = max load of the rank's
// processes (wload_s[0], sorted descending): bA = first block with
// U_b = ckcap - H_b <= L + 7 (no longer alive-far), bD = first block with
// U_b <= 0 (the node is empty for every row whose D_j <= 0); nb when never.
static __global__ void k_trans(const int* __restrict__ hck, const int* __restrict__ ckcap,
                               const int* __restrict__ wload_sorted, int J, int nb, int* __restrict__ bA,
                               int* __restrict__ bD) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int L = wload_sorted[0], HJ = hck_stride(J), c = ckcap[j];
  auto first_ge = [&](long long thr) {  // first b with hck[b][j] >= thr (hck nondecreasing in b)
    int l = 0, r = nb;
    while (l < r) {
      const int mid = (l + r) >> 1;
      if ((long long)hck[(size_t)mid * HJ + j] >= thr) r = mid; else l = mid + 1;
    }
    return l;
  };
  bA[j] = first_ge((long long)c - L - kK + 1);  // U_b <= L + 7  <=>  H_b >= c - L - 7
  bD[j] = first_ge((long long)c);               // U_b <= 0      <=>  H_b >= c
}

// ---------------------------------------------------------------------------
template <bool PROF, int N3>
__global__ void __launch_bounds__(kBlock, 1) k_sweep_inc(IncArgs x, const __grid_constant__ CUtensorMap gmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const TcArgs& a = x.t;
  const SweepArgs& S = a.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = S.J, lo = S.lo, hi = S.hi;
  const int base = hck_base(lo), HJ = hck_stride(J), RJ = (J + 7) & ~7;
  float* sG = (float*)(smem + Layout::g);
  unsigned char* sW = smem + Layout::w;
  const float* sAf = (const float*)(smem + Layout::af);
  const float* sWx = (const float*)(smem + Layout::wx);
  short* sD = (short*)(smem + Layout::d);
  int* sEv = (int*)(smem + Layout::ev);
  float* sIx = (float*)(smem + Layout::ix);
  int* sInfo = (int*)(smem + Layout::info);
  float* sBest = (float*)(smem + Layout::best);
  int* sCk = (int*)(smem + Layout::ck);
  int* sTau = sCk + kMaxJ;
  int* sAb = sTau + kMaxJ;
  int* sAj = sAb + kMaxJ;
  int* sDb = sAj + kMaxJ;
  int* sDj = sDb + kMaxJ;
  float* sWt = (float*)(smem + Layout::wt);
  float* sB2 = sWt + kTcH;
  int* sCtlAll = (int*)(smem + Layout::ctl);
  uint64_t* sBar = (uint64_t*)(smem + Layout::bar);
  uint64_t* sRBar = (uint64_t*)(smem + Layout::rbar);
  uint32_t* sTmem = (uint32_t*)(smem + Layout::tmem);
  const int tile = blockIdx.x;
  const int h = warp >> 3, wq = warp & 7, q = wq & 3, p2 = wq >> 2, th = lane >> 4;
  const int g = 2 * p2 + th;
  const int rr = 16 * q + (lane & 15);
  const int R = kHalfRows * h + rr;
  const bool agent = g == 3;
  const int ht = tid & (kHalfThreads - 1);
  const uint32_t tl = (uint32_t)(32 * q + 16 * h) << 16;
  unsigned char* sAh = smem + Layout::a + 2 * h * kAH;
  int* ctl = sCtlAll + h * kCtl;
  uint64_t* bar = sBar + h;
  const int rowo = ro64(rr);
  const int nchunk = (J + 7) >> 3;
  const int ni = (nchunk - 2 * p2 + 3) >> 2;  // node chunks of this warp pair (warp-uniform)

  // ---------------------------------------------------------------- setup
  if (tid == 0) {  // weights (layers 2 / 3) and the layer-1 tables by bulk copy
    mbar_init(sBar, 1);
    mbar_init(sBar + 1, 1);
    mbar_init(sBar + 2, 1);
    for (int r = 0; r < kTcRows; ++r) mbar_init(sRBar + r, 2);  // G row + event block, 1/x0 chunk
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t tb = (uint32_t)J * kTcH * 4;
    mbar_expect_tx(sBar + 2, (uint32_t)kWBytes + 2 * tb);
    bulk_load(sW, a.wimg2 + 2 * kW1Bytes, kWBytes, sBar + 2);
    bulk_load(smem + Layout::af, x.af, tb, sBar + 2);
    bulk_load(smem + Layout::wx, x.wx, tb, sBar + 2);
  }
  for (int j = tid; j < kMaxJ; j += kBlock) {
    sCk[j] = j < J ? S.ckcap[j] : 0;
    sTau[j] = j < J ? x.tau[j] : INT_MAX;
  }
  if (tid < J) {  // transition lists sorted by block (ties by node)
    const int ba = x.bA[tid], bd = x.bD[tid];
    int ra = 0, rd = 0;
    for (int k = 0; k < J; ++k) {
      const int ka = x.bA[k], kd = x.bD[k];
      ra += ka < ba || (ka == ba && k < tid);
      rd += kd < bd || (kd == bd && k < tid);
    }
    sAb[ra] = ba; sAj[ra] = tid;
    sDb[rd] = bd; sDj[rd] = tid;
  }
  for (int i = tid; i < kTcH; i += kBlock) {
    sWt[i] = x.wt[i];
    sB2[i] = a.b2f[i];
  }
  const int nq = a.wctl[0], dealt = (int)gridDim.x * kTcRows;
  __syncthreads();  // mbarriers initialised before any TMA below
  // start a process on this row: window range, first step, its TMA
  auto begin_proc = [&](int* inf, int m) {
    int pos = 0, end = 0;
    if (m >= 0) {
      const int beg = S.pstart[m], n = S.pstart[m + 1] - beg;
      pos = beg + lower_bound_i32(S.pslots + beg, n, lo);
      end = beg + lower_bound_i32(S.pslots + beg, n, hi);
    }
    inf[RI_M] = m;
    inf[RI_POS] = pos;
    inf[RI_END] = end;
    inf[RI_XDIRTY] = 1;
    inf[RI_XUPD] = -1;
    inf[RI_EVT] = -1;
    inf[RI_DRESET] = 1;
    inf[RI_P] = -1;
    inf[RI_X] = -1;
    if (pos < end) {
      const int t = S.pslots[pos];
      inf[RI_T] = t;
      inf[RI_P] = S.model.product[t];
      inf[RI_X] = S.rid[t];
      inf[RI_RR] = S.model.rrow[t];
      inf[RI_OT] = S.model.order_t ? S.model.order_t[t] : t;
      inf[RI_TN] = pos + 1 < end ? S.pslots[pos + 1] : -1;
      const int b = (t - base) >> kLogK, r = (int)(inf - sInfo) / kInfo;
      fence_async_smem();
      mbar_expect_tx(sRBar + r, kTcH * 4 + kK * 4);
      tma_load_2d(sG + r * kTcH, &gmap, 0, b, sRBar + r);
      bulk_load(sEv + r * kK, S.ev + base + (b << kLogK), kK * 4, sRBar + r);
      mbar_arrive(sRBar + r);  // (no inventory delta before a process's first step)
      inf[RI_GPH] = inf[RI_GCNT] & 1;
      inf[RI_GCNT] += 1;
    }
  };
  auto next_entry = [&]() -> int {
    const int k = dealt + atomicAdd(&a.wctl[1], 1);
    return k < nq ? a.wq[k] : -1;
  };
  if (agent) {
    const int k = R * (int)gridDim.x + tile;
    sInfo[R * kInfo + RI_GCNT] = 0;
    begin_proc(sInfo + R * kInfo, k < nq ? a.wq[k] : -1);
  }
  for (int i = tid; i < 2 * kCtl; i += kBlock) sCtlAll[i] = 0;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  mbar_wait(sBar + 2, 0);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  const uint32_t tD = tmem + ((uint32_t)(16 * h) << 16);  // MMA accumulator base of the half

  const uint32_t aBase = smem_u32(sAh);
  const uint32_t w2 = smem_u32(sW), w3 = w2 + 2 * kW2Bytes;
  const uint32_t id64 = idesc_f16(64, 64), id128 = idesc_f16(64, 128);
  const uint32_t idn3 = idesc_f16(64, N3), id2n3 = idesc_f16(64, 2 * N3);
  uint32_t phase = 0;
  const float invT = S.model.horizon > 0 ? (float)(1.0 / (double)S.model.horizon) : 0.f;
  const uint64_t ldpol = l2_policy_evict_last();

  // per-row incremental state (identical in the row's four threads)
  double acc[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) acc[k] = 0.0;
  uint32_t nA[4] = {0, 0, 0, 0}, nD[4] = {0, 0, 0, 0};  // nodes past their alive-far / stocked (U_b > 0) block
  uint32_t Dp[4] = {0, 0, 0, 0};                        // nodes with D_j > 0 (can be stocked for this row only)
  int cA = 0, cD = 0;
  uint32_t xb = 0;  // x > 0 bits of the thread's score nodes (bit 8i + k: node 8(g + 4i) + k)
  // agent: the row's counters (changed, conflicts, first changed, mismatch delta, evaluations, tc rows)
  int cn_changed = 0, cn_conflicts = 0, cn_first = INT_MAX, cn_mism = 0, cn_nev = 0, cn_tc = 0;

  long long* pacc = (long long*)(smem + Layout::prof);
  if (PROF && tid == 0)
    for (int k = 0; k < 20; ++k) pacc[k] = 0;
  long long plast = PROF ? clock64() : 0;
  const bool prof_on = PROF && blockIdx.x == 0 && tid == 0;
#define PMARK(k) do { if (PROF && prof_on) { const long long now_ = clock64(); if (pacc[16] <= 2) pacc[k] += now_ - plast; plast = now_; } } while (0)

  // acc[k] += s * tab[j][unit k] over the thread's 16 units (8g.., 8(g+4)..)
  auto acc_add = [&](const float* tab, int j, double s) {
    const float4* r = (const float4*)(tab + j * kTcH);
    const float4 v0 = r[2 * g], v1 = r[2 * g + 1], v2 = r[2 * g + 8], v3 = r[2 * g + 9];
    const float v[16] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w,
                         v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = fma((double)v[k], s, acc[k]);
  };
  auto issue_layer = [&](uint32_t accc, uint32_t N, uint32_t wb, int ks0, int ks1, uint32_t idfull, uint32_t idhalf,
                         bool commit) {
    tc_fence_after();
    const uint64_t dA = umma_desc(aBase, kHalfRows * 16, 128), dAl = umma_desc(aBase + kAH, kHalfRows * 16, 128);
    const uint64_t dW = umma_desc(wb, 2 * N * 16, 128);
    for (int s = ks0; s < ks1; ++s) {
      const uint64_t ah = dA + s * ((2 * kChunkB) >> 4), al = dAl + s * ((2 * kChunkB) >> 4);
      const uint64_t b = dW + s * ((4 * N * 16) >> 4);
      mma_f16(tD + accc, ah, b, idfull, s > 0);
      mma_f16(tD + accc + N, al, b, idhalf, 1);
    }
    if (commit) mma_commit(bar);
  };
  auto wait_mma = [&]() {
    mbar_wait(bar, phase);
    phase ^= 1;
    tc_fence_after();
  };

  for (;;) {
    int* inf = sInfo + R * kInfo;
    const bool act = inf[RI_POS] < inf[RI_END];
    // ============================ F': z1 from G, the row accumulator and corrections
    uint32_t capok = 0;  // capacity > 0 bits of the thread's score nodes
    if (agent && act) {  // operands of this row's update (U): async copies into its info row
      const int t = inf[RI_T], pos = inf[RI_POS], end = inf[RI_END], tn = inf[RI_TN];
      cp_async4(inf + RI_UEV, S.ev + t);
      cp_async4(inf + RI_UOLD, S.cache + t);
      cp_async4(inf + RI_UWR, (const int*)(S.written + (t & ~3)));  // byte t & 3 of the word
      if (S.ref) cp_async4(inf + RI_UREF, S.ref + t);
      if (tn >= 0) {
        cp_async4(inf + RI_UPN, S.model.product + tn);
        cp_async4(inf + RI_UXN, S.rid + tn);
        cp_async4(inf + RI_URRN, S.model.rrow + tn);
        if (S.model.order_t) cp_async4(inf + RI_UOTN, S.model.order_t + tn);
        else inf[RI_UOTN] = tn;
      } else {
        inf[RI_UPN] = -1;
        inf[RI_UXN] = -1;
      }
      if (pos + 2 < end) cp_async4(inf + RI_UTNN, S.pslots + pos + 2);
      else inf[RI_UTNN] = -1;
      cp_async_commit();
    }
    if (act) {
      const int t = inf[RI_T], b = (t - base) >> kLogK, p = inf[RI_P];
      const bool dres = inf[RI_DRESET] != 0, dirty = inf[RI_XDIRTY] != 0;
      const short* Drow = sD + R * kMaxJ;
      if (dres) {
#pragma unroll
        for (int w = 0; w < 4; ++w) { nA[w] = 0; nD[w] = 0; Dp[w] = 0; }
        cA = 0;
        cD = 0;
      } else {  // the previous step's deltas (D: +evt, -dec; x: -1 at dec), status at its block
        const int evt = inf[RI_EVT], dec = inf[RI_XUPD];
        auto dpos = [&](int j) {
          const uint32_t m = 1u << (j & 31);
          Dp[j >> 5] = Drow[j] > 0 ? (Dp[j >> 5] | m) : (Dp[j >> 5] & ~m);
        };
        if (evt >= 0) dpos(evt);
        if (dec >= 0) dpos(dec);
        if (!dirty) {
          if (evt >= 0 && !bit128(nA, evt)) acc_add(sAf, evt, 1.0);
          if (dec >= 0 && !bit128(nA, dec)) acc_add(sAf, dec, -1.0);
        }
      }
      while (cA < J && sAb[cA] <= b) {  // alive-far -> near: its linear term leaves acc
        const int j = sAj[cA++];
        if (!dres && !dirty) {
          const int dj = Drow[j];
          if (dj) acc_add(sAf, j, -(double)dj);
        }
        nA[j >> 5] |= 1u << (j & 31);
      }
      while (cD < J && sDb[cD] <= b) {
        const int j = sDj[cD++];
        nD[j >> 5] |= 1u << (j & 31);
      }
      mbar_wait(sRBar + R, (uint32_t)inf[RI_GPH]);
      if (!dirty) {
        const int dec = inf[RI_XUPD];
        if (dec >= 0) acc_add(sWx, dec, -(double)sIx[R * 4 + (int)(((size_t)p * J + dec) & 3)]);
      }
      PMARK(11);
      if (dirty) {  // process / run start: acc from the row's D and the run's inventory
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = 0.0;
        if (!dres)
          for (int j = 0; j < J; ++j) {
            const int dj = Drow[j];
            if (dj && !bit128(nA, j)) acc_add(sAf, j, (double)dj);
          }
        const int* xr = S.xloc + (size_t)inf[RI_X] * J;
        const float* ix = a.inv_x0 + (size_t)p * J;
        uint32_t nb2 = 0;
        for (int j0 = 0; j0 < J; j0 += 16) {  // 32 loads in flight per round
          int xv[16];
          float iv[16];
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            xv[k] = j0 + k < J ? __ldcg(xr + j0 + k) : 0;
            iv[k] = j0 + k < J ? __ldg(ix + j0 + k) : 0.f;
          }
#pragma unroll
          for (int k = 0; k < 16; ++k)
            if (xv[k]) acc_add(sWx, j0 + k, (double)xv[k] * (double)iv[k]);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int jc = j0 + 8 * hh;
            if (((jc >> 3) & 3) == g) {
              uint32_t bb = 0;
#pragma unroll
              for (int k = 0; k < 8; ++k) bb |= (xv[8 * hh + k] > 0 ? 1u : 0u) << k;
              nb2 |= bb << (8 * (jc >> 5));
            }
          }
        }
        xb = nb2;
        if (dres)  // this row's D restarts from 0 (the U phase below is the first writer)
          for (int j = g; j < kMaxJ; j += 4) sD[R * kMaxJ + j] = 0;
      }
      PMARK(12);
      // partial block [max(lo, 8b), t): G_t = G_b - A_j for events that still find j stocked
      float corr[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) corr[k] = 0.f;
      auto corr_add = [&](int j, float s) {
        const float4* r = (const float4*)(sAf + j * kTcH);
        const float4 v0 = r[2 * g], v1 = r[2 * g + 1], v2 = r[2 * g + 8], v3 = r[2 * g + 9];
        const float v[16] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w,
                             v2.x, v2.y, v2.z, v2.w, v3.x, v3.y, v3.z, v3.w};
#pragma unroll
        for (int k = 0; k < 16; ++k) corr[k] = fmaf(v[k], s, corr[k]);
      };
      const int bs = base + (b << kLogK), k0 = max(lo, bs) - bs, k1 = t - bs;
      const int* evb = sEv + R * kK;
      for (int k = k0; k < k1; ++k) {
        const int j = evb[k];
        if (j >= 0 && bs + k < sTau[j]) corr_add(j, -1.f);
      }
      // near nodes: the exact clamp term and capacity
      uint32_t nok[4] = {0, 0, 0, 0};
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        uint32_t m = (nA[w] & ~nD[w]) | (nD[w] & Dp[w]);  // near the clamp, or revived by this row's D
        while (m) {
          const int j = 32 * w + __ffs(m) - 1;
          m &= m - 1;
          if (PROF && prof_on) pacc[14] += 1;
          int part = 0;
          for (int k = k0; k < k1; ++k) part += evb[k] == j;
          const int U = sCk[j] - __ldg(S.hck + (size_t)b * HJ + j) - part;
          const int e = dres ? 0 : (int)Drow[j];
          const int cn = max(0, U + e), c0 = max(0, U);
          if (cn != c0) corr_add(j, (float)(cn - c0));
          if (cn > 0) nok[w] |= 1u << (j & 31);
        }
      }
#pragma unroll
      for (int i = 0; i < kMaxCI; ++i) {  // alive-far nodes, or near with c > 0
        const uint32_t by = ((~nA[i] | nok[i]) >> (8 * g)) & 0xffu;
        capok |= by << (8 * i);
      }
      PMARK(13);
      // z1 -> tanh -> the layer-2 operand
      const float tf = (float)inf[RI_OT] * invT;
      const float* grow = sG + R * kTcH;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int u0 = 8 * (g + 4 * c);
        const float4 g0 = *(const float4*)(grow + u0), g1 = *(const float4*)(grow + u0 + 4);
        const float4 w0 = *(const float4*)(sWt + u0), w1 = *(const float4*)(sWt + u0 + 4);
        const float gv[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
        const float wv[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
        uint32_t ph[4], pl[4];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const float z0 = fmaf(wv[k], tf, (gv[k] + (float)acc[8 * c + k]) + corr[8 * c + k]);
          const float z1 = fmaf(wv[k + 1], tf, (gv[k + 1] + (float)acc[8 * c + k + 1]) + corr[8 * c + k + 1]);
          split2(tanh_mufu(z0), tanh_mufu(z1), ph[k / 2], pl[k / 2]);
        }
        const int off = rowo + kc64(u0);
        *(uint4*)(sAh + off) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
        *(uint4*)(sAh + kAH + off) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
      }
      if (agent) {  // keep the step's event block (the smem copy is refilled by the next TMA)
        const int4 e0 = *(const int4*)evb, e1 = *(const int4*)(evb + 4);
        *(int4*)(inf + RI_EV0) = e0;
        *(int4*)(inf + RI_EV0 + 4) = e1;
        inf[RI_B] = b;
      }
    }
    if (p2 == 0) {
      const uint32_t bal = __ballot_sync(0xffffffffu, act) & 0xffffu;
      if (lane == 0) {
        ctl[CT_QACT + q] = bal != 0;
        if (bal) atomicAdd(&ctl[0], __popc(bal));
      }
    }
    tc_fence_before();
    fence_async_smem();
    bar_half(h);  // ---- B1: the layer-2 operand is published
    PMARK(0);
    if (ctl[0] == 0) break;
    if (PROF && prof_on) {  // per-step trace: rows active in the half, cycles since the last step
      const long long k = pacc[10], now = clock64();
      if (k > 0 && k <= 4096) { a.prof[20 + 2 * (k - 1)] = pacc[16]; a.prof[20 + 2 * (k - 1) + 1] = now - pacc[17]; }
      pacc[16] = ctl[0];
      pacc[17] = now;
      pacc[10] += 1;
    }
    if (ht == 0) issue_layer(kColL2, kTcH, w2, 0, kTcH / 16, id128, id64, true);
    if (ht == kHalfThreads - 1) ctl[1] = 0;
    if (agent && act && inf[RI_POS] + 1 < inf[RI_END]) {  // the next step's G row and event block
      const int bn = (inf[RI_TN] - base) >> kLogK;
      fence_async_smem();
      mbar_expect_tx(sRBar + R, kTcH * 4 + kK * 4);
      tma_load_2d(sG + R * kTcH, &gmap, 0, bn, sRBar + R);
      bulk_load(sEv + R * kK, S.ev + base + (bn << kLogK), kK * 4, sRBar + R);
      inf[RI_GPH] = inf[RI_GCNT] & 1;
      inf[RI_GCNT] += 1;
    }
    const bool qact = ctl[CT_QACT + q] != 0;  // warp-uniform: skip idle row quarters
    wait_mma();
    PMARK(1);

    // ============================ E2: h2 = tanh(z2 + b2); layer 3's first k-steps after the first chunk
    auto hidden_part = [&](int i) {
      if (!qact) return;
      uint32_t vh[8], vx[8];
      ld8s(tmem + tl + kColL2 + 16 * p2 + 32 * i, vh);
      ld8s(tmem + tl + kColL2 + kTcH + 16 * p2 + 32 * i, vx);
      tmem_wait_ld();
      const int u0 = 8 * (g + 4 * i);
      uint32_t ph[4], pl[4];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const float z0 = fmaf(__uint_as_float(vx[k]), kLoInv, __uint_as_float(vh[k])) + sB2[u0 + k];
        const float z1 = fmaf(__uint_as_float(vx[k + 1]), kLoInv, __uint_as_float(vh[k + 1])) + sB2[u0 + k + 1];
        split2(tanh_mufu(z0), tanh_mufu(z1), ph[k / 2], pl[k / 2]);
      }
      const int off = rowo + kc64(u0);
      *(uint4*)(sAh + off) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
      *(uint4*)(sAh + kAH + off) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
    };
    hidden_part(0);
    tc_fence_before();
    fence_async_smem();
    bar_half(h);
    if (ht == 0) issue_layer(kColL3, N3, w3, 0, 2, id2n3, idn3, false);  // k-steps 0-1 (units 0-31)
    tc_fence_after();
    hidden_part(1);
    tc_fence_before();
    fence_async_smem();
    bar_half(h);  // ---- B2
    PMARK(2);
    if (ht == 0) issue_layer(kColL3, N3, w3, 2, kTcH / 16, id2n3, idn3, true);
    // feasibility: capacity bits from F', inventory bits (the previous decision's node)
    uint32_t fmask = act ? capok & xb : 0u;
    int xdec = 1, decb = -1;  // the previous decision's node if it is one of this thread's: its inventory now
    if (act && !inf[RI_XDIRTY]) {
      const int dec = inf[RI_XUPD];
      if (dec >= 0 && ((dec >> 3) & 3) == g) {
        decb = 8 * (dec >> 5) + (dec & 7);
        xdec = __ldcg(S.xloc + (size_t)inf[RI_X] * J + dec);  // the agent's RED of the last step is done
      }
    }
    uint32_t rwv[kMaxCI][8];
    {
      const float* rw = a.rtabq + (size_t)(fmask ? inf[RI_RR] : 0) * RJ;
#pragma unroll
      for (int i = 0; i < kMaxCI; ++i) {
        if ((fmask >> (8 * i)) & 0xffu) {
          ldg256_el(rw + 8 * (g + 4 * i), rwv[i]);
        } else {
#pragma unroll
          for (int k = 0; k < 8; ++k) rwv[i][k] = 0u;
        }
      }
    }
    if (decb >= 0 && xdec <= 0) {
      xb &= ~(1u << decb);
      fmask &= ~(1u << decb);
    }
    wait_mma();
    PMARK(3);

    // ============================ S: scores, argmax, margin (row, group)
    {
      float v1 = -INFINITY, v2 = -INFINITY, ssum = 0.f;
      int i1 = -1;
      if (qact) {
#pragma unroll
        for (int i0 = 0; i0 < kMaxCI; i0 += 2) {
          if (i0 >= ni) break;
          uint32_t vh[2][8], vx[2][8];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (i0 + u < ni) {
              ld8s(tmem + tl + kColL3 + 16 * p2 + 32 * (i0 + u), vh[u]);
              ld8s(tmem + tl + kColL3 + N3 + 16 * p2 + 32 * (i0 + u), vx[u]);
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            const int i = i0 + u;
            if (i >= ni) break;
            const int j0 = 8 * (g + 4 * i);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              if (!((fmask >> (8 * i + k)) & 1u)) continue;
              const float qv = fmaf(__uint_as_float(vx[u][k]), kLoInv, __uint_as_float(vh[u][k]));
              const float sc = __uint_as_float(rwv[i][k]) - qv;
              ssum += sc;
              if (sc > v1) { v2 = v1; v1 = sc; i1 = j0 + k; }
              else if (sc > v2) v2 = sc;
            }
          }
        }
      }
      const bool bad = !isfinite(ssum);
      float* bs = sBest + R * 12 + g * 3;
      bs[0] = v1;
      bs[1] = __int_as_float(bad ? -2 : i1);
      bs[2] = v2;
    }
    if (agent && act) cp_async_wait_all();  // the update operands have landed (read by this thread only)
    tc_fence_before();
    bar_half(h);  // ---- B3
    PMARK(4);
    if (ht == kHalfThreads - 1) ctl[0] = 0;

    // ============================ combine + update (row agents)
    // U: publish the decision, D / x deltas, advance to the next own slot
    auto update = [&]() {
      inf[RI_DRESET] = 0;
      const int t = inf[RI_T], xr = inf[RI_X], dec = inf[RI_DEC];
      const int uo = inf[RI_UOLD], uxn = inf[RI_UXN], uev = inf[RI_UEV];
      inf[RI_EVT] = uev;
      inf[RI_XUPD] = dec;
      short* Dw = sD + R * kMaxJ;
      if (uev >= 0) Dw[uev] += 1;
      if (dec >= 0) {
        Dw[dec] -= 1;
        atomicSub(S.xloc + (size_t)xr * J + dec, 1);  // fire-and-forget RED
      }
      if (dec != uo) {
        cn_changed += 1;
        cn_first = min(cn_first, t);
        cn_conflicts += (inf[RI_UWR] >> (8 * (t & 3))) & 0xff ? 1 : 0;
      }
      if (S.ref) {
        const int ur = inf[RI_UREF];
        cn_mism += (dec != ur ? 1 : 0) - (uo != ur ? 1 : 0);
      }
      S.cache[t] = dec;
      S.written[t] = 1;
      cn_nev += 1;
      const int pos = inf[RI_POS] + 1;
      inf[RI_POS] = pos;
      if (pos < inf[RI_END]) {
        if (dec >= 0 && uxn == xr) {  // the next step's x delta needs 1/x0[p][dec]: 16-byte bulk copy
          const float* src = a.inv_x0 + (size_t)inf[RI_P] * J + dec;
          mbar_expect_tx(sRBar + R, 16);
          bulk_load(sIx + R * 4, (const void*)((uintptr_t)src & ~(uintptr_t)15), 16, sRBar + R);
        } else {
          mbar_arrive(sRBar + R);
        }
        inf[RI_T] = inf[RI_TN];
        inf[RI_XDIRTY] = uxn != xr ? 1 : 0;
        inf[RI_X] = uxn;
        inf[RI_P] = inf[RI_UPN];
        inf[RI_RR] = inf[RI_URRN];
        inf[RI_OT] = inf[RI_UOTN];
        inf[RI_TN] = inf[RI_UTNN];
      } else {  // process done: its evaluation count, then the next work-list entry
        const int m = inf[RI_M];
        const unsigned long long nev = (unsigned)cn_nev;
        atomicMax(&S.scal->max_evals, nev);
        atomicAdd(&S.scal->total_evals, nev);
        if (S.evals_out) S.evals_out[m] = (long long)nev;
        cn_nev = 0;
        begin_proc(inf, next_entry());
      }
    };
    bool flagged = false;
    if (agent) {
      inf[RI_FLAG] = 0;
      if (!act) {
        inf[RI_ANY] = -1;
      } else {
        const float* bs = sBest + R * 12;
        float v1 = bs[0], v2 = bs[2];
        int i1 = __float_as_int(bs[1]);
        bool bad = i1 == -2;
#pragma unroll
        for (int gg = 1; gg < 4; ++gg) {
          const float w1 = bs[3 * gg], w2v = bs[3 * gg + 2];
          const int j1 = __float_as_int(bs[3 * gg + 1]);
          bad |= j1 == -2;
          if (w1 > v1 || (w1 == v1 && j1 >= 0 && (i1 < 0 || j1 < i1))) { v2 = fmaxf(v1, w2v); v1 = w1; i1 = j1; }
          else v2 = fmaxf(v2, w1);
        }
        if (i1 == -1 && !bad) {  // nothing feasible: decline without a forward pass
          inf[RI_ANY] = 0;
          inf[RI_DEC] = -1;
        } else {
          inf[RI_ANY] = 1;
          inf[RI_DEC] = v1 >= 0.f ? i1 : -1;
          const float g = fmaxf(a.guard, a.guard_abs);  // (the derived bound is proven for tc_pp's layer 1)
          const bool flag = bad || i1 < 0 || !(v1 - v2 >= g) || !(fabsf(v1) >= g);
          cn_tc += 1;
          if (flag || a.verify) {
            inf[RI_FLAG] = flag ? 1 : 2;
            const int k = atomicAdd(&ctl[1], 1);
            ctl[2 + k] = R;
            flagged = true;
          }
        }
        if (!flagged) update();
      }
    }
    const int nflag = bar_red_popc(1 + h, kHalfThreads, flagged);  // ---- B4
    PMARK(5);

    // ============================ exact FP64 re-evaluation of flagged rows
    if (nflag) {
      for (int f = 0; f < nflag; ++f) {
        const int Rf = ctl[2 + f];
        const int* infF = sInfo + Rf * kInfo;
        int* caps = (int*)sAh;
        int* xrow = caps + kMaxJ;
        int* res = xrow + kMaxJ;
        {  // the step's capacities: ckcap - H_b - partial + D
          const int tF = infF[RI_T], bF = infF[RI_B], bsF = base + (bF << kLogK);
          const int k0F = max(lo, bsF) - bsF, k1F = tF - bsF;
          const short* DF = sD + Rf * kMaxJ;
          const bool dresF = infF[RI_DRESET] != 0;
          for (int j = ht; j < J; j += kHalfThreads) {
            int part = 0;
            for (int k = k0F; k < k1F; ++k) part += infF[RI_EV0 + k] == j;
            caps[j] = max(0, sCk[j] - __ldg(S.hck + (size_t)bF * HJ + j) - part + (dresF ? 0 : (int)DF[j]));
            xrow[j] = __ldcg(S.xloc + (size_t)infF[RI_X] * J + j);
          }
        }
        bar_half(h);
        rc::half_recheck(S.model, (double*)(sAh + kAH), caps, xrow, infF[RI_T], res, ht, h,
                         nullptr);
        if (ht == 0) {
          int* infw = sInfo + Rf * kInfo;
          const int exact = res[0], nonfinite = res[1];
          if (nonfinite)
            atomicMin(&S.scal->err_nonfinite, ((unsigned long long)infw[RI_M] << 32) | (unsigned)infw[RI_OT]);
          if (infw[RI_FLAG] == 1) {
            ctl[CT_FLAG] += 1;
            ctl[CT_DIS] += exact != infw[RI_DEC] ? 1 : 0;
          } else {
            ctl[CT_BAD] += exact != infw[RI_DEC] ? 1 : 0;
          }
          infw[RI_DEC] = exact;
        }
        bar_half(h);
      }
      if (flagged) update();
      bar_half(h);
    }
    PMARK(6);
  }

  // ---------------------------------------------------------------- teardown
  __syncthreads();
  if (PROF && prof_on)
    for (int k = 0; k < 20; ++k) a.prof[k] = pacc[k];
#undef PMARK
  if (agent) {
    if (cn_changed) {
      atomicAdd(&S.scal->changed, (unsigned long long)(unsigned)cn_changed);
      atomicAdd(&S.scal->conflicts, (unsigned long long)(unsigned)cn_conflicts);
      atomicMin(&S.scal->first_changed, (unsigned long long)(unsigned)cn_first);
    }
    const long long mism = cn_mism;
    if (mism) atomicAdd((unsigned long long*)&S.scal->mismatch_delta, (unsigned long long)mism);
    if (cn_tc) atomicAdd(&a.stats[0], (unsigned long long)(unsigned)cn_tc);
  }
  if (tid == 0) {
    for (int hh = 0; hh < 2; ++hh) {
      const int* c = sCtlAll + hh * kCtl;
      if (c[CT_FLAG]) atomicAdd(&a.stats[1], (unsigned long long)(unsigned)c[CT_FLAG]);
      if (c[CT_DIS]) atomicAdd(&a.stats[2], (unsigned long long)(unsigned)c[CT_DIS]);
      if (c[CT_BAD]) atomicAdd(&a.stats[3], (unsigned long long)(unsigned)c[CT_BAD]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
  (void)ldpol;
}

}  // namespace inc

cudaError_t launch_inc_prep(const IncPrep& p, cudaStream_t stream) {
  const int nseg = (p.nb + inc::kGSeg - 1) / inc::kGSeg;
  if (nseg > 0)
    inc::k_grows<<<nseg, 64, 0, stream>>>(p.hck, p.ev, p.tau, p.ckcap, p.a64, p.b1, p.lo, p.hi, p.J, p.nb, p.grow);
  inc::k_trans<<<(p.J + 127) / 128, 128, 0, stream>>>(p.hck, p.ckcap, p.wload_sorted, p.J, p.nb, p.bA, p.bD);
  return cudaGetLastError();
}

template <bool PROF, int N3>
static cudaError_t launch_inc(const IncArgs& a, const CUtensorMap& gmap, int ntiles, cudaStream_t stream) {
  const size_t smem = inc::Layout::total;
  const cudaError_t e = ensure_dyn_smem((const void*)inc::k_sweep_inc<PROF, N3>, smem);
  if (e != cudaSuccess) return e;
  inc::k_sweep_inc<PROF, N3><<<ntiles, inc::kBlock, smem, stream>>>(a, gmap);
  return cudaGetLastError();
}

cudaError_t launch_tc_inc(const IncArgs& a, const CUtensorMap& gmap, int ntiles, cudaStream_t stream) {
  if (a.t.prof) return launch_inc<true, kTcN3>(a, gmap, ntiles, stream);  // (debug profiles: the C3 shape)
  switch (a.t.n3) {
    case 16: return launch_inc<false, 16>(a, gmap, ntiles, stream);
    case 32: return launch_inc<false, 32>(a, gmap, ntiles, stream);
    case 64: return launch_inc<false, 64>(a, gmap, ntiles, stream);
    default: return launch_inc<false, kTcN3>(a, gmap, ntiles, stream);
  }
}

}  // namespace pcd
