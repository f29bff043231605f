// tc_pp.cu — the tcgen05 run-partition sweep, ping-pong form (see
// tc_common.cuh for the MLP / precision / exactness scheme).
//
// A CTA (one per SM, 16 warps) runs TWO independent 64-row pipelines
// ("halves"). Half h owns warps 8h..8h+7, the TMEM lanes {32q + 16h + i :
// q < 4, i < 16} (an M=64 tcgen05.mma accumulator at lane offset 16h), its
// own 64-row A operand in smem, its own mbarrier and named barrier (1 + h).
// The weights and the tensor core are shared. While one half waits on its
// MMAs or on the checkpoint-row loads of its next step, the other half's
// CUDA-core phases (features, tanh epilogues, scores) run, so latency that a
// single 128-row lockstep exposes is overlapped.
//
// Thread mapping inside a half: warp w = 8h + 4p + q, lane l: row
// r = 16q + (l & 15) (TMEM lane 32q + 16h + (l & 15)), node group
// g = 2p + (l >> 4). TMEM is accessed with the .16x32bx2 shapes (split 8
// columns), so group g of a row owns the 8-node chunks g, g+4, g+8, g+12 of
// every per-node TMEM region and the 8-unit chunks g, g+4 of the hidden
// layers. Group 3 threads are the row agents (per-row bookkeeping, update
// operand loads, publish, work-list pulls).
//
// Per step and half: F (capacities c = max(0, ckcap - H + D - partial),
// features, feasibility) -> L1 / E1 / L2 / E2 / L3 (fp16x3 MMAs, tanh
// epilogues) -> S (scores, per-group argmax + margin) -> agents combine ->
// exact FP64 re-evaluation of rows with margin < guard (half-local) -> U.
// The state algebra is the run-partition closed form of k_sweep_product.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>

#include "tc_common.cuh"
#include "tc_recheck.cuh"

namespace pcd {
namespace pp {

constexpr int kBlock = 512;
constexpr int kHalfRows = 64;
constexpr int kHalfThreads = 256;
constexpr int kInfo = 28;
constexpr int kScrJ = 112;
constexpr int kMaxCI = 4;   // node chunks per thread (13 chunks for J <= 103)
constexpr uint32_t kTmemCols = 512, kColD = 256, kColCap = 384;
constexpr int kAH = kHalfRows * kTcK1 * 2;  // bytes of one of hi / lo for a half
constexpr int kChunkB = kHalfRows * 8 * 2;  // bytes per k-chunk of a half's operand

enum {
  RI_T = 0, RI_P, RI_POS, RI_END, RI_ANY, RI_DEC, RI_FLAG, RI_RR, RI_TN, RI_XDIRTY, RI_XUPD, RI_OT, RI_EVT,
  RI_X, RI_M, RI_DRESET,
  RI_UEV, RI_UOLD, RI_UWR, RI_UREF, RI_UPN, RI_URRN, RI_UOTN, RI_UTNN, RI_UXN,
  RI_WAIT,   // steps this row's current slot has waited for its FP64 re-evaluation
  RI_PAUSE,  // the slot's re-evaluation is deferred: redo the step, no update
  RI_POS0    // the process's first window position (speculation entries)
};
static_assert(RI_POS0 < kInfo, "per-row state fits");
// Flagged rows wait (redoing their step, which is deterministic: same slot,
// same state) until kRcBatch of them are pending in the half, one has waited
// kMaxWait steps, or they are at least half of the active rows; then the
// whole pending set is re-evaluated in batches (tc_recheck.cuh)
constexpr int kMaxWait = 3;
enum { CN_CHANGED = 0, CN_CONFLICTS, CN_FIRST, CN_MISM, CN_NEV, CN_TC, CN_COUNT };
// per-half control block: [0] active rows, [1] flagged rows, [2..66) flagged rows
enum { CT_FLAG = 66, CT_DIS, CT_BAD, CT_QACT, CT_MAXERR = CT_QACT + 4, CT_MAXWAIT, CT_SPEC, kCtl = 80 };

struct Layout {
  static constexpr int w = 0;
  static constexpr int a = kWImgBytes;                       // half h: hi at a + 2h kAH, lo + kAH
  static constexpr int info = a + 4 * kAH;                   // 128 x kInfo ints
  static constexpr int best = info + kTcRows * kInfo * 4;    // 128 x 4 groups x 3
  static constexpr int cap = best + kTcRows * 4 * 3 * 4;     // checkpoint capacities [112]
  static constexpr int ctl = cap + kScrJ * 4;                // 2 x kCtl
  static constexpr int cst = ctl + 2 * kCtl * 4;             // invc0[112] b1[64] b2[64] b3[112]
  static constexpr int gnode = cst + 352 * 4;                // per-node guards: margin [112], |best| [112]
  static constexpr int cnt = gnode + 2 * kTcN3 * 4;          // per-row counters
  static constexpr int prof = cnt + CN_COUNT * kTcRows * 4;  // debug phase clocks [20]
  static constexpr int bar = prof + 20 * 8;                  // one mbarrier per half + the weight load's
  static constexpr int tmem = bar + 32;
  static constexpr int total = tmem + 16;
};
static_assert(Layout::total <= 232448, "ping-pong sweep shared memory budget");
static_assert(Layout::cap % 16 == 0 && Layout::cst % 16 == 0 && Layout::prof % 8 == 0, "aligned smem rows");

// canonical K-major no-swizzle offsets of a 64-row operand
__device__ __forceinline__ int kc64(int k) { return (k >> 3) * kChunkB + (k & 7) * 2; }
__device__ __forceinline__ int ro64(int r) { return (r >> 3) * 128 + (r & 7) * 16; }

__device__ __forceinline__ void bar_half(int h) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(kHalfThreads) : "memory");
}
// .16x32bx2 TMEM access: threads 0-15 -> lanes base..base+15 at columns
// col..col+7, threads 16-31 -> the same lanes at col+8..col+15
__device__ __forceinline__ void ld8s(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], 8;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void st8s(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.16x32bx2.x8.b32 [%0], 8, {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

__device__ __forceinline__ void put_feature(unsigned char* sAh, int off, float v) {
  __half hh, l;
  split_f16(v, hh, l);
  *(__half*)(sAh + off) = hh;
  *(__half*)(sAh + kAH + off) = l;
}

// ---------------------------------------------------------------------------
// Exact FP64 re-evaluation of one flagged row by its half (256 threads):
// DualNetworkPolicy::evaluate (policies.hpp:121-168) in exactly the operation
// order of warp_policy_eval<kDual> — one thread per output neuron runs the
// acc = b; acc += w * x chain on weights read from L2. Scratch lives in the
// first k-chunks of the half's operand (free between layer 3 and the next F).
//   hi [0, ...)  caps / x row / results (ints)
//   lo [0, ...)  f / h1 / h2 / pr (doubles)
constexpr int kRcInts = 0;
using rc::kRcVec;
constexpr int kRcScratchHi = (kRcInts + rc::kRcBatchInts * 4 + 15) & ~15;
constexpr int kRcScratchLo = ((rc::kRcBatch * rc::kRcRow > kRcVec ? rc::kRcBatch * rc::kRcRow : kRcVec) * 8 + 15) & ~15;
static_assert(kRcScratchHi <= 12 * kChunkB && kRcScratchLo <= 12 * kChunkB, "recheck scratch in k-chunks 0..11");
// operand columns the recheck scratch may overwrite (the x/x0 features persist
// across steps only when they lie above these and above the hidden operands)
constexpr int kScratchCols = ((kRcScratchHi > kRcScratchLo ? kRcScratchHi : kRcScratchLo) + kChunkB - 1) / kChunkB * 8;

// N3: layer-3 width class (J <= N3), KS1: layer-1 k-steps (2J + 1 <= 16 KS1);
// the C3 shape is <112, 13>, smaller node counts get narrower MMAs
template <bool PROF, int N3, int KS1>
__global__ void __launch_bounds__(kBlock, 1) k_sweep_pp(TcArgs a, const __grid_constant__ CUtensorMap wmap) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const long long hk0 = PROF ? clock64() : 0;  // (debug) per-half timeline
  const SweepArgs& S = a.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = S.J, lo = S.lo;
  const int base = hck_base(lo), HJ = hck_stride(J), RJ = (J + 7) & ~7;
  unsigned char* sW = smem + Layout::w;
  int* sInfo = (int*)(smem + Layout::info);
  float* sBest = (float*)(smem + Layout::best);
  int* sCap = (int*)(smem + Layout::cap);
  int* sCtlAll = (int*)(smem + Layout::ctl);
  int* sCnt = (int*)(smem + Layout::cnt);
  uint64_t* sBar = (uint64_t*)(smem + Layout::bar);
  uint32_t* sTmem = (uint32_t*)(smem + Layout::tmem);
  float* sInvC0 = (float*)(smem + Layout::cst);
  float* sB1 = sInvC0 + kScrJ;
  float* sB2 = sB1 + 64;
  const int tile = blockIdx.x;
  // half / row / node-group of this thread
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
  const int XO = tc_rj(J);  // first inventory-feature column (capacity chunks are whole)
  const bool xpersist = XO >= kTcH && XO >= kScratchCols;  // x/x0 columns never overwritten

  // ---------------------------------------------------------------- setup
  {
    uint4* da = (uint4*)(smem + Layout::a);
    for (int i = tid; i < 4 * kAH / 16; i += kBlock) da[i] = make_uint4(0, 0, 0, 0);
  }
  for (int j = tid; j < kScrJ; j += kBlock) {
    sCap[j] = j < J ? S.ckcap[j] : 0;
    sInvC0[j] = j < J ? a.inv_c0[j] : 0.f;
  }
  for (int i = tid; i < kTcH; i += kBlock) {
    sB1[i] = a.b1f[i];
    sB2[i] = a.b2f[i];
  }
  float* sGn = (float*)(smem + Layout::gnode);
  for (int i = tid; i < 2 * kTcN3; i += kBlock)
    sGn[i] = a.gnode ? a.gnode[i] : (i < kTcN3 ? a.guard : a.guard_abs);
  const int nq = a.wctl[0], dealt = (int)gridDim.x * kTcRows;
  auto begin_proc = [&](int* inf, int m) {
    int pos = 0, end = 0;
    if (m >= 0) {  // (window positions from the work-list build: one round trip)
      pos = a.wbeg[m];
      end = pos + a.wlen[m];
    }
    inf[RI_M] = m;
    inf[RI_POS] = pos;
    inf[RI_POS0] = pos;
    inf[RI_END] = end;
    inf[RI_XDIRTY] = 1;
    inf[RI_XUPD] = -1;
    inf[RI_EVT] = -1;
    inf[RI_DRESET] = 1;
    inf[RI_P] = -1;
    inf[RI_X] = -1;
    inf[RI_WAIT] = 0;
    inf[RI_PAUSE] = 0;
    if (pos < end) {
      const int t = S.pslots[pos];
      inf[RI_T] = t;
      inf[RI_P] = S.model.product[t];
      inf[RI_X] = S.rid[t];
      inf[RI_RR] = S.model.rrow[t];
      inf[RI_OT] = S.model.order_t ? S.model.order_t[t] : t;
      inf[RI_TN] = pos + 1 < end ? S.pslots[pos + 1] : -1;
    }
  };
  auto next_entry = [&]() -> int {
    const int k = dealt + atomicAdd(&a.wctl[1], 1);
    return k < nq ? a.wq[k] : -1;
  };
  if (agent) {
    const int k = R * (int)gridDim.x + tile;
    begin_proc(sInfo + R * kInfo, k < nq ? a.wq[k] : -1);
    for (int k2 = 0; k2 < CN_COUNT; ++k2) sCnt[k2 * kTcRows + R] = k2 == CN_FIRST ? INT_MAX : 0;
  }
  for (int i = tid; i < 2 * kCtl; i += kBlock) sCtlAll[i] = 0;
  if (tid == 0) {
    mbar_init(sBar, 1);
    mbar_init(sBar + 1, 1);
    mbar_init(sBar + 2, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the B operands of every MMA (weight image, kWImgBytes) by TMA: two
    // [kWImgRows/2][128] fp16 boxes; the MMA issuers wait on sBar[2] before
    // their first layer, so the copy overlaps the first F phase
    mbar_expect_tx(sBar + 2, kWImgBytes);
    tma_load_2d(sW, &wmap, 0, 0, sBar + 2);
    tma_load_2d(sW + kWImgBytes / 2, &wmap, 0, kWImgRows / 2, sBar + 2);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;
  const uint32_t tD = tmem + ((uint32_t)(16 * h) << 16);  // MMA accumulator base of the half
  {  // D = 0
    const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int i = 0; i < ni; ++i) st8s(tmem + tl + kColD + 16 * p2 + 32 * i, z);
    tmem_wait_st();
  }

  const uint32_t aBase = smem_u32(sAh);
  // per layer one [hi; lo] operand of 2N rows (engine.cu prepare_tc, img2)
  const uint32_t w1 = smem_u32(sW), w2 = w1 + 2 * kW1Bytes, w3 = w2 + 2 * kW2Bytes;
  const uint32_t id64 = idesc_f16(64, 64), id128 = idesc_f16(64, 128);
  const uint32_t idn3 = idesc_f16(64, N3), id2n3 = idesc_f16(64, 2 * N3);
  uint32_t phase = 0;
  bool wready = false;  // (MMA issuers) the weight image's TMA load completed
  const float invT = S.model.horizon > 0 ? (float)(1.0 / (double)S.model.horizon) : 0.f;
  uint32_t xb = 0;  // x > 0 bits of the thread's nodes (bit 8i + k: node 8(g + 4i) + k), persistent

  long long* pacc = (long long*)(smem + Layout::prof);
  if (PROF && tid == 0)
    for (int k = 0; k < 20; ++k) pacc[k] = 0;
  long long plast = PROF ? clock64() : 0;
  const long long hl0 = plast;
  long long hsteps = 0, hrcb = 0, hrcc = 0;
  const bool prof_on = PROF && blockIdx.x == 0 && tid == 0;
#define PMARK(k) do { if (PROF && prof_on) { const long long now_ = clock64(); pacc[k] += now_ - plast; plast = now_; } } while (0)

  // the half's MMAs of one layer (N outputs), K16 k-steps: A_hi . [W_hi; W_lo]
  // (one N = 2N MMA: hi.hi into acc, hi.lo into acc + N), then A_lo . W_hi
  // accumulated into acc + N
  auto issue_layer = [&](uint32_t acc, uint32_t N, uint32_t wb, int ksteps, uint32_t idfull, uint32_t idhalf,
                         int s0 = 0, bool commit = true) {
    tc_fence_after();
    const uint64_t dA = umma_desc(aBase, kHalfRows * 16, 128), dAl = umma_desc(aBase + kAH, kHalfRows * 16, 128);
    const uint64_t dW = umma_desc(wb, 2 * N * 16, 128);
    for (int s = s0; s < ksteps; ++s) {
      const uint64_t ah = dA + s * ((2 * kChunkB) >> 4), al = dAl + s * ((2 * kChunkB) >> 4);
      const uint64_t b = dW + s * ((4 * N * 16) >> 4);
      mma_f16(tD + acc, ah, b, idfull, s > 0);
      mma_f16(tD + acc + N, al, b, idhalf, 1);
    }
    if (commit) mma_commit(bar);
  };

  for (;;) {
    // ============================ F: capacities, features, feasibility
    uint32_t fmask = 0;  // feasible nodes of the thread (bit 8i + k)
    int* inf = sInfo + R * kInfo;
    int u_ev = -1, u_old = 0, u_wr = 0, u_ref = 0, u_pn = -1, u_rrn = 0, u_otn = 0, u_tnn = -1, u_xn = -1;
    if (agent) {  // P: the operands of this row's update (U); latency hidden behind F
      const int pos = inf[RI_POS], end = inf[RI_END];
      if (pos < end) {
        const int t = inf[RI_T];
        u_ev = S.nocache ? -1 : S.ev[t];
        u_old = S.cache[t];
        u_wr = S.written[t];
        if (S.ref) u_ref = S.ref[t];
        const int tn = inf[RI_TN];
        if (tn >= 0) {
          u_pn = S.model.product[tn];
          u_xn = S.rid[tn];
          u_rrn = S.model.rrow[tn];
          u_otn = S.model.order_t ? S.model.order_t[tn] : tn;
        }
        if (pos + 2 < end) u_tnn = S.pslots[pos + 2];
      }
    }
    {
      const bool act = inf[RI_POS] < inf[RI_END];
      int t = 0, b = 0, p = 0, x = 0, xd = 0, xu = -1, evt = -1, xuv = 0, dres = 0;
      float xui = 0.f;
      uint32_t hv[kMaxCI][8];
      uint32_t e8[8];
#pragma unroll
      for (int i = 0; i < kMaxCI; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) hv[i][k] = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) e8[k] = 0xffffffffu;
      // the thread's chunk of a node (>= 0) or -1
      auto my_ci = [&](int j) { return (j >= 0 && ((j >> 3) & 3) == g) ? (j >> 5) : -1; };
      if (act) {
        t = inf[RI_T];
        p = inf[RI_P];
        x = inf[RI_X];
        dres = inf[RI_DRESET];
        xd = inf[RI_XDIRTY] | (xpersist ? 0 : 1);
        xu = inf[RI_XUPD];
        evt = inf[RI_EVT];
        b = (t - base) >> kLogK;
        // streamed rows bypass L1, so the reward table (read every step) stays there
        // (and leave L2 first: read about once per iteration)
        if (!S.nocache) {  // nocache (Time Warp): other processes' steps count as declined
          const int* hr = S.hck + (size_t)b * HJ;
          const uint64_t pol = l2_policy_evict_first();
          ldg256_na_ef(S.ev + base + (b << kLogK), e8, pol);
#pragma unroll
          for (int i = 0; i < kMaxCI; ++i)
            if (i < ni && 8 * (g + 4 * i) < J) ldg256_na_ef(hr + 8 * (g + 4 * i), hv[i], pol);
        }
        if (!xd && my_ci(xu) >= 0) {
          xuv = S.xloc[(size_t)x * J + xu];
          xui = __ldg(a.inv_x0 + (size_t)p * J + xu);
        }
      }
      // partial block [max(lo, base + 8b), t): per-chunk packed nibble counts
      uint32_t pk[kMaxCI];
#pragma unroll
      for (int i = 0; i < kMaxCI; ++i) pk[i] = 0;
      {
        const int sb = base + (b << kLogK);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int s = sb + k;
          const int ek = (int)e8[k];
          const int ci = (act && s >= lo && s < t) ? my_ci(ek) : -1;
          const uint32_t nib = 1u << (4 * (ek & 7));
#pragma unroll
          for (int i = 0; i < kMaxCI; ++i) pk[i] += ci == i ? nib : 0u;
        }
      }
      PMARK(12);
      const int ciE = my_ci(evt), ciX = my_ci(xu);
#pragma unroll
      for (int i = 0; i < kMaxCI; ++i) {
        if (i >= ni) break;  // warp-uniform; constant trip count keeps the arrays in registers
        const int j0 = 8 * (g + 4 * i);
        const bool live = j0 < J;
        const int jc = live ? j0 : 0;
        uint32_t dv[8];
        ld8s(tmem + tl + kColD + 16 * p2 + 32 * i, dv);
        tmem_wait_ld();
        // D deltas of the chunk as biased nibbles (1 + [k == evt] - [k == xu]); dres clears D
        const uint32_t dpk = 0x11111111u + (ciE == i ? 1u << (4 * (evt & 7)) : 0u) - (ciX == i ? 1u << (4 * (xu & 7)) : 0u);
        const uint32_t dmask = dres ? 0u : 0xffffffffu;
        const int4 cp0 = *(const int4*)(sCap + jc), cp1 = *(const int4*)(sCap + jc + 4);
        const float4 iv0 = *(const float4*)(sInvC0 + jc), iv1 = *(const float4*)(sInvC0 + jc + 4);
        const int capv[8] = {cp0.x, cp0.y, cp0.z, cp0.w, cp1.x, cp1.y, cp1.z, cp1.w};
        const float inv[8] = {iv0.x, iv0.y, iv0.z, iv0.w, iv1.x, iv1.y, iv1.z, iv1.w};
        uint32_t cv[8], bits = 0;
        float fv[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int d = (int)(dv[k] & dmask) + (int)((dpk >> (4 * k)) & 15u) - 1;
          dv[k] = (uint32_t)d;
          const int cc = j0 + k < J ? max(capv[k] - (int)hv[i][k] + d - (int)((pk[i] >> (4 * k)) & 15u), 0) : 0;
          cv[k] = (uint32_t)cc;
          bits |= (cc > 0 ? 1u : 0u) << k;
          fv[k] = (float)cc * inv[k];
        }
        st8s(tmem + tl + kColD + 16 * p2 + 32 * i, dv);
        st8s(tmem + tl + kColCap + 16 * p2 + 32 * i, cv);
        if (live) {
          fmask |= bits << (8 * i);
          uint32_t h4[4], l4[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) split2(fv[2 * k], fv[2 * k + 1], h4[k], l4[k]);
          if (act) {  // whole chunk: columns [J, RJ) are zero padding (cc = 0 there)
            const int off = rowo + kc64(j0);
            *(uint4*)(sAh + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
            *(uint4*)(sAh + kAH + off) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
          }
        }
      }
      PMARK(13);
      // inventory features x/x0 (columns J + node) and the x > 0 bits
      if (act && xd) {
        const int* xr = S.xloc + (size_t)x * J;
        const float* ix = a.inv_x0 + (size_t)p * J;
        uint32_t nb = 0;
#pragma unroll
        for (int i = 0; i < kMaxCI; ++i) {
          if (i >= ni) break;
          const int j0 = 8 * (g + 4 * i);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            if (j0 + k >= J) break;
            const int xj = xr[j0 + k];
            put_feature(sAh, rowo + kc64(XO + j0 + k), (float)xj * __ldg(ix + j0 + k));
            nb |= (xj > 0 ? 1u : 0u) << (8 * i + k);
          }
        }
        xb = nb;
      } else if (act && ciX >= 0) {
        put_feature(sAh, rowo + kc64(XO + xu), (float)xuv * xui);
        if (xuv <= 0) xb &= ~(1u << (8 * ciX + (xu & 7)));
      }
      if (act && agent) put_feature(sAh, rowo + kc64(XO + J), (float)inf[RI_OT] * invT);
      fmask = act ? (fmask & xb) : 0u;
      if (p2 == 0) {
        const uint32_t bal = __ballot_sync(0xffffffffu, act) & 0xffffu;
        if (lane == 0) {
          ctl[CT_QACT + q] = bal != 0;
          if (bal) atomicAdd(&ctl[0], __popc(bal));
        }
      }
      tmem_wait_st();
      PMARK(14);
    }
    if (agent) {
      inf[RI_UEV] = u_ev;
      inf[RI_UOLD] = u_old;
      inf[RI_UWR] = u_wr;
      inf[RI_UREF] = u_ref;
      inf[RI_UPN] = u_pn;
      inf[RI_URRN] = u_rrn;
      inf[RI_UOTN] = u_otn;
      inf[RI_UTNN] = u_tnn;
      inf[RI_UXN] = u_xn;
    }
    tc_fence_before();
    fence_async_smem();
    bar_half(h);
    PMARK(0);
    if (ctl[0] == 0) break;
    if (PROF && prof_on) pacc[10] += 1;
    if (PROF) hsteps += 1;

    // ============================ layer 1: z1 = F . W1^T (three products)
    if (ht == 0 && !wready) {
      mbar_wait(sBar + 2, 0);  // the TMA weight image has landed
      wready = true;
    }
    if (ht == 0) issue_layer(0, kTcH, w1, KS1, id128, id64);
    if (ht == 0) mbar_wait(bar, phase);  // one waiter; the half sleeps on its named barrier
    bar_half(h);
    PMARK(1);
    phase ^= 1;
    tc_fence_after();

    // ============================ hidden epilogues (z -> tanh -> fp16 hi/lo)
    const bool qact = ctl[CT_QACT + q] != 0;  // warp-uniform: skip idle row quarters
    // one 8-unit chunk (i = 0: units 0-31 of the layer = the next layer's
    // k-steps 0-1; i = 1: units 32-63 = k-steps 2-3), so the next layer's
    // first k-steps run while the second chunk is computed
    auto hidden_part = [&](uint32_t col_hh, uint32_t col_x, const float* bias, int i) {
      if (!qact) return;
      uint32_t vh[8], vx[8];
      ld8s(tmem + tl + col_hh + 16 * p2 + 32 * i, vh);
      ld8s(tmem + tl + col_x + 16 * p2 + 32 * i, vx);
      tmem_wait_ld();
      const int u0 = 8 * (g + 4 * i);
      uint32_t ph[4], pl[4];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const float z0 = fmaf(__uint_as_float(vx[k]), kLoInv, __uint_as_float(vh[k])) + bias[u0 + k];
        const float z1 = fmaf(__uint_as_float(vx[k + 1]), kLoInv, __uint_as_float(vh[k + 1])) + bias[u0 + k + 1];
        split2(tanh_mufu(z0), tanh_mufu(z1), ph[k / 2], pl[k / 2]);
      }
      const int off = rowo + kc64(u0);
      *(uint4*)(sAh + off) = make_uint4(ph[0], ph[1], ph[2], ph[3]);
      *(uint4*)(sAh + kAH + off) = make_uint4(pl[0], pl[1], pl[2], pl[3]);
    };
    auto publish_operand = [&]() {
      tc_fence_before();
      fence_async_smem();
      bar_half(h);
    };
    hidden_part(0, 64, sB1, 0);
    publish_operand();
    if (ht == 0) issue_layer(128, kTcH, w2, 2, id128, id64, 0, false);  // layer 2, k-steps 0-1
    tc_fence_after();
    hidden_part(0, 64, sB1, 1);
    publish_operand();
    PMARK(2);

    // ============================ layer 2 (k-steps 2-3)
    if (ht == 0) issue_layer(128, kTcH, w2, kTcH / 16, id128, id64, 2, true);
    if (ht == 0) mbar_wait(bar, phase);  // one waiter; the half sleeps on its named barrier
    bar_half(h);
    PMARK(3);
    phase ^= 1;
    tc_fence_after();
    // h2 overwrites h1 (layer 2 has completed); no early layer-3 k-steps here:
    // layer 3's accumulators (columns 0..2 N3) overlap layer 2's (128..255)
    hidden_part(128, 192, sB2, 0);
    hidden_part(128, 192, sB2, 1);
    publish_operand();
    PMARK(4);

    // ============================ layer 3: q = h2 . W3'^T (N = 112)
    if (ht == 0) issue_layer(0, N3, w3, kTcH / 16, id2n3, idn3);
    // this thread's reward loads while layer 3 runs
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
    if (ht == 0) mbar_wait(bar, phase);  // one waiter; the half sleeps on its named barrier
    bar_half(h);
    PMARK(5);
    phase ^= 1;
    tc_fence_after();

    // ============================ S: scores, argmax, margin (row, group)
    {
      float v1 = -INFINITY, v2 = -INFINITY, ssum = 0.f;  // ssum: non-finite iff some score is (or overflow: flagged, safe)
      int i1 = -1;
      if (qact) {
#pragma unroll
        for (int i0 = 0; i0 < kMaxCI; i0 += 2) {
          if (i0 >= ni) break;  // warp-uniform
          uint32_t vh[2][8], vx[2][8];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            if (i0 + u < ni) {
              ld8s(tmem + tl + 16 * p2 + 32 * (i0 + u), vh[u]);
              ld8s(tmem + tl + N3 + 16 * p2 + 32 * (i0 + u), vx[u]);
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
              if (!((fmask >> (8 * i + k)) & 1u)) continue;  // feasible implies node < J
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
    tc_fence_before();
    bar_half(h);
    PMARK(6);
    if (agent) {  // combine the groups
      inf[RI_FLAG] = 0;
      if (inf[RI_POS] >= inf[RI_END]) {
        inf[RI_ANY] = -1;
      } else {
        const float* bs = sBest + R * 12;
        float v1 = bs[0], v2 = bs[2];
        int i1 = __float_as_int(bs[1]);
        bool bad = i1 == -2;
#pragma unroll
        for (int gg = 1; gg < 4; ++gg) {
          const float w1 = bs[3 * gg], w2 = bs[3 * gg + 2];
          const int j1 = __float_as_int(bs[3 * gg + 1]);
          bad |= j1 == -2;
          if (w1 > v1 || (w1 == v1 && j1 >= 0 && (i1 < 0 || j1 < i1))) { v2 = fmaxf(v1, w2); v1 = w1; i1 = j1; }
          else v2 = fmaxf(v2, w1);
        }
        if (i1 == -1 && !bad) {  // nothing feasible
          inf[RI_ANY] = 0;
          inf[RI_DEC] = -1;
        } else {
          inf[RI_ANY] = 1;
          inf[RI_DEC] = v1 >= 0.f ? i1 : -1;
          bool flag = bad || i1 < 0;
          if (!flag) {
            const float gd = sGn[i1], ga = sGn[kTcN3 + i1], mg = v1 - v2, av = fabsf(v1);
            if (!(mg >= gd) || !(av >= ga)) {  // within the guard: speculate or re-evaluate here
              flag = true;
              if (a.spec && mg >= gd * a.spec_floor && av >= ga * a.spec_floor) {
                const int qi = atomicAdd(a.spec_n, 1);
                if (qi < a.spec_cap) {  // (a full queue falls back to the re-evaluation here)
                  int* e = a.spec_q + (size_t)qi * kSpecStride;
                  e[0] = inf[RI_T];
                  e[1] = inf[RI_POS];
                  e[2] = inf[RI_POS0];
                  e[3] = inf[RI_END];
                  e[4] = inf[RI_M];
                  e[5] = inf[RI_X];
                  e[6] = inf[RI_P];
                  e[7] = inf[RI_RR];
                  e[8] = inf[RI_OT];
                  // (debug, tests) publish a wrong decision for every 4th
                  // speculated slot: the verification must catch it
                  if (a.spec_flip == 1 && (inf[RI_T] & 3) == 0) inf[RI_DEC] = inf[RI_DEC] >= 0 ? -1 : i1;
                  e[9] = inf[RI_DEC];
                  flag = false;
                  atomicAdd(&ctl[CT_SPEC], 1);
                }
              }
            }
          }
          if (!flag) sCnt[CN_TC * kTcRows + R] += 1;  // (flagged rows: when re-evaluated)
          if (flag || a.verify) {
            inf[RI_FLAG] = flag ? 1 : 2;
            const int k = atomicAdd(&ctl[1], 1);
            ctl[2 + k] = R;
            if (flag) atomicMax(&ctl[CT_MAXWAIT], inf[RI_WAIT]);
          }
        }
      }
    }
    bar_half(h);
    PMARK(7);

    // ============================ exact FP64 re-evaluation of flagged rows
    // in batches of rc::kRcBatch: one order-free FP64 pass certifies most
    // rows (fast_margin), the rest take the reference's ordered chain
    const int nflag = ctl[1];
    const bool rc_run =
        nflag > 0 && (a.verify || nflag >= rc::kRcBatch || ctl[CT_MAXWAIT] >= kMaxWait || 2 * nflag >= ctl[0]);
    if (!rc_run && nflag > 0 && agent && inf[RI_FLAG] == 1) {  // defer: redo this step
      inf[RI_PAUSE] = 1;
      inf[RI_WAIT] += 1;
    }
    const long long hrc0 = PROF ? clock64() : 0;
    if (rc_run) {
      int* rints = (int*)(sAh + kRcInts);
      int* rres = rints + rc::kRcBatch * 2 * kScrJ;
      int* rinfo = rres + 4 * rc::kRcBatch;  // rc::kRcRowInfo per row
      double* rlo = (double*)(sAh + kAH);
      // verify mode: the row's tensor-core scores (TMEM layer-3 columns) against
      // the exact ones; ps2 == nullptr: ps holds summed prices
      auto verify_row = [&](int b, const double* ps, const double* ps2) {
        const int Rf = ctl[2 + b], rf = Rf - kHalfRows * h;
        if ((rf >> 4) != q) return;  // warp-uniform
        const int* caps = rints + (b % rc::kRcBatch) * 2 * kScrJ;
        const int* xrow = caps + kScrJ;
        const int* infF = sInfo + Rf * kInfo;
        const double* rw = S.model.rtab + (size_t)S.model.rrow[infF[RI_T]] * J;
        const float* rq = a.rtabq + (size_t)infF[RI_RR] * RJ;
        float emax = 0.f;
        for (int i = 0; i < ni; ++i) {
          uint32_t vh[8], vx[8];
          ld8s(tmem + tl + 16 * p2 + 32 * i, vh);
          ld8s(tmem + tl + N3 + 16 * p2 + 32 * i, vx);
          tmem_wait_ld();
          const int j0 = 8 * (g + 4 * i);
          if (rr != rf) continue;
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int j = j0 + k;
            if (j >= J || caps[j] <= 0 || xrow[j] <= 0) continue;
            const float sc = rq[j] - fmaf(__uint_as_float(vx[k]), kLoInv, __uint_as_float(vh[k]));
            const double ex = ps2 ? (rw[j] - ps[j]) - ps2[j] : rw[j] - ps[j];
            emax = fmaxf(emax, __double2float_ru(fabs((double)sc - ex)));
          }
        }
        if (rr == rf && emax > 0.f) atomicMax(&ctl[CT_MAXERR], __float_as_int(emax));
      };
      for (int f0 = 0; f0 < nflag; f0 += rc::kRcBatch) {
        const int nb = min(rc::kRcBatch, nflag - f0);
        // the step's capacities (TMEM cap columns, from the rows' threads) and inventory rows
        for (int b = 0; b < nb; ++b) {
          const int rf = ctl[2 + f0 + b] - kHalfRows * h;
          if ((rf >> 4) == q) {  // warp-uniform
            int* caps = rints + b * 2 * kScrJ;
            for (int i = 0; i < ni; ++i) {
              uint32_t v[8];
              ld8s(tmem + tl + kColCap + 16 * p2 + 32 * i, v);
              tmem_wait_ld();
              const int j0 = 8 * (g + 4 * i);
              if (rr == rf && j0 < kScrJ)
#pragma unroll
                for (int k = 0; k < 8; ++k) caps[j0 + k] = (int)v[k];
            }
          }
        }
        if (ht < nb) {
          const int* infF = sInfo + ctl[2 + f0 + ht] * kInfo;
          int* ri = rinfo + rc::kRcRowInfo * ht;
          ri[0] = infF[RI_T];
          ri[1] = infF[RI_P];
          ri[2] = infF[RI_X];
          ri[3] = infF[RI_RR];
          ri[4] = infF[RI_OT];
        }
        bar_half(h);
        rc::half_recheck_fast_batch(S.model, S.xloc, rlo, rints, rinfo, nb, ht, h,
                                    (PROF && prof_on) ? pacc + 15 : nullptr);
        if (PROF && prof_on) pacc[11] += 1 + ((long long)nb << 20);  // batches | rows << 20
        if (a.verify)
          for (int b = 0; b < nb; ++b)
            if (rres[4 * b + 2]) verify_row(f0 + b, rlo + b * rc::kRcRow + kTcH, nullptr);
        // rows the fast path could not certify: the ordered chain (reuses the double scratch)
        for (int b = 0; b < nb; ++b) {
          if (rres[4 * b + 2]) continue;  // uniform (shared memory)
          const int* caps = rints + b * 2 * kScrJ;
          rc::half_recheck_ordered(S.model, rlo, caps, caps + kScrJ, rinfo[rc::kRcRowInfo * b], rres + 4 * b, ht, h);
          if (PROF && prof_on) pacc[11] += 1LL << 40;  // ordered-chain rows
          if (a.verify) verify_row(f0 + b, rlo + rc::kRcOpr, rlo + rc::kRcOpr + J);
        }
        if (ht == 0) {
          for (int b = 0; b < nb; ++b) {
            int* infw = sInfo + ctl[2 + f0 + b] * kInfo;
            const int exact = rres[4 * b], nonfinite = rres[4 * b + 1];
            if (nonfinite)
              atomicMin(&S.scal->err_nonfinite, ((unsigned long long)infw[RI_M] << 32) | (unsigned)infw[RI_OT]);
            infw[RI_WAIT] = 0;
            if (infw[RI_FLAG] == 1) {
              ctl[CT_FLAG] += 1;
              ctl[CT_DIS] += exact != infw[RI_DEC] ? 1 : 0;
              sCnt[CN_TC * kTcRows + ctl[2 + f0 + b]] += 1;
            } else {
              ctl[CT_BAD] += exact != infw[RI_DEC] ? 1 : 0;
            }
            infw[RI_DEC] = exact;
          }
        }
        bar_half(h);
      }
      // the scratch overlaps K-padding columns of the layer-1 operand when
      // 2J+1 < kScratchCols: leave zeros behind, as the setup did
      uint4* zh = (uint4*)sAh;
      uint4* zl = (uint4*)(sAh + kAH);
      for (int i = ht; i < kRcScratchHi / 16; i += kHalfThreads) zh[i] = make_uint4(0, 0, 0, 0);
      for (int i = ht; i < kRcScratchLo / 16; i += kHalfThreads) zl[i] = make_uint4(0, 0, 0, 0);
      bar_half(h);
    }
    PMARK(8);
    if (PROF && rc_run) {
      hrcb += (nflag + rc::kRcBatch - 1) / rc::kRcBatch;
      hrcc += clock64() - hrc0;
    }

    // ============================ U: update + publish (row agents)
    if (agent) {
      inf[RI_DRESET] = 0;
      if (inf[RI_PAUSE]) {  // deferred re-evaluation: same slot next step, no state change
        inf[RI_PAUSE] = 0;
        inf[RI_EVT] = -1;
        inf[RI_XUPD] = -1;
      } else if (inf[RI_ANY] >= 0) {
        const int t = inf[RI_T], x = inf[RI_X], dec = inf[RI_DEC];
        const int uo = inf[RI_UOLD], uxn = inf[RI_UXN];
        // D deltas are applied by the row's F threads next step
        inf[RI_EVT] = inf[RI_UEV];
        inf[RI_XUPD] = dec;
        if (dec >= 0) atomicSub(&S.xloc[(size_t)x * J + dec], 1);  // fire-and-forget RED
        int* cn = sCnt + R;
        if (dec != uo) {
          cn[CN_CHANGED * kTcRows] += 1;
          cn[CN_FIRST * kTcRows] = min(cn[CN_FIRST * kTcRows], t);
          cn[CN_CONFLICTS * kTcRows] += inf[RI_UWR] ? 1 : 0;
        }
        if (S.ref) {
          const int ur = inf[RI_UREF];
          cn[CN_MISM * kTcRows] += (dec != ur ? 1 : 0) - (uo != ur ? 1 : 0);
        }
        S.cache[t] = dec;
        S.written[t] = 1;
        cn[CN_NEV * kTcRows] += 1;
        const int pos = inf[RI_POS] + 1;
        inf[RI_POS] = pos;
        if (pos < inf[RI_END]) {
          const int tp = inf[RI_UTNN];
          if (tp >= 0 && !S.nocache) {  // warm L2 with the checkpoint row and event block of the step after next
            const int bn = (tp - base) >> kLogK;
            const int* hbn = S.hck + (size_t)bn * HJ;
            for (int k = 0; k < HJ; k += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(hbn + k));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(S.ev + base + (bn << kLogK)));
          }
          inf[RI_T] = inf[RI_TN];
          inf[RI_XDIRTY] = uxn != x ? 1 : 0;
          inf[RI_X] = uxn;
          inf[RI_P] = inf[RI_UPN];
          inf[RI_RR] = inf[RI_URRN];
          inf[RI_OT] = inf[RI_UOTN];
          inf[RI_TN] = inf[RI_UTNN];
        } else {
          // process done: its evaluation count, then the next work-list entry
          const int m = inf[RI_M];
          const unsigned long long nev = (unsigned)cn[CN_NEV * kTcRows];
          atomicMax(&S.scal->max_evals, nev);
          atomicAdd(&S.scal->total_evals, nev);
          if (S.evals_out) S.evals_out[m] = (long long)nev;
          cn[CN_NEV * kTcRows] = 0;
          begin_proc(inf, next_entry());
        }
      }
    }
    if (ht == kHalfThreads - 1) {
      ctl[0] = 0;
      ctl[1] = 0;
      ctl[CT_MAXWAIT] = 0;
    }
    bar_half(h);
    PMARK(9);
  }

  // ---------------------------------------------------------------- teardown
  const long long hl1 = PROF ? clock64() : 0;
  __syncthreads();
  if (PROF && prof_on)
    for (int k = 0; k < 20; ++k) a.prof[k] = pacc[k];
  if (PROF && ht == 0) {  // per half: steps, loop cycles, re-evaluation batches / cycles, setup, end wait
    long long* hp = a.prof + 20 + 2 * 4096 + (size_t)(2 * blockIdx.x + h) * 6;
    hp[0] = hsteps;
    hp[1] = hl1 - hl0;
    hp[2] = hrcb;
    hp[3] = hrcc;
    hp[4] = hl0 - hk0;
    hp[5] = clock64() - hl1;
  }
#undef PMARK
  if (agent) {
    const int* cn = sCnt + R;
    if (cn[CN_CHANGED * kTcRows]) {
      atomicAdd(&S.scal->changed, (unsigned long long)(unsigned)cn[CN_CHANGED * kTcRows]);
      atomicAdd(&S.scal->conflicts, (unsigned long long)(unsigned)cn[CN_CONFLICTS * kTcRows]);
      atomicMin(&S.scal->first_changed, (unsigned long long)(unsigned)cn[CN_FIRST * kTcRows]);
    }
    const long long mism = cn[CN_MISM * kTcRows];
    if (mism) atomicAdd((unsigned long long*)&S.scal->mismatch_delta, (unsigned long long)mism);
    if (cn[CN_TC * kTcRows]) atomicAdd(&a.stats[0], (unsigned long long)(unsigned)cn[CN_TC * kTcRows]);
  }
  if (tid == 0) {
    for (int hh = 0; hh < 2; ++hh) {
      const int* c = sCtlAll + hh * kCtl;
      if (c[CT_FLAG]) atomicAdd(&a.stats[1], (unsigned long long)(unsigned)c[CT_FLAG]);
      if (c[CT_DIS]) atomicAdd(&a.stats[2], (unsigned long long)(unsigned)c[CT_DIS]);
      if (c[CT_BAD]) atomicAdd(&a.stats[3], (unsigned long long)(unsigned)c[CT_BAD]);
      if (c[CT_MAXERR]) atomicMax(&a.stats[4], (unsigned long long)(unsigned)c[CT_MAXERR]);
      if (c[CT_SPEC]) atomicAdd(&a.stats[5], (unsigned long long)(unsigned)c[CT_SPEC]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

}  // namespace pp

template <bool PROF, int N3>
static cudaError_t launch_pp(const TcArgs& a, const CUtensorMap& wmap, int ntiles, cudaStream_t stream) {
  // layer-1 k-steps for the width class (tc_k1_needed(J) <= tc_rj(N3) + N3 + 1 = 2 N3 + 1)
  constexpr int KS1 = (2 * N3 + 1 + 15) / 16 < kTcK1 / 16 ? (2 * N3 + 1 + 15) / 16 : kTcK1 / 16;
  const size_t smem = pp::Layout::total;
  const cudaError_t e = ensure_dyn_smem((const void*)pp::k_sweep_pp<PROF, N3, KS1>, smem);
  if (e != cudaSuccess) return e;
  pp::k_sweep_pp<PROF, N3, KS1><<<ntiles, pp::kBlock, smem, stream>>>(a, wmap);
  return cudaGetLastError();
}

int tc_pp_width_class(int J) { return J <= 16 ? 16 : J <= 32 ? 32 : J <= 64 ? 64 : kTcN3; }

cudaError_t launch_tc_pp(const TcArgs& a, const CUtensorMap& wmap, int ntiles, cudaStream_t stream) {
  if (a.prof) return launch_pp<true, kTcN3>(a, wmap, ntiles, stream);  // (debug profiles: the C3 shape)
  switch (a.n3) {
    case 16: return launch_pp<false, 16>(a, wmap, ntiles, stream);
    case 32: return launch_pp<false, 32>(a, wmap, ntiles, stream);
    case 64: return launch_pp<false, 64>(a, wmap, ntiles, stream);
    default: return launch_pp<false, kTcN3>(a, wmap, ntiles, stream);
  }
}

}  // namespace pcd
