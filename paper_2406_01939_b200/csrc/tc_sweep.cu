// tc_sweep.cu — the tcgen05 product-partition sweep (see tc_sweep.cuh).
//
// Per step, for the 128 processes (rows) of the CTA:
//   P  threads 0..127 issue the loads their row's update will need (cache,
//      written, ref, ev at t; product/rrow of the next slot; the slot after) —
//      consumed only in U, so their latency hides behind the step;
//   F  16 warps x 8 rows: batched loads of the checkpoint-count row hck[b],
//      the row's D = Hown - F and the partial block of effective events, then
//      the capacity part of the features (c/c0) and the feasibility mask.
//      The inventory part (x/x0) stays resident in smem between steps (it
//      changes only when the process fulfils from its own product);
//   L1/E1/L2/E2/L3  three tcgen05 GEMM layers (fp16x3, fp32 TMEM accumulate)
//      with tanh epilogues writing the next layer's A operand;
//   S  scores r_j - q_j, argmax, decision margin; rows with margin < guard are
//      re-evaluated exactly (FP64, warp_policy_eval<kDual>);
//   U  publish + counters + state deltas (thread per row).
#include <cuda_runtime.h>

#include "tc_sweep.cuh"

namespace pcd {

constexpr int kTcWarps = 8;
constexpr int kGroups = kTcWarps / 4;             // TMEM column groups per lane quarter
constexpr int kTcBlock = kTcWarps * 32;
constexpr int kRowsPerWarp = kTcRows / kTcWarps;  // 16
constexpr int kInfo = 16;                          // ints of per-row state
constexpr int kMaxJ = 103;                         // 2J+1 <= 208
constexpr int kScrJ = 104;
constexpr int kRecheckWarps = 6;                   // concurrent exact re-evaluations
constexpr int kRecheckStride = 5376;               // bytes of FP64 scratch per warp

// per-row state (sInfo[r*kInfo + .])
enum {
  RI_T = 0,   // slot of the current step
  RI_P,       // its product
  RI_POS,     // CSR position of the current step
  RI_END,     // CSR end of the window
  RI_ANY,     // -1 inactive, 0 nothing feasible, 1 evaluate
  RI_DEC,     // decision
  RI_FLAG,    // 0 / 1 flagged / 2 verify-only
  RI_RR,      // reward row of t
  RI_TN,      // slot of the next step
  RI_XDIRTY,  // reload the inventory features of the row
  RI_XUPD,    // node whose inventory feature changed in the last step (-1)
  RI_OT,      // Order::t of the current step
  RI_EVT      // effective cached attempt at the last step's slot (-1): Hown += 1
};

// spreads the 16 low bits of x onto the even bit positions of a 32-bit word
__device__ __forceinline__ uint32_t spread16(uint32_t x) {
  x &= 0xffffu;
  x = (x | (x << 8)) & 0x00ff00ffu;
  x = (x | (x << 4)) & 0x0f0f0f0fu;
  x = (x | (x << 2)) & 0x33333333u;
  x = (x | (x << 1)) & 0x55555555u;
  return x;
}

struct TcSmemLayout {
  static constexpr int w = 0;
  static constexpr int a = kWImgBytes;                    // 98,304
  static constexpr int scr = a + 2 * kABytes;            // 16 warps x 104 ints
  static constexpr int mask = scr + kTcWarps * kScrJ * 4; // feasibility, 128 x 4 words
  static constexpr int xbit = mask + kTcRows * 4 * 4;     // x > 0, 128 x 4 words
  static constexpr int info = xbit + kTcRows * 4 * 4;     // 128 x 16 ints
  static constexpr int best = info + kTcRows * kInfo * 4; // 128 x 4 groups x 3
  static constexpr int cap = best + kTcRows * 12 * 4;     // checkpoint capacities
  static constexpr int ctl = cap + 128 * 4;               // [0] active [1] nflag [2..130) flagged
  static constexpr int cst = ctl + 136 * 4;               // invc0[104] b1[64] b2[64] b3[112]
  static constexpr int bar = cst + 344 * 4;
  static constexpr int tmem = bar + 8;
  static constexpr int total = tmem + 8;
};
static_assert(TcSmemLayout::total <= 232448, "tc sweep shared memory budget");

__host__ size_t tc_smem_bytes() { return TcSmemLayout::total; }

__device__ __forceinline__ void put_feature(unsigned char* sA, int r, int k, float v) {
  __half h, l;
  split_f16(v, h, l);
  const int off = canon_off(128, r, k);
  *(__half*)(sA + off) = h;
  *(__half*)(sA + kABytes + off) = l;
}
__device__ __forceinline__ void put_feature_at(unsigned char* sA, int off, float v) {
  __half h, l;
  split_f16(v, h, l);
  *(__half*)(sA + off) = h;
  *(__half*)(sA + kABytes + off) = l;
}
// canonical offset of column k for row 0 (add (r>>3)*128 + (r&7)*16 for row r)
__device__ __forceinline__ int kcol_off(int k) { return (k >> 3) * 2048 + (k & 7) * 2; }
__device__ __forceinline__ int row_off(int r) { return (r >> 3) * 128 + (r & 7) * 16; }

// fp32 pair -> (hi, lo) fp16x2 with lo scaled by 2^11
__device__ __forceinline__ void split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 hf = __half22float2(h);
  const __half2 l = __floats2half2_rn((x0 - hf.x) * kLoScale, (x1 - hf.y) * kLoScale);
  hi = *(const uint32_t*)&h;
  lo = *(const uint32_t*)&l;
}

__global__ void __launch_bounds__(kTcBlock, 1) k_sweep_product_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const SweepArgs& S = a.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = S.J, lo = S.lo, hi = S.hi;
  unsigned char* sW = smem + TcSmemLayout::w;
  unsigned char* sA = smem + TcSmemLayout::a;
  int* sScr = (int*)(smem + TcSmemLayout::scr);
  uint32_t* sMask = (uint32_t*)(smem + TcSmemLayout::mask);
  uint32_t* sXbit = (uint32_t*)(smem + TcSmemLayout::xbit);
  int* sInfo = (int*)(smem + TcSmemLayout::info);
  float* sBest = (float*)(smem + TcSmemLayout::best);
  int* sCap = (int*)(smem + TcSmemLayout::cap);
  int* sCtl = (int*)(smem + TcSmemLayout::ctl);
  uint64_t* sBar = (uint64_t*)(smem + TcSmemLayout::bar);
  uint32_t* sTmem = (uint32_t*)(smem + TcSmemLayout::tmem);
  float* sInvC0 = (float*)(smem + TcSmemLayout::cst);
  float* sB1 = sInvC0 + 104;
  float* sB2 = sB1 + 64;
  float* sB3 = sB2 + 64;
  const int tile = blockIdx.x;
  int* Dtile = a.D + (size_t)tile * kTcRows * J;
  // The inventory features persist in smem only if the hidden-layer operands
  // (k-chunks 0..7) never overlap them, i.e. J >= 64.
  const bool xpersist = J >= 64;

  // ---------------------------------------------------------------- setup
  {
    const uint4* src = (const uint4*)a.wimg;
    uint4* dst = (uint4*)sW;
    for (int i = tid; i < kWImgBytes / 16; i += kTcBlock) dst[i] = src[i];
    uint4* da = (uint4*)sA;  // zero padding columns / idle rows once
    for (int i = tid; i < 2 * kABytes / 16; i += kTcBlock) da[i] = make_uint4(0, 0, 0, 0);
  }
  for (int i = tid; i < kTcRows * J; i += kTcBlock) Dtile[i] = 0;
  for (int j = tid; j < J; j += kTcBlock) {
    sCap[j] = S.ckcap[j];
    sInvC0[j] = a.inv_c0[j];
  }
  for (int i = tid; i < kTcH; i += kTcBlock) {
    sB1[i] = a.b1f[i];
    sB2[i] = a.b2f[i];
  }
  for (int i = tid; i < kTcN3; i += kTcBlock) sB3[i] = a.b3f[i];
  if (tid < kTcRows) {
    const int m = a.rows[tile * kTcRows + tid];
    int pos = 0, end = 0;
    if (m >= 0) {
      const int beg = S.pstart[m], n = S.pstart[m + 1] - beg;
      pos = beg + lower_bound_i32(S.pslots + beg, n, lo);
      end = beg + lower_bound_i32(S.pslots + beg, n, hi);
    }
    int* inf = sInfo + tid * kInfo;
    inf[RI_POS] = pos;
    inf[RI_END] = end;
    inf[RI_XDIRTY] = 1;
    inf[RI_XUPD] = -1;
    inf[RI_EVT] = -1;
    inf[RI_P] = -1;
    if (pos < end) {
      const int t = S.pslots[pos];
      inf[RI_T] = t;
      inf[RI_P] = S.model.product[t];
      inf[RI_RR] = S.model.rrow[t];
      inf[RI_OT] = S.model.order_t ? S.model.order_t[t] : t;
      inf[RI_TN] = pos + 1 < end ? S.pslots[pos + 1] : -1;
    }
  }
  if (tid == 0) {
    sCtl[0] = 0;
    sCtl[1] = 0;
    mbar_init(sBar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sTmem)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *sTmem;

  const uint32_t aBase = smem_u32(sA);
  const uint32_t w1h = smem_u32(sW), w1l = w1h + kW1Bytes;
  const uint32_t w2h = w1l + kW1Bytes, w2l = w2h + kW2Bytes;
  const uint32_t w3h = w2l + kW2Bytes, w3l = w3h + kW3Bytes;
  // hidden operands (R=128, K=64) live in k-chunks 0..7 of the feature buffer
  const uint32_t hHi = aBase, hLo = aBase + kABytes;
  const uint32_t id64 = idesc_f16(128, 64), id112 = idesc_f16(128, kTcN3);
  // base UMMA descriptors (issuing thread only); a k-step advances the 14-bit start address
#define UMMA_BASES                                                                               \
  const uint64_t dA = umma_desc(aBase, 2048, 128), dAl = umma_desc(aBase + kABytes, 2048, 128); \
  const uint64_t dW1 = umma_desc(w1h, 1024, 128), dW1l = umma_desc(w1l, 1024, 128);             \
  const uint64_t dW2 = umma_desc(w2h, 1024, 128), dW2l = umma_desc(w2l, 1024, 128);             \
  const uint64_t dW3 = umma_desc(w3h, 16 * kTcN3, 128), dW3l = umma_desc(w3l, 16 * kTcN3, 128); \
  (void)dW1; (void)dW1l; (void)dW2; (void)dW2l; (void)dW3; (void)dW3l
  uint32_t phase = 0;
  // t/T in fp32 (the exact FP64 path recomputes it for flagged rows)
  const float invT = S.model.horizon > 0 ? (float)(1.0 / (double)S.model.horizon) : 0.f;
  int koff[2];  // canonical column offsets of this lane's capacity-feature pairs
#pragma unroll
  for (int c = 0; c < 2; ++c) koff[c] = kcol_off(64 * c + 2 * lane);
  auto Drow_st = [&](int r, int j, int v) { Dtile[(size_t)r * J + j] = v; };

  unsigned long long changed = 0, conflicts = 0, first = ~0ull, st_tc = 0, st_flag = 0, st_dis = 0,
                     st_bad = 0;
  long long mism = 0;
  unsigned long long nev = 0;  // evaluations of row `tid` (tid < 128)

  long long pacc[20] = {0};
  long long fl = 0;
  long long plast = clock64();
  const bool prof_on = a.prof && blockIdx.x == 0 && tid == 0;
#define PMARK(k) do { if (prof_on) { const long long now_ = clock64(); pacc[k] += now_ - plast; plast = now_; } } while (0)
  for (;;) {
    // ============================ P: prefetch the update's operands (rows)
    int u_ev = -1, u_old = 0, u_wr = 0, u_ref = 0, u_pn = -1, u_rrn = 0, u_otn = 0, u_tnn = -1;
    if (tid < kTcRows) {
      const int* inf = sInfo + tid * kInfo;
      const int pos = inf[RI_POS], end = inf[RI_END];
      if (pos < end) {
        const int t = inf[RI_T];
        u_ev = S.ev[t];
        u_old = S.cache[t];
        u_wr = S.written[t];
        if (S.ref) u_ref = S.ref[t];
        const int tn = inf[RI_TN];
        if (tn >= 0) {
          u_pn = S.model.product[tn];
          u_rrn = S.model.rrow[tn];
          u_otn = S.model.order_t ? S.model.order_t[tn] : tn;
        }
        if (pos + 2 < end) u_tnn = S.pslots[pos + 2];
      }
    }

    // ============================ F: local state + capacity features
    {
      int active_w = 0;
#pragma unroll 1
      for (int i0 = 0; i0 < kRowsPerWarp; i0 += 4) {
        int hv[4][2][2], dv[4][2][2], evp[4], xu[4], xdirty[4], xupd[4], evtp[4];
        float xi[4];
        bool act[4];
        if (prof_on) fl = clock64();
        // -- batched loads of 4 rows (one memory round trip)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = warp + kTcWarps * (i0 + i);
          const int* inf = sInfo + r * kInfo;
          act[i] = inf[RI_POS] < inf[RI_END];
          xdirty[i] = inf[RI_XDIRTY];
          xupd[i] = inf[RI_XUPD];
          evtp[i] = inf[RI_EVT];
          evp[i] = -1;
          xu[i] = 0;
          xi[i] = 0.f;
          if (act[i]) {
            const int t = inf[RI_T];
            const int b = a.fake ? 0 : (t - lo) >> kLogK;  // fake: timing experiment only
            const int* hb = S.hck + (size_t)b * J;
            const int* Drow = Dtile + (size_t)r * J;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              const int j0 = 64 * c + 2 * lane;
              hv[i][c][0] = j0 < J ? __ldg(hb + j0) : 0;
              hv[i][c][1] = j0 + 1 < J ? __ldg(hb + j0 + 1) : 0;
              dv[i][c][0] = j0 < J ? Drow[j0] : 0;
              dv[i][c][1] = j0 + 1 < J ? Drow[j0 + 1] : 0;
            }
            const int s = lo + (b << kLogK) + lane;
            if (s < t) evp[i] = S.ev[s];
            if (xupd[i] >= 0 && !xdirty[i]) {
              xu[i] = S.xloc[(size_t)inf[RI_P] * J + xupd[i]];
              xi[i] = __ldg(a.inv_x0 + (size_t)inf[RI_P] * J + xupd[i]);
            }
          }
        }
        __syncwarp();
        if (prof_on) { const long long n_ = clock64(); pacc[12] += n_ - fl; fl = n_; }
        // -- (A) inventory features + D deltas, 4 independent rows
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int r = warp + kTcWarps * (i0 + i);
          int* inf = sInfo + r * kInfo;
          if (!act[i]) {
            if (lane == 0) inf[RI_ANY] = -1;
            continue;
          }
          ++active_w;
          const int ro = row_off(r);
          if (xdirty[i] || !xpersist) {  // full reload (first step / product change)
            const int p = inf[RI_P];
            const int* xr = S.xloc + (size_t)p * J;
            const float* ix0 = a.inv_x0 + (size_t)p * J;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const int j = c * 32 + lane;
              const int xj = j < J ? xr[j] : 0;
              if (j < J) put_feature_at(sA, ro + kcol_off(J + j), (float)xj * ix0[j]);
              const uint32_t bal = __ballot_sync(0xffffffffu, xj > 0);
              if (lane == 0) sXbit[r * 4 + c] = bal;
            }
            if (lane == 0) inf[RI_XDIRTY] = 0;
          } else if (xupd[i] >= 0 && lane == 4 + i) {  // single-entry update
            const int j = xupd[i];
            put_feature_at(sA, ro + kcol_off(J + j), (float)xu[i] * xi[i]);
            if (xu[i] <= 0) sXbit[r * 4 + (j >> 5)] &= ~(1u << (j & 31));
          }
          if (lane == 8 + i) {
            inf[RI_XUPD] = -1;
            inf[RI_EVT] = -1;
          }
          // D = Hown - F: apply last step's two deltas in registers, write back
          const int evt = evtp[i], dl = xupd[i];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int j0 = 64 * c + 2 * lane;
            if (evt == j0) { dv[i][c][0] += 1; Drow_st(r, j0, dv[i][c][0]); }
            if (evt == j0 + 1) { dv[i][c][1] += 1; Drow_st(r, j0 + 1, dv[i][c][1]); }
            if (dl == j0) { dv[i][c][0] -= 1; Drow_st(r, j0, dv[i][c][0]); }
            if (dl == j0 + 1) { dv[i][c][1] -= 1; Drow_st(r, j0 + 1, dv[i][c][1]); }
          }
        }
        if (prof_on) { const long long n_ = clock64(); pacc[13] += n_ - fl; fl = n_; }
        // -- (B) partial block [lo + bK, t): per-row uint8 event counts
        uint32_t* cnt = (uint32_t*)(sScr + warp * kScrJ);  // 4 rows x 26 words
        if (lane < 26) {
#pragma unroll
          for (int i = 0; i < 4; ++i) cnt[i * 26 + lane] = 0u;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (evp[i] >= 0) atomicAdd(&cnt[i * 26 + (evp[i] >> 2)], 1u << (8 * (evp[i] & 3)));
        __syncwarp();
        if (prof_on) { const long long n_ = clock64(); pacc[14] += n_ - fl; fl = n_; }
        // -- (C) capacity features c = max(0, ckcap - H_t + Hown - F)
        //        for 4 independent rows (no syncs between rows: ILP)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (!act[i]) continue;
          const int r = warp + kTcWarps * (i0 + i);
          const int ro = row_off(r);
          const unsigned char* cb = (const unsigned char*)(cnt + i * 26);
          uint32_t any = 0;
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int j0 = 64 * c + 2 * lane;
            bool f0 = false, f1 = false;
            if (j0 < J) {
              const uint16_t pc = *(const uint16_t*)(cb + j0);
              const int c0 = max(sCap[j0] - hv[i][c][0] + dv[i][c][0] - (int)(pc & 0xff), 0);
              const int c1 = j0 + 1 < J ? max(sCap[j0 + 1] - hv[i][c][1] + dv[i][c][1] - (int)(pc >> 8), 0) : 0;
              const uint32_t xb = sXbit[r * 4 + (j0 >> 5)];
              f0 = c0 > 0 && ((xb >> (j0 & 31)) & 1u);
              f1 = c1 > 0 && ((xb >> ((j0 + 1) & 31)) & 1u);
              uint32_t h2, l2;
              split2((float)c0 * sInvC0[j0], (float)c1 * sInvC0[j0 + 1], h2, l2);
              if (j0 + 1 < J) {
                *(uint32_t*)(sA + ro + koff[c]) = h2;
                *(uint32_t*)(sA + kABytes + ro + koff[c]) = l2;
              } else {  // odd J: the neighbour column belongs to the x part
                *(uint16_t*)(sA + ro + koff[c]) = (uint16_t)h2;
                *(uint16_t*)(sA + kABytes + ro + koff[c]) = (uint16_t)l2;
              }
            }
            const uint32_t E = __ballot_sync(0xffffffffu, f0), O = __ballot_sync(0xffffffffu, f1);
            if (lane < 2) {  // two lanes pack the two 32-column words in parallel
              const uint32_t e = lane ? E >> 16 : E & 0xffffu, o = lane ? O >> 16 : O & 0xffffu;
              sMask[r * 4 + 2 * c + lane] = spread16(e) | (spread16(o) << 1);
            }
            any |= E | O;
          }
          int* inf = sInfo + r * kInfo;
          if (lane == 2) put_feature_at(sA, ro + kcol_off(2 * J), (float)inf[RI_OT] * invT);
          if (lane == 3) inf[RI_ANY] = any ? 1 : 0;
        }
        if (prof_on) { const long long n_ = clock64(); pacc[16] += n_ - fl; fl = n_; }
      }
      if (prof_on) pacc[11] += clock64() - plast;  // warp 0's own F work
      if (lane == 0 && active_w) atomicAdd(&sCtl[0], active_w);
    }
    fence_async_smem();
    __syncthreads();
    PMARK(0);
    if (sCtl[0] == 0) break;
    if (prof_on) pacc[10] += 1;

    // ============================ layer 1: z1 = F . W1^T  (3 products)
    if (tid == 0) {
      tc_fence_after();
      UMMA_BASES;
#pragma unroll
      for (int s = 0; s < kTcK1 / 16; ++s) {
        const uint64_t ah = dA + s * (4096 >> 4), al = dAl + s * (4096 >> 4);
        const uint64_t bh = dW1 + s * (2048 >> 4), bl = dW1l + s * (2048 >> 4);
        mma_f16(tmem + 0, ah, bh, id64, s > 0);
        mma_f16(tmem + 64, ah, bl, id64, s > 0);
        mma_f16(tmem + 64, al, bh, id64, 1);
      }
      mma_commit(sBar);
    }
    mbar_wait(sBar, phase);
    PMARK(1);
    phase ^= 1;
    tc_fence_after();

    // ============================ hidden epilogues (z -> tanh -> fp16 hi/lo)
    auto hidden_epilogue = [&](uint32_t col_hh, uint32_t col_x, const float* bias) {
      const int q4 = warp & 3, qc = warp >> 2;  // TMEM lane quarter, column group
      const int r = 32 * q4 + lane;
      const uint32_t lane_off = (uint32_t)(32 * q4) << 16;
#pragma unroll
      for (int cc = 0; cc < kTcH / kGroups; cc += 16) {
        const int cb = qc * (kTcH / kGroups) + cc;
        float vh[16], vx[16];
        tmem_ld16(tmem + lane_off + col_hh + cb, vh);
        tmem_ld16(tmem + lane_off + col_x + cb, vx);
        tmem_wait_ld();
        uint32_t ph[8], pl[8];
#pragma unroll
        for (int i = 0; i < 16; i += 2) {
          const float z0 = fmaf(vx[i], kLoInv, vh[i]) + bias[cb + i];
          const float z1 = fmaf(vx[i + 1], kLoInv, vh[i + 1]) + bias[cb + i + 1];
          split2(tanh_f32(z0), tanh_f32(z1), ph[i / 2], pl[i / 2]);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // two 8-column chunks
          const int off = canon_off(128, r, cb + 8 * h);
          *(uint4*)(sA + off) = make_uint4(ph[4 * h], ph[4 * h + 1], ph[4 * h + 2], ph[4 * h + 3]);
          *(uint4*)(sA + kABytes + off) = make_uint4(pl[4 * h], pl[4 * h + 1], pl[4 * h + 2], pl[4 * h + 3]);
        }
      }
    };
    hidden_epilogue(0, 64, sB1);
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    PMARK(2);

    // ============================ layer 2
    if (tid == 0) {
      tc_fence_after();
      UMMA_BASES;
#pragma unroll
      for (int s = 0; s < kTcH / 16; ++s) {
        const uint64_t ah = dA + s * (4096 >> 4), al = dAl + s * (4096 >> 4);
        const uint64_t bh = dW2 + s * (2048 >> 4), bl = dW2l + s * (2048 >> 4);
        mma_f16(tmem + 128, ah, bh, id64, s > 0);
        mma_f16(tmem + 192, ah, bl, id64, s > 0);
        mma_f16(tmem + 192, al, bh, id64, 1);
      }
      mma_commit(sBar);
    }
    mbar_wait(sBar, phase);
    PMARK(3);
    phase ^= 1;
    tc_fence_after();
    hidden_epilogue(128, 192, sB2);  // h2 overwrites h1 (L2 has completed)
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    PMARK(4);

    // ============================ layer 3: q = h2 . W3'^T (N = 112)
    if (tid == 0) {
      tc_fence_after();
      UMMA_BASES;
#pragma unroll
      for (int s = 0; s < kTcH / 16; ++s) {
        const uint64_t ah = dA + s * (4096 >> 4), al = dAl + s * (4096 >> 4);
        const uint64_t bh = dW3 + s * ((2 * 16 * kTcN3) >> 4), bl = dW3l + s * ((2 * 16 * kTcN3) >> 4);
        mma_f16(tmem + 0, ah, bh, id112, s > 0);
        mma_f16(tmem + kTcN3, ah, bl, id112, s > 0);
        mma_f16(tmem + kTcN3, al, bh, id112, 1);
      }
      mma_commit(sBar);
    }
    // issue this thread's reward loads while layer 3 runs
    const int s_q4 = warp & 3, s_qc = warp >> 2;
    const int s_r = 32 * s_q4 + lane;
    constexpr int kSCols = (kTcN3 / 16 + kGroups - 1) / kGroups * 16;  // 64 for 2 groups
    const int s_c0 = s_qc * kSCols;
    const int s_ncols = min(kSCols, kTcN3 - s_c0);
    const bool s_eval = sInfo[s_r * kInfo + RI_ANY] == 1;
    uint64_t s_mk = 0;
    if (s_eval) {
      s_mk = sMask[s_r * 4 + (s_c0 >> 5)];
      if (kSCols > 32 && (s_c0 >> 5) + 1 < 4) s_mk |= (uint64_t)sMask[s_r * 4 + (s_c0 >> 5) + 1] << 32;
    }
    float rwv[kSCols];
    {
      const float* rw = a.rtabf + (size_t)(s_eval ? sInfo[s_r * kInfo + RI_RR] : 0) * J;
      if ((J & 3) == 0) {  // 16-byte aligned rows: vector loads
#pragma unroll
        for (int i = 0; i < kSCols; i += 4) {
          if (s_c0 + i < J && ((s_mk >> i) & 0xfull)) {
            const float4 v = __ldg((const float4*)(rw + s_c0 + i));
            rwv[i] = v.x; rwv[i + 1] = v.y; rwv[i + 2] = v.z; rwv[i + 3] = v.w;
          } else {
            rwv[i] = rwv[i + 1] = rwv[i + 2] = rwv[i + 3] = 0.f;
          }
        }
      } else {
#pragma unroll
        for (int i = 0; i < kSCols; ++i) rwv[i] = ((s_mk >> i) & 1ull) ? __ldg(rw + s_c0 + i) : 0.f;
      }
    }
    mbar_wait(sBar, phase);
    PMARK(5);
    phase ^= 1;
    tc_fence_after();

    // ============================ S: scores, argmax, margin (column groups)
    {
      const int qc = s_qc, r = s_r, c0 = s_c0;
      const uint32_t lane_off = (uint32_t)(32 * s_q4) << 16;
      const uint64_t mk = s_mk;
      float v1 = -INFINITY, v2 = -INFINITY;
      int i1 = -1;
      bool bad = false;
#pragma unroll
      for (int hf = 0; hf < kSCols / 16; ++hf) {
        if (16 * hf >= s_ncols) break;  // warp-uniform
        float vh[16], vx[16];
        tmem_ld16(tmem + lane_off + c0 + 16 * hf, vh);
        tmem_ld16(tmem + lane_off + kTcN3 + c0 + 16 * hf, vx);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int j = c0 + 16 * hf + i;
          if (!((mk >> (16 * hf + i)) & 1ull)) continue;  // feasible implies j < J
          const float q = fmaf(vx[i], kLoInv, vh[i]) + sB3[j];
          const float sc = rwv[16 * hf + i] - q;
          if (!isfinite(sc)) bad = true;
          if (sc > v1) { v2 = v1; v1 = sc; i1 = j; }
          else if (sc > v2) v2 = sc;
        }
      }
      float* bs = sBest + r * 12 + qc * 3;
      bs[0] = v1;
      bs[1] = __int_as_float(bad ? -2 : i1);
      bs[2] = v2;
    }
    tc_fence_before();
    __syncthreads();
    PMARK(6);
    if (tid < kTcRows) {
      const int r = tid;
      int* inf = sInfo + r * kInfo;
      inf[RI_FLAG] = 0;
      if (inf[RI_ANY] == 0) {
        inf[RI_DEC] = -1;
      } else if (inf[RI_ANY] == 1) {
        const float* bs = sBest + r * 12;
        float v1 = bs[0], v2 = bs[2];
        int i1 = __float_as_int(bs[1]);
        bool bad = i1 == -2;
        for (int g = 1; g < kGroups; ++g) {
          const float w1 = bs[3 * g], w2 = bs[3 * g + 2];
          const int j1 = __float_as_int(bs[3 * g + 1]);
          bad |= j1 == -2;
          if (w1 > v1) { v2 = fmaxf(v1, w2); v1 = w1; i1 = j1; }
          else v2 = fmaxf(v2, w1);
        }
        inf[RI_DEC] = v1 >= 0.f ? i1 : -1;
        const bool flag = bad || i1 < 0 || !(v1 - v2 >= a.guard) || !(fabsf(v1) >= a.guard);
        ++st_tc;
        if (flag || a.verify) {
          inf[RI_FLAG] = flag ? 1 : 2;
          const int k = atomicAdd(&sCtl[1], 1);
          sCtl[2 + k] = r;
        }
      }
    }
    __syncthreads();
    PMARK(7);

    // ============================ exact FP64 re-evaluation of flagged rows
    const int nflag = sCtl[1];
    if (warp < kRecheckWarps) {
      for (int fi = warp; fi < nflag; fi += kRecheckWarps) {
        const int r = sCtl[2 + fi];
        int* inf = sInfo + r * kInfo;
        const int t = inf[RI_T], p = inf[RI_P];
        const int b = (t - lo) >> kLogK;
        // scratch: k-chunks 0..7 of the hi (warps 0-2) / lo (3-5) feature
        // buffers — they held h2, dead since layer 3 completed
        unsigned char* base = sA + (warp < 3 ? 0 : kABytes) + (warp % 3) * kRecheckStride;
        int* caps = (int*)base;
        int* row = caps + kScrJ;
        double* d = (double*)(base + 2 * kScrJ * 4);
        WarpScratch ws{d, d + 2 * kMaxJ + 1, d + 2 * kMaxJ + 1 + kTcH, d + 2 * kMaxJ + 1 + 2 * kTcH};
        const int* hb = S.hck + (size_t)b * J;
        const int* Drow = Dtile + (size_t)r * J;
        for (int j = lane; j < J; j += 32) {
          caps[j] = sCap[j] - hb[j] + Drow[j];
          row[j] = S.xloc[(size_t)p * J + j];
        }
        __syncwarp();
        const int s = lo + (b << kLogK) + lane;
        if (s < t) {
          const int e = S.ev[s];
          if (e >= 0) atomicSub(&caps[e], 1);
        }
        __syncwarp();
        for (int j = lane; j < J; j += 32) caps[j] = max(caps[j], 0);
        __syncwarp();
        int nonfinite = 0;
        const int exact = warp_policy_eval<kDual>(S.model, caps, row, t, ws, lane, &nonfinite);
        if (lane == 0) {
          if (nonfinite) {
            const int m = a.rows[tile * kTcRows + r];
            atomicMin(&S.scal->err_nonfinite, ((unsigned long long)m << 32) | (unsigned)inf[RI_OT]);
          }
          if (inf[RI_FLAG] == 1) {
            ++st_flag;
            st_dis += exact != inf[RI_DEC];
          } else {
            st_bad += exact != inf[RI_DEC];
          }
          inf[RI_DEC] = exact;
        }
        __syncwarp();
      }
    }
    __syncthreads();
    PMARK(8);

    // ============================ U: update + publish (thread r = row r)
    if (tid < kTcRows) {
      const int r = tid;
      int* inf = sInfo + r * kInfo;
      if (inf[RI_ANY] >= 0) {
        const int t = inf[RI_T], p = inf[RI_P], dec = inf[RI_DEC];
        // D deltas are applied by the row's F warp next step (no RMW here)
        inf[RI_EVT] = u_ev;
        if (dec >= 0) {
          atomicSub(&S.xloc[(size_t)p * J + dec], 1);  // fire-and-forget RED
          inf[RI_XUPD] = dec;
        }
        if (dec != u_old) {
          ++changed;
          first = min(first, (unsigned long long)t);
          conflicts += u_wr ? 1 : 0;
        }
        if (S.ref) mism += (long long)(dec != u_ref) - (long long)(u_old != u_ref);
        S.cache[t] = dec;
        S.written[t] = 1;
        ++nev;
        const int pos = inf[RI_POS] + 1;
        inf[RI_POS] = pos;
        if (pos < inf[RI_END]) {
          const int tn = inf[RI_TN];
          // warm L2 with the next step's checkpoint-count row
          const int* hbn = S.hck + (size_t)((tn - lo) >> kLogK) * J;
          for (int q = 0; q < J; q += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(hbn + q));
          inf[RI_T] = tn;
          if (u_pn != p) inf[RI_XDIRTY] = 1;
          inf[RI_P] = u_pn;
          inf[RI_RR] = u_rrn;
          inf[RI_OT] = u_otn;
          inf[RI_TN] = u_tnn;
        }
      }
      if (tid == 0) {
        sCtl[0] = 0;
        sCtl[1] = 0;
      }
    }
    __syncthreads();
    PMARK(9);
  }

  // ---------------------------------------------------------------- teardown
  if (prof_on)
    for (int k = 0; k < 17; ++k) a.prof[k] = pacc[k];
#undef PMARK
  if (tid < kTcRows) {
    const int m = a.rows[tile * kTcRows + tid];
    if (m >= 0) {
      atomicMax(&S.scal->max_evals, nev);
      atomicAdd(&S.scal->total_evals, nev);
      if (S.evals_out) S.evals_out[m] = (long long)nev;
    }
  }
  if (changed) {
    atomicAdd(&S.scal->changed, changed);
    atomicAdd(&S.scal->conflicts, conflicts);
    atomicMin(&S.scal->first_changed, first);
  }
  if (mism) atomicAdd((unsigned long long*)&S.scal->mismatch_delta, (unsigned long long)mism);
  if (st_flag) atomicAdd(&a.stats[1], st_flag);
  if (st_tc) atomicAdd(&a.stats[0], st_tc);
  if (st_dis) atomicAdd(&a.stats[2], st_dis);
  if (st_bad) atomicAdd(&a.stats[3], st_bad);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256));
  }
}

void launch_tc_sweep(const TcArgs& a, int ntiles, cudaStream_t stream) {
  static bool attr = false;
  const size_t smem = tc_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_product_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  k_sweep_product_tc<<<ntiles, kTcBlock, smem, stream>>>(a);
}

}  // namespace pcd
