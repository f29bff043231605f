// tc_sweep.cu — the tcgen05 product-partition sweep (see tc_sweep.cuh).
//
// Work distribution: one CTA per SM, 128 rows (processes in flight). The
// engine sorts the processes with window slots by load (desc) into wq; entry
// k < tiles*128 starts on row k / tiles of tile k % tiles, and a row whose
// process is done pulls the next entry (atomic counter), so every row works
// until the list is drained (list scheduling, longest first).
//
// Thread mapping: thread (warp w, lane l) owns row r = 32*(w%4) + l — the
// TMEM lane it may access — and column group g = w/4 (nodes [32g, 32g+32)).
// Warps 12..15 (group 3, at most one 8-node chunk) are also the row agents:
// per-row bookkeeping, the update's operand loads, publish.
//
// Per-row state that lives on chip for the whole launch:
//   TMEM cols 256..383  D = Hown - F (int32, one lane per row)
//   TMEM cols 384..511  the integer capacities of the current step (read by
//                       the exact re-evaluation of flagged rows)
//   smem                inventory features x/x0 (columns J..2J-1 of the A
//                       operand, updated in place), per-row bookkeeping and
//                       counters
//   registers           x > 0 bits and the feasibility mask of (row, group)
//
// Per step, for the 128 processes (rows) of the CTA:
//   P  row agents issue the loads their row's update will need (cache,
//      written, ref, ev at t; product/rrow of the next slot; the slot after)
//      and warm L2 with the next step's checkpoint row;
//   F  thread (row, group): one batch of loads (the checkpoint row hck[b] for
//      its nodes, the 8-slot event block, D from TMEM), then
//      c = max(0, ckcap - hck + D - partial) per node (partial events as
//      packed nibble counts, the two D deltas of the last step), the capacity
//      features c/c0 (fp16 hi/lo), the feasibility bits;
//   L1/E1/L2/E2/L3  three tcgen05 GEMM layers (fp16x3, fp32 TMEM accumulate)
//      with tanh epilogues writing the next layer's A operand;
//   S  scores r_j - q_j, argmax and decision margin per (row, group); the row
//      agents combine the groups; rows with margin < guard are re-evaluated
//      exactly (FP64, warp_policy_eval<kDual>) by the warp of their TMEM lanes;
//   U  row agents: publish + counters + state deltas.
#include <cuda_runtime.h>

#include <climits>
#include <cstdio>
#include <type_traits>

#include "tc_sweep.cuh"

namespace pcd {

constexpr int kTcWarps = 16;
constexpr int kGroups = kTcWarps / 4;      // column groups (warps w, w+4, ... share TMEM lanes)
constexpr int kTcBlock = kTcWarps * 32;
constexpr int kGC = 32;                    // nodes per column group
constexpr int kGChunks = kGC / 8;          // 8-node chunks per group
constexpr int kInfo = 28;                  // ints of per-row state
constexpr int kMaxJ = 103;                 // 2J+1 <= 208
constexpr int kScrJ = 112;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColD = 256, kColCap = 384;
static_assert(kGroups * kGC >= kTcN3 && kGroups * kGC <= 128, "column groups cover the score columns");
static_assert(kMaxJ <= (kGroups - 1) * kGC + 8, "the row agents' group holds at most one 8-node chunk");

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
  RI_XUPD,    // node whose own inventory dropped in the last step (-1): F += 1
  RI_OT,      // Order::t of the current step
  RI_EVT,     // effective cached attempt at the last step's slot (-1): Hown += 1
  RI_X,       // run of the current step (row of xloc)
  RI_M,       // process of the row (-1 idle)
  RI_DRESET,  // a new process started: D = 0
  // operands of this step's update, loaded by the row agent at the step start
  RI_UEV, RI_UOLD, RI_UWR, RI_UREF, RI_UPN, RI_URRN, RI_UOTN, RI_UTNN, RI_UXN
};
static_assert(RI_UXN < kInfo, "per-row state fits");
// per-row counters of the launch (sCnt[k * 128 + r], row agents)
enum { CN_CHANGED = 0, CN_CONFLICTS, CN_FIRST, CN_MISM, CN_NEV, CN_TC, CN_COUNT };
// sCtl: [0] active rows, [1] flagged rows, [2..130) flagged list, recheck statistics
enum { CT_FLAG = 131, CT_DIS, CT_BAD, CT_QACT };  // CT_QACT + q: lane quarter q has active rows

struct TcSmemLayout {
  static constexpr int w = 0;
  static constexpr int a = kWImgBytes;                          // 98,304
  static constexpr int info = a + 2 * kABytes;                 // 128 x 24 ints
  static constexpr int best = info + kTcRows * kInfo * 4;       // 128 x groups x 3
  static constexpr int cap = best + kTcRows * kGroups * 3 * 4;  // checkpoint capacities [112]
  static constexpr int ctl = cap + kScrJ * 4;
  static constexpr int cst = ctl + 140 * 4;                     // invc0[112] b1[64] b2[64] b3[112]
  static constexpr int cnt = cst + 352 * 4;                     // per-row counters
  static constexpr int prof = cnt + CN_COUNT * kTcRows * 4;     // debug phase clocks [20]
  static constexpr int bar = prof + 20 * 8;
  static constexpr int tmem = bar + 8;
  static constexpr int total = tmem + 8;
};
static_assert(TcSmemLayout::total <= 232448, "tc sweep shared memory budget");
static_assert(TcSmemLayout::cap % 16 == 0 && TcSmemLayout::cst % 16 == 0 && TcSmemLayout::prof % 8 == 0,
              "aligned smem rows");

__host__ size_t tc_smem_bytes() { return TcSmemLayout::total; }

__device__ __forceinline__ void put_feature_at(unsigned char* sA, int off, float v) {
  __half h, l;
  split_f16(v, h, l);
  *(__half*)(sA + off) = h;
  *(__half*)(sA + kABytes + off) = l;
}
// canonical offset of column k for row 0 (add row_off(r) for row r)
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

// ---------------------------------------------------------------------------
// Exact FP64 re-evaluation of up to kRecheckRows flagged rows by the whole CTA:
// DualNetworkPolicy::evaluate (policies.hpp:121-168) with exactly the operation
// order of warp_policy_eval<kDual> (device_policy.cuh) — one thread per
// (row, output neuron) runs the neuron's acc = b; acc += w*x chain — while
// the FP64 weights stream from L2 through two 8 KB smem tiles (cp.async, one
// 16-byte copy per thread per tile), so the chains never wait on a dependent
// global load. Scratch: k-chunks 0..11 of the hi / lo feature buffers (free
// between layer 3 and the next F: h2 is dead, capacity features are rebuilt).
//   hi [0, 16 KB)      weight tiles          lo [0, 8.5 KB)  f / h1 / h2 / pr per row
//   hi [16 KB, ...)    caps, x rows, results
constexpr int kRecheckRows = 2;              // 2 x out(<=206) threads <= 512
constexpr int kRcTile = 8192;                // bytes per weight tile (1024 doubles)
constexpr int kRcInts = 2 * kRcTile;         // offset of the int area in the hi buffer
constexpr int kRcVec = 2 * kMaxJ + 2 + 2 * kTcH + 2 * kMaxJ;  // f, h1, h2, pr doubles per row
constexpr int kRcScratchHi = (kRcInts + (2 * kRecheckRows * kScrJ + 2 * kRecheckRows) * 4 + 15) & ~15;
constexpr int kRcScratchLo = (kRecheckRows * kRcVec * 8 + 15) & ~15;
static_assert(kRcScratchHi <= 12 * 2048 && kRcScratchLo <= 12 * 2048, "recheck scratch stays in k-chunks 0..11");

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// out[k][r] = (tanh?)(bias[r] + sum_c W[c][r] * xin[k][c]) for r < width, k < nb
__device__ void rc_layer(const double* __restrict__ W, const double* __restrict__ bias, int K, int width,
                         const double* xin, double* outv, bool act_tanh, int tanh_fma, int nb,
                         unsigned char* tiles, int tid) {
  const int tc = (kRcTile / 8) / width;  // W rows per tile
  const int ntiles = (K + tc - 1) / tc;
  const int k = tid / width, r = tid - k * width;
  const bool active = k < nb;
  auto issue = [&](int tile) {
    const int c0 = tile * tc, rows = min(tc, K - c0);
    const int n16 = rows * width / 2;  // width is even
    double* dst = (double*)(tiles + (tile & 1) * kRcTile);
    const double* src = W + (size_t)c0 * width;
    for (int i = tid; i < n16; i += kTcBlock) cp_async16(dst + 2 * i, src + 2 * i);
    cp_async_commit();
  };
  double acc = active ? __ldg(bias + r) : 0.0;
  const double* x = xin + k * kRcVec;
  issue(0);
  for (int tile = 0; tile < ntiles; ++tile) {
    if (tile + 1 < ntiles) {
      issue(tile + 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (active) {
      const double* w = (const double*)(tiles + (tile & 1) * kRcTile) + r;
      const int c0 = tile * tc, rows = min(tc, K - c0);
      for (int c = 0; c < rows; ++c) acc = __dadd_rn(acc, __dmul_rn(w[c * width], x[c0 + c]));
    }
    __syncthreads();
  }
  if (active) outv[k * kRcVec + r] = act_tanh ? gt_tanh(acc, tanh_fma) : acc;
  __syncthreads();
}

__device__ void cta_recheck(const DevModel& P, unsigned char* sA, const int* caps, const int* xrow,
                            const int* rows, int nb, const int* sInfo, int tid) {
  const int J = P.J, H = P.H, in = P.in, out = P.out;
  unsigned char* tiles = sA;
  double* vec = (double*)(sA + kABytes);  // per row: f[in] h1[H] h2[H] pr[out] (kRcVec)
  int* res = (int*)(sA + kRcInts) + 2 * kRecheckRows * kScrJ;  // [exact x nb][nonfinite x nb]
  const int warp = tid >> 5, lane = tid & 31;
  // features (DualNetworkPolicy::features, policies.hpp:129-141)
  for (int i = tid; i < nb * in; i += kTcBlock) {
    const int k = i / in, j = i - k * in;
    const int* inf = sInfo + rows[k] * kInfo;
    const int t = inf[RI_T];
    double f;
    if (j < J) {
      const int c0 = __ldg(P.pcap0 + j);
      f = c0 > 0 ? __ddiv_rn((double)caps[k * kScrJ + j], (double)c0) : 0.0;
    } else if (j < 2 * J) {
      const int x0 = __ldg(P.pinv0 + (size_t)P.product[t] * J + (j - J));
      f = x0 > 0 ? __ddiv_rn((double)xrow[k * kScrJ + (j - J)], (double)x0) : 0.0;
    } else {
      const int ot = P.order_t ? P.order_t[t] : t;
      f = P.horizon > 0 ? __ddiv_rn((double)ot, (double)P.horizon) : 0.0;
    }
    vec[k * kRcVec + j] = f;
  }
  __syncthreads();
  const int oh1 = 2 * kMaxJ + 2, oh2 = oh1 + kTcH, opr = oh2 + kTcH;
  rc_layer(P.w1t, P.b1, in, H, vec, vec + oh1, true, P.tanh_fma, nb, tiles, tid);
  rc_layer(P.w2t, P.b2, H, H, vec + oh1, vec + oh2, true, P.tanh_fma, nb, tiles, tid);
  rc_layer(P.w3t, P.b3, H, out, vec + oh2, vec + opr, false, P.tanh_fma, nb, tiles, tid);
  // scores and argmax: warp k for row k (as warp_policy_eval<kDual>)
  if (warp < nb) {
    const int k = warp;
    const int* inf = sInfo + rows[k] * kInfo;
    const int t = inf[RI_T];
    const double* rw = P.rtab + (size_t)P.rrow[t] * J;
    const double* pr = vec + k * kRcVec + opr;
    bool feas = false;
    for (int j = lane; j < J; j += 32) feas |= caps[k * kScrJ + j] > 0 && xrow[k * kScrJ + j] > 0;
    int exact = -1, nonfinite = 0;
    if (__any_sync(0xffffffffu, feas)) {
      double bv = 0.0;
      int bi = -1;
      bool bad = false;
      for (int j = lane; j < J; j += 32) {
        if (caps[k * kScrJ + j] <= 0 || xrow[k * kScrJ + j] <= 0) continue;
        const double sc = __dsub_rn(__dsub_rn(__ldg(rw + j), pr[j]), pr[J + j]);
        if (!isfinite(sc)) { bad = true; continue; }
        argmax_combine(bv, bi, sc, j);
      }
      if (__any_sync(0xffffffffu, bad)) {
        nonfinite = 1;
      } else {
        warp_argmax(bv, bi);
        exact = (bi >= 0 && bv >= 0.0) ? bi : -1;
      }
    }
    if (lane == 0) {
      res[k] = exact;
      res[kRecheckRows + k] = nonfinite;
    }
  }
  __syncthreads();
}

template <bool PROF>
__global__ void __launch_bounds__(kTcBlock, 1) k_sweep_product_tc(TcArgs a) {
  extern __shared__ __align__(1024) unsigned char smem[];
  const SweepArgs& S = a.s;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int J = S.J, lo = S.lo, hi = S.hi;
  const int base = hck_base(lo), HJ = hck_stride(J), RJ = (J + 7) & ~7;
  unsigned char* sW = smem + TcSmemLayout::w;
  unsigned char* sA = smem + TcSmemLayout::a;
  int* sInfo = (int*)(smem + TcSmemLayout::info);
  float* sBest = (float*)(smem + TcSmemLayout::best);
  int* sCap = (int*)(smem + TcSmemLayout::cap);
  int* sCtl = (int*)(smem + TcSmemLayout::ctl);
  int* sCnt = (int*)(smem + TcSmemLayout::cnt);
  uint64_t* sBar = (uint64_t*)(smem + TcSmemLayout::bar);
  uint32_t* sTmem = (uint32_t*)(smem + TcSmemLayout::tmem);
  float* sInvC0 = (float*)(smem + TcSmemLayout::cst);
  float* sB1 = sInvC0 + kScrJ;
  float* sB2 = sB1 + 64;
  float* sB3 = sB2 + 64;
  const int tile = blockIdx.x;
  // (row, group) of this thread for every per-row phase
  const int q4 = warp & 3, grp = warp >> 2;
  const int r = 32 * q4 + lane;
  const bool agent = grp == kGroups - 1;
  const uint32_t tl = (uint32_t)(32 * q4) << 16;  // TMEM lane base of the warp
  const int gc0 = kGC * grp;                      // first node of the group
  const int gcn = max(0, min(kGC, J - gc0));      // nodes of the group
  const int rowo = row_off(r);
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
  for (int j = tid; j < kScrJ; j += kTcBlock) {
    sCap[j] = j < J ? S.ckcap[j] : 0;
    sInvC0[j] = j < J ? a.inv_c0[j] : 0.f;
  }
  for (int i = tid; i < kTcH; i += kTcBlock) {
    sB1[i] = a.b1f[i];
    sB2[i] = a.b2f[i];
  }
  for (int i = tid; i < kTcN3; i += kTcBlock) sB3[i] = a.b3f[i];
  const int nq = a.wctl[0], dealt = (int)gridDim.x * kTcRows;
  // row agent: bind process m (>= 0) or go idle (m < 0)
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
    }
  };
  auto next_entry = [&]() -> int {
    const int k = dealt + atomicAdd(&a.wctl[1], 1);
    return k < nq ? a.wq[k] : -1;
  };
  if (agent) {
    const int k = r * (int)gridDim.x + tile;
    begin_proc(sInfo + r * kInfo, k < nq ? a.wq[k] : -1);
    for (int k = 0; k < CN_COUNT; ++k) sCnt[k * kTcRows + r] = k == CN_FIRST ? INT_MAX : 0;
  }
  if (tid == 0) {
    sCtl[0] = 0;
    sCtl[1] = 0;
    sCtl[CT_FLAG] = sCtl[CT_DIS] = sCtl[CT_BAD] = 0;
    mbar_init(sBar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
  {  // D = 0
    const uint32_t z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < kGChunks; ++c) tmem_st8(tmem + tl + kColD + gc0 + 8 * c, z);
    tmem_wait_st();
  }

  const uint32_t aBase = smem_u32(sA);
  const uint32_t w1h = smem_u32(sW), w1l = w1h + kW1Bytes;
  const uint32_t w2h = w1l + kW1Bytes, w2l = w2h + kW2Bytes;
  const uint32_t w3h = w2l + kW2Bytes, w3l = w3h + kW3Bytes;
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
  uint32_t xb = 0;  // x > 0 bits of (row, group), persistent

  // debug phase profile (PROF instantiation only): clock64 totals of CTA 0, thread 0
  long long* pacc = (long long*)(smem + TcSmemLayout::prof);
  if (PROF && tid == 0)
    for (int k = 0; k < 20; ++k) pacc[k] = 0;
  long long fl = 0;
  long long plast = PROF ? clock64() : 0;
  const bool prof_on = PROF && blockIdx.x == 0 && tid == 0;
#define PMARK(k) do { if (PROF && prof_on) { const long long now_ = clock64(); pacc[k] += now_ - plast; plast = now_; } } while (0)
  for (;;) {
    // ============================ F: capacities, features, feasibility
    uint32_t fmask = 0;  // feasible nodes of (row, group), bit i = node gc0 + i
    auto f_phase = [&](auto nch) {
      constexpr int NCH = decltype(nch)::value;
      if (PROF && prof_on) fl = clock64();
      const int* inf = sInfo + r * kInfo;
      const bool act = inf[RI_POS] < inf[RI_END];
      int t = 0, b = 0, p = 0, x = 0, xd = 0, xu = -1, evt = -1, xuv = 0, dres = 0;
      float xui = 0.f;
      uint32_t hv[NCH][8];  // checkpoint counts of the group's nodes, 8 per chunk
      uint32_t e8[8];       // the 8-slot event block
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int i = 0; i < 8; ++i) hv[c][i] = 0;
#pragma unroll
      for (int i = 0; i < 8; ++i) e8[i] = 0xffffffffu;
      if (act) {
        t = inf[RI_T];
        p = inf[RI_P];
        x = inf[RI_X];
        dres = inf[RI_DRESET];
        xd = inf[RI_XDIRTY] | (xpersist ? 0 : 1);
        xu = inf[RI_XUPD];
        evt = inf[RI_EVT];
        b = (t - base) >> kLogK;
        const int bl = a.pf == 9 ? (r & 7) : b;  // debug timing experiment (wrong results)
        ldg256(S.ev + base + (bl << kLogK), e8);
        const int* hr = S.hck + (size_t)bl * HJ + gc0;
#pragma unroll
        for (int c = 0; c < NCH; ++c)
          if (8 * c < gcn) ldg256(hr + 8 * c, hv[c]);
        if (!xd && xu >= gc0 && xu < gc0 + gcn) {
          xuv = S.xloc[(size_t)x * J + xu];
          xui = __ldg(a.inv_x0 + (size_t)p * J + xu);
        }
      }
      // partial block [max(lo, base + 8b), t): per-chunk packed nibble counts
      uint32_t pk[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) pk[c] = 0;
      {
        const int sb = base + (b << kLogK);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int s = sb + k;
          const int ek = (int)e8[k];
          const int rel = (act && s >= lo && s < t && ek >= 0) ? ek - gc0 : -1;
          const int ch = rel >> 3;  // < 0 for none / other group
          const uint32_t nib = 1u << (4 * (rel & 7));
#pragma unroll
          for (int c = 0; c < NCH; ++c) pk[c] += ch == c ? nib : 0u;
        }
      }
      if (PROF && prof_on) { const long long n_ = clock64(); pacc[12] += n_ - fl; fl = n_; }
      const int relE = evt >= 0 ? evt - gc0 : -1, relX = xu >= 0 ? xu - gc0 : -1;
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const int j0 = gc0 + 8 * c;
        if (j0 >= J) break;  // warp-uniform
        uint32_t dv[8];
        tmem_ld8(tmem + tl + kColD + j0, dv);
        tmem_wait_ld();
        const int eE = (relE >> 3) == c ? (relE & 7) : -1, eX = (relX >> 3) == c ? (relX & 7) : -1;
        const int4 cp0 = *(const int4*)(sCap + j0), cp1 = *(const int4*)(sCap + j0 + 4);
        const float4 iv0 = *(const float4*)(sInvC0 + j0), iv1 = *(const float4*)(sInvC0 + j0 + 4);
        const int capv[8] = {cp0.x, cp0.y, cp0.z, cp0.w, cp1.x, cp1.y, cp1.z, cp1.w};
        const float inv[8] = {iv0.x, iv0.y, iv0.z, iv0.w, iv1.x, iv1.y, iv1.z, iv1.w};
        uint32_t cv[8], bits = 0;
        float fv[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int d = (dres ? 0 : (int)dv[i]) + (i == eE ? 1 : 0) - (i == eX ? 1 : 0);
          dv[i] = (uint32_t)d;
          const int cc = max(capv[i] - (int)hv[c][i] + d - (int)((pk[c] >> (4 * i)) & 15u), 0);
          cv[i] = (uint32_t)cc;
          bits |= (cc > 0 ? 1u : 0u) << i;
          fv[i] = (float)cc * inv[i];
        }
        tmem_st8(tmem + tl + kColD + j0, dv);
        tmem_st8(tmem + tl + kColCap + j0, cv);
        fmask |= bits << (8 * c);
        uint32_t h4[4], l4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) split2(fv[2 * i], fv[2 * i + 1], h4[i], l4[i]);
        if (act) {
          const int off = rowo + kcol_off(j0);
          if (j0 + 8 <= J) {
            *(uint4*)(sA + off) = make_uint4(h4[0], h4[1], h4[2], h4[3]);
            *(uint4*)(sA + kABytes + off) = make_uint4(l4[0], l4[1], l4[2], l4[3]);
          } else {  // last partial chunk: the columns from J on are inventory features
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              if (j0 + 2 * i + 1 < J) {
                *(uint32_t*)(sA + off + 4 * i) = h4[i];
                *(uint32_t*)(sA + kABytes + off + 4 * i) = l4[i];
              } else if (j0 + 2 * i < J) {
                *(uint16_t*)(sA + off + 4 * i) = (uint16_t)h4[i];
                *(uint16_t*)(sA + kABytes + off + 4 * i) = (uint16_t)l4[i];
              }
            }
          }
        }
      }
      if (PROF && prof_on) { const long long n_ = clock64(); pacc[13] += n_ - fl; fl = n_; }
      // inventory features x/x0 (columns J + node) and the x > 0 bits
      if (act && xd) {
        const int* xr = S.xloc + (size_t)x * J + gc0;
        const float* ix = a.inv_x0 + (size_t)p * J + gc0;
        uint32_t nb = 0;
        for (int i = 0; i < gcn; ++i) {
          const int xj = xr[i];
          put_feature_at(sA, rowo + kcol_off(J + gc0 + i), (float)xj * __ldg(ix + i));
          nb |= (xj > 0 ? 1u : 0u) << i;
        }
        xb = nb;
      } else if (act && xu >= gc0 && xu < gc0 + gcn) {
        put_feature_at(sA, rowo + kcol_off(J + xu), (float)xuv * xui);
        if (xuv <= 0) xb &= ~(1u << (xu - gc0));
      }
      if (act && agent) put_feature_at(sA, rowo + kcol_off(2 * J), (float)inf[RI_OT] * invT);
      fmask = act ? (fmask & xb) : 0u;
      if (grp == 0) {
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (lane == 0) {
          sCtl[CT_QACT + q4] = bal != 0;
          if (bal) atomicAdd(&sCtl[0], __popc(bal));
        }
      }
      tmem_wait_st();
      if (PROF && prof_on) { const long long n_ = clock64(); pacc[14] += n_ - fl; fl = n_; }
    };
    if (agent) {
      // P: the loads this row's update (U) needs; their latency hides behind F
      int u_ev = -1, u_old = 0, u_wr = 0, u_ref = 0, u_pn = -1, u_rrn = 0, u_otn = 0, u_tnn = -1, u_xn = -1;
      int* inf = sInfo + r * kInfo;
      const int pos = inf[RI_POS], end = inf[RI_END];
      if (pos < end) {
        const int t = inf[RI_T];
        u_ev = S.ev[t];
        u_old = S.cache[t];
        u_wr = S.written[t];
        if (S.ref) u_ref = S.ref[t];
        const int tn = inf[RI_TN];
        if (tn >= 0) {
          if (a.pf == 1) {  // warm L2 with the next step's checkpoint row and event block
            const int bn = (tn - base) >> kLogK;
            const int* hbn = S.hck + (size_t)bn * HJ;
            for (int k = 0; k < HJ; k += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(hbn + k));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(S.ev + base + (bn << kLogK)));
          }
          u_pn = S.model.product[tn];
          u_xn = S.rid[tn];
          u_rrn = S.model.rrow[tn];
          u_otn = S.model.order_t ? S.model.order_t[tn] : tn;
        }
        if (pos + 2 < end) u_tnn = S.pslots[pos + 2];
      }
      f_phase(std::integral_constant<int, 1>{});
      inf[RI_UEV] = u_ev;
      inf[RI_UOLD] = u_old;
      inf[RI_UWR] = u_wr;
      inf[RI_UREF] = u_ref;
      inf[RI_UPN] = u_pn;
      inf[RI_URRN] = u_rrn;
      inf[RI_UOTN] = u_otn;
      inf[RI_UTNN] = u_tnn;
      inf[RI_UXN] = u_xn;
    } else {
      f_phase(std::integral_constant<int, kGChunks>{});
    }
    tc_fence_before();
    fence_async_smem();
    __syncthreads();
    PMARK(0);
    if (sCtl[0] == 0) break;
    if (PROF && prof_on) pacc[10] += 1;

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
    const bool qact = sCtl[CT_QACT + q4] != 0;  // warp-uniform: skip idle lane quarters
    auto hidden_epilogue = [&](uint32_t col_hh, uint32_t col_x, const float* bias) {
      if (!qact) return;
#pragma unroll
      for (int cc = 0; cc < kTcH / kGroups; cc += 16) {
        const int cb = grp * (kTcH / kGroups) + cc;
        float vh[16], vx[16];
        tmem_ld16(tmem + tl + col_hh + cb, vh);
        tmem_ld16(tmem + tl + col_x + cb, vx);
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
    uint32_t rwv[kGChunks][8];  // fp32 rewards of the group's nodes (rows padded to 8)
    {
      const float* rw = a.rtabf + (size_t)(fmask ? sInfo[r * kInfo + RI_RR] : 0) * RJ + gc0;
#pragma unroll
      for (int c = 0; c < kGChunks; ++c) {
        if ((fmask >> (8 * c)) & 0xffu) {
          ldg256(rw + 8 * c, rwv[c]);
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) rwv[c][i] = 0u;
        }
      }
    }
    mbar_wait(sBar, phase);
    PMARK(5);
    phase ^= 1;
    tc_fence_after();

    // ============================ S: scores, argmax, margin (row, group)
    {
      float v1 = -INFINITY, v2 = -INFINITY;
      int i1 = -1;
      bool bad = false;
      uint32_t vh[kGChunks][8], vx[kGChunks][8];
#pragma unroll
      for (int c = 0; c < kGChunks; ++c) {
        if (qact && gc0 + 8 * c < kTcN3) {  // warp-uniform
          tmem_ld8(tmem + tl + gc0 + 8 * c, vh[c]);
          tmem_ld8(tmem + tl + kTcN3 + gc0 + 8 * c, vx[c]);
        }
      }
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < kGChunks; ++c) {
        if (!qact || gc0 + 8 * c >= kTcN3) break;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int li = 8 * c + i;
          if (!((fmask >> li) & 1u)) continue;  // feasible implies node < J
          const float qv = fmaf(__uint_as_float(vx[c][i]), kLoInv, __uint_as_float(vh[c][i])) + sB3[gc0 + li];
          const float sc = __uint_as_float(rwv[c][i]) - qv;
          if (!isfinite(sc)) bad = true;
          if (sc > v1) { v2 = v1; v1 = sc; i1 = gc0 + li; }
          else if (sc > v2) v2 = sc;
        }
      }
      float* bs = sBest + r * (kGroups * 3) + grp * 3;
      bs[0] = v1;
      bs[1] = __int_as_float(bad ? -2 : i1);
      bs[2] = v2;
    }
    tc_fence_before();
    __syncthreads();
    PMARK(6);
    if (agent) {  // combine the groups
      int* inf = sInfo + r * kInfo;
      inf[RI_FLAG] = 0;
      if (inf[RI_POS] >= inf[RI_END]) {
        inf[RI_ANY] = -1;
      } else {
        const float* bs = sBest + r * (kGroups * 3);
        float v1 = bs[0], v2 = bs[2];
        int i1 = __float_as_int(bs[1]);
        bool bad = i1 == -2;
#pragma unroll
        for (int g = 1; g < kGroups; ++g) {
          const float w1 = bs[3 * g], w2 = bs[3 * g + 2];
          const int j1 = __float_as_int(bs[3 * g + 1]);
          bad |= j1 == -2;
          if (w1 > v1) { v2 = fmaxf(v1, w2); v1 = w1; i1 = j1; }
          else v2 = fmaxf(v2, w1);
        }
        if (i1 == -1 && !bad) {  // nothing feasible
          inf[RI_ANY] = 0;
          inf[RI_DEC] = -1;
        } else {
          inf[RI_ANY] = 1;
          inf[RI_DEC] = v1 >= 0.f ? i1 : -1;
          const bool flag = bad || i1 < 0 || !(v1 - v2 >= a.guard) || !(fabsf(v1) >= a.guard);
          sCnt[CN_TC * kTcRows + r] += 1;
          if (flag || a.verify) {
            inf[RI_FLAG] = flag ? 1 : 2;
            const int k = atomicAdd(&sCtl[1], 1);
            sCtl[2 + k] = r;
          }
        }
      }
    }
    __syncthreads();
    PMARK(7);

    // ============================ exact FP64 re-evaluation of flagged rows
    // by the whole CTA, two rows at a time (cta_recheck)
    const int nflag = sCtl[1];
    for (int f0 = 0; f0 < nflag; f0 += kRecheckRows) {
      const int nb = min(kRecheckRows, nflag - f0);
      int* caps = (int*)(sA + kRcInts);  // [kRecheckRows][kScrJ], then row[kRecheckRows][kScrJ]
      int* xrow = caps + kRecheckRows * kScrJ;
      // capacities of the step (TMEM cols 384+) from the warp of the row's lanes
      if (warp < 4) {
        for (int k = 0; k < nb; ++k) {
          const int rr = sCtl[2 + f0 + k];
          if ((rr >> 5) != warp) continue;  // warp-uniform
          for (int c0 = 0; c0 < kTcN3 / 8; c0 += 7) {  // 14 chunks of 8 nodes
            uint32_t v[7][8];
#pragma unroll
            for (int c = 0; c < 7; ++c) tmem_ld8(tmem + tl + kColCap + 8 * (c0 + c), v[c]);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 7; ++c)
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int x = (int)__shfl_sync(0xffffffffu, v[c][i], rr & 31);
                if (lane == 0) caps[k * kScrJ + 8 * (c0 + c) + i] = x;
              }
          }
        }
      }
      for (int i = tid; i < nb * J; i += kTcBlock) {
        const int k = i / J, j = i - k * J;
        const int* inf = sInfo + sCtl[2 + f0 + k] * kInfo;
        xrow[k * kScrJ + j] = S.xloc[(size_t)inf[RI_X] * J + j];
      }
      __syncthreads();
      cta_recheck(S.model, sA, caps, xrow, sCtl + 2 + f0, nb, sInfo, tid);
      if (lane == 0 && warp < nb) {
        const int rr = sCtl[2 + f0 + warp];
        int* inf = sInfo + rr * kInfo;
        const int* res = (const int*)(sA + kRcInts) + 2 * kRecheckRows * kScrJ;
        const int exact = res[warp], nonfinite = res[kRecheckRows + warp];
        if (nonfinite) {
          const int m = inf[RI_M];
          atomicMin(&S.scal->err_nonfinite, ((unsigned long long)m << 32) | (unsigned)inf[RI_OT]);
        }
        if (inf[RI_FLAG] == 1) {
          atomicAdd(&sCtl[CT_FLAG], 1);
          atomicAdd(&sCtl[CT_DIS], exact != inf[RI_DEC] ? 1 : 0);
        } else {
          atomicAdd(&sCtl[CT_BAD], exact != inf[RI_DEC] ? 1 : 0);
        }
        inf[RI_DEC] = exact;
      }
      __syncthreads();
      if (f0 + kRecheckRows >= nflag) {
        // the scratch overlaps K-padding columns of the layer-1 operand when
        // 2J+1 < 72: leave zeros behind, as the setup did
        uint4* zh = (uint4*)sA;
        uint4* zl = (uint4*)(sA + kABytes);
        for (int i = tid; i < kRcScratchHi / 16; i += kTcBlock) zh[i] = make_uint4(0, 0, 0, 0);
        for (int i = tid; i < kRcScratchLo / 16; i += kTcBlock) zl[i] = make_uint4(0, 0, 0, 0);
      }
    }
    __syncthreads();
    PMARK(8);

    // ============================ U: update + publish (row agents)
    if (agent) {
      int* inf = sInfo + r * kInfo;
      inf[RI_DRESET] = 0;
      if (inf[RI_ANY] >= 0) {
        const int t = inf[RI_T], x = inf[RI_X], dec = inf[RI_DEC];
        const int u_old = inf[RI_UOLD], u_xn = inf[RI_UXN];
        // D deltas are applied by the row's F threads next step
        inf[RI_EVT] = inf[RI_UEV];
        inf[RI_XUPD] = dec;
        if (dec >= 0) atomicSub(&S.xloc[(size_t)x * J + dec], 1);  // fire-and-forget RED
        int* cn = sCnt + r;
        if (dec != u_old) {
          cn[CN_CHANGED * kTcRows] += 1;
          cn[CN_FIRST * kTcRows] = min(cn[CN_FIRST * kTcRows], t);
          cn[CN_CONFLICTS * kTcRows] += inf[RI_UWR] ? 1 : 0;
        }
        if (S.ref) {
          const int u_ref = inf[RI_UREF];
          cn[CN_MISM * kTcRows] += (dec != u_ref ? 1 : 0) - (u_old != u_ref ? 1 : 0);
        }
        S.cache[t] = dec;
        S.written[t] = 1;
        cn[CN_NEV * kTcRows] += 1;
        const int pos = inf[RI_POS] + 1;
        inf[RI_POS] = pos;
        if (pos < inf[RI_END]) {
          if (a.pf == 2) {
            const int bn = (inf[RI_TN] - base) >> kLogK;
            const int* hbn = S.hck + (size_t)bn * HJ;
            for (int k = 0; k < HJ; k += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(hbn + k));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(S.ev + base + (bn << kLogK)));
          }
          inf[RI_T] = inf[RI_TN];
          inf[RI_XDIRTY] = u_xn != x ? 1 : 0;
          inf[RI_X] = u_xn;
          inf[RI_P] = inf[RI_UPN];
          inf[RI_RR] = inf[RI_URRN];
          inf[RI_OT] = inf[RI_UOTN];
          inf[RI_TN] = inf[RI_UTNN];
        } else {
          // process done: its evaluation count (evals_per_process, max and
          // total), then the next entry of the work list
          const int m = inf[RI_M];
          const unsigned long long nev = (unsigned)cn[CN_NEV * kTcRows];
          atomicMax(&S.scal->max_evals, nev);
          atomicAdd(&S.scal->total_evals, nev);
          if (S.evals_out) S.evals_out[m] = (long long)nev;
          cn[CN_NEV * kTcRows] = 0;
          begin_proc(inf, next_entry());
        }
      }
      if (tid == kTcBlock - 1) {
        sCtl[0] = 0;
        sCtl[1] = 0;
      }
    }
    __syncthreads();
    PMARK(9);
  }

  // ---------------------------------------------------------------- teardown
  if (PROF && prof_on)
    for (int k = 0; k < 17; ++k) a.prof[k] = pacc[k];
#undef PMARK
  if (agent) {
    const int* cn = sCnt + r;
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
    if (sCtl[CT_FLAG]) atomicAdd(&a.stats[1], (unsigned long long)(unsigned)sCtl[CT_FLAG]);
    if (sCtl[CT_DIS]) atomicAdd(&a.stats[2], (unsigned long long)(unsigned)sCtl[CT_DIS]);
    if (sCtl[CT_BAD]) atomicAdd(&a.stats[3], (unsigned long long)(unsigned)sCtl[CT_BAD]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
  }
}

void launch_tc_sweep(const TcArgs& a, int ntiles, cudaStream_t stream) {
  static bool attr = false;
  const size_t smem = tc_smem_bytes();
  if (!attr) {
    cudaFuncSetAttribute(k_sweep_product_tc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_sweep_product_tc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  if (a.prof)
    k_sweep_product_tc<true><<<ntiles, kTcBlock, smem, stream>>>(a);
  else
    k_sweep_product_tc<false><<<ntiles, kTcBlock, smem, stream>>>(a);
}

}  // namespace pcd
