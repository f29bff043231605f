// device_policy.cuh — exact FP64 policy evaluation on sm_100a.
//
// The three reference policies (fo/policies.hpp) evaluated by one warp per
// process, reproducing the reference's double-precision results bit for bit:
//   * every multiply/add/divide is an explicit round-to-nearest intrinsic
//     (__dmul_rn/__dadd_rn/...), so nvcc never contracts them into FMAs —
//     the reference is compiled without FMA (mlp.cpp:149-168);
//   * MlpParams::forward's accumulation order acc=b; acc+=w*x (mlp.cpp:141-169)
//     is kept per output neuron;
//   * tanh is glibc 2.39's s_tanh.c with the IFUNC-selected expm1 body
//     (FMA or SSE2 variant, chosen at handle creation to match the host libm
//     the reference links), restated from the libm disassembly.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pcd {

enum : int { kGreedy = 0, kCapacity = 1, kDual = 2, kNull = 3 };

struct DevModel {
  int kind, J, I, H, in, out;
  double gamma;
  const double* w1t;   // [in][H]   (transpose of MlpParams::w1 [H][in])
  const double* b1;    // [H]
  const double* w2t;   // [H][H]
  const double* b2;    // [H]
  const double* w3t;   // [H][out]
  const double* b3;    // [out]
  const int* pcap0;    // [J]   DualNetworkPolicy::initial_ capacities
  const int* pinv0;    // [I*J] DualNetworkPolicy::initial_ inventory
  long long horizon;   // DualNetworkPolicy::horizon_
  int tanh_fma;
  const int* product;  // [T]
  const int* order_t;  // [T] or nullptr
  const int* rrow;     // [T]
  const double* rtab;  // [R*J]
  const double* w3s;   // [H][J] W3[j] + W3[J+j] (transposed) for the order-free recheck, or nullptr
  double fast_margin;  // decision margin above which the order-free FP64 recheck is exact (0 = off)
};

// ---------------------------------------------------------------- glibc tanh
__device__ __forceinline__ double gt_add_exp(double y, int k) {
  unsigned long long b = __double_as_longlong(y);
  unsigned hi = (unsigned)(b >> 32) + ((unsigned)k << 20);
  return __longlong_as_double((long long)(((unsigned long long)hi << 32) | (b & 0xffffffffull)));
}

// glibc expm1 (fdlibm s_expm1.c as built in glibc 2.39; FMA body @0x7ac30,
// SSE2 body @0x2eaf0 of libm.so.6). Reachable range from tanh: |x| < 44.
static __device__ __noinline__ double gt_expm1(double x, int use_fma) {
  const double INVLN2 = 1.4426950408889634, LN2HI = 0.6931471803691238,
               LN2LO = 1.9082149292705877e-10;
  const double Q1 = -3.33333333333331316428e-02, Q2 = 1.58730158725481460165e-03,
               Q3 = -7.93650757867487942473e-05, Q4 = 4.00821782732936239552e-06,
               Q5 = -2.01099218183624371326e-07;
  const unsigned long long bx = __double_as_longlong(x);
  const unsigned hx = (unsigned)(bx >> 32) & 0x7fffffffu;
  const int neg = (int)(bx >> 63);
  double hi, lo, c = 0.0;
  int k;
  if (hx >= 0x4043687Au) {
    if (hx >= 0x40862E42u) {
      if (hx >= 0x7ff00000u) {
        if (((hx & 0xfffffu) | (unsigned)bx) != 0) return __dadd_rn(x, x);
        return neg ? -1.0 : x;
      }
      if (x > 7.09782712893383973096e+02) return __longlong_as_double(0x7ff0000000000000ll);
    }
    if (neg) return -1.0;
  }
  if (hx > 0x3fd62e42u) {
    if (hx < 0x3FF0A2B2u) {
      if (!neg) { hi = __dsub_rn(x, LN2HI); lo = LN2LO; k = 1; }
      else { hi = __dadd_rn(x, LN2HI); lo = -LN2LO; k = -1; }
    } else {
      const double kf = __dadd_rn(neg ? -0.5 : 0.5, __dmul_rn(INVLN2, x));
      k = __double2int_rz(kf);
      const double t = (double)k;
      hi = use_fma ? __fma_rn(-t, LN2HI, x) : __dsub_rn(x, __dmul_rn(LN2HI, t));
      lo = __dmul_rn(t, LN2LO);
    }
    x = __dsub_rn(hi, lo);
    c = __dsub_rn(__dsub_rn(hi, x), lo);
  } else if (hx < 0x3c900000u) {
    return x;
  } else {
    k = 0;
  }
  const double hfx = __dmul_rn(x, 0.5);
  const double hxs = __dmul_rn(x, hfx);
  double r1, t, e;
  if (use_fma) {
    const double R2 = __fma_rn(hxs, Q3, Q2);
    const double R3 = __fma_rn(hxs, Q5, Q4);
    const double h2 = __dmul_rn(hxs, hxs);
    const double R1 = __fma_rn(hxs, Q1, 1.0);
    const double h4 = __dmul_rn(h2, h2);
    r1 = __fma_rn(h4, R3, __fma_rn(h2, R2, R1));
    t = __fma_rn(-r1, hfx, 3.0);
    e = __ddiv_rn(__dsub_rn(r1, t), __fma_rn(-x, t, 6.0));
    e = __dmul_rn(e, hxs);
    if (k == 0) return __dsub_rn(x, __fma_rn(e, x, -hxs));
    e = __fma_rn(__dsub_rn(e, c), x, -c);
    e = __dsub_rn(e, hxs);
    if (k == -1) return __fma_rn(0.5, __dsub_rn(x, e), -0.5);
    if (k == 1) {
      if (x < -0.25) return __dmul_rn(__dsub_rn(e, __dadd_rn(x, 0.5)), -2.0);
      return __fma_rn(__dsub_rn(x, e), 2.0, 1.0);
    }
  } else {
    const double h2 = __dmul_rn(hxs, hxs);
    const double R2 = __dadd_rn(__dmul_rn(Q3, hxs), Q2);
    const double R1 = __dadd_rn(__dmul_rn(Q1, hxs), 1.0);
    const double h4 = __dmul_rn(h2, h2);
    const double R3 = __dadd_rn(__dmul_rn(Q5, hxs), Q4);
    r1 = __dadd_rn(__dadd_rn(__dmul_rn(R2, h2), R1), __dmul_rn(R3, h4));
    t = __dsub_rn(3.0, __dmul_rn(hfx, r1));
    e = __ddiv_rn(__dsub_rn(r1, t), __dsub_rn(6.0, __dmul_rn(t, x)));
    e = __dmul_rn(e, hxs);
    if (k == 0) return __dsub_rn(x, __dsub_rn(__dmul_rn(e, x), hxs));
    e = __dsub_rn(__dmul_rn(__dsub_rn(e, c), x), c);
    e = __dsub_rn(e, hxs);
    if (k == -1) return __dsub_rn(__dmul_rn(__dsub_rn(x, e), 0.5), 0.5);
    if (k == 1) {
      if (x < -0.25) return __dmul_rn(__dsub_rn(e, __dadd_rn(x, 0.5)), -2.0);
      return __dadd_rn(1.0, __dmul_rn(2.0, __dsub_rn(x, e)));
    }
  }
  if (k <= -2 || k > 56) {
    const double y = __dsub_rn(1.0, __dsub_rn(e, x));
    return __dsub_rn(gt_add_exp(y, k), 1.0);
  }
  if (k < 20) {
    const double tt = __longlong_as_double((long long)((unsigned long long)(0x3ff00000u - (0x200000u >> k)) << 32));
    return gt_add_exp(__dsub_rn(tt, __dsub_rn(e, x)), k);
  }
  const double tt = __longlong_as_double((long long)((unsigned long long)((unsigned)(0x3ff - k) << 20) << 32));
  return gt_add_exp(__dadd_rn(__dsub_rn(x, __dadd_rn(e, tt)), 1.0), k);
}

// glibc tanh (s_tanh.c; tanh@0x31620 of libm.so.6).
__device__ __forceinline__ double gt_tanh(double x, int use_fma) {
  const unsigned long long bx = __double_as_longlong(x);
  const unsigned jx = (unsigned)(bx >> 32);
  const unsigned ix = jx & 0x7fffffffu;
  const int neg = (int)(jx >> 31);
  double z;
  if (ix >= 0x7ff00000u) return neg ? __dsub_rn(__ddiv_rn(1.0, x), 1.0) : __dadd_rn(__ddiv_rn(1.0, x), 1.0);
  if (ix < 0x40360000u) {
    if ((ix | (unsigned)bx) == 0) return x;
    if (ix < 0x3c800000u) return __dmul_rn(x, __dadd_rn(1.0, x));
    const double ax = fabs(x);
    if (ix >= 0x3ff00000u) {
      const double t = gt_expm1(__dadd_rn(ax, ax), use_fma);
      z = __dsub_rn(1.0, __ddiv_rn(2.0, __dadd_rn(t, 2.0)));
    } else {
      const double t = gt_expm1(__dmul_rn(-2.0, ax), use_fma);
      z = __ddiv_rn(-t, __dadd_rn(t, 2.0));
    }
  } else {
    z = 1.0;
  }
  return neg ? -z : z;
}

// ------------------------------------------------------------- warp policy
struct WarpScratch {
  double* f;   // [in]
  double* h1;  // [H]
  double* h2;  // [H]
  double* pr;  // [out]
};

// Combine for the argmax: larger score wins, ties -> lower node index. This is
// exactly the sequential scan of policies.hpp:32-41 / :60-73 / :153-167 for
// finite scores (strict '>' keeps the first maximum).
__device__ __forceinline__ void argmax_combine(double& v, int& i, double v2, int i2) {
  if (i2 >= 0 && (i < 0 || v2 > v || (v2 == v && i2 < i))) { v = v2; i = i2; }
}

__device__ __forceinline__ void warp_argmax(double& v, int& i) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, i, o);
    argmax_combine(v, i, v2, i2);
  }
}

// Evaluates the policy for order t at state (caps[J], row[J]) — both readable
// by every lane. Returns the action on every lane; on a non-finite dual score
// sets *nonfinite = 1 (ContractViolation, policies.hpp:158-161).
template <int KIND>
__device__ int warp_policy_eval(const DevModel& P, const int* caps, const int* row, int t,
                                const WarpScratch& s, int lane, int* nonfinite) {
  const int J = P.J;
  const double* rw = P.rtab + (size_t)P.rrow[t] * J;
  if (KIND == kNull) return -1;
  if (KIND == kGreedy || KIND == kCapacity) {
    int maxc = 0;
    if (KIND == kCapacity) {
      for (int j = lane; j < J; j += 32) maxc = max(maxc, caps[j]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) maxc = max(maxc, __shfl_xor_sync(0xffffffffu, maxc, o));
    }
    double bv = 0.0;
    int bi = -1;
    for (int j = lane; j < J; j += 32) {
      if (caps[j] <= 0 || row[j] <= 0) continue;
      double sc = __ldg(rw + j);
      if (KIND == kCapacity)
        sc = __dadd_rn(sc, __ddiv_rn(__dmul_rn(P.gamma, (double)caps[j]), (double)maxc));
      argmax_combine(bv, bi, sc, j);
    }
    warp_argmax(bv, bi);
    return bi;
  }
  // ---- DualNetworkPolicy::evaluate (policies.hpp:121-168)
  bool feas = false;
  for (int j = lane; j < J; j += 32) feas |= caps[j] > 0 && row[j] > 0;
  if (!__any_sync(0xffffffffu, feas)) return -1;
  const int p = P.product[t];
  const int* irow = P.pinv0 + (size_t)p * J;
  for (int j = lane; j < J; j += 32) {
    const int c0 = __ldg(P.pcap0 + j);
    const int x0 = __ldg(irow + j);
    s.f[j] = c0 > 0 ? __ddiv_rn((double)caps[j], (double)c0) : 0.0;
    s.f[J + j] = x0 > 0 ? __ddiv_rn((double)row[j], (double)x0) : 0.0;
  }
  if (lane == 0) {
    const int ot = P.order_t ? P.order_t[t] : t;
    s.f[2 * J] = P.horizon > 0 ? __ddiv_rn((double)ot, (double)P.horizon) : 0.0;
  }
  __syncwarp();
  const int H = P.H, in = P.in, out = P.out;
  // Each output keeps the reference's sequential acc += w * x chain
  // (mlp.cpp:141-169, no contraction); a lane runs several outputs' chains
  // side by side for instruction-level parallelism.
  for (int r = lane; r < H; r += 64) {
    const bool two = r + 32 < H;
    double a0 = __ldg(P.b1 + r), a1 = two ? __ldg(P.b1 + r + 32) : 0.0;
    const double* w = P.w1t + r;
    for (int c = 0; c < in; ++c) {
      const double f = s.f[c];
      a0 = __dadd_rn(a0, __dmul_rn(__ldg(w + (size_t)c * H), f));
      if (two) a1 = __dadd_rn(a1, __dmul_rn(__ldg(w + (size_t)c * H + 32), f));
    }
    s.h1[r] = gt_tanh(a0, P.tanh_fma);
    if (two) s.h1[r + 32] = gt_tanh(a1, P.tanh_fma);
  }
  __syncwarp();
  for (int r = lane; r < H; r += 64) {
    const bool two = r + 32 < H;
    double a0 = __ldg(P.b2 + r), a1 = two ? __ldg(P.b2 + r + 32) : 0.0;
    const double* w = P.w2t + r;
    for (int c = 0; c < H; ++c) {
      const double x = s.h1[c];
      a0 = __dadd_rn(a0, __dmul_rn(__ldg(w + (size_t)c * H), x));
      if (two) a1 = __dadd_rn(a1, __dmul_rn(__ldg(w + (size_t)c * H + 32), x));
    }
    s.h2[r] = gt_tanh(a0, P.tanh_fma);
    if (two) s.h2[r + 32] = gt_tanh(a1, P.tanh_fma);
  }
  __syncwarp();
  for (int r = lane; r < out; r += 128) {
    const bool v1 = r + 32 < out, v2 = r + 64 < out, v3 = r + 96 < out;
    double a0 = __ldg(P.b3 + r), a1 = v1 ? __ldg(P.b3 + r + 32) : 0.0;
    double a2 = v2 ? __ldg(P.b3 + r + 64) : 0.0, a3 = v3 ? __ldg(P.b3 + r + 96) : 0.0;
    const double* w = P.w3t + r;
    for (int c = 0; c < H; ++c) {
      const double x = s.h2[c];
      const double* wc = w + (size_t)c * out;
      a0 = __dadd_rn(a0, __dmul_rn(__ldg(wc), x));
      if (v1) a1 = __dadd_rn(a1, __dmul_rn(__ldg(wc + 32), x));
      if (v2) a2 = __dadd_rn(a2, __dmul_rn(__ldg(wc + 64), x));
      if (v3) a3 = __dadd_rn(a3, __dmul_rn(__ldg(wc + 96), x));
    }
    s.pr[r] = a0;
    if (v1) s.pr[r + 32] = a1;
    if (v2) s.pr[r + 64] = a2;
    if (v3) s.pr[r + 96] = a3;
  }
  __syncwarp();
  double bv = 0.0;
  int bi = -1;
  bool bad = false;
  for (int j = lane; j < J; j += 32) {
    if (caps[j] <= 0 || row[j] <= 0) continue;
    const double sc = __dsub_rn(__dsub_rn(__ldg(rw + j), s.pr[j]), s.pr[J + j]);
    if (!isfinite(sc)) { bad = true; continue; }
    argmax_combine(bv, bi, sc, j);
  }
  if (__any_sync(0xffffffffu, bad)) { *nonfinite = 1; return -1; }
  warp_argmax(bv, bi);
  __syncwarp();
  // best_score starts at 0.0 and declining wins only against negatives.
  return (bi >= 0 && bv >= 0.0) ? bi : -1;
}

}  // namespace pcd
