// tc_recheck.cuh — exact FP64 re-evaluation of one flagged row of a
// tensor-core sweep by its 256-thread half (shared by tc_pp.cu and tc_inc.cu).
//
// DualNetworkPolicy::evaluate (policies.hpp:121-168) in exactly the operation
// order of warp_policy_eval<kDual>: one thread per output neuron runs the
// acc = b; acc += w * x chain on weights read from L2. The caller provides the
// step's capacities and inventory row and a double scratch `vec` of kRcVec
// entries (the half's MMA operand, free between layer 3 and the next step).
#pragma once

#include "tc_common.cuh"

namespace pcd {
namespace rc {

constexpr int kRcThreads = 256;
constexpr int kRcMaxJ = 112;
constexpr int kRcVec = 2 * kRcMaxJ + 2 + 2 * kTcH + 2 * kRcMaxJ;  // f | h1 | h2 | prices

__device__ __forceinline__ void bar_half(int h) {
  asm volatile("bar.sync %0, %1;" ::"r"(1 + h), "r"(kRcThreads) : "memory");
}

// outv[r] = (tanh?)(bias[r] + sum_c W[c][r] * xin[c]) for r < width: one
// thread per output neuron, the weights read straight from L2 (W is [K][width],
// so a warp reads contiguous rows), 16 loads in flight ahead of the chain
__device__ inline void rc_layer(const double* __restrict__ W, const double* __restrict__ bias, int K, int width,
                         const double* xin, double* outv, bool act_tanh, int tanh_fma, int ht, int h) {
  if (ht < width) {
    const uint64_t pol = l2_policy_evict_last();  // the FP64 weights stay L2-resident
    double acc = __ldg(bias + ht);
    const double* w = W + ht;
    int c = 0;
    for (; c + 16 <= K; c += 16) {
      double wv[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) wv[u] = ldg_f64_el(w + (size_t)(c + u) * width, pol);
#pragma unroll
      for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, __dmul_rn(wv[u], xin[c + u]));
    }
    for (; c < K; ++c) acc = __dadd_rn(acc, __dmul_rn(__ldg(w + (size_t)c * width), xin[c]));
    outv[ht] = act_tanh ? gt_tanh(acc, tanh_fma) : acc;
  }
  bar_half(h);
}

// res[0] = exact decision, res[1] = non-finite score flag (res[2] scratch)
__device__ inline void half_recheck(const DevModel& P, double* vec, const int* caps, const int* xrow, int t,
                             int* res, int ht, int h, long long* rprof = nullptr) {
  long long t0 = rprof ? clock64() : 0;
  auto mark = [&](int k) {
    if (rprof) { const long long n = clock64(); rprof[k] += n - t0; t0 = n; }
  };
  const int J = P.J, H = P.H, in = P.in, out = P.out;
  for (int j = ht; j < in; j += kRcThreads) {
    double f;
    if (j < J) {
      const int c0 = __ldg(P.pcap0 + j);
      f = c0 > 0 ? __ddiv_rn((double)caps[j], (double)c0) : 0.0;
    } else if (j < 2 * J) {
      const int x0 = __ldg(P.pinv0 + (size_t)P.product[t] * J + (j - J));
      f = x0 > 0 ? __ddiv_rn((double)xrow[j - J], (double)x0) : 0.0;
    } else {
      const int ot = P.order_t ? P.order_t[t] : t;
      f = P.horizon > 0 ? __ddiv_rn((double)ot, (double)P.horizon) : 0.0;
    }
    vec[j] = f;
  }
  bar_half(h);
  mark(0);
  const int oh1 = 2 * kRcMaxJ + 2, oh2 = oh1 + kTcH, opr = oh2 + kTcH;
  if (P.w3s && H == kTcH && P.fast_margin > 0.0) {
    // Fast path: the same FP64 network in any summation order (four threads
    // per hidden neuron, two per score, fused multiply-adds), scores from the
    // summed price weights W3s = W3[:J] + W3[J:]. Against the reference's
    // ordered FP64 evaluation each score differs by at most E, the rounding
    // bound of the three layers for THESE weights (features in [0, 1], tanh
    // 1-Lipschitz; computed at pcd_create, P.fast_margin = 4E, ~1e-10 for
    // U(-0.1, 0.1) weights). A decision whose margins (best - second, |best|
    // vs the decline score 0) exceed it is therefore the reference's;
    // otherwise the exact ordered chain below decides.
    const int n = ht >> 2, qq = ht & 3;
    {  // layer 1
      const int kq = (in + 3) >> 2, c0 = qq * kq, c1 = min(in, c0 + kq);
      const double* w = P.w1t + n;
      double z = 0.0;
      for (int c = c0; c < c1; c += 8) {
        double wv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) wv[u] = c + u < c1 ? __ldg(w + (size_t)(c + u) * H) : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) z = fma(wv[u], c + u < c1 ? vec[c + u] : 0.0, z);
      }
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      if (qq == 0) vec[oh1 + n] = gt_tanh(z + __ldg(P.b1 + n), P.tanh_fma);
    }
    bar_half(h);
    {  // layer 2
      const int c0 = qq * (kTcH / 4);
      const double* w = P.w2t + n;
      double z = 0.0;
#pragma unroll
      for (int u = 0; u < kTcH / 4; ++u) z = fma(__ldg(w + (size_t)(c0 + u) * H), vec[oh1 + c0 + u], z);
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      z += __shfl_xor_sync(0xffffffffu, z, 2);
      if (qq == 0) vec[oh2 + n] = gt_tanh(z + __ldg(P.b2 + n), P.tanh_fma);
    }
    bar_half(h);
    {  // summed prices ps_j = b3[j] + b3[J+j] + W3s[:, j] . h2, two threads per node
      const int j = ht >> 1, q2 = ht & 1;
      double z = 0.0;
      if (j < J) {
        const double* w = P.w3s + j;
#pragma unroll 8
        for (int u = 0; u < kTcH / 2; ++u) {
          const int l = q2 * (kTcH / 2) + u;
          z = fma(__ldg(w + (size_t)l * J), vec[oh2 + l], z);
        }
      }
      z += __shfl_xor_sync(0xffffffffu, z, 1);
      if (j < J && q2 == 0) vec[opr + j] = z + (__ldg(P.b3 + j) + __ldg(P.b3 + J + j));
    }
    bar_half(h);
    if (ht < 32) {
      const int lane = ht;
      const double* rw = P.rtab + (size_t)P.rrow[t] * J;
      double b1v = -INFINITY, b2v = -INFINITY;
      int bi = -1;
      bool bad = false;
      for (int j = lane; j < J; j += 32) {
        if (caps[j] <= 0 || xrow[j] <= 0) continue;
        const double sc = __ldg(rw + j) - vec[opr + j];
        if (!isfinite(sc)) { bad = true; continue; }
        if (sc > b1v) { b2v = b1v; b1v = sc; bi = j; }
        else if (sc > b2v) b2v = sc;
      }
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double o1 = __shfl_xor_sync(0xffffffffu, b1v, off), o2 = __shfl_xor_sync(0xffffffffu, b2v, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (o1 > b1v || (o1 == b1v && oi >= 0 && (bi < 0 || oi < bi))) {
          b2v = fmax(b1v, o2);
          b1v = o1;
          bi = oi;
        } else {
          b2v = fmax(b2v, o1);
        }
      }
      bad = __any_sync(0xffffffffu, bad);
      // nothing feasible -> decline without a forward pass (policies.hpp:129-131)
      const bool sure = !bad && (bi < 0 || (fabs(b1v) > P.fast_margin && b1v - b2v > P.fast_margin));
      if (lane == 0) {
        res[0] = bi >= 0 && b1v >= 0.0 ? bi : -1;
        res[1] = 0;
        res[2] = sure;
      }
    }
    bar_half(h);
    mark(4);
    if (res[2]) return;
  }
  rc_layer(P.w1t, P.b1, in, H, vec, vec + oh1, true, P.tanh_fma, ht, h);
  mark(1);
  rc_layer(P.w2t, P.b2, H, H, vec + oh1, vec + oh2, true, P.tanh_fma, ht, h);
  mark(2);
  rc_layer(P.w3t, P.b3, H, out, vec + oh2, vec + opr, false, P.tanh_fma, ht, h);
  mark(3);
  if (ht < 32) {  // scores and argmax as warp_policy_eval<kDual>
    const int lane = ht;
    const double* rw = P.rtab + (size_t)P.rrow[t] * J;
    const double* pr = vec + opr;
    bool feas = false;
    for (int j = lane; j < J; j += 32) feas |= caps[j] > 0 && xrow[j] > 0;
    int exact = -1, nonfinite = 0;
    if (__any_sync(0xffffffffu, feas)) {
      double bv = 0.0;
      int bi = -1;
      bool bad = false;
      for (int j = lane; j < J; j += 32) {
        if (caps[j] <= 0 || xrow[j] <= 0) continue;
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
      res[0] = exact;
      res[1] = nonfinite;
    }
  }
  bar_half(h);
  mark(4);
}

}  // namespace rc
}  // namespace pcd
