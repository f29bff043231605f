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
constexpr int kRcOpr = 2 * kRcMaxJ + 2 + 2 * kTcH;                // offset of the prices in vec
// after half_recheck: res[2] = 1 -> vec[kRcOpr + j] holds the summed price
// p_j + p_{J+j} (fast path), 0 -> p_j and p_{J+j} at kRcOpr + j, kRcOpr + J + j

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
  const int oh1 = 2 * kRcMaxJ + 2, oh2 = oh1 + kTcH, opr = kRcOpr;
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
      res[2] = 0;
    }
  }
  bar_half(h);
  mark(4);
}


// k (<= N) 16-byte / 8-byte L2-resident loads issued back to back (volatile:
// ptxas keeps them ahead of their uses, so one L2 round trip covers them all)
template <int N>
__device__ __forceinline__ void ldg2_group(double2 (&v)[N], const double2* p, size_t stride, int k, uint64_t pol) {
#pragma unroll
  for (int u = 0; u < N; ++u) {
    if (u < k)
      asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                   : "=d"(v[u].x), "=d"(v[u].y)
                   : "l"(p + (size_t)u * stride), "l"(pol));
    else
      v[u] = make_double2(0.0, 0.0);
  }
}
__device__ __forceinline__ double2 ldg2_el(const double2* p, uint64_t pol) {
  double2 v;
  asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
  return v;
}
template <int N>
__device__ __forceinline__ void ldg1_group(double (&v)[N], const double* p, size_t stride, uint64_t pol) {
#pragma unroll
  for (int u = 0; u < N; ++u)
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v[u]) : "l"(p + (size_t)u * stride), "l"(pol));
}

// ---------------------------------------------------------------------------
// The fast path for up to kRcBatch flagged rows at once (same arithmetic as
// half_recheck's fast path; each L2 weight load now serves every row of the
// batch). Scratch: per row b, lo + b kRcRow doubles = f[2J+1] | h1[64] at
// kRcH1 (h2 and the summed prices reuse f's slots once layer 1 is done:
// h2 at 0, ps at kTcH); ints + b 2 kRcMaxJ = caps[J] | xrow[J]; per-row
// results rb + 4 b: [0] decision, [1] non-finite, [2] sure (the fast path's
// margins cleared fast_margin; else the caller runs the ordered chain).
constexpr int kRcBatch = 4;
constexpr int kRcH1 = 2 * kRcMaxJ + 2;
constexpr int kRcRow = kRcH1 + kTcH;
// per-row slot description: [0] t, [1] product, [2] run (row of xloc), [3]
// reward row, [4] order time (the row agent's bookkeeping, so no dependent
// lookups through the order tape)
constexpr int kRcRowInfo = 5;
constexpr int kRcBatchInts = kRcBatch * 2 * kRcMaxJ + 4 * kRcBatch + kRcRowInfo * kRcBatch;

// caps[J] of every row must be in ints + b 2 kRcMaxJ; the inventory rows are
// loaded here (xrow[J] filled in for the argmax) together with the
// normalisers, so the whole operand fetch is one round trip
__device__ inline void half_recheck_fast_batch(const DevModel& P, const int* xloc, double* lo, int* ints,
                                               const int* rinfo, int nb, int ht, int h,
                                               long long* rprof = nullptr) {
  long long t0 = rprof ? clock64() : 0;
  auto mark = [&](int k) {
    if (rprof) { const long long n = clock64(); rprof[k] += n - t0; t0 = n; }
  };
  const int J = P.J, H = P.H, in = P.in;
  int* rb = ints + kRcBatch * 2 * kRcMaxJ;
  for (int idx = ht; idx < nb * in; idx += kRcThreads) {
    const int b = idx / in, j = idx - b * in;
    int* caps = ints + b * 2 * kRcMaxJ;
    int* xrow = caps + kRcMaxJ;
    const int* ri = rinfo + kRcRowInfo * b;
    double f;
    if (j < J) {
      const int c0 = __ldg(P.pcap0 + j);
      f = c0 > 0 ? __ddiv_rn((double)caps[j], (double)c0) : 0.0;
    } else if (j < 2 * J) {
      const int x = xloc[(size_t)ri[2] * J + (j - J)];
      const int x0 = __ldg(P.pinv0 + (size_t)ri[1] * J + (j - J));
      xrow[j - J] = x;
      f = x0 > 0 ? __ddiv_rn((double)x, (double)x0) : 0.0;
    } else {
      f = P.horizon > 0 ? __ddiv_rn((double)ri[4], (double)P.horizon) : 0.0;
    }
    lo[b * kRcRow + j] = f;
  }
  bar_half(h);
  mark(0);
  // layers 1 and 2: thread = (neuron pair np, input eighth e); 16-byte weight
  // loads (w1t / w2t are [in][64]), up to 15 in flight per thread
  const int np = ht >> 3, e = ht & 7, n0 = 2 * np;
  // the 8 lanes of a pair reduce, then lane e finishes (neuron n0 + (e & 1), row e >> 1)
  auto finish = [&](double (&z)[kRcBatch][2], const double* bias, int out_off) {
#pragma unroll
    for (int b = 0; b < kRcBatch; ++b)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        z[b][k] += __shfl_xor_sync(0xffffffffu, z[b][k], 1);
        z[b][k] += __shfl_xor_sync(0xffffffffu, z[b][k], 2);
        z[b][k] += __shfl_xor_sync(0xffffffffu, z[b][k], 4);
      }
    const int rb_ = e >> 1, k_ = e & 1;
    double zz = 0.0;
#pragma unroll
    for (int b = 0; b < kRcBatch; ++b)
#pragma unroll
      for (int k = 0; k < 2; ++k) zz = (b == rb_ && k == k_) ? z[b][k] : zz;
    if (rb_ < nb) lo[rb_ * kRcRow + out_off + n0 + k_] = gt_tanh(zz + __ldg(bias + n0 + k_), P.tanh_fma);
  };
  {  // layer 1 -> h1
    const int ke = (in + 7) >> 3, c0 = e * ke, c1 = min(in, c0 + ke);
    const double2* w = (const double2*)(P.w1t + n0);
    const uint64_t pol = l2_policy_evict_last();  // the FP64 weights stay L2-resident
    double z[kRcBatch][2] = {};
    for (int cb = c0; cb < c1; cb += 14) {
      double2 wv[14];
      ldg2_group(wv, w + (size_t)cb * (H / 2), H / 2, c1 - cb, pol);
#pragma unroll
      for (int u = 0; u < 14; ++u)
#pragma unroll
        for (int b = 0; b < kRcBatch; ++b)
          if (b < nb && cb + u < c1) {
            const double f = lo[b * kRcRow + cb + u];
            z[b][0] = fma(wv[u].x, f, z[b][0]);
            z[b][1] = fma(wv[u].y, f, z[b][1]);
          }
    }
    finish(z, P.b1, kRcH1);
  }
  bar_half(h);
  mark(1);
  {  // layer 2 -> h2 (slots 0..63 of the row)
    const int c0 = e * (kTcH / 8);
    const double2* w = (const double2*)(P.w2t + n0);
    const uint64_t pol = l2_policy_evict_last();
    double2 wv[kTcH / 8];
    ldg2_group(wv, w + (size_t)c0 * (H / 2), H / 2, kTcH / 8, pol);
    double z[kRcBatch][2] = {};
#pragma unroll
    for (int u = 0; u < kTcH / 8; ++u)
#pragma unroll
      for (int b = 0; b < kRcBatch; ++b)
        if (b < nb) {
          const double x = lo[b * kRcRow + kRcH1 + c0 + u];
          z[b][0] = fma(wv[u].x, x, z[b][0]);
          z[b][1] = fma(wv[u].y, x, z[b][1]);
        }
    finish(z, P.b2, 0);
  }
  bar_half(h);
  mark(2);
  {  // summed prices ps_j (slots kTcH.. of the row), two threads per node, 16 loads in flight
    const int j = ht >> 1, q2 = ht & 1;
    double z[kRcBatch] = {0.0, 0.0, 0.0, 0.0};
    if (j < J) {
      const double* w = P.w3s + j;
      const uint64_t pol = l2_policy_evict_last();
#pragma unroll
      for (int ub = 0; ub < kTcH / 2; ub += 16) {
        double wv[16];
        ldg1_group(wv, w + (size_t)(q2 * (kTcH / 2) + ub) * J, J, pol);
#pragma unroll
        for (int u = 0; u < 16; ++u)
#pragma unroll
          for (int b = 0; b < kRcBatch; ++b)
            if (b < nb) z[b] = fma(wv[u], lo[b * kRcRow + q2 * (kTcH / 2) + ub + u], z[b]);
      }
    }
#pragma unroll
    for (int b = 0; b < kRcBatch; ++b) z[b] += __shfl_xor_sync(0xffffffffu, z[b], 1);
    if (j < J && q2 == 0) {
      const double b3 = __ldg(P.b3 + j) + __ldg(P.b3 + J + j);
#pragma unroll
      for (int b = 0; b < kRcBatch; ++b)
        if (b < nb) lo[b * kRcRow + kTcH + j] = z[b] + b3;
    }
  }
  bar_half(h);
  mark(3);
  {  // argmax and the fast path's certificate: warp b decides row b
    const int b = ht >> 5, lane = ht & 31;
    if (b < nb) {
      const int* caps = ints + b * 2 * kRcMaxJ;
      const int* xrow = caps + kRcMaxJ;
      const double* rw = P.rtab + (size_t)rinfo[kRcRowInfo * b + 3] * J;
      const double* ps = lo + b * kRcRow + kTcH;
      double b1v = -INFINITY, b2v = -INFINITY;
      int bi = -1;
      bool bad = false;
      for (int j = lane; j < J; j += 32) {
        if (caps[j] <= 0 || xrow[j] <= 0) continue;
        const double sc = __ldg(rw + j) - ps[j];
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
      const bool sure = !bad && (bi < 0 || (fabs(b1v) > P.fast_margin && b1v - b2v > P.fast_margin));
      if (lane == 0) {
        rb[4 * b] = bi >= 0 && b1v >= 0.0 ? bi : -1;
        rb[4 * b + 1] = 0;
        rb[4 * b + 2] = sure;
      }
    }
  }
  bar_half(h);
  mark(4);
}

// The exact ordered chain for one row (no fast path): the reference's
// operation order (rc_layer), for rows the batched fast path could not certify.
__device__ inline void half_recheck_ordered(const DevModel& P, double* vec, const int* caps, const int* xrow, int t,
                                            int* res, int ht, int h) {
  DevModel Q = P;
  Q.fast_margin = 0.0;  // skips half_recheck's fast path
  half_recheck(Q, vec, caps, xrow, t, res, ht, h);
}

}  // namespace rc
}  // namespace pcd
