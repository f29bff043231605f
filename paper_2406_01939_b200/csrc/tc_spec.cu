// tc_spec.cu — verification of the tensor-core sweep's speculated decisions.
//
// A row whose decision margins lie between 1/256 of the derived guards and the
// guards (tc_pp.cu, combine) takes the tensor-core argmax at once and appends
// its slot to a queue instead of stalling its half for an FP64
// re-evaluation. After the sweep this kernel re-derives, for every queued
// slot, the exact state the row saw and evaluates the reference policy on it
// in FP64, in the reference's operation order (warp_policy_eval<kDual>, the
// same code as the FP64 engine). Any disagreement sets Scalars::spec_bad and
// the host re-runs the whole iteration without speculation from backups of
// the window's cache and written flags (engine.cu run_iteration), so every
// published decision is the reference's.
//
// The state of a row at its slot t (run-partition closed form, DESIGN.md
// §4.2/4.2b), from the process's own slots [pos0, end) in pslots:
//   D_j   = sum over own slots s < t of ([ev[s] == j] - [cache[s] == j])
//   c_j   = max(0, ckcap_j - (hck row of t's block)_j - #{ev == j in the block before t} + D_j)
//   x_j   = xloc[run]_j (after the sweep) + #{own slots s >= t of the run with cache[s] == j}
// (cache[] holds the sweep's fresh decisions: every slot has one owner).
#include <cuda_runtime.h>

#include <algorithm>

#include "tc_common.cuh"

namespace pcd {
namespace spec {

constexpr int kWarps = 16;

// shared memory: the FP64 weights (w1t [in][H] | w2t [H][H] | w3s [H][J] | b1 |
// b2 | b3s [J]; J even, so every row of w3s starts 16-byte aligned) then per
// warp: caps[J] | row[J] (ints), f[max(in, out), padded to even] (the ordered
// fallback's prices overwrite f once layer 1 has read it) | h1[H] | h2[H]
__host__ __device__ inline size_t weights_doubles(int J, int in, int H) {
  return (size_t)in * H + (size_t)H * H + (size_t)H * J + 2 * (size_t)H + J;
}
__host__ __device__ inline size_t warp_bytes(int J, int in, int H, int out) {
  const int fo = ((in > out ? in : out) + 1) & ~1;  // f, later the fallback's prices
  return (((size_t)2 * J * 4 + 15) & ~(size_t)15) + (size_t)(fo + 2 * H) * 8;
}

__global__ void __launch_bounds__(kWarps * 32, 1) k_spec_verify(SweepArgs S, const int* __restrict__ q,
                                                               const int* __restrict__ qn, int cap, int force_bad) {
  extern __shared__ __align__(16) unsigned char vsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const DevModel& P = S.model;
  const int J = S.J, H = P.H, in = P.in;
  const int n = min(*qn, cap);
  if (n <= 0 || (int)blockIdx.x * nw >= n) return;
  double* sw = (double*)vsm;
  double* w1 = sw;
  double* w2 = w1 + (size_t)in * H;
  double* w3 = w2 + (size_t)H * H;
  double* b1 = w3 + (size_t)H * J;
  double* b2 = b1 + H;
  double* b3s = b2 + H;
  // the three weight matrices by TMA bulk copies (one thread, one mbarrier)
  __shared__ __align__(8) uint64_t wbar;
  if (threadIdx.x == 0) {
    mbar_init(&wbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const uint32_t n1 = (uint32_t)in * H * 8, n2 = (uint32_t)H * H * 8, n3 = (uint32_t)H * J * 8;
    mbar_expect_tx(&wbar, n1 + n2 + n3);
    bulk_load(w1, P.w1t, n1, &wbar);
    bulk_load(w2, P.w2t, n2, &wbar);
    bulk_load(w3, P.w3s, n3, &wbar);
  }
  for (int i = threadIdx.x; i < H; i += blockDim.x) {
    b1[i] = __ldg(P.b1 + i);
    b2[i] = __ldg(P.b2 + i);
  }
  for (int j = threadIdx.x; j < J; j += blockDim.x) b3s[j] = __ldg(P.b3 + j) + __ldg(P.b3 + J + j);
  __syncthreads();
  mbar_wait(&wbar, 0);
  unsigned char* wb = vsm + weights_doubles(J, in, H) * 8 + (size_t)warp * warp_bytes(J, in, H, P.out);
  int* crow = (int*)wb;
  int* prow = crow + J;
  double* f = (double*)(wb + (((size_t)2 * J * 4 + 15) & ~(size_t)15));
  double* h1 = f + (((in > P.out ? in : P.out) + 1) & ~1);  // (16-byte aligned pairs)
  double* h2 = h1 + H;
  const int base = hck_base(S.lo), HJ = hck_stride(J);
  for (int e = blockIdx.x * nw + warp; e < n; e += gridDim.x * nw) {
    const int* E = q + (size_t)e * kSpecStride;
    const int t = E[0], pos = E[1], pos0 = E[2], end = E[3], x = E[5], p = E[6], rr = E[7], ot = E[8], dec = E[9];
    // ---- the row's state at t (see the file comment); crow holds D first
    for (int j = lane; j < J; j += 32) {
      crow[j] = 0;
      prow[j] = 0;
    }
    __syncwarp();
    // the own slots 32 x kGroup at a time: every load of a group in flight at once
    constexpr int kGroup = 4;
    for (int k0 = pos0; k0 < end; k0 += 32 * kGroup) {
      int sl[kGroup], dd[kGroup], aa[kGroup], rr_[kGroup];
#pragma unroll
      for (int u = 0; u < kGroup; ++u) {
        const int k = k0 + 32 * u + lane;
        sl[u] = k < end ? S.pslots[k] : -1;
      }
#pragma unroll
      for (int u = 0; u < kGroup; ++u) {
        const int k = k0 + 32 * u + lane;
        dd[u] = sl[u] >= 0 ? S.cache[sl[u]] : -1;
        aa[u] = sl[u] >= 0 && k < pos ? S.ev[sl[u]] : -1;
        rr_[u] = sl[u] >= 0 && k >= pos ? S.rid[sl[u]] : -1;
      }
#pragma unroll
      for (int u = 0; u < kGroup; ++u) {
        const int k = k0 + 32 * u + lane;
        if (sl[u] < 0) continue;
        if (k < pos) {
          if (aa[u] >= 0) atomicAdd(&crow[aa[u]], 1);
          if (dd[u] >= 0) atomicSub(&crow[dd[u]], 1);
        } else if (dd[u] >= 0 && rr_[u] == x) {
          atomicAdd(&prow[dd[u]], 1);
        }
      }
    }
    __syncwarp();
    const int b = (t - base) >> kLogK;
    const int sb = max(S.lo, base + (b << kLogK));
    // the <= 7 events of t's block before t, one per lane, counted by shuffles
    const int evk = sb + lane < t && lane < 8 ? S.ev[sb + lane] : -1;
    int evs[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) evs[k] = __shfl_sync(0xffffffffu, evk, k);
    bool feas = false;
    for (int j = lane; j < J; j += 32) {
      int hh = S.hck[(size_t)b * HJ + j];
#pragma unroll
      for (int k = 0; k < 8; ++k) hh += evs[k] == j ? 1 : 0;
      const int c = max(0, S.ckcap[j] - hh + crow[j]);
      const int xv = prow[j] + S.xloc[(size_t)x * J + j];
      crow[j] = c;
      prow[j] = xv;
      feas |= c > 0 && xv > 0;
      const int c0 = __ldg(P.pcap0 + j), x0 = __ldg(P.pinv0 + (size_t)p * J + j);
      f[j] = c0 > 0 ? __ddiv_rn((double)c, (double)c0) : 0.0;
      f[J + j] = x0 > 0 ? __ddiv_rn((double)xv, (double)x0) : 0.0;
    }
    if (lane == 0) f[2 * J] = P.horizon > 0 ? __ddiv_rn((double)ot, (double)P.horizon) : 0.0;
    __syncwarp();
    int exact;
    bool sure = true;
    if (!__any_sync(0xffffffffu, feas)) {
      exact = -1;  // nothing feasible: decline without a forward pass (policies.hpp:129-131)
    } else {
      // ---- order-free FP64 forward from shared memory (the in-sweep fast path's
      // arithmetic and certificate: margins above fast_margin decide exactly)
      // (H == 64: lane l owns outputs 2l and 2l + 1, read as one 16-byte
      // shared-memory word; inputs in pairs on two chains — the certificate
      // holds for any summation order, fast_margin_bound)
      {
        const int o = 2 * lane;
        double2 ae = *(const double2*)(b1 + o), ao = make_double2(0.0, 0.0);
        int c = 0;
        for (; c + 2 <= in; c += 2) {
          const double2 fc = *(const double2*)(f + c);
          const double2 we = *(const double2*)(w1 + (size_t)c * H + o);
          const double2 wo = *(const double2*)(w1 + (size_t)(c + 1) * H + o);
          ae.x = fma(we.x, fc.x, ae.x);
          ae.y = fma(we.y, fc.x, ae.y);
          ao.x = fma(wo.x, fc.y, ao.x);
          ao.y = fma(wo.y, fc.y, ao.y);
        }
        if (c < in) {
          const double fc = f[c];
          const double2 we = *(const double2*)(w1 + (size_t)c * H + o);
          ae.x = fma(we.x, fc, ae.x);
          ae.y = fma(we.y, fc, ae.y);
        }
        *(double2*)(h1 + o) = make_double2(gt_tanh(ae.x + ao.x, P.tanh_fma), gt_tanh(ae.y + ao.y, P.tanh_fma));
      }
      __syncwarp();
      {
        const int o = 2 * lane;
        double2 ae = *(const double2*)(b2 + o), ao = make_double2(0.0, 0.0);
        for (int c = 0; c < H; c += 2) {
          const double2 hc = *(const double2*)(h1 + c);
          const double2 we = *(const double2*)(w2 + (size_t)c * H + o);
          const double2 wo = *(const double2*)(w2 + (size_t)(c + 1) * H + o);
          ae.x = fma(we.x, hc.x, ae.x);
          ae.y = fma(we.y, hc.x, ae.y);
          ao.x = fma(wo.x, hc.y, ao.x);
          ao.y = fma(wo.y, hc.y, ao.y);
        }
        *(double2*)(h2 + o) = make_double2(gt_tanh(ae.x + ao.x, P.tanh_fma), gt_tanh(ae.y + ao.y, P.tanh_fma));
      }
      __syncwarp();
      const double* rw = P.rtab + (size_t)rr * J;
      double b1v = -INFINITY, b2v = -INFINITY;
      int bi = -1;
      bool bad = false;
      // layer 3: lane l owns nodes 2l, 2l + 1 and 64 + 2l, 65 + 2l (J even:
      // 16-byte aligned pairs in the [H][J] rows)
      double2 za = make_double2(0.0, 0.0), zb = make_double2(0.0, 0.0);
      const int ja = 2 * lane, jb = 64 + 2 * lane;
      const bool va = ja < J, vb = jb < J;
      if (va) za = make_double2(b3s[ja], b3s[ja + 1]);
      if (vb) zb = make_double2(b3s[jb], b3s[jb + 1]);
      for (int l = 0; l < H; ++l) {
        const double hl = h2[l];
        const double* wr = w3 + (size_t)l * J;
        if (va) {
          const double2 w = *(const double2*)(wr + ja);
          za.x = fma(w.x, hl, za.x);
          za.y = fma(w.y, hl, za.y);
        }
        if (vb) {
          const double2 w = *(const double2*)(wr + jb);
          zb.x = fma(w.x, hl, zb.x);
          zb.y = fma(w.y, hl, zb.y);
        }
      }
      const double zq[4] = {za.x, za.y, zb.x, zb.y};
      const int jq[4] = {ja, ja + 1, jb, jb + 1};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = jq[u];
        if (j >= J || crow[j] <= 0 || prow[j] <= 0) continue;
        const double sc = __ldg(rw + j) - zq[u];
        if (!isfinite(sc)) { bad = true; continue; }
        if (sc > b1v || (sc == b1v && j < bi)) { b2v = b1v; b1v = sc; bi = j; }
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
      sure = !bad && P.fast_margin > 0.0 &&
             (bi < 0 || (fabs(b1v) > P.fast_margin && b1v - b2v > P.fast_margin));
      exact = bi >= 0 && b1v >= 0.0 ? bi : -1;
    }
    if (!sure) {  // too close to call in any order: the reference's own operation order
      WarpScratch ws;
      ws.f = f;
      ws.h1 = h1;
      ws.h2 = h2;
      ws.pr = f;  // (the prices are written after layer 1 has consumed f)
      int nonfinite = 0;
      exact = warp_policy_eval<kDual>(P, crow, prow, t, ws, lane, &nonfinite);
      if (nonfinite) exact = -2;  // the sweep must report it: re-run without speculation
    }
    if (lane == 0 && (exact != dec || force_bad)) atomicOr(&S.scal->spec_bad, 1);
    __syncwarp();
  }
}

}  // namespace spec

// warps per CTA: as many as fit next to the weights (12 at J = 100)
static int spec_warps(int J, int in, int H, int out) {
  const size_t wbytes = spec::weights_doubles(J, in, H) * 8, per = spec::warp_bytes(J, in, H, out);
  const size_t cap = 232448 - 64;  // (the static mbarrier)
  const size_t avail = cap > wbytes ? cap - wbytes : 0;
  return (int)std::min<size_t>((size_t)spec::kWarps, avail / per);
}

cudaError_t launch_spec_verify(const SweepArgs& S, const int* q, const int* qn, int cap, int force_bad,
                               cudaStream_t stream) {
  const int J = S.J, in = S.model.in, H = S.model.H, out = S.model.out;
  const int nw = spec_warps(J, in, H, out);
  if (nw < 1) return cudaErrorInvalidConfiguration;
  const size_t smem = spec::weights_doubles(J, in, H) * 8 + spec::warp_bytes(J, in, H, out) * nw;
  const cudaError_t e = ensure_dyn_smem((const void*)spec::k_spec_verify, smem);
  if (e != cudaSuccess) return e;
  spec::k_spec_verify<<<148, nw * 32, smem, stream>>>(S, q, qn, cap, force_bad);
  return cudaGetLastError();
}

}  // namespace pcd
