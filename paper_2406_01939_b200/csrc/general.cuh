// general.cuh — closed-form sweep for ANY partition and any cache
// (PCD_ENGINE_GENERAL).
//
// The reference's sweep_one_process (engine.hpp:299-342) replays the frozen
// cache over the whole window for every process. Every attempt on (product i,
// node j) — a non-null cached action at a slot the process does not own, or
// one of its own fresh decisions — succeeds iff node j is alive and
// x[i][j] > 0, so with A^m_u[i][j] = attempts in [lo, u):
//   C_u[j]   = ckcap[j] - sum_i min(x0[i][j], A_u[i][j])      (non-increasing)
//   c_u[j]   = max(0, C_u[j]);   tau_j = first u with C_u[j] <= 0
//   x_u[i][j] = x0[i][j] - min(x0[i][j], A_{min(u, tau_j)}[i][j])
// A = G + delta, G_u[i][j] = non-null cache entries (i, j) in [lo, u) and
// delta = own fresh - own cached. sum_i min(x0, G_u) is process-independent:
// H_u[j], the effective-attempt prefix count of k_effective/k_hist_prefix.
// Each process walks only its own slots and carries the sparse delta as a
// list of (product, node) entries; an entry is dropped once its
// (product, node) group has saturated (its term is zero from then on).
// G_u queries are binary searches in per-(product, node) slot lists of the
// window (one radix sort per iteration); delta at an earlier time comes from
// the chain of the process's earlier own slots of the same product.
#pragma once

#include <climits>

#include "kernels.cuh"

namespace pcd {

// window entries keyed by (product, node); null / out-of-range actions go to
// the bucket nullkey
static __global__ void k_gen_keys(const int* __restrict__ cache, const int* __restrict__ product, int lo, int hi,
                                  int J, int nullkey, int* __restrict__ keys, int* __restrict__ vals) {
  const long long n = hi - lo;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const int s = lo + (int)i, a = cache[s];
    keys[i] = (a >= 0 && a < J) ? product[s] * J + a : nullkey;
    vals[i] = s;
  }
}

// product of every plan position (pslots order: owner-major, time-ordered)
static __global__ void k_plan_pkeys(const int* __restrict__ pslots, const int* __restrict__ product, long long T,
                                    int* __restrict__ keys, int* __restrict__ vals) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < T; k += (long long)gridDim.x * blockDim.x) {
    keys[k] = product[pslots[k]];
    vals[k] = (int)k;
  }
}

// prev[k] = the plan position of the same process's previous slot of the same
// product, -1 if none (input: positions stably sorted by product)
static __global__ void k_prev_same(const int* __restrict__ skeys, const int* __restrict__ spos,
                                   const int* __restrict__ pslots, const int* __restrict__ owner, long long T,
                                   int* __restrict__ prev) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < T; i += (long long)gridDim.x * blockDim.x) {
    const int k = spos[i];
    int pv = -1;
    if (i > 0 && skeys[i - 1] == skeys[i] && owner[pslots[spos[i - 1]]] == owner[pslots[k]]) pv = spos[i - 1];
    prev[k] = pv;
  }
}

struct GenArgs {
  DevModel model;
  int M, J, lo, hi;
  const int* pstart;
  const int* pslots;
  const int* prev;     // [T] same-product chain over plan positions
  const int* ckcap;
  const int* ckinv;
  const int* hck;
  const int* ev;
  const int* gstart;   // [I*J + 2] window entry lists by (product, node)
  const int* gslots;
  int* ocache;         // [T] by plan position: the slot's cached action (null if not an attempt)
  int* ofresh;         // [T] by plan position: the slot's fresh action
  int4* dl;            // [2T] delta entries {key, delta, cursor, node}, 2 per plan position
  int* cache;
  unsigned char* written;
  const int* ref;
  Scalars* scal;
  long long* evals_out;
  const unsigned char* mine;
};

__host__ __device__ inline size_t gen_warp_smem_bytes(int J, int in, int H, int out) {
  const size_t ibytes = ((size_t)5 * J * 4 + 15) & ~(size_t)15;
  return ibytes + (size_t)(in + 2 * H + out) * 8;
}

// min(x0, g + d) - min(x0, g): the term of one delta entry
__device__ __forceinline__ int gen_term(int x0, int g, int d) { return min(x0, g + d) - min(x0, g); }

// H_u[j]: effective cached attempts at node j in [lo, u)
__device__ __forceinline__ int gen_h_at(const GenArgs& a, int u, int j) {
  const int base = hck_base(a.lo), b = (u - base) >> kLogK;
  int h = a.hck[(size_t)b * hck_stride(a.J) + j];
  for (int v = max(a.lo, base + (b << kLogK)); v < u; ++v) h += a.ev[v] == j ? 1 : 0;
  return h;
}

// delta[p][j] from own slots of the chain before slot u (and inside the window)
__device__ __forceinline__ int gen_chain_delta(const GenArgs& a, int pos, int j, int u) {
  int d = 0;
  for (int v = a.prev[pos]; v >= 0; v = a.prev[v]) {
    const int sv = a.pslots[v];
    if (sv < a.lo) break;
    if (sv < u) d += (a.ofresh[v] == j ? 1 : 0) - (a.ocache[v] == j ? 1 : 0);
  }
  return d;
}

template <int KIND>
static __global__ void __launch_bounds__(128) k_sweep_general(GenArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * (blockDim.x >> 5) + warp;
  if (m >= a.M || (a.mine && !a.mine[m])) return;
  const int J = a.J, lo = a.lo, hi = a.hi;
  const size_t ibytes = ((size_t)5 * J * 4 + 15) & ~(size_t)15;
  unsigned char* w = smem + gen_warp_smem_bytes(J, a.model.in, a.model.H, a.model.out) * warp;
  int* cv = (int*)w;    // C_t, then c_t
  int* xr = cv + J;     // x_t[p]
  int* corr = xr + J;   // sum of the delta terms per node
  int* tau = corr + J;  // death slots (INT_MAX: alive so far)
  int* dp = tau + J;    // delta[p][.] of the current product p over own slots in [lo, t)
  WarpScratch ws;
  {
    double* d = (double*)(w + ibytes);
    ws.f = d;
    ws.h1 = d + a.model.in;
    ws.h2 = ws.h1 + a.model.H;
    ws.pr = ws.h2 + a.model.H;
  }
  const int beg = a.pstart[m], n = a.pstart[m + 1] - beg;
  const int* sl = a.pslots + beg;
  int k = lower_bound_i32(sl, n, lo);
  if (k >= n || sl[k] >= hi) return;
  int4* dl = a.dl + 2 * (size_t)beg;
  int nd = 0;
  for (int j = lane; j < J; j += 32) tau[j] = INT_MAX;
  const int HJ = hck_stride(J), base = hck_base(lo);
  const unsigned ltmask = (1u << lane) - 1u;
  int sprev = lo - 1;
  int curp = -1;  // product of the previous own slot (dp and the dead nodes' x are its)
  unsigned long long changed = 0, conflicts = 0, first = ~0ull, nev = 0;
  long long mism = 0;
  __syncwarp();
  for (; k < n; ++k) {
    const int t = sl[k];
    if (t >= hi) break;
    const int pos = beg + k;
    const int p = a.model.product[t];
    const int aold = a.cache[t];
    const int cold = (aold >= 0 && aold < J) ? aold : -1;
    // delta terms at t (cursors advance to t)
    for (int j = lane; j < J; j += 32) corr[j] = 0;
    __syncwarp();
    for (int e = lane; e < nd; e += 32) {
      int4 d = dl[e];
      const int kb = a.gstart[d.x], ke = a.gstart[d.x + 1];
      int cur = d.z;
      while (cur < ke && a.gslots[cur] < t) ++cur;
      dl[e].z = cur;
      const int f = gen_term(a.ckinv[d.x], cur - kb, d.y);
      if (f) atomicAdd(&corr[d.w], f);
    }
    __syncwarp();
    // C_t = ckcap - H_t - corr
    const int b = (t - base) >> kLogK;
    const int* hrow = a.hck + (size_t)b * HJ;
    for (int j = lane; j < J; j += 32) cv[j] = a.ckcap[j] - hrow[j] - corr[j];
    __syncwarp();
    for (int v = max(lo, base + (b << kLogK)) + lane; v < t; v += 32) {
      const int e = a.ev[v];
      if (e >= 0) atomicSub(&cv[e], 1);
    }
    __syncwarp();
    // nodes that died since the previous own slot: tau in (sprev, t]
    for (int j = lane; j < J; j += 32) {
      if (tau[j] != INT_MAX || cv[j] > 0) continue;
      int l = sprev + 1, r = t;
      while (l < r) {
        const int u = l + ((r - l) >> 1);
        int c = a.ckcap[j] - gen_h_at(a, u, j);
        for (int e = 0; e < nd; ++e) {
          const int4 d = dl[e];
          if (d.w != j) continue;
          const int kb = a.gstart[d.x], ke = a.gstart[d.x + 1];
          c -= gen_term(a.ckinv[d.x], lower_bound_i32(a.gslots + kb, ke - kb, u), d.y);
        }
        if (c <= 0) r = u; else l = u + 1;
      }
      tau[j] = l;
    }
    __syncwarp();
    // drop saturated entries (zero from t on; the searches above still saw them)
    {
      int wr = 0;
      for (int e0 = 0; e0 < nd; e0 += 32) {
        const int e = e0 + lane;
        int4 d = make_int4(0, 0, 0, 0);
        bool keep = false;
        if (e < nd) {
          d = dl[e];
          const int g = d.z - a.gstart[d.x], x0 = a.ckinv[d.x];
          keep = d.y > 0 ? g < x0 : (d.y < 0 && g + d.y < x0);
        }
        const unsigned bal = __ballot_sync(0xffffffffu, keep);
        if (keep) dl[wr + __popc(bal & ltmask)] = d;
        wr += __popc(bal);
        __syncwarp();
      }
      nd = wr;
    }
    // local state at t: capacities and the order's inventory row. Runs of own
    // slots of one product update dp incrementally and keep the frozen x of
    // nodes that were already dead; a product switch walks the chain once.
    const bool same = p == curp;
    if (!same)
      for (int j = lane; j < J; j += 32) dp[j] = gen_chain_delta(a, pos, j, t);
    for (int j = lane; j < J; j += 32) {
      const int c = cv[j];
      cv[j] = max(c, 0);
      if (c <= 0 && same && tau[j] <= sprev) continue;  // dead before the previous own slot: x frozen
      const int key = p * J + j;
      const int kb = a.gstart[key], ke = a.gstart[key + 1];
      const int A = c > 0 ? lower_bound_i32(a.gslots + kb, ke - kb, t) + dp[j]
                          : lower_bound_i32(a.gslots + kb, ke - kb, tau[j]) + gen_chain_delta(a, pos, j, tau[j]);
      const int x0 = a.ckinv[key];
      xr[j] = x0 - min(x0, A);
    }
    __syncwarp();
    int nonfinite = 0;
    const int anew = warp_policy_eval<KIND>(a.model, cv, xr, t, ws, lane, &nonfinite);
    ++nev;
    if (nonfinite) {
      const int ot = a.model.order_t ? a.model.order_t[t] : t;
      if (lane == 0) atomicMin(&a.scal->err_nonfinite, ((unsigned long long)m << 32) | (unsigned)ot);
      break;
    }
    const bool infeasible = anew >= J || (anew >= 0 && !(cv[anew] > 0 && xr[anew] > 0));
    __syncwarp();
    if (infeasible) {
      if (lane == 0) atomicMin(&a.scal->err_infeasible, ((unsigned long long)m << 32) | (unsigned)t);
      break;
    }
    // delta entries of (p, cold) and (p, anew)
    if (cold != anew) {
#pragma unroll 1
      for (int q = 0; q < 2; ++q) {
        const int j = q ? anew : cold;
        if (j < 0) continue;  // warp-uniform
        const int dlt = dp[j] + (anew == j ? 1 : 0) - (cold == j ? 1 : 0);
        const int key = p * J + j;
        int found = -1;
        for (int e0 = 0; e0 < nd; e0 += 32) {
          const int e = e0 + lane;
          const unsigned bal = __ballot_sync(0xffffffffu, e < nd && dl[e].x == key);
          if (bal) {
            found = e0 + __ffs(bal) - 1;
            break;
          }
        }
        if (lane == 0) {
          if (found >= 0) {
            dl[found].y = dlt;
          } else if (dlt != 0) {
            const int kb = a.gstart[key], ke = a.gstart[key + 1];
            dl[nd] = make_int4(key, dlt, kb + lower_bound_i32(a.gslots + kb, ke - kb, t), j);
          }
        }
        if (found < 0 && dlt != 0) ++nd;
        __syncwarp();
      }
    }
    if (lane == 0) {
      if (cold >= 0) dp[cold] -= 1;
      if (anew >= 0) dp[anew] += 1;
      a.ocache[pos] = cold;
      a.ofresh[pos] = anew;
      if (anew != aold) {
        ++changed;
        first = min(first, (unsigned long long)t);
        conflicts += a.written[t] ? 1 : 0;
      }
      if (a.ref) mism += (long long)(anew != a.ref[t]) - (long long)(aold != a.ref[t]);
      a.cache[t] = anew;
      a.written[t] = 1;
    }
    __syncwarp();
    sprev = t;
    curp = p;
  }
  if (lane == 0) {
    if (changed) {
      atomicAdd(&a.scal->changed, changed);
      atomicAdd(&a.scal->conflicts, conflicts);
      atomicMin(&a.scal->first_changed, first);
    }
    if (mism) atomicAdd((unsigned long long*)&a.scal->mismatch_delta, (unsigned long long)mism);
    atomicMax(&a.scal->max_evals, nev);
    atomicAdd(&a.scal->total_evals, nev);
    if (a.evals_out) a.evals_out[m] = (long long)nev;
  }
}

}  // namespace pcd
