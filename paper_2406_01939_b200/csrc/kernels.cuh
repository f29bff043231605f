// kernels.cuh — sm_100a kernels of one Picard iteration (engine.hpp:358-444)
// and of the fixed-point driver's checkpoint advance (engine.hpp:514-526).
//
// Device layout (SoA, HBM-resident for the whole run):
//   product[T], rrow[T], order_t[T]       int32   the order tape
//   rtab[R*J]                             f64     rewards, one row per origin
//   owner[T]                              int32   PartitionPlan::owner
//   pstart[M+1], pslots[T]                int32   per-process owned slots (time order)
//   qstart[I+1], qslots[T]                int32   per-product slots (time order)
//   cache[T], fresh[T], ref[T]            int32   ActionCache / fresh / oracle
//   written[T]                            uint8   "slot written before" (conflicts)
//   ckcap[J], ckinv[I*J]                  int32   checkpoint FoState (dense)
//   rid[T]                                int32   run of each slot (run = one process's stretch
//                                                 of one product's slot list)
//   xloc[R*J]                             int32   per-iteration inventory of every run
//   ev[T]                                 int32   effective cached attempt (node or -1)
//   hck[nb*HJ]                            int32   hck[b][j] = H(b)[j] = effective attempts at
//                                                 node j in [lo, base + 8b), base = lo & ~7
//                                                 (K=8 blocks aligned on absolute slots; rows
//                                                 padded to 8 nodes = 32 bytes)
//   seg[nseg*SJ]                          int32   scratch: per-segment totals / offsets
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include "device_policy.cuh"

namespace pcd {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: record the
// largest size set for each (kernel, device) and raise it when a launch needs
// more. Returns the CUDA status of the call (cudaSuccess when nothing to do).
inline cudaError_t ensure_dyn_smem(const void* kernel, size_t bytes) {
  if (bytes <= 48 * 1024) return cudaSuccess;
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& have = done[{kernel, dev}];
  if (have >= bytes) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) have = bytes;
  return e;
}

constexpr int kLogK = 3;  // checkpoint stride K = 8 slots (partial block <= 7 events)
constexpr int kK = 1 << kLogK;
constexpr int kLogSeg = 6;
constexpr int kSegRows = 1 << kLogSeg;  // checkpoint rows per scan segment

__host__ __device__ __forceinline__ int hck_stride(int J) { return (J + 7) & ~7; }  // 32-byte rows
__host__ __device__ __forceinline__ int seg_stride(int J) { return (J + 7) & ~7; }
__host__ __device__ __forceinline__ int hck_base(int lo) { return lo & ~(kK - 1); }
// checkpoint rows covering the window [lo, hi)
__host__ __device__ __forceinline__ int hck_rows(int lo, int hi) {
  return (hi - hck_base(lo) + kK - 1) >> kLogK;
}

struct Scalars {
  unsigned long long changed;
  unsigned long long first_changed;  // min
  unsigned long long conflicts;
  long long mismatch_delta;
  unsigned long long max_evals;
  unsigned long long total_evals;
  unsigned long long err_nonfinite;  // min over (m << 32 | t)
  unsigned long long err_infeasible; // min over (m << 32 | t)
  int neg_flag;
  int spec_bad;                      // a speculated tensor-core decision was wrong (tc_spec.cu)
  long long mismatches;              // full-cache mismatch count (init kernel)
};

__device__ __forceinline__ int lower_bound_i32(const int* a, int n, int key) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// Effective-attempt pass (run-partition closed form).
// For every product, walk its slots of the window in time order; the cached
// attempt at slot t (node a) is *effective* iff fewer than ckinv[p][a]
// earlier cached attempts of the same (product, node) exist in the window —
// i.e. it would succeed inventory-wise with unlimited capacity.
// One warp per product, 32 slots per round: the rank of an attempt among the
// equal (product, node) attempts of the round comes from __match_any_sync,
// the running per-node counts live in the warp's smem row.
// ---------------------------------------------------------------------------
// First index in [0, n) with a[i] >= key (n if none), by the whole warp: a
// 32-ary search (every lane probes one point per round, a ballot picks the
// sub-range), ~log32(n) dependent loads instead of log2(n). Warp-uniform call.
__device__ __forceinline__ int warp_lower_bound(const int* __restrict__ a, int n, int key) {
  const int lane = threadIdx.x & 31;
  int l = 0, r = n;  // the answer lies in [l, r]
  while (l < r) {
    const long long span = r - l;
    const int pos = l + (int)(span * lane / 32);  // in [l, r - 1], nondecreasing in the lane
    const unsigned ge = __ballot_sync(0xffffffffu, a[pos] >= key);
    if (!ge) {
      l = l + (int)(span * 31 / 32) + 1;  // beyond the last probe
    } else {
      const int k = __ffs(ge) - 1;        // first lane at or above the key (a is sorted)
      r = l + (int)(span * k / 32);
      if (k > 0) l = l + (int)(span * (k - 1) / 32) + 1;
    }
  }
  return l;
}

// first index >= from whose entry is >= key (a sorted; from <= the answer):
// two 32-wide forward probes, then the 32-ary search of the rest
__device__ __forceinline__ int warp_advance(const int* __restrict__ a, int n, int from, int key) {
  const int lane = threadIdx.x & 31;
  for (int r = 0; r < 2 && from < n; ++r, from += 32) {
    const int k = from + lane;
    const unsigned ge = __ballot_sync(0xffffffffu, k < n && a[k] >= key);
    if (ge) return from + __ffs(ge) - 1;
  }
  return from >= n ? n : from + warp_lower_bound(a + from, n - from, key);
}

// [k0, k1): product p's slots inside the window [lo, hi) (warp-uniform call).
// cur (or nullptr: 32-ary searches) holds per product the previous window's
// bounds; inside simulate windows only move forward, so both bounds are
// found by a short forward scan from them (mode 1 advances and stores them,
// mode 2 reads this window's, stored by an earlier kernel of the iteration)
__device__ __forceinline__ void product_window(const int* __restrict__ qstart, const int* __restrict__ qslots, int p,
                                               int lo, int hi, const int*& sl, int& k0, int& k1,
                                               int2* cur = nullptr, int mode = 0) {
  const int beg = qstart[p], n = qstart[p + 1] - beg;
  sl = qslots + beg;
  if (cur && mode == 2) {
    const int2 c = cur[p];
    k0 = c.x;
    k1 = c.y;
  } else if (cur) {
    const int2 c = cur[p];
    k0 = warp_advance(sl, n, c.x, lo);
    k1 = warp_advance(sl, n, max(c.y, k0), hi);
    if ((threadIdx.x & 31) == 0) cur[p] = make_int2(k0, k1);
  } else {
    k0 = warp_lower_bound(sl, n, lo);
    k1 = k0 + warp_lower_bound(sl + k0, n - k0, hi);
  }
}

static __global__ void k_effective(const int* __restrict__ qstart, const int* __restrict__ qslots, int I,
                                   int lo, int hi, const int* __restrict__ cache,
                                   const int* __restrict__ ckinv, int J, int* __restrict__ ev,
                                   int2* __restrict__ qcur = nullptr) {
  extern __shared__ int cnt_smem[];  // per warp: cnt[J], x0[J]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int p = blockIdx.x * (blockDim.x >> 5) + warp;
  if (p >= I) return;  // warp-uniform
  int* cnt = cnt_smem + warp * 2 * J;
  int* x0 = cnt + J;
  for (int j = lane; j < J; j += 32) {
    cnt[j] = 0;
    x0[j] = ckinv[(size_t)p * J + j];
  }
  const int* sl;
  int k0, k1;
  product_window(qstart, qslots, p, lo, hi, sl, k0, k1, qcur, 1);
  const unsigned lt = (1u << lane) - 1u;
  __syncwarp();
  // 64 slots per round, both halves' loads in flight before either is ranked
  for (int b = k0; b < k1; b += 64) {
    const int kA = b + lane, kB = b + 32 + lane;
    const bool vA = kA < k1, vB = kB < k1;
    const int tA = vA ? sl[kA] : 0, tB = vB ? sl[kB] : 0;
    const int aA = vA ? cache[tA] : -1, aB = vB ? cache[tB] : -1;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool valid = h ? vB : vA;
      const int t = h ? tB : tA, a = h ? aB : aA;
      const bool att = valid && a >= 0 && a < J;
      const unsigned peers = __match_any_sync(0xffffffffu, att ? a : -1);
      const int rank = __popc(peers & lt);
      const int c = att ? cnt[a] : 0;
      const int e = att && c + rank < x0[a] ? a : -1;
      if (valid) ev[t] = e;
      __syncwarp();
      if (att && rank == 0) cnt[a] = c + __popc(peers);
      __syncwarp();
    }
  }
}

// Death slot of every node under the frozen cache: tau[j] = the slot of the
// effective attempt at node j whose index (in window order) is ckcap[j] —
// the first one that finds the node empty when the cache is replayed from
// the checkpoint; INT_MAX when the node never empties in the window.
// Death slot of every node under the frozen cache: one warp per node runs a
// 32-ary search for the last checkpoint row with H <= ckcap (4 dependent
// rounds over ~4e4 rows instead of 16 binary-search steps), then scans that
// row's <= 8-slot block for the effective attempt numbered ckcap.
static __global__ void k_tau(const int* __restrict__ hck, const int* __restrict__ ev, const int* __restrict__ ckcap,
                             int lo, int hi, int J, int nb, int* __restrict__ tau) {
  const int lane = threadIdx.x & 31;
  const int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (j >= J) return;  // warp-uniform
  const int HJ = hck_stride(J), c = ckcap[j], base = hck_base(lo);
  // last checkpoint row with H <= c (row 0 holds 0); H is nondecreasing in the row
  int l = 0, r = nb - 1;
  while (l < r) {
    const long long span = r - l;
    const int pos = l + (int)((span * (lane + 1) + 31) / 32);  // pos(31) == r, pos(0) >= l + 1
    const unsigned ok = __ballot_sync(0xffffffffu, hck[(size_t)pos * HJ + j] <= c);
    if (!ok) {
      r = l + (int)((span + 31) / 32) - 1;
    } else {
      const int k = 31 - __clz(ok);  // the ok lanes are a prefix
      const int lk = l + (int)((span * (k + 1) + 31) / 32);
      r = k == 31 ? lk : l + (int)((span * (k + 2) + 31) / 32) - 1;
      l = lk;
    }
  }
  if (lane == 0) {
    int h = hck[(size_t)l * HJ + j], out = 0x7fffffff;
    const int s1 = min(hi, base + ((l + 1) << kLogK));
    for (int s = max(lo, base + (l << kLogK)); s < s1; ++s) {
      if (ev[s] != j) continue;
      if (h == c) { out = s; break; }
      ++h;
    }
    tau[j] = out;
  }
}

// Inventory of every run at its first slot in the window (run partitions:
// each (process, product) pair owns one contiguous stretch of the product's
// slot list). Before its first own slot a process holds the replay state of
// the frozen cache, so
//   xloc[run][j] = ckinv[p][j] - #{effective cached attempts (p, j) in
//                                  [lo, first slot) that precede tau[j]}.
// One warp per product walks the window slots in time order with per-node
// counts in smem and writes a row at every run start. (256, 8): 32
// registers, 64 warps per SM, so the 10^4 product warps of C3 take 1.06
// waves instead of 1.4 (prep 7.4 -> 7.3 ms)
static __global__ void __launch_bounds__(256, 8) k_xinit(const int* __restrict__ qstart, const int* __restrict__ qslots, int I, int lo,
                               int hi, const int* __restrict__ ev, const int* __restrict__ rid,
                               const int* __restrict__ tau, const int* __restrict__ ckinv, int J,
                               int* __restrict__ xloc, int2* __restrict__ qcur = nullptr) {
  extern __shared__ int cnt_smem[];  // tau[J] (block), then cnt[J] per warp
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int* stau = cnt_smem;
  for (int j = threadIdx.x; j < J; j += blockDim.x) stau[j] = tau[j];
  __syncthreads();
  const int p = blockIdx.x * (blockDim.x >> 5) + warp;
  if (p >= I) return;  // warp-uniform
  int* cnt = cnt_smem + J + warp * J;
  for (int j = lane; j < J; j += 32) cnt[j] = 0;
  const int* sl;
  int k0, k1;
  product_window(qstart, qslots, p, lo, hi, sl, k0, k1, qcur, 2);
  const int* x0 = ckinv + (size_t)p * J;
  int prev_run = -1;
  __syncwarp();
  for (int b0 = k0; b0 < k1; b0 += 64) {
    const int kA = b0 + lane, kB = b0 + 32 + lane;
    const bool vA = kA < k1, vB = kB < k1;
    const int tA = vA ? sl[kA] : 0, tB = vB ? sl[kB] : 0;
    const int eA = vA ? ev[tA] : -1, eB = vB ? ev[tB] : -1;
    const int rA = vA ? rid[tA] : -1, rB = vB ? rid[tB] : -1;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const bool valid = hh ? vB : vA;
      const int t = hh ? tB : tA, e = hh ? eB : eA, r = hh ? rB : rA;
      const bool contrib = e >= 0 && t < stau[e];
      int pr = __shfl_up_sync(0xffffffffu, r, 1);
      if (lane == 0) pr = prev_run;
      unsigned starts = __ballot_sync(0xffffffffu, valid && r != pr);
      int done = 0;
      while (starts) {
        const int L = __ffs(starts) - 1;
        starts &= starts - 1;
        if (contrib && lane >= done && lane < L) atomicAdd(&cnt[e], 1);
        __syncwarp();
        const int rr = __shfl_sync(0xffffffffu, r, L);
        int* xr = xloc + (size_t)rr * J;
        for (int j = lane; j < J; j += 32) xr[j] = x0[j] - cnt[j];
        __syncwarp();
        done = L;
      }
      if (contrib && lane >= done) atomicAdd(&cnt[e], 1);
      prev_run = __shfl_sync(0xffffffffu, r, 31);
      __syncwarp();
    }
  }
}

// Time Warp windows on product partitions: every product is one run, whose
// inventory at its first window slot is the checkpoint's.
static __global__ void k_xinit_plain(const int* __restrict__ qstart, const int* __restrict__ qslots, int I, int lo,
                                     int hi, const int* __restrict__ rid, const int* __restrict__ ckinv, int J,
                                     int* __restrict__ xloc) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= I) return;
  const int* sl;
  int k0, k1;
  product_window(qstart, qslots, warp, lo, hi, sl, k0, k1);
  if (k0 >= k1) return;
  int* xr = xloc + (size_t)rid[sl[k0]] * J;
  for (int j = lane; j < J; j += 32) xr[j] = ckinv[(size_t)warp * J + j];
}

// Time Warp rollback (fo/timewarp.hpp:150-170): re-execute [lo, hi) strictly
// serially against the global state (one warp, the exact FP64 policy).
// err[0] = time step of the first failure, err[1] = 1 infeasible / 2 non-finite
template <int KIND>
static __global__ void k_serial_window(DevModel model, int lo, int hi, int* __restrict__ ckcap,
                                       int* __restrict__ ckinv, int* __restrict__ cache, long long* err) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, J = model.J;
  int* caps = (int*)smem;
  int* row = caps + J;
  WarpScratch ws;
  double* d = (double*)(smem + ((2 * J * 4 + 15) & ~15));
  ws.f = d;
  ws.h1 = d + model.in;
  ws.h2 = ws.h1 + model.H;
  ws.pr = ws.h2 + model.H;
  for (int j = lane; j < J; j += 32) caps[j] = ckcap[j];
  __syncwarp();
  for (int t = lo; t < hi; ++t) {
    const int p = model.product[t];
    for (int j = lane; j < J; j += 32) row[j] = ckinv[(size_t)p * J + j];
    __syncwarp();
    int nonfinite = 0;
    const int a = warp_policy_eval<KIND>(model, caps, row, t, ws, lane, &nonfinite);
    const bool bad = nonfinite || a >= J || (a >= 0 && !(caps[a] > 0 && row[a] > 0));
    __syncwarp();
    if (bad) {
      if (lane == 0) {
        err[0] = nonfinite ? (model.order_t ? model.order_t[t] : t) : t;
        err[1] = nonfinite ? 2 : 1;
      }
      return;
    }
    if (lane == 0) {
      if (a >= 0) {
        caps[a] -= 1;
        ckinv[(size_t)p * J + a] -= 1;
      }
      cache[t] = a;
    }
    __syncwarp();
  }
  for (int j = lane; j < J; j += 32) ckcap[j] = caps[j];
}

// Depletion profile: keys = node of every fulfilment (J for declines) so a
// stable radix sort lists each node's fulfilments in time order; then
// first_depleted_at[j] = (slot of the cap0[j]-th fulfilment) + 1, or 0 when
// cap0[j] == 0, or T when the node never empties before the last order.
static __global__ void k_fulfil_keys(const int* __restrict__ a, long long T, int J, int* __restrict__ keys) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    const int v = a[t];
    keys[t] = (v >= 0 && v < J) ? v : J;
  }
}
static __global__ void k_depletion(const int* __restrict__ start, const int* __restrict__ slots,
                                   const int* __restrict__ cap0, int J, long long T, long long* __restrict__ out) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int c = cap0[j], n = start[j + 1] - start[j];
  long long d = T;
  if (c <= 0) d = T > 0 ? 0 : T;
  else if (n >= c) d = min(T, (long long)slots[start[j] + c - 1] + 1);
  out[j] = d;
}

// Run structure of a plan along the product slot lists (qslots, time order
// per product): run_start[k] = 1 where a product's list starts or the owner
// changes.
static __global__ void k_run_starts(const int* __restrict__ qslots, const int* __restrict__ product,
                                    const int* __restrict__ owner, long long T, int* __restrict__ flag) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < T; k += (long long)gridDim.x * blockDim.x) {
    const int t = qslots[k];
    int st = 1;
    if (k > 0) {
      const int tp = qslots[k - 1];
      st = product[tp] != product[t] || owner[tp] != owner[t];
    }
    flag[k] = st;
  }
}
// rid[t] = run of slot t; per process the number of runs and whether any of
// them is non-leading (does not start at its product's first slot).
static __global__ void k_run_ids(const int* __restrict__ qslots, const int* __restrict__ qstart,
                                 const int* __restrict__ product, const int* __restrict__ owner,
                                 const int* __restrict__ flag, const int* __restrict__ incl, long long T,
                                 int* __restrict__ rid, int* __restrict__ nruns, int* __restrict__ nonlead) {
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < T; k += (long long)gridDim.x * blockDim.x) {
    const int t = qslots[k];
    rid[t] = incl[k] - 1;
    if (flag[k]) {
      const int m = owner[t];
      atomicAdd(&nruns[m], 1);
      if (k != qstart[product[t]]) atomicOr(&nonlead[m], 1);
    }
  }
}
// The closed form needs every process to hold the replay state of the frozen
// cache before each of its runs: true when the process owns a single run, or
// only leading runs (no other process touches those products earlier).
static __global__ void k_check_runs(const int* __restrict__ nruns, const int* __restrict__ nonlead, int M,
                                    int* flag) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int bad = m < M && nruns[m] > 1 && nonlead[m];
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

// Work list of one iteration: window load of every process of this rank
// (owned slots in [lo, hi)); the engine sorts (load desc) so the rows of the
// tensor-core sweep pull the longest processes first.
static __global__ void k_window_load(const int* __restrict__ pstart, const int* __restrict__ pslots, int M, int lo,
                                     int hi, const unsigned char* __restrict__ mine, int* __restrict__ load,
                                     int* __restrict__ ids, int* __restrict__ nq, int* __restrict__ wbeg) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  int n = 0, k0 = 0;
  const int beg = pstart[m];
  if (!mine || mine[m]) {
    const int c = pstart[m + 1] - beg;
    k0 = lower_bound_i32(pslots + beg, c, lo);
    n = k0 < c && pslots[beg + k0] < hi ? lower_bound_i32(pslots + beg, c, hi) - k0 : 0;
  }
  load[m] = n;
  ids[m] = m;
  if (wbeg) wbeg[m] = beg + k0;  // the process's first window position (the sweep's rows start there)
  if (n) atomicAdd(nq, 1);
}

// Prefix counts of effective attempts, reduce-then-scan over segments of
// kSegRows K-slot blocks: (1) per-segment totals, (2) exclusive scan of the
// totals per node (seg[] then holds H at every segment start), (3) per-block
// histograms in smem scanned from the segment offset and written once as the
// final prefix (ev is read twice, hck written once).
static __global__ void k_seg_count(const int* __restrict__ ev, int lo, int hi, int J, int* __restrict__ seg) {
  extern __shared__ int cs[];  // [J]
  const int sg = blockIdx.x, SJ = seg_stride(J);
  for (int j = threadIdx.x; j < J; j += blockDim.x) cs[j] = 0;
  __syncthreads();
  const int base = hck_base(lo);
  const int s0 = max(lo, base + (sg << (kLogSeg + kLogK))), s1 = min(hi, base + ((sg + 1) << (kLogSeg + kLogK)));
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const int e = ev[s];
    if (e >= 0) atomicAdd(&cs[e], 1);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < SJ; j += blockDim.x) seg[(size_t)sg * SJ + j] = j < J ? cs[j] : 0;
}

// Exclusive scan of the segment totals over segments, per node: the segments
// are cut into gridDim.x ranges; thread j of a block walks node j down its
// range (a row of seg is read coalesced by the block). (a) range totals,
// (b) one block scans the range totals, (c) ranges apply their offsets.
static __global__ void k_seg_scan_a(const int* __restrict__ seg, int nseg, int J, int* __restrict__ tot) {
  const int SJ = seg_stride(J), per = (nseg + gridDim.x - 1) / gridDim.x;
  const int s0 = blockIdx.x * per, s1 = min(nseg, s0 + per);
  for (int j = threadIdx.x; j < SJ; j += blockDim.x) {
    int sum = 0;
#pragma unroll 8
    for (int s = s0; s < s1; ++s) sum += seg[(size_t)s * SJ + j];
    tot[(size_t)blockIdx.x * SJ + j] = sum;
  }
}
// one block per node column, a block-wide scan over the (<= 256) range totals
static __global__ void k_seg_scan_b(int* __restrict__ tot, int nblk, int J) {
  __shared__ int sh[256];
  const int SJ = seg_stride(J), j = blockIdx.x, b = threadIdx.x;
  const int v = b < nblk ? tot[(size_t)b * SJ + j] : 0;
  sh[b] = v;
  __syncthreads();
  for (int off = 1; off < 256; off <<= 1) {
    const int add = b >= off ? sh[b - off] : 0;
    __syncthreads();
    sh[b] += add;
    __syncthreads();
  }
  if (b < nblk) tot[(size_t)b * SJ + j] = sh[b] - v;  // exclusive
}
static __global__ void k_seg_scan_c(int* __restrict__ seg, int nseg, int J, const int* __restrict__ tot) {
  const int SJ = seg_stride(J), per = (nseg + gridDim.x - 1) / gridDim.x;
  const int s0 = blockIdx.x * per, s1 = min(nseg, s0 + per);
  for (int j = threadIdx.x; j < SJ; j += blockDim.x) {
    int acc = tot[(size_t)blockIdx.x * SJ + j];
    for (int s = s0; s < s1; ++s) {
      const int v = seg[(size_t)s * SJ + j];
      seg[(size_t)s * SJ + j] = acc;
      acc += v;
    }
  }
}

static __global__ void k_hist_prefix(const int* __restrict__ ev, int lo, int hi, int J, int nb,
                                     const int* __restrict__ seg, int* __restrict__ hck) {
  extern __shared__ int hs[];  // [kSegRows][J]
  const int sg = blockIdx.x, HJ = hck_stride(J), SJ = seg_stride(J);
  const int b0 = sg << kLogSeg, nrows = min(kSegRows, nb - b0);
  for (int i = threadIdx.x; i < kSegRows * J; i += blockDim.x) hs[i] = 0;
  __syncthreads();
  const int base = hck_base(lo), sb = base + (b0 << kLogK);
  const int s0 = max(lo, sb), s1 = min(hi, sb + (nrows << kLogK));
  for (int s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const int e = ev[s];
    if (e >= 0) atomicAdd(&hs[((s - sb) >> kLogK) * J + e], 1);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    int acc = seg[(size_t)sg * SJ + j];
    for (int r = 0; r < nrows; ++r) {
      const int v = hs[r * J + j];
      hs[r * J + j] = acc;
      acc += v;
    }
  }
  __syncthreads();
  // rows of HJ ints as 16-byte stores: lane -> 4-column group, warp -> rows
  const int nw = blockDim.x >> 5, lane = threadIdx.x & 31, HJ4 = HJ >> 2;
  for (int c = lane; c < HJ4; c += 32)
    for (int r = threadIdx.x >> 5; r < nrows; r += nw) {
      const int j = 4 * c;
      int4 v;
      v.x = j < J ? hs[r * J + j] : 0;
      v.y = j + 1 < J ? hs[r * J + j + 1] : 0;
      v.z = j + 2 < J ? hs[r * J + j + 2] : 0;
      v.w = j + 3 < J ? hs[r * J + j + 3] : 0;
      *(int4*)(hck + (size_t)(b0 + r) * HJ + j) = v;
    }
}

struct SweepArgs {
  DevModel model;
  int M, J, lo, hi;
  const int* pstart;
  const int* pslots;
  const int* ckcap;
  const int* hck;
  const int* ev;
  int* xloc;
  const int* rid;
  int nocache;  // Time Warp windows: every other process's step counts as declined (H = 0)
  int* cache;
  unsigned char* written;
  const int* ref;
  Scalars* scal;
  long long* evals_out;  // optional [M]
  const unsigned char* mine;  // [M] processes of this rank (multi-GPU), nullptr = all
};

__device__ __forceinline__ void carve_warp_smem(unsigned char* base, int warp, int J, int in, int H,
                                                int out, int*& D, int*& crow, int*& prow,
                                                WarpScratch& ws) {
  const size_t ints = (size_t)3 * J;
  const size_t ibytes = (ints * 4 + 15) & ~(size_t)15;
  const size_t per = ibytes + (size_t)(in + 2 * H + out) * 8;
  unsigned char* w = base + per * warp;
  D = (int*)w;
  crow = D + J;
  prow = crow + J;
  double* d = (double*)(w + ibytes);
  ws.f = d;
  ws.h1 = d + in;
  ws.h2 = ws.h1 + H;
  ws.pr = ws.h2 + H;
}

__host__ __device__ inline size_t warp_smem_bytes(int J, int in, int H, int out) {
  const size_t ibytes = ((size_t)3 * J * 4 + 15) & ~(size_t)15;
  return ibytes + (size_t)(in + 2 * H + out) * 8;
}

// ---------------------------------------------------------------------------
// Closed-form sweep for run partitions (product partitions, and product
// chunks: every process's slots of a product form one contiguous stretch of
// the product's slot list, k_check_runs). One warp per process walks ONLY its
// own slots of the window; the local state at own slot t (run r, product p) is
//   c[j] = max(0, ckcap[j] - H_t[j] + Hown_t[j] - F_t[j])
//   x[p][j] = xloc[r][j] - F_t[p][j]           (xloc from k_xinit)
// where H_t = effective cached attempts in [lo,t) (hck + partial block scan),
// Hown_t the effective attempts at own slots before t and F_t the process's
// own fresh fulfilments before t. This equals the state the reference's
// sweep_one_process (engine.hpp:299-342) reaches by replaying the window
// (proof: DESIGN.md §4.2). The barrier publish (engine.hpp:434-443) and the
// driver counters (engine.hpp:543-553) are fused in: each slot has exactly one
// owner and no other process reads cache[t] after the effective pass.
// ---------------------------------------------------------------------------
template <int KIND>
static __global__ void __launch_bounds__(128, 8) k_sweep_product(SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * (blockDim.x >> 5) + warp;
  if (m >= a.M || (a.mine && !a.mine[m])) return;
  const int J = a.J;
  int *D, *crow, *prow;
  WarpScratch ws;
  carve_warp_smem(smem, warp, J, a.model.in, a.model.H, a.model.out, D, crow, prow, ws);
  const int beg = a.pstart[m], n = a.pstart[m + 1] - beg;
  const int* sl = a.pslots + beg;
  int k = lower_bound_i32(sl, n, a.lo);
  if (k >= n || sl[k] >= a.hi) return;
  for (int j = lane; j < J; j += 32) D[j] = 0;
  __syncwarp();
  unsigned long long changed = 0, conflicts = 0, first = ~0ull, nev = 0;
  long long mism = 0;
  for (; k < n; ++k) {
    const int t = sl[k];
    if (t >= a.hi) break;
    const int aold = a.cache[t];
    const int evt = a.nocache ? -1 : a.ev[t];
    const int b = (t - hck_base(a.lo)) >> kLogK;
    const int* hrow = a.nocache ? nullptr : a.hck + (size_t)b * hck_stride(J);
    int* xrow = a.xloc + (size_t)a.rid[t] * J;
    for (int j = lane; j < J; j += 32) {
      crow[j] = a.ckcap[j] - (hrow ? hrow[j] : 0) + D[j];
      prow[j] = xrow[j];
    }
    __syncwarp();
    if (!a.nocache)
      for (int s = max(a.lo, hck_base(a.lo) + (b << kLogK)) + lane; s < t; s += 32) {
        const int e = a.ev[s];
        if (e >= 0) atomicSub(&crow[e], 1);
      }
    __syncwarp();
    for (int j = lane; j < J; j += 32) crow[j] = max(crow[j], 0);
    __syncwarp();
    int nonfinite = 0;
    const int anew = warp_policy_eval<KIND>(a.model, crow, prow, t, ws, lane, &nonfinite);
    ++nev;
    if (nonfinite) {
      const int ot = a.model.order_t ? a.model.order_t[t] : t;
      if (lane == 0) atomicMin(&a.scal->err_nonfinite, ((unsigned long long)m << 32) | (unsigned)ot);
      break;
    }
    const bool infeasible = anew >= J || (anew >= 0 && !(crow[anew] > 0 && prow[anew] > 0));
    __syncwarp();
    if (infeasible) {
      if (lane == 0) atomicMin(&a.scal->err_infeasible, ((unsigned long long)m << 32) | (unsigned)t);
      break;
    }
    if (lane == 0) {
      if (evt >= 0) D[evt] += 1;
      if (anew >= 0) {
        D[anew] -= 1;
        xrow[anew] -= 1;
      }
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

struct ReplayArgs {
  DevModel model;
  int M, J, I, lo, hi, m0, m1;
  const int* owner;
  const int* pstart;
  const int* pslots;
  const int* ckcap;
  const int* ckinv;
  const int* cache;
  int* fresh;
  int* scratch;  // [(m1-m0) * I * J]
  Scalars* scal;
  long long* evals_out;
  const unsigned char* mine;  // [M] or nullptr
};

// ---------------------------------------------------------------------------
// Exact replay sweep for ANY partition (sweep_one_process, engine.hpp:299-342):
// one warp per process replays [lo, stop_after] against the frozen cache with
// a private dense copy of the checkpoint state; fresh values go to fresh[t]
// and are published by k_publish after all processes finished (the barrier).
// ---------------------------------------------------------------------------
template <int KIND>
static __global__ void __launch_bounds__(128) k_sweep_replay(ReplayArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = a.m0 + blockIdx.x * (blockDim.x >> 5) + warp;
  if (m >= a.m1 || (a.mine && !a.mine[m])) return;
  const int J = a.J;
  int *caps, *unused1, *unused2;
  WarpScratch ws;
  carve_warp_smem(smem, warp, J, a.model.in, a.model.H, a.model.out, caps, unused1, unused2, ws);
  const int beg = a.pstart[m], n = a.pstart[m + 1] - beg;
  const int* sl = a.pslots + beg;
  const int k_hi = lower_bound_i32(sl, n, a.hi);
  if (k_hi == 0 || sl[k_hi - 1] < a.lo) return;
  const int stop = sl[k_hi - 1];
  int* inv = a.scratch + (size_t)(m - a.m0) * a.I * J;
  for (int j = lane; j < J; j += 32) caps[j] = a.ckcap[j];
  for (size_t i = lane; i < (size_t)a.I * J; i += 32) inv[i] = a.ckinv[i];
  __syncwarp();
  unsigned long long nev = 0;
  for (int t = a.lo; t <= stop; ++t) {
    const int p = a.model.product[t];
    int* row = inv + (size_t)p * J;
    if (a.owner[t] == m) {
      int nonfinite = 0;
      const int anew = warp_policy_eval<KIND>(a.model, caps, row, t, ws, lane, &nonfinite);
      ++nev;
      if (nonfinite) {
        const int ot = a.model.order_t ? a.model.order_t[t] : t;
        if (lane == 0) atomicMin(&a.scal->err_nonfinite, ((unsigned long long)m << 32) | (unsigned)ot);
        break;
      }
      const bool infeasible = anew >= J || (anew >= 0 && !(caps[anew] > 0 && row[anew] > 0));
      __syncwarp();
      if (infeasible) {
        if (lane == 0) atomicMin(&a.scal->err_infeasible, ((unsigned long long)m << 32) | (unsigned)t);
        break;
      }
      if (lane == 0) {
        if (anew >= 0) { caps[anew] -= 1; row[anew] -= 1; }
        a.fresh[t] = anew;
      }
    } else {
      const int c = a.cache[t];
      const bool ok = c >= 0 && c < J && caps[c] > 0 && row[c] > 0;
      __syncwarp();
      if (ok && lane == 0) { caps[c] -= 1; row[c] -= 1; }
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicMax(&a.scal->max_evals, nev);
    atomicAdd(&a.scal->total_evals, nev);
    if (a.evals_out) a.evals_out[m] = (long long)nev;
  }
}

// Barrier publish (engine.hpp:434-443) + driver counters (engine.hpp:543-553).
static __global__ void k_publish(const int* __restrict__ fresh, int* __restrict__ cache,
                          unsigned char* __restrict__ written, const int* __restrict__ ref, int lo,
                          int hi, Scalars* scal) {
  unsigned long long changed = 0, conflicts = 0, first = ~0ull;
  long long mism = 0;
  for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) {
    const int nw = fresh[t], od = cache[t];
    if (nw != od) {
      ++changed;
      first = min(first, (unsigned long long)t);
      conflicts += written[t] ? 1 : 0;
      if (ref) mism += (long long)(nw != ref[t]) - (long long)(od != ref[t]);
      cache[t] = nw;
    }
    written[t] = 1;
  }
  // warp reduce then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
    conflicts += __shfl_xor_sync(0xffffffffu, conflicts, o);
    mism += __shfl_xor_sync(0xffffffffu, mism, o);
    first = min(first, __shfl_xor_sync(0xffffffffu, first, o));
  }
  if ((threadIdx.x & 31) == 0 && changed) {
    atomicAdd(&scal->changed, changed);
    atomicAdd(&scal->conflicts, conflicts);
    atomicMin(&scal->first_changed, first);
    if (mism) atomicAdd((unsigned long long*)&scal->mismatch_delta, (unsigned long long)mism);
  }
}

static __global__ void k_fill(int* p, int v, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = v;
}

static __global__ void k_mismatches(const int* __restrict__ cache, const int* __restrict__ ref, long long T, Scalars* scal) {
  unsigned long long c = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x)
    c += cache[t] != ref[t];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd((unsigned long long*)&scal->mismatches, c);
}

// Checkpoint advance (engine.hpp:514-526 -> apply_in_place, fo/types.hpp:89-100):
// subtract the cache prefix's fulfilments from the checkpoint state.
// The stable prefix's fulfilments subtracted from the checkpoint (capacity by
// a per-block smem histogram, inventory by atomics). A count that goes
// negative, or an action >= J, is an infeasible cached action: the atomics
// return the old values, and a subtraction that crosses zero is seen by the
// thread (block) that makes it, so the check costs no extra pass over the
// checkpoint (neg |= 1; the serial search then finds the order).
static __global__ void k_advance(const int* __restrict__ cache, const int* __restrict__ product, int lo,
                          int hi, int J, int* __restrict__ ckcap, int* __restrict__ ckinv, int* __restrict__ neg) {
  extern __shared__ int hcap[];
  for (int j = threadIdx.x; j < J; j += blockDim.x) hcap[j] = 0;
  __syncthreads();
  bool bad = false;
  for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) {
    const int a = cache[t];
    if (a >= 0 && a < J) {
      atomicAdd(&hcap[a], 1);
      bad |= atomicSub(&ckinv[(size_t)product[t] * J + a], 1) <= 0;
    } else if (a >= J) {
      bad = true;
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < J; j += blockDim.x)
    if (hcap[j]) bad |= atomicSub(&ckcap[j], hcap[j]) < hcap[j];
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(neg, 1);
}


// k_advance taken back (a rejected speculation, or the error path's replay):
// the same fulfilments added back, so the checkpoint is exactly the one before.
static __global__ void k_unadvance(const int* __restrict__ cache, const int* __restrict__ product, int lo, int hi,
                                   int J, int* __restrict__ ckcap, int* __restrict__ ckinv) {
  extern __shared__ int hcap[];
  for (int j = threadIdx.x; j < J; j += blockDim.x) hcap[j] = 0;
  __syncthreads();
  for (int t = lo + blockIdx.x * blockDim.x + threadIdx.x; t < hi; t += gridDim.x * blockDim.x) {
    const int a = cache[t];
    if (a >= 0 && a < J) {
      atomicAdd(&hcap[a], 1);
      atomicAdd(&ckinv[(size_t)product[t] * J + a], 1);
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < J; j += blockDim.x)
    if (hcap[j]) atomicAdd(&ckcap[j], hcap[j]);
}

// Error path only: serial re-application to find the first infeasible order.
static __global__ void k_advance_serial(const int* __restrict__ cache, const int* __restrict__ product,
                                 const int* __restrict__ order_t, int lo, int hi, int J,
                                 int* __restrict__ ckcap, int* __restrict__ ckinv, long long* err_t) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  *err_t = -1;
  for (int t = lo; t < hi; ++t) {
    const int a = cache[t];
    if (a < 0) continue;
    int* row = ckinv + (size_t)product[t] * J;
    if (a >= J || ckcap[a] <= 0 || row[a] <= 0) {
      *err_t = order_t ? order_t[t] : t;
      return;
    }
    ckcap[a] -= 1;
    row[a] -= 1;
  }
}

// Owned-slot counts per process inside [lo, hi) (evals_per_process).
static __global__ void k_window_evals(const int* __restrict__ pstart, const int* __restrict__ pslots, int M,
                               int lo, int hi, long long* out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= M) return;
  const int beg = pstart[m], n = pstart[m + 1] - beg;
  out[m] = lower_bound_i32(pslots + beg, n, hi) - lower_bound_i32(pslots + beg, n, lo);
}

static __global__ void k_first_out_of_range(const int* __restrict__ a, long long n, int lo, int hi,
                                            unsigned long long* first) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n; t += (long long)gridDim.x * blockDim.x)
    if (a[t] < lo || a[t] >= hi) atomicMin(first, (unsigned long long)t);
}

// out[i] = 1 / x[i] rounded to float (0 where x[i] <= 0): feature scales of the tensor-core sweep
static __global__ void k_inv_f32(const int* __restrict__ x, long long n, float* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = x[i] > 0 ? (float)(1.0 / (double)x[i]) : 0.f;
}

static __global__ void k_iota(int* p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) p[i] = (int)i;
}

// CSR start offsets from sorted keys: start[k] = first index with key >= k.
static __global__ void k_csr_starts(const int* __restrict__ sorted_keys, long long T, int nkeys, int* __restrict__ start) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i > T) return;
  const int prev = i == 0 ? -1 : sorted_keys[i - 1];
  const int cur = i == T ? nkeys : sorted_keys[i];
  for (int k = prev + 1; k <= cur; ++k) start[k] = (int)i;
}

static __global__ void k_transpose_f64(const double* __restrict__ src, int rows, int cols, double* __restrict__ dst) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= (long long)rows * cols) return;
  const int r = (int)(i / cols), c = (int)(i % cols);
  dst[(size_t)c * rows + r] = src[i];
}

// ---------------------------------------------------------------------------
// Multi-GPU exchange: every rank packs the cache values of
// the slots its processes own (rank-major slot CSR, time order) and one
// ncclAllGather delivers every rank's slice; each rank scatters them back.
// ---------------------------------------------------------------------------
static __global__ void k_pack_slots(const int* __restrict__ src, const int* __restrict__ slots, int n,
                                    int* __restrict__ out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = src[slots[i]];
}
// Window slices of every rank's owned-slot list (exchange): rank r's slots
// d_rslots[start[r] .. start[r] + count[r]) arrive at recv[r * maxw ..).
constexpr int kMaxRanks = 64;
struct RankWindow {
  int start[kMaxRanks];
  int count[kMaxRanks];
};
static __global__ void k_unpack_window(const int* __restrict__ in, const int* __restrict__ slots, RankWindow w,
                                       int nranks, int maxw, int* __restrict__ dst) {
  const long long total = (long long)nranks * maxw;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total; g += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(g / maxw), i = (int)(g % maxw);
    if (i < w.count[r]) dst[slots[w.start[r] + i]] = in[g];
  }
}
// Scalars <-> [sum: changed, conflicts, mismatch, total_evals | min: first,
// err_nonfinite, err_infeasible | max: max_evals] (int64 reduction buffer).
static __global__ void k_scalars_pack(const Scalars* s, long long* b) {
  b[0] = (long long)s->changed; b[1] = (long long)s->conflicts; b[2] = s->mismatch_delta;
  b[3] = (long long)s->total_evals;
  b[4] = (long long)s->first_changed; b[5] = (long long)s->err_nonfinite; b[6] = (long long)s->err_infeasible;
  b[7] = (long long)s->max_evals;
}
static __global__ void k_scalars_unpack(const long long* b, Scalars* s) {
  s->changed = (unsigned long long)b[0]; s->conflicts = (unsigned long long)b[1]; s->mismatch_delta = b[2];
  s->total_evals = (unsigned long long)b[3];
  s->first_changed = (unsigned long long)b[4]; s->err_nonfinite = (unsigned long long)b[5];
  s->err_infeasible = (unsigned long long)b[6];
  s->max_evals = (unsigned long long)b[7];
}

}  // namespace pcd
