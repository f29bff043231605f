// linear.cu — the non-SCO environment of the reference (picard::linear,
// linear.hpp / linear.cpp): a time-varying linear system
//   s_{t+1} = A_t s_t + B_t a_t + w_t,   a_t = G s_t  (GainPolicy)
// and its Picard convergence curve with single-step partitions (M = T,
// picard_convergence_curve, linear.cpp:279-330).
//
// With one process per time step, process t replays the cached actions
// a_0..a_{t-1} from the origin and evaluates G at the state it reaches, so
// one Picard iteration is
//   cache_k[t] = G s_t(cache_{k-1}),  s(cache) = rollout of the cache,
// and the curve scores rollout(cache_k) against the closed-loop (sequential)
// trajectory. The reference replays every prefix per process (O(T^2) per
// iteration); here a rollout is an affine scan over time:
//   (1) every thread composes the affine maps of a chunk of L steps,
//   (2) one thread chains the chunk maps (T/L of them) into chunk-start states,
//   (3) every thread rolls its chunk out from its start state,
// O(T n^2) work per iteration. Scores are block-reduced in a fixed order, so
// runs are deterministic. The reference compares real-valued actions with a
// 1e-9 relative tolerance (LinearEnv::actions_equal); the scan's different
// summation order stays far inside it (tests: tests/test_gpu_linear.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "capi_internal.h"
#include "device_policy.cuh"

namespace pcd {
namespace lin {

#define LCK(x)                                                                             \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x);   \
  } while (0)

constexpr int kChunk = 256;  // steps per scan chunk

struct Buf {
  double* p = nullptr;
  explicit Buf(size_t n) { if (n) LCK(cudaMalloc(&p, n * sizeof(double))); }
  ~Buf() { if (p) cudaFree(p); }
  Buf(const Buf&) = delete;
  Buf& operator=(const Buf&) = delete;
};

// c_t = B_t a_t + w_t (a = cache, or nullptr for the zero actions)
template <int N>
__global__ void k_drive(const double* __restrict__ B, const double* __restrict__ w, const double* __restrict__ a,
                        int P, long long T, double* __restrict__ c) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
      if (a)
        for (int k = 0; k < P; ++k) acc += B[((size_t)t * N + i) * P + k] * a[(size_t)t * P + k];
      c[(size_t)t * N + i] = acc + w[(size_t)t * N + i];
    }
  }
}

// Ac_t = A_t + B_t G (the closed-loop map of the sequential trajectory)
template <int N>
__global__ void k_closed_loop(const double* __restrict__ A, const double* __restrict__ B, const double* __restrict__ G,
                              int P, long long T, double* __restrict__ Ac) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
#pragma unroll
    for (int r = 0; r < N; ++r)
#pragma unroll
      for (int cc = 0; cc < N; ++cc) {
        double acc = A[((size_t)t * N + r) * N + cc];
        for (int k = 0; k < P; ++k) acc += B[((size_t)t * N + r) * P + k] * G[(size_t)k * N + cc];
        Ac[((size_t)t * N + r) * N + cc] = acc;
      }
  }
}

// (1) chunk maps: M_c = A_{e-1} ... A_{b}, v_c = rollout of c over the chunk from 0
template <int N>
__global__ void k_chunk_maps(const double* __restrict__ A, const double* __restrict__ c, long long T, int nchunks,
                             double* __restrict__ Mout, double* __restrict__ vout) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch >= nchunks) return;
  const long long b = (long long)ch * kChunk, e = min(T, b + kChunk);
  double M[N][N], v[N];
#pragma unroll
  for (int r = 0; r < N; ++r) {
    v[r] = 0.0;
#pragma unroll
    for (int q = 0; q < N; ++q) M[r][q] = r == q ? 1.0 : 0.0;
  }
  for (long long t = b; t < e; ++t) {
    const double* At = A + (size_t)t * N * N;
    double nv[N], nM[N][N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = c[(size_t)t * N + r];
#pragma unroll
      for (int q = 0; q < N; ++q) acc += At[r * N + q] * v[q];
      nv[r] = acc;
#pragma unroll
      for (int q = 0; q < N; ++q) {
        double m = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) m += At[r * N + k] * M[k][q];
        nM[r][q] = m;
      }
    }
#pragma unroll
    for (int r = 0; r < N; ++r) {
      v[r] = nv[r];
#pragma unroll
      for (int q = 0; q < N; ++q) M[r][q] = nM[r][q];
    }
  }
#pragma unroll
  for (int r = 0; r < N; ++r) {
    vout[(size_t)ch * N + r] = v[r];
#pragma unroll
    for (int q = 0; q < N; ++q) Mout[((size_t)ch * N + r) * N + q] = M[r][q];
  }
}

// (2) chunk-start states S_0 = 0, S_{c+1} = M_c S_c + v_c (one thread)
template <int N>
__global__ void k_chunk_chain(const double* __restrict__ M, const double* __restrict__ v, int nchunks,
                              double* __restrict__ S) {
  double s[N];
#pragma unroll
  for (int r = 0; r < N; ++r) s[r] = 0.0;
  for (int ch = 0; ch < nchunks; ++ch) {
#pragma unroll
    for (int r = 0; r < N; ++r) S[(size_t)ch * N + r] = s[r];
    double ns[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = v[(size_t)ch * N + r];
#pragma unroll
      for (int q = 0; q < N; ++q) acc += M[((size_t)ch * N + r) * N + q] * s[q];
      ns[r] = acc;
    }
#pragma unroll
    for (int r = 0; r < N; ++r) s[r] = ns[r];
  }
}

// (3) rollout of every chunk from its start state: states[t+1] = A_t s_t + c_t
// (A == nullptr: the zero dynamics of state_coupling = 0, states[t+1] = c_t)
template <int N>
__global__ void k_chunk_rollout(const double* __restrict__ A, const double* __restrict__ c, long long T, int nchunks,
                                const double* __restrict__ S, double* __restrict__ states) {
  const int ch = blockIdx.x * blockDim.x + threadIdx.x;
  if (ch == 0) {
#pragma unroll
    for (int r = 0; r < N; ++r) states[r] = 0.0;
  }
  if (ch >= nchunks) return;
  const long long b = (long long)ch * kChunk, e = min(T, b + kChunk);
  double s[N];
#pragma unroll
  for (int r = 0; r < N; ++r) s[r] = A ? S[(size_t)ch * N + r] : 0.0;
  for (long long t = b; t < e; ++t) {
    double ns[N];
#pragma unroll
    for (int r = 0; r < N; ++r) {
      double acc = c[(size_t)t * N + r];
      if (A) {
        const double* At = A + (size_t)t * N * N;
#pragma unroll
        for (int q = 0; q < N; ++q) acc += At[r * N + q] * s[q];
      }
      ns[r] = acc;
      states[(size_t)(t + 1) * N + r] = acc;
    }
#pragma unroll
    for (int r = 0; r < N; ++r) s[r] = ns[r];
  }
}

// GainPolicy::evaluate at every step: a_t = G s_t (linear.hpp:112-126)
template <int N>
__global__ void k_policy(const double* __restrict__ G, const double* __restrict__ states, int P, long long T,
                         double* __restrict__ a) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    for (int r = 0; r < P; ++r) {
      double acc = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) acc += G[(size_t)r * N + q] * states[(size_t)t * N + q];
      a[(size_t)t * P + r] = acc;
    }
  }
}

// per-block partial sums of sum_t ||x[t+1] - y[t+1]|| (y == nullptr: ||x[t+1]||)
template <int N>
__global__ void k_gap_partial(const double* __restrict__ x, const double* __restrict__ y, long long T,
                              double* __restrict__ part) {
  __shared__ double sh[256];
  double acc = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    double d2 = 0.0;
#pragma unroll
    for (int r = 0; r < N; ++r) {
      const double d = x[(size_t)(t + 1) * N + r] - (y ? y[(size_t)(t + 1) * N + r] : 0.0);
      d2 += d * d;
    }
    acc += sqrt(d2);
  }
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int off = blockDim.x / 2; off > 0; off >>= 1) {
    if ((int)threadIdx.x < off) sh[threadIdx.x] += sh[threadIdx.x + off];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}
__global__ void k_sum(const double* __restrict__ part, int n, double* __restrict__ out) {
  double acc = 0.0;
  for (int i = 0; i < n; ++i) acc += part[i];
  *out = acc;
}

template <int N>
struct Runner {
  int P;
  long long T;
  cudaStream_t s;
  int nchunks, grid;
  Runner(int P_, long long T_, cudaStream_t s_) : P(P_), T(T_), s(s_) {
    nchunks = (int)((T + kChunk - 1) / kChunk);
    grid = (int)std::min<long long>(1184, std::max<long long>(1, (T + 255) / 256));
  }
  // states = rollout of the drive c under the dynamics Adyn (nullptr = zero dynamics)
  void rollout(const double* Adyn, const double* c, double* states, double* M, double* v, double* S) {
    if (nchunks == 0) {  // empty horizon: the initial state only
      LCK(cudaMemsetAsync(states, 0, sizeof(double) * N, s));
      return;
    }
    if (Adyn) {
      k_chunk_maps<N><<<(nchunks + 127) / 128, 128, 0, s>>>(Adyn, c, T, nchunks, M, v);
      k_chunk_chain<N><<<1, 1, 0, s>>>(M, v, nchunks, S);
    }
    k_chunk_rollout<N><<<(nchunks + 127) / 128, 128, 0, s>>>(Adyn, c, T, nchunks, S, states);
  }
  double gap(const double* x, const double* y, double* part, double* out) {
    k_gap_partial<N><<<grid, 256, 0, s>>>(x, y, T, part);
    k_sum<<<1, 1, 0, s>>>(part, grid, out);
    double h = 0.0;
    LCK(cudaMemcpyAsync(&h, out, sizeof h, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    return h;
  }
};

template <int N>
static void curve_impl(const pcd_linear_spec* sp, const double* init, double tol, int64_t max_it, int norm,
                       double* curve, int64_t cap, int64_t* len, double* final_cache, double* elapsed_ms) {
  const int P = sp->input_dim;
  const long long T = sp->horizon;
  cudaStream_t s;
  LCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  const size_t TN = (size_t)T * N, TP = (size_t)T * P;
  Buf A(TN * N), B(TN * P), w(TN), G((size_t)P * N), Ac(TN * N), c(TN), cache(std::max<size_t>(TP, 1)),
      ref((TN + N)), draft(TN + N), st(TN + N);
  Runner<N> R(P, T, s);
  Buf M((size_t)R.nchunks * N * N + 1), v((size_t)R.nchunks * N + 1), S((size_t)R.nchunks * N + 1),
      part((size_t)R.grid + 1), out(1);
  bool zeroA = true;
  for (size_t i = 0; i < TN * N && zeroA; ++i) zeroA = sp->dynamics[i] == 0.0;
  LCK(cudaMemcpyAsync(A.p, sp->dynamics, TN * N * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(B.p, sp->input, TN * P * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(w.p, sp->disturbances, TN * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(G.p, sp->gain, (size_t)P * N * 8, cudaMemcpyHostToDevice, s));
  if (init) LCK(cudaMemcpyAsync(cache.p, init, TP * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaStreamSynchronize(s));
  const auto t0 = std::chrono::steady_clock::now();
  // reference: the closed-loop (sequential) trajectory
  k_closed_loop<N><<<R.grid, 256, 0, s>>>(A.p, B.p, G.p, P, T, Ac.p);
  k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, nullptr, P, T, c.p);
  R.rollout(Ac.p, c.p, ref.p, M.p, v.p, S.p);
  // draft: rollout of the initial cache (zero actions when absent)
  k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, init ? cache.p : nullptr, P, T, c.p);
  R.rollout(zeroA ? nullptr : A.p, c.p, draft.p, M.p, v.p, S.p);
  const double denom = norm ? R.gap(ref.p, draft.p, part.p, out.p) : R.gap(ref.p, nullptr, part.p, out.p);
  const int64_t capit = max_it > 0 ? max_it : T;
  const double* cur = draft.p;
  int64_t k = 0;
  for (; k < capit; ++k) {
    if (!(denom > 0.0))  // relative_rmse (linear.cpp:236-262)
      throw ContractViolation(norm ? "relative rmse: baseline equals the reference"
                                   : "relative rmse: reference trajectory is zero");
    // one Picard iteration with single-step processes: cache = G s(cache)
    k_policy<N><<<R.grid, 256, 0, s>>>(G.p, cur, P, T, cache.p);
    k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, cache.p, P, T, c.p);
    R.rollout(zeroA ? nullptr : A.p, c.p, st.p, M.p, v.p, S.p);
    cur = st.p;
    const double r = R.gap(ref.p, st.p, part.p, out.p) / denom;
    if (k < cap) curve[k] = r;
    if (r <= tol) {
      ++k;
      break;
    }
  }
  *len = k;
  LCK(cudaGetLastError());
  if (elapsed_ms)
    *elapsed_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (final_cache && T) LCK(cudaMemcpyAsync(final_cache, cache.p, TP * 8, cudaMemcpyDeviceToHost, s));
  LCK(cudaStreamSynchronize(s));
}


// ---------------------------------------------------------------------------
// MLP feedback policy (BASELINE config 4): a_t = forward(s_t)
// with the reference's MlpParams (mlp.cpp:141-169) in place of GainPolicy.
constexpr int kMlpMaxH = 64;
constexpr int kMlpMaxP = 16;
constexpr int kMlpBlock = 128;

static int host_tanh_fma_lin() {
#if defined(__x86_64__)
  __builtin_cpu_init();
  return (__builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2")) ? 1 : 0;
#else
  return 1;
#endif
}

// Every state's action, one thread per state, in MlpParams::forward's exact
// operation order (acc = b; acc += w * x with explicit round-to-nearest
// multiply and add, glibc tanh restated): each action is bit-identical to the
// reference's forward() of the same state. The weights sit in shared memory
// (w1 | b1 | w2 | b2 | w3 | b3, MlpParams layout), the first hidden layer in
// a [unit][thread] shared array; the second layer is streamed unit by unit
// into the output accumulators, which keeps layer 3's order (c ascending).
template <int N>
__global__ void __launch_bounds__(kMlpBlock) k_mlp_policy(const double* __restrict__ Wg, int H, int P, int tfma,
                                                          const double* __restrict__ states, long long T,
                                                          double* __restrict__ a) {
  extern __shared__ __align__(16) double lsm[];
  const int nw = H * N + H + H * H + H + P * H + P;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) lsm[i] = Wg[i];
  __syncthreads();
  const double *w1 = lsm, *b1 = w1 + H * N, *w2 = b1 + H, *b2 = w2 + H * H, *w3 = b2 + H, *b3 = w3 + P * H;
  double* h1 = lsm + nw + threadIdx.x;  // h1[c] at h1[c * kMlpBlock]
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    double x[N];
#pragma unroll
    for (int c = 0; c < N; ++c) x[c] = states[(size_t)t * N + c];
    for (int r = 0; r < H; ++r) {
      double acc = b1[r];
#pragma unroll
      for (int c = 0; c < N; ++c) acc = __dadd_rn(acc, __dmul_rn(w1[r * N + c], x[c]));
      h1[r * kMlpBlock] = gt_tanh(acc, tfma);
    }
    double out[kMlpMaxP];
#pragma unroll
    for (int k = 0; k < kMlpMaxP; ++k) out[k] = k < P ? b3[k] : 0.0;
    for (int r = 0; r < H; ++r) {
      double acc = b2[r];
      const double* row = w2 + r * H;
      for (int c = 0; c < H; ++c) acc = __dadd_rn(acc, __dmul_rn(row[c], h1[c * kMlpBlock]));
      const double h2 = gt_tanh(acc, tfma);
#pragma unroll
      for (int k = 0; k < kMlpMaxP; ++k)
        if (k < P) out[k] = __dadd_rn(out[k], __dmul_rn(w3[k * H + r], h2));
    }
#pragma unroll
    for (int k = 0; k < kMlpMaxP; ++k)
      if (k < P) a[(size_t)t * P + k] = out[k];
  }
}

// LinearEnv::actions_equal (linear.hpp:64-71) over the whole cache: out[0] +=
// slots that differ beyond 1e-9 relative, out[1] = max relative change (as
// ordered bits of a non-negative double)
__global__ void k_action_change(const double* __restrict__ x, const double* __restrict__ y, int P, long long T,
                                unsigned long long* out) {
  __shared__ unsigned long long sc[8], sm[8];
  unsigned long long cnt = 0, mx = 0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    bool diff = false;
    for (int k = 0; k < P; ++k) {
      const double u = x[(size_t)t * P + k], v = y[(size_t)t * P + k];
      const double scale = fmax(1.0, fmax(fabs(u), fabs(v)));
      const double d = fabs(u - v);
      diff |= d > 1e-9 * scale;
      const double rel = d / scale;
      const unsigned long long b = (unsigned long long)__double_as_longlong(rel == rel ? rel : INFINITY);
      mx = b > mx ? b : mx;
    }
    cnt += diff ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    const unsigned long long m2 = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = m2 > mx ? m2 : mx;
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sc[w] = cnt; sm[w] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long c2 = 0, m3 = 0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { c2 += sc[i]; m3 = sm[i] > m3 ? sm[i] : m3; }
    if (c2) atomicAdd(out, c2);
    atomicMax(out + 1, m3);
  }
}

template <int N>
static void mlp_curve_impl(const pcd_linear_spec* sp, const pcd_linear_mlp* pol, const double* init, double tol,
                           int64_t max_it, int norm, double* curve, int64_t cap, pcd_linear_mlp_result* res,
                           double* final_cache, double* ref_states) {
  const int P = sp->input_dim, H = pol->hidden;
  const long long T = sp->horizon;
  cudaStream_t s;
  LCK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamDestroy(s); }
  } sg{s};
  const size_t TN = (size_t)T * N, TP = (size_t)T * P;
  Buf A(TN * N), B(TN * P), w(TN), c(TN), c0(std::max<size_t>(TP, 1)), ca(std::max<size_t>(TP, 1)),
      cb(std::max<size_t>(TP, 1)), ref(TN + N), draft(TN + N), st(TN + N);
  Runner<N> R(P, T, s);
  Buf M((size_t)R.nchunks * N * N + 1), v((size_t)R.nchunks * N + 1), S((size_t)R.nchunks * N + 1),
      part((size_t)R.grid + 1), out(1);
  // weights, MlpParams layout
  const size_t nw = (size_t)H * N + H + (size_t)H * H + H + (size_t)P * H + P;
  std::vector<double> hw;
  hw.reserve(nw);
  hw.insert(hw.end(), pol->w1, pol->w1 + (size_t)H * N);
  hw.insert(hw.end(), pol->b1, pol->b1 + H);
  hw.insert(hw.end(), pol->w2, pol->w2 + (size_t)H * H);
  hw.insert(hw.end(), pol->b2, pol->b2 + H);
  hw.insert(hw.end(), pol->w3, pol->w3 + (size_t)P * H);
  hw.insert(hw.end(), pol->b3, pol->b3 + P);
  Buf W(nw);
  unsigned long long* chg = nullptr;
  LCK(cudaMalloc(&chg, 2 * sizeof(unsigned long long)));
  struct ChgGuard {
    unsigned long long* p;
    ~ChgGuard() { cudaFree(p); }
  } cg{chg};
  bool zeroA = true;
  for (size_t i = 0; i < TN * N && zeroA; ++i) zeroA = sp->dynamics[i] == 0.0;
  LCK(cudaMemcpyAsync(A.p, sp->dynamics, TN * N * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(B.p, sp->input, TN * P * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(w.p, sp->disturbances, TN * 8, cudaMemcpyHostToDevice, s));
  LCK(cudaMemcpyAsync(W.p, hw.data(), nw * 8, cudaMemcpyHostToDevice, s));
  if (init) LCK(cudaMemcpyAsync(c0.p, init, TP * 8, cudaMemcpyHostToDevice, s));
  else if (TP) LCK(cudaMemsetAsync(c0.p, 0, TP * 8, s));
  const size_t smem = (nw + (size_t)kMlpMaxH * kMlpBlock) * sizeof(double);
  LCK(cudaFuncSetAttribute(k_mlp_policy<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int tfma = host_tanh_fma_lin();
  const int pgrid = (int)std::min<long long>(148 * 8, std::max<long long>(1, (T + kMlpBlock - 1) / kMlpBlock));
  LCK(cudaStreamSynchronize(s));
  // one Picard iteration with single-step processes: dst = pi(rollout(src)); the rollout is left in st
  auto iterate = [&](const double* src, double* dst) {
    k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, src, P, T, c.p);
    R.rollout(zeroA ? nullptr : A.p, c.p, st.p, M.p, v.p, S.p);
    k_mlp_policy<N><<<pgrid, kMlpBlock, smem, s>>>(W.p, H, P, tfma, st.p, T, dst);
  };
  auto change = [&](const double* x, const double* y, unsigned long long* cnt, double* rel) {
    LCK(cudaMemsetAsync(chg, 0, 2 * sizeof(unsigned long long), s));
    k_action_change<<<R.grid, 256, 0, s>>>(x, y, P, T, chg);
    unsigned long long hcg[2];
    LCK(cudaMemcpyAsync(hcg, chg, sizeof hcg, cudaMemcpyDeviceToHost, s));
    LCK(cudaStreamSynchronize(s));
    *cnt = hcg[0];
    double r;
    std::memcpy(&r, &hcg[1], sizeof r);
    *rel = r;
  };
  // pass 1: the sequential trajectory as the Picard fixed point (Prop. 1);
  // also picard_simulate's iterations_to_converged for the single-step plan
  const int64_t hard_cap = 2 * (int64_t)T + 4;  // picard_simulate's safety cap (engine.hpp:485-490)
  const auto t0 = std::chrono::steady_clock::now();
  double* cur = ca.p;
  double* nxt = cb.p;
  LCK(cudaMemcpyAsync(cur, c0.p, std::max<size_t>(TP, 1) * 8, cudaMemcpyDeviceToDevice, s));
  int64_t k = 0, conv = 0;
  double best = INFINITY;
  int stall = 0;
  while (T > 0) {
    if (k >= hard_cap)
      throw IterationLimit("picard iteration cap exceeded (" + std::to_string(hard_cap) +
                           "); the policy may be nondeterministic", k, {});
    iterate(cur, nxt);
    ++k;
    unsigned long long cnt;
    double rel;
    change(cur, nxt, &cnt, &rel);
    std::swap(cur, nxt);
    if (!(rel == rel)) throw ContractViolation("linear mlp policy: non-finite action");
    if (!conv && cnt == 0) conv = k;
    // the fixed point in floating point: no change beyond 2^-46 relative, or
    // the change stopped shrinking once below 1e-12 (last-ulp oscillation)
    if (rel <= 0x1p-46) break;
    if (rel <= 1e-12) {
      stall = rel < best ? 0 : stall + 1;
      if (stall >= 3) break;
    }
    best = std::min(best, rel);
    if (conv && k > conv + 200 && rel <= 1e-9) break;
  }
  if (T > 0) {
    // the reference trajectory is the rollout of the fixed-point cache
    k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, cur, P, T, c.p);
    R.rollout(zeroA ? nullptr : A.p, c.p, ref.p, M.p, v.p, S.p);
  } else {
    LCK(cudaMemsetAsync(ref.p, 0, sizeof(double) * N, s));
  }
  LCK(cudaStreamSynchronize(s));
  const auto t1 = std::chrono::steady_clock::now();
  res->iterations_to_converged = conv;
  res->fixed_point_iterations = k;
  res->fixed_point_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  // pass 2: the curve (linear.cpp:279-318): same iterates, scored against ref
  k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, init ? c0.p : nullptr, P, T, c.p);
  R.rollout(zeroA ? nullptr : A.p, c.p, draft.p, M.p, v.p, S.p);
  const double denom = norm ? R.gap(ref.p, draft.p, part.p, out.p) : R.gap(ref.p, nullptr, part.p, out.p);
  const int64_t capit = max_it > 0 ? max_it : T;
  cur = ca.p;
  nxt = cb.p;
  LCK(cudaMemcpyAsync(cur, c0.p, std::max<size_t>(TP, 1) * 8, cudaMemcpyDeviceToDevice, s));
  int64_t n = 0;
  for (; n < capit; ++n) {
    if (!(denom > 0.0))  // relative_rmse (linear.cpp:236-262)
      throw ContractViolation(norm ? "relative rmse: baseline equals the reference"
                                   : "relative rmse: reference trajectory is zero");
    iterate(cur, nxt);
    std::swap(cur, nxt);
    k_drive<N><<<R.grid, 256, 0, s>>>(B.p, w.p, cur, P, T, c.p);
    R.rollout(zeroA ? nullptr : A.p, c.p, st.p, M.p, v.p, S.p);
    const double r = R.gap(ref.p, st.p, part.p, out.p) / denom;
    if (n < cap) curve[n] = r;
    if (r <= tol) {
      ++n;
      break;
    }
  }
  LCK(cudaGetLastError());
  res->curve_len = n;
  res->curve_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t1).count();
  if (final_cache && T) LCK(cudaMemcpyAsync(final_cache, cur, TP * 8, cudaMemcpyDeviceToHost, s));
  if (ref_states) LCK(cudaMemcpyAsync(ref_states, ref.p, (TN + N) * 8, cudaMemcpyDeviceToHost, s));
  LCK(cudaStreamSynchronize(s));
}
}  // namespace lin
}  // namespace pcd

namespace pcd {
int translate_exception();  // capi.cpp: exception -> status code (same mapping as the FO engine)
}

extern "C" int pcd_linear_convergence_curve(const pcd_linear_spec* spec, const double* initial_cache,
                                            double tolerance, int64_t max_iterations, int32_t normalization,
                                            int32_t device, double* curve, int64_t curve_cap, int64_t* curve_len,
                                            double* final_cache, double* elapsed_ms) {
  try {
    if (!spec || !curve_len) throw pcd::InvalidArgument("null argument");
    if (spec->state_dim < 1 || spec->input_dim < 1 || spec->horizon < 0)
      throw pcd::ContractViolation("linear spec: dimensions must be positive");
    if (spec->state_dim > 8 || spec->input_dim > 64)
      throw pcd::InvalidArgument("linear spec: state_dim <= 8 and input_dim <= 64 on the device");
    if (spec->horizon > 0 && (!spec->dynamics || !spec->input || !spec->disturbances || !spec->gain))
      throw pcd::InvalidArgument("linear spec arrays missing");
    if (curve_cap > 0 && !curve) throw pcd::InvalidArgument("curve buffer missing");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw pcd::CudaError("no CUDA device available: the B200 engine has no CPU fallback");
    }
    if (device < 0 || device >= ndev) throw pcd::InvalidArgument("device index out of range");
    if (cudaSetDevice(device) != cudaSuccess) throw pcd::CudaError("cudaSetDevice failed");
    *curve_len = 0;
    using namespace pcd::lin;
    switch (spec->state_dim) {
#define PCD_LIN_CASE(n) \
  case n: curve_impl<n>(spec, initial_cache, tolerance, max_iterations, normalization, curve, curve_cap, curve_len, final_cache, elapsed_ms); break;
      PCD_LIN_CASE(1) PCD_LIN_CASE(2) PCD_LIN_CASE(3) PCD_LIN_CASE(4)
      PCD_LIN_CASE(5) PCD_LIN_CASE(6) PCD_LIN_CASE(7) PCD_LIN_CASE(8)
#undef PCD_LIN_CASE
    }
    return PCD_OK;
  } catch (...) {
    return pcd::translate_exception();
  }
}

extern "C" int pcd_linear_mlp_convergence_curve(const pcd_linear_spec* spec, const pcd_linear_mlp* policy,
                                                const double* initial_cache, double tolerance,
                                                int64_t max_iterations, int32_t normalization, int32_t device,
                                                double* curve, int64_t curve_cap, pcd_linear_mlp_result* result,
                                                double* final_cache, double* reference_states) {
  try {
    if (!spec || !policy || !result) throw pcd::InvalidArgument("null argument");
    *result = pcd_linear_mlp_result{};
    if (spec->state_dim < 1 || spec->input_dim < 1 || spec->horizon < 0)
      throw pcd::ContractViolation("linear spec: dimensions must be positive");
    if (spec->state_dim > 8 || spec->input_dim > pcd::lin::kMlpMaxP)
      throw pcd::InvalidArgument("linear mlp policy: state_dim <= 8 and input_dim <= 16 on the device");
    if (policy->hidden < 1 || policy->hidden > pcd::lin::kMlpMaxH)
      throw pcd::InvalidArgument("linear mlp policy: hidden width must be in [1, 64]");
    if (!policy->w1 || !policy->b1 || !policy->w2 || !policy->b2 || !policy->w3 || !policy->b3)
      throw pcd::InvalidArgument("linear mlp policy: weight arrays missing");
    if (spec->horizon > 0 && (!spec->dynamics || !spec->input || !spec->disturbances))
      throw pcd::InvalidArgument("linear spec arrays missing");
    if (curve_cap > 0 && !curve) throw pcd::InvalidArgument("curve buffer missing");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw pcd::CudaError("no CUDA device available: the B200 engine has no CPU fallback");
    }
    if (device < 0 || device >= ndev) throw pcd::InvalidArgument("device index out of range");
    if (cudaSetDevice(device) != cudaSuccess) throw pcd::CudaError("cudaSetDevice failed");
    using namespace pcd::lin;
    switch (spec->state_dim) {
#define PCD_LIN_CASE(n) \
  case n: mlp_curve_impl<n>(spec, policy, initial_cache, tolerance, max_iterations, normalization, curve, curve_cap, result, final_cache, reference_states); break;
      PCD_LIN_CASE(1) PCD_LIN_CASE(2) PCD_LIN_CASE(3) PCD_LIN_CASE(4)
      PCD_LIN_CASE(5) PCD_LIN_CASE(6) PCD_LIN_CASE(7) PCD_LIN_CASE(8)
#undef PCD_LIN_CASE
    }
    return PCD_OK;
  } catch (...) {
    return pcd::translate_exception();
  }
}
