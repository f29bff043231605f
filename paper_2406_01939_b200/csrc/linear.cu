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
#include <string>
#include <vector>

#include "capi_internal.h"

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
