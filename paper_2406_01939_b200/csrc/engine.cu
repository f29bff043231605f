// engine.cu — B200-native Picard fixed-point engine behind the C ABI.
//
// Host driver mirroring picard::picard_simulate (engine.hpp:458-590) and
// picard_iterate_once (engine.hpp:358-444); every per-iteration computation
// (sweeps, publish, counters, checkpoint advance) runs in the kernels of
// kernels.cuh on the device. Only the per-iteration scalar block (a few
// dozen bytes) crosses PCIe inside the loop.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <map>
#include <mutex>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <cuda_fp16.h>

#include "capi_internal.h"
#include "general.cuh"
#include "kernels.cuh"
#include "tc_common.cuh"

namespace pcd {

cudaError_t launch_tc_pp(const TcArgs& a, const CUtensorMap& wmap, int ntiles, cudaStream_t stream);
cudaError_t launch_spec_verify(const SweepArgs& S, const int* q, const int* qn, int cap, int force_bad,
                               cudaStream_t stream);  // tc_spec.cu  // tc_pp.cu (two 64-row halves)
cudaError_t launch_tc_inc(const IncArgs& a, const CUtensorMap& gmap, int ntiles, cudaStream_t stream);  // tc_inc.cu
cudaError_t launch_inc_prep(const IncPrep& p, cudaStream_t stream);  // tc_inc.cu: G rows + node transitions
int tc_pp_width_class(int J);  // tc_pp.cu: layer-3 width class of the ping-pong sweep for J nodes
size_t tc_smem_bytes();

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw CudaError(std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #x);   \
  } while (0)

// Process-wide caching allocator (per device): one-shot API calls create and
// destroy a handle each time; recycling the device blocks (~1.5 GB at C3)
// keeps cudaMalloc / cudaFree (and their implicit device syncs) out of the
// end-to-end path. Blocks are only returned here when no work of their
// stream is pending (handles sync before destroy; growth syncs the device).
struct DevicePool {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void*> free;
  void* get(size_t bytes, size_t* got) {
    bytes = (bytes + 511) & ~(size_t)511;
    int dev = 0;
    cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu);
      auto it = free.lower_bound({dev, bytes});
      if (it != free.end() && it->first.first == dev && it->first.second <= 2 * bytes + (1 << 20)) {
        void* p = it->second;
        *got = it->first.second;
        free.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e != cudaSuccess) {  // release the cache and retry once
      cudaGetLastError();
      trim(dev);
      CK(cudaMalloc(&p, bytes));
    }
    *got = bytes;
    return p;
  }
  void put(void* p, size_t bytes) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    free.insert({{dev, bytes}, p});
  }
  void trim(int dev) {
    std::lock_guard<std::mutex> lk(mu);
    for (auto it = free.begin(); it != free.end();) {
      if (it->first.first == dev) {
        cudaFree(it->second);
        it = free.erase(it);
      } else {
        ++it;
      }
    }
  }
};
static DevicePool g_pool;

template <typename T>
struct DBuf {
  T* p = nullptr;
  size_t n = 0;       // elements requested
  size_t bytes = 0;   // block size
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  ~DBuf() { release(); }
  void release() {
    if (p) g_pool.put(p, bytes);
    p = nullptr;
    n = 0;
    bytes = 0;
  }
  void alloc(size_t count) {
    if (count <= n && p) return;
    if (p) {  // growth: the old block may still be read by queued work
      cudaDeviceSynchronize();
      release();
    }
    if (count == 0) return;
    p = (T*)g_pool.get(count * sizeof(T), &bytes);
    n = count;
  }
  void swap(DBuf& o) {
    std::swap(p, o.p);
    std::swap(n, o.n);
    std::swap(bytes, o.bytes);
  }
  void upload(const T* h, size_t count, cudaStream_t s) {
    alloc(count);
    if (count) CK(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, s));
  }
};

// --------------------------------------------------------------- NCCL (dlopen)
// Minimal NCCL surface, loaded lazily so single-GPU use never needs libnccl.
typedef struct { char internal[128]; } nccl_unique_id;
typedef void* nccl_comm;
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(nccl_unique_id*) = nullptr;
  int (*CommInitRank)(nccl_comm*, int, nccl_unique_id, int) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, nccl_comm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, nccl_comm, cudaStream_t) = nullptr;
  int (*CommDestroy)(nccl_comm) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  bool load() {
    if (lib) return true;
    for (const char* n : {"libnccl.so.2", "libnccl.so"}) {
      lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
      if (lib) break;
    }
    if (!lib) return false;
    GetUniqueId = (decltype(GetUniqueId))dlsym(lib, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(lib, "ncclCommInitRank");
    AllGather = (decltype(AllGather))dlsym(lib, "ncclAllGather");
    AllReduce = (decltype(AllReduce))dlsym(lib, "ncclAllReduce");
    CommDestroy = (decltype(CommDestroy))dlsym(lib, "ncclCommDestroy");
    GetErrorString = (decltype(GetErrorString))dlsym(lib, "ncclGetErrorString");
    return GetUniqueId && CommInitRank && AllGather && AllReduce && CommDestroy;
  }
};
static NcclApi g_nccl;
enum { ncclInt32 = 2, ncclInt64 = 4, ncclUint64 = 5, ncclSum = 0, ncclMax = 2, ncclMin = 3 };

// The communicator of one rank: an all-gather of int32
// cache slices and integer all-reduces of the convergence scalars. NCCL over
// NVLink / NVSwitch between processes (one per GPU), or an in-process
// loopback group: N handles on one device, each driven by its own host
// thread — the test harness that runs the multi-rank code path (exchange,
// pack / unpack, per-rank process masks, shards) on a single GPU, where NCCL
// refuses duplicate devices.
enum class RedOp { SumI64, MinU64, MaxU64 };
struct Comm {
  virtual ~Comm() = default;
  virtual void all_gather(const int* send, int* recv, size_t count, cudaStream_t s) = 0;
  virtual void all_reduce(long long* buf, size_t count, RedOp op, cudaStream_t s) = 0;
};

struct NcclComm final : Comm {
  nccl_comm c = nullptr;
  ~NcclComm() override {
    if (c && g_nccl.CommDestroy) g_nccl.CommDestroy(c);
  }
  static void check(int rc, const char* what) {
    if (rc) throw CudaError(std::string(what) + ": " + (g_nccl.GetErrorString ? g_nccl.GetErrorString(rc) : "?"));
  }
  void all_gather(const int* send, int* recv, size_t count, cudaStream_t s) override {
    check(g_nccl.AllGather(send, recv, count, ncclInt32, c, s), "ncclAllGather");
  }
  void all_reduce(long long* buf, size_t count, RedOp op, cudaStream_t s) override {
    const int dt = op == RedOp::SumI64 ? ncclInt64 : ncclUint64;
    const int o = op == RedOp::SumI64 ? ncclSum : op == RedOp::MinU64 ? ncclMin : ncclMax;
    check(g_nccl.AllReduce(buf, buf, count, dt, o, c, s), "ncclAllReduce");
  }
};

struct LoopbackGroup {
  static constexpr size_t kMaxReduce = 64;
  int n = 1;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long long gen = 0;
  int* staging = nullptr;  // device
  size_t staging_cap = 0;  // ints
  std::vector<long long> host;  // n x kMaxReduce
  explicit LoopbackGroup(int nr) : n(nr), host((size_t)nr * kMaxReduce) {}
  ~LoopbackGroup() {
    if (staging) cudaFree(staging);
  }
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long long g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return gen != g; }))
      throw CudaError("loopback group: a rank did not reach the collective (timeout)");
  }
};

struct LoopbackComm final : Comm {
  std::shared_ptr<LoopbackGroup> g;
  int rank = 0;
  void all_gather(const int* send, int* recv, size_t count, cudaStream_t s) override {
    CK(cudaStreamSynchronize(s));  // this rank's send slice is complete
    g->barrier();
    if (rank == 0 && g->staging_cap < count * g->n) {
      if (g->staging) CK(cudaFree(g->staging));
      g->staging = nullptr;
      CK(cudaMalloc(&g->staging, sizeof(int) * count * g->n));
      g->staging_cap = count * g->n;
    }
    g->barrier();
    if (count) {
      CK(cudaMemcpyAsync(g->staging + (size_t)rank * count, send, sizeof(int) * count, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
    }
    g->barrier();
    if (count) {
      CK(cudaMemcpyAsync(recv, g->staging, sizeof(int) * count * g->n, cudaMemcpyDeviceToDevice, s));
      CK(cudaStreamSynchronize(s));
    }
    g->barrier();  // nobody refills the staging buffer before every rank has read it
  }
  void all_reduce(long long* buf, size_t count, RedOp op, cudaStream_t s) override {
    if (count > LoopbackGroup::kMaxReduce) throw InvalidArgument("loopback reduce too large");
    long long mine[LoopbackGroup::kMaxReduce];
    CK(cudaMemcpyAsync(mine, buf, sizeof(long long) * count, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::copy(mine, mine + count, g->host.begin() + (size_t)rank * LoopbackGroup::kMaxReduce);
    g->barrier();
    for (size_t i = 0; i < count; ++i) {
      long long v = g->host[i];
      for (int r = 1; r < g->n; ++r) {
        const long long w = g->host[(size_t)r * LoopbackGroup::kMaxReduce + i];
        if (op == RedOp::SumI64) v += w;
        else if (op == RedOp::MinU64) v = (long long)std::min((unsigned long long)v, (unsigned long long)w);
        else v = (long long)std::max((unsigned long long)v, (unsigned long long)w);
      }
      mine[i] = v;
    }
    g->barrier();  // every rank has read the inputs
    CK(cudaMemcpyAsync(buf, mine, sizeof(long long) * count, cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
  }
};

}  // namespace pcd

struct pcd_handle {
  int device = 0;
  cudaStream_t stream = nullptr;
  int32_t J = 0, I = 0;
  int64_t T = 0, R = 0;
  int tanh_fma = 1;
  // instance
  pcd::DBuf<int> product, order_t, rrow, cap0, inv0;
  pcd::DBuf<double> rtab;
  // policy
  int kind = 0, H = 64;
  double gamma = 0.0;
  int64_t p_horizon = 0;
  pcd::DBuf<double> w1t, b1, w2t, b2, w3t, b3, w3s;
  double fast_margin = 0.0;  // see fast_margin_bound
  int nocache = 0;           // Time Warp windows (pcd_time_warp)
  pcd::DBuf<int> pcap0, pinv0;
  // plan
  int32_t M = 0;
  bool have_plan = false, is_product = false;
  pcd::DBuf<int> owner, pstart, pslots, qstart, qslots;
  pcd::DBuf<int> rid;     // run of every slot (run partitions)
  int64_t runs = 0;       // R
  // per-iteration work list of the tensor-core sweep (window load desc)
  pcd::DBuf<int> wload, wids, wload_s, wq, wctl, wbeg;  // wctl = {nq, head}; wbeg: first window position
  pcd::DBuf<unsigned char> wtmp;
  // dynamic state
  pcd::DBuf<int> cache, ref, fresh, ev, ckcap, ckinv, ckbak, xloc, hck, seg, segtot, scratch, tau;
  int adv_buf = -1;                      // 0: the last checkpoint advance is not yet checked (deferred), -1 none
  struct TimedPhase { cudaEvent_t a, b; double* acc; };
  std::vector<cudaEvent_t> evpool;       // phase-timer events (flush_timers), reused
  size_t evnext = 0;
  std::vector<TimedPhase> tlog;          // recorded, not yet resolved phases
  bool defer_timers = false;
  int64_t adv_from = 0, adv_to = 0;
  pcd::DBuf<unsigned char> written;
  pcd::DBuf<long long> evals;
  // general closed form (general.cuh): same-product chains of the plan,
  // per-iteration (product, node) entry lists, per-position actions, deltas
  bool gen_plan = false;
  pcd::DBuf<int> gprev, gkeys, gkeys_s, gvals, gslots, gstart, ocache, ofresh;
  pcd::DBuf<int4> gdl;
  pcd::DBuf<unsigned char> gtmp;
  pcd::Scalars* scal = nullptr;  // device
  pcd::Scalars* h_scal = nullptr;  // pinned host
  long long* d_errt = nullptr;
  pcd_timing timing{};
  bool resident_valid = false;
  int32_t* history = nullptr;  // host, pcd_set_history
  int64_t history_cap = 0;
  // tensor-core policy (tc_pp.cu)
  bool tc_ok = false;                    // dual policy with 2J+1 <= 208, hidden 64
  double tc_guard = 0.0;                 // derived guard 2B (1 + 2^-10), tc_error_bound
  double tc_bound = 0.0;                 // B: bound on |score_tc - score_ref|
  double tc_guard_abs = 0.0;             // B (1 + 2^-10): the |best| test
  pcd::DBuf<float> tc_gnode;             // per best node: [0, kTcN3) margin, [kTcN3, 2 kTcN3) |best| thresholds
  pcd::DBuf<int> spec_q, spec_n, cbak;   // speculation queue (tc_spec.cu) and the window's cache backup
  pcd::DBuf<unsigned char> wbak;         // ... and written flags backup
  int tc_n3 = 0;                         // layer-3 width class of the ping-pong image (prepare_tc)
  pcd::DBuf<unsigned char> tc_wimg2;
  pcd::DBuf<float> tc_b1, tc_b2, tc_ic0, tc_ix0, tc_rtq;
  int debug = 0;                         // pcd_set_debug flags
  pcd::DBuf<long long> tc_prof;          // PCD_DEBUG_TC_PROFILE: phase clocks of CTA 0
  pcd::DBuf<unsigned long long> tc_stats;
  int32_t tc_tiles = 0;
  int64_t max_load = 0;
  // incremental-layer-1 sweep (tc_inc.cu): layer-1 tables, per-iteration G rows
  bool inc_ok = false;                   // dual policy, J <= kIncMaxJ (prepare_tc)
  int32_t tc_kernel_req = 0;             // pcd_config::tc_kernel of the running simulate
  pcd::DBuf<float> inc_af, inc_wx, inc_wt, grow;
  pcd::DBuf<double> inc_a64, inc_b1;
  pcd::DBuf<int> inc_bA, inc_bD;
  CUtensorMap gmap{};                    // TMA map over grow ([rows][64] fp32, one-row boxes)
  CUtensorMap wmap{};                    // TMA map over tc_wimg2 (make_wmap)
  size_t gmap_rows = 0;
  // multi-GPU
  int32_t rank = 0, nranks = 1;
  std::unique_ptr<pcd::Comm> comm;  // NCCL, or a loopback group (tests)
  std::vector<int32_t> rank_of;
  std::vector<int32_t> h_roff, h_rslots;  // rank-major, time-ordered owned slots (host copy)
  int32_t maxn = 0;
  pcd::DBuf<unsigned char> d_mine;
  pcd::DBuf<int> d_roff, d_rslots, d_send, d_recv;
  pcd::DBuf<long long> d_red;

  pcd::DevModel model() const {
    pcd::DevModel m{};
    m.kind = kind; m.J = J; m.I = I; m.H = H; m.in = 2 * J + 1; m.out = 2 * J;
    m.gamma = gamma;
    m.w1t = w1t.p; m.b1 = b1.p; m.w2t = w2t.p; m.b2 = b2.p; m.w3t = w3t.p; m.b3 = b3.p;
    m.pcap0 = pcap0.p; m.pinv0 = pinv0.p; m.horizon = p_horizon; m.tanh_fma = tanh_fma;
    m.product = product.p; m.order_t = order_t.p; m.rrow = rrow.p; m.rtab = rtab.p;
    m.w3s = w3s.n ? w3s.p : nullptr;
    m.fast_margin = fast_margin;
    return m;
  }
  // auxiliary stream: the tensor-core sweep's work list and the speculation
  // backups are built on it while the cache kernels run on `stream`
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  bool wl_ready = false;  // the work list of the coming sweep is already built (build_worklist)
  // per-product window bounds carried across the iterations of simulate
  // (windows only move forward there; kernels.cuh product_window)
  pcd::DBuf<int2> qcur;
  bool qcur_on = false;
  // post-sweep verification of speculated decisions running on `aux` while
  // the host reads the iteration's scalars and launches the checkpoint
  // advance (simulate: finish_verify); it reads the checkpoint capacities
  // from a snapshot, as the advance may already be rewriting them
  bool verify_pending = false;
  cudaEvent_t ev_sweep = nullptr;
  pcd::DBuf<int> ckcap_v;
  // pipelined verification (simulate): the verification of iteration i runs
  // on `aux` beside iteration i+1's checkpoint advance and cache kernels,
  // which write the spare set of the per-iteration buffers the verification
  // reads (ev, hck, xloc; swapped after each speculated sweep) and back up
  // the next window into the spare backups; the host waits for the
  // verdict (h_vbad, ev_vdone) only before iteration i+1's sweep. The work
  // list and the backups then go on `aux2`, not behind the verification.
  pcd::DBuf<int> ev2, hck2, xloc2, cbak2;
  pcd::DBuf<unsigned char> wbak2;
  cudaStream_t aux2 = nullptr;
  cudaEvent_t ev_vdone = nullptr;
  int* h_vbad = nullptr;  // pinned: the verification's verdict
  bool pipe_verify = false;
  int64_t wl_hint = 0;       // busiest window load of the last iteration (build_worklist's sort width)
  bool nospec_once = false;  // the next iteration re-runs one whose speculation was rejected
  // pinned host destination of the actions (pcd_simulate): the committed
  // prefix streams out on `aux` while later iterations run
  int32_t* dl_out = nullptr;
  int64_t dl_done = 0;  // slots [0, dl_done) are queued for download
  ~pcd_handle() {
    if (stream) cudaStreamSynchronize(stream);
    if (aux) cudaStreamSynchronize(aux);
    if (aux2) cudaStreamSynchronize(aux2);
    for (cudaEvent_t e : evpool) cudaEventDestroy(e);
    if (ev_vdone) cudaEventDestroy(ev_vdone);
    if (aux2) cudaStreamDestroy(aux2);
    if (h_vbad) cudaFreeHost(h_vbad);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_sweep) cudaEventDestroy(ev_sweep);
    if (ev_join) cudaEventDestroy(ev_join);
    if (aux) cudaStreamDestroy(aux);
    comm.reset();
    if (scal) cudaFree(scal);
    if (h_scal) cudaFreeHost(h_scal);
    if (d_errt) cudaFree(d_errt);
    if (stream) cudaStreamDestroy(stream);
  }
};

// multi-GPU helpers (defined with the C ABI below)
static void exchange(pcd_handle* h, int* buf, bool reduce, int lo, int hi);
static void rebuild_shards(pcd_handle* h);

namespace pcd {

static int host_tanh_fma() {
#if defined(__x86_64__)
  __builtin_cpu_init();
  return (__builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2")) ? 1 : 0;
#else
  return 1;
#endif
}

static int grid_for(long long n, int block, int cap = 148 * 16) {
  long long g = (n + block - 1) / block;
  return (int)std::max(1LL, std::min<long long>(g, cap));
}

// Builds a time-ordered CSR of slot indices keyed by `keys` (owner or product).
// first index t with a[t] outside [lo, hi) (device-side input validation), -1 if none
static long long first_out_of_range(pcd_handle* h, const int* a, int64_t n, int lo, int hi) {
  if (n <= 0) return -1;
  DBuf<unsigned long long> first;
  first.alloc(1);
  CK(cudaMemsetAsync(first.p, 0xff, sizeof(unsigned long long), h->stream));
  k_first_out_of_range<<<grid_for(n, 256), 256, 0, h->stream>>>(a, n, lo, hi, first.p);
  unsigned long long r = ~0ull;
  CK(cudaMemcpyAsync(&r, first.p, sizeof r, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return r == ~0ull ? -1 : (long long)r;
}

static void build_csr(pcd_handle* h, const int* d_keys, int nkeys, DBuf<int>& start, DBuf<int>& slots) {
  const int64_t T = h->T;
  start.alloc((size_t)nkeys + 1);
  slots.alloc((size_t)std::max<int64_t>(T, 1));
  if (T == 0) {
    CK(cudaMemsetAsync(start.p, 0, sizeof(int) * ((size_t)nkeys + 1), h->stream));
    return;
  }
  DBuf<int> vals_in, keys_out;
  vals_in.alloc(T);
  keys_out.alloc(T);
  k_iota<<<grid_for(T, 256), 256, 0, h->stream>>>(vals_in.p, T);
  int bits = 1;
  while ((1LL << bits) < (long long)nkeys) ++bits;
  size_t tmp_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, d_keys, keys_out.p, vals_in.p, slots.p,
                                     (int)T, 0, bits, h->stream));
  DBuf<unsigned char> tmp;
  tmp.alloc(tmp_bytes);
  CK(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, d_keys, keys_out.p, vals_in.p, slots.p,
                                     (int)T, 0, bits, h->stream));
  k_csr_starts<<<(int)((T + 1 + 255) / 256), 256, 0, h->stream>>>(keys_out.p, T, nkeys, start.p);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(h->stream));
}

// all = false keeps neg_flag: the checkpoint advance's negativity flag stays
// set on the device until the next scalar read checks it (advance_checkpoint)
static void reset_scalars(pcd_handle* h, bool all = true) {
  Scalars s{};
  s.first_changed = ~0ull;
  s.err_nonfinite = ~0ull;
  s.err_infeasible = ~0ull;
  *h->h_scal = s;
  CK(cudaMemcpyAsync(h->scal, h->h_scal, all ? sizeof(Scalars) : offsetof(Scalars, neg_flag),
                     cudaMemcpyHostToDevice, h->stream));
}

static void read_scalars(pcd_handle* h) {
  CK(cudaMemcpyAsync(h->h_scal, h->scal, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
}

struct IterOut {
  int64_t changed = 0, first_changed = -1, conflicts = 0, mismatch_delta = 0;
  int64_t max_evals = 0, total_evals = 0;
  bool aborted = false;  // the previous iteration's pipelined verification failed (simulate)
};

// Events used for the per-phase device timing (pcd_timing).
// Phase timers: an event pair per phase, resolved into the pcd_timing field
// when the stream is synchronised anyway (flush_timers) -- inside simulate()
// the timers are deferred to its end, so timing a phase costs no host
// round trip (outside, each phase is resolved at once).
static cudaEvent_t timer_event(pcd_handle* h) {
  if (h->evnext == h->evpool.size()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    h->evpool.push_back(e);
  }
  return h->evpool[h->evnext++];
}
static void flush_timers(pcd_handle* h) {
  if (h->tlog.empty()) {
    h->evnext = 0;
    return;
  }
  CK(cudaEventSynchronize(h->tlog.back().b));
  for (const auto& t : h->tlog) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, t.a, t.b));
    *t.acc += ms;
  }
  h->tlog.clear();
  h->evnext = 0;
}
struct PhaseTimer {
  pcd_handle* h;
  cudaEvent_t a = nullptr;
  explicit PhaseTimer(pcd_handle* hh) : h(hh) {}
  void start() {
    a = timer_event(h);
    CK(cudaEventRecord(a, h->stream));
  }
  void stop(double* acc) {
    cudaEvent_t b = timer_event(h);
    CK(cudaEventRecord(b, h->stream));
    h->tlog.push_back({a, b, acc});
    if (!h->defer_timers) flush_timers(h);
  }
};

template <int KIND>
static void launch_product_sweep(pcd_handle* h, int lo, int hi, long long* evals_out) {
  SweepArgs a{};
  a.model = h->model();
  a.M = h->M; a.J = h->J; a.lo = lo; a.hi = hi;
  a.pstart = h->pstart.p; a.pslots = h->pslots.p;
  a.ckcap = h->ckcap.p; a.hck = h->hck.p; a.ev = h->ev.p; a.xloc = h->xloc.p; a.rid = h->rid.p;
  a.nocache = h->nocache;
  a.cache = h->cache.p; a.written = h->written.p; a.ref = h->ref.n ? h->ref.p : nullptr;
  a.scal = h->scal; a.evals_out = evals_out;
  a.mine = h->comm ? h->d_mine.p : nullptr;
  const int wpb = 4;
  const size_t smem = warp_smem_bytes(h->J, 2 * h->J + 1, h->H, 2 * h->J) * wpb;
  CK(ensure_dyn_smem((const void*)k_sweep_product<KIND>, smem));
  k_sweep_product<KIND><<<(h->M + wpb - 1) / wpb, wpb * 32, smem, h->stream>>>(a);
  CK(cudaGetLastError());
}

template <int KIND>
static void launch_replay_sweep(pcd_handle* h, int lo, int hi, long long* evals_out) {
  const size_t per = (size_t)h->I * h->J;
  const size_t budget = (size_t)512 << 20;  // bytes of private state in flight
  int batch = (int)std::max<size_t>(1, std::min<size_t>((size_t)h->M, budget / std::max<size_t>(1, per * 4)));
  h->scratch.alloc(std::max<size_t>(1, per * (size_t)batch));
  const int wpb = 4;
  const size_t smem = warp_smem_bytes(h->J, 2 * h->J + 1, h->H, 2 * h->J) * wpb;
  CK(ensure_dyn_smem((const void*)k_sweep_replay<KIND>, smem));
  for (int m0 = 0; m0 < h->M; m0 += batch) {
    ReplayArgs a{};
    a.model = h->model();
    a.M = h->M; a.J = h->J; a.I = h->I; a.lo = lo; a.hi = hi; a.m0 = m0;
    a.m1 = std::min(h->M, m0 + batch);
    a.owner = h->owner.p; a.pstart = h->pstart.p; a.pslots = h->pslots.p;
    a.ckcap = h->ckcap.p; a.ckinv = h->ckinv.p; a.cache = h->cache.p; a.fresh = h->fresh.p;
    a.scratch = h->scratch.p; a.scal = h->scal; a.evals_out = evals_out;
    a.mine = h->comm ? h->d_mine.p : nullptr;
    const int nproc = a.m1 - a.m0;
    k_sweep_replay<KIND><<<(nproc + wpb - 1) / wpb, wpb * 32, smem, h->stream>>>(a);
    CK(cudaGetLastError());
  }
}

template <typename F>
static void dispatch_kind(int kind, F&& f) {
  switch (kind) {
    case kGreedy: f(std::integral_constant<int, kGreedy>{}); break;
    case kCapacity: f(std::integral_constant<int, kCapacity>{}); break;
    case kDual: f(std::integral_constant<int, kDual>{}); break;
    default: f(std::integral_constant<int, kNull>{}); break;
  }
}

static void throw_sweep_error(pcd_handle* h) {
  const Scalars& s = *h->h_scal;
  if (s.err_nonfinite == ~0ull && s.err_infeasible == ~0ull) return;
  if (s.err_nonfinite <= s.err_infeasible) {
    const int64_t t = (int64_t)(s.err_nonfinite & 0xffffffffull);
    throw ContractViolation("dual network produced a non-finite score", t);
  }
  const int64_t t = (int64_t)(s.err_infeasible & 0xffffffffull);
  throw ContractViolation("policy returned an infeasible action at t=" + std::to_string(t), t);
}

// AUTO's choice between the two tensor-core sweeps when the incremental one applies
constexpr bool kIncDefault = false;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeFn tensor_map_encoder() {
  static EncodeFn encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    encode = (EncodeFn)fn;
  }
  return encode;
}

// TMA map over the sweep's weight image (the B operands of every MMA): the
// kWImgBytes image viewed as [kWImgRows][128] fp16, loaded by two
// [kWImgRows/2][128] boxes (cp.async.bulk.tensor) at the start of every CTA.
static void make_wmap(pcd_handle* h) {
  const auto encode = tensor_map_encoder();
  const cuuint64_t dims[2] = {128, (cuuint64_t)kWImgRows};
  const cuuint64_t strides[1] = {128 * 2};
  const cuuint32_t box[2] = {128, (cuuint32_t)(kWImgRows / 2)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&h->wmap, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, (void*)h->tc_wimg2.p, dims, strides, box,
                            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (weights) failed (" + std::to_string((int)r) + ")");
}

// G-row buffer of the incremental sweep and its TMA map (2-D: 64 fp32 per
// row, one-row boxes), grown to the window's block count.
static void ensure_gmap(pcd_handle* h, size_t rows) {
  rows = std::max<size_t>(rows, 1);
  if (h->gmap_rows >= rows) return;
  const size_t cap = std::max(rows, h->gmap_rows * 2);
  h->grow.alloc(cap * kTcH);
  const auto encode = tensor_map_encoder();
  const cuuint64_t dims[2] = {(cuuint64_t)kTcH, (cuuint64_t)cap};
  const cuuint64_t strides[1] = {(cuuint64_t)kTcH * sizeof(float)};
  const cuuint32_t box[2] = {(cuuint32_t)kTcH, 1};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&h->gmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, h->grow.p, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  h->gmap_rows = cap;
}

// Work list of a tensor-core sweep over [lo, hi): this rank's processes with
// window slots, heaviest first; the first tiles*128 entries are dealt round
// robin over the tiles, the rest are pulled by rows as they finish (wctl[1]
// = next entry)
static void build_worklist(pcd_handle* h, int lo, int hi, cudaStream_t st) {
  const int M = h->M;
  h->wload.alloc(M); h->wids.alloc(M); h->wload_s.alloc(M); h->wq.alloc(M); h->wctl.alloc(2); h->wbeg.alloc(M);
  CK(cudaMemsetAsync(h->wctl.p, 0, 2 * sizeof(int), st));
  k_window_load<<<(M + 255) / 256, 256, 0, st>>>(h->pstart.p, h->pslots.p, M, lo, hi,
                                                 h->comm ? h->d_mine.p : nullptr, h->wload.p, h->wids.p, h->wctl.p,
                                                 h->wbeg.p);
  int bits = 1;
  while ((1LL << bits) <= (long long)h->max_load) ++bits;
  // (simulate) sort on the bits the previous iteration's busiest window load
  // needs, with headroom, instead of the plan's whole-horizon maximum: one
  // radix pass instead of two at C3. A heavier load would only be dealt out
  // of LPT order (the sweep's results do not depend on the order); the
  // incremental sweep reads the maximum off the sorted list, so it keeps
  // every bit.
  const bool inc = h->tc_kernel_req == 2 || (h->debug & PCD_DEBUG_TC_INC) || kIncDefault;
  if (h->wl_hint > 0 && !inc) {
    int hb = 1;
    while ((1LL << hb) <= 4 * h->wl_hint) ++hb;
    bits = std::min(bits, hb);
  }
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairsDescending(nullptr, tb, h->wload.p, h->wload_s.p, h->wids.p, h->wq.p, M, 0,
                                               bits, st));
  h->wtmp.alloc(tb);
  CK(cub::DeviceRadixSort::SortPairsDescending(h->wtmp.p, tb, h->wload.p, h->wload_s.p, h->wids.p, h->wq.p, M, 0,
                                               bits, st));
  h->timing.kernel_launches += 2;
}

// One iteration over [lo, hi) on the resident cache. engine: REPLAY/PRODUCT.
static void ensure_aux(pcd_handle* h) {
  if (h->aux) return;
  CK(cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_sweep, cudaEventDisableTiming));
  CK(cudaStreamCreateWithFlags(&h->aux2, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&h->ev_vdone, cudaEventDisableTiming));
  CK(cudaHostAlloc((void**)&h->h_vbad, sizeof(int), cudaHostAllocDefault));
  *h->h_vbad = 0;
}

static void launch_tc(pcd_handle* h, int lo, int hi, long long* evals_out, double guard, int verify,
                      int tiles_req = 0, bool spec = false, bool verify_async = false) {
  TcArgs a{};
  if (spec) {
    a.spec = 1;
    // rows below 1/256 of the guards (where every observed tensor-core error
    // lies: 18 wrong argmaxes at C3, margins < guard/1024) are re-evaluated in
    // the sweep, the rest speculated (C3: 1/16 -> 1/256 cut the in-sweep
    // re-evaluations 15x, 98 -> 95.4 ms)
    a.spec_floor = 1.f / 256.f;
    a.spec_flip = (h->debug & PCD_DEBUG_SPEC_FLIP) ? 1 : 0;
    a.spec_cap = (int)std::min<int64_t>((int64_t)(hi - lo), 1 << 20);
    h->spec_q.alloc((size_t)a.spec_cap * kSpecStride);
    h->spec_n.alloc(1);
    CK(cudaMemsetAsync(h->spec_n.p, 0, sizeof(int), h->stream));
    a.spec_n = h->spec_n.p;
    a.spec_q = h->spec_q.p;
  }
  SweepArgs& s = a.s;
  s.model = h->model();
  s.M = h->M; s.J = h->J; s.lo = lo; s.hi = hi;
  s.pstart = h->pstart.p; s.pslots = h->pslots.p;
  s.ckcap = h->ckcap.p; s.hck = h->hck.p; s.ev = h->ev.p; s.xloc = h->xloc.p; s.rid = h->rid.p;
  s.nocache = h->nocache;
  s.cache = h->cache.p; s.written = h->written.p; s.ref = h->ref.n ? h->ref.p : nullptr;
  s.scal = h->scal; s.evals_out = evals_out;
  if (!h->wl_ready) build_worklist(h, lo, hi, h->stream);
  h->wl_ready = false;
  a.wq = h->wq.p; a.wctl = h->wctl.p; a.wbeg = h->wbeg.p; a.wlen = h->wload.p; a.wimg2 = h->tc_wimg2.p; a.n3 = h->tc_n3;
  a.b1f = h->tc_b1.p; a.b2f = h->tc_b2.p;
  a.inv_c0 = h->tc_ic0.p; a.inv_x0 = h->tc_ix0.p; a.rtabq = h->tc_rtq.p;
  {  // the guards as floats rounded up, so the kernel's margin tests never undercut them
    auto up = [](double g) {
      float gf = (float)g;
      if ((double)gf < g) gf = nextafterf(gf, INFINITY);
      return gf;
    };
    a.guard = up(guard > 0 ? guard : h->tc_guard);
    a.guard_abs = up(guard > 0 ? guard : h->tc_guard_abs);
    a.gnode = guard > 0 ? nullptr : h->tc_gnode.p;  // (an override applies to every node)
  }
  a.verify = verify;
  a.stats = h->tc_stats.p;
  // PCD_DEBUG_TC_PROFILE: per-phase clock64 totals of CTA 0, printed to stderr
  const bool prof = (h->debug & PCD_DEBUG_TC_PROFILE) != 0;
  if (prof) {
    // phase totals + per-step (active rows, cycles) of CTA 0 half 0 + 6 per half
    h->tc_prof.alloc(20 + 2 * 4096 + 2 * 148 * 6);
    CK(cudaMemsetAsync(h->tc_prof.p, 0, (20 + 2 * 4096 + 2 * 148 * 6) * sizeof(long long), h->stream));
    a.prof = h->tc_prof.p;
  }
  // tiles < SMs (tests): rows pull processes from the work list mid-iteration
  const int tiles = tiles_req > 0 ? std::min(h->tc_tiles, tiles_req) : h->tc_tiles;
  // the incremental-layer-1 sweep needs the frozen-cache prefix counts (not
  // Time Warp's nocache windows), J <= kIncMaxJ and |D| within int16
  const int req = h->tc_kernel_req ? h->tc_kernel_req
                  : (h->debug & PCD_DEBUG_TC_FUSED) ? 1 : (h->debug & PCD_DEBUG_TC_INC) ? 2 : 0;
  const bool inc_fits = h->inc_ok && !h->nocache && std::min<int64_t>(h->max_load, (int64_t)hi - lo) < 32000;
  if (req == 2 && !inc_fits)
    throw InvalidArgument("tc_kernel=incremental does not apply (Time Warp window, J > 104 or window load >= 32000)");
  if (inc_fits && req != 1 && (req == 2 || kIncDefault)) {
    a.spec = 0;  // (the incremental sweep re-evaluates every row within the guard itself)
    const int nb = hck_rows(lo, hi);
    ensure_gmap(h, (size_t)nb);
    IncPrep pr{};
    pr.hck = h->hck.p; pr.ev = h->ev.p; pr.tau = h->tau.p; pr.ckcap = h->ckcap.p;
    pr.a64 = h->inc_a64.p; pr.b1 = h->inc_b1.p; pr.wload_sorted = h->wload_s.p;
    pr.lo = lo; pr.hi = hi; pr.J = h->J; pr.nb = nb;
    pr.grow = h->grow.p; pr.bA = h->inc_bA.p; pr.bD = h->inc_bD.p;
    CK(launch_inc_prep(pr, h->stream));
    IncArgs x{};
    x.t = a;
    x.af = h->inc_af.p; x.wx = h->inc_wx.p; x.wt = h->inc_wt.p;
    x.tau = h->tau.p; x.bA = h->inc_bA.p; x.bD = h->inc_bD.p;
    CK(launch_tc_inc(x, h->gmap, tiles, h->stream));
    h->timing.kernel_launches += 2;
    h->timing.tc_kernel = 2;
    h->timing.tc_inc_iters += 1;
  } else {
    CK(launch_tc_pp(a, h->wmap, tiles, h->stream));
    h->timing.tc_kernel = 1;
    if (a.spec && verify_async) {  // the speculated decisions checked on `aux` (finish_verify)
      ensure_aux(h);
      h->ckcap_v.alloc(std::max(1, h->J));
      CK(cudaMemcpyAsync(h->ckcap_v.p, h->ckcap.p, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaEventRecord(h->ev_sweep, h->stream));
      CK(cudaStreamWaitEvent(h->aux, h->ev_sweep, 0));
      SweepArgs sv = a.s;
      sv.ckcap = h->ckcap_v.p;
      CK(launch_spec_verify(sv, a.spec_q, a.spec_n, a.spec_cap, (h->debug & PCD_DEBUG_SPEC_RERUN) ? 1 : 0, h->aux));
      // the verdict to pinned memory, the flag cleared for the next
      // verification (same stream), an event the host waits on
      CK(cudaMemcpyAsync(h->h_vbad, &h->scal->spec_bad, sizeof(int), cudaMemcpyDeviceToHost, h->aux));
      CK(cudaMemsetAsync(&h->scal->spec_bad, 0, sizeof(int), h->aux));
      CK(cudaEventRecord(h->ev_vdone, h->aux));
      h->verify_pending = true;
      h->timing.kernel_launches += 1;
    } else if (a.spec) {  // the speculated decisions checked against the reference policy
      CK(launch_spec_verify(a.s, a.spec_q, a.spec_n, a.spec_cap, (h->debug & PCD_DEBUG_SPEC_RERUN) ? 1 : 0,
                            h->stream));
      h->timing.kernel_launches += 1;
    }
  }
  if (prof) {
    long long v[20];
    CK(cudaMemcpyAsync(v, h->tc_prof.p, sizeof v, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (h->timing.tc_kernel == 2) {
      std::vector<long long> tr(2 * 4096);
      CK(cudaMemcpy(tr.data(), h->tc_prof.p + 20, tr.size() * sizeof(long long), cudaMemcpyDeviceToHost));
      const int edges[6] = {1, 3, 9, 17, 33, 65};
      long long cyc[5] = {0, 0, 0, 0, 0}, cnt[5] = {0, 0, 0, 0, 0};
      for (int k = 0; k < 4096 && tr[2 * k]; ++k)
        for (int e = 0; e < 5; ++e)
          if (tr[2 * k] >= edges[e] && tr[2 * k] < edges[e + 1]) { cyc[e] += tr[2 * k + 1]; cnt[e] += 1; }
      fprintf(stderr, "incsteps active[1-2]=%lld@%lld [3-8]=%lld@%lld [9-16]=%lld@%lld [17-32]=%lld@%lld [33-64]=%lld@%lld (steps@cycles/step)\n",
              cnt[0], cnt[0] ? cyc[0] / cnt[0] : 0, cnt[1], cnt[1] ? cyc[1] / cnt[1] : 0, cnt[2], cnt[2] ? cyc[2] / cnt[2] : 0,
              cnt[3], cnt[3] ? cyc[3] / cnt[3] : 0, cnt[4], cnt[4] ? cyc[4] / cnt[4] : 0);
    }
    if (h->timing.tc_kernel == 2)
      fprintf(stderr, "incprof steps=%lld exact_nodes=%lld pre=%lld dirty=%lld part/near=%lld zB1=%lld L2=%lld E2=%lld L3=%lld S=%lld UB4=%lld chk=%lld\n",
              v[10], v[14], v[11], v[12], v[13], v[0], v[1], v[2], v[3], v[4], v[5], v[6]);
    else
    fprintf(stderr, "tcprof steps=%lld F=%lld L1=%lld E1=%lld L2=%lld E2=%lld L3=%lld S=%lld fin=%lld chk=%lld U=%lld\n",
            v[10], v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], v[9]);
    if (h->timing.tc_kernel == 1) {
      const int nh = 2 * std::min(148, h->tc_tiles);
      std::vector<long long> hp((size_t)nh * 6);
      CK(cudaMemcpy(hp.data(), h->tc_prof.p + 20 + 2 * 4096, hp.size() * 8, cudaMemcpyDeviceToHost));
      int im = 2;  // (CTA 0 carries the phase clocks: excluded)
      std::vector<long long> cyc(nh);
      for (int i = 2; i < nh; ++i) {
        cyc[i] = hp[6 * i + 1];
        if (cyc[i] > cyc[im]) im = i;
      }
      std::vector<long long> sc = cyc;
      std::sort(sc.begin(), sc.end());
      const long long* m = &hp[6 * im];
      fprintf(stderr, "tchalf max: half %d steps=%lld loop=%lld (%.0f/step) rc_batches=%lld rc_cycles=%lld setup=%lld endwait=%lld | loop cycles median %lld p10 %lld\n",
              im, m[0], m[1], m[0] ? (double)m[1] / m[0] : 0.0, m[2], m[3], m[4], m[5], sc[nh / 2], sc[nh / 10]);
    }
    fprintf(stderr, "tcprof F: loads=%lld feat=%lld x=%lld | recheck batches=%lld rows=%lld ordered=%lld feat=%lld L1=%lld L2=%lld L3=%lld score=%lld\n",
            v[12], v[13], v[14], v[11] & 0xfffff, (v[11] >> 20) & 0xfffff, v[11] >> 40, v[15], v[16], v[17], v[18], v[19]);
  }
}

// Effective attempts of the frozen cache and their checkpointed per-node
// prefix counts H (k_effective, k_seg_*, k_hist_prefix); returns the row count.
static int build_hck(pcd_handle* h, int lo, int hi) {
  const int J = h->J;
  const int wpb = 8;  // warps (products) per block
  const int pgrid = (h->I + wpb - 1) / wpb;
  k_effective<<<pgrid, wpb * 32, (size_t)wpb * 2 * J * 4, h->stream>>>(h->qstart.p, h->qslots.p, h->I, lo, hi,
                                                                   h->cache.p, h->ckinv.p, J, h->ev.p,
                                                                   h->qcur_on ? h->qcur.p : nullptr);
  const int nb = hck_rows(lo, hi);
  const int nseg = (nb + kSegRows - 1) / kSegRows;
  const size_t hsm = (size_t)kSegRows * J * 4;
  CK(ensure_dyn_smem((const void*)k_hist_prefix, hsm));
  k_seg_count<<<nseg, 256, (size_t)J * 4, h->stream>>>(h->ev.p, lo, hi, J, h->seg.p);
  {
    const int nblk = std::max(1, std::min(256, nseg));
    h->segtot.alloc((size_t)nblk * seg_stride(J));
    k_seg_scan_a<<<nblk, 128, 0, h->stream>>>(h->seg.p, nseg, J, h->segtot.p);
    k_seg_scan_b<<<seg_stride(J), 256, 0, h->stream>>>(h->segtot.p, nblk, J);
    k_seg_scan_c<<<nblk, 128, 0, h->stream>>>(h->seg.p, nseg, J, h->segtot.p);
  }
  k_hist_prefix<<<nseg, 256, hsm, h->stream>>>(h->ev.p, lo, hi, J, nb, h->seg.p, h->hck.p);
  CK(cudaGetLastError());
  h->timing.kernel_launches += 6;
  return nb;
}

// General closed form: same-product chains of the plan (once per plan) and the
// window's entry lists by (product, node) (every iteration).
static void build_gen_lists(pcd_handle* h, int lo, int hi) {
  const int64_t T = h->T;
  const int W = hi - lo;
  if (!h->gen_plan) {
    h->gprev.alloc((size_t)std::max<int64_t>(T, 1));
    h->ocache.alloc((size_t)std::max<int64_t>(T, 1));
    h->ofresh.alloc((size_t)std::max<int64_t>(T, 1));
    h->gdl.alloc(2 * (size_t)std::max<int64_t>(T, 1));
    if (T > 0) {
      DBuf<int> k0, v0, k1, v1;
      k0.alloc(T); v0.alloc(T); k1.alloc(T); v1.alloc(T);
      k_plan_pkeys<<<grid_for(T, 256), 256, 0, h->stream>>>(h->pslots.p, h->product.p, T, k0.p, v0.p);
      int bits = 1;
      while ((1LL << bits) < (long long)h->I) ++bits;
      size_t tb = 0;
      CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k0.p, k1.p, v0.p, v1.p, (int)T, 0, bits, h->stream));
      h->gtmp.alloc(tb);
      CK(cub::DeviceRadixSort::SortPairs(h->gtmp.p, tb, k0.p, k1.p, v0.p, v1.p, (int)T, 0, bits, h->stream));
      k_prev_same<<<grid_for(T, 256), 256, 0, h->stream>>>(k1.p, v1.p, h->pslots.p, h->owner.p, T, h->gprev.p);
      CK(cudaGetLastError());
      CK(cudaStreamSynchronize(h->stream));
    }
    h->gen_plan = true;
  }
  const long long nkeys = (long long)h->I * h->J + 1;  // + the null bucket
  if (nkeys >= INT32_MAX) throw InvalidArgument("general engine: products x nodes must fit int32");
  h->gstart.alloc((size_t)nkeys + 1);
  h->gkeys.alloc((size_t)std::max(W, 1)); h->gkeys_s.alloc((size_t)std::max(W, 1));
  h->gvals.alloc((size_t)std::max(W, 1)); h->gslots.alloc((size_t)std::max(W, 1));
  k_gen_keys<<<grid_for(W, 256), 256, 0, h->stream>>>(h->cache.p, h->product.p, lo, hi, h->J, (int)(nkeys - 1),
                                                     h->gkeys.p, h->gvals.p);
  int bits = 1;
  while ((1LL << bits) < nkeys) ++bits;
  size_t tb = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, h->gkeys.p, h->gkeys_s.p, h->gvals.p, h->gslots.p, W, 0, bits,
                                     h->stream));
  h->gtmp.alloc(tb);
  CK(cub::DeviceRadixSort::SortPairs(h->gtmp.p, tb, h->gkeys.p, h->gkeys_s.p, h->gvals.p, h->gslots.p, W, 0, bits,
                                     h->stream));
  k_csr_starts<<<(int)((W + 1 + 255) / 256), 256, 0, h->stream>>>(h->gkeys_s.p, W, (int)nkeys, h->gstart.p);
  CK(cudaGetLastError());
  h->timing.kernel_launches += 5;
}

template <int KIND>
static void launch_general_sweep(pcd_handle* h, int lo, int hi, long long* evals_out) {
  GenArgs a{};
  a.model = h->model();
  a.M = h->M; a.J = h->J; a.lo = lo; a.hi = hi;
  a.pstart = h->pstart.p; a.pslots = h->pslots.p; a.prev = h->gprev.p;
  a.ckcap = h->ckcap.p; a.ckinv = h->ckinv.p; a.hck = h->hck.p; a.ev = h->ev.p;
  a.gstart = h->gstart.p; a.gslots = h->gslots.p;
  a.ocache = h->ocache.p; a.ofresh = h->ofresh.p; a.dl = h->gdl.p;
  a.cache = h->cache.p; a.written = h->written.p; a.ref = h->ref.n ? h->ref.p : nullptr;
  a.scal = h->scal; a.evals_out = evals_out;
  a.mine = h->comm ? h->d_mine.p : nullptr;
  const int wpb = 4;
  const size_t smem = gen_warp_smem_bytes(h->J, 2 * h->J + 1, h->H, 2 * h->J) * wpb;
  CK(ensure_dyn_smem((const void*)k_sweep_general<KIND>, smem));
  k_sweep_general<KIND><<<(h->M + wpb - 1) / wpb, wpb * 32, smem, h->stream>>>(a);
  CK(cudaGetLastError());
}

static void check_advance(pcd_handle* h);

static IterOut iter_out(pcd_handle* h) {
  IterOut out;
  const Scalars& s = *h->h_scal;
  out.changed = (int64_t)s.changed;
  out.first_changed = s.changed ? (int64_t)s.first_changed : -1;
  out.conflicts = (int64_t)s.conflicts;
  out.mismatch_delta = (int64_t)s.mismatch_delta;
  out.max_evals = (int64_t)s.max_evals;
  out.total_evals = (int64_t)s.total_evals;
  return out;
}

// A speculated decision differs from the reference policy: the iteration
// again from the backed-up window without speculation (every row within the
// guard re-evaluated in the sweep); the scalars are read afterwards.
static void rerun_without_spec(pcd_handle* h, int64_t lo64, int64_t hi64, long long* evals_out, double guard,
                               int verify, int tiles) {
  PhaseTimer tm(h);
  tm.start();
  const int W = (int)(hi64 - lo64);
  CK(cudaMemcpyAsync(h->cache.p + lo64, h->cbak.p, sizeof(int) * (size_t)W, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemcpyAsync(h->written.p + lo64, h->wbak.p, (size_t)W, cudaMemcpyDeviceToDevice, h->stream));
  const int J = h->J, wpb = 8, pgrid = (h->I + wpb - 1) / wpb;
  k_xinit<<<pgrid, wpb * 32, (size_t)(wpb + 1) * J * 4, h->stream>>>(h->qstart.p, h->qslots.p, h->I, (int)lo64,
                                                               (int)hi64, h->ev.p, h->rid.p, h->tau.p, h->ckinv.p, J,
                                                               h->xloc.p, h->qcur_on ? h->qcur.p : nullptr);
  reset_scalars(h, false);
  CK(cudaMemsetAsync(&h->scal->spec_bad, 0, sizeof(int), h->stream));
  launch_tc(h, (int)lo64, (int)hi64, evals_out, guard, verify, tiles, false);
  tm.stop(&h->timing.sweep_ms);
  h->timing.tc_spec_reruns += 1;
  h->timing.kernel_launches += 2;
  read_scalars(h);
}

// Waits for a deferred verification; true if a speculated decision was wrong.
static bool finish_verify(pcd_handle* h) {
  if (!h->verify_pending) return false;
  h->verify_pending = false;
  CK(cudaEventSynchronize(h->ev_vdone));
  return *h->h_vbad != 0;
}

static IterOut run_iteration(pcd_handle* h, int engine, int64_t lo64, int64_t hi64, long long* evals_out,
                             double guard = 0.0, int verify = 0, int tiles = 0, bool defer_verify = false) {
  IterOut out;
  bool spec = false;  // the tensor-core sweep speculated (tc_spec.cu)
  const int lo = (int)lo64, hi = (int)hi64, W = hi - lo;
  if (h->verify_pending && (W <= 0 || engine != PCD_ENGINE_PRODUCT) && finish_verify(h)) {
    out.aborted = true;  // (a pipelined verification outside the tensor-core path: settled first)
    return out;
  }
  reset_scalars(h, false);
  if (W <= 0) return out;
  PhaseTimer tm(h);
  if (engine == PCD_ENGINE_GENERAL) {
    tm.start();
    build_hck(h, lo, hi);
    build_gen_lists(h, lo, hi);
    tm.stop(&h->timing.prep_ms);
    tm.start();
    dispatch_kind(h->kind, [&](auto k) { launch_general_sweep<decltype(k)::value>(h, lo, hi, evals_out); });
    exchange(h, h->cache.p, true, lo, hi);  // N>1: owned window slots + convergence scalars
    if (h->comm) CK(cudaMemsetAsync(h->written.p + lo, 1, (size_t)W, h->stream));
    tm.stop(&h->timing.sweep_ms);
    h->timing.kernel_launches += 1;
    h->timing.sweep_launches += 1;
  } else if (engine == PCD_ENGINE_PRODUCT || engine == PCD_ENGINE_PRODUCT_FP64) {
    const bool tc = engine == PCD_ENGINE_PRODUCT && h->tc_ok && h->kind == kDual;
    // speculation (tc_spec.cu) needs the derived per-node guards and a
    // single rank; the window's cache / written flags are backed up for the
    // re-run a wrong speculated decision triggers
    spec = tc && !(h->debug & PCD_DEBUG_NO_SPEC) && !h->nospec_once && !verify && !(guard > 0) && !h->nocache &&
           !h->comm && h->tc_gnode.n > 0 && h->J % 2 == 0;  // (the verification's paired loads)
    h->nospec_once = false;
    if (tc) {  // work list and backups on the second auxiliary stream, beside the cache kernels
      ensure_aux(h);
      CK(cudaEventRecord(h->ev_fork, h->stream));
      CK(cudaStreamWaitEvent(h->aux2, h->ev_fork, 0));
      build_worklist(h, lo, hi, h->aux2);
      if (spec) {
        h->cbak.alloc((size_t)W);
        h->wbak.alloc((size_t)W);
        CK(cudaMemcpyAsync(h->cbak.p, h->cache.p + lo, sizeof(int) * (size_t)W, cudaMemcpyDeviceToDevice, h->aux2));
        CK(cudaMemcpyAsync(h->wbak.p, h->written.p + lo, (size_t)W, cudaMemcpyDeviceToDevice, h->aux2));
        // (a verification in flight clears the flag on `aux` after its verdict)
        if (!h->verify_pending) CK(cudaMemsetAsync(&h->scal->spec_bad, 0, sizeof(int), h->aux2));
      }
      CK(cudaEventRecord(h->ev_join, h->aux2));
    }
    tm.start();
    const int J = h->J;
    const int wpb = 8;  // warps (products) per block
    const int pgrid = (h->I + wpb - 1) / wpb;
    const int nb = build_hck(h, lo, hi);
    k_tau<<<(32 * J + 127) / 128, 128, 0, h->stream>>>(h->hck.p, h->ev.p, h->ckcap.p, lo, hi, J, nb, h->tau.p);
    k_xinit<<<pgrid, wpb * 32, (size_t)(wpb + 1) * J * 4, h->stream>>>(h->qstart.p, h->qslots.p, h->I, lo, hi, h->ev.p,
                                                                 h->rid.p, h->tau.p, h->ckinv.p, J, h->xloc.p,
                                                                 h->qcur_on ? h->qcur.p : nullptr);
    CK(cudaGetLastError());
    tm.stop(&h->timing.prep_ms);
    h->timing.kernel_launches += 2;
    // the previous iteration's pipelined verification: its verdict is needed
    // before this sweep publishes anything; a rejected one abandons this
    // iteration (its cache kernels wrote only per-iteration buffers)
    if (h->verify_pending && finish_verify(h)) {
      h->wl_ready = false;
      out.aborted = true;
      return out;
    }
    tm.start();
    if (tc) {
      CK(cudaStreamWaitEvent(h->stream, h->ev_join, 0));
      h->wl_ready = true;
      launch_tc(h, lo, hi, evals_out, guard, verify, tiles, spec, spec && defer_verify);
      h->timing.tc_used = 1;
      h->timing.tc_tiles = h->tc_tiles;
    } else {
      dispatch_kind(h->kind, [&](auto k) { launch_product_sweep<decltype(k)::value>(h, lo, hi, evals_out); });
    }
    exchange(h, h->cache.p, true, lo, hi);  // N>1: owned window slots + convergence scalars
    if (h->comm)  // every window slot is owned by some rank: all written now
      CK(cudaMemsetAsync(h->written.p + lo, 1, (size_t)W, h->stream));
    tm.stop(&h->timing.sweep_ms);
    h->timing.kernel_launches += 1;
    h->timing.sweep_launches += 1;
  } else {
    tm.start();
    dispatch_kind(h->kind, [&](auto k) { launch_replay_sweep<decltype(k)::value>(h, lo, hi, evals_out); });
    if (h->comm) {  // fresh[] slices to every rank; then a replicated publish
      exchange(h, h->fresh.p, false, lo, hi);
      k_scalars_pack<<<1, 1, 0, h->stream>>>(h->scal, h->d_red.p);
      h->comm->all_reduce(h->d_red.p + 3, 1, RedOp::SumI64, h->stream);
      h->comm->all_reduce(h->d_red.p + 5, 2, RedOp::MinU64, h->stream);
      h->comm->all_reduce(h->d_red.p + 7, 1, RedOp::MaxU64, h->stream);
      k_scalars_unpack<<<1, 1, 0, h->stream>>>(h->d_red.p, h->scal);
    }
    tm.stop(&h->timing.sweep_ms);
    h->timing.sweep_launches += 1;
    h->timing.kernel_launches += 1;
    // errors surface before publishing (the reference throws out of the sweep)
    read_scalars(h);
    check_advance(h);
    throw_sweep_error(h);
    tm.start();
    k_publish<<<grid_for(W, 256), 256, 0, h->stream>>>(h->fresh.p, h->cache.p, h->written.p,
                                                        h->ref.n ? h->ref.p : nullptr, lo, hi, h->scal);
    CK(cudaGetLastError());
    tm.stop(&h->timing.publish_ms);
    h->timing.kernel_launches += 1;
  }
  read_scalars(h);
  check_advance(h);  // the previous iteration's checkpoint advance (deferred check)
  if (spec && defer_verify && (h->h_scal->err_nonfinite != ~0ull || h->h_scal->err_infeasible != ~0ull)) {
    // an error on a speculated trajectory counts only once it is verified
    if (finish_verify(h)) rerun_without_spec(h, lo64, hi64, evals_out, guard, verify, tiles);
  } else if (spec && !defer_verify && h->h_scal->spec_bad) {
    rerun_without_spec(h, lo64, hi64, evals_out, guard, verify, tiles);
  }
  throw_sweep_error(h);
  return iter_out(h);
}

// advance_checkpoint (engine.hpp:514-526): subtract the stable prefix's
// fulfilments from the checkpoint; a negative count means an infeasible
// cached action, for which the reference throws ContractViolation at the
// first such order. The check is deferred: the flag stays set on the device
// and is read with the next iteration's scalars (no extra host round trip per
// iteration); the state before the advance is recovered by the exact inverse
// (unadvance) so the serial error search can replay it. defer = false checks now.
static void advance_checkpoint(pcd_handle* h, int64_t from, int64_t to, bool defer = true) {
  if (to <= from) return;
  PhaseTimer tm(h);
  tm.start();
  k_advance<<<grid_for(to - from, 256), 256, (size_t)h->J * 4, h->stream>>>(
      h->cache.p, h->product.p, (int)from, (int)to, h->J, h->ckcap.p, h->ckinv.p, &h->scal->neg_flag);
  CK(cudaGetLastError());
  h->adv_buf = 0;
  h->adv_from = from;
  h->adv_to = to;
  tm.stop(&h->timing.advance_ms);
  h->timing.kernel_launches += 1;
  if (!defer) {
    CK(cudaMemcpyAsync(&h->h_scal->neg_flag, &h->scal->neg_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    check_advance(h);
  }
}

// The checkpoint before the last advance: k_advance's atomic subtractions
// added back (exact integer inverse; the advanced slots of the cache are
// unchanged until the next sweep, which starts at the advance's end).
static void unadvance(pcd_handle* h) {
  const int from = (int)h->adv_from, to = (int)h->adv_to;
  k_unadvance<<<grid_for(to - from, 256), 256, (size_t)h->J * 4, h->stream>>>(h->cache.p, h->product.p, from, to,
                                                                             h->J, h->ckcap.p, h->ckinv.p);
  CK(cudaGetLastError());
  h->timing.kernel_launches += 1;
}

// h_scal->neg_flag was just read from the device: a set flag belongs to the
// last advance (earlier ones were checked at earlier reads)
static void check_advance(pcd_handle* h) {
  if (!h->h_scal->neg_flag) return;
  if (h->adv_buf < 0) {  // a stale flag of another path (Time Warp checks its own merges)
    CK(cudaMemsetAsync(&h->scal->neg_flag, 0, sizeof(int), h->stream));
    h->h_scal->neg_flag = 0;
    return;
  }
  unadvance(h);
  CK(cudaMemsetAsync(&h->scal->neg_flag, 0, sizeof(int), h->stream));
  k_advance_serial<<<1, 1, 0, h->stream>>>(h->cache.p, h->product.p, h->order_t.n ? h->order_t.p : nullptr,
                                           (int)h->adv_from, (int)h->adv_to, h->J, h->ckcap.p, h->ckinv.p,
                                           h->d_errt);
  long long et = -1;
  CK(cudaMemcpyAsync(&et, h->d_errt, sizeof(long long), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->adv_buf = -1;
  throw ContractViolation("infeasible fulfillment at t=" + std::to_string(et), et);
}

// the pending advance checked now (before returning or throwing otherwise)
// Takes back the last checkpoint advance (its prefix held a speculated
// decision that the verification rejected): the state before it, no pending
// negativity flag.
static void undo_advance(pcd_handle* h) {
  if (h->adv_buf < 0) return;
  unadvance(h);
  CK(cudaMemsetAsync(&h->scal->neg_flag, 0, sizeof(int), h->stream));
  h->h_scal->neg_flag = 0;
  h->adv_buf = -1;
}

static void flush_advance_check(pcd_handle* h) {
  if (h->adv_buf < 0) return;
  CK(cudaMemcpyAsync(&h->h_scal->neg_flag, &h->scal->neg_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  check_advance(h);
}

static int choose_engine(pcd_handle* h, int requested) {
  if (requested == PCD_ENGINE_REPLAY || requested == PCD_ENGINE_GENERAL) return requested;
  if (requested == PCD_ENGINE_PRODUCT || requested == PCD_ENGINE_PRODUCT_FP64) {
    if (!h->is_product)
      throw InvalidArgument("engine=PRODUCT requires a run partition (each process owns one contiguous stretch of a product's orders, or whole products)");
    return requested;
  }
  if (requested != PCD_ENGINE_AUTO) throw InvalidArgument("unknown engine " + std::to_string(requested));
  return h->is_product ? PCD_ENGINE_PRODUCT : PCD_ENGINE_GENERAL;
}

static void ensure_state_buffers(pcd_handle* h) {
  const size_t T = (size_t)std::max<int64_t>(h->T, 1);
  const size_t IJ = std::max<size_t>(1, (size_t)h->I * h->J);
  h->cache.alloc(T);
  h->fresh.alloc(T);
  h->ev.alloc(T + kK);  // + kK: the sweep reads whole K-slot blocks
  h->written.alloc(T + 4);  // + 4: the incremental sweep copies whole 4-byte words
  h->ckcap.alloc(std::max(1, h->J));
  h->ckinv.alloc(IJ);
  h->ckbak.alloc(IJ + h->J);  // Time Warp's merge backup
  h->xloc.alloc(std::max<size_t>(1, (size_t)h->runs * std::max(1, h->J)));
  h->tau.alloc(std::max(1, h->J));
  const size_t nb = (T + kK - 1) / kK + 1;  // + 1: blocks start at lo & ~(K-1)
  h->hck.alloc(nb * hck_stride(std::max(1, h->J)));
  h->seg.alloc(((nb + kSegRows - 1) / kSegRows + 1) * seg_stride(std::max(1, h->J)));
  h->evals.alloc(std::max(1, h->M));
}

// picard_simulate (engine.hpp:458-590) over the resident cache.
static void simulate(pcd_handle* h, const pcd_config* cfg, bool track, pcd_result* res,
                     pcd_trace_row* trace, int64_t trace_cap) {
  const int64_t T = h->T;
  *res = pcd_result{0, -1, 0, 0, 0, 0, 0, -1};
  if (!h->have_plan) throw InvalidArgument("no partition plan set (pcd_set_plan)");
  if (cfg->processes != 0 && cfg->processes != h->M)
    throw ContractViolation("config process count disagrees with the plan");
  if (cfg->max_steps < 0 || cfg->max_iterations < 0)
    throw ContractViolation("picard config values must be non-negative");
  const int engine = choose_engine(h, cfg->engine);
  if (cfg->tc_kernel < 0 || cfg->tc_kernel > 2) throw InvalidArgument("tc_kernel must be 0, 1 or 2");
  h->tc_kernel_req = cfg->tc_kernel;
  h->tlog.clear();  // (phases of an earlier call that threw: their fields are reset next)
  if (h->aux) CK(cudaStreamSynchronize(h->aux));  // (a verification left by a call that threw)
  if (h->aux2) CK(cudaStreamSynchronize(h->aux2));
  h->verify_pending = false;
  struct CursorOff {
    pcd_handle* h;
    ~CursorOff() { h->qcur_on = false; }
  } cursor_guard{h};
  h->qcur.alloc((size_t)std::max(1, h->I));
  CK(cudaMemsetAsync(h->qcur.p, 0, sizeof(int2) * (size_t)std::max(1, h->I), h->stream));
  h->qcur_on = true;
  h->wl_hint = 0;
  struct HintOff {
    pcd_handle* h;
    ~HintOff() { h->wl_hint = 0; }
  } hint_guard{h};
  h->evnext = 0;
  struct DeferTimers {
    pcd_handle* h;
    ~DeferTimers() { h->defer_timers = false; }
  } defer_guard{h};
  h->timing = pcd_timing{};
  h->timing.engine_used = engine;
  h->timing.device = h->device;
  h->defer_timers = true;
  if (h->tc_stats.n) CK(cudaMemsetAsync(h->tc_stats.p, 0, sizeof(unsigned long long) * kTcStats, h->stream));
  const int64_t cap_it = cfg->max_iterations > 0 ? cfg->max_iterations : 2 * T + 4;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, h->stream));
  // checkpoint = initial state; written = 0
  CK(cudaMemcpyAsync(h->ckcap.p, h->cap0.p, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemcpyAsync(h->ckinv.p, h->inv0.p, sizeof(int) * (size_t)h->I * h->J, cudaMemcpyDeviceToDevice, h->stream));
  if (T) CK(cudaMemsetAsync(h->written.p, 0, (size_t)T, h->stream));
  int64_t mismatches = 0;
  if (track) {
    reset_scalars(h);
    k_mismatches<<<grid_for(T, 256), 256, 0, h->stream>>>(h->cache.p, h->ref.p, T, h->scal);
    read_scalars(h);
    mismatches = h->h_scal->mismatches;
    if (mismatches == 0) res->iterations_to_correct = 0;
  }
  std::vector<pcd_trace_row> rows;
  int64_t ws = 0, iteration = 0, episodes = 0;
  h->adv_buf = -1;
  CK(cudaMemsetAsync(&h->scal->neg_flag, 0, sizeof(int), h->stream));
  // Pipelined verification (engine_used PRODUCT with speculation): iteration
  // i's verification runs beside iteration i+1's advance and cache kernels
  // and is settled before i+1's sweep (run_iteration). Until then iteration
  // i's bookkeeping is provisional: `pend` keeps what a rejection takes back
  // (its window, whether it advanced the checkpoint, the counters before it).
  // Not with a per-iteration history (it copies each iteration's cache).
  h->pipe_verify = !h->history;
  struct Acc {
    pcd_result res;
    int64_t mismatches, episodes, rows, steps_critical, total_evals;
  };
  struct Pending {
    bool on = false, advanced = false;
    int64_t ws = 0, W = 0, iteration = 0;
    Acc acc{};
  } pend;
  auto settle = [&](const IterOut* aborted_by) -> bool {  // true: iteration pend.iteration must re-run
    if (!pend.on) return false;
    const bool bad = aborted_by ? aborted_by->aborted : finish_verify(h);
    if (!bad) {
      pend.on = false;
      return false;
    }
    // rejected: back to the state before iteration pend.iteration
    *res = pend.acc.res;
    mismatches = pend.acc.mismatches;
    episodes = pend.acc.episodes;
    rows.resize((size_t)pend.acc.rows);
    h->timing.steps_critical = pend.acc.steps_critical;
    h->timing.total_evals = pend.acc.total_evals;
    if (pend.advanced) undo_advance(h);
    // (the pending window's backups were swapped out to the spares)
    CK(cudaMemcpyAsync(h->cache.p + pend.ws, h->cbak2.p, sizeof(int) * (size_t)pend.W, cudaMemcpyDeviceToDevice,
                       h->stream));
    CK(cudaMemcpyAsync(h->written.p + pend.ws, h->wbak2.p, (size_t)pend.W, cudaMemcpyDeviceToDevice, h->stream));
    CK(cudaMemsetAsync(h->qcur.p, 0, sizeof(int2) * (size_t)std::max(1, h->I), h->stream));  // windows back
    ws = pend.ws;
    iteration = pend.iteration - 1;
    h->nospec_once = true;
    h->timing.tc_spec_reruns += 1;
    pend.on = false;
    return true;
  };
  for (;;) {
    if (ws >= T) {
      if (settle(nullptr)) continue;
      break;
    }
    const int64_t we = cfg->max_steps > 0 ? std::min(T, ws + cfg->max_steps) : T;
    if (iteration >= cap_it) {
      if (settle(nullptr)) continue;
      flush_advance_check(h);  // the reference throws from the advance before reaching the cap
      res->iterations_run = iteration;
      res->trace_rows = (int64_t)rows.size();
      throw IterationLimit("picard iteration cap exceeded (" + std::to_string(cap_it) +
                               "); the policy may be nondeterministic",
                           iteration, rows);
    }
    ++iteration;
    const Acc before{*res, mismatches, episodes, (int64_t)rows.size(), h->timing.steps_critical,
                     h->timing.total_evals};
    IterOut it = run_iteration(h, engine, ws, we, nullptr, cfg->tc_guard, cfg->tc_verify, cfg->tc_tiles, true);
    if (it.aborted) {  // the previous iteration's speculation was rejected: re-run it
      settle(&it);
      continue;
    }
    pend.on = false;  // (run_iteration settled the previous verification)
    // the checkpoint advance goes out while a deferred verification of
    // speculated decisions still runs; a rejected one takes it back and the
    // iteration is re-run without speculation
    auto next_ws = [&](const IterOut& o) { return o.changed == 0 ? we : std::max(ws, o.first_changed); };
    int64_t nws = next_ws(it);
    if (nws > ws) advance_checkpoint(h, ws, nws);
    if (h->verify_pending && h->pipe_verify) {
      // verdict later: the next iteration's cache kernels and backups go to
      // the spare buffers
      h->ev2.alloc(h->ev.n);
      h->hck2.alloc(h->hck.n);
      h->xloc2.alloc(h->xloc.n);
      h->ev.swap(h->ev2);
      h->hck.swap(h->hck2);
      h->xloc.swap(h->xloc2);
      h->cbak.swap(h->cbak2);
      h->wbak.swap(h->wbak2);
      pend.on = true;
      pend.W = we - ws;
      pend.advanced = nws > ws;
      pend.ws = ws;
      pend.iteration = iteration;
      pend.acc = before;
    } else if (finish_verify(h)) {
      if (nws > ws) undo_advance(h);
      rerun_without_spec(h, ws, we, nullptr, cfg->tc_guard, cfg->tc_verify, cfg->tc_tiles);
      throw_sweep_error(h);
      it = iter_out(h);
      nws = next_ws(it);
      if (nws > ws) advance_checkpoint(h, ws, nws);
    }
    h->wl_hint = it.max_evals;
    res->iterations_to_converged += 1;
    res->policy_eval_count_sequential_equivalent += it.max_evals;
    res->total_policy_evals += it.total_evals;
    res->conflicts += it.conflicts;
    mismatches += it.mismatch_delta;
    if (cfg->record_trace) rows.push_back({episodes, iteration, it.changed, it.max_evals, ws});
    if (track && res->iterations_to_correct < 0 && mismatches == 0) res->iterations_to_correct = iteration;
    if (h->history && iteration - 1 < h->history_cap && T)
      CK(cudaMemcpy(h->history + (iteration - 1) * T, h->cache.p, (size_t)T * 4, cudaMemcpyDeviceToHost));
    h->timing.steps_critical += it.max_evals;
    h->timing.total_evals += it.total_evals;
    if (it.changed == 0) ++episodes;
    ws = nws;
    // slots before the checkpoint are final (before the pending iteration's
    // window while its verification runs): copy them out beside the next
    // iterations (batches of >= 1M slots)
    const int64_t fin = pend.on ? pend.ws : ws;
    if (h->dl_out && fin - h->dl_done >= (1 << 20)) {
      ensure_aux(h);
      CK(cudaEventRecord(h->ev_fork, h->stream));
      CK(cudaStreamWaitEvent(h->aux, h->ev_fork, 0));
      CK(cudaMemcpyAsync(h->dl_out + h->dl_done, h->cache.p + h->dl_done, sizeof(int32_t) * (size_t)(fin - h->dl_done),
                         cudaMemcpyDeviceToHost, h->aux));
      h->dl_done = fin;
    }
  }
  flush_advance_check(h);
  h->adv_buf = -1;
  CK(cudaEventRecord(e1, h->stream));
  CK(cudaEventSynchronize(e1));
  flush_timers(h);
  h->defer_timers = false;
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  h->timing.total_ms = ms;
  h->timing.iterations = iteration;
  if (h->tc_stats.n) {
    unsigned long long st[kTcStats];
    CK(cudaMemcpy(st, h->tc_stats.p, sizeof st, cudaMemcpyDeviceToHost));
    h->timing.tc_rows = (int64_t)st[0];
    h->timing.tc_flagged = (int64_t)st[1];
    h->timing.tc_disagree = (int64_t)st[2];
    h->timing.tc_unflagged_bad = (int64_t)st[3];
    h->timing.tc_max_score_err = (double)__uint_as_float_host((uint32_t)st[4]);
    h->timing.tc_speculated = (int64_t)st[5];
  }
  h->timing.tc_guard = cfg->tc_guard > 0 ? cfg->tc_guard : h->tc_guard;
  h->timing.tc_score_bound = h->tc_bound;
  res->iterations_run = iteration;
  res->trace_rows = (int64_t)rows.size();
  for (int64_t i = 0; i < (int64_t)rows.size() && i < trace_cap; ++i) trace[i] = rows[(size_t)i];
}

}  // namespace pcd

// ============================================================== C ABI (device)
using namespace pcd;

namespace pcd {
int translate_exception();  // capi.cpp
}

#define PCD_TRY try {
#define PCD_CATCH \
  }               \
  catch (...) { return pcd::translate_exception(); }

// pinned host pool (pcd_host_alloc / pcd_host_free)
static std::mutex g_hmu;
static std::multimap<size_t, void*> g_hfree;
static std::map<void*, size_t> g_hsize;
extern "C" void* pcd_host_alloc(size_t bytes) {
  bytes = (bytes + 4095) & ~(size_t)4095;
  {
    std::lock_guard<std::mutex> lk(g_hmu);
    auto it = g_hfree.lower_bound(bytes);
    if (it != g_hfree.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      g_hfree.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  if (cudaHostAlloc(&p, bytes, cudaHostAllocPortable) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lk(g_hmu);
  g_hsize[p] = bytes;
  return p;
}
extern "C" void pcd_host_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_hmu);
  auto it = g_hsize.find(p);
  if (it != g_hsize.end()) g_hfree.insert({it->second, p});
}

extern "C" int pcd_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

static void validate_instance(const pcd_instance* in) {
  if (!in) throw InvalidArgument("instance is null");
  if (in->nodes < 1) throw InvalidArgument("instance needs at least one node");
  if (in->nodes > 32767) throw InvalidArgument("node count above 32767 is not supported");
  if (in->products < 1) throw InvalidArgument("product count must be >= 1");
  if (in->horizon < 0 || in->horizon > 0x7ffffff0LL) throw InvalidArgument("horizon out of range");
  if (in->horizon > 0 && (!in->product || !in->reward_row || !in->reward_table))
    throw InvalidArgument("instance arrays missing");
  if (!in->capacity || !in->inventory) throw InvalidArgument("instance state missing");
  // per-order range checks run on the device after the upload (pcd_create)
  for (int64_t i = 0; i < in->reward_rows * in->nodes; ++i)
    if (!std::isfinite(in->reward_table[i])) throw InvalidArgument("rewards must be finite");
}

// Process sharding (this rank's processes; all ranks' slot lists for the
// exchange) and the tensor-core tiles of this rank's processes.
static void rebuild_shards(pcd_handle* h) {
  if (!h->have_plan) return;
  const int32_t M = h->M;
  const int64_t T = h->T;
  // per-process loads from the owned-slot CSR (device)
  std::vector<int32_t> pst((size_t)M + 1);
  CK(cudaMemcpyAsync(pst.data(), h->pstart.p, sizeof(int32_t) * ((size_t)M + 1), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  std::vector<int64_t> load((size_t)M, 0);
  for (int32_t m = 0; m < M; ++m) load[(size_t)m] = pst[(size_t)m + 1] - pst[(size_t)m];
  h->rank_of.assign((size_t)M, 0);
  if (h->comm) {
    std::vector<int32_t> owner((size_t)std::max<int64_t>(T, 1));
    if (T) CK(cudaMemcpy(owner.data(), h->owner.p, sizeof(int32_t) * (size_t)T, cudaMemcpyDeviceToHost));
    shard_processes(owner.data(), T, M, h->nranks, h->rank_of.data());
    std::vector<unsigned char> mine((size_t)M);
    for (int32_t m = 0; m < M; ++m) mine[(size_t)m] = h->rank_of[(size_t)m] == h->rank;
    h->d_mine.upload(mine.data(), mine.size(), h->stream);
    // rank-major, time-ordered slot lists (counting sort) for pack / unpack
    std::vector<int32_t> off((size_t)h->nranks + 1, 0), slots((size_t)std::max<int64_t>(T, 1));
    for (int64_t t = 0; t < T; ++t) off[(size_t)h->rank_of[(size_t)owner[(size_t)t]] + 1] += 1;
    for (int32_t r = 0; r < h->nranks; ++r) off[(size_t)r + 1] += off[(size_t)r];
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int64_t t = 0; t < T; ++t) slots[(size_t)fill[(size_t)h->rank_of[(size_t)owner[(size_t)t]]]++] = (int32_t)t;
    h->h_roff = off;
    h->h_rslots = slots;
    h->maxn = 0;
    for (int32_t r = 0; r < h->nranks; ++r) h->maxn = std::max(h->maxn, off[(size_t)r + 1] - off[(size_t)r]);
    h->d_roff.upload(off.data(), off.size(), h->stream);
    h->d_rslots.upload(slots.data(), slots.size(), h->stream);
    h->d_send.alloc((size_t)std::max(1, h->maxn));
    h->d_recv.alloc((size_t)std::max(1, h->maxn) * h->nranks);
    h->d_red.alloc(8);
  }
  // tensor-core sweep: one CTA per SM; rows pull this rank's processes from
  // the per-iteration work list (launch_tc), so only the largest load (for
  // the sort key width) is kept here
  h->max_load = 0;
  for (int32_t m = 0; m < M; ++m)
    if (h->rank_of[(size_t)m] == h->rank) h->max_load = std::max(h->max_load, load[(size_t)m]);
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, h->device);
  h->tc_tiles = nsm;
  CK(cudaStreamSynchronize(h->stream));
}

// After a sweep on N>1 ranks: gather every rank's owned slots of `buf` inside
// the window [lo, hi) (the cache for the fused run-partition / general
// sweeps, fresh[] for the replay sweep) and, for the fused sweeps, reduce
// the per-rank convergence scalars. Each rank's owned slots are one
// time-ordered list, so its window slice is a contiguous range [a_r, a_r +
// n_r); the all-gather ships max_r n_r int32 per rank (padded).
static void exchange(pcd_handle* h, int* buf, bool reduce, int lo, int hi) {
  if (!h->comm) return;  // single GPU without a communicator
  if (h->nranks > kMaxRanks) throw InvalidArgument("too many ranks");
  RankWindow w{};
  int maxw = 0;
  for (int r = 0; r < h->nranks; ++r) {
    const int32_t* b = h->h_rslots.data() + h->h_roff[(size_t)r];
    const int32_t* e = h->h_rslots.data() + h->h_roff[(size_t)r + 1];
    const int32_t* a0 = std::lower_bound(b, e, lo);
    const int32_t* a1 = std::lower_bound(a0, e, hi);
    w.start[r] = h->h_roff[(size_t)r] + (int)(a0 - b);
    w.count[r] = (int)(a1 - a0);
    maxw = std::max(maxw, w.count[r]);
  }
  if (maxw > 0) {
    const int r = h->rank;
    k_pack_slots<<<grid_for(std::max(1, w.count[r]), 256), 256, 0, h->stream>>>(buf, h->d_rslots.p + w.start[r],
                                                                                w.count[r], h->d_send.p);
    h->comm->all_gather(h->d_send.p, h->d_recv.p, (size_t)maxw, h->stream);
    k_unpack_window<<<grid_for((long long)maxw * h->nranks, 256), 256, 0, h->stream>>>(h->d_recv.p, h->d_rslots.p, w,
                                                                                      h->nranks, maxw, buf);
  }
  if (reduce) {
    k_scalars_pack<<<1, 1, 0, h->stream>>>(h->scal, h->d_red.p);
    h->comm->all_reduce(h->d_red.p, 4, RedOp::SumI64, h->stream);
    h->comm->all_reduce(h->d_red.p + 4, 3, RedOp::MinU64, h->stream);
    h->comm->all_reduce(h->d_red.p + 7, 1, RedOp::MaxU64, h->stream);
    k_scalars_unpack<<<1, 1, 0, h->stream>>>(h->d_red.p, h->scal);
  }
  CK(cudaGetLastError());
  h->timing.kernel_launches += reduce ? 4 : 2;
}

// Largest dual-network feature (policies.hpp:136-148): c / c0 and x / x0 with
// the policy's normalisers (states never exceed the instance's initial one),
// t / T with the policy's horizon; at least 1.
static double feature_max(const pcd_instance* in, const int32_t* pcap, const int32_t* pinv, int64_t horizon,
                          int J) {
  double fmax = 1.0;
  if (pcap != in->capacity)  // the instance's own normalisers give ratios <= 1
    for (int j = 0; j < J; ++j)
      if (pcap[j] > 0) fmax = std::max(fmax, (double)in->capacity[j] / pcap[j]);
  if (pinv != in->inventory)
    for (size_t i = 0; i < (size_t)in->products * J; ++i)
      if (pinv[i] > 0) fmax = std::max(fmax, (double)in->inventory[i] / pinv[i]);
  if (horizon > 0) {
    double tmax = (double)std::max<int64_t>(in->horizon - 1, 0);
    if (in->order_t)
      for (int64_t t = 0; t < in->horizon; ++t) tmax = std::max(tmax, (double)in->order_t[t]);
    fmax = std::max(fmax, tmax / (double)horizon);
  }
  return fmax;
}

// Rounding bound E between two FP64 evaluations of the dual network's scores
// that differ only in summation order / FMA use (the reference's ordered
// acc = b; acc += w*x vs the order-free recheck), for features in [0, 1]:
//   layer 1: |dz1| <= 2 g(in+1) S1,                 S1 = max_n |b1| + fmax sum|W1[n]|
//   h1:      |dh1| <= |dz1| + 2u                    (tanh 1-Lipschitz, <= 1 ulp each)
//   layer 2: |dz2| <= A2 |dh1| + 2 g(H+1) S2,       A2 = max_n sum|W2[n]|
//   score:   |ds|  <= A3 |dh2| + 2 g(H+2) S3 + 4u (|r| + S3)
// with g(n) = n u / (1 - n u), u = 2^-53; the fast path needs both decision
// margins above 4E (pp::half_recheck). Returns 4E, or 0 (fast path off) when
// the bound is not small.
static double fast_margin_bound(const pcd_policy* pol, int J, int H, double rmax, double fmax) {
  const int in = 2 * J + 1, out = 2 * J;
  const double u = std::ldexp(1.0, -53);
  auto g = [&](double n) { return n * u / (1.0 - n * u); };
  double S1 = 0, A2 = 0, S2 = 0, A3 = 0, S3 = 0;
  for (int n = 0; n < H; ++n) {
    double a = 0;
    for (int c = 0; c < in; ++c) a += std::fabs(pol->w1[(size_t)n * in + c]);
    S1 = std::max(S1, std::fabs(pol->b1[n]) + fmax * a);
    double b = 0;
    for (int c = 0; c < H; ++c) b += std::fabs(pol->w2[(size_t)n * H + c]);
    A2 = std::max(A2, b);
    S2 = std::max(S2, b + std::fabs(pol->b2[n]));
  }
  for (int j = 0; j < J; ++j) {
    double a = 0;
    for (int l = 0; l < H; ++l) a += std::fabs(pol->w3[(size_t)j * H + l]) + std::fabs(pol->w3[(size_t)(J + j) * H + l]);
    A3 = std::max(A3, a);
    S3 = std::max(S3, a + std::fabs(pol->b3[j]) + std::fabs(pol->b3[J + j]));
  }
  (void)out;
  const double dz1 = 2 * g(in + 1) * S1, dh1 = dz1 + 2 * u;
  const double dz2 = A2 * dh1 + 2 * g(H + 1) * S2, dh2 = dz2 + 2 * u;
  const double ds = A3 * dh2 + 2 * g(H + 2) * S3 + 4 * u * (rmax + S3);
  const double m = 4 * ds;
  return (std::isfinite(m) && m < 1e-6) ? std::max(m, 1e-13) : 0.0;
}

// Tensor-core exactness guard, DERIVED: an a-priori bound B
// on |score_tc - score_ref| for every row of every step, from
//   * the fp16 hi + 2^-11 lo split of operands (|x - hi - lo 2^-11| <=
//     2^-22 |x| + 2^-36, fp16 subnormals included), the fp32 rounding of
//     weights, reciprocals and features, and the dropped lo.lo product;
//   * the tcgen05.mma kind::f16 fp32 accumulation measured on this B200
//     (tools/mma_accum_probe.cu, profiles/r02_mma_accum_probe.log): per MMA
//     the 16 products and the accumulator are aligned to the largest
//     exponent e with the bits below 2^(e-24) truncated, and the sum is
//     truncated to fp32, so one MMA errs by < u (17 max|x_i| + 2 |D|),
//     u = 2^-24, bounded here by 19 u P(s) with P(s) the k-step's bound on
//     the partial sums;
//   * tanh_mufu's error, measured exhaustively over every float
//     (tools/tanh_mufu_probe.cu): kTanhErr;
//   * first-order propagation with the weights themselves, unit by unit
//     (|dz2_m| <= sum_c |W2_mc| |dh1_c| + ..., tanh 1-Lipschitz), per-column
//     feature maxima (capacities never exceed the instance's, inventories
//     likewise, t < T), and the reference's own FP64 rounding E64.
// A row whose best score beats the second by >= 2B (and |best| >= 2B) has
// the reference's decision; guard = 2B (1 + 2^-10) also absorbs the fp32
// subtraction v1 - v2. Returns B, or 0 when the tensor-core path must not be
// used (non-finite weights, operands outside fp16 range, features > 1e4).
constexpr double kTanhErr = 0x1p-22;  // >= max |tanh_mufu(z) - tanh(z)| over all floats (probe)
// Per node j (optional outputs): babs[j] >= |score_tc_j - score_ref_j| and
// rdiff[j] >= max_{i != j} error of s_j - s_i (the margin test's threshold
// when j is the best node); B = max babs, *bdiff = max rdiff.
static double tc_error_bound(const pcd_policy* pol, const pcd_instance* in, const int32_t* pcap,
                             const int32_t* pinv, int64_t horizon, int J, int H, double* bdiff,
                             std::vector<double>* babs = nullptr, std::vector<double>* rdiff = nullptr) {
  *bdiff = 0.0;
  const int inw = 2 * J + 1;
  const double u = 0x1p-24, t36 = 0x1p-36;
  double wmax = 0;
  auto scan = [&](const double* w, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      if (!std::isfinite(w[i])) return false;
      wmax = std::max(wmax, std::fabs(w[i]));
    }
    return true;
  };
  if (!scan(pol->w1, (size_t)H * inw) || !scan(pol->b1, H) || !scan(pol->w2, (size_t)H * H) || !scan(pol->b2, H) ||
      !scan(pol->w3, (size_t)2 * J * H) || !scan(pol->b3, 2 * J))
    return 0.0;
  if (wmax > 3.0e4) return 0.0;  // fp16 hi parts (65504) and W3' = W3[j] + W3[J+j]
  // per-column feature maxima
  std::vector<double> F((size_t)inw, 0.0);
  for (int j = 0; j < J; ++j) {
    if (pcap[j] > 0) F[j] = (double)in->capacity[j] / pcap[j];
    double m = 0;
    for (int64_t i = 0; i < in->products; ++i) {
      const int32_t x0 = pinv[(size_t)i * J + j];
      if (x0 > 0) m = std::max(m, (double)in->inventory[(size_t)i * J + j] / x0);
    }
    F[J + j] = m;
  }
  {
    double tmax = (double)std::max<int64_t>(in->horizon - 1, 0);
    if (in->order_t)
      for (int64_t t = 0; t < in->horizon; ++t) tmax = std::max(tmax, (double)in->order_t[t]);
    F[2 * J] = horizon > 0 ? tmax / (double)horizon : 0.0;
  }
  for (double f : F)
    if (!(f <= 1.0e4)) return 0.0;
  double rmax = 0.0;
  for (int64_t i = 0; i < in->reward_rows * in->nodes; ++i) rmax = std::max(rmax, std::fabs(in->reward_table[i]));
  if (!(rmax <= 1.0e6)) return 0.0;
  const double slack = 1.0 + 0x1p-9;  // second-order terms of the splits (|hi| <= |x| (1 + 2^-11) ...)
  // one layer: inputs with magnitude bound X[c] and error bound dX[c] (relative
  // representation error of the inputs themselves: rel_in), weights w(r, c);
  // returns the error bound of every output (before the activation)
  // nonneg: the inputs are >= 0 (layer 1's features), so each hi.hi product has
  // its weight's sign and the per-term truncations (toward zero) of one MMA
  // can only add up within one sign class: max(n+, n-) + 1 (the accumulator,
  // sign unknown) terms instead of 17
  auto layer = [&](int rows, int K, auto w, const std::vector<double>& X, const std::vector<double>& dX,
                   double rel_in, auto bias, bool nonneg) {
    std::vector<double> dz((size_t)rows);
    const int steps = (K + 15) / 16;
    for (int r = 0; r < rows; ++r) {
      // P: sum |w| X over the inputs so far; Pp / Pn: the same over positive /
      // negative weights. With nonneg inputs (0 <= x <= X) every partial sum
      // lies in [-Pn, Pp], so |C|, |D| <= max(Pp, Pn) (a linear form over a box
      // peaks at a vertex); otherwise they are bounded by P.
      double P = 0, Pp = 0, Pn = 0, accsum = 0, psum = 0, prop = 0, absw = 0;
      for (int s = 0; s < steps; ++s) {
        int npos = 0, nneg = 0;
        const double Cin = nonneg ? std::max(Pp, Pn) : P;  // bound on the accumulator entering the MMA
        double pmax = 0;                                   // bound on its largest product
        for (int c = 16 * s; c < std::min(K, 16 * s + 16); ++c) {
          const double wv = w(r, c), aw = std::fabs(wv), t = aw * X[(size_t)c] * slack;
          P += t;
          (wv > 0 ? Pp : Pn) += t;
          pmax = std::max(pmax, t);
          prop += aw * dX[(size_t)c];
          absw += aw + X[(size_t)c];
          npos += wv > 0 && X[(size_t)c] > 0;
          nneg += wv < 0 && X[(size_t)c] > 0;
        }
        const double Dout = nonneg ? std::max(Pp, Pn) : P;
        // one MMA errs by < n u 2^e + 2u |D|: n truncated terms (the products,
        // or with nonneg inputs one sign class of them, plus the accumulator),
        // 2^e <= max(|C|, max |p|)
        accsum += (nonneg ? std::max(npos, nneg) + 1 : 17) * std::max(Cin, pmax) + 2 * Dout;
        psum += P;
      }
      const double b = std::fabs(bias(r));
      // per product: feature/weight roundings + both splits + dropped lo.lo
      const double terms = (rel_in + 2 * 0x1p-22 + u + 0x1p-22) * P + 2 * t36 * absw;
      const double acc_hh = u * accsum;                       // hi.hi MMAs
      const double acc_x = 0x1p-11 * 2 * 19 * u * 2 * psum;  // hi.lo + lo.hi MMAs (x2 terms, x2 per k-step)
      const double rnd = u * P * 1.01 + u * b + u * (P + b) * 1.01;  // fmaf combine, fp32 bias, bias add
      dz[(size_t)r] = prop + terms + acc_hh + acc_x + rnd;
    }
    return dz;
  };
  // layer 1 (features: 3 fp32 roundings each), in the operand's column order
  // (tc_l1_input: the k-steps group the inputs as the MMAs do)
  const int K1 = tc_k1_needed(J);
  std::vector<double> Fk((size_t)K1, 0.0), zeros((size_t)K1, 0.0);
  for (int k = 0; k < K1; ++k) {
    const int c = tc_l1_input(k, J);
    Fk[(size_t)k] = c >= 0 ? F[(size_t)c] : 0.0;
  }
  const auto dz1 = layer(H, K1, [&](int r, int k) {
                           const int c = tc_l1_input(k, J);
                           return c >= 0 ? pol->w1[(size_t)r * inw + c] : 0.0;
                         }, Fk, zeros, 3 * u, [&](int r) { return pol->b1[r]; }, true);
  std::vector<double> X2((size_t)H, 1.0), dh1((size_t)H);
  for (int n = 0; n < H; ++n) dh1[(size_t)n] = dz1[(size_t)n] + kTanhErr;
  const auto dz2 = layer(H, H, [&](int r, int c) { return pol->w2[(size_t)r * H + c]; }, X2, dh1, 0.0,
                         [&](int r) { return pol->b2[r]; }, false);
  std::vector<double> dh2((size_t)H);
  for (int n = 0; n < H; ++n) dh2[(size_t)n] = dz2[(size_t)n] + kTanhErr;
  const auto dq = layer(J, H, [&](int r, int c) { return pol->w3[(size_t)r * H + c] + pol->w3[(size_t)(J + r) * H + c]; },
                        X2, dh2, 0.0, [&](int) { return 0.0; }, false);
  double B = 0;
  std::vector<double> own((size_t)J), bj((size_t)J), rj((size_t)J, 0.0);
  auto w3s = [&](int j, int l) { return pol->w3[(size_t)j * H + l] + pol->w3[(size_t)(J + j) * H + l]; };
  for (int j = 0; j < J; ++j) {
    double P3 = 0, prop = 0;
    for (int l = 0; l < H; ++l) {
      P3 += std::fabs(w3s(j, l));
      prop += std::fabs(w3s(j, l)) * dh2[(size_t)l];
    }
    const double b3s = std::fabs(pol->b3[j] + pol->b3[J + j]);
    // rtabq = fl32(r - b3s), score = fl32(rtabq - q)
    const double ds = dq[(size_t)j] + u * (rmax + b3s) + u * (rmax + b3s + P3) * 1.01;
    own[(size_t)j] = ds - prop;  // everything but the propagated h2 error
    bj[(size_t)j] = ds;
    B = std::max(B, ds);
  }
  // the margin test compares two scores of the same row: their h2 error is
  // shared, so the difference s_i - s_j errs by at most
  //   sum_l |W3'_il - W3'_jl| |dh2_l| + own_i + own_j
  double D = 0;
  for (int i = 0; i < J; ++i)
    for (int j = i + 1; j < J; ++j) {
      double a = 0;
      for (int l = 0; l < H; ++l) a += std::fabs(w3s(i, l) - w3s(j, l)) * dh2[(size_t)l];
      const double dij = a + own[(size_t)i] + own[(size_t)j];
      D = std::max(D, dij);
      rj[(size_t)i] = std::max(rj[(size_t)i], dij);
      rj[(size_t)j] = std::max(rj[(size_t)j], dij);
    }
  // the reference's FP64 scores against exact arithmetic (the same analysis as
  // fast_margin_bound with u = 2^-53 and one ordered chain)
  double fmaxall = 1.0;
  for (double f : F) fmaxall = std::max(fmaxall, f);
  const double fm = fast_margin_bound(pol, J, H, rmax, fmaxall);
  if (!(fm > 0)) return 0.0;  // the FP64 scores themselves are not known to 1e-6
  B += fm;
  *bdiff = std::isfinite(D) ? D + 2 * fm : 0.0;
  if (babs && rdiff) {
    babs->resize((size_t)J);
    rdiff->resize((size_t)J);
    for (int j = 0; j < J; ++j) {
      (*babs)[(size_t)j] = bj[(size_t)j] + fm;
      (*rdiff)[(size_t)j] = rj[(size_t)j] + 2 * fm;
    }
  }
  return std::isfinite(B) && std::isfinite(D) ? B : 0.0;
}
constexpr double kMaxTcGuard = 2e-2;  // beyond this most rows would be re-evaluated: FP64 path

// Weight images for the tcgen05 sweep (tc_sweep.cuh): fp16 hi + 2^11-scaled lo
// parts in the canonical K-major no-swizzle UMMA layout, W3' = W3[:J] + W3[J:]
// (the score needs only p_j + p_{J+j}), fp32 biases and feature reciprocals.
static void prepare_tc(pcd_handle* h, const pcd_policy* pol, const int32_t* pcap, const int32_t* pinv,
                       const double* rtab) {
  const int J = h->J, I = h->I, in = 2 * J + 1;
  std::vector<unsigned char> img2(kWImgBytes, 0);
  const int n3 = tc_pp_width_class(J);
  h->tc_n3 = n3;
  // per layer the hi rows 0..R-1 and lo rows R..2R-1 as one 2R-row K-major
  // operand, so hi.hi and hi.lo are one N = 2R MMA (layer 3: R = the width
  // class of J); the layers sit at the offsets of hi + lo images of widths
  // kTcH / kTcH / kTcN3
  auto put = [&](size_t base, int R, int r, int k, double w) {
    const float wf = (float)w;
    const __half hi = __float2half_rn(wf);
    const __half lo = __float2half_rn((wf - __half2float(hi)) * kLoScale);
    const int R2 = R == kTcN3 ? n3 : R;
    if (r < R2) {
      std::memcpy(&img2[base + (size_t)canon_off(2 * R2, r, k)], &hi, 2);
      std::memcpy(&img2[base + (size_t)canon_off(2 * R2, R2 + r, k)], &lo, 2);
    }
  };
  const size_t w2base = 2 * (size_t)kW1Bytes, w3base = w2base + 2 * (size_t)kW2Bytes;
  for (int r = 0; r < kTcH; ++r)
    for (int k = 0; k < kTcK1; ++k) {
      const int c = tc_l1_input(k, J);
      put(0, kTcH, r, k, c >= 0 ? pol->w1[(size_t)r * in + c] : 0.0);
    }
  for (int r = 0; r < kTcH; ++r)
    for (int k = 0; k < kTcH; ++k) put(w2base, kTcH, r, k, pol->w2[(size_t)r * kTcH + k]);
  for (int r = 0; r < kTcN3; ++r)
    for (int k = 0; k < kTcH; ++k)
      put(w3base, kTcN3, r, k, r < J ? pol->w3[(size_t)r * kTcH + k] + pol->w3[(size_t)(J + r) * kTcH + k] : 0.0);
  std::vector<float> b1(kTcH), b2(kTcH), ic0(J);
  for (int r = 0; r < kTcH; ++r) { b1[r] = (float)pol->b1[r]; b2[r] = (float)pol->b2[r]; }
  for (int j = 0; j < J; ++j) ic0[j] = pcap[j] > 0 ? (float)(1.0 / pcap[j]) : 0.f;
  h->tc_wimg2.upload(img2.data(), img2.size(), h->stream);
  make_wmap(h);
  h->tc_b1.upload(b1.data(), b1.size(), h->stream);
  h->tc_b2.upload(b2.data(), b2.size(), h->stream);
  h->tc_ic0.upload(ic0.data(), ic0.size(), h->stream);
  // 1/x0 of the policy's inventory normalisers, on the device (pinv0 is resident)
  h->tc_ix0.alloc((size_t)I * J + 4);  // + 4: the incremental sweep copies aligned 16-byte chunks
  if ((size_t)I * J > 0)
    k_inv_f32<<<grid_for((long long)I * J, 256), 256, 0, h->stream>>>(h->pinv0.p, (long long)I * J, h->tc_ix0.p);
  CK(cudaGetLastError());
  // score = r - (q + b3) is computed as (r - b3) - q: one rounding of the
  // FP64 difference instead of a bias add per node per step; 32-byte rows for
  // the 256-bit loads of the score phase
  const int RJ = (J + 7) & ~7;
  std::vector<float> rtq((size_t)h->R * RJ, 0.f);
  for (int64_t rr = 0; rr < h->R; ++rr)
    for (int j = 0; j < J; ++j)
      rtq[(size_t)rr * RJ + j] = (float)(rtab[(size_t)rr * J + j] - (pol->b3[j] + pol->b3[J + j]));
  h->tc_rtq.upload(rtq.data(), rtq.size(), h->stream);
  h->tc_stats.alloc(kTcStats);
  // incremental sweep (tc_inc.cu): A_j = W1[:, j] / c0_j (FP64 for the G rows,
  // fp32 for the per-row updates), W1[:, J + j], W1[:, 2J], b1
  h->inc_ok = J <= kIncMaxJ && h->H == kTcH;
  if (h->inc_ok) {
    std::vector<double> a64((size_t)J * kTcH), b1d(kTcH);
    std::vector<float> af((size_t)J * kTcH), wx((size_t)J * kTcH), wt(kTcH);
    for (int j = 0; j < J; ++j)
      for (int u = 0; u < kTcH; ++u) {
        const double w = pol->w1[(size_t)u * in + j];
        a64[(size_t)j * kTcH + u] = pcap[j] > 0 ? w / (double)pcap[j] : 0.0;
        af[(size_t)j * kTcH + u] = (float)a64[(size_t)j * kTcH + u];
        wx[(size_t)j * kTcH + u] = (float)pol->w1[(size_t)u * in + J + j];
      }
    for (int u = 0; u < kTcH; ++u) {
      wt[u] = (float)pol->w1[(size_t)u * in + 2 * J];
      b1d[u] = pol->b1[u];
    }
    h->inc_a64.upload(a64.data(), a64.size(), h->stream);
    h->inc_b1.upload(b1d.data(), b1d.size(), h->stream);
    h->inc_af.upload(af.data(), af.size(), h->stream);
    h->inc_wx.upload(wx.data(), wx.size(), h->stream);
    h->inc_wt.upload(wt.data(), wt.size(), h->stream);
    h->inc_bA.alloc(J);
    h->inc_bD.alloc(J);
  }
  CK(cudaStreamSynchronize(h->stream));
  h->tc_ok = true;
}

extern "C" int pcd_create(const pcd_instance* in, const pcd_policy* pol, int32_t device, pcd_handle** out) {
  PCD_TRY
  if (!out) throw InvalidArgument("out is null");
  *out = nullptr;
  validate_instance(in);
  if (!pol) throw InvalidArgument("policy is null");
  if (pol->kind < 0 || pol->kind > 3) throw InvalidArgument("unknown policy kind");
  if (pol->kind == PCD_POLICY_CAPACITY && !std::isfinite(pol->gamma)) throw InvalidArgument("gamma must be finite");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device available: the B200 engine has no CPU fallback");
  }
  if (device < 0 || device >= ndev) throw InvalidArgument("device index out of range");
  CK(cudaSetDevice(device));
  auto h = std::make_unique<pcd_handle>();
  h->device = device;
  CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
  h->J = in->nodes; h->I = in->products; h->T = in->horizon; h->R = in->reward_rows;
  h->tanh_fma = host_tanh_fma();
  const size_t T = (size_t)h->T, J = (size_t)h->J, IJ = (size_t)h->I * J;
  cudaStream_t s = h->stream;
  h->product.upload(in->product, T, s);
  if (in->order_t) h->order_t.upload(in->order_t, T, s);
  h->rrow.upload(in->reward_row, T, s);
  if (in->reward_rows > 0x7fffffffLL) throw InvalidArgument("too many reward rows");
  // per-order range checks on the device, read back with create's final
  // synchronisation (nothing below indexes with products or reward rows), so
  // the uploads overlap the host-side bound computations
  DBuf<unsigned long long> oor;
  oor.alloc(2);
  CK(cudaMemsetAsync(oor.p, 0xff, 2 * sizeof(unsigned long long), s));
  if (h->T > 0) {
    k_first_out_of_range<<<grid_for(h->T, 256), 256, 0, s>>>(h->product.p, h->T, 0, h->I, oor.p);
    k_first_out_of_range<<<grid_for(h->T, 256), 256, 0, s>>>(h->rrow.p, h->T, 0, (int)h->R, oor.p + 1);
    CK(cudaGetLastError());
  }
  h->rtab.upload(in->reward_table, (size_t)h->R * J, s);
  h->cap0.upload(in->capacity, J, s);
  h->inv0.upload(in->inventory, IJ, s);
  h->kind = pol->kind;
  h->gamma = pol->gamma;
  h->H = pol->hidden > 0 ? pol->hidden : 64;
  if (pol->kind == PCD_POLICY_DUAL) {
    if (!pol->w1 || !pol->b1 || !pol->w2 || !pol->b2 || !pol->w3 || !pol->b3)
      throw InvalidArgument("dual network: parameters missing");
    const int inw = 2 * h->J + 1, outw = 2 * h->J, H = h->H;
    // staging buffers live until the sync at the end of this block, so the
    // uploads, transposes and the host-side bound computations below overlap
    DBuf<double> tmp[3];
    int nt = 0;
    auto upload_t = [&](const double* src, int rows, int cols, DBuf<double>& dst) {
      DBuf<double>& t = tmp[nt++];
      t.upload(src, (size_t)rows * cols, s);
      dst.alloc((size_t)rows * cols);
      k_transpose_f64<<<(rows * cols + 255) / 256, 256, 0, s>>>(t.p, rows, cols, dst.p);
      CK(cudaGetLastError());
    };
    upload_t(pol->w1, H, inw, h->w1t);
    upload_t(pol->w2, H, H, h->w2t);
    upload_t(pol->w3, outw, H, h->w3t);
    {  // W3s[l][j] = W3[j][l] + W3[J+j][l]: summed prices for the order-free recheck
      const int Jn = h->J;
      std::vector<double> w3s((size_t)H * Jn);
      for (int l = 0; l < H; ++l)
        for (int j = 0; j < Jn; ++j)
          w3s[(size_t)l * Jn + j] = pol->w3[(size_t)j * H + l] + pol->w3[(size_t)(Jn + j) * H + l];
      h->w3s.upload(w3s.data(), w3s.size(), s);
      double rmax = 0;
      for (int64_t i = 0; i < in->reward_rows * in->nodes; ++i) rmax = std::max(rmax, std::fabs(in->reward_table[i]));
      const int32_t* pc = pol->init_capacity ? pol->init_capacity : in->capacity;
      const int32_t* pi = pol->init_capacity ? (pol->init_inventory ? pol->init_inventory : in->inventory)
                                             : in->inventory;
      const int64_t ph = pol->horizon >= 0 ? pol->horizon : in->horizon;
      h->fast_margin = fast_margin_bound(pol, Jn, H, rmax, feature_max(in, pc, pi, ph, Jn));
    }
    h->b1.upload(pol->b1, H, s);
    h->b2.upload(pol->b2, H, s);
    h->b3.upload(pol->b3, outw, s);
    if (pol->init_capacity) {
      h->pcap0.upload(pol->init_capacity, J, s);
      h->pinv0.upload(pol->init_inventory ? pol->init_inventory : in->inventory, IJ, s);
    } else {
      h->pcap0.upload(in->capacity, J, s);
      h->pinv0.upload(in->inventory, IJ, s);
    }
    h->p_horizon = pol->horizon >= 0 ? pol->horizon : in->horizon;
    if (tc_k1_needed(h->J) <= kTcK1 && h->J <= kTcN3 && H == kTcH) {
      const int32_t* pc = pol->init_capacity ? pol->init_capacity : in->capacity;
      const int32_t* pi = pol->init_capacity ? (pol->init_inventory ? pol->init_inventory : in->inventory)
                                             : in->inventory;
      double Bd = 0;
      std::vector<double> babs, rdiff;
      const double B = tc_error_bound(pol, in, pc, pi, h->p_horizon, h->J, H, &Bd, &babs, &rdiff);
      const double g = Bd * (1.0 + 0x1p-10);
      if (B > 0 && g <= kMaxTcGuard) {
        prepare_tc(h.get(), pol, pc, pi, in->reward_table);
        h->tc_guard = g;
        h->tc_guard_abs = B * (1.0 + 0x1p-10);
        h->tc_bound = B;
        // per-node thresholds (indexed by the best node), as floats rounded up
        std::vector<float> gt(2 * (size_t)kTcN3, 0.f);
        auto up = [](double x) {
          float f = (float)x;
          if ((double)f < x) f = nextafterf(f, INFINITY);
          return f;
        };
        for (int j = 0; j < h->J; ++j) {
          gt[(size_t)j] = up(rdiff[(size_t)j] * (1.0 + 0x1p-10));
          gt[(size_t)kTcN3 + j] = up(babs[(size_t)j] * (1.0 + 0x1p-10));
        }
        h->tc_gnode.upload(gt.data(), gt.size(), s);
      }
    }
    CK(cudaStreamSynchronize(s));  // the staging buffers (tmp) are released below
  }
  CK(cudaMalloc(&h->scal, sizeof(Scalars)));
  CK(cudaMallocHost(&h->h_scal, sizeof(Scalars)));
  CK(cudaMalloc(&h->d_errt, sizeof(long long)));
  CK(cudaStreamSynchronize(s));
  {  // the range checks (first offending t, product before reward row)
    unsigned long long r[2];
    CK(cudaMemcpy(r, oor.p, sizeof r, cudaMemcpyDeviceToHost));
    const long long bp = r[0] == ~0ull ? -1 : (long long)r[0], br = r[1] == ~0ull ? -1 : (long long)r[1];
    if (bp >= 0 && (br < 0 || bp <= br))
      throw InvalidArgument("order product out of range at t=" + std::to_string(bp));
    if (br >= 0) throw InvalidArgument("reward row out of range at t=" + std::to_string(br));
  }
  *out = h.release();
  return PCD_OK;
  PCD_CATCH
}

// The derived tensor-core bound of a dual policy on an instance, host only
// (pcd_create applies the same computation).
extern "C" int pcd_tc_error_bound(const pcd_instance* in, const pcd_policy* pol, double* bound, double* guard) {
  PCD_TRY
  validate_instance(in);
  if (!pol || !bound || !guard) throw InvalidArgument("null argument");
  *bound = 0.0;
  *guard = 0.0;
  if (pol->kind != PCD_POLICY_DUAL) return PCD_OK;
  const int J = in->nodes, H = pol->hidden;
  if (!(tc_k1_needed(J) <= kTcK1 && J <= kTcN3 && H == kTcH)) return PCD_OK;
  if (!pol->w1 || !pol->b1 || !pol->w2 || !pol->b2 || !pol->w3 || !pol->b3) throw InvalidArgument("policy weights missing");
  const int32_t* pc = pol->init_capacity ? pol->init_capacity : in->capacity;
  const int32_t* pi = pol->init_capacity ? (pol->init_inventory ? pol->init_inventory : in->inventory) : in->inventory;
  const int64_t ph = pol->horizon >= 0 ? pol->horizon : in->horizon;
  double Bd = 0;
  const double B = tc_error_bound(pol, in, pc, pi, ph, J, H, &Bd);
  const double g = Bd * (1.0 + 0x1p-10);
  *bound = B;
  *guard = (B > 0 && g <= kMaxTcGuard) ? g : 0.0;
  return PCD_OK;
  PCD_CATCH
}

extern "C" void pcd_destroy(pcd_handle* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);  // buffers go back to the pool idle
  delete h;
}

extern "C" int pcd_set_plan(pcd_handle* h, const int32_t* owner, int32_t M) {
  PCD_TRY
  if (!h) throw InvalidArgument("handle is null");
  CK(cudaSetDevice(h->device));
  // PartitionPlan::validate (engine.hpp:82-95)
  if (M < 1) throw ContractViolation("partition plan: process count must be >= 1");
  if (h->T > 0 && !owner) throw ContractViolation("partition plan does not cover the horizon");
  {  // validate into a scratch buffer: a rejected plan leaves the handle's plan intact
    DBuf<int> nowner;
    nowner.upload(owner, (size_t)h->T, h->stream);
    const long long bad = first_out_of_range(h, nowner.p, h->T, 0, M);
    if (bad >= 0) throw ContractViolation("partition plan: owner out of range", bad);
    h->have_plan = false;  // until the new plan's CSR / runs / shards are built
    nowner.swap(h->owner);
  }
  h->M = M;
  build_csr(h, h->owner.p, M, h->pstart, h->pslots);
  build_csr(h, h->product.p, h->I, h->qstart, h->qslots);
  // runs along the product slot lists (kernels.cuh: k_run_starts / k_run_ids /
  // k_check_runs): the closed-form engines need a run partition
  h->rid.alloc((size_t)std::max<int64_t>(h->T, 1));
  int hf = 0;
  h->runs = 0;
  if (h->T > 0) {
    DBuf<int> flagk, incl, nruns, nonlead, flag;
    flagk.alloc(h->T); incl.alloc(h->T); nruns.alloc(M); nonlead.alloc(M); flag.alloc(1);
    CK(cudaMemsetAsync(nruns.p, 0, sizeof(int) * (size_t)M, h->stream));
    CK(cudaMemsetAsync(nonlead.p, 0, sizeof(int) * (size_t)M, h->stream));
    CK(cudaMemsetAsync(flag.p, 0, sizeof(int), h->stream));
    k_run_starts<<<grid_for(h->T, 256), 256, 0, h->stream>>>(h->qslots.p, h->product.p, h->owner.p, h->T, flagk.p);
    size_t tb = 0;
    CK(cub::DeviceScan::InclusiveSum(nullptr, tb, flagk.p, incl.p, (int)h->T, h->stream));
    DBuf<unsigned char> tmp;
    tmp.alloc(tb);
    CK(cub::DeviceScan::InclusiveSum(tmp.p, tb, flagk.p, incl.p, (int)h->T, h->stream));
    k_run_ids<<<grid_for(h->T, 256), 256, 0, h->stream>>>(h->qslots.p, h->qstart.p, h->product.p, h->owner.p,
                                                          flagk.p, incl.p, h->T, h->rid.p, nruns.p, nonlead.p);
    k_check_runs<<<(M + 255) / 256, 256, 0, h->stream>>>(nruns.p, nonlead.p, M, flag.p);
    CK(cudaGetLastError());
    int nr = 0;
    CK(cudaMemcpyAsync(&nr, incl.p + h->T - 1, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(&hf, flag.p, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    h->runs = nr;
    // xloc is R x J int32: refuse the closed form for pathological plans
    if ((double)nr * h->J * 4 > 8e9) hf = 1;
  }
  h->is_product = hf == 0;
  h->gen_plan = false;
  h->have_plan = true;
  ensure_state_buffers(h);
  rebuild_shards(h);
  return PCD_OK;
  PCD_CATCH
}

static void upload_cache_ref(pcd_handle* h, const int32_t* initial_cache, const int32_t* reference) {
  ensure_state_buffers(h);
  const size_t T = (size_t)h->T;
  if (initial_cache) CK(cudaMemcpyAsync(h->cache.p, initial_cache, T * 4, cudaMemcpyHostToDevice, h->stream));
  else k_fill<<<grid_for((long long)T, 256), 256, 0, h->stream>>>(h->cache.p, -1, (long long)T);
  if (reference) {
    h->ref.alloc(std::max<size_t>(T, 1));
    CK(cudaMemcpyAsync(h->ref.p, reference, T * 4, cudaMemcpyHostToDevice, h->stream));
  } else if (h->ref.p) {
    h->ref.release();
  }
  CK(cudaGetLastError());
}

extern "C" int pcd_upload_cache(pcd_handle* h, const int32_t* initial_cache, const int32_t* reference) {
  PCD_TRY
  if (!h) throw InvalidArgument("handle is null");
  if (!h->have_plan) throw InvalidArgument("no partition plan set (pcd_set_plan)");
  CK(cudaSetDevice(h->device));
  upload_cache_ref(h, initial_cache, reference);
  CK(cudaStreamSynchronize(h->stream));
  h->resident_valid = true;
  return PCD_OK;
  PCD_CATCH
}

static int fill_limit(pcd_result* res, pcd_trace_row* trace, int64_t trace_cap, const IterationLimit& e) {
  res->iterations_run = e.iterations_run;
  res->trace_rows = (int64_t)e.partial_trace.size();
  for (int64_t i = 0; i < (int64_t)e.partial_trace.size() && i < trace_cap; ++i) trace[i] = e.partial_trace[(size_t)i];
  set_last_error(e.what());
  return PCD_ITERATION_LIMIT;
}

extern "C" int pcd_simulate(pcd_handle* h, const pcd_config* cfg, const int32_t* initial_cache,
                            const int32_t* reference, int32_t* actions_out, pcd_result* res,
                            pcd_trace_row* trace, int64_t trace_cap) {
  pcd_result dummy;
  if (!res) res = &dummy;
  *res = pcd_result{0, -1, 0, 0, 0, 0, 0, -1};
  PCD_TRY
  if (!h || !cfg) throw InvalidArgument("null argument");
  if (!h->have_plan) throw InvalidArgument("no partition plan set (pcd_set_plan)");
  CK(cudaSetDevice(h->device));
  upload_cache_ref(h, initial_cache, reference);
  // a pinned destination receives the committed prefix during the run
  struct DlReset {
    pcd_handle* h;
    ~DlReset() {
      if (h->aux) cudaStreamSynchronize(h->aux);
      h->dl_out = nullptr;
      h->dl_done = 0;
    }
  } dl_guard{h};
  h->dl_done = 0;
  h->dl_out = nullptr;
  if (actions_out && h->T) {
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, actions_out) == cudaSuccess && pa.type == cudaMemoryTypeHost)
      h->dl_out = actions_out;
    cudaGetLastError();
  }
  try {
    simulate(h, cfg, reference != nullptr, res, trace, trace_cap);
  } catch (const IterationLimit& e) {
    return fill_limit(res, trace, trace_cap, e);
  } catch (const ContractViolation& e) {
    res->error_time_step = e.time_step;
    throw;
  }
  const int64_t from = h->dl_out ? h->dl_done : 0;
  if (actions_out && h->T > from)
    CK(cudaMemcpyAsync(actions_out + from, h->cache.p + from, (size_t)(h->T - from) * 4, cudaMemcpyDeviceToHost,
                       h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_simulate_resident(pcd_handle* h, const pcd_config* cfg, int32_t use_initial_cache,
                                     int32_t use_reference, pcd_result* res, pcd_trace_row* trace,
                                     int64_t trace_cap) {
  pcd_result dummy;
  if (!res) res = &dummy;
  *res = pcd_result{0, -1, 0, 0, 0, 0, 0, -1};
  PCD_TRY
  if (!h || !cfg) throw InvalidArgument("null argument");
  if (!h->have_plan) throw InvalidArgument("no partition plan set (pcd_set_plan)");
  CK(cudaSetDevice(h->device));
  ensure_state_buffers(h);
  if (!use_initial_cache)
    k_fill<<<grid_for(h->T, 256), 256, 0, h->stream>>>(h->cache.p, -1, (long long)h->T);
  else if (!h->resident_valid)
    throw InvalidArgument("no resident initial cache (pcd_upload_cache)");
  if (use_reference && !h->ref.n) throw InvalidArgument("no resident reference (pcd_upload_cache)");
  h->resident_valid = false;  // the cache is overwritten by the run
  try {
    simulate(h, cfg, use_reference != 0, res, trace, trace_cap);
  } catch (const IterationLimit& e) {
    return fill_limit(res, trace, trace_cap, e);
  } catch (const ContractViolation& e) {
    res->error_time_step = e.time_step;
    throw;
  }
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_download_actions(pcd_handle* h, int32_t* actions_out) {
  PCD_TRY
  if (!h || !actions_out) throw InvalidArgument("null argument");
  CK(cudaSetDevice(h->device));
  if (h->T) CK(cudaMemcpyAsync(actions_out, h->cache.p, (size_t)h->T * 4, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_iterate_once(pcd_handle* h, int32_t engine, int32_t* cache, int64_t t_lo, int64_t t_hi,
                                const int32_t* ckpt_capacity, const int32_t* ckpt_inventory,
                                int64_t* evals_per_process, int64_t* changed_slots, int64_t* n_changed) {
  PCD_TRY
  if (!h || !cache) throw InvalidArgument("null argument");
  if (!h->have_plan) throw InvalidArgument("no partition plan set (pcd_set_plan)");
  if (t_lo < 0 || t_hi > h->T) throw InvalidArgument("window outside the horizon");
  CK(cudaSetDevice(h->device));
  ensure_state_buffers(h);
  const int eng = choose_engine(h, engine);
  const size_t T = (size_t)h->T;
  std::vector<int32_t> before(cache, cache + T);
  CK(cudaMemcpyAsync(h->cache.p, cache, T * 4, cudaMemcpyHostToDevice, h->stream));
  if (ckpt_capacity) CK(cudaMemcpyAsync(h->ckcap.p, ckpt_capacity, sizeof(int) * h->J, cudaMemcpyHostToDevice, h->stream));
  else CK(cudaMemcpyAsync(h->ckcap.p, h->cap0.p, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
  if (ckpt_inventory) CK(cudaMemcpyAsync(h->ckinv.p, ckpt_inventory, sizeof(int) * (size_t)h->I * h->J, cudaMemcpyHostToDevice, h->stream));
  else CK(cudaMemcpyAsync(h->ckinv.p, h->inv0.p, sizeof(int) * (size_t)h->I * h->J, cudaMemcpyDeviceToDevice, h->stream));
  if (T) CK(cudaMemsetAsync(h->written.p, 0, T, h->stream));
  CK(cudaMemsetAsync(h->evals.p, 0, sizeof(long long) * h->M, h->stream));
  DBuf<int> saved_ref;  // iterate_once has no reference
  std::swap(saved_ref.p, h->ref.p);
  std::swap(saved_ref.n, h->ref.n);
  h->tc_kernel_req = 0;
  try {
    run_iteration(h, eng, t_lo, t_hi, h->evals.p);
  } catch (...) {
    std::swap(saved_ref.p, h->ref.p);
    std::swap(saved_ref.n, h->ref.n);
    throw;
  }
  std::swap(saved_ref.p, h->ref.p);
  std::swap(saved_ref.n, h->ref.n);
  if (T) CK(cudaMemcpyAsync(cache, h->cache.p, T * 4, cudaMemcpyDeviceToHost, h->stream));
  std::vector<long long> ev((size_t)h->M, 0);
  k_window_evals<<<(h->M + 255) / 256, 256, 0, h->stream>>>(h->pstart.p, h->pslots.p, h->M, (int)t_lo,
                                                             (int)t_hi, h->evals.p);
  CK(cudaMemcpyAsync(ev.data(), h->evals.p, sizeof(long long) * h->M, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  if (evals_per_process)
    for (int32_t m = 0; m < h->M; ++m) evals_per_process[m] = ev[(size_t)m];
  int64_t n = 0;
  for (int64_t t = std::max<int64_t>(t_lo, 0); t < t_hi; ++t)
    if (before[(size_t)t] != cache[t]) {
      if (changed_slots) changed_slots[n] = t;
      ++n;
    }
  if (n_changed) *n_changed = n;
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_sequential(pcd_handle* h, int32_t* actions_out, int64_t* policy_evals) {
  PCD_TRY
  if (!h) throw InvalidArgument("handle is null");
  CK(cudaSetDevice(h->device));
  // Prop. 1: the Picard fixed point is the serial trajectory.
  const int32_t M = std::max(1, std::min<int32_t>(h->I, 8192));
  std::vector<int32_t> owner((size_t)h->T);
  std::vector<int32_t> prod((size_t)h->T);
  CK(cudaMemcpy(prod.data(), h->product.p, (size_t)h->T * 4, cudaMemcpyDeviceToHost));
  product_partition(prod.data(), h->T, h->I, M, 1, owner.data());
  // save / restore any user plan
  const bool had = h->have_plan;
  std::vector<int32_t> saved;
  if (had) {
    saved.resize((size_t)h->T);
    if (h->T) CK(cudaMemcpy(saved.data(), h->owner.p, sizeof(int32_t) * (size_t)h->T, cudaMemcpyDeviceToHost));
  }
  const int32_t savedM = h->M;
  int rc = pcd_set_plan(h, owner.data(), M);
  if (rc) return rc;
  pcd_config cfg{0, 0, 0, 0, 1, PCD_ENGINE_PRODUCT};
  pcd_result res;
  rc = pcd_simulate(h, &cfg, nullptr, nullptr, actions_out, &res, nullptr, 0);
  if (rc == PCD_CONTRACT_VIOLATION) {
    // A Picard sweep may evaluate the policy at non-serial states; reproduce
    // the serial error exactly with the single-process fixed point.
    std::vector<int32_t> one((size_t)h->T, 0);
    pcd_set_plan(h, one.data(), 1);
    rc = pcd_simulate(h, &cfg, nullptr, nullptr, actions_out, &res, nullptr, 0);
  }
  if (had) pcd_set_plan(h, saved.data(), savedM);
  if (policy_evals) *policy_evals = h->T;
  return rc;
  PCD_CATCH
}

// time_warp_simulate (fo/timewarp.hpp:56-181). Each window is one sweep of
// the run-partition engine with the cache treated as all-declined (nocache:
// H = 0, so a process sees the synchronized state minus its own decisions),
// then the merge is the checkpoint advance over the window; a merge that
// would go negative is undone and the window re-executed serially.
extern "C" int pcd_time_warp(pcd_handle* h, int32_t processes, uint64_t seed, int32_t rule, int32_t record_trace,
                             int32_t* actions_out, pcd_tw_result* res, pcd_tw_trace_row* trace, int64_t trace_cap) {
  pcd_tw_result dummy;
  if (!res) res = &dummy;
  *res = pcd_tw_result{0, 0, 0, 0, 0, -1};
  PCD_TRY
  if (!h) throw InvalidArgument("handle is null");
  CK(cudaSetDevice(h->device));
  const int64_t T = h->T;
  // the plan: make_product_partition(instance, processes, seed)
  std::vector<int32_t> prod((size_t)std::max<int64_t>(T, 1)), owner((size_t)std::max<int64_t>(T, 1));
  if (T) CK(cudaMemcpy(prod.data(), h->product.p, sizeof(int32_t) * (size_t)T, cudaMemcpyDeviceToHost));
  product_partition(prod.data(), T, h->I, processes, seed, owner.data());
  {
    const int rc = pcd_set_plan(h, owner.data(), processes);
    if (rc) return rc;
  }
  ensure_state_buffers(h);
  const size_t IJ = (size_t)h->I * h->J;
  CK(cudaMemcpyAsync(h->ckcap.p, h->cap0.p, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemcpyAsync(h->ckinv.p, h->inv0.p, sizeof(int) * IJ, cudaMemcpyDeviceToDevice, h->stream));
  if (T) k_fill<<<grid_for(T, 256), 256, 0, h->stream>>>(h->cache.p, -1, (long long)T);
  if (T) CK(cudaMemsetAsync(h->written.p, 0, (size_t)T, h->stream));
  h->ref.release();
  h->timing = pcd_timing{};
  h->nocache = 1;
  struct Reset {
    pcd_handle* h;
    ~Reset() { h->nocache = 0; }
  } reset{h};
  DBuf<long long> derr;
  derr.alloc(2);
  std::vector<int32_t> caps((size_t)h->J);
  std::vector<pcd_tw_trace_row> rows;
  const bool tc = h->tc_ok && h->kind == kDual;
  int64_t t0 = 0;
  while (t0 < T) {
    CK(cudaMemcpyAsync(caps.data(), h->ckcap.p, sizeof(int32_t) * h->J, cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    int64_t delta = 0;
    if (rule == 0) {
      int32_t mc = caps.empty() ? 0 : caps[0];
      for (int32_t c : caps) mc = std::min(mc, c);
      delta = std::max<int64_t>(1, mc);
    } else {
      int32_t ms = 0;
      bool any = false;
      for (int32_t c : caps) {
        if (c <= 0) continue;
        ms = any ? std::min(ms, c) : c;
        any = true;
      }
      delta = any ? std::max<int64_t>(1, ms) : T - t0;
    }
    const int64_t hi = std::min(T, t0 + delta);
    const int lo32 = (int)t0, hi32 = (int)hi;
    // local decisions of every process over the window
    reset_scalars(h);
    k_xinit_plain<<<(h->I * 32 + 255) / 256, 256, 0, h->stream>>>(h->qstart.p, h->qslots.p, h->I, lo32, hi32,
                                                                   h->rid.p, h->ckinv.p, h->J, h->xloc.p);
    if (tc) launch_tc(h, lo32, hi32, nullptr, 0.0, 0);
    else dispatch_kind(h->kind, [&](auto k) { launch_product_sweep<decltype(k)::value>(h, lo32, hi32, nullptr); });
    exchange(h, h->cache.p, true, lo32, hi32);
    read_scalars(h);
    throw_sweep_error(h);
    const int64_t max_evals = (int64_t)h->h_scal->max_evals, sum_evals = (int64_t)h->h_scal->total_evals;
    res->policy_eval_count_sequential_equivalent += max_evals;
    res->total_policy_evals += sum_evals;
    h->timing.kernel_launches += 3;
    // synchronize: apply the merged decisions in time order
    bool merged = true;
    {
      CK(cudaMemcpyAsync(h->ckbak.p, h->ckinv.p, sizeof(int) * IJ, cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaMemcpyAsync(h->ckbak.p + IJ, h->ckcap.p, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaMemsetAsync(&h->scal->neg_flag, 0, sizeof(int), h->stream));
      k_advance<<<grid_for(hi - t0, 256), 256, (size_t)h->J * 4, h->stream>>>(
          h->cache.p, h->product.p, lo32, hi32, h->J, h->ckcap.p, h->ckinv.p, &h->scal->neg_flag);
      int flag = 0;
      CK(cudaMemcpyAsync(&flag, &h->scal->neg_flag, sizeof(int), cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      merged = flag == 0;
    }
    if (!merged) {  // roll back, re-execute the window serially (charged at serial cost)
      CK(cudaMemcpyAsync(h->ckinv.p, h->ckbak.p, sizeof(int) * IJ, cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaMemcpyAsync(h->ckcap.p, h->ckbak.p + IJ, sizeof(int) * h->J, cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaMemsetAsync(derr.p, 0xff, 2 * sizeof(long long), h->stream));
      const size_t smem = ((size_t)2 * h->J * 4 + 15 & ~(size_t)15) +
                          (size_t)(2 * h->J + 1 + 2 * h->H + 2 * h->J) * 8;
      dispatch_kind(h->kind, [&](auto k) {
        k_serial_window<decltype(k)::value><<<1, 32, smem, h->stream>>>(h->model(), lo32, hi32, h->ckcap.p,
                                                                          h->ckinv.p, h->cache.p, derr.p);
      });
      CK(cudaGetLastError());
      long long e[2];
      CK(cudaMemcpyAsync(e, derr.p, sizeof e, cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      if (e[1] == 2) throw ContractViolation("dual network produced a non-finite score", e[0]);
      if (e[1] == 1)
        throw ContractViolation("policy returned an infeasible action at t=" + std::to_string(e[0]), e[0]);
      res->rollbacks += 1;
      res->policy_eval_count_sequential_equivalent += hi - t0;
      res->total_policy_evals += hi - t0;
    }
    res->sync_rounds += 1;
    if (record_trace) rows.push_back({res->sync_rounds, t0, hi - t0, max_evals, merged ? 0 : 1, 0});
    t0 = hi;
  }
  if (actions_out && T)
    CK(cudaMemcpyAsync(actions_out, h->cache.p, sizeof(int32_t) * (size_t)T, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  res->trace_rows = (int64_t)rows.size();
  for (int64_t i = 0; i < (int64_t)rows.size() && i < trace_cap; ++i) trace[i] = rows[(size_t)i];
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_depletion_profile(pcd_handle* h, const int32_t* actions, int64_t* first_depleted_at,
                                     int64_t* depleted_count) {
  PCD_TRY
  if (!h || !first_depleted_at) throw InvalidArgument("null argument");
  CK(cudaSetDevice(h->device));
  const int64_t T = h->T;
  const int J = h->J;
  DBuf<int> acts, keys, start, slots;
  DBuf<long long> out;
  out.alloc(std::max(1, J));
  const int* a = h->cache.p;
  if (actions) {
    acts.upload(actions, (size_t)std::max<int64_t>(T, 1), h->stream);
    a = acts.p;
  } else if (!h->cache.p) {
    throw InvalidArgument("no resident trajectory (run pcd_simulate first or pass actions)");
  }
  if (T > 0) {
    keys.alloc((size_t)T);
    k_fulfil_keys<<<grid_for(T, 256), 256, 0, h->stream>>>(a, T, J, keys.p);
    build_csr(h, keys.p, J + 1, start, slots);
  } else {
    start.alloc((size_t)J + 2);
    CK(cudaMemsetAsync(start.p, 0, sizeof(int) * ((size_t)J + 2), h->stream));
    slots.alloc(1);
  }
  k_depletion<<<(J + 127) / 128, 128, 0, h->stream>>>(start.p, slots.p, h->cap0.p, J, T, out.p);
  CK(cudaGetLastError());
  std::vector<long long> d((size_t)J);
  CK(cudaMemcpyAsync(d.data(), out.p, sizeof(long long) * (size_t)J, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  int64_t cnt = 0;
  for (int j = 0; j < J; ++j) {
    first_depleted_at[j] = d[(size_t)j];
    cnt += d[(size_t)j] < T;
  }
  if (depleted_count) *depleted_count = cnt;
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_checkpoint_state(pcd_handle* h, int32_t* capacity, int32_t* inventory) {
  PCD_TRY
  if (!h || !capacity || !inventory) throw InvalidArgument("null argument");
  if (!h->ckcap.p) throw InvalidArgument("no simulation has run on this handle");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(capacity, h->ckcap.p, sizeof(int32_t) * (size_t)h->J, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(inventory, h->ckinv.p, sizeof(int32_t) * (size_t)h->I * h->J, cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_set_history(pcd_handle* h, int32_t* history, int64_t cap_iterations) {
  if (!h) return PCD_INVALID_ARGUMENT;
  h->history = history;
  h->history_cap = history ? cap_iterations : 0;
  return PCD_OK;
}

extern "C" int pcd_set_debug(pcd_handle* h, int32_t flags) {
  if (!h) return PCD_INVALID_ARGUMENT;
  h->debug = flags;
  return PCD_OK;
}

extern "C" int pcd_last_timing(const pcd_handle* h, pcd_timing* out) {
  if (!h || !out) return PCD_INVALID_ARGUMENT;
  *out = h->timing;
  return PCD_OK;
}

extern "C" int pcd_picard_simulate(const pcd_instance* inst, const pcd_policy* policy, const int32_t* owner,
                                   int32_t processes, const pcd_config* cfg, const int32_t* initial_cache,
                                   const int32_t* reference, int32_t* actions_out, pcd_result* result,
                                   pcd_trace_row* trace, int64_t trace_cap) {
  pcd_handle* h = nullptr;
  int rc = pcd_create(inst, policy, 0, &h);
  if (rc) return rc;
  rc = pcd_set_plan(h, owner, processes);
  if (rc == PCD_OK) rc = pcd_simulate(h, cfg, initial_cache, reference, actions_out, result, trace, trace_cap);
  pcd_destroy(h);
  return rc;
}

extern "C" int pcd_nccl_unique_id(unsigned char out[128]) {
  PCD_TRY
  if (!g_nccl.load()) throw CudaError("libnccl.so.2 could not be loaded");
  nccl_unique_id id;
  const int rc = g_nccl.GetUniqueId(&id);
  if (rc != 0) throw CudaError(std::string("ncclGetUniqueId failed: ") + g_nccl.GetErrorString(rc));
  std::memcpy(out, id.internal, 128);
  return PCD_OK;
  PCD_CATCH
}

extern "C" int pcd_attach_comm(pcd_handle* h, const unsigned char id[128], int32_t rank, int32_t nranks) {
  PCD_TRY
  if (!h) throw InvalidArgument("handle is null");
  if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("bad rank / nranks");
  if (!g_nccl.load()) throw CudaError("libnccl.so.2 could not be loaded");
  CK(cudaSetDevice(h->device));
  nccl_unique_id uid;
  std::memcpy(uid.internal, id, 128);
  auto c = std::make_unique<NcclComm>();
  const int rc = g_nccl.CommInitRank(&c->c, nranks, uid, rank);
  if (rc != 0) throw CudaError(std::string("ncclCommInitRank failed: ") + g_nccl.GetErrorString(rc));
  h->comm = std::move(c);
  h->rank = rank;
  h->nranks = nranks;
  rebuild_shards(h);
  return PCD_OK;
  PCD_CATCH
}

// ------------------------------------------------ in-process loopback group
struct pcd_loopback {
  std::shared_ptr<pcd::LoopbackGroup> g;
};

extern "C" pcd_loopback* pcd_loopback_create(int32_t nranks) {
  if (nranks < 1 || nranks > kMaxRanks) {
    set_last_error("loopback group: nranks out of range");
    return nullptr;
  }
  auto* l = new pcd_loopback;
  l->g = std::make_shared<pcd::LoopbackGroup>(nranks);
  return l;
}

extern "C" void pcd_loopback_destroy(pcd_loopback* l) { delete l; }

extern "C" int pcd_attach_loopback(pcd_handle* h, pcd_loopback* l, int32_t rank) {
  PCD_TRY
  if (!h || !l) throw InvalidArgument("null argument");
  if (rank < 0 || rank >= l->g->n) throw InvalidArgument("bad rank");
  CK(cudaSetDevice(h->device));
  auto c = std::make_unique<LoopbackComm>();
  c->g = l->g;
  c->rank = rank;
  h->comm = std::move(c);
  h->rank = rank;
  h->nranks = l->g->n;
  rebuild_shards(h);
  return PCD_OK;
  PCD_CATCH
}
