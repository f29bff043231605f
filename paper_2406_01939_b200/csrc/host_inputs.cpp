// host_inputs.cpp — host-side inputs of the B200 Picard engine.
//
// Instance generation, partitioners and seeded MLP parameters are driven by
// serial mt19937_64 streams, so they stay on the host and must reproduce the
// reference's streams bit for bit:
//   generate_instance        instance.cpp:80-140 (+ geometry.cpp, rng.hpp)
//   make_product_partition   instance.cpp:142-186
//   make_uniform_time_partition engine.hpp:99-114
//   MlpParams::seeded_uniform mlp.cpp:117-129
// The synthetic J>30 geometry is the SURVEY.md §8(d) extension.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <queue>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_internal.h"

namespace pcd {

namespace {

using Engine = std::mt19937_64;  // bit-specified by the standard (rng.hpp:14)

uint64_t below(Engine& g, uint64_t n) {  // rng.hpp:41-49
  if (n <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t v;
  do { v = g(); } while (v >= limit);
  return v % n;
}
double unit(Engine& g) { return static_cast<double>(g() >> 11) * 0x1.0p-53; }  // rng.hpp:52-54
double range(Engine& g, double lo, double hi) { return lo + (hi - lo) * unit(g); }

template <typename T>
void shuffle(T* v, size_t n, Engine& g) {  // rng.hpp:60-66 (Fisher-Yates, top down)
  for (size_t i = n; i > 1; --i) std::swap(v[i - 1], v[(size_t)below(g, i)]);
}

std::vector<int64_t> apportion(const std::vector<double>& w, int64_t total) {
  const size_t n = w.size();
  std::vector<int64_t> out(n, 0);
  if (n == 0 || total <= 0) return out;
  double sum = 0.0;
  for (double x : w) {
    if (!(x >= 0.0)) throw InvalidArgument("apportion weights must be non-negative");
    sum += x;
  }
  if (!(sum > 0.0)) throw InvalidArgument("apportion weights must not all be zero");
  std::vector<double> frac(n);
  int64_t assigned = 0;
  for (size_t i = 0; i < n; ++i) {
    const double share = static_cast<double>(total) * w[i] / sum;
    out[i] = static_cast<int64_t>(std::floor(share));
    frac[i] = share - static_cast<double>(out[i]);
    assigned += out[i];
  }
  std::vector<size_t> order(n);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return frac[a] > frac[b]; });
  for (int64_t r = 0; r < total - assigned; ++r) out[order[(size_t)r]] += 1;
  return out;
}

// Largest city per state, 30 most populous U.S. states (geometry.cpp:15-46).
constexpr double kLat[30] = {34.05, 29.76, 30.33, 40.71, 39.95, 41.88, 39.96, 33.75, 35.23, 42.33,
                             40.74, 36.85, 47.61, 33.45, 42.36, 36.16, 39.77, 39.29, 39.10, 43.04,
                             39.74, 44.98, 32.78, 33.52, 29.95, 38.25, 45.52, 35.47, 41.19, 40.76};
constexpr double kLon[30] = {-118.24, -95.37, -81.66, -74.01,  -75.17,  -87.63, -83.00, -84.39,
                             -80.84,  -83.05, -74.17, -75.98,  -122.33, -112.07, -71.06, -86.78,
                             -86.16,  -76.61, -94.58, -87.91,  -104.99, -93.27, -79.93, -86.81,
                             -90.07,  -85.76, -122.68, -97.52, -73.20,  -111.89};
constexpr double kPop[30] = {39.54e6, 29.15e6, 21.54e6, 20.20e6, 13.00e6, 12.81e6, 11.80e6, 10.71e6,
                             10.44e6, 10.08e6, 9.29e6,  8.63e6,  7.71e6,  7.15e6,  7.03e6,  6.91e6,
                             6.79e6,  6.18e6,  6.15e6,  5.89e6,  5.77e6,  5.71e6,  5.12e6,  5.02e6,
                             4.66e6,  4.51e6,  4.24e6,  3.96e6,  3.61e6,  3.27e6};

double great_circle_km(double la, double lo_a, double lb, double lo_b) {  // geometry.cpp:52-61
  constexpr double kPi = 3.14159265358979323846;
  const double pa = la * kPi / 180.0, pb = lb * kPi / 180.0;
  const double dp = (lb - la) * kPi / 180.0, dl = (lo_b - lo_a) * kPi / 180.0;
  const double s = std::sin(dp / 2.0), t = std::sin(dl / 2.0);
  const double h = s * s + std::cos(pa) * std::cos(pb) * t * t;
  return 2.0 * 6371.0 * std::asin(std::sqrt(std::min(1.0, h)));
}

struct Geometry {
  int32_t n;
  std::vector<double> pop, dist;
};

Geometry make_geometry(int32_t J, int32_t kind) {
  if (kind == 0 && (J < 1 || J > 30))
    throw InvalidArgument("node count must be in [1, 30]");
  if (J < 1) throw InvalidArgument("geometry needs at least one node");
  std::vector<double> lat(J), lon(J);
  Geometry g{J, std::vector<double>(J), std::vector<double>((size_t)J * J, 0.0)};
  if (kind == 0) {
    for (int32_t j = 0; j < J; ++j) { lat[j] = kLat[j]; lon[j] = kLon[j]; g.pop[j] = kPop[j]; }
  } else {
    Engine gen(12345);
    for (int32_t j = 0; j < J; ++j) {
      lat[j] = range(gen, 25.0, 49.0);
      lon[j] = range(gen, -124.0, -67.0);
      g.pop[j] = range(gen, 1e6, 4e7);
    }
  }
  for (int32_t a = 0; a < J; ++a)
    for (int32_t b = a + 1; b < J; ++b) {
      const double d = great_circle_km(lat[a], lon[a], lat[b], lon[b]);
      g.dist[(size_t)a * J + b] = d;
      g.dist[(size_t)b * J + a] = d;
    }
  return g;
}

void reward_vector(const Geometry& g, int32_t origin, double* out) {  // geometry.cpp:104-128
  const double* d = g.dist.data() + (size_t)origin * g.n;
  double max_d = 0.0;
  for (int32_t j = 0; j < g.n; ++j) max_d = std::max(max_d, d[j]);
  for (int32_t j = 0; j < g.n; ++j) out[j] = 1.0;
  if (max_d <= 0.0) return;
  for (int32_t j = 0; j < g.n; ++j) out[j] = std::round((max_d - d[j]) / max_d * 1e9) / 1e9;
}

}  // namespace

void generate_instance(int32_t J, int32_t I, int64_t T, double beta, double coverage,
                       uint64_t seed, int32_t geometry, int32_t* product, int32_t* origin,
                       double* reward_table, int32_t* capacity, int32_t* inventory) {
  if (I < 1) throw InvalidArgument("product count must be >= 1");
  if (T < 1) throw InvalidArgument("horizon must be >= 1");
  if (!(coverage > 0.0 && coverage <= 1.0)) throw InvalidArgument("coverage must be in (0, 1]");
  if (!(beta <= 0.0 && beta >= -8.0)) throw InvalidArgument("beta must be in [-8, 0]");
  const Geometry g = make_geometry(J, geometry);
  // demand_counts (instance.cpp:67-78)
  std::vector<double> w(I);
  for (int32_t i = 0; i < I; ++i) w[i] = std::pow(static_cast<double>(i + 1), -std::abs(beta));
  const auto counts = apportion(w, T);
  for (int32_t j = 0; j < J; ++j) reward_vector(g, j, reward_table + (size_t)j * J);
  Engine gen(seed);
  std::vector<double> cum(J);
  double tot = 0.0;
  for (int32_t j = 0; j < J; ++j) cum[j] = (tot += g.pop[j]);
  // Orders in product order, origin by WeightedSampler (rng.hpp:70-96),
  // then one Fisher-Yates shuffle of the (product, origin) records.
  struct Rec { int32_t product, origin; };
  std::vector<Rec> recs;
  recs.reserve((size_t)T);
  for (int32_t i = 0; i < I; ++i)
    for (int64_t q = 0; q < counts[(size_t)i]; ++q) {
      const double u = unit(gen) * cum.back();
      int32_t lo = 0, hi = J - 1;
      while (lo < hi) {
        const int32_t mid = (lo + hi) / 2;
        if (cum[mid] <= u) lo = mid + 1; else hi = mid;
      }
      recs.push_back({i, lo});
    }
  shuffle(recs.data(), recs.size(), gen);
  for (int64_t t = 0; t < T; ++t) { product[t] = recs[(size_t)t].product; origin[t] = recs[(size_t)t].origin; }
  const auto cap = apportion(g.pop, std::llround(coverage * static_cast<double>(T)));
  for (int32_t j = 0; j < J; ++j) capacity[j] = static_cast<int32_t>(cap[(size_t)j]);
  std::memset(inventory, 0, sizeof(int32_t) * (size_t)I * J);
  for (int32_t i = 0; i < I; ++i) {
    const int64_t units = std::llround(coverage * static_cast<double>(counts[(size_t)i]));
    if (units <= 0) continue;
    const auto row = apportion(g.pop, units);
    for (int32_t j = 0; j < J; ++j) inventory[(size_t)i * J + j] = static_cast<int32_t>(row[(size_t)j]);
  }
}

void product_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, uint64_t seed,
                       int32_t* owner) {
  if (M < 1) throw InvalidArgument("process count must be >= 1");
  std::vector<int64_t> counts((size_t)I, 0);
  for (int64_t t = 0; t < T; ++t) counts[(size_t)product[t]] += 1;
  std::vector<int32_t> order((size_t)I);
  std::iota(order.begin(), order.end(), 0);
  Engine gen(seed);
  shuffle(order.data(), order.size(), gen);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return counts[(size_t)a] > counts[(size_t)b]; });
  using Load = std::pair<int64_t, int32_t>;
  std::priority_queue<Load, std::vector<Load>, std::greater<>> lightest;
  for (int32_t g = 0; g < M; ++g) lightest.emplace(0, g);
  std::vector<int32_t> group_of((size_t)I, 0);
  for (int32_t p : order) {
    auto [load, group] = lightest.top();
    lightest.pop();
    group_of[(size_t)p] = group;
    lightest.emplace(load + counts[(size_t)p], group);
  }
  for (int64_t t = 0; t < T; ++t) owner[t] = group_of[(size_t)product[t]];
}

// Product-chunk partition (ours; no reference counterpart): every product's
// orders, in time order, are cut into k_i = ceil(Q_i / L) contiguous chunks of
// near-equal size, one process per chunk, with L the smallest chunk length for
// which sum_i k_i <= M. A run partition (engine.cu: k_check_runs), so the
// closed-form engines apply; with M >= I it spreads the window over up to M
// processes instead of I. Falls back to make_product_partition when M is
// below the number of ordered products.
void product_chunk_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, uint64_t seed,
                             int32_t* owner) {
  if (M < 1) throw InvalidArgument("process count must be >= 1");
  std::vector<int64_t> counts((size_t)I, 0);
  for (int64_t t = 0; t < T; ++t) counts[(size_t)product[t]] += 1;
  int64_t used = 0, qmax = 0;
  for (int64_t q : counts) {
    used += q > 0;
    qmax = std::max(qmax, q);
  }
  if (used > M || T == 0) return product_partition(product, T, I, M, seed, owner);
  auto chunks = [&](int64_t L) {
    int64_t k = 0;
    for (int64_t q : counts) k += (q + L - 1) / L;
    return k;
  };
  int64_t lo = 1, hi = qmax;  // chunks(qmax) = used <= M
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (chunks(mid) <= M) hi = mid; else lo = mid + 1;
  }
  const int64_t L = lo;
  std::vector<int32_t> first((size_t)I, 0);  // first process of each product
  std::vector<int64_t> seen((size_t)I, 0);
  int32_t next = 0;
  for (int32_t i = 0; i < I; ++i) {
    first[(size_t)i] = next;
    next += (int32_t)((counts[(size_t)i] + L - 1) / L);
  }
  for (int64_t t = 0; t < T; ++t) {
    const int32_t i = product[t];
    const int64_t q = counts[(size_t)i], k = (q + L - 1) / L, c = seen[(size_t)i]++;
    // chunk c' holds ranks [floor(c' q / k), floor((c'+1) q / k))
    owner[t] = first[(size_t)i] + (int32_t)(((c + 1) * k - 1) / q);
  }
}

// Window-aware product chunks (ours; no reference counterpart). A Picard
// iteration's critical path is its busiest process's own slots inside the
// window [ws, ws + W) (engine.hpp:120-126, max_steps = W), so cutting a
// product whose orders are sparse in time buys nothing, while a product with a
// dense stretch bounds every window. Each product's orders, in time order,
// are cut greedily: a chunk grows while no W-long interval holds more than L
// of its orders (checked at every new order against the chunk's orders in
// (t - W, t]); greedy is minimal per product since the constraint holds for
// every sub-run of a valid chunk. L is the smallest bound with at most M
// chunks in total, so every window's per-process chain is <= L. W <= 0 or
// W >= T: the whole horizon is one window (chunks of at most L orders).
// Falls back to make_product_partition when M is below the ordered products.
void product_window_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, int64_t W,
                              uint64_t seed, int32_t* owner) {
  if (M < 1) throw InvalidArgument("process count must be >= 1");
  if (W <= 0 || W > T) W = T;
  std::vector<int64_t> start((size_t)I + 1, 0);
  for (int64_t t = 0; t < T; ++t) start[(size_t)product[t] + 1] += 1;
  int64_t used = 0, qmax = 0;
  for (int32_t i = 0; i < I; ++i) {
    used += start[(size_t)i + 1] > 0;
    qmax = std::max(qmax, start[(size_t)i + 1]);
    start[(size_t)i + 1] += start[(size_t)i];
  }
  if (used > M || T == 0) return product_partition(product, T, I, M, seed, owner);
  std::vector<int64_t> ts((size_t)T);  // each product's order times, ascending
  {
    std::vector<int64_t> fill(start.begin(), start.end() - 1);
    for (int64_t t = 0; t < T; ++t) ts[(size_t)fill[(size_t)product[t]]++] = t;
  }
  // chunks of product i under bound L; cut[] (optional) receives each chunk's
  // first rank within the product
  auto cut_product = [&](int32_t i, int64_t L, std::vector<int64_t>* cut) {
    const int64_t* a = ts.data() + start[(size_t)i];
    const int64_t q = start[(size_t)i + 1] - start[(size_t)i];
    int64_t n = q > 0, k0 = 0, j = 0;  // j: first rank with time > a[k] - W
    if (cut && q > 0) cut->push_back(0);
    for (int64_t k = 0; k < q; ++k) {
      while (a[j] <= a[k] - W) ++j;
      if (k - std::max(k0, j) + 1 > L) {
        k0 = k;
        ++n;
        if (cut) cut->push_back(k);
      }
    }
    return n;
  };
  auto chunks = [&](int64_t L) {
    int64_t k = 0;
    for (int32_t i = 0; i < I && k <= M; ++i) k += cut_product(i, L, nullptr);
    return k;
  };
  int64_t lo = 1, hi = qmax;  // chunks(qmax) = used <= M
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (chunks(mid) <= M) hi = mid; else lo = mid + 1;
  }
  int32_t next = 0;
  std::vector<int64_t> cut;
  for (int32_t i = 0; i < I; ++i) {
    cut.clear();
    cut_product(i, lo, &cut);
    const int64_t b = start[(size_t)i], q = start[(size_t)i + 1] - b;
    size_t c = 0;
    for (int64_t k = 0; k < q; ++k) {
      while (c + 1 < cut.size() && cut[c + 1] <= k) ++c;
      owner[ts[(size_t)(b + k)]] = next + (int32_t)c;
    }
    next += (int32_t)cut.size();
  }
}

void uniform_partition(int64_t T, int32_t M, uint64_t seed, int32_t* owner) {
  if (M < 1) throw ContractViolation("uniform partition: process count must be >= 1");
  Engine gen(seed);
  for (int64_t t = 0; t < T; ++t) owner[t] = static_cast<int32_t>(below(gen, (uint64_t)M));
}

// ---------------------------------------------------------------- linear env
namespace {
// spectral_norm (linear.cpp:68-98): 200 power iterations on M^T M
double lin_spectral_norm(const double* m, int rows, int cols) {
  const size_t r = (size_t)rows, c = (size_t)cols;
  std::vector<double> v(c, 1.0 / std::sqrt(static_cast<double>(c)));
  std::vector<double> mv(r, 0.0), mtmv(c, 0.0);
  auto norm2 = [](const std::vector<double>& x) {
    double acc = 0.0;
    for (double e : x) acc += e * e;
    return std::sqrt(acc);
  };
  double sigma = 0.0;
  for (int iter = 0; iter < 200; ++iter) {
    for (size_t i = 0; i < r; ++i) {
      double acc = 0.0;
      for (size_t j = 0; j < c; ++j) acc += m[i * c + j] * v[j];
      mv[i] = acc;
    }
    const double mv_norm = norm2(mv);
    if (mv_norm < 1e-300) return 0.0;
    std::fill(mtmv.begin(), mtmv.end(), 0.0);
    for (size_t i = 0; i < r; ++i)
      for (size_t j = 0; j < c; ++j) mtmv[j] += m[i * c + j] * mv[i];
    const double mtmv_norm = norm2(mtmv);
    if (mtmv_norm < 1e-300) return mv_norm;
    for (size_t j = 0; j < c; ++j) v[j] = mtmv[j] / mtmv_norm;
    sigma = mv_norm;
  }
  return sigma;
}
}  // namespace

// make_contractive_spec (linear.cpp:126-218) and closed_loop_contraction
// (linear.cpp:100-117), in the reference's operation order.
void linear_contractive_spec(int32_t n_, int32_t p_, int64_t T, double rho, uint64_t seed, double coupling,
                             double* A, double* B, double* W, double* G, double* contraction) {
  if (rho <= 0.0) throw ContractViolation("rho must be positive");
  if (coupling < 0.0 || coupling >= 1.0) throw ContractViolation("state_coupling must be in [0, 1)");
  if (n_ < 1 || p_ < 1 || T < 0) throw ContractViolation("linear spec: dimensions must be positive");
  const size_t n = (size_t)n_, p = (size_t)p_;
  Engine gen(seed);
  for (size_t i = 0; i < p * n; ++i) G[i] = range(gen, -1.0, 1.0);
  std::vector<double> a(n * n), b(n * p), bg(n * n), closed(n * n);
  for (int64_t t = 0; t < T; ++t) {
    std::fill(a.begin(), a.end(), 0.0);
    if (coupling > 0.0) {
      for (auto& x : a) x = range(gen, -1.0, 1.0);
      const double norm = lin_spectral_norm(a.data(), n_, n_);
      const double target = coupling * rho;
      for (auto& x : a) x *= norm > 0.0 ? target / norm : 0.0;
    }
    for (auto& x : b) x = range(gen, -1.0, 1.0);
    for (size_t r = 0; r < n; ++r)
      for (size_t c = 0; c < n; ++c) {
        double acc = 0.0;
        for (size_t k = 0; k < p; ++k) acc += b[r * p + k] * G[k * n + c];
        bg[r * n + c] = acc;
      }
    const double bg_norm = lin_spectral_norm(bg.data(), n_, n_);
    if (bg_norm < 1e-12) throw ContractViolation("degenerate random draw: B_t G is zero");
    double scale;
    if (coupling == 0.0) {
      scale = rho / bg_norm;
    } else {
      auto closed_norm = [&](double s) {
        for (size_t i = 0; i < n * n; ++i) closed[i] = a[i] + s * bg[i];
        return lin_spectral_norm(closed.data(), n_, n_);
      };
      double lo = 0.0, hi = (rho + coupling * rho + 1.0) / bg_norm;
      while (closed_norm(hi) < rho) hi *= 2.0;
      for (int iter = 0; iter < 120; ++iter) {
        const double mid = 0.5 * (lo + hi);
        (closed_norm(mid) < rho ? lo : hi) = mid;
      }
      scale = 0.5 * (lo + hi);
    }
    for (auto& x : b) x *= scale;
    std::copy(a.begin(), a.end(), A + (size_t)t * n * n);
    std::copy(b.begin(), b.end(), B + (size_t)t * n * p);
    for (size_t i = 0; i < n; ++i) W[(size_t)t * n + i] = range(gen, -1.0, 1.0);
  }
  double worst = 0.0;
  for (int64_t t = 0; t < T; ++t) {
    for (size_t r = 0; r < n; ++r)
      for (size_t c = 0; c < n; ++c) {
        double acc = A[(size_t)t * n * n + r * n + c];
        for (size_t k = 0; k < p; ++k) acc += B[(size_t)t * n * p + r * p + k] * G[k * n + c];
        closed[r * n + c] = acc;
      }
    worst = std::max(worst, lin_spectral_norm(closed.data(), n_, n_));
  }
  *contraction = worst;
}

void seeded_mlp(int32_t in, int32_t out, uint64_t seed, int32_t h, double* w1, double* b1,
                double* w2, double* b2, double* w3, double* b3) {
  Engine gen(seed);
  auto fill = [&](double* p, int64_t n) { for (int64_t i = 0; i < n; ++i) p[i] = range(gen, -0.1, 0.1); };
  fill(w1, (int64_t)h * in);
  fill(b1, h);
  fill(w2, (int64_t)h * h);
  fill(b2, h);
  fill(w3, (int64_t)out * h);
  fill(b3, out);
}

// LPT of per-process loads onto `ranks` shards (heaviest first, lightest
// shard, ties -> lower index), so every rank gets a balanced share of the
// critical-path work.
void shard_processes(const int32_t* owner, int64_t T, int32_t M, int32_t ranks, int32_t* rank_of) {
  if (ranks < 1) throw InvalidArgument("ranks must be >= 1");
  std::vector<int64_t> load((size_t)M, 0);
  for (int64_t t = 0; t < T; ++t) load[(size_t)owner[t]] += 1;
  std::vector<int32_t> order((size_t)M);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return load[(size_t)a] > load[(size_t)b]; });
  using Load = std::pair<int64_t, int32_t>;
  std::priority_queue<Load, std::vector<Load>, std::greater<>> q;
  for (int32_t r = 0; r < ranks; ++r) q.emplace(0, r);
  for (int32_t m : order) {
    auto [l, r] = q.top();
    q.pop();
    rank_of[(size_t)m] = r;
    q.emplace(l + load[(size_t)m], r);
  }
}

}  // namespace pcd
