/*
 * picard_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference's hot path (arXiv 2406.01939 artifact,
 * /root/reference/proj), used as the CPU checker for the B200 engine. It is
 * pinned against (a) the golden vectors / known-answer tests of the reference
 * test suite (tests/golden, tests/test_oracle.py) and (b) the unmodified
 * reference library built into oracle/_ref (ref_harness.cpp). Only tests/,
 * __graft_entry__.smoke() and bench.py's CPU legs may load it; the product
 * path (paper_2406_01939_b200) never does.
 *
 * Every function cites the reference file:line it restates.
 */
#define _GNU_SOURCE
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "glibc_tanh.h"
#include "oracle.h"

/* ------------------------------------------------------------------ errors */
static __thread char g_err[512];
static void set_err(const char* s) { snprintf(g_err, sizeof g_err, "%s", s); }
const char* orc_last_error(void) { return g_err; }

enum { OK = 0, INVALID = 1, CONTRACT = 2, ITERLIMIT = 3 };

/* ------------------------------------------------- mt19937_64 (rng.hpp:14) */
/* std::mt19937_64 is bit-specified by the C++ standard [rand.predef]. */
typedef struct { uint64_t mt[312]; int idx; } mt64;

static void mt_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

/* rng::below (rng.hpp:41-49): rejection sampling, then modulo. */
static uint64_t rng_below(mt64* g, uint64_t n) {
  if (n <= 1) return 0;
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t v;
  do { v = mt_next(g); } while (v >= limit);
  return v % n;
}
/* rng::unit (rng.hpp:52-54) and rng::range (:56-58). */
static double rng_unit(mt64* g) { return (double)(mt_next(g) >> 11) * 0x1.0p-53; }
static double rng_range(mt64* g, double lo, double hi) { return lo + (hi - lo) * rng_unit(g); }

/* ----------------------------------------------------------- tanh (libm) */
static int g_tanh_fma = -1;
static int tanh_fma(void) {
  if (g_tanh_fma < 0) {
#if defined(__x86_64__)
    __builtin_cpu_init();
    g_tanh_fma = (__builtin_cpu_supports("fma") && __builtin_cpu_supports("avx2")) ? 1 : 0;
#else
    g_tanh_fma = 1;
#endif
  }
  return g_tanh_fma;
}
void orc_set_tanh_variant(int fma) { g_tanh_fma = fma ? 1 : 0; }
int orc_tanh_variant(void) { return tanh_fma(); }
double orc_tanh(double x) { return gt_tanh(x, 1); }
double orc_tanh_nofma(double x) { return gt_tanh(x, 0); }
double orc_expm1(double x) { return gt_expm1(x, 1); }
double orc_expm1_nofma(double x) { return gt_expm1(x, 0); }

/* ---------------------------------------------- instance generation inputs */
/* largest_remainder_apportion (instance.cpp:34-65). */
static int apportion(const double* w, int64_t n, int64_t total, int64_t* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = 0;
  if (n == 0 || total <= 0) return OK;
  double sum = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    if (!(w[i] >= 0.0)) { set_err("apportion weights must be non-negative"); return INVALID; }
    sum += w[i];
  }
  if (!(sum > 0.0)) { set_err("apportion weights must not all be zero"); return INVALID; }
  double* frac = (double*)malloc(sizeof(double) * (size_t)n);
  int64_t* order = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t assigned = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double share = (double)total * w[i] / sum;
    out[i] = (int64_t)floor(share);
    frac[i] = share - (double)out[i];
    assigned += out[i];
  }
  /* stable sort of indices by fraction descending (insertion/merge keeps
   * ties in index order, as std::stable_sort does). */
  for (int64_t i = 0; i < n; ++i) order[i] = i;
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t width = 1; width < n; width *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * width) {
      int64_t mid = lo + width < n ? lo + width : n;
      int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
      int64_t a = lo, b = mid, k = lo;
      while (a < mid && b < hi) {
        if (frac[order[b]] > frac[order[a]]) tmp[k++] = order[b++];
        else tmp[k++] = order[a++];
      }
      while (a < mid) tmp[k++] = order[a++];
      while (b < hi) tmp[k++] = order[b++];
    }
    memcpy(order, tmp, sizeof(int64_t) * (size_t)n);
  }
  for (int64_t r = 0; r < total - assigned; ++r) out[order[r]] += 1;
  free(tmp); free(order); free(frac);
  return OK;
}
int orc_apportion(const double* w, int64_t n, int64_t total, int64_t* out) {
  return apportion(w, n, total, out);
}

/* demand_counts (instance.cpp:67-78). */
int orc_demand_counts(int32_t products, int64_t horizon, double beta, int64_t* out) {
  if (products < 1) { set_err("product count must be >= 1"); return INVALID; }
  if (horizon < 0) { set_err("horizon must be non-negative"); return INVALID; }
  const double e = fabs(beta);
  double* w = (double*)malloc(sizeof(double) * (size_t)products);
  for (int32_t i = 0; i < products; ++i) w[i] = pow((double)(i + 1), -e);
  int rc = apportion(w, products, horizon, out);
  free(w);
  return rc;
}

/* The 30-city table of default_geometry (geometry.cpp:15-46): latitude,
 * longitude, state population (data restated, ordered by population). */
static const double kLat[30] = {34.05, 29.76, 30.33, 40.71, 39.95, 41.88, 39.96, 33.75, 35.23, 42.33,
                                40.74, 36.85, 47.61, 33.45, 42.36, 36.16, 39.77, 39.29, 39.10, 43.04,
                                39.74, 44.98, 32.78, 33.52, 29.95, 38.25, 45.52, 35.47, 41.19, 40.76};
static const double kLon[30] = {-118.24, -95.37, -81.66, -74.01,  -75.17, -87.63, -83.00, -84.39,
                                -80.84,  -83.05, -74.17, -75.98,  -122.33, -112.07, -71.06, -86.78,
                                -86.16,  -76.61, -94.58, -87.91,  -104.99, -93.27, -79.93, -86.81,
                                -90.07,  -85.76, -122.68, -97.52, -73.20,  -111.89};
static const double kPop[30] = {39.54e6, 29.15e6, 21.54e6, 20.20e6, 13.00e6, 12.81e6, 11.80e6, 10.71e6,
                                10.44e6, 10.08e6, 9.29e6,  8.63e6,  7.71e6,  7.15e6,  7.03e6,  6.91e6,
                                6.79e6,  6.18e6,  6.15e6,  5.89e6,  5.77e6,  5.71e6,  5.12e6,  5.02e6,
                                4.66e6,  4.51e6,  4.24e6,  3.96e6,  3.61e6,  3.27e6};

/* great_circle_km (geometry.cpp:52-61). */
static double great_circle_km(double lat_a, double lon_a, double lat_b, double lon_b) {
  const double kPi = 3.14159265358979323846;
  const double phi_a = lat_a * kPi / 180.0;
  const double phi_b = lat_b * kPi / 180.0;
  const double d_phi = (lat_b - lat_a) * kPi / 180.0;
  const double d_lambda = (lon_b - lon_a) * kPi / 180.0;
  const double s = sin(d_phi / 2.0);
  const double t = sin(d_lambda / 2.0);
  const double h = s * s + cos(phi_a) * cos(phi_b) * t * t;
  return 2.0 * 6371.0 * asin(sqrt(h < 1.0 ? h : 1.0));
}

typedef struct { int32_t n; double* lat; double* lon; double* pop; double* dist; } geometry_t;

static void geometry_free(geometry_t* g) { free(g->lat); free(g->lon); free(g->pop); free(g->dist); }

/* NetworkGeometry ctor (geometry.cpp:63-82) over either the city table
 * (default_geometry, :93-102) or the seeded synthetic J-node extension
 * (SURVEY.md §8(d)). */
static int make_geometry(int32_t J, int32_t kind, geometry_t* g) {
  if (kind == 0 && (J < 1 || J > 30)) { set_err("node count must be in [1, 30]"); return INVALID; }
  if (J < 1) { set_err("geometry needs at least one node"); return INVALID; }
  g->n = J;
  g->lat = (double*)malloc(sizeof(double) * J);
  g->lon = (double*)malloc(sizeof(double) * J);
  g->pop = (double*)malloc(sizeof(double) * J);
  g->dist = (double*)calloc((size_t)J * J, sizeof(double));
  if (kind == 0) {
    for (int32_t j = 0; j < J; ++j) { g->lat[j] = kLat[j]; g->lon[j] = kLon[j]; g->pop[j] = kPop[j]; }
  } else {
    mt64 gen; mt_seed(&gen, 12345);
    for (int32_t j = 0; j < J; ++j) {
      g->lat[j] = rng_range(&gen, 25.0, 49.0);
      g->lon[j] = rng_range(&gen, -124.0, -67.0);
      g->pop[j] = rng_range(&gen, 1e6, 4e7);
    }
  }
  for (int32_t a = 0; a < J; ++a)
    for (int32_t b = a + 1; b < J; ++b) {
      const double d = great_circle_km(g->lat[a], g->lon[a], g->lat[b], g->lon[b]);
      g->dist[(size_t)a * J + b] = d;
      g->dist[(size_t)b * J + a] = d;
    }
  return OK;
}

/* reward_vector / rewards_from_distances (geometry.cpp:104-128). */
static void reward_vector(const geometry_t* g, int32_t origin, double* out) {
  const int32_t J = g->n;
  const double* d = g->dist + (size_t)origin * J;
  double max_d = 0.0;
  for (int32_t j = 0; j < J; ++j) max_d = d[j] > max_d ? d[j] : max_d;
  for (int32_t j = 0; j < J; ++j) out[j] = 1.0;
  if (max_d <= 0.0) return;
  for (int32_t j = 0; j < J; ++j) {
    const double r = (max_d - d[j]) / max_d;
    out[j] = round(r * 1e9) / 1e9;
  }
}

/* generate_instance (instance.cpp:80-140). */
int orc_generate_instance(int32_t J, int32_t I, int64_t T, double beta, double coverage,
                          uint64_t seed, int32_t geometry, int32_t* product, int32_t* origin,
                          double* reward_table, int32_t* capacity, int32_t* inventory) {
  if (I < 1) { set_err("product count must be >= 1"); return INVALID; }
  if (T < 1) { set_err("horizon must be >= 1"); return INVALID; }
  if (!(coverage > 0.0 && coverage <= 1.0)) { set_err("coverage must be in (0, 1]"); return INVALID; }
  if (!(beta <= 0.0 && beta >= -8.0)) { set_err("beta must be in [-8, 0]"); return INVALID; }
  geometry_t g;
  int rc = make_geometry(J, geometry, &g);
  if (rc) return rc;
  int64_t* counts = (int64_t*)malloc(sizeof(int64_t) * (size_t)I);
  rc = orc_demand_counts(I, T, beta, counts);
  if (rc) { free(counts); geometry_free(&g); return rc; }
  for (int32_t j = 0; j < J; ++j) reward_vector(&g, j, reward_table + (size_t)j * J);

  mt64 gen; mt_seed(&gen, seed);
  /* rng::WeightedSampler (rng.hpp:70-96) over populations */
  double* cum = (double*)malloc(sizeof(double) * J);
  double total = 0.0;
  for (int32_t j = 0; j < J; ++j) { total += g.pop[j]; cum[j] = total; }
  int64_t n = 0;
  for (int32_t i = 0; i < I; ++i)
    for (int64_t q = 0; q < counts[i]; ++q) {
      const double u = rng_unit(&gen) * cum[J - 1];
      int32_t lo = 0, hi = J - 1;
      while (lo < hi) {
        const int32_t mid = (lo + hi) / 2;
        if (cum[mid] <= u) lo = mid + 1; else hi = mid;
      }
      product[n] = i;
      origin[n] = lo;
      ++n;
    }
  /* rng::shuffle (rng.hpp:60-66) of the order records */
  for (int64_t i = n; i > 1; --i) {
    const int64_t j = (int64_t)rng_below(&gen, (uint64_t)i);
    int32_t tp = product[i - 1]; product[i - 1] = product[j]; product[j] = tp;
    int32_t to = origin[i - 1]; origin[i - 1] = origin[j]; origin[j] = to;
  }
  int64_t* cap = (int64_t*)malloc(sizeof(int64_t) * J);
  rc = apportion(g.pop, J, llround(coverage * (double)T), cap);
  for (int32_t j = 0; j < J; ++j) capacity[j] = (int32_t)cap[j];
  memset(inventory, 0, sizeof(int32_t) * (size_t)I * J);
  for (int32_t i = 0; i < I && rc == OK; ++i) {
    const int64_t units = llround(coverage * (double)counts[i]);
    if (units <= 0) continue;
    rc = apportion(g.pop, J, units, cap);
    for (int32_t j = 0; j < J; ++j) inventory[(size_t)i * J + j] = (int32_t)cap[j];
  }
  free(cap); free(cum); free(counts); geometry_free(&g);
  return rc;
}

/* test::small_random_instance parameters (test_helpers.hpp:31-41). */
int orc_small_random_params(uint64_t seed, int32_t* nodes, int32_t* products, int64_t* horizon,
                            double* beta, double* coverage, uint64_t* inst_seed) {
  mt64 gen; mt_seed(&gen, seed);
  *nodes = (int32_t)(2 + rng_below(&gen, 4));
  *products = (int32_t)(1 + rng_below(&gen, 12));
  *horizon = (int64_t)(1 + rng_below(&gen, 60));
  *beta = -(double)rng_below(&gen, 11) / 10.0;
  *coverage = 0.5 + 0.5 * rng_unit(&gen);
  *inst_seed = seed ^ 0x9e3779b97f4a7c15ULL;
  return OK;
}

/* ------------------------------------------------------------ partitions */
/* make_uniform_time_partition (engine.hpp:99-114). */
int orc_uniform_partition(int64_t T, int32_t M, uint64_t seed, int32_t* owner) {
  if (M < 1) { set_err("uniform partition: process count must be >= 1"); return CONTRACT; }
  mt64 gen; mt_seed(&gen, seed);
  for (int64_t t = 0; t < T; ++t) owner[t] = (int32_t)rng_below(&gen, (uint64_t)M);
  return OK;
}

/* make_product_partition (instance.cpp:142-186): seeded shuffle, stable sort
 * by demand descending, LPT onto the lightest (load, group) min-heap. */
int orc_product_partition(const orc_instance* in, int32_t M, uint64_t seed, int32_t* owner) {
  if (M < 1) { set_err("process count must be >= 1"); return INVALID; }
  const int32_t I = in->products;
  int64_t* counts = (int64_t*)calloc((size_t)I, sizeof(int64_t));
  for (int64_t t = 0; t < in->horizon; ++t) counts[in->product[t]] += 1;
  int32_t* ord = (int32_t*)malloc(sizeof(int32_t) * (size_t)(I > 0 ? I : 1));
  for (int32_t i = 0; i < I; ++i) ord[i] = i;
  mt64 gen; mt_seed(&gen, seed);
  for (int64_t i = I; i > 1; --i) {
    const int64_t j = (int64_t)rng_below(&gen, (uint64_t)i);
    int32_t tmp = ord[i - 1]; ord[i - 1] = ord[j]; ord[j] = tmp;
  }
  /* stable merge sort by count descending */
  int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(I > 0 ? I : 1));
  for (int64_t width = 1; width < I; width *= 2) {
    for (int64_t lo = 0; lo < I; lo += 2 * width) {
      int64_t mid = lo + width < I ? lo + width : I;
      int64_t hi = lo + 2 * width < I ? lo + 2 * width : I;
      int64_t a = lo, b = mid, k = lo;
      while (a < mid && b < hi) {
        if (counts[ord[b]] > counts[ord[a]]) tmp[k++] = ord[b++];
        else tmp[k++] = ord[a++];
      }
      while (a < mid) tmp[k++] = ord[a++];
      while (b < hi) tmp[k++] = ord[b++];
    }
    memcpy(ord, tmp, sizeof(int32_t) * (size_t)I);
  }
  /* binary min-heap of (load, group); keys are unique so any heap order
   * pops the same sequence as std::priority_queue<..., std::greater<>>. */
  int64_t* hl = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
  int32_t* hg = (int32_t*)malloc(sizeof(int32_t) * (size_t)M);
  for (int32_t g = 0; g < M; ++g) { hl[g] = 0; hg[g] = g; } /* already a heap */
  int32_t* group_of = (int32_t*)calloc((size_t)(I > 0 ? I : 1), sizeof(int32_t));
#define LESS(a, b) (hl[a] < hl[b] || (hl[a] == hl[b] && hg[a] < hg[b]))
  for (int32_t k = 0; k < I; ++k) {
    const int32_t p = ord[k];
    group_of[p] = hg[0];
    hl[0] += counts[p]; /* replace top, sift down */
    int32_t i = 0;
    for (;;) {
      int32_t l = 2 * i + 1, r = l + 1, s = i;
      if (l < M && LESS(l, s)) s = l;
      if (r < M && LESS(r, s)) s = r;
      if (s == i) break;
      int64_t tl = hl[i]; hl[i] = hl[s]; hl[s] = tl;
      int32_t tg = hg[i]; hg[i] = hg[s]; hg[s] = tg;
      i = s;
    }
  }
#undef LESS
  for (int64_t t = 0; t < in->horizon; ++t) owner[t] = group_of[in->product[t]];
  free(group_of); free(hg); free(hl); free(tmp); free(ord); free(counts);
  return OK;
}

/* ------------------------------------------------------------------ MLP */
/* MlpParams::seeded_uniform (mlp.cpp:117-129). */
int orc_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden, double* w1,
                   double* b1, double* w2, double* b2, double* w3, double* b3) {
  mt64 gen; mt_seed(&gen, seed);
  for (int64_t i = 0; i < (int64_t)hidden * input; ++i) w1[i] = rng_range(&gen, -0.1, 0.1);
  for (int64_t i = 0; i < hidden; ++i) b1[i] = rng_range(&gen, -0.1, 0.1);
  for (int64_t i = 0; i < (int64_t)hidden * hidden; ++i) w2[i] = rng_range(&gen, -0.1, 0.1);
  for (int64_t i = 0; i < hidden; ++i) b2[i] = rng_range(&gen, -0.1, 0.1);
  for (int64_t i = 0; i < (int64_t)output * hidden; ++i) w3[i] = rng_range(&gen, -0.1, 0.1);
  for (int64_t i = 0; i < output; ++i) b3[i] = rng_range(&gen, -0.1, 0.1);
  return OK;
}

/* MlpParams::forward (mlp.cpp:141-169): acc = b; acc += w*x, in order. */
static void mlp_forward(const orc_policy* p, int32_t in, int32_t out, const double* x,
                        double* y, double* h1, double* h2) {
  const int32_t h = p->hidden;
  const int fm = tanh_fma();
  for (int32_t r = 0; r < h; ++r) {
    double acc = p->b1[r];
    const double* row = p->w1 + (size_t)r * in;
    for (int32_t c = 0; c < in; ++c) acc += row[c] * x[c];
    h1[r] = gt_tanh(acc, fm);
  }
  for (int32_t r = 0; r < h; ++r) {
    double acc = p->b2[r];
    const double* row = p->w2 + (size_t)r * h;
    for (int32_t c = 0; c < h; ++c) acc += row[c] * h1[c];
    h2[r] = gt_tanh(acc, fm);
  }
  for (int32_t r = 0; r < out; ++r) {
    double acc = p->b3[r];
    const double* row = p->w3 + (size_t)r * h;
    for (int32_t c = 0; c < h; ++c) acc += row[c] * h2[c];
    y[r] = acc;
  }
}

int orc_mlp_forward(const orc_policy* p, int32_t in, int32_t out, const double* x, double* y) {
  double* h1 = (double*)malloc(sizeof(double) * p->hidden);
  double* h2 = (double*)malloc(sizeof(double) * p->hidden);
  mlp_forward(p, in, out, x, y, h1, h2);
  free(h1); free(h2);
  return OK;
}

/* ------------------------------------------------------------- policies */
typedef struct {
  const orc_instance* in;
  const orc_policy* p;
  const int32_t* init_cap;
  const int32_t* init_inv;
  int64_t horizon;
  double* scratch; /* features, prices, h1, h2 */
} policy_ctx;

static void ctx_init(policy_ctx* c, const orc_instance* in, const orc_policy* p) {
  c->in = in;
  c->p = p;
  c->init_cap = p->init_capacity ? p->init_capacity : in->capacity;
  c->init_inv = p->init_capacity ? (p->init_inventory ? p->init_inventory : in->inventory)
                                 : in->inventory;
  c->horizon = p->horizon >= 0 ? p->horizon : in->horizon;
  const int32_t J = in->nodes;
  const int32_t h = p->hidden > 0 ? p->hidden : 1;
  c->scratch = (double*)malloc(sizeof(double) * (size_t)(4 * J + 1 + 2 * h));
}
static void ctx_free(policy_ctx* c) { free(c->scratch); }

/* Evaluates the policy at (caps[J], row[J]) for order t. Returns CONTRACT on a
 * non-finite dual score (policies.hpp:158-161). */
static int policy_eval(policy_ctx* c, const int32_t* caps, const int32_t* row, int64_t t,
                       int32_t* action) {
  const int32_t J = c->in->nodes;
  const double* rw = c->in->reward_table + (size_t)c->in->reward_row[t] * J;
  const int32_t ot = c->in->order_t ? c->in->order_t[t] : (int32_t)t;
  int32_t best = -1;
  switch (c->p->kind) {
    case 0: { /* GreedyPolicy::evaluate (policies.hpp:28-43) */
      double br = 0.0;
      for (int32_t j = 0; j < J; ++j) {
        if (caps[j] <= 0 || row[j] <= 0) continue;
        if (best < 0 || rw[j] > br) { best = j; br = rw[j]; }
      }
      break;
    }
    case 1: { /* CapacityPenalizedPolicy::evaluate (policies.hpp:55-74) */
      int32_t maxc = 0;
      for (int32_t j = 0; j < J; ++j) maxc = caps[j] > maxc ? caps[j] : maxc;
      double bs = 0.0;
      for (int32_t j = 0; j < J; ++j) {
        if (caps[j] <= 0 || row[j] <= 0) continue;
        const double s = rw[j] + c->p->gamma * (double)caps[j] / (double)maxc;
        if (best < 0 || s > bs) { best = j; bs = s; }
      }
      break;
    }
    case 2: { /* DualNetworkPolicy::evaluate (policies.hpp:121-168) */
      int any = 0;
      for (int32_t j = 0; j < J && !any; ++j) any = caps[j] > 0 && row[j] > 0;
      if (!any) break;
      double* f = c->scratch;
      double* pr = f + 2 * J + 1;
      double* h1 = pr + 2 * J;
      double* h2 = h1 + c->p->hidden;
      const int32_t* irow = c->init_inv + (size_t)c->in->product[t] * J;
      for (int32_t j = 0; j < J; ++j) {
        f[j] = c->init_cap[j] > 0 ? (double)caps[j] / (double)c->init_cap[j] : 0.0;
        f[J + j] = irow[j] > 0 ? (double)row[j] / (double)irow[j] : 0.0;
      }
      f[2 * J] = c->horizon > 0 ? (double)ot / (double)c->horizon : 0.0;
      mlp_forward(c->p, 2 * J + 1, 2 * J, f, pr, h1, h2);
      double bs = 0.0;
      for (int32_t j = 0; j < J; ++j) {
        if (caps[j] <= 0 || row[j] <= 0) continue;
        const double s = rw[j] - pr[j] - pr[J + j];
        if (!isfinite(s)) {
          set_err("dual network produced a non-finite score");
          *action = ot; /* carries time_step */
          return CONTRACT;
        }
        if (s > bs || (s == bs && best < 0)) { best = j; bs = s; }
      }
      break;
    }
    default: /* NullOnlyPolicy (test_engine.cpp:17-22) */
      break;
  }
  *action = best;
  return OK;
}

int orc_policy_evaluate(const orc_instance* in, const orc_policy* p, const int32_t* cap,
                        const int32_t* inv, int64_t t, int32_t* action) {
  policy_ctx c;
  ctx_init(&c, in, p);
  int rc = policy_eval(&c, cap, inv + (size_t)in->product[t] * in->nodes, t, action);
  ctx_free(&c);
  return rc;
}

/* ------------------------------------------------------- state & dynamics */
/* action_feasible (fo/types.hpp:76-85): null is always feasible; nodes >= J
 * are infeasible; else capacity and the product's inventory must be > 0. */
static int feasible(int32_t J, const int32_t* caps, const int32_t* row, int32_t a) {
  if (a < 0) return 1;
  if (a >= J) return 0;
  return caps[a] > 0 && row[a] > 0;
}

/* Copy-on-write local view (fo/local_state.hpp:120-202 semantics): caps are
 * copied, inventory rows on first write. */
typedef struct {
  int32_t J, I;
  int32_t* caps;
  const int32_t* base_inv;
  uint32_t* stamp;
  int64_t* slot;
  int32_t* rows;
  int64_t nrows, rows_cap;
  uint32_t epoch;
} local_t;

static void local_init(local_t* l, int32_t J, int32_t I) {
  memset(l, 0, sizeof *l);
  l->J = J; l->I = I;
  l->caps = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J > 0 ? J : 1));
  l->stamp = (uint32_t*)calloc((size_t)(I > 0 ? I : 1), sizeof(uint32_t));
  l->slot = (int64_t*)calloc((size_t)(I > 0 ? I : 1), sizeof(int64_t));
}
static void local_free(local_t* l) { free(l->caps); free(l->stamp); free(l->slot); free(l->rows); }
static void local_rebind(local_t* l, const int32_t* cap, const int32_t* inv) {
  memcpy(l->caps, cap, sizeof(int32_t) * (size_t)l->J);
  l->base_inv = inv;
  l->nrows = 0;
  if (++l->epoch == 0) { memset(l->stamp, 0, sizeof(uint32_t) * (size_t)l->I); l->epoch = 1; }
}
static const int32_t* local_row(const local_t* l, int32_t p) {
  if (l->stamp[p] == l->epoch) return l->rows + l->slot[p] * l->J;
  return l->base_inv + (size_t)p * l->J;
}
static int32_t* local_touch(local_t* l, int32_t p) {
  if (l->stamp[p] != l->epoch) {
    if (l->nrows == l->rows_cap) {
      l->rows_cap = l->rows_cap ? 2 * l->rows_cap : 16;
      l->rows = (int32_t*)realloc(l->rows, sizeof(int32_t) * (size_t)(l->rows_cap * l->J));
    }
    l->stamp[p] = l->epoch;
    l->slot[p] = l->nrows++;
    memcpy(l->rows + l->slot[p] * l->J, l->base_inv + (size_t)p * l->J, sizeof(int32_t) * (size_t)l->J);
  }
  return l->rows + l->slot[p] * l->J;
}
/* FoLocalState::apply (local_state.hpp:154-162), caller checked feasibility. */
static void local_apply(local_t* l, int32_t p, int32_t a) {
  if (a < 0) return;
  l->caps[a] -= 1;
  local_touch(l, p)[a] -= 1;
}

/* sequential_simulate (engine.hpp:237-267). */
int orc_sequential(const orc_instance* in, const orc_policy* p, int32_t* actions, int64_t* evals,
                   int64_t* error_t) {
  const int32_t J = in->nodes;
  policy_ctx c;
  ctx_init(&c, in, p);
  local_t l;
  local_init(&l, J, in->products);
  local_rebind(&l, in->capacity, in->inventory);
  int rc = OK;
  *evals = 0;
  for (int64_t t = 0; t < in->horizon; ++t) {
    const int32_t prod = in->product[t];
    int32_t a;
    rc = policy_eval(&c, l.caps, local_row(&l, prod), t, &a);
    if (rc) { if (error_t) *error_t = a; break; }
    ++*evals;
    if (!feasible(J, l.caps, local_row(&l, prod), a)) {
      set_err("policy returned an infeasible action");
      if (error_t) *error_t = t;
      rc = CONTRACT;
      break;
    }
    local_apply(&l, prod, a);
    actions[t] = a;
  }
  local_free(&l);
  ctx_free(&c);
  return rc;
}

/* ------------------------------------------------------- Picard iteration */
/* picard_iterate_once (engine.hpp:358-444) with sweep_one_process
 * (:299-342). `fresh` is scratch of length >= t_hi - t_lo. */
static int iterate_once(policy_ctx* c, local_t* l, const int32_t* owner, int32_t M,
                        int32_t* cache, int64_t lo, int64_t hi, const int32_t* ck_cap,
                        const int32_t* ck_inv, int64_t* evals, int64_t* changed,
                        int64_t* n_changed, int64_t* error_t) {
  const orc_instance* in = c->in;
  const int32_t J = in->nodes;
  const int64_t W = hi - lo;
  for (int32_t m = 0; m < M; ++m) evals[m] = 0;
  *n_changed = 0;
  if (W <= 0) return OK;
  int64_t* stop_after = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
  for (int32_t m = 0; m < M; ++m) stop_after[m] = -1;
  for (int64_t t = lo; t < hi; ++t) stop_after[owner[t]] = t;
  int32_t* fresh = (int32_t*)malloc(sizeof(int32_t) * (size_t)W);
  for (int64_t i = 0; i < W; ++i) fresh[i] = -1;
  int rc = OK;
  for (int32_t m = 0; m < M && rc == OK; ++m) {
    if (stop_after[m] < 0) continue;
    local_rebind(l, ck_cap, ck_inv);
    for (int64_t t = lo; t <= stop_after[m]; ++t) {
      const int32_t prod = in->product[t];
      if (owner[t] == m) {
        int32_t a;
        rc = policy_eval(c, l->caps, local_row(l, prod), t, &a);
        if (rc) { if (error_t) *error_t = a; break; }
        ++evals[m];
        if (!feasible(J, l->caps, local_row(l, prod), a)) {
          set_err("policy returned an infeasible action");
          if (error_t) *error_t = t;
          rc = CONTRACT;
          break;
        }
        local_apply(l, prod, a);
        fresh[t - lo] = a;
      } else {
        const int32_t a = cache[t];
        if (feasible(J, l->caps, local_row(l, prod), a)) local_apply(l, prod, a);
      }
    }
  }
  if (rc == OK) {
    for (int64_t t = lo; t < hi; ++t) {
      if (cache[t] != fresh[t - lo]) changed[(*n_changed)++] = t;
      cache[t] = fresh[t - lo];
    }
  }
  free(fresh);
  free(stop_after);
  return rc;
}

static int validate_plan(const int32_t* owner, int64_t T, int32_t M, int64_t* error_t) {
  if (M < 1) { set_err("partition plan: process count must be >= 1"); return CONTRACT; }
  for (int64_t t = 0; t < T; ++t)
    if (owner[t] < 0 || owner[t] >= M) {
      set_err("partition plan: owner out of range");
      if (error_t) *error_t = t;
      return CONTRACT;
    }
  return OK;
}

int orc_iterate_once(const orc_instance* in, const orc_policy* p, const int32_t* owner, int32_t M,
                     int32_t* cache, int64_t lo, int64_t hi, const int32_t* ck_cap,
                     const int32_t* ck_inv, int64_t* evals, int64_t* changed, int64_t* n_changed,
                     int64_t* error_t) {
  policy_ctx c;
  ctx_init(&c, in, p);
  local_t l;
  local_init(&l, in->nodes, in->products);
  int rc = iterate_once(&c, &l, owner, M, cache, lo, hi, ck_cap, ck_inv, evals, changed,
                        n_changed, error_t);
  local_free(&l);
  ctx_free(&c);
  return rc;
}

/* apply_in_place over a cache range (engine.hpp:514-526 advance_checkpoint;
 * fo/types.hpp:89-100 throws on an infeasible entry with order.t). */
static int advance_checkpoint(const orc_instance* in, const int32_t* cache, int64_t from,
                              int64_t to, int32_t* cap, int32_t* inv, int64_t* error_t) {
  const int32_t J = in->nodes;
  for (int64_t t = from; t < to; ++t) {
    const int32_t a = cache[t];
    if (a < 0) continue;
    int32_t* row = inv + (size_t)in->product[t] * J;
    if (!feasible(J, cap, row, a)) {
      set_err("infeasible fulfillment while advancing the checkpoint");
      if (error_t) *error_t = in->order_t ? in->order_t[t] : t;
      return CONTRACT;
    }
    cap[a] -= 1;
    row[a] -= 1;
  }
  return OK;
}

/* picard_simulate (engine.hpp:458-590). `history` (optional) receives the
 * full cache after every iteration, like theory::CacheTraceRecorder. */
int orc_picard(const orc_instance* in, const orc_policy* p, const int32_t* owner, int32_t M,
               const orc_config* cfg, const int32_t* initial_cache, const int32_t* reference,
               int32_t* actions, orc_result* res, orc_trace_row* trace, int64_t trace_cap,
               int32_t* history, int64_t history_cap) {
  const int64_t T = in->horizon;
  const int32_t J = in->nodes, I = in->products;
  memset(res, 0, sizeof *res);
  res->iterations_to_correct = -1;
  res->error_time_step = -1;
  int rc = validate_plan(owner, T, M, &res->error_time_step);
  if (rc) return rc;
  if (cfg->processes != 0 && cfg->processes != M) {
    set_err("config process count disagrees with the plan");
    return CONTRACT;
  }
  if (cfg->max_steps < 0 || cfg->max_iterations < 0) {
    set_err("picard config values must be non-negative");
    return CONTRACT;
  }
  const int64_t cap_it = cfg->max_iterations > 0 ? cfg->max_iterations : 2 * T + 4;
  int32_t* cache = actions;
  for (int64_t t = 0; t < T; ++t) cache[t] = initial_cache ? initial_cache[t] : -1;
  int64_t mismatches = 0;
  if (reference) {
    for (int64_t t = 0; t < T; ++t) mismatches += cache[t] != reference[t];
    if (mismatches == 0) res->iterations_to_correct = 0;
  }
  uint8_t* written = (uint8_t*)calloc((size_t)(T > 0 ? T : 1), 1);
  int32_t* ck_cap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J > 0 ? J : 1));
  int32_t* ck_inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)((int64_t)I * J > 0 ? (int64_t)I * J : 1));
  memcpy(ck_cap, in->capacity, sizeof(int32_t) * (size_t)J);
  memcpy(ck_inv, in->inventory, sizeof(int32_t) * (size_t)I * J);
  int64_t* evals = (int64_t*)malloc(sizeof(int64_t) * (size_t)M);
  int64_t* changed = (int64_t*)malloc(sizeof(int64_t) * (size_t)(T > 0 ? T : 1));
  policy_ctx c;
  ctx_init(&c, in, p);
  local_t l;
  local_init(&l, J, I);
  int64_t ws = 0, iteration = 0, episodes = 0;
  while (ws < T) {
    const int64_t we = cfg->max_steps > 0 ? (ws + cfg->max_steps < T ? ws + cfg->max_steps : T) : T;
    if (iteration >= cap_it) {
      set_err("picard iteration cap exceeded; the policy may be nondeterministic");
      res->iterations_run = iteration;
      rc = ITERLIMIT;
      break;
    }
    ++iteration;
    int64_t n_changed = 0;
    if (reference) /* subtract the window's contribution; re-add after publish */
      for (int64_t t = ws; t < we; ++t) mismatches -= cache[t] != reference[t];
    rc = iterate_once(&c, &l, owner, M, cache, ws, we, ck_cap, ck_inv, evals, changed,
                      &n_changed, &res->error_time_step);
    if (rc) break;
    if (reference)
      for (int64_t t = ws; t < we; ++t) mismatches += cache[t] != reference[t];
    int64_t mx = 0, tot = 0;
    for (int32_t m = 0; m < M; ++m) { mx = evals[m] > mx ? evals[m] : mx; tot += evals[m]; }
    res->iterations_to_converged += 1;
    res->policy_eval_count_sequential_equivalent += mx;
    res->total_policy_evals += tot;
    for (int64_t i = 0; i < n_changed; ++i) res->conflicts += written[changed[i]] ? 1 : 0;
    for (int64_t t = ws; t < we; ++t) written[t] = 1;
    if (cfg->record_trace) {
      if (res->trace_rows < trace_cap) {
        orc_trace_row* r = &trace[res->trace_rows];
        r->chunk = episodes; r->iteration = iteration; r->changed_slots = n_changed;
        r->max_process_evals = mx; r->t_reset = ws;
      }
      res->trace_rows += 1;
    }
    if (history && iteration - 1 < history_cap)
      memcpy(history + (iteration - 1) * T, cache, sizeof(int32_t) * (size_t)T);
    if (reference && res->iterations_to_correct < 0 && mismatches == 0)
      res->iterations_to_correct = iteration;
    if (n_changed == 0) {
      rc = advance_checkpoint(in, cache, ws, we, ck_cap, ck_inv, &res->error_time_step);
      if (rc) break;
      ws = we;
      ++episodes;
    } else if (changed[0] > ws) {
      rc = advance_checkpoint(in, cache, ws, changed[0], ck_cap, ck_inv, &res->error_time_step);
      if (rc) break;
      ws = changed[0];
    }
  }
  if (rc != ITERLIMIT) res->iterations_run = iteration;
  local_free(&l);
  ctx_free(&c);
  free(changed); free(evals); free(ck_inv); free(ck_cap); free(written);
  return rc;
}

/* naive_fixed_point (test_engine.cpp:236-266): the textbook Algorithm 1 over
 * plain states — every process sweeps the whole horizon from the initial
 * state each iteration. history[k*T..] = cache after iteration k+1. */
int orc_naive_fixed_point(const orc_instance* in, const orc_policy* p, const int32_t* owner,
                          int32_t M, int32_t* history, int64_t history_cap, int64_t* iterations) {
  const int64_t T = in->horizon;
  const int32_t J = in->nodes, I = in->products;
  int32_t* cache = (int32_t*)malloc(sizeof(int32_t) * (size_t)(T > 0 ? T : 1));
  int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(T > 0 ? T : 1));
  int32_t* cap = (int32_t*)malloc(sizeof(int32_t) * (size_t)(J > 0 ? J : 1));
  int32_t* inv = (int32_t*)malloc(sizeof(int32_t) * (size_t)((int64_t)I * J > 0 ? (int64_t)I * J : 1));
  for (int64_t t = 0; t < T; ++t) cache[t] = -1;
  policy_ctx c;
  ctx_init(&c, in, p);
  int rc = OK;
  *iterations = 0;
  for (int64_t k = 0; k < 2 * T + 4 && rc == OK; ++k) {
    for (int64_t t = 0; t < T; ++t) next[t] = -1;
    for (int32_t m = 0; m < M && rc == OK; ++m) {
      memcpy(cap, in->capacity, sizeof(int32_t) * (size_t)J);
      memcpy(inv, in->inventory, sizeof(int32_t) * (size_t)I * J);
      for (int64_t t = 0; t < T; ++t) {
        int32_t* row = inv + (size_t)in->product[t] * J;
        int32_t a;
        if (owner[t] == m) {
          rc = policy_eval(&c, cap, row, t, &a);
          if (rc) break;
          next[t] = a;
        } else {
          a = feasible(J, cap, row, cache[t]) ? cache[t] : -1;
        }
        if (a >= 0) {
          if (!feasible(J, cap, row, a)) { set_err("infeasible"); rc = CONTRACT; break; }
          cap[a] -= 1;
          row[a] -= 1;
        }
      }
    }
    if (rc) break;
    int same = 1;
    for (int64_t t = 0; t < T; ++t) same &= next[t] == cache[t];
    memcpy(cache, next, sizeof(int32_t) * (size_t)T);
    if (history && k < history_cap) memcpy(history + k * T, cache, sizeof(int32_t) * (size_t)T);
    *iterations = k + 1;
    if (same) break;
  }
  ctx_free(&c);
  free(inv); free(cap); free(next); free(cache);
  return rc;
}

/* fo_total_reward (env.hpp:298-310). */
int orc_total_reward(const orc_instance* in, const int32_t* actions, double* total) {
  double s = 0.0;
  for (int64_t t = 0; t < in->horizon; ++t)
    if (actions[t] >= 0) s += in->reward_table[(size_t)in->reward_row[t] * in->nodes + actions[t]];
  *total = s;
  return OK;
}
