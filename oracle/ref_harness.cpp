// ref_harness.cpp — TEST INFRASTRUCTURE ONLY.
//
// Flat extern "C" wrapper around the UNMODIFIED reference library
// (/root/reference/proj/include + proj/src/{instance,geometry,mlp}.cpp), built
// by oracle/Makefile into oracle/_ref/libpicard_ref.so. Nothing from the
// reference is copied here: this file only marshals flat arrays into the
// reference's own types and calls its public API:
//   picard::sequential_simulate      engine.hpp:237-267
//   picard::picard_simulate          engine.hpp:458-590
//   picard::picard_iterate_once      engine.hpp:358-444
//   picard::make_uniform_time_partition engine.hpp:99-114
//   picard::fo::generate_instance    instance.cpp:80-140
//   picard::fo::make_product_partition instance.cpp:142-186
//   picard::fo::MlpParams            mlp.cpp:104-169
//   picard::fo::{Greedy,CapacityPenalized,DualNetwork}Policy policies.hpp
//   picard::timewarp::time_warp_simulate     fo/timewarp.hpp:56-181
//   picard::linear::{make_contractive_spec, picard_convergence_curve,
//     rollout_states, GainPolicy, LinearEnv}   linear.hpp / linear.cpp
// The only logic of our own is (a) the J>30 synthetic geometry (SURVEY.md
// §8(d)) assembled from the reference's building blocks exactly as
// generate_instance does (instance.cpp:95-138), and (b) the fixture recipe of
// test_helpers.hpp:31-41 (small_random_instance parameters).

#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <span>
#include <string>
#include <vector>

#include "picard/engine.hpp"
#include "picard/fo/env.hpp"
#include "picard/fo/geometry.hpp"
#include "picard/fo/instance.hpp"
#include "picard/fo/mlp.hpp"
#include "picard/fo/policies.hpp"
#include "picard/fo/timewarp.hpp"
#include "picard/linear.hpp"
#include "picard/rng.hpp"
#include "picard/theory.hpp"

#include "oracle.h"

using namespace picard;
using namespace picard::fo;

namespace {

thread_local std::string g_err;

struct NullOnlyPolicy {  // test_engine.cpp:17-22
  template <FoStateView V>
  FoAction evaluate(const V&, const Order&) const { return kNoFulfill; }
};

FoState make_state(int32_t J, int32_t I, const int32_t* cap, const int32_t* inv) {
  FoState s;
  s.capacity.assign(cap, cap + J);
  for (int32_t i = 0; i < I; ++i) {
    const int32_t* row = inv + (size_t)i * J;
    bool any = false;
    for (int32_t j = 0; j < J; ++j) any |= row[j] != 0;
    if (any) s.inventory[i].assign(row, row + J);
  }
  return s;
}

Instance make_instance(const orc_instance* in) {
  Instance inst;
  inst.nodes = in->nodes;
  inst.products = in->products;
  inst.horizon = in->horizon;
  inst.initial = make_state(in->nodes, in->products, in->capacity, in->inventory);
  inst.orders.resize((size_t)in->horizon);
  for (int64_t t = 0; t < in->horizon; ++t) {
    Order& o = inst.orders[(size_t)t];
    o.t = in->order_t ? in->order_t[t] : (int32_t)t;
    o.product = in->product[t];
    o.origin_node = in->reward_row[t];
    const double* r = in->reward_table + (size_t)in->reward_row[t] * in->nodes;
    o.rewards.assign(r, r + in->nodes);
  }
  return inst;
}

MlpParams make_params(const orc_policy* p, int32_t J) {
  MlpParams m;
  const int32_t in = 2 * J + 1, out = 2 * J, h = p->hidden;
  m.widths = {in, h, h, out};
  m.w1.assign(p->w1, p->w1 + (size_t)h * in);
  m.b1.assign(p->b1, p->b1 + h);
  m.w2.assign(p->w2, p->w2 + (size_t)h * h);
  m.b2.assign(p->b2, p->b2 + h);
  m.w3.assign(p->w3, p->w3 + (size_t)out * h);
  m.b3.assign(p->b3, p->b3 + out);
  return m;
}

PartitionPlan make_plan(const int32_t* owner, int64_t T, int32_t M) {
  PartitionPlan plan;
  plan.processes = M;
  plan.owner.assign(owner, owner + T);
  return plan;
}

// Calls fn(instance, policy) with the reference policy object of the kind.
template <typename Fn>
int with_policy(const orc_instance* in, const orc_policy* p, const Instance& inst,
                Fn&& fn) {
  switch (p->kind) {
    case 0: return fn(GreedyPolicy{});
    case 1: return fn(CapacityPenalizedPolicy{p->gamma});
    case 2: {
      auto init = std::make_shared<const FoState>(
          p->init_capacity
              ? make_state(in->nodes, in->products, p->init_capacity,
                           p->init_inventory ? p->init_inventory : in->inventory)
              : inst.initial);
      const int64_t horizon = p->horizon >= 0 ? p->horizon : in->horizon;
      return fn(DualNetworkPolicy(make_params(p, in->nodes), init, horizon));
    }
    case 3: return fn(NullOnlyPolicy{});
    default: throw std::invalid_argument("unknown policy kind");
  }
}

template <typename Body>
int guarded(Body&& body, int64_t* error_t = nullptr, orc_result* res = nullptr,
            orc_trace_row* trace = nullptr, int64_t trace_cap = 0) {
  try {
    return body();
  } catch (const IterationLimitError& e) {
    g_err = e.what();
    if (res) {
      res->iterations_run = e.iterations_run();
      res->trace_rows = (int64_t)e.partial_trace().size();
      for (size_t i = 0; i < e.partial_trace().size() && (int64_t)i < trace_cap; ++i) {
        const auto& r = e.partial_trace()[i];
        trace[i] = {r.chunk, r.iteration, r.changed_slots, r.max_process_evals, r.t_reset};
      }
    }
    return 3;
  } catch (const ContractViolation& e) {
    g_err = e.what();
    if (error_t) *error_t = e.time_step();
    if (res) res->error_time_step = e.time_step();
    return 2;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

struct HistoryRecorder {  // same shape as theory::CacheTraceRecorder (theory.hpp:120-126)
  int32_t* history;
  int64_t cap;
  int64_t T;
  int64_t rows = 0;
  void on_iteration(std::int64_t, std::int64_t, std::int64_t, std::int64_t,
                    std::span<const FoAction> cache) {
    if (history && rows < cap) {
      for (int64_t t = 0; t < T; ++t) history[rows * T + t] = cache[(size_t)t].node;
    }
    ++rows;
  }
};

// Seeded synthetic geometry for J > 30 (SURVEY.md §8(d), Appendix B probe100).
NetworkGeometry synthetic_geometry(int32_t J) {
  auto gen = rng::make(12345);
  std::vector<GeoNode> nodes;
  for (int32_t j = 0; j < J; ++j) {
    GeoNode n;
    n.name = "N" + std::to_string(j);
    n.state = "XX";
    n.latitude = rng::range(gen, 25.0, 49.0);
    n.longitude = rng::range(gen, -124.0, -67.0);
    n.population = rng::range(gen, 1e6, 4e7);
    nodes.push_back(n);
  }
  return NetworkGeometry(std::move(nodes));
}

// generate_instance (instance.cpp:80-140) with an injected geometry: the same
// calls in the same order, so geometry==default reproduces generate_instance.
Instance generate_with_geometry(int32_t J, int32_t I, int64_t T, double beta,
                                double coverage, uint64_t seed,
                                const NetworkGeometry& geometry) {
  Instance instance;
  instance.nodes = J;
  instance.products = I;
  instance.horizon = T;
  instance.meta = {beta, coverage, seed};
  const auto counts = demand_counts(I, T, beta);
  const auto populations = geometry.population_weights();
  auto gen = rng::make(seed);
  rng::WeightedSampler origin_sampler(populations);
  std::vector<std::vector<double>> node_rewards;
  for (int32_t j = 0; j < J; ++j) node_rewards.push_back(reward_vector(j, geometry));
  instance.orders.reserve((size_t)T);
  for (int32_t i = 0; i < I; ++i) {
    for (int64_t q = 0; q < counts[(size_t)i]; ++q) {
      Order order;
      order.product = i;
      order.origin_node = (int32_t)origin_sampler.sample(gen);
      instance.orders.push_back(std::move(order));  // rewards filled below
    }
  }
  rng::shuffle(std::span<Order>(instance.orders), gen);
  for (int64_t t = 0; t < T; ++t) instance.orders[(size_t)t].t = (int32_t)t;
  const auto capacity = largest_remainder_apportion(
      populations, std::llround(coverage * static_cast<double>(T)));
  for (auto c : capacity) instance.initial.capacity.push_back((int32_t)c);
  for (int32_t i = 0; i < I; ++i) {
    const int64_t units = std::llround(coverage * static_cast<double>(counts[(size_t)i]));
    if (units <= 0) continue;
    const auto row = largest_remainder_apportion(populations, units);
    auto& stored = instance.initial.inventory[i];
    for (auto x : row) stored.push_back((int32_t)x);
  }
  // rewards are a function of the origin only; return them as a table.
  instance.orders.shrink_to_fit();
  (void)node_rewards;
  return instance;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

double ref_tanh(double x) { return std::tanh(x); }

int ref_demand_counts(int32_t products, int64_t horizon, double beta, int64_t* out) {
  return guarded([&] {
    auto c = demand_counts(products, horizon, beta);
    for (size_t i = 0; i < c.size(); ++i) out[i] = c[i];
    return 0;
  });
}

int ref_apportion(const double* weights, int64_t n, int64_t total, int64_t* out) {
  return guarded([&] {
    auto c = largest_remainder_apportion(std::span<const double>(weights, (size_t)n), total);
    for (size_t i = 0; i < c.size(); ++i) out[i] = c[i];
    return 0;
  });
}

int ref_generate_instance(int32_t J, int32_t I, int64_t T, double beta,
                          double coverage, uint64_t seed, int32_t geometry,
                          int32_t* product, int32_t* origin, double* reward_table,
                          int32_t* capacity, int32_t* inventory) {
  return guarded([&] {
    Instance inst;
    NetworkGeometry geo = geometry == 0 ? default_geometry(J) : synthetic_geometry(J);
    if (geometry == 0) {
      inst = generate_instance(J, I, T, beta, coverage, seed);
    } else {
      if (!(I >= 1) || !(T >= 1) || !(coverage > 0.0 && coverage <= 1.0) ||
          !(beta <= 0.0 && beta >= -8.0))
        throw std::invalid_argument("bad instance parameters");
      inst = generate_with_geometry(J, I, T, beta, coverage, seed, geo);
    }
    for (int32_t j = 0; j < J; ++j) {
      auto r = reward_vector(j, geo);
      for (int32_t k = 0; k < J; ++k) reward_table[(size_t)j * J + k] = r[(size_t)k];
    }
    for (int64_t t = 0; t < T; ++t) {
      const Order& o = inst.orders[(size_t)t];
      product[t] = o.product;
      origin[t] = o.origin_node;
      if (geometry == 0) {  // the generated rewards must equal the table row
        for (int32_t k = 0; k < J; ++k)
          if (o.rewards[(size_t)k] != reward_table[(size_t)o.origin_node * J + k])
            throw std::runtime_error("reward row is not a function of the origin");
      }
    }
    for (int32_t j = 0; j < J; ++j) capacity[j] = inst.initial.capacity[(size_t)j];
    std::memset(inventory, 0, sizeof(int32_t) * (size_t)I * J);
    for (const auto& [i, row] : inst.initial.inventory)
      for (int32_t j = 0; j < J; ++j) inventory[(size_t)i * J + j] = row[(size_t)j];
    return 0;
  });
}

int ref_small_random_params(uint64_t seed, int32_t* nodes, int32_t* products,
                            int64_t* horizon, double* beta, double* coverage,
                            uint64_t* inst_seed) {
  // test_helpers.hpp:31-41
  auto gen = rng::make(seed);
  *nodes = (int32_t)(2 + rng::below(gen, 4));
  *products = (int32_t)(1 + rng::below(gen, 12));
  *horizon = (int64_t)(1 + rng::below(gen, 60));
  *beta = -static_cast<double>(rng::below(gen, 11)) / 10.0;
  *coverage = 0.5 + 0.5 * rng::unit(gen);
  *inst_seed = seed ^ 0x9e3779b97f4a7c15ull;
  return 0;
}

int ref_product_partition(const orc_instance* in, int32_t M, uint64_t seed,
                          int32_t* owner) {
  return guarded([&] {
    Instance inst = make_instance(in);
    auto plan = make_product_partition(inst, M, seed);
    for (int64_t t = 0; t < in->horizon; ++t) owner[t] = plan.owner[(size_t)t];
    return 0;
  });
}

int ref_uniform_partition(int64_t T, int32_t M, uint64_t seed, int32_t* owner) {
  return guarded([&] {
    auto plan = make_uniform_time_partition(T, M, seed);
    for (int64_t t = 0; t < T; ++t) owner[t] = plan.owner[(size_t)t];
    return 0;
  });
}

int ref_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden,
                   double* w1, double* b1, double* w2, double* b2, double* w3,
                   double* b3) {
  return guarded([&] {
    auto p = MlpParams::seeded_uniform(input, output, seed, hidden);
    std::copy(p.w1.begin(), p.w1.end(), w1);
    std::copy(p.b1.begin(), p.b1.end(), b1);
    std::copy(p.w2.begin(), p.w2.end(), w2);
    std::copy(p.b2.begin(), p.b2.end(), b2);
    std::copy(p.w3.begin(), p.w3.end(), w3);
    std::copy(p.b3.begin(), p.b3.end(), b3);
    return 0;
  });
}

int ref_mlp_forward(const orc_policy* pol, int32_t input, int32_t output,
                    const double* x, double* out) {
  return guarded([&] {
    MlpParams m;
    const int32_t h = pol->hidden;
    m.widths = {input, h, h, output};
    m.w1.assign(pol->w1, pol->w1 + (size_t)h * input);
    m.b1.assign(pol->b1, pol->b1 + h);
    m.w2.assign(pol->w2, pol->w2 + (size_t)h * h);
    m.b2.assign(pol->b2, pol->b2 + h);
    m.w3.assign(pol->w3, pol->w3 + (size_t)output * h);
    m.b3.assign(pol->b3, pol->b3 + output);
    m.forward(std::span<const double>(x, (size_t)input), std::span<double>(out, (size_t)output));
    return 0;
  });
}

int ref_policy_evaluate(const orc_instance* in, const orc_policy* pol,
                        const int32_t* cap, const int32_t* inv, int64_t t,
                        int32_t* action) {
  return guarded([&] {
    Instance inst = make_instance(in);
    FoState state = make_state(in->nodes, in->products, cap, inv);
    return with_policy(in, pol, inst, [&](const auto& policy) {
      *action = policy.evaluate(state, inst.orders[(size_t)t]).node;
      return 0;
    });
  });
}

int ref_sequential(const orc_instance* in, const orc_policy* pol, int32_t* actions,
                   int64_t* evals, int64_t* error_t) {
  return guarded(
      [&] {
        Instance inst = make_instance(in);
        auto env = inst.make_env();
        return with_policy(in, pol, inst, [&](const auto& policy) {
          auto out = sequential_simulate(env, policy, std::span<const Order>(inst.orders));
          for (size_t t = 0; t < out.actions.size(); ++t) actions[t] = out.actions[t].node;
          *evals = out.policy_evals;
          return 0;
        });
      },
      error_t);
}

// Wall-clock of sequential_simulate alone (instance marshalling excluded), the
// CPU-baseline leg of bench.py (BASELINE.md §4 protocol step 3).
int ref_sequential_timed(const orc_instance* in, const orc_policy* pol, int32_t* actions,
                         double* seconds) {
  return guarded([&] {
    Instance inst = make_instance(in);
    auto env = inst.make_env();
    return with_policy(in, pol, inst, [&](const auto& policy) {
      const auto t0 = std::chrono::steady_clock::now();
      auto out = sequential_simulate(env, policy, std::span<const Order>(inst.orders));
      const auto t1 = std::chrono::steady_clock::now();
      *seconds = std::chrono::duration<double>(t1 - t0).count();
      for (size_t t = 0; t < out.actions.size(); ++t) actions[t] = out.actions[t].node;
      return 0;
    });
  });
}

// Wall-clock of picard_simulate alone with PicardConfig::threads = `threads`.
int ref_picard_timed(const orc_instance* in, const orc_policy* pol, const int32_t* owner,
                     int32_t M, int64_t max_steps, int32_t threads, int32_t* actions,
                     int64_t* iterations, int64_t* seq_equiv, double* seconds) {
  return guarded([&] {
    Instance inst = make_instance(in);
    auto env = inst.make_env();
    auto plan = make_plan(owner, in->horizon, M);
    PicardConfig config;
    config.max_steps = max_steps;
    config.threads = threads;
    return with_policy(in, pol, inst, [&](const auto& policy) {
      const auto t0 = std::chrono::steady_clock::now();
      auto r = picard_simulate(env, policy, std::span<const Order>(inst.orders), plan, config);
      const auto t1 = std::chrono::steady_clock::now();
      *seconds = std::chrono::duration<double>(t1 - t0).count();
      *iterations = r.iterations_to_converged;
      *seq_equiv = r.policy_eval_count_sequential_equivalent;
      for (size_t t = 0; t < r.actions.size(); ++t) actions[t] = r.actions[t].node;
      return 0;
    });
  });
}

int ref_picard(const orc_instance* in, const orc_policy* pol, const int32_t* owner,
               int32_t M, const orc_config* cfg, const int32_t* initial_cache,
               const int32_t* reference, int32_t* actions, orc_result* res,
               orc_trace_row* trace, int64_t trace_cap, int32_t* history,
               int64_t history_cap) {
  *res = orc_result{0, -1, 0, 0, 0, 0, 0, -1};
  return guarded(
      [&] {
        Instance inst = make_instance(in);
        auto env = inst.make_env();
        auto plan = make_plan(owner, in->horizon, M);
        PicardConfig config;
        config.processes = cfg->processes;
        config.max_steps = cfg->max_steps;
        config.max_iterations = cfg->max_iterations;
        config.record_trace = cfg->record_trace != 0;
        config.threads = cfg->threads > 0 ? cfg->threads : 1;
        std::vector<FoAction> init, ref;
        if (initial_cache)
          for (int64_t t = 0; t < in->horizon; ++t) init.push_back(FoAction{initial_cache[t]});
        if (reference)
          for (int64_t t = 0; t < in->horizon; ++t) ref.push_back(FoAction{reference[t]});
        HistoryRecorder rec{history, history_cap, in->horizon};
        return with_policy(in, pol, inst, [&](const auto& policy) {
          auto r = picard_simulate(env, policy, std::span<const Order>(inst.orders), plan,
                                   config, std::span<const FoAction>(init),
                                   std::span<const FoAction>(ref), &rec);
          for (size_t t = 0; t < r.actions.size(); ++t) actions[t] = r.actions[t].node;
          res->iterations_to_converged = r.iterations_to_converged;
          res->iterations_to_correct =
              r.iterations_to_correct.has_value() ? *r.iterations_to_correct : -1;
          res->conflicts = r.conflicts;
          res->policy_eval_count_sequential_equivalent =
              r.policy_eval_count_sequential_equivalent;
          res->total_policy_evals = r.total_policy_evals;
          res->trace_rows = (int64_t)r.trace.size();
          res->iterations_run = r.iterations_to_converged;
          for (size_t i = 0; i < r.trace.size() && (int64_t)i < trace_cap; ++i) {
            const auto& row = r.trace[i];
            trace[i] = {row.chunk, row.iteration, row.changed_slots, row.max_process_evals,
                        row.t_reset};
          }
          return 0;
        });
      },
      nullptr, res, trace, trace_cap);
}

int ref_iterate_once(const orc_instance* in, const orc_policy* pol, const int32_t* owner,
                     int32_t M, int32_t* cache, int64_t t_lo, int64_t t_hi,
                     const int32_t* ckpt_cap, const int32_t* ckpt_inv,
                     int64_t* evals_per_process, int64_t* changed, int64_t* n_changed,
                     int64_t* error_t) {
  return guarded(
      [&] {
        Instance inst = make_instance(in);
        auto env = inst.make_env();
        auto plan = make_plan(owner, in->horizon, M);
        ActionCache<FoAction> c;
        for (int64_t t = 0; t < in->horizon; ++t) c.push_back(FoAction{cache[t]});
        FoState ckpt = make_state(in->nodes, in->products, ckpt_cap, ckpt_inv);
        return with_policy(in, pol, inst, [&](const auto& policy) {
          auto out = picard_iterate_once(env, policy, std::span<const Order>(inst.orders),
                                         plan, c, t_lo, t_hi, ckpt);
          for (int64_t t = 0; t < in->horizon; ++t) cache[t] = c[(size_t)t].node;
          for (int32_t m = 0; m < M; ++m) evals_per_process[m] = out.evals_per_process[(size_t)m];
          for (size_t i = 0; i < out.changed_slots.size(); ++i) changed[i] = out.changed_slots[i];
          *n_changed = (int64_t)out.changed_slots.size();
          return 0;
        });
      },
      error_t);
}

int ref_total_reward(const orc_instance* in, const int32_t* actions, double* total) {
  return guarded([&] {
    Instance inst = make_instance(in);
    std::vector<FoAction> a;
    for (int64_t t = 0; t < in->horizon; ++t) a.push_back(FoAction{actions[t]});
    *total = fo_total_reward(std::span<const Order>(inst.orders), std::span<const FoAction>(a));
    return 0;
  });
}

// ------------------------------------------------------- serial sessions
// One sequential trajectory run as consecutive segments (bench.py's reference
// arm): the instance is marshalled once; each segment is the reference's own
// sequential_simulate over orders [t0, t1) on an FoEnv built from the state
// the previous segments reached (carried with the reference's apply_in_place,
// types.hpp:89-100), the policy keeping the instance's normalisation state
// and horizon. Concatenated segments are exactly one sequential_simulate of
// the whole horizon: its state at t0 is that same carried state.
struct RefSession {
  orc_instance in;
  orc_policy pol;
  Instance inst;
  FoState state;
  int64_t at = 0;
};

void* ref_session_create(const orc_instance* in, const orc_policy* pol) {
  try {
    auto s = std::make_unique<RefSession>();
    s->in = *in;
    s->pol = *pol;
    s->inst = make_instance(in);
    s->state = s->inst.initial;
    return s.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_session_destroy(void* p) { delete static_cast<RefSession*>(p); }

// state at time t (cap[J], dense inv[I*J]); the next segment must start at t
int ref_session_set_state(void* p, int64_t t, const int32_t* cap, const int32_t* inv) {
  return guarded([&] {
    auto* s = static_cast<RefSession*>(p);
    if (t < 0 || t > s->in.horizon) throw std::invalid_argument("session time out of range");
    s->state = make_state(s->in.nodes, s->in.products, cap, inv);
    s->at = t;
    return 0;
  });
}

int ref_session_get_state(void* p, int64_t* t, int32_t* cap, int32_t* inv) {
  return guarded([&] {
    auto* s = static_cast<RefSession*>(p);
    const int32_t J = s->in.nodes;
    *t = s->at;
    for (int32_t j = 0; j < J; ++j) cap[j] = s->state.capacity[(size_t)j];
    std::memset(inv, 0, sizeof(int32_t) * (size_t)s->in.products * J);
    for (const auto& [i, row] : s->state.inventory)
      for (int32_t j = 0; j < J; ++j) inv[(size_t)i * J + j] = row[(size_t)j];
    return 0;
  });
}

// fo_total_reward (env.hpp) of a whole-horizon trajectory over the session's orders
int ref_session_total_reward(void* p, const int32_t* actions, double* total) {
  return guarded([&] {
    auto* s = static_cast<RefSession*>(p);
    std::vector<FoAction> a((size_t)s->in.horizon);
    for (int64_t t = 0; t < s->in.horizon; ++t) a[(size_t)t] = FoAction{actions[t]};
    *total = fo_total_reward(std::span<const Order>(s->inst.orders), std::span<const FoAction>(a));
    return 0;
  });
}

// sequential_simulate over orders [at, t1) (timed alone), then the state carry
int ref_session_sequential(void* p, int64_t t1, int32_t* actions, double* seconds, int64_t* error_t) {
  auto* s = static_cast<RefSession*>(p);
  return guarded(
      [&] {
        if (t1 < s->at || t1 > s->in.horizon) throw std::invalid_argument("segment end out of range");
        const std::span<const Order> seg(s->inst.orders.data() + s->at, (size_t)(t1 - s->at));
        FoEnv env(s->state, s->in.products);
        return with_policy(&s->in, &s->pol, s->inst, [&](const auto& policy) {
          const auto c0 = std::chrono::steady_clock::now();
          auto out = sequential_simulate(env, policy, seg);
          const auto c1 = std::chrono::steady_clock::now();
          *seconds = std::chrono::duration<double>(c1 - c0).count();
          for (size_t k = 0; k < out.actions.size(); ++k) {
            actions[k] = out.actions[k].node;
            apply_in_place(s->state, seg[k], out.actions[k]);
          }
          s->at = t1;
          return 0;
        });
      },
      error_t);
}

// theory::compute_depletion_from_capacities on the capacities of the
// trajectory `actions` replayed from the initial state (fo_transition)
int ref_depletion(const orc_instance* in, const int32_t* actions, int64_t* first_depleted_at) {
  return guarded([&] {
    Instance inst = make_instance(in);
    FoState s = inst.initial;
    std::vector<std::vector<int32_t>> caps;
    caps.push_back(s.capacity);
    for (int64_t t = 0; t < in->horizon; ++t) {
      apply_in_place(s, inst.orders[(size_t)t], FoAction{actions[t]});
      caps.push_back(s.capacity);
    }
    const auto prof = theory::compute_depletion_from_capacities(caps);
    for (size_t j = 0; j < prof.first_depleted_at.size(); ++j) first_depleted_at[j] = prof.first_depleted_at[j];
    return 0;
  });
}

// ---------------------------------------------------------------- Time Warp
// counters = {sync_rounds, rollbacks, seq_equiv, total_evals}; trace rows of
// 5 int64 {round, t_start, window_length, max_process_evals, rolled_back}
int ref_time_warp(const orc_instance* in, const orc_policy* pol, int32_t processes, uint64_t seed, int32_t rule,
                  int32_t record_trace, int32_t* actions, int64_t* counters, int64_t* trace, int64_t trace_cap,
                  int64_t* trace_rows, int64_t* error_t) {
  return guarded(
      [&] {
        Instance inst = make_instance(in);
        return with_policy(in, pol, inst, [&](const auto& policy) {
          const auto r = timewarp::time_warp_simulate(inst, policy, processes, seed, record_trace != 0,
                                                      rule ? timewarp::WindowRule::min_stocked_capacity
                                                           : timewarp::WindowRule::min_capacity);
          for (size_t t = 0; t < r.actions.size(); ++t) actions[t] = r.actions[t].node;
          counters[0] = r.sync_rounds;
          counters[1] = r.rollbacks;
          counters[2] = r.policy_eval_count_sequential_equivalent;
          counters[3] = r.total_policy_evals;
          *trace_rows = (int64_t)r.trace.size();
          for (size_t i = 0; i < r.trace.size() && (int64_t)i < trace_cap; ++i) {
            const auto& row = r.trace[i];
            int64_t* o = trace + 5 * i;
            o[0] = row.round; o[1] = row.t_start; o[2] = row.window_length; o[3] = row.max_process_evals;
            o[4] = row.rolled_back ? 1 : 0;
          }
          return 0;
        });
      },
      error_t);
}

// ---------------------------------------------------------------- linear env
// Flat layout: A[T][n][n], B[T][n][p], w[T][n], G[p][n] (row-major).
static linear::LinearSystemSpec make_linear(int32_t n, int32_t p, int64_t T, const double* A, const double* B,
                                            const double* w, const double* G) {
  linear::LinearSystemSpec s;
  s.state_dim = n;
  s.input_dim = p;
  s.horizon = T;
  s.gain.assign(G, G + (size_t)p * n);
  for (int64_t t = 0; t < T; ++t) {
    s.dynamics.emplace_back(A + (size_t)t * n * n, A + (size_t)(t + 1) * n * n);
    s.input.emplace_back(B + (size_t)t * n * p, B + (size_t)(t + 1) * n * p);
    s.disturbances.emplace_back(w + (size_t)t * n, w + (size_t)(t + 1) * n);
  }
  s.contraction = linear::closed_loop_contraction(s);
  return s;
}

int ref_linear_spec(int32_t n, int32_t p, int64_t T, double rho, uint64_t seed, double coupling, double* A,
                    double* B, double* w, double* G, double* contraction) {
  return guarded([&] {
    const auto s = linear::make_contractive_spec(n, p, T, rho, seed, coupling);
    std::memcpy(G, s.gain.data(), sizeof(double) * s.gain.size());
    for (int64_t t = 0; t < T; ++t) {
      std::memcpy(A + (size_t)t * n * n, s.dynamics[(size_t)t].data(), sizeof(double) * n * n);
      std::memcpy(B + (size_t)t * n * p, s.input[(size_t)t].data(), sizeof(double) * n * p);
      std::memcpy(w + (size_t)t * n, s.disturbances[(size_t)t].data(), sizeof(double) * n);
    }
    *contraction = s.contraction;
    return 0;
  });
}

// picard_convergence_curve (linear.cpp): curve[k] for k < *len (<= cap)
int ref_linear_curve(int32_t n, int32_t p, int64_t T, const double* A, const double* B, const double* w,
                     const double* G, const double* init, double tolerance, int64_t max_iterations,
                     int32_t normalization, double* curve, int64_t cap, int64_t* len) {
  return guarded([&] {
    const auto s = make_linear(n, p, T, A, B, w, G);
    std::vector<std::vector<double>> ic;
    if (init)
      for (int64_t t = 0; t < T; ++t) ic.emplace_back(init + (size_t)t * p, init + (size_t)(t + 1) * p);
    linear::ConvergenceCurveOptions o;
    o.tolerance = tolerance;
    o.max_iterations = max_iterations;
    o.normalization = normalization ? linear::RmseNormalization::draft : linear::RmseNormalization::reference;
    const auto c = linear::picard_convergence_curve(s, ic, o);
    *len = (int64_t)c.size();
    for (size_t k = 0; k < c.size() && (int64_t)k < cap; ++k) curve[k] = c[k];
    return 0;
  });
}

// sequential_simulate of (LinearEnv, GainPolicy): actions[T][p], states[T+1][n]
int ref_linear_sequential(int32_t n, int32_t p, int64_t T, const double* A, const double* B, const double* w,
                          const double* G, double* actions, double* states) {
  return guarded([&] {
    const auto s = make_linear(n, p, T, A, B, w, G);
    linear::LinearEnv env(s);
    linear::GainPolicy pol(s);
    const auto steps = linear::make_steps(s);
    const auto r = sequential_simulate_with_states(env, pol, std::span<const linear::LinearStep>(steps));
    for (int64_t t = 0; t < T; ++t) std::memcpy(actions + (size_t)t * p, r.actions[(size_t)t].data(), sizeof(double) * p);
    for (int64_t t = 0; t <= T; ++t) std::memcpy(states + (size_t)t * n, r.states[(size_t)t].data(), sizeof(double) * n);
    return 0;
  });
}


// ---------------------------------------------------------------- linear env, MLP feedback
// The reference's MlpParams (mlp.cpp:141-169) as a PolicyFor<LinearEnv>
// (engine.hpp:57-61): a_t = forward(s_t). Test-only policy for BASELINE
// config 4 ("non-SCO env with MLP policy"); everything else is the unmodified
// reference (LinearEnv, make_steps, rollout_states, relative_rmse and the engine).
struct MlpFeedbackPolicy {
  static constexpr EvalCost cost_class = EvalCost::expensive;
  const MlpParams* mlp;
  std::vector<double> evaluate(const std::vector<double>& s, const linear::LinearStep&) const {
    std::vector<double> a(static_cast<std::size_t>(mlp->widths[3]));
    mlp->forward(s, a);
    return a;
  }
};
static_assert(PolicyFor<MlpFeedbackPolicy, linear::LinearEnv>);

static MlpParams make_lin_mlp(int32_t n, int32_t p, int32_t H, const double* w1, const double* b1,
                              const double* w2, const double* b2, const double* w3, const double* b3) {
  MlpParams m;
  m.widths = {n, H, H, p};
  m.w1.assign(w1, w1 + (size_t)H * n);
  m.b1.assign(b1, b1 + H);
  m.w2.assign(w2, w2 + (size_t)H * H);
  m.b2.assign(b2, b2 + H);
  m.w3.assign(w3, w3 + (size_t)p * H);
  m.b3.assign(b3, b3 + p);
  return m;
}

// picard_convergence_curve (linear.cpp:267-318) with MlpFeedbackPolicy in
// place of GainPolicy: the same statements, the policy type swapped.
int ref_linear_mlp_curve(int32_t n, int32_t p, int64_t T, const double* A, const double* B, const double* w,
                         int32_t H, const double* w1, const double* b1, const double* w2, const double* b2,
                         const double* w3, const double* b3, const double* init, double tolerance,
                         int64_t max_iterations, int32_t normalization, double* curve, int64_t cap, int64_t* len) {
  return guarded([&] {
    std::vector<double> G((size_t)p * n, 0.0);
    const auto spec = make_linear(n, p, T, A, B, w, G.data());
    const auto mlp = make_lin_mlp(n, p, H, w1, b1, w2, b2, w3, b3);
    linear::LinearEnv env(spec);
    MlpFeedbackPolicy policy{&mlp};
    const auto steps = linear::make_steps(spec);
    const std::int64_t horizon = spec.horizon;
    PartitionPlan plan;
    plan.processes = static_cast<std::int32_t>(std::max<std::int64_t>(1, horizon));
    plan.owner.resize(static_cast<std::size_t>(horizon));
    for (std::int64_t t = 0; t < horizon; ++t) plan.owner[(size_t)t] = static_cast<std::int32_t>(t);
    ActionCache<std::vector<double>> cache;
    if (init) {
      for (int64_t t = 0; t < T; ++t) cache.emplace_back(init + (size_t)t * p, init + (size_t)(t + 1) * p);
    } else {
      cache.assign(static_cast<std::size_t>(horizon), env.null_action());
    }
    const auto reference = sequential_simulate_with_states(env, policy, std::span<const linear::LinearStep>(steps));
    const auto draft = linear::rollout_states(spec, cache);
    auto score = [&](const std::vector<std::vector<double>>& states) {
      const std::span<const std::vector<double>> cand(states.begin() + 1, states.end());
      const std::span<const std::vector<double>> ref(reference.states.begin() + 1, reference.states.end());
      if (normalization) {
        const std::span<const std::vector<double>> base(draft.begin() + 1, draft.end());
        return linear::relative_rmse(cand, ref, base);
      }
      return linear::relative_rmse(cand, ref);
    };
    const std::int64_t capit = max_iterations > 0 ? max_iterations : horizon;
    const auto checkpoint = env.initial_state();
    std::vector<double> c;
    for (std::int64_t k = 1; k <= capit; ++k) {
      picard_iterate_once(env, policy, std::span<const linear::LinearStep>(steps), plan, cache, 0, horizon,
                          checkpoint);
      c.push_back(score(linear::rollout_states(spec, cache)));
      if (c.back() <= tolerance) break;
    }
    *len = (int64_t)c.size();
    for (size_t k = 0; k < c.size() && (int64_t)k < cap; ++k) curve[k] = c[k];
    return 0;
  });
}

// sequential_simulate_with_states of (LinearEnv, MlpFeedbackPolicy): actions[T][p], states[T+1][n]
int ref_linear_mlp_sequential(int32_t n, int32_t p, int64_t T, const double* A, const double* B, const double* w,
                              int32_t H, const double* w1, const double* b1, const double* w2, const double* b2,
                              const double* w3, const double* b3, double* actions, double* states) {
  return guarded([&] {
    std::vector<double> G((size_t)p * n, 0.0);
    const auto spec = make_linear(n, p, T, A, B, w, G.data());
    const auto mlp = make_lin_mlp(n, p, H, w1, b1, w2, b2, w3, b3);
    linear::LinearEnv env(spec);
    MlpFeedbackPolicy pol{&mlp};
    const auto steps = linear::make_steps(spec);
    const auto r = sequential_simulate_with_states(env, pol, std::span<const linear::LinearStep>(steps));
    for (int64_t t = 0; t < T; ++t) std::memcpy(actions + (size_t)t * p, r.actions[(size_t)t].data(), sizeof(double) * p);
    for (int64_t t = 0; t <= T; ++t) std::memcpy(states + (size_t)t * n, r.states[(size_t)t].data(), sizeof(double) * n);
    return 0;
  });
}

// picard_simulate (engine.hpp:458-590) of (LinearEnv, MlpFeedbackPolicy) with
// the single-step plan (M = T) and the whole horizon as window:
// iterations_to_converged and the converged actions[T][p]
int ref_linear_mlp_picard(int32_t n, int32_t p, int64_t T, const double* A, const double* B, const double* w,
                          int32_t H, const double* w1, const double* b1, const double* w2, const double* b2,
                          const double* w3, const double* b3, const double* init, int32_t threads,
                          int64_t* iterations, double* actions) {
  return guarded([&] {
    std::vector<double> G((size_t)p * n, 0.0);
    const auto spec = make_linear(n, p, T, A, B, w, G.data());
    const auto mlp = make_lin_mlp(n, p, H, w1, b1, w2, b2, w3, b3);
    linear::LinearEnv env(spec);
    MlpFeedbackPolicy pol{&mlp};
    const auto steps = linear::make_steps(spec);
    PartitionPlan plan;
    plan.processes = static_cast<std::int32_t>(std::max<std::int64_t>(1, T));
    plan.owner.resize(static_cast<std::size_t>(T));
    for (std::int64_t t = 0; t < T; ++t) plan.owner[(size_t)t] = static_cast<std::int32_t>(t);
    std::vector<std::vector<double>> ic;
    if (init)
      for (int64_t t = 0; t < T; ++t) ic.emplace_back(init + (size_t)t * p, init + (size_t)(t + 1) * p);
    PicardConfig cfg;
    cfg.threads = threads;
    const auto r = picard_simulate(env, pol, std::span<const linear::LinearStep>(steps), plan, cfg,
                                   std::span<const std::vector<double>>(ic));
    *iterations = r.iterations_to_converged;
    for (int64_t t = 0; t < T; ++t) std::memcpy(actions + (size_t)t * p, r.actions[(size_t)t].data(), sizeof(double) * p);
    return 0;
  });
}

}  // extern "C"
