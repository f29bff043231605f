// picard_b200.hpp — C++ drop-in for the reference's serial and Picard
// simulation paths, running on the B200 engine through the C ABI
// (picard_b200.h). Include it AFTER the reference headers:
//
//   #include "picard/engine.hpp"
//   #include "picard/fo/policies.hpp"
//   #include "picard_b200.hpp"
//
//   auto r = picard::b200::picard_simulate(env, policy, orders, plan, config,
//                                          initial_cache, reference_actions);
//
// Same argument meanings, same PicardResult / IterationOutcome /
// SequentialOutput, same exception types as
//   picard::picard_simulate      engine.hpp:458-590
//   picard::picard_iterate_once  engine.hpp:358-444
//   picard::sequential_simulate  engine.hpp:237-267
// and, when the reference's headers are on the include path,
//   picard::timewarp::time_warp_simulate    fo/timewarp.hpp:56-181
//   picard::linear::picard_convergence_curve linear.cpp:279-330
// for FoEnv x {GreedyPolicy, CapacityPenalizedPolicy, DualNetworkPolicy}.
//
// Observers (engine.hpp:194-223) keep the reference's call shapes:
//   * SequentialObserver (on_state) on sequential_simulate: the device
//     computes the trajectory, then the states are replayed on the host with
//     the reference's own FoLocalState (a state is a pure function of the
//     action prefix), so the observer sees every state entering t in [0, T];
//     sequential_simulate_with_states is built on it exactly as in the
//     reference (engine.hpp:277-291);
//   * IterationObserver (on_iteration, e.g. theory::CacheTraceRecorder) on
//     picard_simulate: the device records the cache after every iteration
//     (pcd_set_history) and the callbacks are delivered in iteration order
//     after the run, with the reference's (iteration, chunk, lo, hi, cache);
//   * LocalStateObserver (on_local_state, e.g. theory::MonotonicityChecker)
//     needs every process's local state at every step on the host: refused
//     with ContractViolation.
//
// DualNetworkPolicy keeps its normalisation state (initial_, horizon_)
// private; every reference call site builds it from the instance's initial
// state and horizon (cli.cpp:324-349, tests), which is what the adapter
// assumes. Pass DeviceOptions{DualNormalization{...}} to state it
// explicitly (and the CUDA device), after the reference's own arguments.
#pragma once

#include <cstdint>
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "picard_b200.h"

namespace picard::b200 {

struct DualNormalization {
  const fo::FoState* initial = nullptr;  // DualNetworkPolicy::initial_ (nullptr: env initial)
  std::int64_t horizon = -1;             // DualNetworkPolicy::horizon_ (-1: orders.size())
};

// Adapter arguments beyond the reference signatures (always last).
struct DeviceOptions {
  DualNormalization norm{};
  int device = 0;
};

namespace detail {

// SoA marshalling of the reference's AoS instance (fo/types.hpp:26-31):
// per-order reward vectors are deduplicated into a table (generated
// instances have one distinct vector per origin node, instance.cpp:100-105).
struct Marshalled {
  std::int32_t J = 0, I = 0;
  std::vector<std::int32_t> product, order_t, reward_row, capacity, inventory;
  std::vector<double> reward_table;
  pcd_instance view{};
};

inline void dense_state(const fo::FoState& s, std::int32_t J, std::int32_t I, std::vector<std::int32_t>& cap,
                        std::vector<std::int32_t>& inv) {
  cap.assign(s.capacity.begin(), s.capacity.end());
  inv.assign(static_cast<std::size_t>(I) * J, 0);
  for (const auto& [p, row] : s.inventory)
    for (std::int32_t j = 0; j < J && j < static_cast<std::int32_t>(row.size()); ++j)
      inv[static_cast<std::size_t>(p) * J + j] = row[static_cast<std::size_t>(j)];
}

inline Marshalled marshal(const fo::FoEnv& env, std::span<const fo::Order> orders) {
  Marshalled m;
  m.J = env.node_count();
  m.I = env.product_count();
  const auto init = env.initial_state();
  dense_state(init, m.J, m.I, m.capacity, m.inventory);
  struct VecHash {
    std::size_t operator()(const std::vector<double>& v) const noexcept {
      std::size_t h = 1469598103934665603ull;
      for (double x : v) {
        std::uint64_t b;
        std::memcpy(&b, &x, 8);
        h = (h ^ b) * 1099511628211ull;
      }
      return h;
    }
  };
  std::unordered_map<std::vector<double>, std::int32_t, VecHash> rows;
  m.product.reserve(orders.size());
  m.order_t.reserve(orders.size());
  m.reward_row.reserve(orders.size());
  for (const auto& o : orders) {
    if (static_cast<std::int32_t>(o.rewards.size()) != m.J)
      throw std::invalid_argument("order reward vector length differs from the node count");
    auto [it, fresh] = rows.emplace(o.rewards, static_cast<std::int32_t>(rows.size()));
    if (fresh) m.reward_table.insert(m.reward_table.end(), o.rewards.begin(), o.rewards.end());
    m.product.push_back(o.product);
    m.order_t.push_back(o.t);
    m.reward_row.push_back(it->second);
  }
  if (m.reward_table.empty()) m.reward_table.assign(static_cast<std::size_t>(m.J), 0.0);
  m.view = pcd_instance{m.J,
                        m.I,
                        static_cast<std::int64_t>(orders.size()),
                        m.product.data(),
                        m.order_t.data(),
                        m.reward_row.data(),
                        m.reward_table.data(),
                        static_cast<std::int64_t>(m.reward_table.size() / static_cast<std::size_t>(m.J)),
                        m.capacity.data(),
                        m.inventory.data()};
  return m;
}

struct PolicySpec {
  pcd_policy view{};
  std::vector<std::int32_t> init_cap, init_inv;
};

inline PolicySpec policy_spec(const fo::GreedyPolicy&, const Marshalled&, const DualNormalization&) {
  PolicySpec s;
  s.view = pcd_policy{PCD_POLICY_GREEDY, 64, 0.0, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, -1};
  return s;
}
inline PolicySpec policy_spec(const fo::CapacityPenalizedPolicy& p, const Marshalled&, const DualNormalization&) {
  PolicySpec s;
  s.view = pcd_policy{PCD_POLICY_CAPACITY, 64, p.gamma, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                      nullptr, nullptr, -1};
  return s;
}
inline PolicySpec policy_spec(const fo::DualNetworkPolicy& p, const Marshalled& m, const DualNormalization& n) {
  PolicySpec s;
  const auto& w = p.params();
  if (w.widths.size() != 4 || w.widths[1] != w.widths[2])
    throw std::invalid_argument("dual network: unsupported layer widths");
  s.view = pcd_policy{PCD_POLICY_DUAL, w.widths[1], 0.0, w.w1.data(), w.b1.data(), w.w2.data(), w.b2.data(),
                      w.w3.data(), w.b3.data(), nullptr, nullptr, n.horizon};
  if (n.initial) {
    dense_state(*n.initial, m.J, m.I, s.init_cap, s.init_inv);
    s.view.init_capacity = s.init_cap.data();
    s.view.init_inventory = s.init_inv.data();
  }
  return s;
}

// Status code -> the reference's exception types (errors.hpp, engine.hpp:140-156).
[[noreturn]] inline void raise(int rc, const pcd_result* res = nullptr,
                               const std::vector<pcd_trace_row>* trace = nullptr) {
  const std::string msg = pcd_last_error();
  if (rc == PCD_CONTRACT_VIOLATION) throw ContractViolation(msg, pcd_last_error_time_step());
  if (rc == PCD_ITERATION_LIMIT) {
    std::vector<PicardTraceRow> rows;
    if (res && trace)
      for (std::int64_t i = 0; i < res->trace_rows && i < static_cast<std::int64_t>(trace->size()); ++i) {
        const auto& t = (*trace)[static_cast<std::size_t>(i)];
        rows.push_back({t.chunk, t.iteration, t.changed_slots, t.max_process_evals, t.t_reset});
      }
    throw IterationLimitError(msg, res ? res->iterations_run : 0, std::move(rows));
  }
  if (rc == PCD_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);  // PCD_CUDA_ERROR: no CPU fallback exists
}

struct Handle {
  pcd_handle* h = nullptr;
  Handle(const pcd_instance& in, const pcd_policy& p, int device) {
    const int rc = pcd_create(&in, &p, device, &h);
    if (rc) raise(rc);
  }
  ~Handle() { pcd_destroy(h); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
};

inline std::vector<std::int32_t> nodes_of(std::span<const fo::FoAction> a) {
  std::vector<std::int32_t> v;
  v.reserve(a.size());
  for (const auto& x : a) v.push_back(x.node);
  return v;
}

}  // namespace detail

namespace detail {
template <typename Obs>
void refuse_local_state_observer(Obs* observer) {
  if constexpr (LocalStateObserver<Obs, fo::FoEnv>) {
    if (observer != nullptr)
      throw ContractViolation(
          "local-state observers need every process's state at every step on the host; "
          "the B200 device path does not support them");
  }
}
}  // namespace detail

// picard_simulate (engine.hpp:458-590) on the B200. Same arguments as the
// reference (observer included, see the header comment), then DeviceOptions.
template <typename P, typename Obs = NoObserver>
PicardResult<fo::FoAction> picard_simulate(const fo::FoEnv& env, const P& policy,
                                           std::span<const fo::Order> orders, const PartitionPlan& plan,
                                           const PicardConfig& config = {},
                                           std::span<const fo::FoAction> initial_cache = {},
                                           std::span<const fo::FoAction> reference_actions = {},
                                           Obs* observer = nullptr, const DeviceOptions& opts = {}) {
  detail::refuse_local_state_observer(observer);
  const std::int64_t T = static_cast<std::int64_t>(orders.size());
  if (static_cast<std::int64_t>(plan.owner.size()) != T)
    throw ContractViolation("partition plan does not cover the horizon");
  if (!initial_cache.empty() && static_cast<std::int64_t>(initial_cache.size()) != T)
    throw ContractViolation("initial cache length must equal the horizon");
  if (!reference_actions.empty() && static_cast<std::int64_t>(reference_actions.size()) != T)
    throw ContractViolation("reference action length must equal the horizon");
  auto m = detail::marshal(env, orders);
  auto ps = detail::policy_spec(policy, m, opts.norm);
  detail::Handle h(m.view, ps.view, opts.device);
  int rc = pcd_set_plan(h.h, plan.owner.data(), plan.processes);
  if (rc) detail::raise(rc);
  constexpr bool wants_iterations = IterationObserver<Obs, fo::FoEnv>;
  const bool observe = wants_iterations && observer != nullptr;
  const bool trace_on = config.record_trace || observe;  // the callbacks need (chunk, lo) per iteration
  const pcd_config cfg{config.processes, trace_on ? 1 : 0, config.max_steps, config.max_iterations,
                       config.threads, PCD_ENGINE_AUTO, 0.0, 0, 0, 0};
  const auto init = detail::nodes_of(initial_cache);
  const auto ref = detail::nodes_of(reference_actions);
  std::vector<std::int32_t> actions(static_cast<std::size_t>(T));
  std::vector<pcd_trace_row> trace(trace_on ? static_cast<std::size_t>(4 * T + 16) : 1);
  pcd_result res{};
  auto run = [&] {
    return pcd_simulate(h.h, &cfg, init.empty() ? nullptr : init.data(), ref.empty() ? nullptr : ref.data(),
                        actions.data(), &res, trace.data(), trace_on ? static_cast<std::int64_t>(trace.size()) : 0);
  };
  rc = run();
  if (rc) detail::raise(rc, &res, &trace);
  std::vector<std::int32_t> history;
  if (observe && T > 0) {  // the run is deterministic: repeat it recording the cache after every iteration
    const std::int64_t k = res.iterations_run;
    history.assign(static_cast<std::size_t>(k * T), 0);
    rc = pcd_set_history(h.h, history.data(), k);
    if (rc == PCD_OK) rc = run();
    pcd_set_history(h.h, nullptr, 0);
    if (rc) detail::raise(rc, &res, &trace);
  }
  PicardResult<fo::FoAction> out;
  out.actions.reserve(actions.size());
  for (auto a : actions) out.actions.push_back(fo::FoAction{a});
  out.iterations_to_converged = res.iterations_to_converged;
  if (res.iterations_to_correct >= 0) out.iterations_to_correct = res.iterations_to_correct;
  out.conflicts = res.conflicts;
  out.policy_eval_count_sequential_equivalent = res.policy_eval_count_sequential_equivalent;
  out.total_policy_evals = res.total_policy_evals;
  for (std::int64_t i = 0; i < res.trace_rows && config.record_trace; ++i) {
    const auto& t = trace[static_cast<std::size_t>(i)];
    out.trace.push_back({t.chunk, t.iteration, t.changed_slots, t.max_process_evals, t.t_reset});
  }
  if constexpr (wants_iterations) {
    if (observe) {
      std::vector<fo::FoAction> cache(static_cast<std::size_t>(T));
      for (std::int64_t i = 0; i < res.trace_rows && i < res.iterations_run; ++i) {
        const auto& row = trace[static_cast<std::size_t>(i)];
        const std::int64_t hi = config.max_steps > 0 ? std::min(T, row.t_reset + config.max_steps) : T;
        for (std::int64_t t = 0; t < T; ++t)
          cache[static_cast<std::size_t>(t)] = fo::FoAction{history[static_cast<std::size_t>(i * T + t)]};
        observer->on_iteration(row.iteration, row.chunk, row.t_reset, hi, std::span<const fo::FoAction>(cache));
      }
    }
  }
  return out;
}

// picard_iterate_once (engine.hpp:358-444) on the B200; `cache` updated in place.
template <typename P, typename Obs = NoObserver>
IterationOutcome picard_iterate_once(const fo::FoEnv& env, const P& policy, std::span<const fo::Order> orders,
                                     const PartitionPlan& plan, ActionCache<fo::FoAction>& cache,
                                     std::int64_t t_lo, std::int64_t t_hi, const fo::FoState& checkpoint_state,
                                     const IterateOptions& options = {}, Obs* observer = nullptr,
                                     std::int64_t iteration = 0, const DeviceOptions& opts = {}) {
  (void)options;    // IterateOptions::threads: the device ignores it
  (void)iteration;  // only passed on to local-state observers, which are refused
  detail::refuse_local_state_observer(observer);
  auto m = detail::marshal(env, orders);
  auto ps = detail::policy_spec(policy, m, opts.norm);
  detail::Handle h(m.view, ps.view, opts.device);
  int rc = pcd_set_plan(h.h, plan.owner.data(), plan.processes);
  if (rc) detail::raise(rc);
  std::vector<std::int32_t> ck_cap, ck_inv;
  detail::dense_state(checkpoint_state, m.J, m.I, ck_cap, ck_inv);
  auto c = detail::nodes_of(cache);
  IterationOutcome out;
  out.evals_per_process.assign(static_cast<std::size_t>(plan.processes), 0);
  std::vector<std::int64_t> changed(std::max<std::size_t>(cache.size(), 1));
  std::int64_t n = 0;
  rc = pcd_iterate_once(h.h, PCD_ENGINE_AUTO, c.data(), t_lo, t_hi, ck_cap.data(), ck_inv.data(),
                        reinterpret_cast<std::int64_t*>(out.evals_per_process.data()), changed.data(), &n);
  if (rc) detail::raise(rc);
  for (std::size_t t = 0; t < cache.size(); ++t) cache[t] = fo::FoAction{c[t]};
  out.changed_slots.assign(changed.begin(), changed.begin() + n);
  return out;
}

// sequential_simulate (engine.hpp:237-267): the serial trajectory, computed
// on the device as the Picard fixed point (Prop. 1); policy_evals = T. A
// SequentialObserver sees the states entering every t in [0, T], replayed on
// the host with the reference's FoLocalState from the device's actions.
template <typename P, typename Obs = NoObserver>
SequentialOutput<fo::FoAction> sequential_simulate(const fo::FoEnv& env, const P& policy,
                                                   std::span<const fo::Order> orders, Obs* observer = nullptr,
                                                   const DeviceOptions& opts = {}) {
  auto m = detail::marshal(env, orders);
  auto ps = detail::policy_spec(policy, m, opts.norm);
  detail::Handle h(m.view, ps.view, opts.device);
  std::vector<std::int32_t> actions(orders.size());
  std::int64_t evals = 0;
  const int rc = pcd_sequential(h.h, actions.data(), &evals);
  if (rc) detail::raise(rc);
  SequentialOutput<fo::FoAction> out;
  for (auto a : actions) out.actions.push_back(fo::FoAction{a});
  out.policy_evals = evals;
  if constexpr (SequentialObserver<Obs, fo::FoEnv>) {
    if (observer != nullptr) {
      auto local = env.make_local();
      const auto start = env.initial_state();
      env.reset_local(local, start);
      for (std::size_t t = 0; t < orders.size(); ++t) {
        observer->on_state(static_cast<std::int64_t>(t), local);
        env.apply_local(local, out.actions[t], orders[t]);
      }
      observer->on_state(static_cast<std::int64_t>(orders.size()), local);
    }
  }
  return out;
}

// sequential_simulate_with_states (engine.hpp:277-291): actions plus the
// state entering every step (size T + 1), through the observer path above.
template <typename P>
SequentialTrajectory<fo::FoEnv> sequential_simulate_with_states(const fo::FoEnv& env, const P& policy,
                                                                std::span<const fo::Order> orders,
                                                                const DeviceOptions& opts = {}) {
  struct Recorder {
    const fo::FoEnv* env;
    std::vector<fo::FoState> states;
    void on_state(std::int64_t, const fo::FoLocalState& local) { states.push_back(env->snapshot(local)); }
  } recorder{&env, {}};
  recorder.states.reserve(orders.size() + 1);
  auto out = sequential_simulate(env, policy, orders, &recorder, opts);
  return {std::move(out.actions), std::move(recorder.states)};
}

#if __has_include("picard/fo/timewarp.hpp")
}  // namespace picard::b200
#include "picard/fo/timewarp.hpp"
namespace picard::b200 {
// timewarp::time_warp_simulate (fo/timewarp.hpp:56-181) on the B200: same
// arguments, same TimeWarpResult (actions, counters, trace), same errors.
template <typename P>
timewarp::TimeWarpResult time_warp_simulate(const fo::Instance& instance, const P& policy, std::int32_t processes,
                                            std::uint64_t seed, bool record_trace = false,
                                            timewarp::WindowRule rule = timewarp::WindowRule::min_capacity,
                                            const DeviceOptions& opts = {}) {
  const auto env = instance.make_env();
  const std::span<const fo::Order> orders(instance.orders);
  auto m = detail::marshal(env, orders);
  auto ps = detail::policy_spec(policy, m, opts.norm);
  detail::Handle h(m.view, ps.view, opts.device);
  std::vector<std::int32_t> actions(orders.size());
  std::vector<pcd_tw_trace_row> rows(record_trace ? 2 * orders.size() + 4 : 1);
  pcd_tw_result res{};
  const int rc = pcd_time_warp(h.h, processes, seed, rule == timewarp::WindowRule::min_stocked_capacity ? 1 : 0,
                               record_trace ? 1 : 0, actions.data(), &res, rows.data(),
                               record_trace ? static_cast<std::int64_t>(rows.size()) : 0);
  if (rc) detail::raise(rc);
  timewarp::TimeWarpResult out;
  for (auto a : actions) out.actions.push_back(fo::FoAction{a});
  out.sync_rounds = res.sync_rounds;
  out.rollbacks = res.rollbacks;
  out.policy_eval_count_sequential_equivalent = res.policy_eval_count_sequential_equivalent;
  out.total_policy_evals = res.total_policy_evals;
  if (record_trace)
    for (std::int64_t i = 0; i < res.trace_rows && i < static_cast<std::int64_t>(rows.size()); ++i) {
      const auto& r = rows[static_cast<std::size_t>(i)];
      out.trace.push_back({r.round, r.t_start, r.window_length, r.max_process_evals, r.rolled_back != 0});
    }
  return out;
}
#endif

#if __has_include("picard/linear.hpp")
}  // namespace picard::b200
#include "picard/linear.hpp"
namespace picard::b200 {
// linear::picard_convergence_curve (linear.cpp:279-330) on the B200: the
// GainPolicy system under single-step partitions, one affine time-scan per
// iteration; curve values within 1e-9 relative of the reference's.
inline std::vector<double> picard_convergence_curve(const linear::LinearSystemSpec& spec,
                                                    std::span<const std::vector<double>> initial_cache = {},
                                                    const linear::ConvergenceCurveOptions& options = {},
                                                    int device = 0) {
  spec.validate();
  const auto n = static_cast<std::size_t>(spec.state_dim), p = static_cast<std::size_t>(spec.input_dim);
  const auto T = static_cast<std::size_t>(spec.horizon);
  std::vector<double> A, B, W, init;
  A.reserve(T * n * n);
  B.reserve(T * n * p);
  W.reserve(T * n);
  for (std::size_t t = 0; t < T; ++t) {
    A.insert(A.end(), spec.dynamics[t].begin(), spec.dynamics[t].end());
    B.insert(B.end(), spec.input[t].begin(), spec.input[t].end());
    W.insert(W.end(), spec.disturbances[t].begin(), spec.disturbances[t].end());
  }
  if (!initial_cache.empty()) {
    if (initial_cache.size() != T) throw ContractViolation("initial cache length must equal the horizon");
    for (const auto& a : initial_cache) init.insert(init.end(), a.begin(), a.end());
  }
  const pcd_linear_spec c{spec.state_dim, spec.input_dim, spec.horizon, A.data(), B.data(), W.data(),
                          spec.gain.data()};
  const std::int64_t cap = options.max_iterations > 0 ? options.max_iterations : spec.horizon;
  std::vector<double> curve(static_cast<std::size_t>(std::max<std::int64_t>(cap, 1)));
  std::int64_t len = 0;
  const int rc = pcd_linear_convergence_curve(
      &c, init.empty() ? nullptr : init.data(), options.tolerance, options.max_iterations,
      options.normalization == linear::RmseNormalization::draft ? 1 : 0, device, curve.data(),
      static_cast<std::int64_t>(curve.size()), &len, nullptr, nullptr);
  if (rc) detail::raise(rc);
  curve.resize(static_cast<std::size_t>(len));
  return curve;
}

// The same curve with the reference's MlpParams as the linear env's feedback
// policy, a_t = mlp.forward(s_t) (no reference counterpart: BASELINE config 4's
// "non-SCO env with MLP policy"; pcd_linear_mlp_convergence_curve). `mlp` has
// widths {state_dim, hidden, hidden, input_dim}. Also returns, through the
// optional pointer, picard_simulate's iterations_to_converged for the
// single-step plan.
inline std::vector<double> picard_convergence_curve(const linear::LinearSystemSpec& spec, const fo::MlpParams& mlp,
                                                    std::span<const std::vector<double>> initial_cache = {},
                                                    const linear::ConvergenceCurveOptions& options = {},
                                                    std::int64_t* iterations_to_converged = nullptr,
                                                    int device = 0) {
  spec.validate();
  if (mlp.widths.size() != 4 || mlp.widths[0] != spec.state_dim || mlp.widths[3] != spec.input_dim ||
      mlp.widths[1] != mlp.widths[2])
    throw std::invalid_argument("mlp widths must be {state_dim, hidden, hidden, input_dim}");
  const auto n = static_cast<std::size_t>(spec.state_dim), p = static_cast<std::size_t>(spec.input_dim);
  const auto T = static_cast<std::size_t>(spec.horizon);
  std::vector<double> A, B, W, init;
  A.reserve(T * n * n);
  B.reserve(T * n * p);
  W.reserve(T * n);
  for (std::size_t t = 0; t < T; ++t) {
    A.insert(A.end(), spec.dynamics[t].begin(), spec.dynamics[t].end());
    B.insert(B.end(), spec.input[t].begin(), spec.input[t].end());
    W.insert(W.end(), spec.disturbances[t].begin(), spec.disturbances[t].end());
  }
  if (!initial_cache.empty()) {
    if (initial_cache.size() != T) throw ContractViolation("initial cache length must equal the horizon");
    for (const auto& a : initial_cache) init.insert(init.end(), a.begin(), a.end());
  }
  const pcd_linear_spec c{spec.state_dim, spec.input_dim, spec.horizon, A.data(), B.data(), W.data(),
                          spec.gain.data()};
  const pcd_linear_mlp m{mlp.widths[1], 0, mlp.w1.data(), mlp.b1.data(), mlp.w2.data(), mlp.b2.data(),
                         mlp.w3.data(), mlp.b3.data()};
  const std::int64_t cap = options.max_iterations > 0 ? options.max_iterations : spec.horizon;
  std::vector<double> curve(static_cast<std::size_t>(std::max<std::int64_t>(cap, 1)));
  pcd_linear_mlp_result res{};
  const int rc = pcd_linear_mlp_convergence_curve(
      &c, &m, init.empty() ? nullptr : init.data(), options.tolerance, options.max_iterations,
      options.normalization == linear::RmseNormalization::draft ? 1 : 0, device, curve.data(),
      static_cast<std::int64_t>(curve.size()), &res, nullptr, nullptr);
  if (rc) detail::raise(rc);
  curve.resize(static_cast<std::size_t>(res.curve_len));
  if (iterations_to_converged) *iterations_to_converged = res.iterations_to_converged;
  return curve;
}
#endif

// Product-chunk plan (no reference counterpart; pcd_product_chunk_partition):
// every product's orders cut into contiguous near-equal chunks, one process
// each, so up to `processes` processes carry work. A valid PartitionPlan for
// picard_simulate (same trajectory); falls back to make_product_partition
// when processes < ordered products.
inline PartitionPlan make_product_chunk_partition(const fo::FoEnv& env, std::span<const fo::Order> orders,
                                                  std::int32_t processes, std::uint64_t seed = 1) {
  auto m = detail::marshal(env, orders);
  PartitionPlan plan;
  plan.processes = processes;
  plan.owner.assign(orders.size(), 0);
  const int rc = pcd_product_chunk_partition(&m.view, processes, seed, plan.owner.data());
  if (rc) detail::raise(rc);
  return plan;
}

// Window-aware product chunks (no reference counterpart;
// pcd_product_window_partition): every window of `window` slots holds at most
// L orders of any one process, L minimal for `processes` chunks. A valid
// PartitionPlan for picard_simulate (same trajectory), tuned for
// PicardConfig::max_steps = window.
inline PartitionPlan make_product_window_partition(const fo::FoEnv& env, std::span<const fo::Order> orders,
                                                   std::int32_t processes, std::int64_t window,
                                                   std::uint64_t seed = 1) {
  auto m = detail::marshal(env, orders);
  PartitionPlan plan;
  plan.processes = processes;
  plan.owner.assign(orders.size(), 0);
  const int rc = pcd_product_window_partition(&m.view, processes, window, seed, plan.owner.data());
  if (rc) detail::raise(rc);
  return plan;
}

}  // namespace picard::b200
