// dropin_test.cpp — the reference's own engine scenarios driven through the
// B200 drop-in (include/picard_b200.hpp) and checked against the UNMODIFIED
// reference CPU engine (compiled from /root/reference/proj). Restates the
// engine cases of test_engine.cpp (:81-138, :140-173, :301-348, :350-371,
// :395-414, :455-477, :525-545) with the same fixtures (test_helpers.hpp).
// Build: make -C tests/cpp (here, where the reference tree exists); the
// binary travels to the GPU box. Exit code = number of failed checks.
#include <cstdio>
#include <memory>
#include <span>
#include <vector>

#include "picard/engine.hpp"
#include "picard/fo/env.hpp"
#include "picard/fo/instance.hpp"
#include "picard/fo/policies.hpp"
#include "picard/rng.hpp"
#include "picard/theory.hpp"
#include "picard_b200.hpp"

using namespace picard;
using namespace picard::fo;

static int failures = 0, checks = 0;
#define CHECK(c)                                                             \
  do {                                                                       \
    ++checks;                                                                \
    if (!(c)) {                                                              \
      ++failures;                                                            \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);    \
    }                                                                        \
  } while (0)

static Instance toy() {  // test_helpers.hpp:17-29 (fixture restated)
  Instance inst;
  inst.nodes = 2;
  inst.products = 1;
  inst.horizon = 2;
  inst.initial.capacity = {1, 1};
  inst.initial.inventory[0] = {1, 1};
  inst.orders.resize(2);
  inst.orders[0] = {0, 0, 0, {0.9, 0.1}};
  inst.orders[1] = {1, 0, 0, {0.8, 0.2}};
  return inst;
}

static Instance small_random(std::uint64_t seed) {  // test_helpers.hpp:31-41
  auto gen = rng::make(seed);
  const auto nodes = static_cast<std::int32_t>(2 + rng::below(gen, 4));
  const auto products = static_cast<std::int32_t>(1 + rng::below(gen, 12));
  const auto horizon = static_cast<std::int64_t>(1 + rng::below(gen, 60));
  const double beta = -static_cast<double>(rng::below(gen, 11)) / 10.0;
  const double coverage = 0.5 + 0.5 * rng::unit(gen);
  return generate_instance(nodes, products, horizon, beta, coverage, seed ^ 0x9e3779b97f4a7c15ull);
}

template <typename P>
static void compare(const Instance& inst, const P& policy, const PartitionPlan& plan, PicardConfig cfg,
                    std::span<const FoAction> init = {}) {
  const auto env = inst.make_env();
  const std::span<const Order> orders(inst.orders);
  const auto oracle = sequential_simulate(env, policy, orders);
  cfg.record_trace = true;
  const auto want = picard_simulate(env, policy, orders, plan, cfg, init, std::span<const FoAction>(oracle.actions));
  const auto got = b200::picard_simulate(env, policy, orders, plan, cfg, init, std::span<const FoAction>(oracle.actions));
  CHECK(got.actions == want.actions);
  CHECK(got.actions == oracle.actions);
  CHECK(got.iterations_to_converged == want.iterations_to_converged);
  CHECK(got.iterations_to_correct == want.iterations_to_correct);
  CHECK(got.conflicts == want.conflicts);
  CHECK(got.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent);
  CHECK(got.total_policy_evals == want.total_policy_evals);
  CHECK(got.trace.size() == want.trace.size());
  for (std::size_t i = 0; i < std::min(got.trace.size(), want.trace.size()); ++i) {
    CHECK(got.trace[i].iteration == want.trace[i].iteration);
    CHECK(got.trace[i].changed_slots == want.trace[i].changed_slots);
    CHECK(got.trace[i].max_process_evals == want.trace[i].max_process_evals);
    CHECK(got.trace[i].t_reset == want.trace[i].t_reset);
    CHECK(got.trace[i].chunk == want.trace[i].chunk);
  }
  const auto seq = b200::sequential_simulate(env, policy, orders);
  CHECK(seq.actions == oracle.actions);
  CHECK(seq.policy_evals == oracle.policy_evals);
}

// the reference's MlpParams as a PolicyFor<linear::LinearEnv> (engine.hpp:57-61)
struct MlpFeedback {
  static constexpr picard::EvalCost cost_class = picard::EvalCost::expensive;
  const picard::fo::MlpParams* m;
  std::vector<double> evaluate(const std::vector<double>& s, const picard::linear::LinearStep&) const {
    std::vector<double> a(static_cast<std::size_t>(m->widths[3]));
    m->forward(s, a);
    return a;
  }
};

int main() {
  // toy two-process hand trace (test_engine.cpp:100-138)
  {
    const auto inst = toy();
    const auto env = inst.make_env();
    PartitionPlan plan;
    plan.processes = 2;
    plan.owner = {0, 1};
    ActionCache<FoAction> cache(2, kNoFulfill);
    const auto first = b200::picard_iterate_once(env, GreedyPolicy{}, std::span<const Order>(inst.orders), plan,
                                                 cache, 0, 2, env.initial_state());
    CHECK(cache[0] == FoAction{0});
    CHECK(cache[1] == FoAction{0});
    CHECK(first.changed_slots == (std::vector<std::int64_t>{0, 1}));
    CHECK(first.evals_per_process == (std::vector<std::int64_t>{1, 1}));
    compare(inst, GreedyPolicy{}, plan, {});
  }
  // infeasible cached action degrades to declining (test_engine.cpp:140-173)
  {
    Instance inst;
    inst.nodes = 1;
    inst.products = 1;
    inst.horizon = 3;
    inst.initial.capacity = {1};
    inst.initial.inventory[0] = {3};
    for (std::int32_t t = 0; t < 3; ++t) inst.orders.push_back(Order{t, 0, 0, {1.0}});
    PartitionPlan plan;
    plan.processes = 2;
    plan.owner = {0, 1, 0};
    const std::vector<FoAction> over(3, FoAction{0});
    compare(inst, GreedyPolicy{}, plan, {}, std::span<const FoAction>(over));
  }
  // oracle equivalence grid (test_engine.cpp:301-348)
  for (std::uint64_t seed = 100; seed < 140; ++seed) {
    const auto inst = small_random(seed);
    auto gen = rng::make(seed * 977);
    const auto M = static_cast<std::int32_t>(1 + rng::below(gen, 8));
    const bool product = rng::below(gen, 2) == 0;
    const auto plan = product ? make_product_partition(inst, M, seed)
                              : make_uniform_time_partition(inst.horizon, M, seed);
    PicardConfig cfg;
    cfg.max_steps = static_cast<std::int64_t>(rng::below(gen, 3) == 0 ? 0 : 1 + rng::below(gen, 20));
    compare(inst, GreedyPolicy{}, plan, cfg);
    compare(inst, CapacityPenalizedPolicy{rng::unit(gen) * 2.0}, plan, cfg);
    if (seed % 4 == 0) compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, seed + 5), plan, cfg);
  }
  // warm starts with windows (test_engine.cpp:350-371, :395-414)
  for (std::uint64_t seed = 200; seed < 212; ++seed) {
    const auto inst = small_random(seed);
    const auto env = inst.make_env();
    const auto plan = make_product_partition(inst, 4, seed);
    const auto draft = sequential_simulate(env, CapacityPenalizedPolicy{1.0}, std::span<const Order>(inst.orders));
    for (std::int64_t ms : {0, 5}) {
      PicardConfig cfg;
      cfg.max_steps = ms;
      compare(inst, GreedyPolicy{}, plan, cfg, std::span<const FoAction>(draft.actions));
    }
  }
  // a J=30 dual run at a larger size (generated instance, product partition)
  {
    const auto inst = generate_instance(30, 200, 6000, -0.3, 0.8, 7);
    compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, 5),
            make_product_partition(inst, 64, 1), {});
    compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, 5),
            make_uniform_time_partition(inst.horizon, 16, 3), {});
  }
  // product-chunk plans (b200::make_product_chunk_partition) through the
  // unmodified reference engine and the B200 engine
  {
    const auto inst = generate_instance(30, 200, 6000, -0.3, 0.8, 7);
    const auto env = inst.make_env();
    const auto plan = b200::make_product_chunk_partition(env, std::span<const Order>(inst.orders), 900);
    compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, 5), plan, {});
    PicardConfig cfg;
    cfg.max_steps = 700;
    compare(inst, GreedyPolicy{}, plan, cfg);
  }
  // window-aware product chunks (b200::make_product_window_partition), at the
  // window they are cut for and at the whole horizon
  {
    const auto inst = generate_instance(30, 200, 6000, -0.3, 0.8, 7);
    const auto env = inst.make_env();
    const auto plan = b200::make_product_window_partition(env, std::span<const Order>(inst.orders), 900, 700);
    PicardConfig cfg;
    cfg.max_steps = 700;
    compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, 5), plan, cfg);
    compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, 5), plan, {});
    compare(inst, CapacityPenalizedPolicy{0.7}, plan, cfg);
  }
  for (std::uint64_t seed = 300; seed < 316; ++seed) {
    const auto inst = small_random(seed);
    const auto env = inst.make_env();
    auto gen = rng::make(seed * 31);
    const auto M = static_cast<std::int32_t>(inst.products + rng::below(gen, 3 * inst.products + 4));
    const auto plan = b200::make_product_chunk_partition(env, std::span<const Order>(inst.orders), M);
    compare(inst, CapacityPenalizedPolicy{0.7}, plan, {});
    if (seed % 2 == 0) compare(inst, DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, seed), plan, {});
  }
  // Time Warp (fo/timewarp.hpp) through the drop-in vs the unmodified reference
  for (std::uint64_t seed = 60; seed < 66; ++seed) {
    const auto inst = small_random(seed);
    for (auto rule : {timewarp::WindowRule::min_capacity, timewarp::WindowRule::min_stocked_capacity}) {
      auto check_tw = [&](const auto& policy) {
        const auto want = timewarp::time_warp_simulate(inst, policy, 4, seed, true, rule);
        const auto got = b200::time_warp_simulate(inst, policy, 4, seed, true, rule);
        CHECK(got.actions == want.actions);
        CHECK(got.sync_rounds == want.sync_rounds);
        CHECK(got.rollbacks == want.rollbacks);
        CHECK(got.policy_eval_count_sequential_equivalent == want.policy_eval_count_sequential_equivalent);
        CHECK(got.total_policy_evals == want.total_policy_evals);
        CHECK(got.trace.size() == want.trace.size());
        for (std::size_t i = 0; i < std::min(got.trace.size(), want.trace.size()); ++i) {
          CHECK(got.trace[i].t_start == want.trace[i].t_start);
          CHECK(got.trace[i].window_length == want.trace[i].window_length);
          CHECK(got.trace[i].max_process_evals == want.trace[i].max_process_evals);
          CHECK(got.trace[i].rolled_back == want.trace[i].rolled_back);
        }
      };
      check_tw(GreedyPolicy{});
      check_tw(CapacityPenalizedPolicy{5.0});
      check_tw(DualNetworkPolicy::seeded(inst.shared_initial(), inst.horizon, seed));
    }
  }
  // linear env convergence curve (linear.cpp:279-330) vs the unmodified reference
  for (double coupling : {0.0, 0.4}) {
    const auto spec = linear::make_contractive_spec(4, 3, 400, 0.6, 17, coupling);
    linear::ConvergenceCurveOptions o;
    o.tolerance = 1e-7;
    const auto want = linear::picard_convergence_curve(spec, {}, o);
    const auto got = b200::picard_convergence_curve(spec, {}, o);
    CHECK(got.size() == want.size());
    for (std::size_t k = 0; k < std::min(got.size(), want.size()); ++k)
      CHECK(std::abs(got[k] - want[k]) <= 1e-9 * std::max(1.0, std::abs(want[k])));
  }
  // linear env with the reference's MlpParams as the feedback policy (BASELINE
  // config 4): the device curve's iteration count equals the reference
  // picard_simulate's for the single-step plan
  {
    const auto spec = linear::make_contractive_spec(4, 3, 300, 0.6, 17, 0.3);
    auto mlp = MlpParams::seeded_uniform(4, 3, 5);
    for (auto& w : mlp.w3) w *= 20.0;
    for (auto& b : mlp.b3) b *= 20.0;
    linear::ConvergenceCurveOptions o;
    o.tolerance = 1e-7;
    std::int64_t it = -1;
    const auto got = b200::picard_convergence_curve(spec, mlp, {}, o, &it);
    const linear::LinearEnv lenv(spec);
    const auto steps = linear::make_steps(spec);
    PartitionPlan plan;
    plan.processes = static_cast<std::int32_t>(spec.horizon);
    for (std::int64_t t = 0; t < spec.horizon; ++t) plan.owner.push_back(static_cast<std::int32_t>(t));
    const auto ref = picard_simulate(lenv, MlpFeedback{&mlp}, std::span<const linear::LinearStep>(steps), plan);
    CHECK(it == ref.iterations_to_converged);
    CHECK(!got.empty() && got.back() <= 1e-7);
  }
  // iteration cap (test_engine.cpp:525-545)
  {
    const auto inst = toy();
    const auto env = inst.make_env();
    PartitionPlan plan;
    plan.processes = 2;
    plan.owner = {0, 1};
    PicardConfig cfg;
    cfg.max_iterations = 1;
    cfg.record_trace = true;
    bool thrown = false;
    try {
      b200::picard_simulate(env, GreedyPolicy{}, std::span<const Order>(inst.orders), plan, cfg);
    } catch (const IterationLimitError& e) {
      thrown = true;
      CHECK(e.iterations_run() == 1);
      CHECK(e.partial_trace().size() == 1);
    }
    CHECK(thrown);
    PartitionPlan bad;
    bad.processes = 2;
    bad.owner = {0, 5};
    bool cv = false;
    try {
      b200::picard_simulate(env, GreedyPolicy{}, std::span<const Order>(inst.orders), bad, {});
    } catch (const ContractViolation&) {
      cv = true;
    }
    CHECK(cv);
  }
  // the reference's full call shapes (engine.hpp:237-291, :358-365,
  // :458-465; theory.hpp:120-126, :160-216, :258-268)
  for (std::uint64_t seed = 900; seed < 912; ++seed) {
    const auto inst = small_random(seed);
    const auto env = inst.make_env();
    const std::span<const Order> orders(inst.orders);
    const auto plan = make_product_partition(inst, 3, seed);
    PicardConfig cfg;
    cfg.max_steps = seed % 3 == 0 ? 7 : 0;
    // IterationObserver: per-iteration caches (CacheTraceRecorder) in order
    theory::CacheTraceRecorder want_rec, got_rec;
    const auto want = picard_simulate(env, GreedyPolicy{}, orders, plan, cfg, {}, {}, &want_rec);
    const auto got = b200::picard_simulate(env, GreedyPolicy{}, orders, plan, cfg, {}, {}, &got_rec);
    CHECK(got.actions == want.actions);
    CHECK(got_rec.caches == want_rec.caches);
    CHECK(got.trace.empty());  // the observer's trace rows are not returned unless record_trace
    // evaluation_speedup_proxy on the drop-in's PicardResult
    if (want.policy_eval_count_sequential_equivalent > 0)
      CHECK(theory::evaluation_speedup_proxy(got, (std::int64_t)orders.size()) ==
            theory::evaluation_speedup_proxy(want, (std::int64_t)orders.size()));
    // SequentialObserver + sequential_simulate_with_states (states entering every t)
    theory::CapacityRecorder want_caps, got_caps;
    sequential_simulate(env, GreedyPolicy{}, orders, &want_caps);
    b200::sequential_simulate(env, GreedyPolicy{}, orders, &got_caps);
    CHECK(got_caps.capacities == want_caps.capacities);
    const auto ws = sequential_simulate_with_states(env, GreedyPolicy{}, orders);
    const auto gs = b200::sequential_simulate_with_states(env, GreedyPolicy{}, orders);
    CHECK(gs.actions == ws.actions);
    CHECK(gs.states.size() == ws.states.size());
    for (std::size_t t = 0; t < std::min(gs.states.size(), ws.states.size()); ++t) {
      CHECK(gs.states[t].capacity == ws.states[t].capacity);
      CHECK(gs.states[t].inventory == ws.states[t].inventory);
    }
    // LocalStateObserver (theory::MonotonicityChecker, theory.hpp:216's call
    // shape): refused with ContractViolation
    theory::MonotonicityChecker checker(std::span<const FoState>(ws.states), inst.products, 1);
    bool refused = false;
    try {
      b200::picard_simulate(env, GreedyPolicy{}, orders, plan, cfg, {}, {}, &checker);
    } catch (const ContractViolation&) {
      refused = true;
    }
    CHECK(refused);
    // picard_iterate_once with IterateOptions / observer / iteration
    ActionCache<FoAction> c1(orders.size(), kNoFulfill), c2(orders.size(), kNoFulfill);
    IterateOptions io;
    io.threads = 2;
    const auto o1 = picard_iterate_once(env, GreedyPolicy{}, orders, plan, c1, 0, (std::int64_t)orders.size(),
                                        env.initial_state(), io, static_cast<NoObserver*>(nullptr), 1);
    const auto o2 = b200::picard_iterate_once(env, GreedyPolicy{}, orders, plan, c2, 0, (std::int64_t)orders.size(),
                                              env.initial_state(), io, static_cast<NoObserver*>(nullptr), 1);
    CHECK(c1 == c2);
    CHECK(o1.changed_slots == o2.changed_slots);
    CHECK(o1.evals_per_process == o2.evals_per_process);
  }
  std::printf("dropin_test: %d checks, %d failures\n", checks, failures);
  return failures;
}
