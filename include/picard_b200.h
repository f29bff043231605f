/*
 * picard_b200.h — C ABI of the B200-native Picard-iteration policy simulator.
 *
 * This is the drop-in boundary for the reference's serial and Picard
 * simulation paths (arXiv 2406.01939 artifact, /root/reference/proj):
 *
 *   reference C++ entry point (file:line)                   replaced by
 *   ------------------------------------------------------   ---------------------
 *   picard::sequential_simulate      engine.hpp:237-267      pcd_sequential
 *   picard::picard_iterate_once      engine.hpp:358-444      pcd_iterate_once
 *   picard::picard_simulate          engine.hpp:458-590      pcd_simulate
 *                                                             (pcd_picard_simulate = one-shot)
 *   picard::compare_to_oracle        engine.hpp:601-614      pcd_compare_actions
 *   picard::make_uniform_time_partition engine.hpp:99-114    pcd_uniform_partition
 *   picard::fo::make_product_partition  instance.cpp:142-186 pcd_product_partition
 *   picard::fo::generate_instance       instance.cpp:80-140  pcd_generate_instance
 *   picard::fo::MlpParams::seeded_uniform mlp.cpp:117-129     pcd_seeded_mlp
 *   picard::fo::fo_total_reward         env.hpp:298-310      pcd_total_reward
 *   Policy::evaluate (Greedy / CapacityPenalized / DualNetwork, policies.hpp:24-174)
 *                                                             pcd_policy (kind + params)
 *
 * Conventions
 *  - All pointers are caller-owned HOST memory; the library owns every device
 *    buffer behind a pcd_handle.  Nothing here takes or returns torch types.
 *  - Actions are int32 node indices, -1 = decline (fo/types.hpp:15-22).
 *  - Inventory is dense row-major [products x nodes]; an all-zero row is the
 *    reference's "absent row" (fo/types.hpp:45-51, 65-71).
 *  - Rewards are a table [reward_rows x nodes] plus reward_row[t]; generated
 *    instances use one row per origin node (instance.cpp:100-105), loaded
 *    instances may use one row per order.
 *  - Status codes mirror the reference's exception types:
 *      PCD_OK                 0
 *      PCD_INVALID_ARGUMENT   1  (std::invalid_argument)
 *      PCD_CONTRACT_VIOLATION 2  (picard::ContractViolation, errors.hpp:11-20;
 *                                 result->error_time_step carries time_step())
 *      PCD_ITERATION_LIMIT    3  (picard::IterationLimitError, engine.hpp:140-156;
 *                                 result->iterations_run + partial trace)
 *      PCD_CUDA_ERROR         4  (device / NCCL failure; no CPU fallback exists)
 *    pcd_last_error() returns the message of the last failure on this thread.
 *  - One handle per host thread; no callbacks.
 */
#ifndef PICARD_B200_H_
#define PICARD_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PCD_OK = 0,
  PCD_INVALID_ARGUMENT = 1,
  PCD_CONTRACT_VIOLATION = 2,
  PCD_ITERATION_LIMIT = 3,
  PCD_CUDA_ERROR = 4
};

/* Policy kinds (fo/policies.hpp). PCD_POLICY_NULL is the always-decline
 * policy the reference tests use (test_engine.cpp:17-22). */
enum {
  PCD_POLICY_GREEDY = 0,    /* GreedyPolicy            policies.hpp:24-44  */
  PCD_POLICY_CAPACITY = 1,  /* CapacityPenalizedPolicy policies.hpp:50-75  */
  PCD_POLICY_DUAL = 2,      /* DualNetworkPolicy       policies.hpp:88-174 */
  PCD_POLICY_NULL = 3
};

/* Sweep engine selection for pcd_simulate / pcd_iterate_once. */
enum {
  PCD_ENGINE_AUTO = 0,          /* run-partition closed form when the plan is a run
                                   partition (tensor-core policy when eligible),
                                   else the general closed form                   */
  PCD_ENGINE_REPLAY = 1,        /* exact per-process window replay (any plan)     */
  PCD_ENGINE_PRODUCT = 2,       /* closed-form run-partition sweep (checked): each
                                   process owns one contiguous stretch of a
                                   product's orders, or only whole products      */
  PCD_ENGINE_PRODUCT_FP64 = 3,  /* ... with the FP64 SIMT policy only             */
  PCD_ENGINE_GENERAL = 4        /* closed form for any plan and any cache: every
                                   process walks only its own slots (FP64 SIMT
                                   policy); AUTO's choice for non-run plans       */
};

/* A fulfillment-optimization instance (fo/instance.hpp:25-37). */
typedef struct pcd_instance {
  int32_t nodes;              /* J */
  int32_t products;           /* I */
  int64_t horizon;            /* T */
  const int32_t* product;     /* [T] Order::product */
  const int32_t* order_t;     /* [T] Order::t, or NULL meaning order_t[t] == t */
  const int32_t* reward_row;  /* [T] row of reward_table holding Order::rewards */
  const double* reward_table; /* [reward_rows * J] */
  int64_t reward_rows;
  const int32_t* capacity;    /* [J] initial FoState::capacity */
  const int32_t* inventory;   /* [I * J] initial FoState::inventory (dense) */
} pcd_instance;

/* A policy. For PCD_POLICY_DUAL the MLP is {2J+1, hidden, hidden, 2J}
 * (fo/mlp.hpp:13-36) with row-major weights; init_* and horizon are the
 * DualNetworkPolicy's normalisation state (policies.hpp:92-96, 136-148). */
typedef struct pcd_policy {
  int32_t kind;
  int32_t hidden;               /* 64 in the reference */
  double gamma;                 /* CapacityPenalizedPolicy::gamma */
  const double* w1;             /* [hidden * (2J+1)] */
  const double* b1;             /* [hidden] */
  const double* w2;             /* [hidden * hidden] */
  const double* b2;             /* [hidden] */
  const double* w3;             /* [2J * hidden] */
  const double* b3;             /* [2J] */
  const int32_t* init_capacity; /* [J]   NULL -> instance capacity  */
  const int32_t* init_inventory;/* [I*J] NULL -> instance inventory */
  int64_t horizon;              /* <0 -> instance horizon */
} pcd_policy;

/* PicardConfig (engine.hpp:120-126) plus B200 engine knobs. */
typedef struct pcd_config {
  int32_t processes;       /* 0 = take M from the plan */
  int32_t record_trace;    /* bool */
  int64_t max_steps;       /* window width; 0 = whole horizon */
  int64_t max_iterations;  /* 0 = 2T + 4 */
  int32_t threads;         /* accepted for API parity; the device ignores it */
  int32_t engine;          /* PCD_ENGINE_* */
  double tc_guard;         /* tensor-core decision margin below which a row is
                              re-evaluated in exact FP64. 0 = the DERIVED guards
                              of pcd_tc_error_bound (an a-priori bound on the
                              tensor-core score errors for this policy and
                              instance), which make every accepted decision the
                              reference's. A value > 0 overrides both tests
                              (tuning / experiments only).                    */
  int32_t tc_verify;       /* debug: re-evaluate EVERY row in FP64 and count
                              unflagged disagreements (pcd_timing.tc_unflagged_bad) */
  int32_t tc_tiles;        /* CTAs of the tensor-core sweep; 0 = one per SM (tests
                              use fewer, so rows pull processes mid-iteration) */
  int32_t tc_kernel;       /* tensor-core sweep: 0 = auto (incremental layer 1 when
                              it applies), 1 = fused layer 1 (tc_pp), 2 = incremental
                              layer 1 (tc_inc; error when it does not apply)        */
} pcd_config;

/* PicardTraceRow (engine.hpp:128-134). */
typedef struct pcd_trace_row {
  int64_t chunk;
  int64_t iteration;
  int64_t changed_slots;
  int64_t max_process_evals;
  int64_t t_reset;
} pcd_trace_row;

/* PicardResult (engine.hpp:158-176) minus the action vector and trace, which
 * are written into caller buffers. */
typedef struct pcd_result {
  int64_t iterations_to_converged;
  int64_t iterations_to_correct;   /* -1 = not measured / never correct */
  int64_t conflicts;
  int64_t policy_eval_count_sequential_equivalent;
  int64_t total_policy_evals;
  int64_t trace_rows;              /* rows produced (may exceed trace_cap) */
  int64_t iterations_run;          /* == iterations_to_converged unless a cap fired */
  int64_t error_time_step;         /* ContractViolation::time_step(), -1 if none */
} pcd_result;

/* Device-side timing of the last pcd_simulate (CUDA events, milliseconds). */
typedef struct pcd_timing {
  double total_ms;        /* first kernel of iteration 1 .. last scalar read */
  double sweep_ms;        /* sum over iterations of the sweep kernel(s) */
  double prep_ms;         /* eff / checkpoint-count kernels */
  double publish_ms;      /* publish / convergence kernels (replay engine) */
  double advance_ms;      /* checkpoint-advance kernels */
  int64_t iterations;
  int64_t kernel_launches;
  int64_t sweep_launches;
  int64_t steps_critical; /* sum over iterations of max per-process evals */
  int64_t total_evals;
  int32_t engine_used;    /* PCD_ENGINE_REPLAY / PRODUCT / PRODUCT_FP64 / GENERAL */
  int32_t device;
  int64_t tc_rows;        /* policy evaluations through the tcgen05 path */
  int64_t tc_flagged;     /* ... re-evaluated exactly (margin < guard) */
  int64_t tc_disagree;    /* flagged rows where the fp16x3 argmax was wrong */
  int64_t tc_unflagged_bad; /* tc_verify only: unflagged rows that were wrong (must be 0) */
  int32_t tc_used;        /* the sweep ran on tensor cores */
  int32_t tc_tiles;       /* CTAs (128 processes each) */
  int32_t tc_kernel;      /* sweep kernel of the last tensor-core iteration: 1 fused, 2 incremental */
  int32_t tc_inc_iters;   /* iterations that ran the incremental-layer-1 sweep */
  double tc_guard;        /* best-minus-second margin guard the sweep used */
  double tc_score_bound;  /* B: derived bound on |score_tc - score_ref| (0: no tensor-core path) */
  double tc_max_score_err;/* tc_verify only: largest observed |score_tc - score_exact| (<= B) */
  int64_t tc_speculated;  /* rows within the guard decided speculatively and verified after the sweep */
  int64_t tc_spec_reruns; /* iterations re-run because a speculated decision was wrong */
} pcd_timing;

typedef struct pcd_handle pcd_handle;

/* ---------------------------------------------------------------- misc */
const char* pcd_version(void);
const char* pcd_last_error(void);
/* ContractViolation::time_step() of the last PCD_CONTRACT_VIOLATION on this
 * thread (-1 if none / not applicable). */
int64_t pcd_last_error_time_step(void);
/* Number of CUDA devices visible (0 on a CPU-only host; never fails). */
int pcd_device_count(void);

/* ------------------------------------------------------------------------
 * Depletion profile (theory::compute_depletion, theory.hpp:21-86) of a
 * trajectory on the device: first_depleted_at[j] = first t in [0, T) whose
 * entering capacity of node j is 0, T when never; *depleted_count = nodes
 * that deplete (theory::DepletionProfile::iteration_bound() = count + 1).
 * actions[T] (host) or NULL for the handle's resident cache. */
int pcd_depletion_profile(pcd_handle* h, const int32_t* actions, int64_t* first_depleted_at,
                          int64_t* depleted_count);

/* Binary SoA instance files (no reference counterpart; the reference's CSV
 * carries a J-vector of rewards per order, ~10^9 fields at C3): a 48-byte
 * header ("PCDINST1", J, I, T, R, has_order_t) followed by product[T],
 * reward_row[T], order_t[T] (if present) as int32, reward_table[R*J] as f64,
 * capacity[J] and inventory[I*J] as int32, little endian. */
int pcd_save_instance_bin(const pcd_instance* inst, const char* path);
int pcd_instance_bin_info(const char* path, int32_t* nodes, int32_t* products, int64_t* horizon,
                          int64_t* reward_rows, int32_t* has_order_t);
int pcd_load_instance_bin(const char* path, int32_t* product, int32_t* reward_row, int32_t* order_t,
                          double* reward_table, int32_t* capacity, int32_t* inventory);

/* ------------------------------------------------------------------------
 * Time Warp safe-window baseline (timewarp::time_warp_simulate,
 * fo/timewarp.hpp:56-181) on the device: product partition of `processes`
 * (seed), windows [t0, t0 + delta) with delta the minimum remaining capacity
 * (rule 0: over all nodes, clamped to >= 1; rule 1: over still-stocked
 * nodes), every process evaluating its own steps against the synchronized
 * state with all other steps declined, then an in-order merge; an infeasible
 * merge rolls the window back and re-executes it serially. Replaces the
 * handle's plan. */
typedef struct pcd_tw_result {
  int64_t sync_rounds;
  int64_t rollbacks;
  int64_t policy_eval_count_sequential_equivalent;
  int64_t total_policy_evals;
  int64_t trace_rows;
  int64_t error_time_step;
} pcd_tw_result;
typedef struct pcd_tw_trace_row {
  int64_t round, t_start, window_length, max_process_evals;
  int32_t rolled_back, pad;
} pcd_tw_trace_row;
int pcd_time_warp(pcd_handle* h, int32_t processes, uint64_t seed, int32_t rule, int32_t record_trace,
                  int32_t* actions_out, pcd_tw_result* result, pcd_tw_trace_row* trace, int64_t trace_cap);

/* ------------------------------------------------------------------------
 * Non-SCO environment (picard::linear, linear.hpp / linear.cpp): the
 * time-varying linear system s_{t+1} = A_t s_t + B_t a_t + w_t under the
 * linear feedback a_t = G s_t (GainPolicy). Row-major flat arrays:
 * dynamics[T][n][n], input[T][n][p], disturbances[T][n], gain[p][n]. */
typedef struct pcd_linear_spec {
  int32_t state_dim;            /* n (<= 8 on the device) */
  int32_t input_dim;            /* p */
  int64_t horizon;              /* T */
  const double* dynamics;
  const double* input;
  const double* disturbances;
  const double* gain;
} pcd_linear_spec;

/* make_contractive_spec (linear.cpp:126-218), bit-identical streams: fills
 * the four arrays and the closed-loop contraction max_t ||A_t + B_t G||_2. */
int pcd_linear_contractive_spec(int32_t state_dim, int32_t input_dim, int64_t horizon, double rho,
                                uint64_t seed, double state_coupling, double* dynamics, double* input,
                                double* disturbances, double* gain, double* contraction);

/* picard_convergence_curve (linear.cpp:279-330) on the device: single-step
 * partitions (M = T), curve[k] = relative RMSE of the cache-induced state
 * trajectory after iteration k+1 (normalization 1 = draft, 0 = reference),
 * stopping once it is <= tolerance or after max_iterations (0 = T).
 * initial_cache[T][p] or NULL (zero actions). *curve_len = iterations run;
 * final_cache[T][p] (optional) receives the last cache; *elapsed_ms
 * (optional) the device time of the iterations. */
int pcd_linear_convergence_curve(const pcd_linear_spec* spec, const double* initial_cache,
                                 double tolerance, int64_t max_iterations, int32_t normalization,
                                 int32_t device, double* curve, int64_t curve_cap, int64_t* curve_len,
                                 double* final_cache, double* elapsed_ms);

/* MLP feedback policy on the linear env (BASELINE config 4):
 * a_t = MlpParams::forward(s_t) (mlp.cpp:141-169) with widths
 * {state_dim, hidden, hidden, input_dim}: tanh hidden layers, linear output,
 * row-major as MlpParams: w1[hidden][n], b1[hidden], w2[hidden][hidden],
 * b2[hidden], w3[p][hidden], b3[p]. The reference pairs the linear env only
 * with GainPolicy (linear.hpp:104-126); this policy plugs the reference's own
 * MLP into the same env and engine (PolicyFor, engine.hpp:57-61). */
typedef struct pcd_linear_mlp {
  int32_t hidden;               /* <= 64 */
  int32_t pad;
  const double* w1;
  const double* b1;
  const double* w2;
  const double* b2;
  const double* w3;
  const double* b3;
} pcd_linear_mlp;

typedef struct pcd_linear_mlp_result {
  int64_t curve_len;               /* iterations of the curve (as pcd_linear_convergence_curve) */
  int64_t iterations_to_converged; /* picard_simulate's count for the single-step plan (M = T,
                                      whole-horizon window): the first iteration that changes no
                                      action under LinearEnv::actions_equal (linear.hpp:64-71) */
  int64_t fixed_point_iterations;  /* iterations of the pass that computes the sequential
                                      trajectory as the Picard fixed point (Prop. 1) */
  double fixed_point_ms;           /* device time of that pass */
  double curve_ms;                 /* device time of the curve pass */
} pcd_linear_mlp_result;

/* picard_convergence_curve (linear.cpp:267-318) with the MLP feedback policy:
 * single-step partitions, one affine time-scan rollout plus one batched FP64
 * MLP evaluation of all T states per iteration. The closed loop is no longer
 * affine, so the sequential reference trajectory is computed first as the
 * Picard fixed point (iterated until the cache stops changing beyond 2^-46
 * relative), then the curve is scored against it. Arguments as
 * pcd_linear_convergence_curve; reference_states[T+1][n] (optional) receives
 * the sequential trajectory. */
int pcd_linear_mlp_convergence_curve(const pcd_linear_spec* spec, const pcd_linear_mlp* policy,
                                     const double* initial_cache, double tolerance, int64_t max_iterations,
                                     int32_t normalization, int32_t device, double* curve, int64_t curve_cap,
                                     pcd_linear_mlp_result* result, double* final_cache,
                                     double* reference_states);

/* The tensor-core sweep's derived exactness bound (no
 * reference counterpart, host only, no device needed): *bound = B, an
 * a-priori bound on |score_tc - score_ref| of the dual policy on this
 * instance (the |best| test uses B (1 + 2^-10)); *guard = D (1 + 2^-10), D a
 * bound on the error of the difference of two scores of one row (<= 2B: the
 * hidden-layer error is shared), the best-minus-second margin pcd_create
 * uses; 0 when the policy keeps the exact FP64 path (non-finite weights,
 * bound too large, shapes the tensor-core sweep does not take). */
int pcd_tc_error_bound(const pcd_instance* instance, const pcd_policy* policy, double* bound, double* guard);

/* Page-locked host buffers from a process-wide pool (no reference
 * counterpart): result arrays allocated here are written by the device at
 * full PCIe bandwidth and recycled by pcd_host_free instead of being pinned
 * and unpinned per call. NULL on failure. */
void* pcd_host_alloc(size_t bytes);
void pcd_host_free(void* p);

/* ------------------------------------------------------- host-side inputs
 * These run on the host CPU (they are serial-RNG bound and must reproduce the
 * reference's mt19937_64 streams bit for bit). */

/* generate_instance (instance.cpp:80-140). geometry 0 = the reference's
 * 30-city table (default_geometry, geometry.cpp:93-102, J <= 30);
 * geometry 1 = the seeded synthetic J-node geometry used for J > 30
 * (mt19937_64(12345), lat U(25,49), lon U(-124,-67),
 * population U(1e6,4e7), drawn per node in that order).
 * Outputs: product[T], origin[T] (== reward_row), reward_table[J*J],
 * capacity[J], inventory[I*J]. */
int pcd_generate_instance(int32_t nodes, int32_t products, int64_t horizon,
                          double beta, double coverage, uint64_t seed,
                          int32_t geometry, int32_t* product, int32_t* origin,
                          double* reward_table, int32_t* capacity,
                          int32_t* inventory);

/* make_product_partition (instance.cpp:142-186): owner[T]. */
int pcd_product_partition(const pcd_instance* inst, int32_t processes,
                          uint64_t seed, int32_t* owner);
/* Product-chunk partition (no reference counterpart; any PartitionPlan is
 * valid input to picard_simulate, engine.hpp:74-96): each product's orders
 * in time order are cut into contiguous chunks of near-equal length L, one
 * process per chunk, L the smallest length with at most `processes` chunks.
 * Falls back to pcd_product_partition(seed) when processes < ordered
 * products. A run partition, so PCD_ENGINE_PRODUCT applies. owner[T]. */
int pcd_product_chunk_partition(const pcd_instance* inst, int32_t processes,
                                uint64_t seed, int32_t* owner);
/* Window-aware product chunks (no reference counterpart): each product's
 * orders in time order are cut greedily so that no `window`-long interval
 * (PicardConfig::max_steps, engine.hpp:120-126) holds more than L orders of
 * one chunk, L the smallest bound with at most `processes` chunks; products
 * sparse in time stay whole. Bounds every iteration's per-process chain by L
 * at that window. window <= 0: the whole horizon. Falls back to
 * pcd_product_partition(seed) when processes < ordered products. A run
 * partition, so PCD_ENGINE_PRODUCT applies. owner[T]. */
int pcd_product_window_partition(const pcd_instance* inst, int32_t processes,
                                 int64_t window, uint64_t seed, int32_t* owner);
/* make_uniform_time_partition (engine.hpp:99-114): owner[T]. */
int pcd_uniform_partition(int64_t horizon, int32_t processes, uint64_t seed,
                          int32_t* owner);
/* MlpParams::seeded_uniform (mlp.cpp:117-129). */
int pcd_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden,
                   double* w1, double* b1, double* w2, double* b2, double* w3,
                   double* b3);
/* fo_total_reward (env.hpp:298-310). */
int pcd_total_reward(const pcd_instance* inst, const int32_t* actions,
                     double* total);
/* compare_to_oracle (engine.hpp:601-614): *first_mismatch = -1 when equal. */
int pcd_compare_actions(const int32_t* a, const int32_t* b, int64_t n,
                        int64_t* first_mismatch);

/* Multi-GPU sharding of processes: LPT over per-process
 * owned-slot loads onto `ranks` shards; rank_of[M]. Pure host logic. */
int pcd_shard_processes(const int32_t* owner, int64_t horizon, int32_t processes,
                        int32_t ranks, int32_t* rank_of);

/* --------------------------------------------------------- device engine */
int pcd_create(const pcd_instance* inst, const pcd_policy* policy, int32_t device,
               pcd_handle** out);
void pcd_destroy(pcd_handle* h);

/* Uploads a partition plan (PartitionPlan, engine.hpp:74-96) and builds the
 * per-process slot CSR on the device. Validates like PartitionPlan::validate. */
int pcd_set_plan(pcd_handle* h, const int32_t* owner, int32_t processes);

/* picard_simulate (engine.hpp:458-590). initial_cache / reference may be NULL.
 * actions_out[T] receives the converged actions; trace[trace_cap] the rows. */
int pcd_simulate(pcd_handle* h, const pcd_config* cfg,
                 const int32_t* initial_cache, const int32_t* reference,
                 int32_t* actions_out, pcd_result* result, pcd_trace_row* trace,
                 int64_t trace_cap);

/* Same, but with the cache / reference already resident (no host copies);
 * the converged actions stay on the device until pcd_download_actions. Used
 * by bench.py for the HBM-resident throughput number. */
int pcd_simulate_resident(pcd_handle* h, const pcd_config* cfg,
                          int32_t use_initial_cache, int32_t use_reference,
                          pcd_result* result, pcd_trace_row* trace,
                          int64_t trace_cap);
int pcd_upload_cache(pcd_handle* h, const int32_t* initial_cache,
                     const int32_t* reference);
int pcd_download_actions(pcd_handle* h, int32_t* actions_out);

/* picard_iterate_once (engine.hpp:358-444) over [t_lo, t_hi) from the given
 * checkpoint state. cache[T] is read and updated in place (host memory).
 * evals_per_process[M]; changed_slots receives ascending time indices
 * (capacity T), *n_changed their count. */
int pcd_iterate_once(pcd_handle* h, int32_t engine, int32_t* cache, int64_t t_lo,
                     int64_t t_hi, const int32_t* ckpt_capacity,
                     const int32_t* ckpt_inventory, int64_t* evals_per_process,
                     int64_t* changed_slots, int64_t* n_changed);

/* sequential_simulate (engine.hpp:237-267): the serial trajectory. Computed on
 * the device as the Picard fixed point of a product partition over
 * min(I, 8192) processes (Prop. 1: identical actions); policy_evals = T. */
int pcd_sequential(pcd_handle* h, int32_t* actions_out, int64_t* policy_evals);

int pcd_last_timing(const pcd_handle* h, pcd_timing* out);

/* Debug flags of a handle (not for production runs). */
enum { PCD_DEBUG_TC_PROFILE = 1, /* per-phase clock64 totals of the tensor-core
                                    sweep's CTA 0, printed to stderr per launch */
       PCD_DEBUG_TC_FUSED = 2,    /* entry points without a pcd_config (pcd_iterate_once,
                                    pcd_sequential) use the fused-layer-1 sweep ... */
       PCD_DEBUG_TC_INC = 4,      /* ... or the incremental-layer-1 sweep (tests) */
       PCD_DEBUG_NO_SPEC = 8,     /* no speculative decisions (every row within the
                                    guard re-evaluated in the sweep, as in verify mode) */
       PCD_DEBUG_SPEC_RERUN = 16, /* treat every speculated decision as wrong: the
                                    iteration is re-run without speculation (tests) */
       PCD_DEBUG_SPEC_FLIP = 32 }; /* publish a wrong decision for every 4th speculated
                                    slot: the verification must detect it and re-run (tests) */
int pcd_set_debug(pcd_handle* h, int32_t flags);

/* The device checkpoint FoState (capacity[J], dense inventory[I*J]): the
 * state at the start of the current window; after a converged pcd_simulate
 * it is the trajectory's final state (advance_checkpoint, engine.hpp:514-526). */
int pcd_checkpoint_state(pcd_handle* h, int32_t* capacity, int32_t* inventory);

/* Debug/parity hook (theory::CacheTraceRecorder, theory.hpp:120-126): when
 * set, pcd_simulate copies the full cache into history[k*T .. (k+1)*T) after
 * iteration k+1 (first `cap_iterations` iterations). NULL disables. */
int pcd_set_history(pcd_handle* h, int32_t* history, int64_t cap_iterations);

/* One-shot convenience mirroring the reference call shape. */
int pcd_picard_simulate(const pcd_instance* inst, const pcd_policy* policy,
                        const int32_t* owner, int32_t processes,
                        const pcd_config* cfg, const int32_t* initial_cache,
                        const int32_t* reference, int32_t* actions_out,
                        pcd_result* result, pcd_trace_row* trace,
                        int64_t trace_cap);

/* ----------------------------------------------- multi-GPU (NCCL, NVLink)
 * One process per GPU. Rank 0 calls pcd_nccl_unique_id and broadcasts the
 * 128 bytes (e.g. via torch.distributed); every rank then attaches. After
 * attaching, pcd_simulate runs only the processes with rank_of[m] == rank and
 * exchanges fresh cache slices with ncclAllGather plus one ncclAllReduce of
 * the convergence scalars per iteration; every rank returns identical results. */
int pcd_nccl_unique_id(unsigned char out[128]);
int pcd_attach_comm(pcd_handle* h, const unsigned char id[128], int32_t rank,
                    int32_t nranks);

/* In-process loopback group (tests; no reference counterpart): the same
 * multi-rank protocol (per-rank process shards, window-slot all-gather,
 * scalar all-reduces) between N handles in ONE process — e.g. N handles on
 * one GPU, each driven by its own host thread, since NCCL refuses duplicate
 * devices. Every rank must call pcd_simulate concurrently; results are
 * identical to a single rank. The group outlives pcd_loopback_destroy while
 * handles remain attached. */
typedef struct pcd_loopback pcd_loopback;
pcd_loopback* pcd_loopback_create(int32_t nranks);
void pcd_loopback_destroy(pcd_loopback* group);
int pcd_attach_loopback(pcd_handle* h, pcd_loopback* group, int32_t rank);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif  /* PICARD_B200_H_ */
