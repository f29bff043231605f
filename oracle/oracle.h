/*
 * oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Flat C interface shared by the two CPU oracles of the Picard hot path:
 *   - orc_*  : oracle/picard_oracle.c, a plain-C restatement of the
 *              reference algorithm (each function cites reference file:line);
 *   - ref_*  : oracle/ref_harness.cpp linked against the UNMODIFIED reference
 *              library compiled from /root/reference/proj/src (built into
 *              oracle/_ref/ by oracle/Makefile) — used to pin the restatement.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load these; the product path never does.
 *
 * Struct layouts are identical to include/picard_b200.h so the same ctypes
 * structures describe both.
 */
#ifndef PICARD_ORACLE_H_
#define PICARD_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_instance {
  int32_t nodes;
  int32_t products;
  int64_t horizon;
  const int32_t* product;
  const int32_t* order_t;
  const int32_t* reward_row;
  const double* reward_table;
  int64_t reward_rows;
  const int32_t* capacity;
  const int32_t* inventory;
} orc_instance;

typedef struct orc_policy {
  int32_t kind; /* 0 greedy, 1 capacity, 2 dual, 3 null */
  int32_t hidden;
  double gamma;
  const double* w1;
  const double* b1;
  const double* w2;
  const double* b2;
  const double* w3;
  const double* b3;
  const int32_t* init_capacity;
  const int32_t* init_inventory;
  int64_t horizon;
} orc_policy;

typedef struct orc_config {
  int32_t processes;
  int32_t record_trace;
  int64_t max_steps;
  int64_t max_iterations;
  int32_t threads;
  int32_t engine;
} orc_config;

typedef struct orc_trace_row {
  int64_t chunk, iteration, changed_slots, max_process_evals, t_reset;
} orc_trace_row;

typedef struct orc_result {
  int64_t iterations_to_converged;
  int64_t iterations_to_correct;
  int64_t conflicts;
  int64_t policy_eval_count_sequential_equivalent;
  int64_t total_policy_evals;
  int64_t trace_rows;
  int64_t iterations_run;
  int64_t error_time_step;
} orc_result;

/* Status codes: 0 ok, 1 invalid argument, 2 contract violation,
 * 3 iteration limit (same as picard_b200.h). */

/* ---- restatement (picard_oracle.c) ---- */
const char* orc_last_error(void);
double orc_tanh(double x);               /* glibc 2.39 tanh, FMA-variant expm1 */
double orc_tanh_nofma(double x);         /* glibc 2.39 tanh, SSE2-variant expm1 */
double orc_expm1(double x);
double orc_expm1_nofma(double x);
void orc_set_tanh_variant(int fma);      /* which variant the MLP uses (default 1) */
int orc_tanh_variant(void);
int orc_demand_counts(int32_t products, int64_t horizon, double beta, int64_t* out);
int orc_apportion(const double* weights, int64_t n, int64_t total, int64_t* out);
int orc_generate_instance(int32_t nodes, int32_t products, int64_t horizon,
                          double beta, double coverage, uint64_t seed,
                          int32_t geometry, int32_t* product, int32_t* origin,
                          double* reward_table, int32_t* capacity,
                          int32_t* inventory);
int orc_small_random_params(uint64_t seed, int32_t* nodes, int32_t* products,
                            int64_t* horizon, double* beta, double* coverage,
                            uint64_t* inst_seed);
int orc_product_partition(const orc_instance* inst, int32_t processes,
                          uint64_t seed, int32_t* owner);
int orc_uniform_partition(int64_t horizon, int32_t processes, uint64_t seed,
                          int32_t* owner);
int orc_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden,
                   double* w1, double* b1, double* w2, double* b2, double* w3,
                   double* b3);
int orc_mlp_forward(const orc_policy* pol, int32_t input, int32_t output,
                    const double* x, double* out);
int orc_policy_evaluate(const orc_instance* inst, const orc_policy* pol,
                        const int32_t* cap, const int32_t* inv, int64_t t,
                        int32_t* action);
int orc_sequential(const orc_instance* inst, const orc_policy* pol,
                   int32_t* actions, int64_t* evals, int64_t* error_t);
int orc_picard(const orc_instance* inst, const orc_policy* pol,
               const int32_t* owner, int32_t processes, const orc_config* cfg,
               const int32_t* initial_cache, const int32_t* reference,
               int32_t* actions, orc_result* res, orc_trace_row* trace,
               int64_t trace_cap, int32_t* history, int64_t history_cap);
int orc_iterate_once(const orc_instance* inst, const orc_policy* pol,
                     const int32_t* owner, int32_t processes, int32_t* cache,
                     int64_t t_lo, int64_t t_hi, const int32_t* ckpt_cap,
                     const int32_t* ckpt_inv, int64_t* evals_per_process,
                     int64_t* changed, int64_t* n_changed, int64_t* error_t);
int orc_naive_fixed_point(const orc_instance* inst, const orc_policy* pol,
                          const int32_t* owner, int32_t processes,
                          int32_t* history, int64_t history_cap,
                          int64_t* iterations);
int orc_total_reward(const orc_instance* inst, const int32_t* actions,
                     double* total);

/* ---- reference harness (ref_harness.cpp, links /root/reference) ---- */
const char* ref_last_error(void);
double ref_tanh(double x);
int ref_demand_counts(int32_t products, int64_t horizon, double beta, int64_t* out);
int ref_apportion(const double* weights, int64_t n, int64_t total, int64_t* out);
int ref_generate_instance(int32_t nodes, int32_t products, int64_t horizon,
                          double beta, double coverage, uint64_t seed,
                          int32_t geometry, int32_t* product, int32_t* origin,
                          double* reward_table, int32_t* capacity,
                          int32_t* inventory);
int ref_small_random_params(uint64_t seed, int32_t* nodes, int32_t* products,
                            int64_t* horizon, double* beta, double* coverage,
                            uint64_t* inst_seed);
int ref_product_partition(const orc_instance* inst, int32_t processes,
                          uint64_t seed, int32_t* owner);
int ref_uniform_partition(int64_t horizon, int32_t processes, uint64_t seed,
                          int32_t* owner);
int ref_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden,
                   double* w1, double* b1, double* w2, double* b2, double* w3,
                   double* b3);
int ref_mlp_forward(const orc_policy* pol, int32_t input, int32_t output,
                    const double* x, double* out);
int ref_policy_evaluate(const orc_instance* inst, const orc_policy* pol,
                        const int32_t* cap, const int32_t* inv, int64_t t,
                        int32_t* action);
int ref_sequential(const orc_instance* inst, const orc_policy* pol,
                   int32_t* actions, int64_t* evals, int64_t* error_t);
int ref_picard(const orc_instance* inst, const orc_policy* pol,
               const int32_t* owner, int32_t processes, const orc_config* cfg,
               const int32_t* initial_cache, const int32_t* reference,
               int32_t* actions, orc_result* res, orc_trace_row* trace,
               int64_t trace_cap, int32_t* history, int64_t history_cap);
int ref_iterate_once(const orc_instance* inst, const orc_policy* pol,
                     const int32_t* owner, int32_t processes, int32_t* cache,
                     int64_t t_lo, int64_t t_hi, const int32_t* ckpt_cap,
                     const int32_t* ckpt_inv, int64_t* evals_per_process,
                     int64_t* changed, int64_t* n_changed, int64_t* error_t);
int ref_total_reward(const orc_instance* inst, const int32_t* actions,
                     double* total);
int ref_sequential_timed(const orc_instance* inst, const orc_policy* pol,
                         int32_t* actions, double* seconds);
int ref_picard_timed(const orc_instance* inst, const orc_policy* pol,
                     const int32_t* owner, int32_t processes, int64_t max_steps,
                     int32_t threads, int32_t* actions, int64_t* iterations,
                     int64_t* seq_equiv, double* seconds);
/* segmented serial trajectory (bench.py reference arm) */
void* ref_session_create(const orc_instance* inst, const orc_policy* pol);
void ref_session_destroy(void* session);
int ref_session_set_state(void* session, int64_t t, const int32_t* cap, const int32_t* inv);
int ref_session_get_state(void* session, int64_t* t, int32_t* cap, int32_t* inv);
int ref_session_total_reward(void* session, const int32_t* actions, double* total);
int ref_session_sequential(void* session, int64_t t1, int32_t* actions, double* seconds,
                           int64_t* error_t);

#ifdef __cplusplus
}
#endif

#endif
