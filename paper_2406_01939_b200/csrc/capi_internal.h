// capi_internal.h — shared declarations of the B200 engine's host side.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/picard_b200.h"

namespace pcd {

// Exception types map 1:1 onto the C-ABI status codes (picard_b200.h) and onto
// the reference's exception classes (errors.hpp:11-20, engine.hpp:140-156).
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct ContractViolation : std::runtime_error {
  int64_t time_step;
  explicit ContractViolation(const std::string& w, int64_t t = -1)
      : std::runtime_error(w), time_step(t) {}
};
struct IterationLimit : std::runtime_error {
  int64_t iterations_run;
  std::vector<pcd_trace_row> partial_trace;
  IterationLimit(const std::string& w, int64_t k, std::vector<pcd_trace_row> tr)
      : std::runtime_error(w), iterations_run(k), partial_trace(std::move(tr)) {}
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

void set_last_error(const std::string& s);

// host_inputs.cpp
void generate_instance(int32_t J, int32_t I, int64_t T, double beta, double coverage,
                       uint64_t seed, int32_t geometry, int32_t* product, int32_t* origin,
                       double* reward_table, int32_t* capacity, int32_t* inventory);
void product_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, uint64_t seed,
                       int32_t* owner);
void product_chunk_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, uint64_t seed,
                             int32_t* owner);
void product_window_partition(const int32_t* product, int64_t T, int32_t I, int32_t M, int64_t W,
                              uint64_t seed, int32_t* owner);
void uniform_partition(int64_t T, int32_t M, uint64_t seed, int32_t* owner);
void seeded_mlp(int32_t in, int32_t out, uint64_t seed, int32_t h, double* w1, double* b1,
                double* w2, double* b2, double* w3, double* b3);
void linear_contractive_spec(int32_t n, int32_t p, int64_t T, double rho, uint64_t seed, double coupling,
                             double* A, double* B, double* W, double* G, double* contraction);
void shard_processes(const int32_t* owner, int64_t T, int32_t M, int32_t ranks, int32_t* rank_of);

}  // namespace pcd
