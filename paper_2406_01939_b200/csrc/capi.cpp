// capi.cpp — host-only entry points of the C ABI (include/picard_b200.h) and
// the exception -> status-code translation shared with engine.cu.
#include <cstdio>
#include <cstring>
#include <string>

#include "capi_internal.h"

namespace pcd {

static thread_local std::string g_last_error;
static thread_local int64_t g_last_time_step = -1;

void set_last_error(const std::string& s) {
  g_last_error = s;
  g_last_time_step = -1;
}

// Maps the in-flight exception onto the status codes of picard_b200.h, which
// mirror the reference's exception classes (errors.hpp, engine.hpp:140-156).
int translate_exception() {
  try {
    throw;
  } catch (const IterationLimit& e) {
    set_last_error(e.what());
    return PCD_ITERATION_LIMIT;
  } catch (const ContractViolation& e) {
    set_last_error(e.what());
    g_last_time_step = e.time_step;
    return PCD_CONTRACT_VIOLATION;
  } catch (const InvalidArgument& e) {
    set_last_error(e.what());
    return PCD_INVALID_ARGUMENT;
  } catch (const CudaError& e) {
    set_last_error(e.what());
    return PCD_CUDA_ERROR;
  } catch (const std::bad_alloc&) {
    set_last_error("host allocation failed");
    return PCD_INVALID_ARGUMENT;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return PCD_INVALID_ARGUMENT;
  } catch (...) {
    set_last_error("unknown error");
    return PCD_INVALID_ARGUMENT;
  }
}

}  // namespace pcd

#define PCD_TRY try {
#define PCD_CATCH \
  }               \
  catch (...) { return pcd::translate_exception(); }

extern "C" {

const char* pcd_version(void) { return "picard_b200 0.1.0 (sm_100a)"; }

const char* pcd_last_error(void) { return pcd::g_last_error.c_str(); }

int64_t pcd_last_error_time_step(void) { return pcd::g_last_time_step; }

int pcd_generate_instance(int32_t nodes, int32_t products, int64_t horizon, double beta,
                          double coverage, uint64_t seed, int32_t geometry, int32_t* product,
                          int32_t* origin, double* reward_table, int32_t* capacity,
                          int32_t* inventory) {
  PCD_TRY
  if (!product || !origin || !reward_table || !capacity || !inventory)
    throw pcd::InvalidArgument("null output buffer");
  pcd::generate_instance(nodes, products, horizon, beta, coverage, seed, geometry, product, origin,
                         reward_table, capacity, inventory);
  return PCD_OK;
  PCD_CATCH
}

int pcd_product_partition(const pcd_instance* inst, int32_t processes, uint64_t seed, int32_t* owner) {
  PCD_TRY
  if (!inst || !owner) throw pcd::InvalidArgument("null argument");
  for (int64_t t = 0; t < inst->horizon; ++t)
    if (inst->product[t] < 0 || inst->product[t] >= inst->products)
      throw pcd::InvalidArgument("order product out of range");
  pcd::product_partition(inst->product, inst->horizon, inst->products, processes, seed, owner);
  return PCD_OK;
  PCD_CATCH
}

int pcd_product_chunk_partition(const pcd_instance* inst, int32_t processes, uint64_t seed, int32_t* owner) {
  PCD_TRY
  if (!inst || !owner) throw pcd::InvalidArgument("null argument");
  for (int64_t t = 0; t < inst->horizon; ++t)
    if (inst->product[t] < 0 || inst->product[t] >= inst->products)
      throw pcd::InvalidArgument("order product out of range");
  pcd::product_chunk_partition(inst->product, inst->horizon, inst->products, processes, seed, owner);
  return PCD_OK;
  PCD_CATCH
}

int pcd_product_window_partition(const pcd_instance* inst, int32_t processes, int64_t window, uint64_t seed,
                                 int32_t* owner) {
  PCD_TRY
  if (!inst || !owner) throw pcd::InvalidArgument("null argument");
  for (int64_t t = 0; t < inst->horizon; ++t)
    if (inst->product[t] < 0 || inst->product[t] >= inst->products)
      throw pcd::InvalidArgument("order product out of range");
  pcd::product_window_partition(inst->product, inst->horizon, inst->products, processes, window, seed, owner);
  return PCD_OK;
  PCD_CATCH
}

int pcd_linear_contractive_spec(int32_t state_dim, int32_t input_dim, int64_t horizon, double rho, uint64_t seed,
                                double state_coupling, double* dynamics, double* input, double* disturbances,
                                double* gain, double* contraction) {
  PCD_TRY
  if (horizon > 0 && (!dynamics || !input || !disturbances)) throw pcd::InvalidArgument("null argument");
  if (!gain || !contraction) throw pcd::InvalidArgument("null argument");
  pcd::linear_contractive_spec(state_dim, input_dim, horizon, rho, seed, state_coupling, dynamics, input,
                               disturbances, gain, contraction);
  return PCD_OK;
  PCD_CATCH
}

// ---------------------------------------------------------------- binary instances
namespace {
struct InstHeader {
  char magic[8];
  int32_t nodes, products;
  int64_t horizon, reward_rows;
  int32_t has_order_t, pad;
  int64_t reserved;
};
static_assert(sizeof(InstHeader) == 48, "header layout");
struct File {
  FILE* f;
  ~File() { if (f) std::fclose(f); }
};
void write_all(FILE* f, const void* p, size_t bytes) {
  if (bytes && std::fwrite(p, 1, bytes, f) != bytes) throw pcd::InvalidArgument("instance file: write failed");
}
void read_all(FILE* f, void* p, size_t bytes) {
  if (bytes && std::fread(p, 1, bytes, f) != bytes) throw pcd::InvalidArgument("instance file: truncated");
}
InstHeader read_header(FILE* f) {
  InstHeader h{};
  read_all(f, &h, sizeof h);
  if (std::memcmp(h.magic, "PCDINST1", 8) != 0) throw pcd::InvalidArgument("instance file: bad magic");
  if (h.nodes < 1 || h.products < 1 || h.horizon < 0 || h.reward_rows < 0)
    throw pcd::InvalidArgument("instance file: bad header");
  return h;
}
}  // namespace

int pcd_save_instance_bin(const pcd_instance* in, const char* path) {
  PCD_TRY
  if (!in || !path) throw pcd::InvalidArgument("null argument");
  File fw{std::fopen(path, "wb")};
  if (!fw.f) throw pcd::InvalidArgument(std::string("cannot open ") + path);
  InstHeader h{};
  std::memcpy(h.magic, "PCDINST1", 8);
  h.nodes = in->nodes;
  h.products = in->products;
  h.horizon = in->horizon;
  h.reward_rows = in->reward_rows;
  h.has_order_t = in->order_t ? 1 : 0;
  write_all(fw.f, &h, sizeof h);
  const size_t T = (size_t)in->horizon, J = (size_t)in->nodes;
  write_all(fw.f, in->product, T * 4);
  write_all(fw.f, in->reward_row, T * 4);
  if (in->order_t) write_all(fw.f, in->order_t, T * 4);
  write_all(fw.f, in->reward_table, (size_t)in->reward_rows * J * 8);
  write_all(fw.f, in->capacity, J * 4);
  write_all(fw.f, in->inventory, (size_t)in->products * J * 4);
  return PCD_OK;
  PCD_CATCH
}

int pcd_instance_bin_info(const char* path, int32_t* nodes, int32_t* products, int64_t* horizon,
                          int64_t* reward_rows, int32_t* has_order_t) {
  PCD_TRY
  if (!path) throw pcd::InvalidArgument("null argument");
  File fr{std::fopen(path, "rb")};
  if (!fr.f) throw pcd::InvalidArgument(std::string("cannot open ") + path);
  const InstHeader h = read_header(fr.f);
  if (nodes) *nodes = h.nodes;
  if (products) *products = h.products;
  if (horizon) *horizon = h.horizon;
  if (reward_rows) *reward_rows = h.reward_rows;
  if (has_order_t) *has_order_t = h.has_order_t;
  return PCD_OK;
  PCD_CATCH
}

int pcd_load_instance_bin(const char* path, int32_t* product, int32_t* reward_row, int32_t* order_t,
                          double* reward_table, int32_t* capacity, int32_t* inventory) {
  PCD_TRY
  if (!path) throw pcd::InvalidArgument("null argument");
  File fr{std::fopen(path, "rb")};
  if (!fr.f) throw pcd::InvalidArgument(std::string("cannot open ") + path);
  const InstHeader h = read_header(fr.f);
  const size_t T = (size_t)h.horizon, J = (size_t)h.nodes;
  if ((T && (!product || !reward_row)) || !reward_table || !capacity || !inventory)
    throw pcd::InvalidArgument("null argument");
  read_all(fr.f, product, T * 4);
  read_all(fr.f, reward_row, T * 4);
  if (h.has_order_t) {
    if (order_t) read_all(fr.f, order_t, T * 4);
    else if (std::fseek(fr.f, (long)(T * 4), SEEK_CUR) != 0) throw pcd::InvalidArgument("instance file: truncated");
  }
  read_all(fr.f, reward_table, (size_t)h.reward_rows * J * 8);
  read_all(fr.f, capacity, J * 4);
  read_all(fr.f, inventory, (size_t)h.products * J * 4);
  return PCD_OK;
  PCD_CATCH
}

int pcd_uniform_partition(int64_t horizon, int32_t processes, uint64_t seed, int32_t* owner) {
  PCD_TRY
  if (horizon > 0 && !owner) throw pcd::InvalidArgument("null argument");
  pcd::uniform_partition(horizon, processes, seed, owner);
  return PCD_OK;
  PCD_CATCH
}

int pcd_seeded_mlp(int32_t input, int32_t output, uint64_t seed, int32_t hidden, double* w1,
                   double* b1, double* w2, double* b2, double* w3, double* b3) {
  PCD_TRY
  if (!w1 || !b1 || !w2 || !b2 || !w3 || !b3) throw pcd::InvalidArgument("null output buffer");
  pcd::seeded_mlp(input, output, seed, hidden, w1, b1, w2, b2, w3, b3);
  return PCD_OK;
  PCD_CATCH
}

int pcd_total_reward(const pcd_instance* inst, const int32_t* actions, double* total) {
  PCD_TRY
  if (!inst || !actions || !total) throw pcd::InvalidArgument("null argument");
  double s = 0.0;  // fo_total_reward (env.hpp:298-310): in order, declines earn 0
  for (int64_t t = 0; t < inst->horizon; ++t)
    if (actions[t] >= 0)
      s += inst->reward_table[(size_t)inst->reward_row[t] * inst->nodes + actions[t]];
  *total = s;
  return PCD_OK;
  PCD_CATCH
}

int pcd_compare_actions(const int32_t* a, const int32_t* b, int64_t n, int64_t* first_mismatch) {
  PCD_TRY
  if ((n > 0 && (!a || !b)) || !first_mismatch) throw pcd::InvalidArgument("null argument");
  *first_mismatch = -1;
  for (int64_t t = 0; t < n; ++t)
    if (a[t] != b[t]) {
      *first_mismatch = t;
      break;
    }
  return PCD_OK;
  PCD_CATCH
}

int pcd_shard_processes(const int32_t* owner, int64_t horizon, int32_t processes, int32_t ranks,
                        int32_t* rank_of) {
  PCD_TRY
  if ((horizon > 0 && !owner) || !rank_of) throw pcd::InvalidArgument("null argument");
  if (processes < 1) throw pcd::InvalidArgument("processes must be >= 1");
  for (int64_t t = 0; t < horizon; ++t)
    if (owner[t] < 0 || owner[t] >= processes) throw pcd::InvalidArgument("owner out of range");
  pcd::shard_processes(owner, horizon, processes, ranks, rank_of);
  return PCD_OK;
  PCD_CATCH
}

}  // extern "C"
