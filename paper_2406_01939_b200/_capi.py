"""ctypes binding of the C ABI in include/picard_b200.h.

The shared library is the in-tree ``libpicard_b200.so`` (built by
``paper_2406_01939_b200/build.py``). There is no fallback: if the library is
missing, importing the package raises, and every device entry point fails
with ``CudaError`` on a host without a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libpicard_b200.so")

I32P = C.POINTER(C.c_int32)
I64P = C.POINTER(C.c_int64)
F64P = C.POINTER(C.c_double)

PCD_OK, PCD_INVALID_ARGUMENT, PCD_CONTRACT_VIOLATION, PCD_ITERATION_LIMIT, PCD_CUDA_ERROR = range(5)
PCD_POLICY_GREEDY, PCD_POLICY_CAPACITY, PCD_POLICY_DUAL, PCD_POLICY_NULL = range(4)
PCD_ENGINE_AUTO, PCD_ENGINE_REPLAY, PCD_ENGINE_PRODUCT, PCD_ENGINE_PRODUCT_FP64, PCD_ENGINE_GENERAL = range(5)


class pcd_linear_spec(C.Structure):
    _fields_ = [("state_dim", C.c_int32), ("input_dim", C.c_int32), ("horizon", C.c_int64),
                ("dynamics", F64P), ("input", F64P), ("disturbances", F64P), ("gain", F64P)]


class pcd_linear_mlp(C.Structure):
    _fields_ = [("hidden", C.c_int32), ("pad", C.c_int32), ("w1", F64P), ("b1", F64P), ("w2", F64P),
                ("b2", F64P), ("w3", F64P), ("b3", F64P)]


class pcd_linear_mlp_result(C.Structure):
    _fields_ = [("curve_len", C.c_int64), ("iterations_to_converged", C.c_int64),
                ("fixed_point_iterations", C.c_int64), ("fixed_point_ms", C.c_double), ("curve_ms", C.c_double)]


class pcd_tw_result(C.Structure):
    _fields_ = [("sync_rounds", C.c_int64), ("rollbacks", C.c_int64),
                ("policy_eval_count_sequential_equivalent", C.c_int64), ("total_policy_evals", C.c_int64),
                ("trace_rows", C.c_int64), ("error_time_step", C.c_int64)]


class pcd_tw_trace_row(C.Structure):
    _fields_ = [("round", C.c_int64), ("t_start", C.c_int64), ("window_length", C.c_int64),
                ("max_process_evals", C.c_int64), ("rolled_back", C.c_int32), ("pad", C.c_int32)]


class pcd_instance(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("products", C.c_int32), ("horizon", C.c_int64),
                ("product", I32P), ("order_t", I32P), ("reward_row", I32P),
                ("reward_table", F64P), ("reward_rows", C.c_int64),
                ("capacity", I32P), ("inventory", I32P)]


class pcd_policy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("hidden", C.c_int32), ("gamma", C.c_double),
                ("w1", F64P), ("b1", F64P), ("w2", F64P), ("b2", F64P), ("w3", F64P), ("b3", F64P),
                ("init_capacity", I32P), ("init_inventory", I32P), ("horizon", C.c_int64)]


class pcd_config(C.Structure):
    _fields_ = [("processes", C.c_int32), ("record_trace", C.c_int32), ("max_steps", C.c_int64),
                ("max_iterations", C.c_int64), ("threads", C.c_int32), ("engine", C.c_int32),
                ("tc_guard", C.c_double), ("tc_verify", C.c_int32), ("tc_tiles", C.c_int32),
                ("tc_kernel", C.c_int32)]


class pcd_trace_row(C.Structure):
    _fields_ = [("chunk", C.c_int64), ("iteration", C.c_int64), ("changed_slots", C.c_int64),
                ("max_process_evals", C.c_int64), ("t_reset", C.c_int64)]


class pcd_result(C.Structure):
    _fields_ = [("iterations_to_converged", C.c_int64), ("iterations_to_correct", C.c_int64),
                ("conflicts", C.c_int64), ("policy_eval_count_sequential_equivalent", C.c_int64),
                ("total_policy_evals", C.c_int64), ("trace_rows", C.c_int64),
                ("iterations_run", C.c_int64), ("error_time_step", C.c_int64)]


class pcd_timing(C.Structure):
    _fields_ = [("total_ms", C.c_double), ("sweep_ms", C.c_double), ("prep_ms", C.c_double),
                ("publish_ms", C.c_double), ("advance_ms", C.c_double), ("iterations", C.c_int64),
                ("kernel_launches", C.c_int64), ("sweep_launches", C.c_int64),
                ("steps_critical", C.c_int64), ("total_evals", C.c_int64),
                ("engine_used", C.c_int32), ("device", C.c_int32), ("tc_rows", C.c_int64),
                ("tc_flagged", C.c_int64), ("tc_disagree", C.c_int64), ("tc_unflagged_bad", C.c_int64),
                ("tc_used", C.c_int32), ("tc_tiles", C.c_int32),
                ("tc_kernel", C.c_int32), ("tc_inc_iters", C.c_int32),
                ("tc_guard", C.c_double), ("tc_score_bound", C.c_double), ("tc_max_score_err", C.c_double),
                ("tc_speculated", C.c_int64), ("tc_spec_reruns", C.c_int64)]


# name -> (restype, argtypes); every symbol declared in include/picard_b200.h
SIGNATURES = {
    "pcd_version": (C.c_char_p, []),
    "pcd_last_error": (C.c_char_p, []),
    "pcd_last_error_time_step": (C.c_int64, []),
    "pcd_device_count": (C.c_int, []),
    "pcd_generate_instance": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_double,
                                        C.c_uint64, C.c_int32, I32P, I32P, F64P, I32P, I32P]),
    "pcd_product_partition": (C.c_int, [C.POINTER(pcd_instance), C.c_int32, C.c_uint64, I32P]),
    "pcd_linear_contractive_spec": (C.c_int, [C.c_int32, C.c_int32, C.c_int64, C.c_double, C.c_uint64, C.c_double,
                                               F64P, F64P, F64P, F64P, C.POINTER(C.c_double)]),
    "pcd_linear_convergence_curve": (C.c_int, [C.POINTER(pcd_linear_spec), F64P, C.c_double, C.c_int64, C.c_int32,
                                                C.c_int32, F64P, C.c_int64, C.POINTER(C.c_int64), F64P,
                                                C.POINTER(C.c_double)]),
    "pcd_linear_mlp_convergence_curve": (C.c_int, [C.POINTER(pcd_linear_spec), C.POINTER(pcd_linear_mlp), F64P,
                                                    C.c_double, C.c_int64, C.c_int32, C.c_int32, F64P, C.c_int64,
                                                    C.POINTER(pcd_linear_mlp_result), F64P, F64P]),
    "pcd_tc_error_bound": (C.c_int, [C.POINTER(pcd_instance), C.POINTER(pcd_policy), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double)]),
    "pcd_time_warp": (C.c_int, [C.c_void_p, C.c_int32, C.c_uint64, C.c_int32, C.c_int32, I32P,
                                 C.POINTER(pcd_tw_result), C.POINTER(pcd_tw_trace_row), C.c_int64]),
    "pcd_depletion_profile": (C.c_int, [C.c_void_p, I32P, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "pcd_save_instance_bin": (C.c_int, [C.POINTER(pcd_instance), C.c_char_p]),
    "pcd_instance_bin_info": (C.c_int, [C.c_char_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                        C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "pcd_load_instance_bin": (C.c_int, [C.c_char_p, I32P, I32P, I32P, F64P, I32P, I32P]),
    "pcd_host_alloc": (C.c_void_p, [C.c_size_t]),
    "pcd_host_free": (None, [C.c_void_p]),
    "pcd_product_chunk_partition": (C.c_int, [C.POINTER(pcd_instance), C.c_int32, C.c_uint64, I32P]),
    "pcd_product_window_partition": (C.c_int, [C.POINTER(pcd_instance), C.c_int32, C.c_int64, C.c_uint64, I32P]),
    "pcd_uniform_partition": (C.c_int, [C.c_int64, C.c_int32, C.c_uint64, I32P]),
    "pcd_seeded_mlp": (C.c_int, [C.c_int32, C.c_int32, C.c_uint64, C.c_int32,
                                 F64P, F64P, F64P, F64P, F64P, F64P]),
    "pcd_total_reward": (C.c_int, [C.POINTER(pcd_instance), I32P, C.POINTER(C.c_double)]),
    "pcd_compare_actions": (C.c_int, [I32P, I32P, C.c_int64, I64P]),
    "pcd_shard_processes": (C.c_int, [I32P, C.c_int64, C.c_int32, C.c_int32, I32P]),
    "pcd_create": (C.c_int, [C.POINTER(pcd_instance), C.POINTER(pcd_policy), C.c_int32,
                             C.POINTER(C.c_void_p)]),
    "pcd_destroy": (None, [C.c_void_p]),
    "pcd_set_plan": (C.c_int, [C.c_void_p, I32P, C.c_int32]),
    "pcd_simulate": (C.c_int, [C.c_void_p, C.POINTER(pcd_config), I32P, I32P, I32P,
                               C.POINTER(pcd_result), C.POINTER(pcd_trace_row), C.c_int64]),
    "pcd_simulate_resident": (C.c_int, [C.c_void_p, C.POINTER(pcd_config), C.c_int32, C.c_int32,
                                        C.POINTER(pcd_result), C.POINTER(pcd_trace_row), C.c_int64]),
    "pcd_upload_cache": (C.c_int, [C.c_void_p, I32P, I32P]),
    "pcd_download_actions": (C.c_int, [C.c_void_p, I32P]),
    "pcd_iterate_once": (C.c_int, [C.c_void_p, C.c_int32, I32P, C.c_int64, C.c_int64, I32P, I32P,
                                   I64P, I64P, I64P]),
    "pcd_sequential": (C.c_int, [C.c_void_p, I32P, I64P]),
    "pcd_last_timing": (C.c_int, [C.c_void_p, C.POINTER(pcd_timing)]),
    "pcd_set_history": (C.c_int, [C.c_void_p, I32P, C.c_int64]),
    "pcd_checkpoint_state": (C.c_int, [C.c_void_p, I32P, I32P]),
    "pcd_set_debug": (C.c_int, [C.c_void_p, C.c_int32]),
    "pcd_picard_simulate": (C.c_int, [C.POINTER(pcd_instance), C.POINTER(pcd_policy), I32P, C.c_int32,
                                      C.POINTER(pcd_config), I32P, I32P, I32P, C.POINTER(pcd_result),
                                      C.POINTER(pcd_trace_row), C.c_int64]),
    "pcd_nccl_unique_id": (C.c_int, [C.POINTER(C.c_ubyte * 128)]),
    "pcd_attach_comm": (C.c_int, [C.c_void_p, C.POINTER(C.c_ubyte * 128), C.c_int32, C.c_int32]),
    "pcd_loopback_create": (C.c_void_p, [C.c_int32]),
    "pcd_loopback_destroy": (None, [C.c_void_p]),
    "pcd_attach_loopback": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
}


def load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a extension first "
            "(python -m paper_2406_01939_b200.build). There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


LIB = load()
