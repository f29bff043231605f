"""B200-native Picard-iteration policy simulator (arXiv 2406.01939).

A drop-in for the reference's serial and Picard simulation paths
(``proj/include/picard``): the fixed-point iteration runs in hand-written
sm_100a kernels behind the C ABI in ``include/picard_b200.h``; this package is
the Python mirror of the reference interface (see :mod:`.api`).
"""
from .api import (  # noqa: F401
    NO_FULFILL, CapacityPenalizedPolicy, LinearCurve, MlpFeedbackPolicy, LinearSystemSpec, make_contractive_spec,
    picard_convergence_curve, TimeWarpResult, time_warp_simulate, DepletionProfile, depletion_profile,
    check_iteration_bound, save_instance_binary, load_instance_binary, ContractViolation, CudaError, DualNetworkPolicy, GreedyPolicy,
    Instance, InvalidArgument, IterationLimitError, IterationOutcome, MlpParams, NullOnlyPolicy,
    PartitionPlan, PicardConfig, PicardError, PicardResult, PicardTraceRow, Policy, SequentialOutput,
    Simulator, compare_to_oracle, device_count, fo_total_reward, generate_instance,
    make_product_chunk_partition, make_product_partition, make_product_window_partition, make_uniform_time_partition, nccl_unique_id, picard_iterate_once,
    LoopbackGroup, tc_error_bound,
    picard_simulate, sequential_simulate, shard_processes)

__version__ = "0.1.0"
