"""Python mirror of the reference's simulator / policy / task-assignment API.

Names, argument meanings and error behaviour follow ``proj/include/picard``:

=====================================  =====================================
reference (file:line)                  here
=====================================  =====================================
fo::Instance (instance.hpp:25-37)      :class:`Instance`
fo::generate_instance (instance.cpp:80) :func:`generate_instance`
fo::make_product_partition (:142-186)  :func:`make_product_partition`
(ours, no reference counterpart)       :func:`make_product_chunk_partition`
(ours, no reference counterpart)       :func:`make_product_window_partition`
make_uniform_time_partition (engine.hpp:99-114) :func:`make_uniform_time_partition`
linear::make_contractive_spec (linear.cpp:126) :func:`make_contractive_spec`
linear::picard_convergence_curve (linear.cpp:279) :func:`picard_convergence_curve`
(ours: MLP policy on the linear env)   :class:`MlpFeedbackPolicy`
PartitionPlan (engine.hpp:74-96)       :class:`PartitionPlan`
PicardConfig (engine.hpp:120-126)      :class:`PicardConfig`
PicardResult / PicardTraceRow          :class:`PicardResult` / :class:`PicardTraceRow`
IterationOutcome (engine.hpp:178-192)  :class:`IterationOutcome`
GreedyPolicy / CapacityPenalizedPolicy / DualNetworkPolicy (policies.hpp)
MlpParams (mlp.hpp:13-36)              :class:`MlpParams`
sequential_simulate (engine.hpp:237)   :func:`sequential_simulate`
picard_iterate_once (engine.hpp:358)   :func:`picard_iterate_once`
picard_simulate (engine.hpp:458)       :func:`picard_simulate`
compare_to_oracle (engine.hpp:601)     :func:`compare_to_oracle`
fo_total_reward (env.hpp:298)          :func:`fo_total_reward`
ContractViolation (errors.hpp:11)      :class:`ContractViolation`
IterationLimitError (engine.hpp:140)   :class:`IterationLimitError`
=====================================  =====================================

Everything below the Python surface runs in ``libpicard_b200.so``: host-side
serial-RNG inputs in C++, and the whole fixed-point iteration in sm_100a
kernels. Actions are ints, ``-1`` = decline (``kNoFulfill``).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _capi as K

LIB = K.LIB
NO_FULFILL = -1
ENGINES = {"auto": K.PCD_ENGINE_AUTO, "replay": K.PCD_ENGINE_REPLAY, "product": K.PCD_ENGINE_PRODUCT,
           "product_fp64": K.PCD_ENGINE_PRODUCT_FP64, "general": K.PCD_ENGINE_GENERAL}
TC_KERNELS = {"auto": 0, "fused": 1, "incremental": 2}


# ------------------------------------------------------------------ errors
class PicardError(RuntimeError):
    pass


class ContractViolation(PicardError):
    """picard::ContractViolation (errors.hpp:11-20)."""

    def __init__(self, what: str, time_step: int = -1):
        super().__init__(what)
        self.time_step = time_step


class IterationLimitError(PicardError):
    """picard::IterationLimitError (engine.hpp:140-156)."""

    def __init__(self, what: str, iterations_run: int, partial_trace):
        super().__init__(what)
        self.iterations_run = iterations_run
        self.partial_trace = partial_trace


class InvalidArgument(ValueError):
    """std::invalid_argument thrown by the reference's generators."""


class CudaError(PicardError):
    """Device / NCCL failure. There is no CPU fallback."""


def _err() -> str:
    return LIB.pcd_last_error().decode()


def _check(rc: int, time_step: int = -1):
    if rc == K.PCD_OK:
        return
    msg = _err()
    if rc == K.PCD_CONTRACT_VIOLATION:
        if time_step < 0:
            time_step = int(LIB.pcd_last_error_time_step())
        raise ContractViolation(msg, time_step)
    if rc == K.PCD_INVALID_ARGUMENT:
        raise InvalidArgument(msg)
    if rc == K.PCD_CUDA_ERROR:
        raise CudaError(msg)
    raise PicardError(f"[{rc}] {msg}")


def _ptr(a, ctype=C.c_int32):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


def _i32(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.int32)


def _pinned_i32(n: int) -> np.ndarray:
    """int32 array in page-locked host memory from the library's pool (the
    device writes results into it at full bandwidth); the buffer returns to
    the pool when the array is garbage collected. Falls back to pageable."""
    import weakref
    nbytes = max(int(n), 1) * 4
    ptr = LIB.pcd_host_alloc(nbytes)
    if not ptr:
        return np.zeros(max(int(n), 1), np.int32)
    buf = (C.c_int32 * max(int(n), 1)).from_address(ptr)
    arr = np.frombuffer(buf, dtype=np.int32)
    weakref.finalize(buf, LIB.pcd_host_free, C.c_void_p(ptr))
    return arr


# --------------------------------------------------------------- instances
@dataclass
class Instance:
    """A fulfillment instance (fo/instance.hpp:25-37) in SoA form.

    ``reward_table[reward_row[t]]`` is Order::rewards of order t; generated
    instances have one row per origin node (instance.cpp:100-105).
    ``inventory`` is dense ``[products, nodes]`` (absent rows are zeros).
    """
    nodes: int
    products: int
    horizon: int
    product: np.ndarray
    reward_row: np.ndarray
    reward_table: np.ndarray
    capacity: np.ndarray
    inventory: np.ndarray
    order_t: Optional[np.ndarray] = None
    meta: dict = field(default_factory=dict)

    def __post_init__(self):
        self.product = _i32(self.product)
        self.reward_row = _i32(self.reward_row)
        J = int(self.nodes)
        self.reward_table = np.ascontiguousarray(self.reward_table, np.float64).reshape(-1, J)
        self.capacity = _i32(self.capacity)
        self.inventory = _i32(self.inventory).reshape(int(self.products), J)
        if self.order_t is not None:
            self.order_t = _i32(self.order_t)

    @property
    def origin(self) -> np.ndarray:
        return self.reward_row

    def rewards(self, t: int) -> np.ndarray:
        return self.reward_table[self.reward_row[t]]

    def to_c(self):
        c = K.pcd_instance(int(self.nodes), int(self.products), int(self.horizon),
                           _ptr(self.product), _ptr(self.order_t), _ptr(self.reward_row),
                           _ptr(self.reward_table, C.c_double), int(self.reward_table.shape[0]),
                           _ptr(self.capacity), _ptr(self.inventory))
        return c

    @staticmethod
    def from_orders(nodes: int, products: int, capacity, inventory, orders: Sequence[tuple],
                    order_t=None) -> "Instance":
        """Builds an instance from (product, rewards[J]) records, deduplicating
        reward vectors into a table (rewards are per order in the reference)."""
        rows, index, rr, prod = [], {}, [], []
        for product, rewards in orders:
            key = tuple(float(x) for x in rewards)
            if key not in index:
                index[key] = len(rows)
                rows.append(key)
            rr.append(index[key])
            prod.append(product)
        table = np.array(rows, np.float64).reshape(-1, nodes) if rows else np.zeros((1, nodes))
        inv = np.zeros((products, nodes), np.int32)
        if isinstance(inventory, dict):
            for p, row in inventory.items():
                inv[p] = row
        else:
            inv[:] = np.asarray(inventory).reshape(products, nodes)
        return Instance(nodes, products, len(prod), np.array(prod, np.int32), np.array(rr, np.int32),
                        table, np.asarray(capacity, np.int32), inv, order_t)


def generate_instance(nodes: int, products: int, horizon: int, beta: float, coverage: float = 0.8,
                      seed: int = 0, geometry: Optional[int] = None) -> Instance:
    """fo::generate_instance (instance.cpp:80-140). ``geometry`` None selects the
    reference's 30-city table for nodes <= 30 and the seeded synthetic J-node
    geometry beyond."""
    if geometry is None:
        geometry = 0 if nodes <= 30 else 1
    J, I, T = int(nodes), int(products), int(horizon)
    product = np.zeros(max(T, 1), np.int32)
    origin = np.zeros(max(T, 1), np.int32)
    table = np.zeros(max(J, 1) * max(J, 1), np.float64)
    cap = np.zeros(max(J, 1), np.int32)
    inv = np.zeros(max(I, 1) * max(J, 1), np.int32)
    _check(LIB.pcd_generate_instance(J, I, T, float(beta), float(coverage), int(seed) & (2**64 - 1),
                                     int(geometry), _ptr(product), _ptr(origin), _ptr(table, C.c_double),
                                     _ptr(cap), _ptr(inv)))
    return Instance(J, I, T, product[:T], origin[:T], table[:J * J], cap[:J], inv[:I * J],
                    meta=dict(beta=beta, coverage=coverage, seed=seed, geometry=geometry))


# -------------------------------------------------------------- partitions
@dataclass
class PartitionPlan:
    """PartitionPlan (engine.hpp:74-96): owner[t] in [0, processes)."""
    processes: int
    owner: np.ndarray

    def __post_init__(self):
        self.owner = _i32(self.owner)

    def horizon(self) -> int:
        return int(self.owner.size)


def make_product_partition(instance: Instance, processes: int, seed: int) -> PartitionPlan:
    owner = np.zeros(max(int(instance.horizon), 1), np.int32)
    c = instance.to_c()
    _check(LIB.pcd_product_partition(C.byref(c), int(processes), int(seed) & (2**64 - 1), _ptr(owner)))
    return PartitionPlan(int(processes), owner[:int(instance.horizon)])


def make_product_chunk_partition(instance: Instance, processes: int, seed: int = 1) -> PartitionPlan:
    """Product chunks (ours, ``pcd_product_chunk_partition``): each product's
    orders cut into contiguous near-equal chunks, one process per chunk, so
    up to ``processes`` processes carry work (a product partition activates
    at most I). Falls back to :func:`make_product_partition` when
    ``processes`` is below the number of ordered products."""
    owner = np.zeros(max(int(instance.horizon), 1), np.int32)
    c = instance.to_c()
    _check(LIB.pcd_product_chunk_partition(C.byref(c), int(processes), int(seed) & (2**64 - 1), _ptr(owner)))
    return PartitionPlan(int(processes), owner[:int(instance.horizon)])


def make_product_window_partition(instance: Instance, processes: int, window: int,
                                  seed: int = 1) -> PartitionPlan:
    """Window-aware product chunks (ours, ``pcd_product_window_partition``):
    each product's orders cut greedily so that no ``window``-long interval
    holds more than L orders of one process, L minimal for ``processes``
    chunks. An iteration's critical path at ``PicardConfig(max_steps=window)``
    is then at most L steps; products sparse in time stay whole. Falls back
    to :func:`make_product_partition` when ``processes`` is below the number
    of ordered products."""
    owner = np.zeros(max(int(instance.horizon), 1), np.int32)
    c = instance.to_c()
    _check(LIB.pcd_product_window_partition(C.byref(c), int(processes), int(window), int(seed) & (2**64 - 1),
                                            _ptr(owner)))
    return PartitionPlan(int(processes), owner[:int(instance.horizon)])


def make_uniform_time_partition(horizon: int, processes: int, seed: int) -> PartitionPlan:
    owner = np.zeros(max(int(horizon), 1), np.int32)
    _check(LIB.pcd_uniform_partition(int(horizon), int(processes), int(seed) & (2**64 - 1), _ptr(owner)))
    return PartitionPlan(int(processes), owner[:int(horizon)])


def shard_processes(plan: PartitionPlan, ranks: int) -> np.ndarray:
    """LPT assignment of the plan's processes to ``ranks`` GPUs (rank_of[M])."""
    out = np.zeros(plan.processes, np.int32)
    _check(LIB.pcd_shard_processes(_ptr(plan.owner), int(plan.owner.size), int(plan.processes),
                                   int(ranks), _ptr(out)))
    return out


# ---------------------------------------------------------------- policies
@dataclass
class MlpParams:
    """MlpParams (fo/mlp.hpp:13-36): {input, hidden, hidden, output}, row-major."""
    widths: List[int]
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray
    w3: np.ndarray
    b3: np.ndarray

    @staticmethod
    def zeros(input: int, output: int, hidden: int = 64) -> "MlpParams":
        z = np.zeros
        return MlpParams([input, hidden, hidden, output], z(hidden * input), z(hidden), z(hidden * hidden),
                         z(hidden), z(output * hidden), z(output))

    @staticmethod
    def seeded_uniform(input: int, output: int, seed: int, hidden: int = 64) -> "MlpParams":
        p = MlpParams.zeros(input, output, hidden)
        _check(LIB.pcd_seeded_mlp(int(input), int(output), int(seed) & (2**64 - 1), int(hidden),
                                  *[_ptr(a, C.c_double) for a in (p.w1, p.b1, p.w2, p.b2, p.w3, p.b3)]))
        return p

    def all_zero(self) -> bool:
        return not any(np.any(a) for a in (self.w1, self.b1, self.w2, self.b2, self.w3, self.b3))

    def save(self, path: str):
        """Binary format of MlpParams::save (mlp.cpp:171-183)."""
        with open(path, "wb") as f:
            f.write(np.asarray(self.widths, "<u4").tobytes())
            for a in (self.w1, self.b1, self.w2, self.b2, self.w3, self.b3):
                f.write(np.asarray(a, "<f8").tobytes())

    @staticmethod
    def load(path: str) -> "MlpParams":
        """MlpParams::load (mlp.cpp:185-206); truncated files raise."""
        with open(path, "rb") as f:
            data = f.read()
        if len(data) < 16:
            raise RuntimeError(f"truncated parameter file {path}")
        inp, h, h2, out = np.frombuffer(data[:16], "<u4").astype(int)
        sizes = [h * inp, h, h * h, h, out * h, out]
        need = 16 + 8 * sum(sizes)
        if len(data) < need:
            raise RuntimeError(f"truncated parameter file {path}")
        arrs, off = [], 16
        for n in sizes:
            arrs.append(np.frombuffer(data[off:off + 8 * n], "<f8").copy())
            off += 8 * n
        return MlpParams([int(inp), int(h), int(h2), int(out)], *arrs)


class Policy:
    kind: int = K.PCD_POLICY_NULL
    gamma: float = 0.0
    hidden: int = 64
    horizon: Optional[int] = None
    init_capacity = None
    init_inventory = None
    w1 = b1 = w2 = b2 = w3 = b3 = None

    def to_c(self):
        d = lambda a: None if a is None else a.ctypes.data_as(K.F64P)
        return K.pcd_policy(int(self.kind), int(self.hidden), float(self.gamma),
                            d(self.w1), d(self.b1), d(self.w2), d(self.b2), d(self.w3), d(self.b3),
                            _ptr(self.init_capacity), _ptr(self.init_inventory),
                            -1 if self.horizon is None else int(self.horizon))


class GreedyPolicy(Policy):
    """GreedyPolicy (policies.hpp:24-44)."""
    kind = K.PCD_POLICY_GREEDY


class NullOnlyPolicy(Policy):
    """The always-decline policy of the reference tests (test_engine.cpp:17-22)."""
    kind = K.PCD_POLICY_NULL


class CapacityPenalizedPolicy(Policy):
    """CapacityPenalizedPolicy (policies.hpp:50-75): r_j + gamma * c_j / max c."""
    kind = K.PCD_POLICY_CAPACITY

    def __init__(self, gamma: float = 0.0):
        self.gamma = float(gamma)


class DualNetworkPolicy(Policy):
    """DualNetworkPolicy (policies.hpp:88-174).

    ``initial_capacity``/``initial_inventory``/``horizon`` are the policy's
    normalisation state (``initial_``/``horizon_``); None = the instance's."""
    kind = K.PCD_POLICY_DUAL

    def __init__(self, params: MlpParams, initial_capacity=None, initial_inventory=None,
                 horizon: Optional[int] = None, nodes: Optional[int] = None):
        self.params = params
        J = nodes if nodes is not None else (params.widths[3] // 2)
        if params.widths[0] != 2 * J + 1 or params.widths[3] != 2 * J:
            raise ContractViolation("dual network: layer sizes do not match J")
        self.hidden = params.widths[1]
        self.w1, self.b1, self.w2, self.b2, self.w3, self.b3 = (
            np.ascontiguousarray(a, np.float64) for a in (params.w1, params.b1, params.w2, params.b2,
                                                          params.w3, params.b3))
        self.init_capacity = _i32(initial_capacity)
        self.init_inventory = _i32(initial_inventory)
        self.horizon = horizon

    @staticmethod
    def seeded(instance: Instance, seed: int, horizon: Optional[int] = None) -> "DualNetworkPolicy":
        J = instance.nodes
        return DualNetworkPolicy(MlpParams.seeded_uniform(2 * J + 1, 2 * J, seed), None, None,
                                 instance.horizon if horizon is None else horizon, J)

    @staticmethod
    def zero(instance: Instance, horizon: Optional[int] = None) -> "DualNetworkPolicy":
        J = instance.nodes
        return DualNetworkPolicy(MlpParams.zeros(2 * J + 1, 2 * J), None, None,
                                 instance.horizon if horizon is None else horizon, J)


# ------------------------------------------------------------ config/result
@dataclass
class PicardConfig:
    """PicardConfig (engine.hpp:120-126) + ``engine`` ("auto"/"replay"/"product"/"product_fp64"/"general")."""
    processes: int = 0
    max_steps: int = 0
    max_iterations: int = 0
    record_trace: bool = False
    threads: int = 1
    engine: str = "auto"
    tc_guard: float = 0.0
    tc_verify: bool = False
    tc_tiles: int = 0
    tc_kernel: str = "auto"  # tensor-core sweep: "auto" / "fused" (tc_pp) / "incremental" (tc_inc)

    def to_c(self):
        return K.pcd_config(int(self.processes), 1 if self.record_trace else 0, int(self.max_steps),
                            int(self.max_iterations), int(self.threads), ENGINES[self.engine],
                            float(self.tc_guard), 1 if self.tc_verify else 0, int(self.tc_tiles),
                            TC_KERNELS[self.tc_kernel])


@dataclass
class PicardTraceRow:
    chunk: int
    iteration: int
    changed_slots: int
    max_process_evals: int
    t_reset: int

    def astuple(self):
        return (self.chunk, self.iteration, self.changed_slots, self.max_process_evals, self.t_reset)


@dataclass
class PicardResult:
    actions: np.ndarray
    iterations_to_converged: int = 0
    iterations_to_correct: Optional[int] = None
    conflicts: int = 0
    policy_eval_count_sequential_equivalent: int = 0
    total_policy_evals: int = 0
    trace: List[PicardTraceRow] = field(default_factory=list)
    timing: Optional[dict] = None
    history: Optional[np.ndarray] = None


@dataclass
class IterationOutcome:
    evals_per_process: np.ndarray
    changed_slots: np.ndarray

    def max_process_evals(self) -> int:
        return int(self.evals_per_process.max()) if self.evals_per_process.size else 0

    def total_evals(self) -> int:
        return int(self.evals_per_process.sum())


@dataclass
class SequentialOutput:
    actions: np.ndarray
    policy_evals: int


def _timing_dict(t: K.pcd_timing) -> dict:
    return {name: getattr(t, name) for name, _ in K.pcd_timing._fields_}


# -------------------------------------------------------------- simulator
class Simulator:
    """Device handle: the instance and policy stay resident in HBM across
    calls (pcd_create / pcd_set_plan / pcd_simulate)."""

    def __init__(self, instance: Instance, policy: Policy, device: int = 0):
        self.instance = instance
        self.policy = policy
        self._h = C.c_void_p()
        ci = instance.to_c()
        cp = policy.to_c()
        _check(LIB.pcd_create(C.byref(ci), C.byref(cp), int(device), C.byref(self._h)))
        self.plan: Optional[PartitionPlan] = None

    def close(self):
        if self._h:
            LIB.pcd_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def set_plan(self, plan: PartitionPlan):
        owner = _i32(plan.owner)
        _check(LIB.pcd_set_plan(self._h, _ptr(owner), int(plan.processes)))
        self.plan = plan

    def _trace_buf(self, config: PicardConfig):
        cap = 4 * int(self.instance.horizon) + 16 if config.record_trace else 0
        return (K.pcd_trace_row * max(cap, 1))(), cap

    def _result(self, rc, res, trace, cap, actions):
        rows = [PicardTraceRow(r.chunk, r.iteration, r.changed_slots, r.max_process_evals, r.t_reset)
                for r in trace[:min(res.trace_rows, cap)]]
        if rc == K.PCD_ITERATION_LIMIT:
            raise IterationLimitError(_err(), res.iterations_run, rows)
        _check(rc, res.error_time_step)
        return PicardResult(actions, res.iterations_to_converged,
                            None if res.iterations_to_correct < 0 else res.iterations_to_correct,
                            res.conflicts, res.policy_eval_count_sequential_equivalent,
                            res.total_policy_evals, rows, self.timing())

    def simulate(self, config: Optional[PicardConfig] = None, initial_cache=None,
                 reference_actions=None, record_history: bool = False) -> PicardResult:
        """picard_simulate; ``record_history`` also returns the cache after every
        iteration (like theory::CacheTraceRecorder) in ``result.history``."""
        config = config or PicardConfig()
        T = int(self.instance.horizon)
        init = _i32(initial_cache)
        ref = _i32(reference_actions)
        if init is not None and init.size != T:
            raise ContractViolation("initial cache length must equal the horizon")
        if ref is not None and ref.size != T:
            raise ContractViolation("reference action length must equal the horizon")
        actions = _pinned_i32(T)
        res = K.pcd_result()
        trace, cap = self._trace_buf(config)
        cfg = config.to_c()
        hist = None
        if record_history:
            hcap = 2 * T + 4 if config.max_iterations <= 0 else int(config.max_iterations)
            hist = np.zeros((hcap, max(T, 1)), np.int32)
            _check(LIB.pcd_set_history(self._h, _ptr(hist), hcap))
        try:
            rc = LIB.pcd_simulate(self._h, C.byref(cfg), _ptr(init), _ptr(ref), _ptr(actions), C.byref(res),
                                  trace, cap)
        finally:
            if record_history:
                LIB.pcd_set_history(self._h, None, 0)
        out = self._result(rc, res, trace, cap, actions[:T])
        if record_history:
            out.history = hist[:res.iterations_run, :T].copy()
        return out

    # resident-input variant used by bench.py for the HBM-resident number
    def upload_cache(self, initial_cache=None, reference_actions=None):
        _check(LIB.pcd_upload_cache(self._h, _ptr(_i32(initial_cache)), _ptr(_i32(reference_actions))))

    def simulate_resident(self, config: Optional[PicardConfig] = None, use_initial_cache=False,
                          use_reference=False) -> PicardResult:
        config = config or PicardConfig()
        res = K.pcd_result()
        trace, cap = self._trace_buf(config)
        cfg = config.to_c()
        rc = LIB.pcd_simulate_resident(self._h, C.byref(cfg), int(use_initial_cache), int(use_reference),
                                       C.byref(res), trace, cap)
        return self._result(rc, res, trace, cap, None)

    def download_actions(self) -> np.ndarray:
        a = np.zeros(max(int(self.instance.horizon), 1), np.int32)
        _check(LIB.pcd_download_actions(self._h, _ptr(a)))
        return a[:int(self.instance.horizon)]

    def set_debug(self, flags: int):
        """pcd_set_debug: PCD_DEBUG_* flags (profiling, the sweep kernel of config-less calls)."""
        _check(LIB.pcd_set_debug(self._h, int(flags)))

    def iterate_once(self, cache: np.ndarray, t_lo: int, t_hi: int, checkpoint_capacity=None,
                     checkpoint_inventory=None, engine: str = "auto", tc_kernel: str = "auto") -> IterationOutcome:
        eng = ENGINES[engine]
        self.set_debug({"auto": 0, "fused": 2, "incremental": 4}[tc_kernel])
        assert cache.dtype == np.int32 and cache.flags.c_contiguous
        M = self.plan.processes
        evals = np.zeros(M, np.int64)
        changed = np.zeros(max(int(self.instance.horizon), 1), np.int64)
        n = C.c_int64()
        cc = _i32(checkpoint_capacity)
        ci = _i32(checkpoint_inventory)
        _check(LIB.pcd_iterate_once(self._h, eng, _ptr(cache), int(t_lo), int(t_hi), _ptr(cc), _ptr(ci),
                                    _ptr(evals, C.c_int64), _ptr(changed, C.c_int64), C.byref(n)))
        return IterationOutcome(evals, changed[:n.value].copy())

    def sequential(self) -> SequentialOutput:
        T = int(self.instance.horizon)
        actions = np.zeros(max(T, 1), np.int32)
        ev = C.c_int64()
        _check(LIB.pcd_sequential(self._h, _ptr(actions), C.byref(ev)))
        return SequentialOutput(actions[:T], ev.value)

    def checkpoint_state(self):
        """The device checkpoint FoState (capacities [J], inventory [I, J]);
        after a converged simulate, the trajectory's final state."""
        J, I = int(self.instance.nodes), int(self.instance.products)
        cap = np.zeros(J, np.int32)
        inv = np.zeros(I * J, np.int32)
        _check(LIB.pcd_checkpoint_state(self._h, _ptr(cap), _ptr(inv)))
        return cap, inv.reshape(I, J)

    def timing(self) -> dict:
        t = K.pcd_timing()
        LIB.pcd_last_timing(self._h, C.byref(t))
        return _timing_dict(t)

    def attach_loopback(self, group: "LoopbackGroup", rank: int):
        _check(LIB.pcd_attach_loopback(self._h, C.c_void_p(group._g), int(rank)))

    def attach_comm(self, unique_id: bytes, rank: int, nranks: int):
        buf = (C.c_ubyte * 128).from_buffer_copy(unique_id)
        _check(LIB.pcd_attach_comm(self._h, C.byref(buf), int(rank), int(nranks)))


class LoopbackGroup:
    """In-process loopback communicator of ``nranks`` ranks
    (pcd_loopback_create): the multi-GPU protocol between handles of one
    process, e.g. N Simulators on one GPU each driven by its own thread."""

    def __init__(self, nranks: int):
        self._g = LIB.pcd_loopback_create(int(nranks))
        if not self._g:
            raise InvalidArgument(_err())
        self.nranks = int(nranks)

    def close(self):
        if self._g:
            LIB.pcd_loopback_destroy(self._g)
            self._g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(LIB.pcd_nccl_unique_id(C.byref(buf)))
    return bytes(buf)


# ------------------------------------------------------- functional surface
def picard_simulate(instance: Instance, policy: Policy, plan: PartitionPlan,
                    config: Optional[PicardConfig] = None, initial_cache=None, reference_actions=None,
                    device: int = 0) -> PicardResult:
    """picard_simulate (engine.hpp:458-590) on the B200."""
    config = config or PicardConfig()
    if plan.owner.size != int(instance.horizon):
        raise ContractViolation("partition plan does not cover the horizon")
    with Simulator(instance, policy, device) as sim:
        sim.set_plan(plan)
        return sim.simulate(config, initial_cache, reference_actions)


def picard_iterate_once(instance: Instance, policy: Policy, plan: PartitionPlan, cache: np.ndarray,
                        t_lo: int, t_hi: int, checkpoint_capacity=None, checkpoint_inventory=None,
                        engine: str = "auto", device: int = 0, tc_kernel: str = "auto") -> IterationOutcome:
    """picard_iterate_once (engine.hpp:358-444); ``cache`` is updated in place."""
    with Simulator(instance, policy, device) as sim:
        sim.set_plan(plan)
        return sim.iterate_once(cache, t_lo, t_hi, checkpoint_capacity, checkpoint_inventory, engine, tc_kernel)


def sequential_simulate(instance: Instance, policy: Policy, device: int = 0) -> SequentialOutput:
    """sequential_simulate (engine.hpp:237-267): the serial trajectory (computed
    on the device as the Picard fixed point, Prop. 1)."""
    with Simulator(instance, policy, device) as sim:
        return sim.sequential()


def compare_to_oracle(candidate, oracle):
    """compare_to_oracle (engine.hpp:601-614) -> (equal, first_mismatch|None)."""
    a, b = _i32(candidate), _i32(oracle)
    if a.size != b.size:
        raise ContractViolation("oracle comparison: length mismatch")
    fm = C.c_int64()
    _check(LIB.pcd_compare_actions(_ptr(a), _ptr(b), int(a.size), C.byref(fm)))
    return (fm.value < 0, None if fm.value < 0 else fm.value)


def fo_total_reward(instance: Instance, actions) -> float:
    """fo_total_reward (env.hpp:298-310)."""
    a = _i32(actions)
    if a.size != int(instance.horizon):
        raise ContractViolation("total reward: order/action length mismatch")
    out = C.c_double()
    c = instance.to_c()
    _check(LIB.pcd_total_reward(C.byref(c), _ptr(a), C.byref(out)))
    return out.value


def device_count() -> int:
    return int(LIB.pcd_device_count())


def tc_error_bound(instance: "Instance", policy: "Policy") -> tuple:
    """(B, guard) of the tensor-core sweep for a dual policy on an instance
    (pcd_tc_error_bound; host only): B bounds |score_tc - score_ref| a priori
    (the |best| test uses B (1 + 2^-10)); guard bounds the error of a
    difference of two scores of one row, times 1 + 2^-10 (the best-minus-second
    margin the sweep uses by default); 0 when the policy keeps the exact FP64
    path."""
    b, g = C.c_double(), C.c_double()
    ci, cp = instance.to_c(), policy.to_c()
    _check(LIB.pcd_tc_error_bound(C.byref(ci), C.byref(cp), C.byref(b), C.byref(g)))
    return b.value, g.value


# ------------------------------------------------------------ linear env
@dataclass
class LinearSystemSpec:
    """picard::linear::LinearSystemSpec (linear.hpp:16-31): s_{t+1} = A_t s_t +
    B_t a_t + w_t with dynamics[T, n, n], input[T, n, p], disturbances[T, n],
    gain[p, n] (the GainPolicy a = G s)."""
    state_dim: int
    input_dim: int
    horizon: int
    dynamics: np.ndarray
    input: np.ndarray
    disturbances: np.ndarray
    gain: np.ndarray
    contraction: float = 0.0

    def contractive(self) -> bool:
        return self.contraction < 1.0

    def to_c(self):
        n, p, T = int(self.state_dim), int(self.input_dim), int(self.horizon)
        self._keep = [np.ascontiguousarray(a, np.float64).reshape(-1)
                      for a in (self.dynamics, self.input, self.disturbances, self.gain)]
        if any(k.size != want for k, want in zip(self._keep, (T * n * n, T * n * p, T * n, p * n))):
            raise ContractViolation("linear spec: matrix dimensions disagree")
        return K.pcd_linear_spec(n, p, T, *[_ptr(k, C.c_double) for k in self._keep])


def make_contractive_spec(state_dim: int, input_dim: int, horizon: int, rho: float, seed: int,
                          state_coupling: float = 0.0) -> LinearSystemSpec:
    """linear::make_contractive_spec (linear.cpp:126-218), bit-identical."""
    n, p, T = int(state_dim), int(input_dim), int(horizon)
    A = np.zeros((max(T, 1), n, n))
    B = np.zeros((max(T, 1), n, p))
    W = np.zeros((max(T, 1), n))
    G = np.zeros((p, n))
    rho_out = C.c_double()
    _check(LIB.pcd_linear_contractive_spec(n, p, T, float(rho), int(seed) & (2**64 - 1), float(state_coupling),
                                           _ptr(A, C.c_double), _ptr(B, C.c_double), _ptr(W, C.c_double),
                                           _ptr(G, C.c_double), C.byref(rho_out)))
    return LinearSystemSpec(n, p, T, A[:T], B[:T], W[:T], G, rho_out.value)


@dataclass
class LinearCurve:
    curve: np.ndarray          # relative RMSE after each iteration
    final_cache: np.ndarray    # [T, p] actions after the last iteration
    device_ms: float
    # MLP feedback policy only (None for GainPolicy): picard_simulate's
    # iteration count for the single-step plan, the iterations and device time
    # of the fixed-point pass, and the sequential trajectory [T+1, n]
    iterations_to_converged: Optional[int] = None
    fixed_point_iterations: Optional[int] = None
    fixed_point_ms: Optional[float] = None
    reference_states: Optional[np.ndarray] = None


@dataclass
class MlpFeedbackPolicy:
    """a_t = MlpParams::forward(s_t) (mlp.cpp:141-169) on the linear env: the
    reference's own MLP ({n, H, H, p}, tanh hidden layers, linear output) as a
    PolicyFor<LinearEnv> (engine.hpp:57-61). The reference pairs the linear env
    only with GainPolicy (linear.hpp:104-126); BASELINE config 4 asks for an
    MLP policy."""
    params: MlpParams

    @staticmethod
    def seeded(state_dim: int, input_dim: int, seed: int, hidden: int = 64, output_scale: float = 1.0):
        """MlpParams::seeded_uniform(n, p, seed, hidden) (mlp.cpp:117-129), the
        output layer (w3, b3) multiplied by ``output_scale`` (sets the policy's
        Lipschitz constant, hence the closed-loop contraction)."""
        m = MlpParams.seeded_uniform(state_dim, input_dim, seed, hidden)
        m.w3 = m.w3 * float(output_scale)
        m.b3 = m.b3 * float(output_scale)
        return MlpFeedbackPolicy(m)

    def to_c(self, state_dim: int, input_dim: int):
        m = self.params
        n, H, H2, p = (int(x) for x in m.widths)
        if n != state_dim or p != input_dim or H != H2:
            raise InvalidArgument("mlp widths must be {state_dim, hidden, hidden, input_dim}")
        self._keep = [np.ascontiguousarray(a, np.float64).reshape(-1) for a in (m.w1, m.b1, m.w2, m.b2, m.w3, m.b3)]
        want = (H * n, H, H * H, H, p * H, p)
        if any(k.size != w for k, w in zip(self._keep, want)):
            raise InvalidArgument("mlp parameter sizes disagree with the widths")
        return K.pcd_linear_mlp(H, 0, *[_ptr(k, C.c_double) for k in self._keep])


def picard_convergence_curve(spec: LinearSystemSpec, initial_cache=None, tolerance: float = 1e-3,
                             max_iterations: int = 0, normalization: str = "draft",
                             device: int = 0, policy: Optional[MlpFeedbackPolicy] = None) -> LinearCurve:
    """linear::picard_convergence_curve (linear.cpp:279-330) on the B200:
    single-step partitions (M = T), one affine time-scan per iteration.
    ``policy=None`` is the reference's GainPolicy a = G s; an
    :class:`MlpFeedbackPolicy` evaluates the MLP at all T states per iteration
    (pcd_linear_mlp_convergence_curve)."""
    T, p, n = int(spec.horizon), int(spec.input_dim), int(spec.state_dim)
    cs = spec.to_c()
    init = None if initial_cache is None else np.ascontiguousarray(initial_cache, np.float64).reshape(-1)
    if init is not None and init.size != T * p:
        raise ContractViolation("initial cache length must equal the horizon")
    cap = max(int(max_iterations) if max_iterations > 0 else T, 1)
    curve = np.zeros(cap)
    fin = np.zeros(max(T * p, 1))
    norm = 1 if normalization == "draft" else 0
    if policy is not None:
        cm = policy.to_c(n, p)
        res = K.pcd_linear_mlp_result()
        ref = np.zeros((T + 1) * n)
        _check(LIB.pcd_linear_mlp_convergence_curve(C.byref(cs), C.byref(cm), _ptr(init, C.c_double),
                                                    float(tolerance), int(max_iterations), norm, int(device),
                                                    _ptr(curve, C.c_double), cap, C.byref(res),
                                                    _ptr(fin, C.c_double), _ptr(ref, C.c_double)))
        return LinearCurve(curve[:res.curve_len].copy(), fin[:T * p].reshape(T, p),
                           res.fixed_point_ms + res.curve_ms, res.iterations_to_converged,
                           res.fixed_point_iterations, res.fixed_point_ms, ref.reshape(T + 1, n))
    n_out = C.c_int64()
    ms = C.c_double()
    _check(LIB.pcd_linear_convergence_curve(C.byref(cs), _ptr(init, C.c_double), float(tolerance),
                                            int(max_iterations), norm,
                                            int(device), _ptr(curve, C.c_double), cap, C.byref(n_out),
                                            _ptr(fin, C.c_double), C.byref(ms)))
    return LinearCurve(curve[:n_out.value].copy(), fin[:T * p].reshape(T, p), ms.value)


# ------------------------------------------------------------ Time Warp
@dataclass
class TimeWarpTraceRow:
    round: int
    t_start: int
    window_length: int
    max_process_evals: int
    rolled_back: bool

    def astuple(self):
        return (self.round, self.t_start, self.window_length, self.max_process_evals, int(self.rolled_back))


@dataclass
class TimeWarpResult:
    """timewarp::TimeWarpResult (fo/timewarp.hpp:36-43)."""
    actions: np.ndarray
    sync_rounds: int
    rollbacks: int
    policy_eval_count_sequential_equivalent: int
    total_policy_evals: int
    trace: List[TimeWarpTraceRow]


def time_warp_simulate(instance: Instance, policy: Policy, processes: int, seed: int, record_trace: bool = False,
                       rule: str = "min_capacity", device: int = 0) -> TimeWarpResult:
    """timewarp::time_warp_simulate (fo/timewarp.hpp:56-181) on the B200: the
    safe-window baseline over make_product_partition(processes, seed);
    ``rule`` is "min_capacity" or "min_stocked_capacity"."""
    if rule not in ("min_capacity", "min_stocked_capacity"):
        raise InvalidArgument("unknown window rule")
    T = int(instance.horizon)
    with Simulator(instance, policy, device) as sim:
        actions = _pinned_i32(T)
        res = K.pcd_tw_result()
        cap = 2 * T + 4 if record_trace else 0
        trace = (K.pcd_tw_trace_row * max(cap, 1))()
        rc = LIB.pcd_time_warp(sim._h, int(processes), int(seed) & (2**64 - 1),
                               1 if rule == "min_stocked_capacity" else 0, 1 if record_trace else 0,
                               _ptr(actions), C.byref(res), trace, cap)
        _check(rc, res.error_time_step)
        rows = [TimeWarpTraceRow(r.round, r.t_start, r.window_length, r.max_process_evals, bool(r.rolled_back))
                for r in trace[:min(res.trace_rows, cap)]]
        return TimeWarpResult(actions[:T].copy(), res.sync_rounds, res.rollbacks,
                              res.policy_eval_count_sequential_equivalent, res.total_policy_evals, rows)


# ------------------------------------------------------------ theory / files
@dataclass
class DepletionProfile:
    """theory::DepletionProfile (theory.hpp:30-51)."""
    horizon: int
    first_depleted_at: np.ndarray
    depleted_nodes: np.ndarray
    sorted_depletion_times: np.ndarray

    def depleted_count(self) -> int:
        return int(self.depleted_nodes.size)

    def depleted_before_order(self, node: int, t: int) -> bool:
        return bool(self.first_depleted_at[node] <= t)

    def iteration_bound(self) -> int:
        return self.depleted_count() + 1


def depletion_profile(instance: Instance, actions, device: int = 0) -> DepletionProfile:
    """theory::compute_depletion (theory.hpp:53-86) of the trajectory
    ``actions`` (computed on the device)."""
    T, J = int(instance.horizon), int(instance.nodes)
    a = _i32(actions)
    if a.size != T:
        raise ContractViolation("trajectory length must equal the horizon")
    out = np.zeros(J, np.int64)
    cnt = C.c_int64()
    with Simulator(instance, NullOnlyPolicy(), device) as sim:
        _check(LIB.pcd_depletion_profile(sim._h, _ptr(a), _ptr(out, C.c_int64), C.byref(cnt)))
    nodes = np.flatnonzero(out < T).astype(np.int32)
    return DepletionProfile(T, out, nodes, np.sort(out))


def check_iteration_bound(iterations_to_correct, profile: DepletionProfile):
    """theory::check_iteration_bound (theory.hpp:228-236) -> (bound, satisfied)."""
    bound = profile.iteration_bound()
    return bound, iterations_to_correct is not None and iterations_to_correct <= bound


def save_instance_binary(instance: Instance, path: str) -> None:
    """Binary SoA instance file (pcd_save_instance_bin)."""
    c = instance.to_c()
    _check(LIB.pcd_save_instance_bin(C.byref(c), str(path).encode()))


def load_instance_binary(path: str) -> Instance:
    J, I, T, R, ho = C.c_int32(), C.c_int32(), C.c_int64(), C.c_int64(), C.c_int32()
    _check(LIB.pcd_instance_bin_info(str(path).encode(), C.byref(J), C.byref(I), C.byref(T), C.byref(R),
                                     C.byref(ho)))
    J, I, T, R = J.value, I.value, T.value, R.value
    product = np.zeros(max(T, 1), np.int32)
    rrow = np.zeros(max(T, 1), np.int32)
    ot = np.zeros(max(T, 1), np.int32) if ho.value else None
    table = np.zeros(max(R * J, 1))
    cap = np.zeros(J, np.int32)
    inv = np.zeros(I * J, np.int32)
    _check(LIB.pcd_load_instance_bin(str(path).encode(), _ptr(product), _ptr(rrow), _ptr(ot),
                                     _ptr(table, C.c_double), _ptr(cap), _ptr(inv)))
    return Instance(J, I, T, product[:T], rrow[:T], table[:R * J].reshape(R, J), cap, inv.reshape(I, J),
                    None if ot is None else ot[:T])
