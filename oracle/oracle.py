"""TEST INFRASTRUCTURE ONLY — ctypes front-end to the two CPU oracles.

``ORC``  : oracle/liboracle.so — plain-C restatement of the reference hot path
           (oracle/picard_oracle.c), pinned by tests/test_oracle.py.
``REF``  : oracle/_ref/libpicard_ref.so — the unmodified reference library
           (/root/reference/proj) + oracle/ref_harness.cpp; ``None`` when it
           was not built (e.g. the reference tree is absent and no prebuilt
           copy travelled with the repo).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs import this
module.  It duck-types instances/policies (any object with the attributes of
``paper_2406_01939_b200.api.Instance`` / ``Policy``) so it never imports the
product package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_I32P = C.POINTER(C.c_int32)
_I64P = C.POINTER(C.c_int64)
_F64P = C.POINTER(C.c_double)


class CInstance(C.Structure):
    _fields_ = [("nodes", C.c_int32), ("products", C.c_int32), ("horizon", C.c_int64),
                ("product", _I32P), ("order_t", _I32P), ("reward_row", _I32P),
                ("reward_table", _F64P), ("reward_rows", C.c_int64),
                ("capacity", _I32P), ("inventory", _I32P)]


class CPolicy(C.Structure):
    _fields_ = [("kind", C.c_int32), ("hidden", C.c_int32), ("gamma", C.c_double),
                ("w1", _F64P), ("b1", _F64P), ("w2", _F64P), ("b2", _F64P),
                ("w3", _F64P), ("b3", _F64P), ("init_capacity", _I32P),
                ("init_inventory", _I32P), ("horizon", C.c_int64)]


class CConfig(C.Structure):
    _fields_ = [("processes", C.c_int32), ("record_trace", C.c_int32),
                ("max_steps", C.c_int64), ("max_iterations", C.c_int64),
                ("threads", C.c_int32), ("engine", C.c_int32)]


class CTraceRow(C.Structure):
    _fields_ = [("chunk", C.c_int64), ("iteration", C.c_int64), ("changed_slots", C.c_int64),
                ("max_process_evals", C.c_int64), ("t_reset", C.c_int64)]


class CResult(C.Structure):
    _fields_ = [("iterations_to_converged", C.c_int64), ("iterations_to_correct", C.c_int64),
                ("conflicts", C.c_int64),
                ("policy_eval_count_sequential_equivalent", C.c_int64),
                ("total_policy_evals", C.c_int64), ("trace_rows", C.c_int64),
                ("iterations_run", C.c_int64), ("error_time_step", C.c_int64)]


def _p(a, ctype):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ctype))


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str, time_step: int = -1):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.time_step = time_step


@dataclass
class OracleResult:
    actions: np.ndarray
    iterations_to_converged: int
    iterations_to_correct: Optional[int]
    conflicts: int
    policy_eval_count_sequential_equivalent: int
    total_policy_evals: int
    trace: list
    history: Optional[np.ndarray]


def _keep(*arrays):
    return [np.ascontiguousarray(a) if a is not None else None for a in arrays]


class _Lib:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib
        f = lambda n: getattr(L, f"{prefix}_{n}")
        f("last_error").restype = C.c_char_p
        f("tanh").restype = C.c_double
        f("tanh").argtypes = [C.c_double]

    def fn(self, name):
        return getattr(self.lib, f"{self.prefix}_{name}")

    def err(self) -> str:
        return self.fn("last_error")().decode()

    def check(self, rc, time_step=-1):
        if rc != 0:
            raise OracleError(rc, self.err(), time_step)

    # -------------------------------------------------------------- inputs
    def _inst(self, inst):
        arrays = dict(product=np.ascontiguousarray(inst.product, np.int32),
                      order_t=None if getattr(inst, "order_t", None) is None
                      else np.ascontiguousarray(inst.order_t, np.int32),
                      reward_row=np.ascontiguousarray(inst.reward_row, np.int32),
                      reward_table=np.ascontiguousarray(inst.reward_table, np.float64),
                      capacity=np.ascontiguousarray(inst.capacity, np.int32),
                      inventory=np.ascontiguousarray(inst.inventory, np.int32))
        c = CInstance(int(inst.nodes), int(inst.products), int(inst.horizon),
                      _p(arrays["product"], C.c_int32), _p(arrays["order_t"], C.c_int32),
                      _p(arrays["reward_row"], C.c_int32), _p(arrays["reward_table"], C.c_double),
                      int(arrays["reward_table"].size // max(1, int(inst.nodes))),
                      _p(arrays["capacity"], C.c_int32), _p(arrays["inventory"], C.c_int32))
        return c, arrays

    def _pol(self, pol):
        keep = {}
        def arr(name, dt):
            v = getattr(pol, name, None)
            if v is None:
                return None
            keep[name] = np.ascontiguousarray(v, dt)
            return keep[name]
        c = CPolicy(int(pol.kind), int(getattr(pol, "hidden", 64)), float(getattr(pol, "gamma", 0.0)),
                    _p(arr("w1", np.float64), C.c_double), _p(arr("b1", np.float64), C.c_double),
                    _p(arr("w2", np.float64), C.c_double), _p(arr("b2", np.float64), C.c_double),
                    _p(arr("w3", np.float64), C.c_double), _p(arr("b3", np.float64), C.c_double),
                    _p(arr("init_capacity", np.int32), C.c_int32),
                    _p(arr("init_inventory", np.int32), C.c_int32),
                    int(getattr(pol, "horizon", -1) if getattr(pol, "horizon", None) is not None else -1))
        return c, keep

    def tanh(self, x: float) -> float:
        return self.fn("tanh")(float(x))

    def demand_counts(self, products, horizon, beta):
        out = np.zeros(products, np.int64)
        self.check(self.fn("demand_counts")(C.c_int32(products), C.c_int64(horizon),
                                            C.c_double(beta), _p(out, C.c_int64)))
        return out

    def apportion(self, weights, total):
        w = np.ascontiguousarray(weights, np.float64)
        out = np.zeros(len(w), np.int64)
        self.check(self.fn("apportion")(_p(w, C.c_double), C.c_int64(len(w)), C.c_int64(total),
                                        _p(out, C.c_int64)))
        return out

    def generate_instance_arrays(self, J, I, T, beta, coverage=0.8, seed=0, geometry=0):
        product = np.zeros(T, np.int32)
        origin = np.zeros(T, np.int32)
        table = np.zeros(J * J, np.float64)
        cap = np.zeros(J, np.int32)
        inv = np.zeros(I * J, np.int32)
        self.check(self.fn("generate_instance")(
            C.c_int32(J), C.c_int32(I), C.c_int64(T), C.c_double(beta), C.c_double(coverage),
            C.c_uint64(seed), C.c_int32(geometry), _p(product, C.c_int32), _p(origin, C.c_int32),
            _p(table, C.c_double), _p(cap, C.c_int32), _p(inv, C.c_int32)))
        return dict(nodes=J, products=I, horizon=T, product=product, order_t=None,
                    reward_row=origin, reward_table=table, capacity=cap, inventory=inv)

    def small_random_params(self, seed):
        n = C.c_int32(); p = C.c_int32(); h = C.c_int64(); b = C.c_double(); cv = C.c_double()
        s = C.c_uint64()
        self.fn("small_random_params")(C.c_uint64(seed), C.byref(n), C.byref(p), C.byref(h),
                                       C.byref(b), C.byref(cv), C.byref(s))
        return n.value, p.value, h.value, b.value, cv.value, s.value

    def product_partition(self, inst, M, seed):
        c, keep = self._inst(inst)
        owner = np.zeros(int(inst.horizon), np.int32)
        self.check(self.fn("product_partition")(C.byref(c), C.c_int32(M), C.c_uint64(seed),
                                                _p(owner, C.c_int32)))
        return owner

    def uniform_partition(self, T, M, seed):
        owner = np.zeros(int(T), np.int32)
        self.check(self.fn("uniform_partition")(C.c_int64(T), C.c_int32(M), C.c_uint64(seed),
                                                _p(owner, C.c_int32)))
        return owner

    def seeded_mlp(self, inp, out, seed, hidden=64):
        a = [np.zeros(hidden * inp), np.zeros(hidden), np.zeros(hidden * hidden), np.zeros(hidden),
             np.zeros(out * hidden), np.zeros(out)]
        self.check(self.fn("seeded_mlp")(C.c_int32(inp), C.c_int32(out), C.c_uint64(seed),
                                         C.c_int32(hidden), *[_p(x, C.c_double) for x in a]))
        return a

    def mlp_forward(self, pol, x):
        c, keep = self._pol(pol)
        x = np.ascontiguousarray(x, np.float64)
        nout = len(pol.b3)
        out = np.zeros(nout)
        self.check(self.fn("mlp_forward")(C.byref(c), C.c_int32(len(x)), C.c_int32(nout),
                                          _p(x, C.c_double), _p(out, C.c_double)))
        return out

    def policy_evaluate(self, inst, pol, cap, inv, t):
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        cap = np.ascontiguousarray(cap, np.int32)
        inv = np.ascontiguousarray(inv, np.int32)
        a = C.c_int32()
        self.check(self.fn("policy_evaluate")(C.byref(ci), C.byref(cp), _p(cap, C.c_int32),
                                              _p(inv, C.c_int32), C.c_int64(t), C.byref(a)))
        return a.value

    # -------------------------------------------------------------- engine
    def sequential(self, inst, pol):
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        actions = np.zeros(int(inst.horizon), np.int32)
        ev = C.c_int64()
        et = C.c_int64(-1)
        rc = self.fn("sequential")(C.byref(ci), C.byref(cp), _p(actions, C.c_int32), C.byref(ev),
                                   C.byref(et))
        self.check(rc, et.value)
        return actions, ev.value

    def picard(self, inst, pol, owner, M, max_steps=0, max_iterations=0, record_trace=False,
               threads=1, initial_cache=None, reference=None, history=False, processes=0):
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        T = int(inst.horizon)
        owner, initial_cache, reference = _keep(np.asarray(owner, np.int32),
                                                None if initial_cache is None else np.asarray(initial_cache, np.int32),
                                                None if reference is None else np.asarray(reference, np.int32))
        cfg = CConfig(processes, 1 if record_trace else 0, max_steps, max_iterations, threads, 0)
        actions = np.zeros(max(T, 1), np.int32)
        res = CResult()
        cap = 4 * T + 16
        trace = (CTraceRow * cap)()
        hist = np.zeros((cap if history else 0, T), np.int32) if history else None
        rc = self.fn("picard")(C.byref(ci), C.byref(cp), _p(owner, C.c_int32), C.c_int32(M),
                               C.byref(cfg), _p(initial_cache, C.c_int32), _p(reference, C.c_int32),
                               _p(actions, C.c_int32), C.byref(res), trace, C.c_int64(cap),
                               _p(hist, C.c_int32) if history else None,
                               C.c_int64(cap if history else 0))
        rows = [(r.chunk, r.iteration, r.changed_slots, r.max_process_evals, r.t_reset)
                for r in trace[:min(res.trace_rows, cap)]]
        if rc != 0:
            e = OracleError(rc, self.err(), res.error_time_step)
            e.iterations_run = res.iterations_run
            e.partial_trace = rows
            raise e
        k = res.iterations_run
        return OracleResult(actions[:T].copy(), res.iterations_to_converged,
                            None if res.iterations_to_correct < 0 else res.iterations_to_correct,
                            res.conflicts, res.policy_eval_count_sequential_equivalent,
                            res.total_policy_evals, rows, hist[:k].copy() if history else None)

    def iterate_once(self, inst, pol, owner, M, cache, lo, hi, ck_cap=None, ck_inv=None):
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        T = int(inst.horizon)
        owner = np.ascontiguousarray(owner, np.int32)
        cache = np.array(cache, np.int32, copy=True)
        ck_cap = np.ascontiguousarray(inst.capacity if ck_cap is None else ck_cap, np.int32)
        ck_inv = np.ascontiguousarray(inst.inventory if ck_inv is None else ck_inv, np.int32)
        evals = np.zeros(M, np.int64)
        changed = np.zeros(max(T, 1), np.int64)
        n = C.c_int64()
        et = C.c_int64(-1)
        rc = self.fn("iterate_once")(C.byref(ci), C.byref(cp), _p(owner, C.c_int32), C.c_int32(M),
                                     _p(cache, C.c_int32), C.c_int64(lo), C.c_int64(hi),
                                     _p(ck_cap, C.c_int32), _p(ck_inv, C.c_int32),
                                     _p(evals, C.c_int64), _p(changed, C.c_int64), C.byref(n),
                                     C.byref(et))
        self.check(rc, et.value)
        return cache, evals, changed[:n.value].copy()

    def naive_fixed_point(self, inst, pol, owner, M):
        assert self.prefix == "orc"
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        T = int(inst.horizon)
        owner = np.ascontiguousarray(owner, np.int32)
        cap = 2 * T + 4
        hist = np.zeros((cap, max(T, 1)), np.int32)
        k = C.c_int64()
        self.check(self.fn("naive_fixed_point")(C.byref(ci), C.byref(cp), _p(owner, C.c_int32),
                                                C.c_int32(M), _p(hist, C.c_int32), C.c_int64(cap),
                                                C.byref(k)))
        return hist[:k.value, :T].copy()

    def sequential_timed(self, inst, pol):
        """REF only: (actions, seconds of sequential_simulate alone)."""
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        actions = np.zeros(max(int(inst.horizon), 1), np.int32)
        sec = C.c_double()
        self.check(self.fn("sequential_timed")(C.byref(ci), C.byref(cp), _p(actions, C.c_int32), C.byref(sec)))
        return actions[:int(inst.horizon)], sec.value

    def picard_timed(self, inst, pol, owner, M, max_steps=0, threads=1):
        """REF only: (actions, iterations, seq_equiv, seconds of picard_simulate alone)."""
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        owner = np.ascontiguousarray(owner, np.int32)
        actions = np.zeros(max(int(inst.horizon), 1), np.int32)
        it = C.c_int64()
        se = C.c_int64()
        sec = C.c_double()
        self.check(self.fn("picard_timed")(C.byref(ci), C.byref(cp), _p(owner, C.c_int32), C.c_int32(M),
                                           C.c_int64(max_steps), C.c_int32(threads), _p(actions, C.c_int32),
                                           C.byref(it), C.byref(se), C.byref(sec)))
        return actions[:int(inst.horizon)], it.value, se.value, sec.value

    def session(self, inst, pol):
        """REF only: a segmented sequential trajectory (RefSession)."""
        return RefSession(self, inst, pol)

    def depletion(self, inst, actions):
        ci, k1 = self._inst(inst)
        out = np.zeros(int(inst.nodes), np.int64)
        a = np.ascontiguousarray(actions, np.int32)
        self.check(self.fn("depletion")(C.byref(ci), _p(a, C.c_int32), _p(out, C.c_int64)))
        return out

    # ---------------------------------------------------------- Time Warp
    # (reference harness only: ref_time_warp, fo/timewarp.hpp:56-181)
    def time_warp(self, inst, pol, processes, seed, rule=0, record_trace=True):
        ci, k1 = self._inst(inst)
        cp, k2 = self._pol(pol)
        T = int(inst.horizon)
        actions = np.zeros(max(T, 1), np.int32)
        counters = np.zeros(4, np.int64)
        cap = 2 * T + 4
        trace = np.zeros((cap, 5), np.int64)
        rows = C.c_int64()
        et = C.c_int64(-1)
        rc = self.fn("time_warp")(C.byref(ci), C.byref(cp), C.c_int32(processes), C.c_uint64(seed), C.c_int32(rule),
                                  C.c_int32(1 if record_trace else 0), _p(actions, C.c_int32),
                                  _p(counters, C.c_int64), _p(trace, C.c_int64), C.c_int64(cap), C.byref(rows),
                                  C.byref(et))
        self.check(rc, et.value)
        return actions[:T], counters, trace[:min(rows.value, cap)]

    # ---------------------------------------------------------- linear env
    # (reference harness only: ref_linear_* in ref_harness.cpp)
    def linear_spec(self, n, p, T, rho, seed, coupling=0.0):
        A = np.zeros((max(T, 1), n, n)); B = np.zeros((max(T, 1), n, p)); W = np.zeros((max(T, 1), n))
        G = np.zeros((p, n)); c = C.c_double()
        self.check(self.fn("linear_spec")(C.c_int32(n), C.c_int32(p), C.c_int64(T), C.c_double(rho),
                                          C.c_uint64(seed), C.c_double(coupling), _p(A, C.c_double),
                                          _p(B, C.c_double), _p(W, C.c_double), _p(G, C.c_double), C.byref(c)))
        return A[:T], B[:T], W[:T], G, c.value

    def linear_curve(self, spec, initial_cache=None, tolerance=1e-3, max_iterations=0, normalization="draft"):
        n, p, T = spec.state_dim, spec.input_dim, spec.horizon
        arrs = [np.ascontiguousarray(a, np.float64) for a in (spec.dynamics, spec.input, spec.disturbances, spec.gain)]
        init = None if initial_cache is None else np.ascontiguousarray(initial_cache, np.float64)
        cap = max(max_iterations if max_iterations > 0 else T, 1)
        curve = np.zeros(cap); ln = C.c_int64()
        self.check(self.fn("linear_curve")(C.c_int32(n), C.c_int32(p), C.c_int64(T),
                                           *[_p(a, C.c_double) for a in arrs], _p(init, C.c_double),
                                           C.c_double(tolerance), C.c_int64(max_iterations),
                                           C.c_int32(1 if normalization == "draft" else 0), _p(curve, C.c_double),
                                           C.c_int64(cap), C.byref(ln)))
        return curve[:ln.value].copy()

    def linear_sequential(self, spec):
        n, p, T = spec.state_dim, spec.input_dim, spec.horizon
        arrs = [np.ascontiguousarray(a, np.float64) for a in (spec.dynamics, spec.input, spec.disturbances, spec.gain)]
        acts = np.zeros((max(T, 1), p)); states = np.zeros((T + 1, n))
        self.check(self.fn("linear_sequential")(C.c_int32(n), C.c_int32(p), C.c_int64(T),
                                                *[_p(a, C.c_double) for a in arrs], _p(acts, C.c_double),
                                                _p(states, C.c_double)))
        return acts[:T], states

    # MLP feedback policy on the linear env (ref_linear_mlp_* in ref_harness.cpp:
    # the reference's MlpParams::forward as a PolicyFor<LinearEnv>)
    def _lin_mlp_args(self, spec, mlp):
        n, p, T = spec.state_dim, spec.input_dim, spec.horizon
        arrs = [np.ascontiguousarray(a, np.float64) for a in (spec.dynamics, spec.input, spec.disturbances)]
        ws = [np.ascontiguousarray(a, np.float64) for a in (mlp.w1, mlp.b1, mlp.w2, mlp.b2, mlp.w3, mlp.b3)]
        self._lin_keep = arrs + ws
        return ([C.c_int32(n), C.c_int32(p), C.c_int64(T)] + [_p(a, C.c_double) for a in arrs]
                + [C.c_int32(int(mlp.widths[1]))] + [_p(a, C.c_double) for a in ws])

    def linear_mlp_curve(self, spec, mlp, initial_cache=None, tolerance=1e-3, max_iterations=0,
                         normalization="draft"):
        T = spec.horizon
        init = None if initial_cache is None else np.ascontiguousarray(initial_cache, np.float64)
        cap = max(max_iterations if max_iterations > 0 else T, 1)
        curve = np.zeros(cap); ln = C.c_int64()
        self.check(self.fn("linear_mlp_curve")(*self._lin_mlp_args(spec, mlp), _p(init, C.c_double),
                                               C.c_double(tolerance), C.c_int64(max_iterations),
                                               C.c_int32(1 if normalization == "draft" else 0),
                                               _p(curve, C.c_double), C.c_int64(cap), C.byref(ln)))
        return curve[:ln.value].copy()

    def linear_mlp_sequential(self, spec, mlp):
        n, p, T = spec.state_dim, spec.input_dim, spec.horizon
        acts = np.zeros((max(T, 1), p)); states = np.zeros((T + 1, n))
        self.check(self.fn("linear_mlp_sequential")(*self._lin_mlp_args(spec, mlp), _p(acts, C.c_double),
                                                    _p(states, C.c_double)))
        return acts[:T], states

    def linear_mlp_picard(self, spec, mlp, initial_cache=None, threads=1):
        p, T = spec.input_dim, spec.horizon
        init = None if initial_cache is None else np.ascontiguousarray(initial_cache, np.float64)
        acts = np.zeros((max(T, 1), p)); it = C.c_int64()
        self.check(self.fn("linear_mlp_picard")(*self._lin_mlp_args(spec, mlp), _p(init, C.c_double),
                                                C.c_int32(threads), C.byref(it), _p(acts, C.c_double)))
        return it.value, acts[:T]

    def total_reward(self, inst, actions):
        ci, k1 = self._inst(inst)
        a = np.ascontiguousarray(actions, np.int32)
        out = C.c_double()
        self.check(self.fn("total_reward")(C.byref(ci), _p(a, C.c_int32), C.byref(out)))
        return out.value


class RefSession:
    """The reference's sequential_simulate run as consecutive segments over one
    marshalled instance (ref_session_* in ref_harness.cpp): ``run(t1)`` times
    sequential_simulate over [at, t1) from the carried state and returns
    (actions, seconds). Concatenated segments are one serial trajectory."""

    def __init__(self, lib, inst, pol):
        self.lib = lib
        self.J, self.I, self.T = int(inst.nodes), int(inst.products), int(inst.horizon)
        self._ci, self._k1 = lib._inst(inst)
        self._cp, self._k2 = lib._pol(pol)
        f = lib.fn("session_create")
        f.restype = C.c_void_p
        self.h = f(C.byref(self._ci), C.byref(self._cp))
        if not self.h:
            raise OracleError(1, lib.err())
        lib.fn("session_destroy").argtypes = [C.c_void_p]
        lib.fn("session_sequential").argtypes = [C.c_void_p, C.c_int64, _I32P, C.POINTER(C.c_double),
                                                 C.POINTER(C.c_int64)]
        lib.fn("session_set_state").argtypes = [C.c_void_p, C.c_int64, _I32P, _I32P]
        lib.fn("session_get_state").argtypes = [C.c_void_p, C.POINTER(C.c_int64), _I32P, _I32P]

    def run(self, t1):
        t1 = int(t1)
        _, at, _, _ = self.state()
        actions = np.zeros(max(t1 - at, 1), np.int32)
        sec = C.c_double()
        et = C.c_int64(-1)
        rc = self.lib.fn("session_sequential")(self.h, t1, _p(actions, C.c_int32), C.byref(sec), C.byref(et))
        self.lib.check(rc, et.value)
        return actions[:t1 - at], sec.value

    def total_reward(self, actions):
        a = np.ascontiguousarray(actions, np.int32)
        out = C.c_double()
        f = self.lib.fn("session_total_reward")
        f.argtypes = [C.c_void_p, _I32P, C.POINTER(C.c_double)]
        self.lib.check(f(self.h, _p(a, C.c_int32), C.byref(out)))
        return out.value

    def set_state(self, t, cap, inv):
        cap = np.ascontiguousarray(cap, np.int32)
        inv = np.ascontiguousarray(inv, np.int32)
        self.lib.check(self.lib.fn("session_set_state")(self.h, int(t), _p(cap, C.c_int32), _p(inv, C.c_int32)))

    def state(self):
        cap = np.zeros(self.J, np.int32)
        inv = np.zeros(self.I * self.J, np.int32)
        t = C.c_int64()
        self.lib.check(self.lib.fn("session_get_state")(self.h, C.byref(t), _p(cap, C.c_int32), _p(inv, C.c_int32)))
        return None, t.value, cap, inv

    def close(self):
        if self.h:
            self.lib.fn("session_destroy")(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def build(quiet=True):
    """Builds liboracle.so (+ _ref when the reference tree exists)."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def _load(path, prefix):
    return _Lib(path, prefix) if os.path.exists(path) else None


_orc_path = os.path.join(HERE, "liboracle.so")
if not os.path.exists(_orc_path):
    build()
ORC = _load(_orc_path, "orc")
REF = _load(os.path.join(HERE, "_ref", "libpicard_ref.so"), "ref")
if ORC is not None:
    ORC.lib.orc_tanh_nofma.restype = C.c_double
    ORC.lib.orc_tanh_nofma.argtypes = [C.c_double]
    ORC.lib.orc_expm1.restype = C.c_double
    ORC.lib.orc_expm1.argtypes = [C.c_double]
    ORC.lib.orc_expm1_nofma.restype = C.c_double
    ORC.lib.orc_expm1_nofma.argtypes = [C.c_double]
    ORC.lib.orc_tanh_variant.restype = C.c_int
