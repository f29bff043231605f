"""TEST INFRASTRUCTURE — regenerates tests/golden/ from the UNMODIFIED reference.

Runs the reference library (oracle/_ref/libpicard_ref.so, built from
/root/reference/proj by oracle/Makefile) on the known-answer cases of the
reference test suite and on seeded grids that restate its property tests,
and writes the outputs as fixtures. /root/reference does not exist on the GPU
box, so the committed fixtures are what pins the oracle there.

    python oracle/make_golden.py            # writes tests/golden/golden.json.gz

Case recipes (reference test file:line they restate):
  toy_two_order        test_helpers.hpp:17-29, test_engine.cpp:100-138
  infeasible_cache     test_engine.cpp:140-173
  oracle_grid          test_engine.cpp:301-348 (seeds 100..139, same RNG draws)
  textbook_grid        test_engine.cpp:229-299 (seeds 500..511)
  initial_cache_grid   test_engine.cpp:350-371 (seeds 200..211)
  window_grid          test_engine.cpp:455-477 (seeds 300..309, widths 0/1/3/17)
  dual_forward         test_policies.cpp:134-188
  demand / apportion   test_instance.cpp:28-54
  product_hand_trace   test_instance.cpp:213-241
  medium               generate_instance(10, 100, 5000) + dual seed 5 (product / uniform, M=64)
"""
from __future__ import annotations

import gzip
import json
import os
import sys
from types import SimpleNamespace as NS

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path[0] = ROOT

from oracle.oracle import REF  # noqa: E402


class MT64:
    """std::mt19937_64 (only used to re-derive the test-suite's parameter draws)."""

    def __init__(self, seed):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def __call__(self):
        M = 0xFFFFFFFFFFFFFFFF
        if self.idx >= 312:
            for i in range(312):
                x = (self.mt[i] & 0xFFFFFFFF80000000) | (self.mt[(i + 1) % 312] & 0x7FFFFFFF)
                xa = x >> 1
                if x & 1:
                    xa ^= 0xB5026F5AA96619E9
                self.mt[i] = self.mt[(i + 156) % 312] ^ xa
            self.idx = 0
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000 & M
        y ^= (y << 37) & 0xFFF7EEE000000000 & M
        y ^= y >> 43
        return y & M

    def below(self, n):
        if n <= 1:
            return 0
        M = 0xFFFFFFFFFFFFFFFF
        limit = M - M % n
        while True:
            v = self()
            if v < limit:
                return v % n

    def unit(self):
        return (self() >> 11) * 2.0 ** -53


def small_random(seed, lib=None):
    lib = lib or REF
    J, I, T, beta, cov, s = lib.small_random_params(seed)
    d = lib.generate_instance_arrays(J, I, T, beta, cov, s)
    return NS(**d), dict(kind="small_random", seed=seed)


def policy(kind, inst=None, seed=None, gamma=0.0, lib=None):
    lib = lib or REF
    p = NS(kind=kind, hidden=64, gamma=float(gamma), horizon=None)
    spec = dict(kind=kind, gamma=float(gamma), seed=seed)
    if kind == 2:
        J = inst.nodes
        w = lib.seeded_mlp(2 * J + 1, 2 * J, seed)
        p.w1, p.b1, p.w2, p.b2, p.w3, p.b3 = w
    return p, spec


def L(a):
    return None if a is None else np.asarray(a).tolist()


def run_case(inst, inst_spec, pol, pol_spec, owner, M, cfg, initial=None, history=False):
    seq, _ = REF.sequential(inst, pol)
    r = REF.picard(inst, pol, owner, M, max_steps=cfg.get("max_steps", 0), record_trace=True,
                   reference=seq, history=history, initial_cache=initial)
    return dict(instance=inst_spec, policy=pol_spec, owner=L(owner), processes=int(M), config=cfg,
                initial_cache=L(initial), sequential=L(seq), actions=L(r.actions),
                iterations_to_converged=r.iterations_to_converged,
                iterations_to_correct=r.iterations_to_correct, conflicts=r.conflicts,
                seq_equiv=r.policy_eval_count_sequential_equivalent,
                total_evals=r.total_policy_evals, trace=[list(x) for x in r.trace],
                history=L(r.history) if history else None,
                total_reward=REF.total_reward(inst, r.actions))


def explicit_instance(J, I, cap, inv, products, rewards):
    table = np.array(rewards, np.float64).reshape(-1, J)
    return NS(nodes=J, products=I, horizon=len(products), product=np.array(products, np.int32),
              order_t=None, reward_row=np.arange(len(products), dtype=np.int32), reward_table=table,
              capacity=np.array(cap, np.int32), inventory=np.array(inv, np.int32).ravel())


def explicit_spec(inst):
    return dict(kind="explicit", nodes=inst.nodes, products=inst.products, capacity=L(inst.capacity),
                inventory=L(inst.inventory), product=L(inst.product), reward_row=L(inst.reward_row),
                reward_table=L(inst.reward_table.ravel()))


def main():
    assert REF is not None, "oracle/_ref not built (make -C oracle)"
    out = dict(meta=dict(source="/root/reference/proj via oracle/_ref/libpicard_ref.so",
                         tanh_variant="host libm"), cases={})
    C = out["cases"]

    # ---- toy two-order (test_helpers.hpp:17-29)
    toy = explicit_instance(2, 1, [1, 1], [[1, 1]], [0, 0], [[0.9, 0.1], [0.8, 0.2]])
    g, gs = policy(0)
    C["toy_two_order"] = run_case(toy, explicit_spec(toy), g, gs, [0, 1], 2, dict(max_steps=0), history=True)
    cache, evals, changed = REF.iterate_once(toy, g, np.array([0, 1], np.int32), 2, np.array([-1, -1], np.int32), 0, 2)
    C["toy_two_order"]["iterate_once_1"] = dict(cache=L(cache), evals=L(evals), changed=L(changed))
    cache2, _, _ = REF.iterate_once(toy, g, np.array([0, 1], np.int32), 2, cache, 0, 2)
    C["toy_two_order"]["iterate_once_2"] = dict(cache=L(cache2))
    C["toy_single_process"] = run_case(toy, explicit_spec(toy), g, gs, [0, 0], 1, dict(max_steps=0))

    # ---- infeasible cached action (test_engine.cpp:140-173)
    inf = explicit_instance(1, 1, [1], [[3]], [0, 0, 0], [[1.0], [1.0], [1.0]])
    C["infeasible_cache"] = run_case(inf, explicit_spec(inf), g, gs, [0, 1, 0], 2, dict(max_steps=0),
                                     initial=np.array([0, 0, 0], np.int32), history=True)

    # ---- oracle equivalence grid (test_engine.cpp:301-348)
    grid = []
    for seed in range(100, 140):
        inst, spec = small_random(seed)
        gen = MT64(seed * 977)
        M = 1 + gen.below(8)
        product_part = gen.below(2) == 0
        owner = REF.product_partition(inst, M, seed) if product_part else REF.uniform_partition(inst.horizon, M, seed)
        ms = 0 if gen.below(3) == 0 else 1 + gen.below(20)
        pols = [policy(0)]
        gamma = gen.unit() * 2.0
        pols.append(policy(1, gamma=gamma))
        if seed % 4 == 0:
            pols.append(policy(2, inst, seed + 5))
        for p, ps in pols:
            grid.append(run_case(inst, spec, p, ps, owner, M, dict(max_steps=ms), history=True))
    C["oracle_grid"] = grid

    # ---- textbook iterates (test_engine.cpp:229-299)
    tb = []
    for seed in range(500, 512):
        gen = MT64(seed)
        inst, spec = small_random(seed)
        M = 2 + gen.below(3)
        owner = REF.product_partition(inst, M, seed) if seed % 2 == 0 else REF.uniform_partition(inst.horizon, M, seed)
        for p, ps in (policy(0), policy(1, gamma=1.5)):
            tb.append(run_case(inst, spec, p, ps, owner, M, dict(max_steps=0), history=True))
    C["textbook_grid"] = tb

    # ---- initial-cache independence (test_engine.cpp:350-371) + windows (:395-414)
    ic = []
    for seed in list(range(200, 212)) + [401]:
        inst, spec = small_random(seed)
        owner = REF.product_partition(inst, 4, seed if seed != 401 else 1)
        gamma = 1.0 if seed != 401 else 2.0
        draft, _ = REF.sequential(inst, policy(1, gamma=gamma)[0])
        for ms in (0, 5):
            ic.append(run_case(inst, spec, *policy(0), owner, 4, dict(max_steps=ms), initial=draft, history=True))
    C["initial_cache_grid"] = ic

    # ---- window-width invariance (test_engine.cpp:455-477)
    wg = []
    for seed in range(300, 310):
        inst, spec = small_random(seed)
        owner = REF.uniform_partition(inst.horizon, 3, seed)
        for ms in (0, 1, 3, 17):
            wg.append(run_case(inst, spec, *policy(0), owner, 3, dict(max_steps=ms), history=True))
    C["window_grid"] = wg

    # ---- dual forward-pass oracle (test_policies.cpp:134-188)
    J = 3
    init_inst = explicit_instance(3, 1, [4, 4, 4], [[2, 2, 2]], [0] * 10, [[0.3, 0.8, 0.6]] * 10)
    init_inst.order_t = np.arange(10, dtype=np.int32)
    p, ps = policy(2, init_inst, 99)
    p.horizon = 10
    a = REF.policy_evaluate(init_inst, p, np.array([2, 4, 1], np.int32), np.array([1, 0, 2], np.int32), 4)
    f = np.array([2 / 4, 4 / 4, 1 / 4, 1 / 2, 0 / 2, 2 / 2, 4 / 10])
    prices = REF.mlp_forward(p, f)
    C["dual_forward"] = dict(seed=99, state_capacity=[2, 4, 1], state_inventory=[1, 0, 2], t=4, horizon=10,
                             rewards=[0.3, 0.8, 0.6], init_capacity=[4, 4, 4], init_inventory=[2, 2, 2],
                             action=a, features=L(f), prices=[float(x).hex() for x in prices])

    # ---- instance pieces (test_instance.cpp)
    C["demand_counts"] = [dict(args=[4, 8, 0.0], out=L(REF.demand_counts(4, 8, 0.0))),
                          dict(args=[4, 120000, -1.0], out=L(REF.demand_counts(4, 120000, -1.0))),
                          dict(args=[50, 12345, -0.7], out=L(REF.demand_counts(50, 12345, -0.7)))]
    C["apportion"] = [dict(weights=[3e6, 1e6], total=80, out=L(REF.apportion([3e6, 1e6], 80))),
                      dict(weights=[1.0, 1.0, 1.0], total=7, out=L(REF.apportion([1.0, 1.0, 1.0], 7)))]
    hand = explicit_instance(1, 4, [10], [[0]] * 4, [0, 0, 0, 0, 1, 1, 1, 2, 2, 3], [[1.0]] * 10)
    C["product_hand_trace"] = dict(owner_m2=L(REF.product_partition(hand, 2, 3)),
                                   owner_m1=L(REF.product_partition(hand, 1, 3)))
    C["uniform_partition"] = dict(args=[10000, 10, 1234], owner_sha=None,
                                  counts=L(np.bincount(REF.uniform_partition(10000, 10, 1234), minlength=10)))
    gi = []
    for args in [(5, 40, 1000, -0.6, 0.8, 1), (3, 20, 200, 0.0, 0.8, 5), (1, 10, 10000, 0.0, 0.8, 7),
                 (30, 300, 3000, -0.4, 0.8, 7)]:
        d = REF.generate_instance_arrays(*args)
        gi.append(dict(args=list(args), product=L(d["product"]), origin=L(d["reward_row"]),
                       reward_table=[float(x).hex() for x in d["reward_table"]], capacity=L(d["capacity"]),
                       inventory=L(d["inventory"])))
    d = REF.generate_instance_arrays(100, 50, 2000, 0.0, 0.8, 7, geometry=1)
    gi.append(dict(args=[100, 50, 2000, 0.0, 0.8, 7], geometry=1, product=L(d["product"]), origin=L(d["reward_row"]),
                   reward_table=[float(x).hex() for x in d["reward_table"]], capacity=L(d["capacity"]),
                   inventory=L(d["inventory"])))
    C["generate_instance"] = gi

    # ---- medium dual runs (no history)
    med = []
    for geometry, (J, I, T) in ((0, (10, 100, 5000)), (1, (40, 100, 4000))):
        d = REF.generate_instance_arrays(J, I, T, 0.0, 0.8, 7, geometry=geometry)
        inst = NS(**d)
        spec = dict(kind="generated", args=[J, I, T, 0.0, 0.8, 7], geometry=geometry)
        for part in ("product", "uniform"):
            owner = REF.product_partition(inst, 64, 1) if part == "product" else REF.uniform_partition(T, 64, 1)
            p, ps = policy(2, inst, 5)
            med.append(run_case(inst, spec, p, ps, owner, 64, dict(max_steps=0)))
    C["medium"] = med

    # ---- tanh bit patterns of the host libm
    rng = np.random.default_rng(7)
    xs = np.concatenate([rng.uniform(-3, 3, 1500), rng.uniform(-25, 25, 300), rng.standard_normal(200) * 1e-3])
    C["tanh"] = [[float(x).hex(), float(REF.tanh(float(x))).hex()] for x in xs]

    os.makedirs(os.path.join(ROOT, "tests", "golden"), exist_ok=True)
    path = os.path.join(ROOT, "tests", "golden", "golden.json.gz")
    with gzip.open(path, "wt") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path))


if __name__ == "__main__":
    main()
