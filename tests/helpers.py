"""Shared test helpers: golden fixtures, oracle/product instance builders."""
from __future__ import annotations

import gzip
import json
import os
from types import SimpleNamespace as NS

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden", "golden.json.gz")


def load_golden():
    with gzip.open(GOLDEN, "rt") as f:
        return json.load(f)


def oracle_instance(spec, lib):
    """Rebuilds a golden case's instance with an oracle library (ORC or REF)."""
    if spec["kind"] == "small_random":
        J, I, T, beta, cov, s = lib.small_random_params(spec["seed"])
        return NS(**lib.generate_instance_arrays(J, I, T, beta, cov, s))
    if spec["kind"] == "generated":
        J, I, T, beta, cov, seed = spec["args"]
        return NS(**lib.generate_instance_arrays(J, I, T, beta, cov, seed, geometry=spec.get("geometry", 0)))
    J = spec["nodes"]
    return NS(nodes=J, products=spec["products"], horizon=len(spec["product"]),
              product=np.array(spec["product"], np.int32), order_t=None,
              reward_row=np.array(spec["reward_row"], np.int32),
              reward_table=np.array(spec["reward_table"], np.float64),
              capacity=np.array(spec["capacity"], np.int32), inventory=np.array(spec["inventory"], np.int32))


def oracle_policy(spec, inst, lib):
    p = NS(kind=spec["kind"], hidden=64, gamma=spec["gamma"], horizon=None)
    if spec["kind"] == 2:
        J = inst.nodes
        p.w1, p.b1, p.w2, p.b2, p.w3, p.b3 = lib.seeded_mlp(2 * J + 1, 2 * J, spec["seed"])
    return p


def product_instance(ns):
    """Product-API Instance from an oracle namespace (same arrays)."""
    from paper_2406_01939_b200 import Instance
    return Instance(ns.nodes, ns.products, ns.horizon, ns.product, ns.reward_row, ns.reward_table,
                    ns.capacity, ns.inventory, getattr(ns, "order_t", None))


def product_policy(spec, inst):
    import paper_2406_01939_b200 as P
    k = spec["kind"]
    if k == 0:
        return P.GreedyPolicy()
    if k == 1:
        return P.CapacityPenalizedPolicy(spec["gamma"])
    if k == 3:
        return P.NullOnlyPolicy()
    J = inst.nodes
    return P.DualNetworkPolicy(P.MlpParams.seeded_uniform(2 * J + 1, 2 * J, spec["seed"]), nodes=J)


def all_cases(golden, groups=("toy_two_order", "toy_single_process", "infeasible_cache", "oracle_grid",
                              "textbook_grid", "initial_cache_grid", "window_grid", "medium")):
    out = []
    for g in groups:
        v = golden["cases"][g]
        for i, c in enumerate(v if isinstance(v, list) else [v]):
            out.append((f"{g}[{i}]", c))
    return out


def is_run_partition(owner, product):
    """The closed-form engines' plan condition (engine.cu: k_check_runs): every
    (process, product) stretch is contiguous in the product's slot list, and a
    process with several stretches owns only whole products."""
    owner = np.asarray(owner)
    product = np.asarray(product)
    runs = {}
    for p in np.unique(product):
        own = owner[product == p]
        cut = np.flatnonzero(np.diff(own)) + 1
        for k, o in enumerate(np.split(own, cut)):
            runs.setdefault(int(o[0]), []).append(k == 0)
    return all(len(v) == 1 or all(v) for v in runs.values())
