"""Multi-GPU host logic on CPU: world_size-2 `gloo` emulation of the engine's
per-iteration exchange.

Each rank owns the processes `shard_processes` assigns it (LPT over loads),
computes fresh values only for their slots (here with the CPU oracle as the
stand-in for the device sweep), packs them in rank-major time order, and an
all_gather (ncclAllGather on the B200 path) plus SUM/MIN/MAX all_reduces of
the convergence scalars rebuild the identical cache and counters on every
rank. The full Picard loop driven this way must reproduce the single-rank
oracle iterate-by-iterate.
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2406_01939_b200 as P


def _slot_lists(owner, rank_of, nranks):
    r_of_t = rank_of[owner]
    order = np.argsort(r_of_t, kind="stable")  # rank-major, time order within a rank
    counts = np.bincount(r_of_t, minlength=nranks)
    off = np.concatenate([[0], np.cumsum(counts)])
    return order.astype(np.int64), off


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from types import SimpleNamespace as NS
        from oracle.oracle import ORC
        ons = NS(**ORC.generate_instance_arrays(10, 60, 3000, 0.0, 0.8, 7))
        inst = P.Instance(ons.nodes, ons.products, ons.horizon, ons.product, ons.reward_row, ons.reward_table,
                          ons.capacity, ons.inventory)
        plan = P.make_product_partition(inst, 24, 1)
        rank_of = P.shard_processes(plan, world)
        slots, off = _slot_lists(plan.owner, rank_of, world)
        maxn = int(np.max(off[1:] - off[:-1]))
        pol = NS(kind=2, hidden=64, gamma=0.0, horizon=None)
        pol.w1, pol.b1, pol.w2, pol.b2, pol.w3, pol.b3 = ORC.seeded_mlp(21, 20, 5)
        T = int(inst.horizon)
        seq, _ = ORC.sequential(ons, pol)
        want = ORC.picard(ons, pol, plan.owner, 24, record_trace=True, reference=seq, history=True)

        cache = np.full(T, -1, np.int32)
        cap, inv = ons.capacity.copy(), ons.inventory.copy()
        written = np.zeros(T, bool)
        ws, it, conflicts, rows = 0, 0, 0, []
        mine_slots = slots[off[rank]:off[rank + 1]]
        while ws < T:
            it += 1
            full, evals, _ = ORC.iterate_once(ons, pol, plan.owner, 24, cache, ws, T, cap, inv)
            # this rank's contribution: its own slots only (the device sweep's output)
            own = mine_slots[(mine_slots >= ws)]
            send = np.full(maxn, -2, np.int64)
            send[:len(mine_slots)] = full[mine_slots]
            recv = [torch.zeros(maxn, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(recv, torch.from_numpy(send))
            new = cache.copy()
            for r in range(world):
                seg = slots[off[r]:off[r + 1]]
                new[seg] = recv[r].numpy()[:len(seg)]
            assert np.array_equal(new, full), "exchange must rebuild the full cache"
            # scalar reductions (per-owner counts -> SUM / MIN / MAX)
            ch = own[new[own] != cache[own]]
            s = torch.tensor([len(ch), int(written[ch].sum())], dtype=torch.int64)
            dist.all_reduce(s, op=dist.ReduceOp.SUM)
            fc = torch.tensor([int(ch.min()) if len(ch) else T], dtype=torch.int64)
            dist.all_reduce(fc, op=dist.ReduceOp.MIN)
            mine_procs = np.nonzero(rank_of == rank)[0]
            mx = torch.tensor([int(evals[mine_procs].max()) if len(mine_procs) else 0], dtype=torch.int64)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)
            n_changed, conf, first = int(s[0]), int(s[1]), int(fc[0])
            assert n_changed == int((new[ws:] != cache[ws:]).sum())
            assert mx.item() == int(evals.max())
            conflicts += conf
            written[ws:] = True
            rows.append((0, it, n_changed, int(mx.item()), ws))
            cache = new
            assert np.array_equal(cache, want.history[it - 1]), f"iteration {it}"
            if n_changed == 0:
                break
            if first > ws:  # checkpoint advance (replicated on every rank)
                for t in range(ws, first):
                    a = cache[t]
                    if a >= 0:
                        cap[a] -= 1
                        inv[ons.product[t] * ons.nodes + a] -= 1
                ws = first
        assert np.array_equal(cache, seq)
        assert conflicts == want.conflicts
        assert rows == [tuple(r) for r in want.trace]
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_exchange_reproduces_single_rank_iterates():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert out == {0: "ok", 1: "ok"}, out


def test_shards_cover_every_process_once():
    inst = P.generate_instance(10, 1000, 100000, 0.0, 0.8, 7)
    plan = P.make_product_partition(inst, 4096, 1)
    for world in (2, 4, 8):
        r = P.shard_processes(plan, world)
        slots, off = _slot_lists(plan.owner, r, world)
        assert sorted(slots.tolist()) == list(range(inst.horizon))
        for k in range(world):
            seg = slots[off[k]:off[k + 1]]
            assert np.all(np.diff(seg) > 0)
            assert np.all(r[plan.owner[seg]] == k)
