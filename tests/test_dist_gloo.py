"""N > 1 host path on CPU: world_size-2 torch.distributed (gloo) processes run
the data-parallel protocol of SURVEY §8(e) with the product's sharding helpers
(paper_2211_03578_b200.dist) and the CPU oracle for the arithmetic:

* scoring: contiguous 5-aligned candidate shards, per-rank top-k with global
  indices, all_gather, merge  ==  unsharded top-k;
* training: whole groups per rank, all_reduce of the per-task strict-pair
  counts (C-0), per-rank gradients scaled by the global counts, all_reduce of
  the gradients (C-1)  ==  unsharded gradient.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import synth
from oracle import model as OM
from oracle import rank_loss as OLR
from oracle import select as SEL
from oracle.dp import full_grad
from paper_2211_03578_b200 import dist as D

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # ---- scoring: sharded top-k merge
        rng = np.random.default_rng(0)
        N, T, k = 1003, 7, 16
        scores = rng.choice(np.float32([0.0, -0.0, 1.0, 0.5]), size=N).astype(np.float32)
        scores[rng.random(N) < 0.5] = rng.normal(size=int((rng.random(N) < 0.5).sum()) or 1)[0]
        task_off = np.sort(np.concatenate([[0, N], rng.integers(0, N, T - 1)])).astype(np.int64)
        lo, hi = D.shard_range(N, world, rank)
        assert lo % D.TILE == 0
        idx, val = SEL.topk(scores[lo:hi], D.local_task_off(task_off, lo, hi), k, base=lo)
        gathered = [None] * world
        dist.all_gather_object(gathered, (idx, val))
        merged = []
        for t in range(T):
            cand = [(float(v), int(i)) for (ii, vv) in gathered for v, i in zip(vv[t], ii[t]) if i >= 0]
            cand.sort(key=lambda c: (-(c[0] + 0.0), c[1]))
            merged.append([i for _, i in cand[:k]])
        ref_idx, _ = SEL.topk(scores, task_off, k)
        ok_topk = all(merged[t] == [i for i in ref_idx[t] if i >= 0] for t in range(T))

        # ---- training: data-parallel gradient with global pair counts
        cfg = OM.Config(L=6, E=8, T=3, hidden=16, up_dims=(16,), attn_heads=4, head_dim=8, n_tasks=2)
        flat = np.concatenate([v.ravel() for v in synth.init_params(3, OM.param_shapes(cfg), bf16=False)])
        r2 = np.random.default_rng(1)
        goff = np.array([0, 5, 9, 17, 20, 28, 33, 40], np.int64)
        X = r2.normal(size=(40, cfg.L, cfg.E))
        lab = r2.uniform(0.05, 1, (40, 2))
        lab[r2.random(40) < 0.5, 0] = np.nan
        groups = D.assign_groups(goff, world, seed=5)[rank]
        rows, loff = D.gather_groups(goff, groups)
        P_local = OLR.strict_pair_counts(lab[rows], loff).astype(np.float64)
        P = torch.tensor(P_local)
        dist.all_reduce(P)                                   # C-0
        _, g = full_grad(cfg, flat, X[rows], lab[rows], loff, P.numpy())
        gt = torch.tensor(g)
        dist.all_reduce(gt)                                  # C-1
        _, g_ref = full_grad(cfg, flat, X, lab, goff)
        ok_grad = bool(np.abs(gt.numpy() - g_ref).max() <= 1e-12 * np.abs(g_ref).max())
        q.put((rank, ok_topk, ok_grad, lo, hi))
    finally:
        dist.destroy_process_group()


def test_world2_protocol_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    assert all(r[1] for r in res), res   # sharded top-k == unsharded
    assert all(r[2] for r in res), res   # DP gradient == unsharded
    assert res[0][3] == 0 and res[0][4] == res[1][3] and res[1][4] == 1003  # shards tile [0, N)


@pytest.mark.parametrize("n,world", [(0, 1), (7, 2), (409600, 8), (1003, 3), (4, 4)])
def test_shard_range_tiles_and_aligns(n, world):
    prev = 0
    for r in range(world):
        lo, hi = D.shard_range(n, world, r)
        assert lo == prev and (lo % D.TILE == 0 or lo == n) and hi >= lo
        prev = hi
    assert prev == n


def test_assign_groups_partitions_all_groups():
    goff = np.concatenate([[0], np.cumsum(synth.group_sizes(0, 37, lo=24, hi=4000, mean=2000))])
    parts = D.assign_groups(goff, 8, seed=1)
    allg = np.sort(np.concatenate(parts))
    assert np.array_equal(allg, np.arange(37))
    loads = [int(np.diff(goff)[p].sum()) for p in parts]
    assert max(loads) - min(loads) <= 4000


# ---------------------------------------------------------------- NEXT-1 sharded tuning
def _tune_worker(rank, world, port, q):
    """Each rank tunes its contiguous block of subgraphs (dist.shard_subgraphs)
    with global ids; Tuner-style gather of the per-subgraph bests over gloo."""
    import synth
    from oracle import search as OS
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S = 5
        ts = [synth.make_template(41, s) for s in range(S)]
        lo, hi = D.shard_subgraphs(S, world, rank)
        lat = lambda s, g: float(synth.template_latency(ts[s], g, 41, s)[0])  # noqa: E731
        cost = lambda s, g: -np.log(synth.template_latency(ts[s], g, 41, s)) + 0.2 * np.cos(g.sum(1))  # noqa: E731
        traj = OS.tune(ts[lo:hi], cost, lat, rounds=2, measure=3, seed=4, n_pop=8, n_child=16, iters=2,
                       p_cross=0.5, p_mut=0.3, ids=list(range(lo, hi)))
        parts = [None] * world
        dist.all_gather_object(parts, (lo, traj["best"][-1], [m for r in traj["measured"] for m in r]))
        q.put((rank, sorted(parts, key=lambda x: x[0])))
    finally:
        dist.destroy_process_group()


def test_sharded_tuning_equals_unsharded():
    import synth
    from oracle import search as OS
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_tune_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    S = 5
    ts = [synth.make_template(41, s) for s in range(S)]
    lat = lambda s, g: float(synth.template_latency(ts[s], g, 41, s)[0])  # noqa: E731
    cost = lambda s, g: -np.log(synth.template_latency(ts[s], g, 41, s)) + 0.2 * np.cos(g.sum(1))  # noqa: E731
    full = OS.tune(ts, cost, lat, rounds=2, measure=3, seed=4, n_pop=8, n_child=16, iters=2,
                   p_cross=0.5, p_mut=0.3)
    for rank in range(WORLD):
        parts = res[rank]
        best = [b for _, bs, _ in parts for b in bs]
        assert best == full["best"][-1]
        measured = sorted(m for _, _, ms in parts for m in ms)
        assert measured == sorted(m for r in full["measured"] for m in r)
    assert [D.shard_subgraphs(S, WORLD, r) for r in range(WORLD)] == [(0, 3), (3, 5)]
