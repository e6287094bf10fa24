"""Host side of the NEXT-1 tuning loop: rounds of
``TLP.ga_round`` (every step of a round runs in libtlp's kernels) plus the
measurement bookkeeping an auto-tuner does between rounds.

P:558: "Put the last selected n tensor programs on the target machine to
measure the latency. ... All our experiments are tuned for 200 rounds, each
round picking 10 tensor programs to measure".  Multi-GPU: one process per GPU,
each tuning a contiguous block of subgraphs (dist.shard_subgraphs, id_base =
the block's first global id) -- the tuning round has no exchange step, so
there is no collective on the data path; ``Tuner.gather`` collects the
per-subgraph bests afterwards.  The "target machine" is a
caller-supplied ``measure(s, genes) -> latency`` (synth.template_latency in
the tests and the bench); a measured program is cached and never re-measured
(R48).  Subgraphs are visited round-robin.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Dict, List, Tuple

import numpy as np


@dataclass
class Trajectory:
    measurements: List[int] = field(default_factory=list)   # cumulative, per round
    best: List[List[float]] = field(default_factory=list)   # per round, per subgraph
    measured: List[List[Tuple[int, Tuple[int, ...], float]]] = field(default_factory=list)


class Tuner:
    """Round-robin tuner over a ctx whose search space is set (ga_set_space)."""

    def __init__(self, model, n_subgraphs: int, knob_counts, n_pop: int = 512, n_child: int = 1920,
                 iters: int = 4, p_cross: float = 0.5, p_mut: float = 0.2, seed: int = 0, head: int = 0,
                 id_base: int = 0):
        self.m = model
        self.S = n_subgraphs
        self.id_base = id_base  # global id of this ctx's subgraph 0 (sharded tuning)
        self.K = [int(k) for k in knob_counts]
        self.kw = dict(n_pop=n_pop, n_child=n_child, iters=iters, p_cross=p_cross, p_mut=p_mut,
                       seed=seed, head=head)
        self.seen: List[Dict[Tuple[int, ...], float]] = [dict() for _ in range(n_subgraphs)]
        self.best = [float("inf")] * n_subgraphs
        self.total = 0
        self.traj = Trajectory()

    def run_round(self, rnd: int, measure: Callable[[int, np.ndarray], float], per_round: int = 10):
        kw = self.kw
        genes, scores = self.m.ga_round(kw["n_pop"], kw["n_child"], kw["iters"], kw["p_cross"],
                                        kw["p_mut"], kw["seed"], rnd, kw["head"])
        g = genes.cpu().numpy().reshape(self.S, kw["n_pop"], -1)
        sc = scores.cpu().numpy().reshape(self.S, kw["n_pop"])
        picked = []
        for s in range(self.S):
            got = 0
            for row, v in zip(g[s], sc[s]):
                if got == per_round:
                    break
                if not np.isfinite(v):
                    continue
                key = tuple(int(x) for x in row[:self.K[s]])
                if key in self.seen[s]:
                    continue
                lat = float(measure(self.id_base + s, np.asarray(key, np.int64)))
                self.seen[s][key] = lat
                self.best[s] = min(self.best[s], lat)
                picked.append((self.id_base + s, key, lat))
                got += 1
                self.total += 1
        self.traj.measurements.append(self.total)
        self.traj.best.append(list(self.best))
        self.traj.measured.append(picked)
        return picked

    def gather(self, group=None):
        """Multi-rank bookkeeping (after tuning; not on the data path): every
        rank receives the global per-subgraph best latencies and measurement
        count, in global subgraph order (torch.distributed all_gather_object)."""
        import torch.distributed as dist
        if not dist.is_initialized() or dist.get_world_size(group) == 1:
            return list(self.best), self.total
        parts = [None] * dist.get_world_size(group)
        dist.all_gather_object(parts, (self.id_base, list(self.best), self.total), group=group)
        parts.sort(key=lambda x: x[0])
        return [b for _, bs, _ in parts for b in bs], sum(t for _, _, t in parts)

    def tune(self, rounds: int, measure, per_round: int = 10) -> Trajectory:
        for rnd in range(rounds):
            self.run_round(rnd, measure, per_round)
        return self.traj
