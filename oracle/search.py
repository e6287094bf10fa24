"""O11 the synthetic Ansor-style tuning round.
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:558 (§6.3): "Ansor will first generate some initial tensor programs for a
subgraph according to predefined rules.  Then use the cost model to pick out
potential tensor programs.  Use these potential tensor programs to generate
more tensor programs through the genetic algorithm and use the cost model
again to prune the poor performers.  This step will iterate multiple times.
Put the last selected n tensor programs on the target machine to measure the
latency.  The above is called a tuning round. ... All our experiments are
tuned for 200 rounds, each round picking 10 tensor programs to measure".
P:598: "approximately 10,000 schedule primitive sequences are performed for
feature extraction and latency prediction for each subgraph in one round".

The paper fixes neither the genetic operators nor the pool sizes; SPEC
S:515-521 names them (fitness-proportional parent selection, numeric-argument
mutation by a step within the domain, crossover at primitive boundaries).
Readings (R44-R48):
  R44  random numbers: Philox4x64-10 (pinned against numpy's Philox) with
       key (seed, 0x544C50) and counter (c, s, round<<16 | iter,
       stream<<32 | block); word j of a block is the j-th output.  Every
       integer decision uses only integer arithmetic on the words:
       uniform index in [0, n) = floor(w * n / 2^64); a Bernoulli(p) draw is
       (w >> 11) < floor(p * 2^53).
  R45  a candidate is one domain index per knob (synth.Template); the initial
       programs are uniform draws of every knob (stream 1, block j/4).
  R46  fitness-proportional selection over the survivors ranked by (score
       desc, index asc): the rank-r survivor has fitness n - r (linear
       ranking, so the decision is exact integer arithmetic and independent
       of the scores' scale); u = floor(w * F / 2^64), F = n(n+1)/2, picks the
       smallest r with C(r) = (r+1) n - r(r+1)/2 > u.
  R47  child = parent A; with probability p_cross (if the subgraph has >= 2
       knob-bearing primitives) one-point crossover at a primitive boundary:
       knobs of the primitives with group ordinal >= cut come from parent B,
       cut uniform in [1, groups).  Then each knob mutates with probability
       p_mut by one step up (bit 0 of its word = 1) or down inside its domain,
       reflected at the ends (stream 3, block j/4).  Selection words are
       stream 2 block 0: (A, B, crossover coin, cut).
  R48  a round per subgraph: n_pop + n_child initial programs are scored and
       the n_pop best survive; then `iters` times n_child children are bred
       from the survivors, scored, and the best n_pop of survivors + children
       survive (ties by position: survivors first, then children).  A program
       equal to an earlier one of the same pool (pool order) is a duplicate
       and gets score -inf before the pruning (Ansor keeps unique states), so
       survivors are distinct unless the pool has fewer than n_pop distinct
       programs; parents are drawn from the n_eff finite-score survivors only.
       The round's output is the survivors in rank order; the tuner measures
       the first `measure` finite-score ones whose gene vectors were never
       measured before (a measured program is cached and never re-measured,
       SPEC S:529).
"""
from __future__ import annotations

from typing import Callable, Dict, List, Sequence, Tuple

import numpy as np

MASK64 = (1 << 64) - 1
KEY1 = 0x544C50
STREAM_INIT, STREAM_SEL, STREAM_MUT = 1, 2, 3


def philox4x64_10(ctr: Sequence[int], key: Sequence[int]) -> List[int]:
    """Philox4x64 with 10 rounds (Salmon et al., SC'11): four 64-bit words."""
    x = [int(v) & MASK64 for v in ctr]
    k0, k1 = int(key[0]) & MASK64, int(key[1]) & MASK64
    for r in range(10):
        if r:
            k0 = (k0 + 0x9E3779B97F4A7C15) & MASK64
            k1 = (k1 + 0xBB67AE8584CAA73B) & MASK64
        p0 = 0xD2E7470EE14C6C93 * x[0]
        p1 = 0xCA5A826395121157 * x[2]
        x = [(p1 >> 64) ^ x[1] ^ k0, p1 & MASK64, (p0 >> 64) ^ x[3] ^ k1, p0 & MASK64]
    return x


def word(seed: int, c: int, s: int, rnd: int, it: int, stream: int, j: int) -> int:
    """R44: word j of stream `stream` for candidate c of subgraph s."""
    ctr = (c, s, (rnd << 16) | it, (stream << 32) | (j >> 2))
    return philox4x64_10(ctr, (seed, KEY1))[j & 3]


def uniform_index(w: int, n: int) -> int:
    return (w * n) >> 64


def bernoulli(w: int, p: float) -> bool:
    return (w >> 11) < int(p * 9007199254740992.0)


def init_genes(dom_sizes: Sequence[int], n: int, seed: int, s: int, rnd: int) -> np.ndarray:
    """R45: n uniform programs of subgraph s."""
    G = len(dom_sizes)
    out = np.zeros((n, G), np.int64)
    for c in range(n):
        for j in range(G):
            out[c, j] = uniform_index(word(seed, c, s, rnd, 0, STREAM_INIT, j), int(dom_sizes[j]))
    return out


def rank_order(scores: np.ndarray) -> np.ndarray:
    """Positions sorted by (score desc, position asc) (R21, R46)."""
    sc = [float(v) + 0.0 for v in np.asarray(scores, np.float64)]
    return np.array(sorted(range(len(sc)), key=lambda i: (-sc[i], i)), np.int64)


def cumulative_fitness(r: int, n: int) -> int:
    """C(r) = sum_{q<=r} (n - q)."""
    return (r + 1) * n - r * (r + 1) // 2


def select_rank(u: int, n: int) -> int:
    """R46: smallest r with C(r) > u, by scanning the ranks in order."""
    for r in range(n):
        if cumulative_fitness(r, n) > u:
            return r
    raise ValueError("u outside [0, F)")


def drop_duplicates(genes: np.ndarray, scores: np.ndarray) -> np.ndarray:
    """R48: scores with every row equal to an earlier row replaced by -inf."""
    out = np.array(scores, np.float64, copy=True)
    first = {}
    for i, row in enumerate(np.asarray(genes)):
        key = tuple(int(v) for v in row)
        if key in first:
            out[i] = -np.inf
        else:
            first[key] = i
    return out


def evolve(pop: np.ndarray, dom_sizes: Sequence[int], groups: Sequence[int], n_child: int,
           p_cross: float, p_mut: float, seed: int, s: int, rnd: int, it: int,
           n_eff: int | None = None) -> np.ndarray:
    """R46/R47: n_child children of the survivors ``pop`` (rank order, best
    first) of subgraph s; parents come from the first n_eff survivors."""
    pop = np.asarray(pop, np.int64)
    n, G = pop.shape
    if n_eff is not None:
        n = n_eff
    groups = np.asarray(groups, np.int64)
    n_groups = int(groups.max()) + 1 if G else 0
    F = n * (n + 1) // 2
    out = np.zeros((n_child, G), np.int64)
    for c in range(n_child):
        wa, wb, wx, wc = (word(seed, c, s, rnd, it, STREAM_SEL, j) for j in range(4))
        ra = select_rank(uniform_index(wa, F), n)
        rb = select_rank(uniform_index(wb, F), n)
        child = pop[ra].copy()
        if n_groups >= 2 and bernoulli(wx, p_cross):
            cut = 1 + uniform_index(wc, n_groups - 1)
            take_b = groups >= cut
            child[take_b] = pop[rb][take_b]
        for j in range(G):
            D = int(dom_sizes[j])
            w = word(seed, c, s, rnd, it, STREAM_MUT, j)
            if D >= 2 and bernoulli(w, p_mut):
                v = int(child[j])
                if w & 1:
                    v = v + 1 if v + 1 < D else v - 1
                else:
                    v = v - 1 if v > 0 else v + 1
                child[j] = v
        out[c] = child
    return out


def materialize(tmpl, genes: np.ndarray) -> List[list]:
    """The abstract primitive sequences of gene vectors: the
    skeleton with knob g's argument replaced by domains[g][gene[g]]."""
    out = []
    for row in np.atleast_2d(genes):
        seq = [(t, list(a)) for t, a in tmpl.prims]
        for g in range(tmpl.G):
            seq[tmpl.knob_prim[g]][1][tmpl.knob_arg[g]] = tmpl.domains[g][int(row[g])]
        out.append(seq)
    return out


CostModel = Callable[[int, np.ndarray], np.ndarray]


def search_round(tmpl, s: int, cost_model: CostModel, seed: int, rnd: int, n_pop: int,
                 n_child: int, iters: int, p_cross: float, p_mut: float
                 ) -> Tuple[np.ndarray, np.ndarray]:
    """R48: survivors (genes [n_pop, G] in rank order, scores) of one round of
    subgraph s; ``cost_model(s, genes)`` returns one score per gene row."""
    D = tmpl.dom_sizes()
    grp = tmpl.knob_groups()
    genes = init_genes(D, n_pop + n_child, seed, s, rnd)
    scores = drop_duplicates(genes, np.asarray(cost_model(s, genes), np.float64))
    keep = rank_order(scores)[:n_pop]
    pop, ps = genes[keep], scores[keep]
    for it in range(1, iters + 1):
        n_eff = int(np.isfinite(ps).sum())
        ch = evolve(pop, D, grp, n_child, p_cross, p_mut, seed, s, rnd, it, n_eff)
        cs = np.asarray(cost_model(s, ch), np.float64)
        allg = np.concatenate([pop, ch])
        alls = drop_duplicates(allg, np.concatenate([ps, cs]))
        keep = rank_order(alls)[:n_pop]
        pop, ps = allg[keep], alls[keep]
    return pop, ps


def tune(templates, cost_model: CostModel, latency: Callable[[int, np.ndarray], float],
         rounds: int, measure: int, seed: int, n_pop: int, n_child: int, iters: int,
         p_cross: float, p_mut: float, ids: Sequence[int] | None = None) -> Dict[str, list]:
    """Round-robin over the subgraphs: every round every subgraph
    runs search_round and measures its first `measure` never-measured
    survivors.  Returns the trajectory: per round the measurements spent and
    the best measured latency per subgraph so far.  ``ids`` are the subgraphs'
    global ids (the random-number counters and the callables' first argument;
    default 0..S-1)."""
    S = len(templates)
    seen: List[Dict[Tuple[int, ...], float]] = [dict() for _ in range(S)]
    best = [float("inf")] * S
    traj: Dict[str, list] = {"measurements": [], "best": [], "measured": []}
    total = 0
    for rnd in range(rounds):
        picked = []
        for s in range(S):
            sid = s if ids is None else int(ids[s])
            pop, ps = search_round(templates[s], sid, cost_model, seed, rnd, n_pop, n_child, iters,
                                   p_cross, p_mut)
            got = 0
            for row, sc in zip(pop, ps):
                if got == measure:
                    break
                if not np.isfinite(sc):
                    continue
                key = tuple(int(v) for v in row)
                if key in seen[s]:
                    continue
                lat = float(latency(sid, row))
                seen[s][key] = lat
                best[s] = min(best[s], lat)
                picked.append((sid, key, lat))
                got += 1
                total += 1
        traj["measurements"].append(total)
        traj["best"].append(list(best))
        traj["measured"].append(picked)
    return traj
