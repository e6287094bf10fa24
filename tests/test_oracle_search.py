"""Pins of oracle/search.py (O11, NEXT-1: the synthetic Ansor-style tuning
round; readings R44-R48).

What fixes each part from outside the oracle:
  * the Philox4x64-10 generator equals numpy's ``np.random.Philox`` (a
    library routine) word for word;
  * fitness-proportional selection is checked by enumerating every u in
    [0, F): rank r is chosen exactly n - r times (the definition of
    linear-ranking roulette), and empirically over Philox draws;
  * the genetic operators against SPEC S:515-521's properties: rates 0 ->
    offspring are parents; crossover only at primitive boundaries; mutation is
    one step inside the domain; validity over 10^4 children;
  * the round / tuner against SPEC S:524-533: a cost model equal to the
    hardware reaches the brute-force optimum of a 64-point template in one
    round of 10 measurements; a constant cost model IS random search (the
    measured programs are exactly the first unseen uniform draws); budget and
    monotonicity invariants.
"""
import itertools

import numpy as np
import pytest

import synth
from oracle import search as O


# ------------------------------------------------------------------ R44 RNG
@pytest.mark.parametrize("ctr,key", [((0, 0, 0, 0), (7, 9)), ((5, 1, 2, 3), (2**64 - 1, 0x544C50)),
                                     ((2**63, 2**64 - 2, 17, 1 << 40), (123456789, 42))])
def test_philox_matches_numpy(ctr, key):
    # numpy's Philox increments the 256-bit counter before each block
    g = np.random.Philox(counter=np.array(ctr, np.uint64), key=np.array(key, np.uint64))
    got = [int(v) for v in g.random_raw(8)]
    c = sum(int(v) << (64 * i) for i, v in enumerate(ctr))
    blocks = []
    for b in (1, 2):
        cc = (c + b) % (1 << 256)
        blocks += O.philox4x64_10([(cc >> (64 * i)) & O.MASK64 for i in range(4)], key)
    assert got == blocks


def test_uniform_index_and_bernoulli():
    rng = np.random.default_rng(0)
    ws = [int(v) for v in rng.integers(0, 2**63, 4000, dtype=np.int64)] + [0, O.MASK64]
    for w in ws:
        assert 0 <= O.uniform_index(w, 7) < 7
        assert not O.bernoulli(w, 0.0)
        assert O.bernoulli(w, 1.0)
    assert O.uniform_index(O.MASK64, 7) == 6 and O.uniform_index(0, 7) == 0
    # p = 0.25: threshold 2^51 on the top 53 bits
    assert O.bernoulli((1 << 62) - 1, 0.25) and not O.bernoulli(1 << 62, 0.25)


# ------------------------------------------------------------------ R46 selection
@pytest.mark.parametrize("n", list(range(1, 13)) + [40])
def test_select_rank_is_fitness_proportional_exactly(n):
    F = n * (n + 1) // 2
    counts = np.zeros(n, np.int64)
    for u in range(F):
        counts[O.select_rank(u, n)] += 1
    assert counts.tolist() == [n - r for r in range(n)]


def test_select_rank_frequencies_over_philox():
    n, draws = 8, 20000
    F = n * (n + 1) // 2
    counts = np.zeros(n)
    for c in range(draws):
        counts[O.select_rank(O.uniform_index(O.word(3, c, 0, 0, 1, O.STREAM_SEL, 0), F), n)] += 1
    expect = draws * (n - np.arange(n)) / F
    chi2 = ((counts - expect) ** 2 / expect).sum()
    assert chi2 < 24.3  # 7 dof, p = 0.001


# ------------------------------------------------------------------ R47 operators
def _pop(tmpl, n, seed):
    return O.init_genes(tmpl.dom_sizes(), n, seed, 0, 0)


def test_rates_zero_offspring_are_parents():
    tmpl = synth.make_template(2, 5)
    pop = _pop(tmpl, 16, 1)
    ch = O.evolve(pop, tmpl.dom_sizes(), tmpl.knob_groups(), 200, 0.0, 0.0, 9, 0, 0, 1)
    rows = {tuple(r) for r in pop}
    assert all(tuple(r) in rows for r in ch)


def test_crossover_at_primitive_boundaries():
    tmpl = synth.make_template(4, 1)
    D, grp = tmpl.dom_sizes(), tmpl.knob_groups()
    assert grp.max() >= 2
    pop = _pop(tmpl, 6, 5)
    ch = O.evolve(pop, D, grp, 300, 1.0, 0.0, 11, 0, 0, 1)
    n_groups = int(grp.max()) + 1
    crossed = 0
    for r in ch:
        ok = False
        for a, b in itertools.product(range(len(pop)), repeat=2):
            for cut in range(1, n_groups):
                want = np.where(grp >= cut, pop[b], pop[a])
                if np.array_equal(want, r):
                    ok = True
                    crossed += int(not np.array_equal(pop[a], r))
                    break
            if ok:
                break
        assert ok
    assert crossed > 100


def test_mutation_is_one_step_inside_the_domain():
    tmpl = synth.small_template((2, 3, 7, 7, 1))
    D = tmpl.dom_sizes()
    pop = _pop(tmpl, 5, 2)
    ch = O.evolve(pop, D, tmpl.knob_groups(), 200, 0.0, 1.0, 4, 0, 0, 1)
    for r in ch:
        diffs = [np.abs(r - p) for p in pop]
        assert any(np.array_equal(d, (D >= 2).astype(np.int64)) for d in diffs)
        assert (r >= 0).all() and (r < D).all()


def test_offspring_validity_sweep_and_reproducibility():
    total = 0
    for k in range(20):
        tmpl = synth.make_template(100 + k, k)
        D, grp = tmpl.dom_sizes(), tmpl.knob_groups()
        pop = _pop(tmpl, 12, k)
        ch = O.evolve(pop, D, grp, 500, 0.6, 0.1, k, k, 3, 2)
        assert ((ch >= 0) & (ch < D)).all()
        total += len(ch)
        again = O.evolve(pop, D, grp, 500, 0.6, 0.1, k, k, 3, 2)
        assert np.array_equal(ch, again)
        other = O.evolve(pop, D, grp, 500, 0.6, 0.1, k + 1, k, 3, 2)
        assert not np.array_equal(ch, other)
    assert total == 10 ** 4


def test_init_genes_uniform_and_valid():
    tmpl = synth.small_template((7, 3))
    g = O.init_genes(tmpl.dom_sizes(), 7000, 1, 0, 0)
    assert ((g >= 0) & (g < tmpl.dom_sizes())).all()
    c0 = np.bincount(g[:, 0], minlength=7)
    assert ((c0 - 1000) ** 2 / 1000).sum() < 22.5  # 6 dof, p = 0.001


def test_materialize_places_domain_values():
    tmpl = synth.small_template((4, 4, 4))
    seq = O.materialize(tmpl, np.array([[1, 2, 3]]))[0]
    assert [seq[p][1][3] for p in (1, 2, 3)] == [2.0, 4.0, 8.0]
    assert seq[0] == tmpl.prims[0] and len(seq) == len(tmpl.prims)
    t2 = synth.make_template(7, 2)
    genes = _pop(t2, 3, 0)
    for row, s in zip(genes, O.materialize(t2, genes)):
        for g in range(t2.G):
            assert s[t2.knob_prim[g]][1][t2.knob_arg[g]] == t2.domains[g][row[g]]


# ------------------------------------------------------------------ R48 round / tuner
def test_latency_closed_forms():
    tmpl = synth.make_template(1, 0)
    base, w, v = synth.template_weights(1, 0, tmpl.G)
    assert synth.template_latency(tmpl, np.zeros(tmpl.G, np.int64), 1, 0)[0] == pytest.approx(base, rel=1e-15)
    top = tmpl.dom_sizes() - 1
    assert synth.template_latency(tmpl, top, 1, 0)[0] == pytest.approx(
        base * np.exp(w.sum() + v.sum()), rel=1e-12)


def test_cheating_model_finds_the_brute_force_optimum():
    tmpl = synth.small_template((4, 4, 4))
    lat = lambda s, g: synth.template_latency(tmpl, g, 5, s)
    space = np.array(list(itertools.product(range(4), repeat=3)))
    opt = lat(0, space).min()
    traj = O.tune([tmpl], lambda s, g: -lat(s, g), lambda s, g: lat(s, g)[0], rounds=1,
                  measure=10, seed=1, n_pop=64, n_child=64, iters=2, p_cross=0.5, p_mut=0.2)
    assert traj["measurements"] == [10]
    assert traj["best"][0][0] == opt


def test_constant_model_is_random_search():
    tmpl = synth.small_template((4, 4, 4))
    lat = lambda s, g: float(synth.template_latency(tmpl, g, 2, s)[0])
    kw = dict(measure=5, seed=8, n_pop=16, n_child=16, iters=3, p_cross=0.5, p_mut=0.3)
    traj = O.tune([tmpl], lambda s, g: np.zeros(len(g)), lat, rounds=4, **kw)
    # random search: each round draw n_pop + n_child uniform programs, keep the
    # first n_pop distinct ones, measure the first unseen of those
    seen = []
    for rnd in range(4):
        g = []
        for row in O.init_genes(tmpl.dom_sizes(), 32, 8, 0, rnd):
            if len(g) < 16 and not any(np.array_equal(row, x) for x in g):
                g.append(row)
        got = 0
        for row in g:
            key = tuple(int(v) for v in row)
            if got < 5 and key not in seen:
                seen.append(key); got += 1
    measured = [k for r in traj["measured"] for (_, k, _) in r]
    assert measured == seen


def test_tuner_invariants():
    ts = [synth.make_template(3, s) for s in range(2)]
    lat = lambda s, g: float(synth.template_latency(ts[s], g, 3, s)[0])
    cost = lambda s, g: -np.log(synth.template_latency(ts[s], g, 3, s)) + 0.3 * np.sin(g.sum(1))
    traj = O.tune(ts, cost, lat, rounds=3, measure=4, seed=2, n_pop=16, n_child=24, iters=2,
                  p_cross=0.5, p_mut=0.2)
    assert traj["measurements"] == [8, 16, 24]
    b = np.array(traj["best"])
    assert (np.diff(b, axis=0) <= 0).all()
    keys = [(s, k) for r in traj["measured"] for (s, k, _) in r]
    assert len(keys) == len(set(keys))
    assert O.tune(ts, cost, lat, rounds=0, measure=4, seed=2, n_pop=16, n_child=24, iters=2,
                  p_cross=0.5, p_mut=0.2)["measurements"] == []
