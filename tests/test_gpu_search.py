"""GPU parity of the NEXT-1 tuning round (k_search.cu through the C-ABI)
against oracle/search.py on the same seeded search spaces (synth templates):
initial genes, children, duplicate dropping and materialised primitive
sequences bit-exact; a whole device round (fp32 context) equal to the oracle's
round driven by the oracle's fp64 forward -- survivors bit-exact, their scores
within 1e-5 -- when the oracle's scores separate every pair of distinct
programs by more than twice the tolerance (checked by brute force, so a rank
can only be decided one way); tuner invariants on the device loop; a
paper-shape bf16 round self-consistent with tlp_score."""
import numpy as np
import pytest
import torch

import synth
import oracle
from oracle import model as OM
from oracle import search as OS

from helpers import fit_scales, flat_params, oracle_cfg, product_cfg, rel_err, token_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03578_b200 as tp
    tp._lib.load()
    return tp


@pytest.fixture(scope="module")
def env(tp):
    tokens = token_table()
    scale = fit_scales(tokens)
    ocfg = oracle_cfg(hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, 5)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    m.set_params(flat.astype(np.float32))
    return dict(tokens=tokens, scale=scale, ocfg=ocfg, params=OM.unflatten(ocfg, flat), m=m)


def _space(seed, S):
    ts = [synth.make_template(seed, s) for s in range(S)]
    return ts, synth.pack_space(ts)


def _rows(genes_dev, S, n, ts):
    g = genes_dev.cpu().numpy().reshape(S, n, -1)
    return [g[s][:, :ts[s].G].astype(np.int64) for s in range(S)], g


@pytest.mark.parametrize("n", [1, 37, 256])
def test_init_bit_exact(env, n):
    m = env["m"]
    ts, sp = _space(11, 5)
    m.ga_set_space(sp)
    got, full = _rows(m.ga_init(n, seed=2**64 - 5, rnd=3), 5, n, ts)
    for s in range(5):
        assert np.array_equal(got[s], OS.init_genes(ts[s].dom_sizes(), n, 2**64 - 5, s, 3))
        assert (full[s][:, ts[s].G:] == 0).all()


@pytest.mark.parametrize("p_cross,p_mut", [(0.0, 0.0), (0.5, 0.2), (1.0, 1.0)])
def test_evolve_bit_exact(env, p_cross, p_mut):
    m = env["m"]
    S, n_pop, n_child = 4, 24, 300
    ts, sp = _space(13, S)
    m.ga_set_space(sp)
    G = m.ga_G
    rng = np.random.default_rng(1)
    pop = np.zeros((S, n_pop, G), np.uint8)
    sc = np.zeros((S, n_pop), np.float32)
    n_eff = [n_pop, 1, 7, 20]
    for s in range(S):
        pop[s, :, :ts[s].G] = OS.init_genes(ts[s].dom_sizes(), n_pop, 9, s, 0)
        v = np.sort(rng.normal(size=n_pop).astype(np.float32))[::-1].copy()
        v[n_eff[s]:] = -np.inf   # duplicate survivors at the tail
        sc[s] = v
    ch = m.ga_evolve(torch.from_numpy(pop.reshape(S * n_pop, G)).cuda(), torch.from_numpy(sc.ravel()).cuda(),
                     n_pop, n_child, p_cross, p_mut, seed=77, rnd=4, it=2)
    got, full = _rows(ch, S, n_child, ts)
    for s in range(S):
        want = OS.evolve(pop[s, :, :ts[s].G].astype(np.int64), ts[s].dom_sizes(), ts[s].knob_groups(),
                         n_child, p_cross, p_mut, 77, s, 4, 2, n_eff[s])
        assert np.array_equal(got[s], want)
        assert (full[s][:, ts[s].G:] == 0).all()


def test_drop_duplicates_bit_exact(env):
    m = env["m"]
    S, n = 3, 3000
    ts, sp = _space(17, S)
    m.ga_set_space(sp)
    G = m.ga_G
    g = np.zeros((S, n, G), np.uint8)
    rng = np.random.default_rng(4)
    for s in range(S):
        g[s, :, :ts[s].G] = OS.init_genes(ts[s].dom_sizes(), n, 5, s, 0)
        for d, src in zip(rng.integers(0, n, 400), rng.integers(0, n, 400)):
            g[s, d] = g[s, src]
    g[0, 5:9] = g[0, 4]   # a chain of copies
    sc = rng.normal(size=S * n).astype(np.float32)
    out = m.ga_drop_duplicates(torch.from_numpy(g.reshape(S * n, G)).cuda(), n,
                               torch.from_numpy(sc).cuda()).cpu().numpy()
    for s in range(S):
        want = OS.drop_duplicates(g[s].astype(np.int64), sc[s * n:(s + 1) * n]).astype(np.float32)
        assert np.array_equal(out[s * n:(s + 1) * n], want)
    assert np.isneginf(out).sum() > 1000


def test_materialize_and_encode_bit_exact(env):
    m, tokens, scale = env["m"], env["tokens"], env["scale"]
    S, n = 6, 40
    ts, sp = _space(19, S)
    m.ga_set_space(sp)
    genes = m.ga_init(n, seed=3, rnd=0)
    b = m.ga_materialize(genes, n)
    rows, _ = _rows(genes, S, n, ts)
    host = synth.PackedBatch(b.seq_off.cpu().numpy()[:b.N + 1], b.prim_type.cpu().numpy()[:b.P],
                             b.arg_off.cpu().numpy()[:b.P + 1], b.arg_kind.cpu().numpy()[:b.A],
                             b.arg_num.cpu().numpy()[:b.A], b.arg_name.cpu().numpy()[:b.A],
                             list(sp.tmpl.strings))
    want = [seq for s in range(S) for seq in OS.materialize(ts[s], rows[s])]
    got = host.to_lists()
    assert got == [[(t, list(a)) for t, a in seq] for seq in want]
    X = m.encode(b).cpu().numpy()
    Xo = oracle.encode(want, tokens, scale)
    assert np.array_equal(X.view(np.uint32), Xo.view(np.uint32))


ROUND_DOMAINS = ((3, 3, 3), (2, 4, 3), (5, 5), (2, 3), (4, 4, 2))


def test_round_matches_oracle(tp):
    """Small search spaces whose every program the oracle scores (brute
    force) with pairwise gaps > 2e-5 of the largest |score| (argument columns
    scaled by 4 so the split factors move the score), so each ranking decision
    of the round is unique: two scores each within the 1e-5 fp32 tolerance of
    their exact values cannot swap across a gap wider than twice it.  The (2, 3) space has fewer
    distinct programs than n_pop: duplicate survivors (-inf) and the n_eff <
    n_pop parent draw are exercised."""
    import itertools
    tokens = token_table()
    scale = np.ones(22, np.float32)
    scale[11:] = 4.0
    ocfg = oracle_cfg(hidden=64, up=(32, 64), head_dim=32)
    flat = flat_params(ocfg, 138)
    params = OM.unflatten(ocfg, flat)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    m.set_params(flat.astype(np.float32))
    ts = [synth.small_template(d) for d in ROUND_DOMAINS]
    S = len(ts)
    cost = lambda s, g: OM.forward(ocfg, params, oracle.encode(OS.materialize(ts[s], g), tokens, scale))[:, 0]  # noqa: E731
    vmax = []
    for s, d in enumerate(ROUND_DOMAINS):
        v = np.sort(cost(s, np.array(list(itertools.product(*[range(x) for x in d])))))
        vmax.append(np.abs(v).max())
        assert np.diff(v).min() > 2e-5 * vmax[s]
    m.ga_set_space(synth.pack_space(ts))
    n_pop, n_child, iters = 8, 24, 3
    want = [OS.search_round(ts[s], s, cost, 31, 2, n_pop, n_child, iters, 0.5, 0.3) for s in range(S)]
    genes, scores = m.ga_round(n_pop, n_child, iters, 0.5, 0.3, seed=31, rnd=2)
    m.sync()
    got, _ = _rows(genes, S, n_pop, ts)
    sc = scores.cpu().numpy().reshape(S, n_pop)
    assert not np.isfinite(want[3][1]).all()  # the 6-point space has duplicate survivors
    for s in range(S):
        fin = np.isfinite(want[s][1])
        assert np.array_equal(np.isfinite(sc[s]), fin)
        assert np.array_equal(got[s], want[s][0])  # -inf rows too: same pool, same index order
        # R25 norm-wise over the batch the round scored: the subgraph's programs
        assert np.abs(sc[s][fin] - want[s][1][fin]).max() <= 1e-5 * vmax[s]
        # duplicate survivors: whichever rows, each equals an earlier survivor
        for r in np.nonzero(~fin)[0]:
            assert any(np.array_equal(got[s][r], got[s][q]) for q in range(r))


def test_device_tuner_invariants(env, tp):
    from paper_2211_03578_b200.search import Tuner
    m = env["m"]
    S = 4
    ts, sp = _space(29, S)
    m.ga_set_space(sp)
    tuner = Tuner(m, S, [t.G for t in ts], n_pop=32, n_child=96, iters=2, seed=5)
    traj = tuner.tune(3, lambda s, g: float(synth.template_latency(ts[s], g, 29, s)[0]), per_round=6)
    assert traj.measurements == [24, 48, 72]
    b = np.array(traj.best)
    assert (np.diff(b, axis=0) <= 0).all()
    keys = [(s, k) for r in traj.measured for (s, k, _) in r]
    assert len(keys) == len(set(keys))
    for s, k, lat in (x for r in traj.measured for x in r):
        assert all(0 <= k[j] < ts[s].dom_sizes()[j] for j in range(ts[s].G))
        assert lat == float(synth.template_latency(ts[s], np.array(k), 29, s)[0])


def test_round_argument_errors(env, tp):
    m = env["m"]
    ts, sp = _space(31, 2)
    m.ga_set_space(sp)
    with pytest.raises(tp.TLPError):
        m.ga_round(0, 8, 1, 0.5, 0.2, seed=1, rnd=0)
    with pytest.raises(tp.TLPError):
        m.ga_round(8, 8, 1, 1.5, 0.2, seed=1, rnd=0)
    bad = synth.pack_space(ts)
    bad.dom_name[0] = 0 if bad.dom_name[0] < 0 else -1   # kind mismatch with the skeleton
    with pytest.raises(tp.TLPError):
        m.ga_set_space(bad)


def test_paper_shape_bf16_round(tp):
    """The bench configuration's kernels (bf16 fused forward, paper shape) on a
    small round: every survivor's score equals tlp_score of its materialised
    program (batch invariance, R34) bit for bit, and the oracle's fp64 score
    within 1e-2 (R25); survivors are distinct and in rank order."""
    tokens = token_table()
    scale = fit_scales(tokens)
    ocfg = oracle_cfg(n_attn=2)
    flat = flat_params(ocfg, 3)
    m = tp.TLP(product_cfg(ocfg, "bf16"))
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(scale)
    m.set_params(flat.astype(np.float32))
    S, n_pop = 4, 64
    ts, sp = _space(37, S)
    m.ga_set_space(sp)
    genes, scores = m.ga_round(n_pop, 192, 2, 0.5, 0.2, seed=9, rnd=0)
    b = m.ga_materialize(genes, n_pop)
    again = m.score(m.encode(b)).cpu().numpy()[:, 0]
    sc = scores.cpu().numpy()
    assert np.isfinite(sc).all()
    assert np.array_equal(again.view(np.uint32), sc.view(np.uint32))
    rows, _ = _rows(genes, S, n_pop, ts)
    params = OM.unflatten(ocfg, flat)
    for s in range(S):
        assert len({tuple(r) for r in rows[s]}) == n_pop
        v = sc[s * n_pop:(s + 1) * n_pop]
        assert (np.diff(v) <= 0).all()
        ref = OM.forward(ocfg, params, oracle.encode(OS.materialize(ts[s], rows[s]), tokens, scale))[:, 0]
        assert rel_err(v, ref) <= 1e-2


def test_sharded_device_rounds_equal_the_full_round(env, tp):
    """Multi-GPU protocol on one GPU: two contexts, each with a contiguous
    block of the subgraphs (dist.shard_subgraphs, id_base = its first global
    id), produce exactly the full space's survivors (no exchange step)."""
    from paper_2211_03578_b200 import dist as D
    m = env["m"]
    S, n_pop = 5, 16
    ts = [synth.make_template(43, s) for s in range(S)]
    m.ga_set_space(synth.pack_space(ts))
    g_full, s_full = m.ga_round(n_pop, 48, 2, 0.5, 0.2, seed=3, rnd=1)
    g_full = g_full.cpu().numpy().reshape(S, n_pop, -1)
    s_full = s_full.cpu().numpy().reshape(S, n_pop)
    for rank in range(2):
        lo, hi = D.shard_subgraphs(S, 2, rank)
        m.ga_set_space(synth.pack_space(ts[lo:hi]), id_base=lo)
        g, sc = m.ga_round(n_pop, 48, 2, 0.5, 0.2, seed=3, rnd=1)
        g = g.cpu().numpy().reshape(hi - lo, n_pop, -1)
        sc = sc.cpu().numpy().reshape(hi - lo, n_pop)
        for j, s in enumerate(range(lo, hi)):
            K = ts[s].G
            assert np.array_equal(g[j][:, :K], g_full[s][:, :K])
            assert np.array_equal(sc[j].view(np.uint32), s_full[s].view(np.uint32))
