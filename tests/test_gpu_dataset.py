"""GPU parity of the NEXT-2 dataset scans (tlp_dedup, tlp_topk_score) against
oracle/dataset.py on the same seeded inputs: classes, kept samples, max labels
and counts bit-exact; the top-k score within 1e-12 (fp64 sums in another
order)."""
import numpy as np
import pytest
import torch

import synth
from oracle import dataset as OD

from helpers import encoded_batch, fit_scales, token_table

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03578_b200 as tp
    tp._lib.load()
    return tp


@pytest.fixture(scope="module")
def store():
    """Encoded synthetic candidates (TenSet-shaped sequences) with planted
    duplicates: within groups, across groups, chains of several copies, and a
    one-ulp near-duplicate that must stay distinct."""
    tokens = token_table()
    scale = fit_scales(tokens)
    _, X = encoded_batch(71, 3000, tokens, scale)
    rng = np.random.default_rng(7)
    src = rng.integers(0, 3000, 120)
    dst = rng.integers(0, 3000, 120)
    for d, s in zip(dst, src):
        X[d] = X[s]
    X[11] = X[10]
    X[11, 0, 0] = np.nextafter(X[11, 0, 0], np.float32(2))
    return X


def _groups(n, sizes):
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    assert off[-1] == n
    return off


@pytest.mark.parametrize("sizes", [(3000,), (500, 0, 1, 1499, 1000), (7,) * 428 + (4,)])
def test_dedup_parity(tp, store, sizes):
    X = store
    off = _groups(len(X), sizes)
    labels = np.random.default_rng(3).uniform(0.05, 1.0, len(X)).astype(np.float32)
    keep_ref, lab_ref, n_ref = OD.dedup_labels(X, off, labels)
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    keep, lab, n = m.dedup(torch.from_numpy(X).cuda(), off, torch.from_numpy(labels).cuda())
    m.sync()
    assert n == n_ref
    assert np.array_equal(keep.cpu().numpy().astype(bool), keep_ref)
    assert np.array_equal(lab.cpu().numpy().view(np.uint32), lab_ref.view(np.uint32))


def test_duplicate_rate_full_size(tp):
    """C2-size store (409,600 encoded candidates) with 1% planted duplicates:
    the duplicate rate equals the oracle's exactly."""
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    tokens = token_table()
    m.set_token_table(sorted(tokens, key=tokens.get))
    m.set_norm_scales(fit_scales(tokens))
    N = 409600
    X = m.encode(tp.DeviceBatch.from_packed(synth.generate(1000, N)))
    rng = np.random.default_rng(11)
    src = torch.from_numpy(rng.integers(0, N, N // 100)).cuda()
    dst = torch.from_numpy(rng.integers(0, N, N // 100)).cuda()
    X[dst] = X[src]
    keep, _, n = m.dedup(X, [0, N])
    m.sync()
    rate_ref, n_ref = OD.duplicate_rate(X.cpu().numpy())
    assert n == n_ref and 1.0 - n / N == pytest.approx(rate_ref, rel=1e-12)
    assert int(keep.sum().item()) == n


def test_dedup_errors(tp, store):
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    X = torch.from_numpy(store[:10].copy()).cuda()
    with pytest.raises(tp.TLPError) as e:
        m.dedup(X, [0, 4, 9])
    assert e.value.code == "ERR_SHAPE"
    bad = torch.ones(10, device="cuda")
    bad[3] = float("nan")
    m.dedup(X, [0, 10], bad)
    with pytest.raises(tp.TLPError) as e:
        m.sync()
    assert e.value.code == "ERR_NONFINITE"


@pytest.mark.parametrize("k", [1, 5, 64])
def test_topk_score_parity(tp, k):
    rng = np.random.default_rng(20 + k)
    sizes = synth.group_sizes(5, 40, lo=24, hi=4000, mean=1500.0)
    sizes[3] = 0
    sizes[7] = 1
    off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    N = int(off[-1])
    lat = rng.lognormal(0.0, 0.7, N).astype(np.float32)
    # scores quantised so ties occur: tie-breaking by index matters
    s = np.round(rng.normal(size=N) * 8).astype(np.float32) / 8
    w = rng.integers(1, 6, len(sizes)).astype(np.float64)
    ref = OD.topk_score(s, lat.astype(np.float64), off, w, k)
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    got = m.topk_score(torch.from_numpy(s).cuda(), torch.from_numpy(lat).cuda(), off, w, k)
    assert got == pytest.approx(ref, rel=1e-12)
    assert 0.0 < got <= 1.0


def test_topk_score_spec_example(tp):
    """S:450-452 worked example through the GPU path."""
    m = tp.TLP(tp.TLPConfig(precision="bf16"))
    lat = torch.tensor([2.0, 4.0, 8.0], device="cuda")
    s = torch.tensor([0.1, 0.9, 0.5], device="cuda")
    assert m.topk_score(s, lat, [0, 3], [2.0], 1) == 0.5
    assert m.topk_score(torch.tensor([0.8, 0.9, 0.1], device="cuda"), lat, [0, 3], [2.0], 2) == 1.0
