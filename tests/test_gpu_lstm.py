"""GPU parity of the NEXT-4 LSTM backbone (R49; "the self-attention or
LSTM module") through the C-ABI against the fp64 oracle (oracle/model.py
lstm_forward / lstm_backward, itself pinned to torch.nn.LSTM): scores and
every gradient within 1e-5 (fp32 SIMT) / 1e-2 (bf16 context: bf16x3 tcgen05
GEMMs for the input projection, every recurrent step and the weight
gradients), norm-wise per tensor (R25); batch invariance of the recurrent
scoring path; one Adam step."""
import numpy as np
import pytest
import torch

from oracle import model as OM
from oracle import rank_loss as OLR
from oracle.optim import AdamState, adam_step

from helpers import (encoded_batch, fit_scales, flat_params, grad_mismatches, oracle_cfg, product_cfg, rel_err,
                     token_table)
from test_gpu_parity import min_rel_gap, train_inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tp():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_2211_03578_b200 as tp
    tp._lib.load()
    return tp


@pytest.fixture(scope="module")
def tokscale():
    tokens = token_table()
    return tokens, fit_scales(tokens)


def lstm_cfg(**kw):
    c = oracle_cfg(**kw)
    c.backbone = "lstm"
    return c


@pytest.mark.parametrize("precision,tol,kw", [
    ("fp32", 1e-5, dict(hidden=64, up=(32, 64), head_dim=32)),
    ("fp32", 1e-5, dict(hidden=64, up=(32, 64), head_dim=32, n_attn=2, n_tasks=2)),
    ("bf16", 1e-2, dict()),                       # paper widths, 1 LSTM layer
    ("bf16", 1e-2, dict(n_attn=2)),
])
def test_lstm_forward_parity(tp, tokscale, precision, tol, kw):
    tokens, scale = tokscale
    ocfg = lstm_cfg(**kw)
    flat = flat_params(ocfg, seed=51)
    _, X = encoded_batch(53, 263, tokens, scale)
    ref = OM.forward(ocfg, OM.unflatten(ocfg, flat), X)
    m = tp.TLP(product_cfg(ocfg, precision))
    assert m.num_params == OM.n_params(ocfg)
    m.set_params(flat.astype(np.float32))
    s = m.score(torch.from_numpy(X).cuda())
    m.sync()
    assert rel_err(s.cpu().numpy(), ref) <= tol


def test_lstm_scoring_batch_invariance(tp, tokscale):
    """A candidate's score does not depend on the batch it is scored in
    (chunks of 8,192 and the GEMM tiling never mix candidates)."""
    tokens, scale = tokscale
    ocfg = lstm_cfg(hidden=64, up=(32, 64), head_dim=32)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat_params(ocfg, seed=3).astype(np.float32))
    _, X = encoded_batch(5, 8200, tokens, scale)
    Xd = torch.from_numpy(X).cuda()
    full = m.score(Xd).cpu().numpy()
    part = m.score(Xd[8191:8200].contiguous()).cpu().numpy()
    assert np.array_equal(full[8191:8200].view(np.uint32), part.view(np.uint32))


@pytest.mark.parametrize("precision,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_lstm_grads_parity(tp, tokscale, precision, tol):
    tokens, scale = tokscale
    ocfg = lstm_cfg(hidden=64, up=(32, 64), head_dim=32, n_attn=1)
    X, y, off = train_inputs(tokens, scale, 1)
    for seed in range(60, 120):  # within-group score gaps > 2e-4 (R26): ranks decided identically
        flat = flat_params(ocfg, seed=seed)
        p = OM.unflatten(ocfg, flat)
        s_ref, acts = OM.forward(ocfg, p, X, save=True)
        if min_rel_gap(s_ref, off) > 2e-4:
            break
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    m = tp.TLP(product_cfg(ocfg, precision))
    m.set_params(flat.astype(np.float32))
    loss = m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    assert abs(float(loss.cpu()) - loss_ref) <= tol * abs(loss_ref)
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, tol)
    assert not bad, bad


def test_lstm_grads_parity_two_layers_mtl(tp, tokscale):
    tokens, scale = tokscale
    ocfg = lstm_cfg(hidden=32, up=(16, 32), head_dim=16, n_attn=2, n_tasks=2, heads=4)
    X, y, off = train_inputs(tokens, scale, 2, sizes=(8, 6, 9, 7, 10, 8))
    for seed in range(60, 160):
        flat = flat_params(ocfg, seed=seed)
        p = OM.unflatten(ocfg, flat)
        s_ref, acts = OM.forward(ocfg, p, X, save=True)
        if min_rel_gap(s_ref, off) > 2e-4:
            break
    loss_ref, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads_ref = OM.backward(ocfg, p, acts, g)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat.astype(np.float32))
    m.compute_grads(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    got = OM.unflatten(ocfg, m.get_grads().astype(np.float64))
    bad = grad_mismatches(ocfg, p, acts, g, got, grads_ref, 1e-5)
    assert not bad, bad


def test_lstm_train_step_adam(tp, tokscale):
    """One tlp_train_step = the oracle's gradient followed by its Adam step (R23)."""
    tokens, scale = tokscale
    ocfg = lstm_cfg(hidden=64, up=(32, 64), head_dim=32)
    X, y, off = train_inputs(tokens, scale, 1)
    for seed in range(60, 120):
        flat = flat_params(ocfg, seed=seed)
        p = OM.unflatten(ocfg, flat)
        s_ref, acts = OM.forward(ocfg, p, X, save=True)
        if min_rel_gap(s_ref, off) > 2e-4:
            break
    _, g = OLR.mtl_lambdarank(s_ref, y.astype(np.float64), off)
    grads = OM.flatten(ocfg, OM.backward(ocfg, p, acts, g))
    st = AdamState.zeros(flat.size)
    want = adam_step(flat, grads, st)
    m = tp.TLP(product_cfg(ocfg, "fp32"))
    m.set_params(flat.astype(np.float32))
    m.train_step(torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda(), off)
    m.sync()
    got = m.get_params().astype(np.float64)
    # Adam moves each weight by ~lr; compare the update itself, per tensor
    upd_got = OM.unflatten(ocfg, got - flat)
    upd_ref = OM.unflatten(ocfg, want - flat)
    for name, _ in OM.param_shapes(ocfg):
        if name.startswith("lstm"):
            assert rel_err(upd_got[name], upd_ref[name]) <= 1e-3, name
