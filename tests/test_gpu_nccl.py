"""The NCCL code paths of the library on ONE GPU (gpurun grants one): a 1-rank
communicator (tlp_set_comm with world 1 and an id) runs the real collectives --
the per-task loss-count allreduce (C-0), the gradient allreduce (C-1) and the
top-k allgather + merge (C-2) of SURVEY §8(e) -- which for one rank must leave
every result bit-identical to the communicator-free path.  The multi-rank
protocol itself is pinned on CPU (tests/test_dist_gloo.py, oracle O8)."""
import os
import socket

import numpy as np
import pytest
import torch

from helpers import encoded_batch, flat_params, oracle_cfg, product_cfg, token_table, fit_scales

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.distributed as dist
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


@pytest.mark.parametrize("precision", ["fp32", "bf16"])
def test_one_rank_collectives_equal_local_path(nccl_group, precision):
    import paper_2211_03578_b200 as tp
    import synth
    import oracle
    tokens = token_table()
    scale = fit_scales(tokens)
    ocfg = oracle_cfg(n_attn=1, n_tasks=2) if precision == "bf16" else \
        oracle_cfg(hidden=64, up=(32, 64), head_dim=32, n_tasks=2)
    flat = flat_params(ocfg, seed=31).astype(np.float32)
    b, X = encoded_batch(41, 600, tokens, scale)
    off = np.array([0, 150, 151, 400, 600], np.int64)
    lat = synth.latencies(b, off, 2)
    y = np.stack([oracle.normalize_labels(lat, off)] * 2, axis=1).astype(np.float32)
    y[::3, 0] = np.nan  # MTL: task 0 labels on a subset
    Xd, yd = torch.from_numpy(X).cuda(), torch.from_numpy(y).cuda()
    models = []
    for with_comm in (False, True):
        m = tp.TLP(product_cfg(ocfg, precision))
        m.set_params(flat)
        if with_comm:
            m.init_comm()
        losses = [float(m.train_step(Xd, yd, off).cpu()) for _ in range(2)]
        s = m.score(Xd)
        idx, val = m.topk(s, off, 8)
        m.sync()
        models.append((losses, m.get_params(), idx.cpu().numpy(), val.cpu().numpy()))
    (l0, p0, i0, v0), (l1, p1, i1, v1) = models
    assert np.array_equal(np.float32(l0).view(np.uint32), np.float32(l1).view(np.uint32))
    assert np.array_equal(p0.view(np.uint32), p1.view(np.uint32))
    assert np.array_equal(i0, i1)
    assert np.array_equal(v0.view(np.uint32), v1.view(np.uint32))
