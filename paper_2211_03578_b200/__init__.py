"""B200-native hot path of TLP / MTL-TLP (arXiv 2211.03578).

Thin Python binding over libtlp.so (include/tlp.h): argument marshalling only.
Every step of the path -- tokenizer, network forward/backward, LambdaRank,
Adam, top-k, label normalisation -- runs in the sm_100a kernels of the
library.  PyTorch is used for device memory, streams and torch.distributed
rendezvous.  There is no CPU or eager fallback: if the library is missing the
import of any op raises.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

import numpy as np
import torch

from . import _lib
from ._lib import tlp_config, tlp_seq_batch

__all__ = ["TLPConfig", "TLP", "DeviceBatch", "TLPError", "paper_config", "tiny_config"]


class TLPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s (%d): %s" % (_lib.TLP_STATUS.get(status, "?"), status, msg))
        self.status = status
        self.code = _lib.TLP_STATUS.get(status, "?")


@dataclass
class TLPConfig:
    """Mirror of tlp_config.  Paper defaults: P:273; R11, R13, R23."""
    L: int = 25
    E: int = 22
    T: int = 11
    hidden: int = 256
    up_dims: Tuple[int, ...] = (128, 256)
    attn_heads: int = 8
    n_attn: int = 1
    n_res: int = 2
    head_dim: int = 128
    n_tasks: int = 1
    precision: str = "bf16"  # "bf16" (tcgen05 scoring) | "fp32" (SIMT, 1e-5 path)
    lr: float = 1e-3
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8
    loss: str = "lambdarank"  # "lambdarank" (R16, the paper's choice) | "mse" (NEXT-3)
    attn_mask: bool = False   # NEXT-3 / R42: mask padding keys (the paper: no mask, R8)
    pos_enc: bool = False     # NEXT-3 / R43: learned positional table (the paper: none, R9)
    backbone: str = "attn"    # NEXT-4 / R49: "attn" (the paper's choice) | "lstm"

    def param_shapes(self):
        """[(name, shape)] of the flat parameter vector in the library's R24 order
        (include/tlp.h tlp_set_params): upsample (W [in, out], b)...; the R43
        table; per attention layer Wq bq Wk bk Wv bv Wo bo (per LSTM layer Wih
        bih Whh bhh); per residual block Wa a Wb b; per task W1 c1 w2 c2."""
        out, d_in, H = [], self.E, self.hidden
        for i, d in enumerate(self.up_dims):
            out += [("up%d.W" % i, (d_in, d)), ("up%d.b" % i, (d,))]
            d_in = d
        if self.pos_enc:
            out.append(("pos", (self.L, H)))
        for l in range(self.n_attn):
            if self.backbone == "lstm":
                out += [("lstm%d.Wih" % l, (H, 4 * H)), ("lstm%d.bih" % l, (4 * H,)),
                        ("lstm%d.Whh" % l, (H, 4 * H)), ("lstm%d.bhh" % l, (4 * H,))]
            else:
                for nm in "qkvo":
                    out += [("attn%d.W%s" % (l, nm), (H, H)), ("attn%d.b%s" % (l, nm), (H,))]
        for r in range(self.n_res):
            out += [("res%d.Wa" % r, (H, H)), ("res%d.a" % r, (H,)), ("res%d.Wb" % r, (H, H)),
                    ("res%d.b" % r, (H,))]
        for t in range(self.n_tasks):
            out += [("head%d.W1" % t, (H, self.head_dim)), ("head%d.c1" % t, (self.head_dim,)),
                    ("head%d.w2" % t, (self.head_dim, 1)), ("head%d.c2" % t, (1,))]
        return out

    def to_c(self) -> tlp_config:
        c = tlp_config()
        c.L, c.E, c.T, c.hidden = self.L, self.E, self.T, self.hidden
        for i, d in enumerate(self.up_dims):
            c.up_dims[i] = d
        c.n_up = len(self.up_dims)
        c.attn_heads, c.n_attn, c.n_res = self.attn_heads, self.n_attn, self.n_res
        c.head_dim, c.n_tasks = self.head_dim, self.n_tasks
        c.precision = {"fp32": 0, "bf16": 1}[self.precision]
        c.lr, c.beta1, c.beta2, c.eps = self.lr, self.beta1, self.beta2, self.eps
        c.loss = {"lambdarank": 0, "mse": 1}[self.loss]
        c.attn_mask = 1 if self.attn_mask else 0
        c.pos_enc = 1 if self.pos_enc else 0
        c.backbone = {"attn": 0, "lstm": 1}[self.backbone]
        return c


def paper_config(**kw) -> TLPConfig:
    return TLPConfig(**kw)


def tiny_config(**kw) -> TLPConfig:
    """C1: hidden 64, upsample 22->32->64, head 64->32->1 (BASELINE configs[0])."""
    base = dict(hidden=64, up_dims=(32, 64), head_dim=32, precision="fp32")
    base.update(kw)
    return TLPConfig(**base)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream_ptr(stream, device: Optional[int] = None) -> Optional[int]:
    """The cudaStream_t of `stream`; None = the current stream OF `device` (the
    ctx's GPU), not of whatever device happens to be current."""
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream.cuda_stream


@dataclass
class DeviceBatch:
    """Packed abstract primitives on the device (tlp_seq_batch).  Built from any
    object exposing seq_off, prim_type, arg_off, arg_kind, arg_num, arg_name
    (numpy) and strings (list of str)."""
    seq_off: torch.Tensor
    prim_type: torch.Tensor
    arg_off: torch.Tensor
    arg_kind: torch.Tensor
    arg_num: torch.Tensor
    arg_name: torch.Tensor
    str_blob: torch.Tensor
    str_off: torch.Tensor
    N: int = 0
    P: int = 0
    A: int = 0
    U: int = 0

    @staticmethod
    def host_arrays(packed):
        enc = [s.encode("utf-8") for s in packed.strings]
        off = np.zeros(len(enc) + 1, np.int64)
        if enc:
            off[1:] = np.cumsum([len(e) for e in enc])
        blob = np.frombuffer(b"".join(enc), np.uint8).copy() if enc else np.zeros(1, np.uint8)
        return dict(seq_off=np.ascontiguousarray(packed.seq_off, np.int64),
                    prim_type=np.ascontiguousarray(packed.prim_type, np.uint8),
                    arg_off=np.ascontiguousarray(packed.arg_off, np.int64),
                    arg_kind=np.ascontiguousarray(packed.arg_kind, np.uint8),
                    arg_num=np.ascontiguousarray(packed.arg_num, np.float64),
                    arg_name=np.ascontiguousarray(packed.arg_name, np.int32),
                    str_blob=blob, str_off=off)

    @classmethod
    def from_packed(cls, packed, device="cuda", pin: bool = False) -> "DeviceBatch":
        arrs = cls.host_arrays(packed)
        ts = {}
        for k, v in arrs.items():
            t = torch.from_numpy(v if v.size else np.zeros(1, v.dtype))
            ts[k] = t.pin_memory() if pin else t.to(device)
        return cls(N=len(arrs["seq_off"]) - 1, P=len(arrs["arg_off"]) - 1,
                   A=int(arrs["arg_off"][-1]), U=len(arrs["str_off"]) - 1, **ts)

    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in
                   (self.seq_off, self.prim_type, self.arg_off, self.arg_kind, self.arg_num,
                    self.arg_name, self.str_blob, self.str_off))

    def to(self, device, non_blocking: bool = False) -> "DeviceBatch":
        f = lambda t: t.to(device, non_blocking=non_blocking)  # noqa: E731
        return DeviceBatch(f(self.seq_off), f(self.prim_type), f(self.arg_off), f(self.arg_kind),
                           f(self.arg_num), f(self.arg_name), f(self.str_blob), f(self.str_off),
                           self.N, self.P, self.A, self.U)

    def c_struct(self) -> tlp_seq_batch:
        b = tlp_seq_batch()
        b.seq_off, b.prim_type, b.arg_off = _ptr(self.seq_off), _ptr(self.prim_type), _ptr(self.arg_off)
        b.arg_kind, b.arg_num, b.arg_name = _ptr(self.arg_kind), _ptr(self.arg_num), _ptr(self.arg_name)
        b.str_blob, b.str_off = _ptr(self.str_blob), _ptr(self.str_off)
        b.P, b.A, b.U = self.P, self.A, self.U
        return b


class TLP:
    """One libtlp context on one GPU (single-threaded, include/tlp.h)."""

    def __init__(self, cfg: TLPConfig, device: int = 0):
        self.lib = _lib.load()
        self.cfg = cfg
        self.device = device
        torch.cuda.init()
        with torch.cuda.device(device):
            h = C.c_void_p()
            c = cfg.to_c()
            st = self.lib.tlp_create(C.byref(c), device, C.byref(h))
            if st != 0:
                raise TLPError(st, self.lib.tlp_last_error(None).decode())
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) is not None and getattr(self, "lib", None) is not None:
            self.lib.tlp_destroy(self.h)
            self.h = None

    def _check(self, st: int):
        if st != 0:
            raise TLPError(st, self.lib.tlp_last_error(self.h).decode())

    # --- state -------------------------------------------------------------
    @property
    def num_params(self) -> int:
        return int(self.lib.tlp_num_params(self.h))

    def set_token_table(self, names: Sequence[str]):
        enc = [s.encode("utf-8") for s in names]
        off = np.zeros(len(enc) + 1, np.int64)
        if enc:
            off[1:] = np.cumsum([len(e) for e in enc])
        blob = np.frombuffer(b"".join(enc) or b"\0", np.uint8).copy()
        self._check(self.lib.tlp_set_token_table(self.h, blob.ctypes.data, off.ctypes.data, len(enc)))

    def set_norm_scales(self, scale):
        s = np.ascontiguousarray(scale, np.float32)
        assert s.shape == (self.cfg.E,)
        self._check(self.lib.tlp_set_norm_scales(self.h, s.ctypes.data))

    def fit_token_table(self, packed):
        """tlp_fit_token_table (R1) from a host packed batch (anything
        DeviceBatch.host_arrays accepts, or a host DeviceBatch)."""
        hb = packed if isinstance(packed, DeviceBatch) else DeviceBatch.from_packed(packed, device="cpu")
        assert not hb.seq_off.is_cuda
        b = hb.c_struct()
        self._check(self.lib.tlp_fit_token_table(self.h, C.byref(b), hb.N))

    def fit_norm_scales(self, batch: "DeviceBatch", stream=None) -> np.ndarray:
        """tlp_fit_norm_scales (R3) from a device batch; returns the [E] scales."""
        out = np.zeros(self.cfg.E, np.float32)
        b = batch.c_struct()
        self._check(self.lib.tlp_fit_norm_scales(self.h, C.byref(b), batch.N, out.ctypes.data,
                                                 _stream_ptr(stream, self.device)))
        torch.cuda.synchronize(self.device)
        return out

    def set_params(self, flat):
        if isinstance(flat, torch.Tensor):
            t = flat.detach().to(torch.float32).contiguous()
            self._check(self.lib.tlp_set_params(self.h, t.data_ptr(), t.numel()))
        else:
            a = np.ascontiguousarray(flat, np.float32)
            self._check(self.lib.tlp_set_params(self.h, a.ctypes.data, a.size))

    def get_params(self) -> np.ndarray:
        a = np.zeros(self.num_params, np.float32)
        self._check(self.lib.tlp_get_params(self.h, a.ctypes.data, a.size))
        return a

    def get_grads(self) -> np.ndarray:
        a = np.zeros(self.num_params, np.float32)
        self._check(self.lib.tlp_get_grads(self.h, a.ctypes.data, a.size))
        return a

    def get_train_scores(self, B: int) -> np.ndarray:
        """Scores [B, n_tasks] of the last training forward (test hook, R26)."""
        a = np.zeros((B, self.cfg.n_tasks), np.float32)
        self._check(self.lib.tlp_get_train_scores(self.h, a.ctypes.data, a.size))
        return a

    def init_comm(self, group=None):
        """Create the library's NCCL communicator over torch.distributed ranks:
        rank 0 makes the ncclUniqueId, torch.distributed broadcasts its bytes."""
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        buf = (C.c_char * 128)()
        if rank == 0:
            self._check(self.lib.tlp_get_unique_id(buf))
        t = torch.tensor(list(bytes(buf)), dtype=torch.uint8)
        if dist.get_backend(group) == "nccl":
            t = t.cuda(self.device)
        dist.broadcast(t, 0, group=group)
        raw = bytes(t.cpu().tolist())
        C.memmove(buf, raw, 128)
        with torch.cuda.device(self.device):
            self._check(self.lib.tlp_set_comm(self.h, buf, rank, world))

    def broadcast_state(self, root: int = 0, stream=None):
        """tlp_broadcast_state (C-3): parameters + Adam state, scales and token
        table from rank `root` to every rank of the communicator."""
        self._check(self.lib.tlp_broadcast_state(self.h, root, _stream_ptr(stream, self.device)))

    def sync(self):
        self._check(self.lib.tlp_sync(self.h))

    @property
    def launches(self) -> int:
        return int(self.lib.tlp_launch_count(self.h))

    # --- hot path ------------------------------------------------------------
    def encode(self, batch: DeviceBatch, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        c = self.cfg
        if out is None:
            out = torch.empty((batch.N, c.L, c.E), dtype=torch.float32, device="cuda:%d" % self.device)
        b = batch.c_struct()
        self._check(self.lib.tlp_encode(self.h, C.byref(b), batch.N, out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def score(self, feats: torch.Tensor, out: Optional[torch.Tensor] = None, stream=None) -> torch.Tensor:
        assert feats.dtype == torch.float32 and feats.is_contiguous()
        N = feats.shape[0]
        if out is None:
            out = torch.empty((N, self.cfg.n_tasks), dtype=torch.float32, device=feats.device)
        self._check(self.lib.tlp_score(self.h, feats.data_ptr(), N, out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def _train(self, fn, feats, labels, group_off, loss_out, stream):
        assert feats.is_contiguous() and labels.is_contiguous()
        B = feats.shape[0]
        goff = np.ascontiguousarray(group_off, np.int64)
        if loss_out is None:
            loss_out = torch.empty(1, dtype=torch.float32, device=feats.device)
        self._check(fn(self.h, feats.data_ptr(), labels.data_ptr(), goff.ctypes.data, B,
                       len(goff) - 1, loss_out.data_ptr(), _stream_ptr(stream, self.device)))
        return loss_out

    def train_step(self, feats, labels, group_off, loss_out=None, stream=None) -> torch.Tensor:
        return self._train(self.lib.tlp_train_step, feats, labels, group_off, loss_out, stream)

    def compute_grads(self, feats, labels, group_off, loss_out=None, stream=None) -> torch.Tensor:
        return self._train(self.lib.tlp_compute_grads, feats, labels, group_off, loss_out, stream)

    def lambdarank(self, scores, labels, group_off, stream=None):
        B = scores.shape[0]
        goff = np.ascontiguousarray(group_off, np.int64)
        loss = torch.empty(1, dtype=torch.float32, device=scores.device)
        ds = torch.empty_like(scores)
        self._check(self.lib.tlp_lambdarank(self.h, scores.data_ptr(), labels.data_ptr(),
                                            goff.ctypes.data, B, len(goff) - 1, loss.data_ptr(),
                                            ds.data_ptr(), _stream_ptr(stream, self.device)))
        return loss, ds

    def mse(self, scores, labels, stream=None):
        """tlp_mse: the NEXT-3 MSE unit (loss [1], dscores like scores)."""
        B = scores.shape[0]
        loss = torch.empty(1, dtype=torch.float32, device=scores.device)
        ds = torch.empty_like(scores)
        self._check(self.lib.tlp_mse(self.h, scores.data_ptr(), labels.data_ptr(), B, loss.data_ptr(),
                                     ds.data_ptr(), _stream_ptr(stream, self.device)))
        return loss, ds

    def topk(self, scores: torch.Tensor, task_off, k: int, head: int = 0, shard_base: int = 0,
             idx_out=None, val_out=None, stream=None):
        toff = np.ascontiguousarray(task_off, np.int64)
        T = len(toff) - 1
        stride = scores.shape[1] if scores.dim() == 2 else 1
        if idx_out is None:
            idx_out = torch.empty((T, k), dtype=torch.int64, device=scores.device)
        if val_out is None:
            val_out = torch.empty((T, k), dtype=torch.float32, device=scores.device)
        self._check(self.lib.tlp_topk(self.h, scores.data_ptr(), stride, head, toff.ctypes.data, T, k,
                                      shard_base, idx_out.data_ptr(), val_out.data_ptr(),
                                      _stream_ptr(stream, self.device)))
        return idx_out, val_out

    def search_round(self, host_batch: DeviceBatch, task_off, k: int, head: int = 0,
                     shard_base: int = 0, chunks: int = 16, idx_out=None, val_out=None, stream=None):
        """One search round from host memory (tlp_search_round): encode -> score ->
        per-task top-k of a HOST batch (DeviceBatch.from_packed(..., pin=True)),
        the chunked host->device copy overlapped with the kernels.  Returns host
        (pinned) idx [T, k] int64 and val [T, k] fp32, valid after stream sync."""
        toff = np.ascontiguousarray(task_off, np.int64)
        T = len(toff) - 1
        if idx_out is None:
            idx_out = torch.empty((T, k), dtype=torch.int64).pin_memory()
        if val_out is None:
            val_out = torch.empty((T, k), dtype=torch.float32).pin_memory()
        assert not idx_out.is_cuda and not val_out.is_cuda
        cs = host_batch.c_struct()
        self._check(self.lib.tlp_search_round(self.h, C.byref(cs), host_batch.N, toff.ctypes.data, T, k,
                                              head, shard_base, chunks, idx_out.data_ptr(),
                                              val_out.data_ptr(), _stream_ptr(stream, self.device)))
        return idx_out, val_out

    def dedup(self, feats: torch.Tensor, group_off, labels: Optional[torch.Tensor] = None,
              stream=None):
        """tlp_dedup: duplicate classes of the rows of `feats` ([N, ...] fp32 device)
        within groups.  Returns (keep int32 [N], label_out fp32 [N] or None,
        n_distinct)."""
        assert feats.dtype == torch.float32 and feats.is_contiguous()
        N = feats.shape[0]
        row_len = feats.numel() // N if N else 1
        goff = np.ascontiguousarray(group_off, np.int64)
        keep = torch.empty(N, dtype=torch.int32, device=feats.device)
        lab = None
        if labels is not None:
            assert labels.dtype == torch.float32 and labels.is_contiguous()
            lab = torch.empty(N, dtype=torch.float32, device=feats.device)
        n = C.c_int64(0)
        self._check(self.lib.tlp_dedup(self.h, feats.data_ptr() if N else None, N, row_len,
                                       goff.ctypes.data, len(goff) - 1,
                                       labels.data_ptr() if labels is not None else None,
                                       keep.data_ptr() if N else None,
                                       lab.data_ptr() if lab is not None else None,
                                       C.byref(n), _stream_ptr(stream, self.device)))
        return keep, lab, int(n.value)

    def topk_score(self, scores: torch.Tensor, latency: torch.Tensor, group_off, weight, k: int,
                   head: int = 0, stream=None) -> float:
        """tlp_topk_score: the paper's top-k score metric."""
        goff = np.ascontiguousarray(group_off, np.int64)
        w = np.ascontiguousarray(weight, np.float64)
        stride = scores.shape[1] if scores.dim() == 2 else 1
        out = C.c_double(0.0)
        self._check(self.lib.tlp_topk_score(self.h, scores.data_ptr(), stride, head, latency.data_ptr(),
                                            goff.ctypes.data, w.ctypes.data, len(goff) - 1, k,
                                            C.byref(out), _stream_ptr(stream, self.device)))
        return float(out.value)

    def topk_merge(self, vals: torch.Tensor, idx: torch.Tensor, idx_out=None, val_out=None,
                   stream=None):
        """Merge per-shard top-k lists vals/idx [W, T, k] into the global [T, k]."""
        W, T, k = vals.shape
        vals, idx = vals.contiguous(), idx.contiguous()
        if idx_out is None:
            idx_out = torch.empty((T, k), dtype=torch.int64, device=vals.device)
        if val_out is None:
            val_out = torch.empty((T, k), dtype=torch.float32, device=vals.device)
        self._check(self.lib.tlp_topk_merge(self.h, vals.data_ptr(), idx.data_ptr(), W, T, k,
                                            idx_out.data_ptr(), val_out.data_ptr(),
                                            _stream_ptr(stream, self.device)))
        return idx_out, val_out

    def normalize_labels(self, latency: torch.Tensor, group_off, out=None, stream=None):
        goff = np.ascontiguousarray(group_off, np.int64)
        if out is None:
            out = torch.empty_like(latency)
        self._check(self.lib.tlp_normalize_labels(self.h, latency.data_ptr(), goff.ctypes.data,
                                                  len(goff) - 1, out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    # ---------------------------------------------------------------- NEXT-1
    def ga_set_space(self, space, id_base: int = 0):
        """tlp_ga_set_space from a host search space (any object with the
        fields of synth.PackedSpace: tmpl (packed batch), knob_off, knob_arg,
        knob_grp, dom_off, dom_num, dom_name); id_base = global id of its
        first subgraph (sharded tuning, dist.shard_subgraphs)."""
        arrs = DeviceBatch.host_arrays(space.tmpl)
        keep = dict(arrs)
        keep["knob_off"] = np.ascontiguousarray(space.knob_off, np.int64)
        keep["knob_arg"] = np.ascontiguousarray(space.knob_arg, np.int64)
        keep["knob_grp"] = np.ascontiguousarray(space.knob_grp, np.int32)
        keep["dom_off"] = np.ascontiguousarray(space.dom_off, np.int64)
        keep["dom_num"] = np.ascontiguousarray(space.dom_num, np.float64)
        keep["dom_name"] = np.ascontiguousarray(space.dom_name, np.int32)
        sp = _lib.tlp_ga_space()
        t = sp.tmpl
        t.seq_off, t.prim_type, t.arg_off = (keep[k].ctypes.data for k in ("seq_off", "prim_type", "arg_off"))
        t.arg_kind, t.arg_num, t.arg_name = (keep[k].ctypes.data for k in ("arg_kind", "arg_num", "arg_name"))
        t.str_blob, t.str_off = keep["str_blob"].ctypes.data, keep["str_off"].ctypes.data
        t.P, t.A, t.U = len(arrs["prim_type"]), len(arrs["arg_kind"]), len(arrs["str_off"]) - 1
        sp.S = len(keep["knob_off"]) - 1
        sp.id_base = id_base
        for k in ("knob_off", "knob_arg", "knob_grp", "dom_off", "dom_num", "dom_name"):
            setattr(sp, k, keep[k].ctypes.data)
        self._check(self.lib.tlp_ga_set_space(self.h, C.byref(sp)))
        self._ga_S = sp.S
        self._ga_strings = (arrs["str_blob"], arrs["str_off"])
        self.ga_G = int(self.lib.tlp_ga_num_genes(self.h))

    def ga_init(self, n: int, seed: int, rnd: int, out=None, stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self._ga_S * n, self.ga_G), dtype=torch.uint8, device="cuda")
        self._check(self.lib.tlp_ga_init(self.h, n, seed, rnd, out.data_ptr(), _stream_ptr(stream, self.device)))
        return out

    def ga_evolve(self, pop: torch.Tensor, pop_scores: torch.Tensor, n_pop: int, n_child: int,
                  p_cross: float, p_mut: float, seed: int, rnd: int, it: int, out=None,
                  stream=None) -> torch.Tensor:
        if out is None:
            out = torch.empty((self._ga_S * n_child, self.ga_G), dtype=torch.uint8, device="cuda")
        self._check(self.lib.tlp_ga_evolve(self.h, pop.data_ptr(), pop_scores.data_ptr(), n_pop, n_child,
                                           p_cross, p_mut, seed, rnd, it, out.data_ptr(),
                                           _stream_ptr(stream, self.device)))
        return out

    def ga_materialize(self, genes: torch.Tensor, n: int, stream=None) -> DeviceBatch:
        """The packed abstract primitives of S*n gene rows (a DeviceBatch
        sharing the space's string table)."""
        P, A = C.c_int64(0), C.c_int64(0)
        self._check(self.lib.tlp_ga_batch_size(self.h, n, C.byref(P), C.byref(A)))
        dev = genes.device
        N = self._ga_S * n
        e = lambda k, dt: torch.empty(max(k, 1), dtype=dt, device=dev)  # noqa: E731
        b = DeviceBatch(e(N + 1, torch.int64), e(P.value, torch.uint8), e(P.value + 1, torch.int64),
                        e(A.value, torch.uint8), e(A.value, torch.float64), e(A.value, torch.int32),
                        torch.from_numpy(self._ga_strings[0]).to(dev),
                        torch.from_numpy(self._ga_strings[1]).to(dev),
                        N=N, P=P.value, A=A.value, U=len(self._ga_strings[1]) - 1)
        self._check(self.lib.tlp_ga_materialize(self.h, genes.data_ptr(), n, b.seq_off.data_ptr(),
                                                b.prim_type.data_ptr(), b.arg_off.data_ptr(),
                                                b.arg_kind.data_ptr(), b.arg_num.data_ptr(),
                                                b.arg_name.data_ptr(), _stream_ptr(stream, self.device)))
        return b

    def ga_drop_duplicates(self, genes: torch.Tensor, n: int, scores: torch.Tensor, stream=None):
        self._check(self.lib.tlp_ga_drop_duplicates(self.h, genes.data_ptr(), n, scores.data_ptr(),
                                                    _stream_ptr(stream, self.device)))
        return scores

    def ga_round(self, n_pop: int, n_child: int, iters: int, p_cross: float, p_mut: float,
                 seed: int, rnd: int, head: int = 0, genes_out=None, scores_out=None, stream=None):
        """tlp_ga_round: one device-resident tuning round of every subgraph.
        Returns (genes [S*n_pop, G] uint8, scores [S*n_pop] fp32) on the device,
        each subgraph's survivors in rank order."""
        S = self._ga_S
        if genes_out is None:
            genes_out = torch.empty((S * n_pop, self.ga_G), dtype=torch.uint8, device="cuda")
        if scores_out is None:
            scores_out = torch.empty(S * n_pop, dtype=torch.float32, device="cuda")
        self._check(self.lib.tlp_ga_round(self.h, n_pop, n_child, iters, p_cross, p_mut, seed, rnd, head,
                                          genes_out.data_ptr(), scores_out.data_ptr(),
                                          _stream_ptr(stream, self.device)))
        return genes_out, scores_out
