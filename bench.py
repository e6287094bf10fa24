"""Benchmark of the TLP / MTL-TLP hot path on B200 (the driver's contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One STEP = one pass of the whole hot path on synthetic
TenSet-shaped inputs:
  scoring round  (BASELINE configs[1], C2): 409,600 candidates = 100 tasks x 4096,
                 tlp_encode -> tlp_score (hidden 256, 2 attention layers) ->
                 tlp_topk (k = 16 per task; + NCCL allgather merge when N > 1);
  training step  (configs[2], C3 shape): tlp_normalize_labels of the batch's
                 groups + tlp_train_step on 16 groups x 512 = 8,192 samples
                 (1 attention layer, LambdaRank, backward, allreduce, Adam).
`value` = candidates scored/s over the scoring phase (all ranks, max-over-ranks
device time); `train_samples_per_s` = the training phase likewise.  Weak
scaling: per-GPU work is fixed as N grows.  Inputs are larger than L2 (901 MB
of features per round), so no explicit flush is needed between iterations.

`--impl reference` times the CPU oracle (oracle/, the only reference this
paper-only tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "candidates scored/s and LambdaRank train samples/s at 1/2/4/8 B200; % tensor peak"
T_TASKS, PER_TASK, TOPK = 100, 4096, 16
N_ROUND = T_TASKS * PER_TASK
TRAIN_GROUPS, TRAIN_PER_GROUP = 16, 512
B_TRAIN = TRAIN_GROUPS * TRAIN_PER_GROUP


def _traffic(kernel: str):
    """DRAM bytes per launch of `kernel` from the newest profiles/*_traffic.json."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    for f in reversed(files):
        d = json.load(open(f))
        if kernel in d:
            return d[kernel]["dram_read_bytes"] + d[kernel]["dram_write_bytes"]
    return None


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
            "sm_max_mhz": 1965.0}, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    def __init__(self, device: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        nv = self.nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwSlowdown", 0x8),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwThermalSlowdown", 0x40),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksThrottleReasonSwThermalSlowdown", 0x20),
            "sw_power_cap": getattr(nv, "nvmlClocksThrottleReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksThrottleReasonHwPowerBrakeSlowdown", 0x80),
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for k, bit in names.items():
                    if r & bit:
                        self.reasons.add(k)
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# ------------------------------------------------------------------ FLOP model
def fwd_flops_per_cand(L=25, E=22, H=256, up=(128, 256), heads=8, n_attn=2, n_res=2, hd=128,
                       n_tasks=1):
    """Algorithmic forward FLOPs per candidate."""
    f, d = 0, E
    for w in up:
        f += 2 * L * d * w
        d = w
    dh = H // heads
    f += n_attn * (2 * L * H * 3 * H + heads * 2 * (2 * L * L * dh) + 2 * L * H * H)
    f += n_res * 2 * (2 * L * H * H)
    f += n_tasks * (2 * L * H * hd + 2 * hd)
    return f


def train_flops_per_sample(n_attn=1, n_tasks=1, **kw):
    """Algorithmic forward + backward FLOPs per training sample: every dense
    layer costs its forward GEMM plus the dgrad and wgrad GEMMs (2x), except
    the first upsample layer, whose input is data (no dgrad); the attention
    core QK^T / PV likewise 3x (90.68 M at 1 layer)."""
    L, E, up = kw.get("L", 25), kw.get("E", 22), kw.get("up", (128, 256))
    return 3 * fwd_flops_per_cand(n_attn=n_attn, n_tasks=n_tasks, **kw) - 2 * L * E * up[0]


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2211_03578_b200 as tp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    precision = args.precision
    dev = torch.device("cuda", local)
    # --- model state through the library only (no oracle code on this arm):
    # rank 0 fits the token table (R1) and the normalisation scales (R3) on a
    # seeded training split and initialises the weights; tlp_broadcast_state
    # (C-3) hands the state to the other ranks ---
    packed = synth.generate(1000 + rank, N_ROUND)
    task_off = synth.uniform_task_off(T_TASKS, PER_TASK)

    def init_flat(cfg, seed):
        return np.concatenate([v.ravel() for v in synth.init_params(seed, cfg.param_shapes())]).astype(np.float32)

    def make(cfg, seed):
        m = tp.TLP(cfg, device=local)
        if rank == 0:
            m.fit_token_table(synth.generate(12345, 2000, unseen_rate=0.0))
            m.fit_norm_scales(tp.DeviceBatch.from_packed(synth.generate(99, 2000, unseen_rate=0.0), device=dev))
            m.set_params(init_flat(cfg, seed))
        if world > 1:
            m.init_comm()
            m.broadcast_state(root=0)
        return m

    cfg2 = tp.TLPConfig(n_attn=2, precision=precision)
    scorer = make(cfg2, 7)
    cfg1 = tp.TLPConfig(n_attn=1, precision=precision)
    trainer = make(cfg1, 8)

    dbatch = tp.DeviceBatch.from_packed(packed, device=dev)
    feats = torch.empty((N_ROUND, 25, 22), dtype=torch.float32, device=dev)
    scores = torch.empty((N_ROUND, 1), dtype=torch.float32, device=dev)
    idx = torch.empty((T_TASKS, TOPK), dtype=torch.int64, device=dev)
    val = torch.empty((T_TASKS, TOPK), dtype=torch.float32, device=dev)
    # training data: 16 groups x 512, latencies -> labels on device
    tpacked = synth.generate(2000 + rank, B_TRAIN)
    goff = np.arange(TRAIN_GROUPS + 1, dtype=np.int64) * TRAIN_PER_GROUP
    lat = torch.from_numpy(synth.latencies(tpacked, goff, 5 + rank).astype(np.float32)).to(dev)
    tfeats = trainer.encode(tp.DeviceBatch.from_packed(tpacked, device=dev))
    labels = torch.empty((B_TRAIN, 1), dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    shard_base = rank * N_ROUND

    def step(ev):
        ev[0].record(stream)
        scorer.encode(dbatch, out=feats, stream=stream)
        ev[1].record(stream)
        scorer.score(feats, out=scores, stream=stream)
        ev[2].record(stream)
        scorer.topk(scores, task_off, TOPK, shard_base=shard_base, idx_out=idx, val_out=val, stream=stream)
        ev[3].record(stream)
        trainer.normalize_labels(lat, goff, out=labels.view(-1), stream=stream)
        trainer.train_step(tfeats, labels, goff, loss_out=loss, stream=stream)
        ev[4].record(stream)

    mk = lambda: [torch.cuda.Event(enable_timing=True) for _ in range(5)]  # noqa: E731
    for _ in range(args.warmup):
        step(mk())
    scorer.sync(); trainer.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = scorer.launches + trainer.launches
    evs = [mk() for _ in range(args.steps)]
    clk = ClockSampler(local)
    with clk:
        t_start = torch.cuda.Event(enable_timing=True); t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        t_end.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    scorer.sync(); trainer.sync()
    launches = scorer.launches + trainer.launches - l0
    total_ms = t_start.elapsed_time(t_end)
    enc_ms = sum(e[0].elapsed_time(e[1]) for e in evs)
    score_ms = sum(e[1].elapsed_time(e[2]) for e in evs)
    topk_ms = sum(e[2].elapsed_time(e[3]) for e in evs)
    train_ms = sum(e[3].elapsed_time(e[4]) for e in evs)
    round_ms = enc_ms + score_ms + topk_ms
    times = torch.tensor([total_ms, round_ms, train_ms, score_ms, enc_ms, topk_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(times, op=dist.ReduceOp.MAX)
    total_ms, round_ms, train_ms, score_ms, enc_ms, topk_ms = times.tolist()

    # --- e2e: one C-ABI call per round from host buffers (tlp_search_round: pinned
    # H2D of the packed round in chunks overlapped with encode + score, top-k,
    # D2H of the top-k) ---
    hbatch = tp.DeviceBatch.from_packed(packed, pin=True)
    idx_host = torch.empty((T_TASKS, TOPK), dtype=torch.int64).pin_memory()
    val_host = torch.empty((T_TASKS, TOPK), dtype=torch.float32).pin_memory()
    def e2e_step():
        scorer.search_round(hbatch, task_off, TOPK, shard_base=shard_base, chunks=args.chunks,
                            idx_out=idx_host, val_out=val_host, stream=stream)
    for _ in range(max(1, args.warmup)):
        e2e_step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # --- host side, reported separately: the H2D copy of one packed
    # round from pinned memory alone, and host packing of candidate sequences
    # (synth.pack, pure Python) on a bounded sample; neither is in `value` ---
    import time
    hb = hbatch.nbytes()
    src_h = torch.empty(hb, dtype=torch.uint8).pin_memory()
    dst_d = torch.empty(hb, dtype=torch.uint8, device=dev)
    dst_d.copy_(src_h, non_blocking=True)
    torch.cuda.synchronize()
    h0 = torch.cuda.Event(enable_timing=True); h1 = torch.cuda.Event(enable_timing=True)
    h0.record(); dst_d.copy_(src_h, non_blocking=True); h1.record(); h1.synchronize()
    h2d_ms = h0.elapsed_time(h1)
    del src_h, dst_d
    sample = packed.to_lists()[:20000]
    t0 = time.perf_counter()
    synth.pack(sample)
    pack_s = time.perf_counter() - t0
    host_side = {"h2d_ms_per_round": h2d_ms, "h2d_GBps": hb / (h2d_ms / 1e3) / 1e9,
                 "pack_us_per_candidate": pack_s / len(sample) * 1e6,
                 "pack_sample": "synth.pack of %d candidates (Python, one core)" % len(sample)}

    # --- NEXT-2 rows: duplicate scan of this round's features and
    # the §6.1 top-k score of its scores against synthetic latencies ---
    next_rows = next2_measure(scorer, feats, scores, task_off, args, stream, dev)
    next_rows.update(next1_measure(scorer, args, stream, rank))
    next_rows.update(next4_measure(feats, tfeats, labels, goff, precision, args, stream, local))
    next_rows.update(c5_measure(scorer, feats, args, stream, world))
    next_rows.update(k9_measure(trainer, labels, goff, args, stream))

    K = args.steps
    cand_s = world * N_ROUND * K / (round_ms / 1e3)
    train_s = world * B_TRAIN * K / (train_ms / 1e3)
    peaks, peaks_kind = load_peaks()
    fl = fwd_flops_per_cand()
    score_launch_ms = score_ms / K
    clocks = clk.summary()
    # burst peak for a kernel that ran at (near) the maximum clock -- the
    # sustained figure was measured at a lower median clock (MEASURED_PEAKS.json
    # clocks_under_load); both fractions are reported
    at_max = bool(clocks.get("sm_mhz") and clocks.get("sm_max_mhz") and
                  clocks["sm_mhz"] >= 0.95 * clocks["sm_max_mhz"])
    burst, sust = peaks["bf16_tflops"], peaks["bf16_tflops_sustained"]
    peak_used, kind_used = (burst, "bf16 burst") if at_max else (sust, "bf16 sustained")
    if precision == "bf16":
        achieved = fl * N_ROUND / (score_launch_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "kernel": "tc_forward_kernel (tlp_score, 1 launch/round)",
                "achieved": achieved, "peak": peak_used, "unit": "TFLOP/s", "frac": achieved / peak_used,
                "frac_burst": achieved / burst, "frac_sustained": achieved / sust,
                "traffic": _traffic("tc_forward_kernel"), "peak_kind": peaks_kind + " " + kind_used +
                " (burst when the timed region's median SM clock >= 95% of max)",
                "flops_per_launch": fl * N_ROUND,
                "traffic_note": "dram__bytes_read+write per launch from profiles/*_traffic.json "
                                "(ncu --set full of the same command); algorithmic input 2,200 B/cand"}
    else:
        achieved = fl * N_ROUND / (score_launch_ms / 1e3) / 1e12
        sm_mhz = peaks.get("sm_max_mhz", 1965.0)
        peak = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
        roof = {"bound": "alu", "kernel": "tlp_score fp32 SIMT chain (all launches of one call)",
                "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None, "peak_kind": "derived FP32 FFMA peak 148 SM x 128 lanes x 2 x sm_max_mhz",
                "flops_per_launch": fl * N_ROUND}
    out = {
        "metric": METRIC, "value": cand_s, "unit": "candidates/s", "n_gpus": world,
        "steps": K, "warmup": args.warmup, "ms_per_step": total_ms / K,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16" if precision == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": "C2 scoring round: 409,600 candidates (100 tasks x 4096), hidden 256, "
                               "2 attention layers, top-16/task; + C3-shape LambdaRank train step "
                               "8,192 samples (16 groups x 512), 1 attention layer",
                   "candidates_per_gpu_per_round": N_ROUND, "train_batch_per_gpu": B_TRAIN,
                   "precision": precision, "parallelism": "dp%d" % world,
                   "l2": "inputs larger than L2 (901 MB features/round), no flush"},
        "train_samples_per_s": train_s,
        "phase_ms_per_step": {"encode": enc_ms / K, "score": score_ms / K, "topk": topk_ms / K,
                              "train": train_ms / K},
        "score_only": {"value": world * N_ROUND * K / (score_ms / 1e3), "unit": "candidates/s"},
        "host_side": host_side,
        "roofline": roof,
        "e2e": {"value": world * N_ROUND * K / (e2e_ms / 1e3), "unit": "candidates/s",
                "h2d_bytes_per_step": hbatch.nbytes(), "d2h_bytes_per_step": T_TASKS * TOPK * 12,
                "call": "tlp_search_round, %d chunks" % args.chunks},
        "gpu_launches": launches,
        "next_rows": next_rows,
        "clocks": clocks,
    }
    tfl = train_flops_per_sample(n_attn=1)
    t_ach = tfl * B_TRAIN / (train_ms / K / 1e3) / 1e12
    out["roofline_train"] = {
        "bound": "tensor", "scope": "whole C3 train step (label normalisation, forward, LambdaRank, "
                                    "backward, allreduce, Adam; all kernels)",
        "achieved": t_ach, "peak": peak_used, "unit": "TFLOP/s", "frac": t_ach / peak_used,
        "frac_burst": t_ach / burst, "flops_per_step": tfl * B_TRAIN,
        "flops_note": "algorithmic fwd + bwd (bwd = dgrad + wgrad) per sample %.2f M x %d samples; "
                      "the bf16 context executes the dense layers as bf16x3 (3 MMAs per product, R37)"
                      % (tfl / 1e6, B_TRAIN)}
    out["c4_mtl"] = c4_measure(scorer, feats, args, stream, local, dev, world)
    out["c1_tiny"] = c1_measure(args, local, dev)
    if world > 1:
        out["allreduce"] = allreduce_measure(trainer, dev)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(seconds_hint=12.0)
        out["cpu_baseline_1core"] = cpu_baseline(seconds_hint=8.0, threads=1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


GA_S, GA_POP, GA_CHILD, GA_ITERS = 100, 512, 1920, 4


def c4_measure(enc, feats, args, stream, local, dev, world):
    """C4 (BASELINE configs[3]): MTL-TLP, a shared 1-layer encoder and 4
    hardware heads, the target head's labels on a seeded 7%
    Bernoulli subset, tasks 1..3 fully labelled.  Training: the C3-shape
    step (16 groups x 512) through tlp_train_step; scoring: tlp_score (4 scores
    per candidate, fused bf16 kernel) over the round's 409,600 encoded
    candidates.  CUDA events, W warm-up + K timed calls; model state as the
    main line (library-initialised weights, device-side labels)."""
    import torch
    import paper_2211_03578_b200 as tp
    cfg = tp.TLPConfig(n_attn=1, n_tasks=4, precision=args.precision)
    m = tp.TLP(cfg, device=local)
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(10, cfg.param_shapes())]).astype(np.float32))
    if world > 1:
        m.init_comm()
    rank = int(os.environ.get("RANK", "0"))
    tp_b = synth.generate(3000 + rank, B_TRAIN)
    goff = np.arange(TRAIN_GROUPS + 1, dtype=np.int64) * TRAIN_PER_GROUP
    lab = np.stack([synth.latencies(tp_b, goff, 40 + rank, task_noise=0.3 * (t > 0)) for t in range(4)], 1)
    lab_d = torch.from_numpy(lab.astype(np.float32)).to(dev)
    y = torch.empty((B_TRAIN, 4), dtype=torch.float32, device=dev)
    for t in range(4):
        col = m.normalize_labels(lab_d[:, t].contiguous(), goff, stream=stream)
        y[:, t] = col
    keep = torch.from_numpy(np.random.default_rng(41 + rank).random(B_TRAIN) < 0.07).to(dev)
    y[:, 0] = torch.where(keep, y[:, 0], torch.full_like(y[:, 0], float("nan")))
    y = y.contiguous()
    X = enc.encode(tp.DeviceBatch.from_packed(tp_b, device=dev), stream=stream)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    sc = torch.empty((feats.shape[0], 4), dtype=torch.float32, device=dev)

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    steps = max(1, args.steps)
    t_ms = timed(lambda: m.train_step(X, y, goff, loss_out=loss, stream=stream), steps)
    s_ms = timed(lambda: m.score(feats, out=sc, stream=stream), max(1, min(steps, 5)))
    m.sync()
    fl_t, fl_s = train_flops_per_sample(n_attn=1, n_tasks=4), fwd_flops_per_cand(n_attn=1, n_tasks=4)
    return {"train": {"value": world * B_TRAIN / (t_ms / 1e3), "unit": "samples/s", "ms_per_step": t_ms,
                      "tflops": fl_t * B_TRAIN / (t_ms / 1e3) / 1e12},
            "score": {"value": world * feats.shape[0] / (s_ms / 1e3), "unit": "candidates/s",
                      "ms_per_call": s_ms, "tflops": fl_s * feats.shape[0] / (s_ms / 1e3) / 1e12},
            "target_label_frac": float(keep.float().mean().item()),
            "config": "MTL-TLP 4 heads, 1 attention layer, hidden 256, %s; train 16 groups x 512 "
                      "(target head on 7%% of samples); score 409,600 candidates" % args.precision}


def c1_measure(args, local, dev):
    """C1 (BASELINE configs[0]): the tiny model (hidden 64, 1 layer, 1 task) on
    256 synthetic candidates: tlp_encode -> tlp_score -> LambdaRank (loss +
    dL/ds) -> top-16, the fp32 SIMT context (the bf16 tensor-core kernels need
    the paper shape).  Launch-latency bound: reported as wall time per call
    (host clock around the synchronised sequence, median of K) and as device
    time (CUDA events)."""
    import time
    import torch
    import paper_2211_03578_b200 as tp
    cfg = tp.tiny_config()
    m = tp.TLP(cfg, device=local)
    m.fit_token_table(synth.generate(12345, 500, unseen_rate=0.0))
    b = tp.DeviceBatch.from_packed(synth.generate(77, 256), device=dev)
    m.fit_norm_scales(b)
    m.set_params(np.concatenate([v.ravel() for v in synth.init_params(11, cfg.param_shapes())]).astype(np.float32))
    goff = np.array([0, 256], np.int64)
    lat = torch.from_numpy(synth.latencies(synth.generate(77, 256), goff, 3).astype(np.float32)).to(dev)
    y = m.normalize_labels(lat, goff).view(256, 1).contiguous()
    stream = torch.cuda.current_stream(dev)

    def call():
        X = m.encode(b, stream=stream)
        s = m.score(X, stream=stream)
        m.lambdarank(s, y, goff, stream=stream)
        m.topk(s, goff, TOPK, stream=stream)
    for _ in range(args.warmup):
        call()
    torch.cuda.synchronize()
    walls = []
    for _ in range(max(5, args.steps)):
        t0 = time.perf_counter()
        call()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(max(5, args.steps)):
        call()
    e1.record(stream)
    torch.cuda.synchronize()
    return {"wall_ms_per_call": statistics.median(walls),
            "device_ms_per_call": e0.elapsed_time(e1) / max(5, args.steps),
            "config": "256 candidates, hidden 64, 1 attention layer, fp32: encode + score + LambdaRank + top-16"}


def allreduce_measure(m, dev):
    """The C-1 gradient allreduce alone: ncclAllReduce (sum, fp32) of the
    trainer's gradient vector through torch.distributed (the same NCCL, same
    size as the library's in-step allreduce), CUDA events, max over ranks."""
    import torch
    import torch.distributed as dist
    n = m.num_params
    buf = torch.zeros(n, dtype=torch.float32, device=dev)
    for _ in range(5):
        dist.all_reduce(buf)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        dist.all_reduce(buf)
    e1.record()
    torch.cuda.synchronize()
    us = torch.tensor([e0.elapsed_time(e1) * 1e3 / reps], dtype=torch.float64, device=dev)
    dist.all_reduce(us, op=dist.ReduceOp.MAX)
    return {"us_per_allreduce": float(us.item()), "bytes": 4 * n,
            "nccl_debug_file": os.environ.get("NCCL_DEBUG_FILE"),
            "note": "torch.distributed NCCL allreduce of the same fp32 gradient size; NCCL_DEBUG=INFO "
                    "log (algorithm / protocol / NVLS selection) written to nccl_debug_file"}


def next4_measure(feats, tfeats, labels, goff, precision, args, stream, local):
    """NEXT-4: the LSTM backbone (R49, 1 layer, paper widths) in
    place of attention -- scoring the round's 409,600 encoded candidates and
    one C3-shape LambdaRank train step (8,192 samples), CUDA events, W warm-up
    + K timed calls.  Layer-by-layer path: bf16x3 tcgen05 GEMMs for the input
    projection and each of the 25 recurrent steps, SIMT cells."""
    import torch
    import paper_2211_03578_b200 as tp
    cfg = tp.TLPConfig(n_attn=1, precision=precision, backbone="lstm")
    flat = np.concatenate([v.ravel() for v in synth.init_params(9, cfg.param_shapes())]).astype(np.float32)
    out = {}
    m = tp.TLP(cfg, device=local)
    m.set_params(flat)
    sc = torch.empty((feats.shape[0], 1), dtype=torch.float32, device=feats.device)
    loss = torch.empty(1, dtype=torch.float32, device=feats.device)

    def timed(fn, steps):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    steps = max(1, min(args.steps, 3))
    ms = timed(lambda: m.score(feats, out=sc, stream=stream), steps)
    fl = 25 * (2 * (2 * 256 * 1024)) + (fwd_flops_per_cand(n_attn=0))  # LSTM GEMMs + the rest
    out["lstm_score"] = {"value": feats.shape[0] / (ms / 1e3), "unit": "candidates/s", "ms_per_call": ms,
                         "tflops": fl * feats.shape[0] / (ms / 1e3) / 1e12,
                         "config": "409,600 candidates, 1 LSTM layer (hidden 256), %s" % precision}
    ms = timed(lambda: m.train_step(tfeats, labels, goff, loss_out=loss, stream=stream), steps)
    out["lstm_train"] = {"value": tfeats.shape[0] / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms,
                         "config": "8,192 samples (16 groups x 512), LambdaRank, 1 LSTM layer, %s" % precision}
    return out


def k9_measure(m, labels, goff, args, stream):
    """K9: the LambdaRank loss + dL/ds kernel alone on the
    training batch (16 groups x 512, seeded scores), CUDA events over K calls.
    Work = ordered pairs evaluated (sum over groups of n^2), ~30 FLOP + 2 SFU per
    pair; roofline: the FP32 SIMT peak SMs x 128 x 2 x clock."""
    import torch
    g = torch.Generator(device=labels.device).manual_seed(5)
    sc = torch.randn(labels.shape, generator=g, device=labels.device, dtype=torch.float32)
    steps = max(1, args.steps)
    for _ in range(args.warmup):
        m.lambdarank(sc, labels, goff, stream=stream)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        m.lambdarank(sc, labels, goff, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    sizes = np.diff(np.asarray(goff, np.int64))
    pairs = float((sizes.astype(np.float64) ** 2).sum())
    props = torch.cuda.get_device_properties(labels.device)
    peak = props.multi_processor_count * 128 * 2 * 1.965e9 / 1e12
    ach = 30.0 * pairs / (ms / 1e3) / 1e12
    return {"k9_lambdarank": {"value": pairs / (ms / 1e3), "unit": "ordered pairs/s", "ms_per_call": ms,
                              "roofline": {"bound": "alu", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
                                           "frac": ach / peak,
                                           "peak_kind": "derived: SMs x 128 FP32 lanes x 2 x 1965 MHz"},
                              "note": "one call incl. the host group offsets; 16 groups x 512"}}


def c5_measure(m, feats, args, stream, world):
    """C5 (BASELINE configs[4]): candidates per round swept over
    10^4 .. 10^7 on each GPU -- tlp_score + per-task top-16 over 100 tasks
    (with the NCCL allgather merge when N > 1 GPUs: world x N candidates per
    round) on device-resident encoded features; beyond the C2 round's 409,600
    rows the features repeat.  Encode is excluded here (the main line times it:
    0.64 ms per 409,600).  Shows the small-N regime, where a round is one
    partial wave of the 148-SM persistent forward plus launch latency."""
    import torch
    points = []
    steps = max(1, min(args.steps, 3))
    for n in (10_000, 100_000, 1_000_000, 10_000_000):
        if n <= feats.shape[0]:
            x = feats[:n]
        else:
            x = feats.repeat((n + feats.shape[0] - 1) // feats.shape[0], 1, 1)[:n].contiguous()
        sc = torch.empty((n, 1), dtype=torch.float32, device=feats.device)
        off = np.linspace(0, n, T_TASKS + 1).astype(np.int64)
        ti = torch.empty((T_TASKS, TOPK), dtype=torch.int64, device=feats.device)
        tv = torch.empty((T_TASKS, TOPK), dtype=torch.float32, device=feats.device)

        def call():
            m.score(x, out=sc, stream=stream)
            m.topk(sc, off, TOPK, idx_out=ti, val_out=tv, stream=stream)
        for _ in range(args.warmup):
            call()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            call()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        points.append({"N_per_gpu": n, "value": world * n / (ms / 1e3), "ms_per_round": ms})
        del x, sc
    torch.cuda.empty_cache()
    return {"c5_sweep": {"unit": "candidates/s", "points": points,
                         "config": "score + top-16 per task over 100 tasks, 2-layer bf16 model, "
                                   "device-resident features, %d GPU(s)" % world}}


def next1_measure(m, args, stream, rank):
    """NEXT-1: one device-resident tuning round of 100 synthetic
    subgraphs (tlp_ga_round): 512 + 1,920 initial programs, then 4 GA
    iterations of 1,920 children per subgraph = 10,112 programs featurised and
    scored per subgraph per round ("approximately 10,000 ... for each
    subgraph in one round"), the paper-size 2-layer bf16 model.  Timed with CUDA
    events over K rounds after W warm-up rounds; then 3 rounds of the host
    tuner (round + survivors D2H + 10 synthetic measurements per subgraph,
    P:558) timed by the host clock around synchronised rounds."""
    import time
    import torch
    from paper_2211_03578_b200.search import Tuner
    ts = [synth.make_template(2000 + rank, s) for s in range(GA_S)]
    m.ga_set_space(synth.pack_space(ts))
    per_round = GA_S * (GA_POP + GA_CHILD + GA_ITERS * GA_CHILD)
    for r in range(args.warmup):
        m.ga_round(GA_POP, GA_CHILD, GA_ITERS, 0.5, 0.2, seed=1, rnd=r, stream=stream)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for r in range(args.steps):
        m.ga_round(GA_POP, GA_CHILD, GA_ITERS, 0.5, 0.2, seed=1, rnd=100 + r, stream=stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    tuner = Tuner(m, GA_S, [t.G for t in ts], n_pop=GA_POP, n_child=GA_CHILD, iters=GA_ITERS, seed=2)
    lat = lambda s, g: float(synth.template_latency(ts[s], g, 2000 + rank, s)[0])  # noqa: E731
    tuner.run_round(0, lat)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for r in range(1, 4):
        tuner.run_round(r, lat)
    host_ms = (time.perf_counter() - t0) * 1e3 / 3
    return {"tune_round": {"value": per_round / (ms / 1e3), "unit": "candidates/s", "ms_per_round": ms,
                           "candidates_per_round": per_round,
                           "config": "100 subgraphs x (512 + 1920 + 4 x 1920) programs, 2-layer bf16 model",
                           "tuner_ms_per_round": host_ms,
                           "tuner_measurements": tuner.total}}


# ------------------------------------------------------------------ oracle arm
def next2_measure(m, feats, scores, task_off, args, stream, dev):
    """Time tlp_dedup over the round's 409,600 feature matrices (1% planted
    duplicates inside the 100 groups = the round's tasks) and tlp_topk_score (k=1, 5) over
    its scores, CUDA events on the launching stream, W warm-up + K timed calls.
    dedup roofline: HBM, algorithmic bytes = each 2,200-byte row read once + a
    duplicate's row re-read for verification + 8 B key + 16 B table slot per
    row."""
    import torch
    N = feats.shape[0]
    rng = np.random.default_rng(11)
    X = feats.clone()
    goff = np.asarray(task_off, np.int64)
    per = int(goff[1] - goff[0])  # uniform task segments: plant duplicates inside groups
    src_h = rng.integers(0, N, N // 100)
    dst_h = (src_h // per) * per + rng.integers(0, per, N // 100)
    X[torch.from_numpy(dst_h).to(dev)] = X[torch.from_numpy(src_h).to(dev)]
    lat = torch.from_numpy(np.random.default_rng(5).lognormal(0.0, 0.7, N).astype(np.float32)).to(dev)
    w = np.random.default_rng(6).integers(1, 6, len(goff) - 1).astype(np.float64)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    res = {}
    ms = timed(lambda: m.dedup(X, goff, stream=stream))
    _, _, n = m.dedup(X, goff, stream=stream)
    peaks, kind = load_peaks()
    dup = N - n
    bytes_alg = N * (2200 + 8 + 16) + dup * 2200
    res["dedup"] = {"value": N / (ms / 1e3), "unit": "candidates/s", "ms_per_call": ms,
                    "duplicate_rate": dup / N, "distinct": n,
                    "roofline": {"bound": "hbm", "achieved": bytes_alg / (ms / 1e3) / 1e9,
                                 "peak": peaks["hbm_gbs"], "unit": "GB/s",
                                 "frac": bytes_alg / (ms / 1e3) / 1e9 / peaks["hbm_gbs"],
                                 "peak_kind": kind + " HBM copy bandwidth"},
                    "note": "synchronous call: includes the host read-back of the distinct count"}
    for k in (1, 5):
        ms = timed(lambda: m.topk_score(scores, lat, goff, w, k, stream=stream))
        res["topk_score_k%d" % k] = {"value": N / (ms / 1e3), "unit": "candidates/s", "ms_per_call": ms,
                                     "score": m.topk_score(scores, lat, goff, w, k, stream=stream)}
    return res


def _oracle_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(n_cand: int, seed: int = 0):
    """One bounded sample of the step on the CPU oracle: encode + forward (2
    layers) + top-k of n_cand candidates (1 task); returns seconds."""
    import oracle
    from oracle import model as OM
    tokens = oracle.build_token_table(synth.training_stream())
    train_raw = synth.generate(99, 500, unseen_rate=0.0)
    raw = np.stack([oracle.extract_rows(s, tokens, 25, 22, 11) for s in train_raw.to_lists()])
    scale = oracle.fit_scales(raw)
    cfg = OM.Config(n_attn=2)
    p = OM.unflatten(cfg, np.concatenate([v.ravel() for v in synth.init_params(7, OM.param_shapes(cfg))]))
    b = synth.generate(1000 + seed, n_cand)
    t0 = time.perf_counter()
    X = oracle.encode(b.to_lists(), tokens, scale)
    s = OM.forward(cfg, p, X)
    oracle.topk(s[:, 0].astype(np.float32), np.array([0, n_cand]), TOPK)
    return time.perf_counter() - t0


def cpu_baseline(seconds_hint=15.0, threads=None):
    """The oracle as it stands on the host cores: all BLAS threads (threads=None)
    or limited with threadpoolctl (threads=1: one core, SURVEY §8(d) "time it
    twice")."""
    import contextlib
    ctx = contextlib.nullcontext()
    if threads is not None:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=threads)
    with ctx:
        cores = _oracle_threads()
        n = 128
        dt = oracle_sample(n)
        # scale the sample to ~seconds_hint of CPU work
        n2 = int(min(16384, max(128, n * seconds_hint / max(dt, 1e-3))))
        dt2 = oracle_sample(n2, seed=1)
    return {"value": n2 / dt2, "unit": "candidates/s", "cores": cores, "kind": "oracle",
            "host_cpus": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            "sample": "%d candidates of the C2 round (1 task): oracle encode + fp64 forward (2 attention "
                      "layers, hidden 256) + top-16, %.1f s, %d BLAS thread(s)" % (n2, dt2, cores)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n = 512
    for w in range(args.warmup):
        oracle_sample(n, seed=100 + w)
    t = 0.0
    for k in range(args.steps):
        t += oracle_sample(n, seed=k)
    v = n * args.steps / t
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "candidates/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * t / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": "C2 scoring round, bounded sample per step: %d candidates "
                                  "(encode + fp64 forward 2 layers + top-16) on host cores" % n},
           "cpu_baseline": {"value": v, "unit": "candidates/s", "cores": _oracle_threads(),
                            "kind": "oracle", "sample": "%d candidates per step" % n},
           "e2e": {"value": v, "unit": "candidates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def spawn(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: re-launch this command under
    torch.distributed.run with N local ranks (one per GPU, 127.0.0.1
    rendezvous), the way the driver launches it; rank 0 prints the line."""
    import socket
    import subprocess
    import torch
    have = torch.cuda.device_count()
    if have < n:
        print(json.dumps({"metric": METRIC, "error": "--gpus %d but only %d visible GPU(s)" % (n, have)}),
              flush=True)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--precision", default=os.environ.get("TLP_BENCH_PRECISION", "bf16"),
                    choices=["bf16", "fp32"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--chunks", type=int, default=16, help="tlp_search_round chunks (e2e leg)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn(args.gpus))
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        print("bench.py: --gpus %d but WORLD_SIZE=%s; measuring WORLD_SIZE ranks"
              % (args.gpus, os.environ["WORLD_SIZE"]), file=sys.stderr)
    if int(os.environ.get("WORLD_SIZE", "1")) > 1:
        # NCCL's algorithm / protocol choice (NVLS, ring, tree) for the scaling record
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,TUNING")
        logdir = os.path.join(ROOT, "gpurun_out")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(
            logdir if os.path.isdir(logdir) else "/tmp", "nccl_bench.%h.%p.log"))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
