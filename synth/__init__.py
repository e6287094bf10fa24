"""Seeded synthetic TenSet-shaped inputs shared by the oracle tests, the GPU
parity tests and bench.py.

This module holds NONE of the method's arithmetic (no one-hot, no token
assignment, no normalisation, no model math).  It only draws abstract
schedule-primitive sequences (fig 3_1_feature_extraction_abstract
(a): ``S ::= p*``, ``p ::= tau (id | num)*``) and packs them into the
structure-of-arrays layout the C-ABI consumes (include/tlp.h, ``tlp_seq_batch``).

Recipe (restated in DESIGN.md "Input recipe"):

* lengths: with p=0.209 len=21 (the paper's mode, 1,807,960 of 8.65M programs,
  P:273); with p=0.001 len~U{26..54} (the paper's maximum 54); otherwise
  clip(rint(exp(N(ln 20, 0.20^2))), 4, 54) redrawn while ==21.
* types: the 11 Ansor CPU primitive types in the registry order of
  tab 3_1_step_len; per-type maximum argument counts equal the
  table's maximum embedding size minus the 11-wide one-hot.
* arguments: TVM auto_scheduler step-record templates (outside knowledge; it
  only shapes synthetic data).  Names: pragma / scope strings, 1% unseen.
* groups ("subgraphs"): sizes from dozens to 4,000.
* latencies: a smooth log-linear function of the RAW arguments (not of the
  encoded features) times a per-group base, so labels are learnable but the
  generator never calls the method.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Sequence, Tuple, Union

import numpy as np

# Registry order R6: tab 3_1_step_len order.
TYPE_NAMES = ("RE", "FU", "SP", "FSP", "CA", "AN", "RF", "PR", "CHW", "CR", "CI")
T_DEFAULT = len(TYPE_NAMES)
RE, FU, SP, FSP, CA, AN, RF, PR, CHW, CR, CI = range(11)

# Max embedding sizes of tab 3_1_step_len; args = value - 11.
TABLE_MAX_EMBED = {"RE": 40, "FU": 22, "SP": 18, "FSP": 15, "CA": 14, "AN": 14,
                   "RF": 14, "PR": 14, "CHW": 13, "CR": 12, "CI": 12}

# Per-sequence type frequencies (a proposal; paper gives none).
TYPE_WEIGHTS = {"SP": .30, "AN": .15, "FU": .12, "RE": .08, "FSP": .08, "CA": .07,
                "CI": .07, "PR": .05, "CHW": .03, "CR": .03, "RF": .02}

PRAGMAS = tuple("auto_unroll_max_step$%d" % v for v in (0, 16, 64, 512, 1024))
SCOPES = ("local", "global", "shared")
UNSEEN_RATE = 0.01

Arg = Union[float, str]
Prim = Tuple[int, List[Arg]]


@dataclass
class PackedBatch:
    """SoA layout of ``tlp_seq_batch`` (include/tlp.h).  All arrays host numpy."""
    seq_off: np.ndarray    # int64 [N+1]
    prim_type: np.ndarray  # uint8 [P]
    arg_off: np.ndarray    # int64 [P+1]
    arg_kind: np.ndarray   # uint8 [A]  0 = Number, 1 = NameParam
    arg_num: np.ndarray    # float64 [A]
    arg_name: np.ndarray   # int32 [A]  index into strings (or -1 for numbers)
    strings: List[str] = field(default_factory=list)  # batch string table

    @property
    def N(self) -> int:
        return len(self.seq_off) - 1

    @property
    def P(self) -> int:
        return len(self.prim_type)

    @property
    def A(self) -> int:
        return len(self.arg_kind)

    def str_blob(self) -> Tuple[np.ndarray, np.ndarray]:
        """UTF-8 blob (uint8) and int64 offsets [U+1] for the batch string table."""
        enc = [s.encode("utf-8") for s in self.strings]
        off = np.zeros(len(enc) + 1, dtype=np.int64)
        if enc:
            off[1:] = np.cumsum([len(e) for e in enc])
        blob = np.frombuffer(b"".join(enc), dtype=np.uint8).copy() if enc else np.zeros(0, np.uint8)
        return blob, off

    def to_lists(self) -> List[List[Prim]]:
        """Unpack to the abstract form [(type_id, [num | name, ...]), ...] per candidate."""
        out: List[List[Prim]] = []
        for n in range(self.N):
            seq: List[Prim] = []
            for p in range(int(self.seq_off[n]), int(self.seq_off[n + 1])):
                args: List[Arg] = []
                for a in range(int(self.arg_off[p]), int(self.arg_off[p + 1])):
                    if self.arg_kind[a] == 1:
                        args.append(self.strings[int(self.arg_name[a])])
                    else:
                        args.append(float(self.arg_num[a]))
                seq.append((int(self.prim_type[p]), args))
            out.append(seq)
        return out

    def slice(self, lo: int, hi: int) -> "PackedBatch":
        """Candidates [lo, hi) as a new packed batch (string table kept whole)."""
        p0, p1 = int(self.seq_off[lo]), int(self.seq_off[hi])
        a0, a1 = int(self.arg_off[p0]), int(self.arg_off[p1])
        return PackedBatch(self.seq_off[lo:hi + 1] - p0, self.prim_type[p0:p1].copy(),
                           self.arg_off[p0:p1 + 1] - a0, self.arg_kind[a0:a1].copy(),
                           self.arg_num[a0:a1].copy(), self.arg_name[a0:a1].copy(),
                           list(self.strings))


def pack(seqs: Sequence[Sequence[Prim]]) -> PackedBatch:
    """Pack abstract sequences into the SoA layout (string table = first-seen order)."""
    seq_off = [0]
    prim_type: List[int] = []
    arg_off = [0]
    kind: List[int] = []
    num: List[float] = []
    name: List[int] = []
    strings: List[str] = []
    sidx = {}
    for seq in seqs:
        for t, args in seq:
            prim_type.append(t)
            for a in args:
                if isinstance(a, str):
                    if a not in sidx:
                        sidx[a] = len(strings)
                        strings.append(a)
                    kind.append(1); num.append(0.0); name.append(sidx[a])
                else:
                    kind.append(0); num.append(float(a)); name.append(-1)
            arg_off.append(len(kind))
        seq_off.append(len(prim_type))
    return PackedBatch(np.asarray(seq_off, np.int64), np.asarray(prim_type, np.uint8),
                       np.asarray(arg_off, np.int64), np.asarray(kind, np.uint8),
                       np.asarray(num, np.float64), np.asarray(name, np.int32), strings)


# ----------------------------------------------------------------------------
# Vectorised generator
# ----------------------------------------------------------------------------

def draw_lengths(rng: np.random.Generator, n: int) -> np.ndarray:
    """Sequence lengths with the paper's constraints: max 54, mode 21."""
    u = rng.random(n)
    out = np.empty(n, np.int64)
    mode = u < 0.209
    tail = (u >= 0.209) & (u < 0.210)
    rest = ~(mode | tail)
    out[mode] = 21
    out[tail] = rng.integers(26, 55, int(tail.sum()))
    idx = np.nonzero(rest)[0]
    while idx.size:
        v = np.clip(np.rint(np.exp(rng.normal(np.log(20.0), 0.20, idx.size))), 4, 54).astype(np.int64)
        ok = v != 21
        out[idx[ok]] = v[ok]
        idx = idx[~ok]
    return out


def _arg_counts(rng: np.random.Generator, types: np.ndarray) -> np.ndarray:
    n = np.empty(types.size, np.int64)
    lo_hi = {RE: (3, 29), FU: (3, 11), SP: (5, 7), FSP: (4, 4), CA: (3, 3), AN: (3, 3),
             RF: (3, 3), PR: (3, 3), CHW: (2, 2), CR: (1, 1), CI: (1, 1)}
    for t, (lo, hi) in lo_hi.items():
        m = types == t
        k = int(m.sum())
        if k:
            n[m] = rng.integers(lo, hi + 1, k)
    return n


def generate(seed: int, n: int, *, min_len: int = 1, max_len: int = 54,
             unseen_rate: float = UNSEEN_RATE, lengths: np.ndarray | None = None) -> PackedBatch:
    """Draw ``n`` TenSet-shaped candidates; fully vectorised."""
    rng = np.random.default_rng(seed)
    if lengths is None:
        lengths = np.clip(draw_lengths(rng, n), min_len, max_len)
    lengths = np.asarray(lengths, np.int64)
    P = int(lengths.sum())
    wt = np.array([TYPE_WEIGHTS[t] for t in TYPE_NAMES], np.float64)
    types = rng.choice(len(TYPE_NAMES), size=P, p=wt / wt.sum()).astype(np.uint8)
    nargs = _arg_counts(rng, types)
    A = int(nargs.sum())
    arg_off = np.zeros(P + 1, np.int64)
    np.cumsum(nargs, out=arg_off[1:])
    prim_of = np.repeat(np.arange(P), nargs)
    pos = np.arange(A) - arg_off[prim_of]
    last = pos == (nargs[prim_of] - 1)
    ty = types[prim_of]

    small = rng.integers(0, 17, A).astype(np.float64)           # stage / iter ids
    extent = 2.0 ** rng.integers(0, 11, A)                      # loop extents
    factor = 2.0 ** rng.integers(0, 7, A)                       # split factors
    enum6 = rng.integers(0, 6, A).astype(np.float64)
    nsplit = rng.integers(1, 5, A).astype(np.float64)
    boolv = rng.integers(0, 2, A).astype(np.float64)

    num = small.copy()
    m = (ty == SP) & (pos == 2); num[m] = extent[m]
    m = (ty == SP) & (pos >= 3) & ~last; num[m] = factor[m]
    m = (ty == SP) & last; num[m] = boolv[m]
    m = (ty == AN) & (pos == 2); num[m] = enum6[m]
    m = (ty == FSP) & (pos == 3); num[m] = nsplit[m]

    is_name = ((ty == PR) & (pos == 2)) | ((ty == CHW) & (pos == 1))
    kind = is_name.astype(np.uint8)
    names_idx = np.nonzero(is_name)[0]
    strings: List[str] = []
    arg_name = np.full(A, -1, np.int32)
    if names_idx.size:
        vocab = list(PRAGMAS) + list(SCOPES)
        pr = ty[names_idx] == PR
        pick = np.where(pr, rng.integers(0, len(PRAGMAS), names_idx.size),
                        len(PRAGMAS) + rng.integers(0, len(SCOPES), names_idx.size))
        unseen = rng.random(names_idx.size) < unseen_rate
        uid = rng.integers(0, 1 << 20, names_idx.size)
        labels = [("unseen_%d" % uid[i]) if unseen[i] else vocab[pick[i]] for i in range(names_idx.size)]
        table = {}
        for i, s in zip(names_idx, labels):
            j = table.get(s)
            if j is None:
                j = table[s] = len(strings)
                strings.append(s)
            arg_name[i] = j
    num[is_name] = 0.0
    seq_off = np.zeros(n + 1, np.int64)
    np.cumsum(lengths, out=seq_off[1:])
    return PackedBatch(seq_off, types, arg_off, kind, num, arg_name, strings)


def training_stream(seed: int = 12345, n: int = 2000) -> List[str]:
    """Names in first-occurrence order over a seeded 'training split' (no unseen names)."""
    b = generate(seed, n, unseen_rate=0.0)
    order: List[str] = []
    seen = set()
    for a in np.nonzero(b.arg_kind == 1)[0]:
        s = b.strings[int(b.arg_name[a])]
        if s not in seen:
            seen.add(s)
            order.append(s)
    return order


def group_sizes(seed: int, n_groups: int, lo: int = 24, hi: int = 4000,
                mean: float = 3500.0) -> np.ndarray:
    """Subgraph sizes 'from dozens to 4,000' with the requested mean."""
    rng = np.random.default_rng(seed)
    # Beta-shaped mass near the top of the range; clipped to [lo, hi].
    a = (mean - lo) / (hi - lo)
    conc = 6.0
    x = rng.beta(a * conc, (1 - a) * conc, n_groups)
    return np.clip(np.rint(lo + x * (hi - lo)), lo, hi).astype(np.int64)


def latencies(batch: PackedBatch, group_off: np.ndarray, seed: int,
              task_noise: float = 0.0) -> np.ndarray:
    """Synthetic latencies: base_g * exp(w . phi(raw args)).  phi uses raw values only."""
    rng = np.random.default_rng(seed)
    P = batch.P
    w_type = rng.normal(0.0, 0.3, T_DEFAULT) + task_noise * rng.normal(0.0, 1.0, T_DEFAULT)
    nargs = np.diff(batch.arg_off)
    first = np.zeros(P)
    has = nargs > 0
    first[has] = batch.arg_num[batch.arg_off[:-1][has]]
    contrib = w_type[batch.prim_type] * np.log1p(np.abs(first)) / 4.0
    per_cand = np.add.reduceat(contrib, batch.seq_off[:-1]) if P else np.zeros(batch.N)
    per_cand = np.where(np.diff(batch.seq_off) > 0, per_cand, 0.0)
    lens = np.diff(batch.seq_off).astype(np.float64)
    per_cand = per_cand + 0.05 * lens + 1e-3 * rng.normal(size=batch.N)
    G = len(group_off) - 1
    base = 10.0 ** rng.uniform(-4, -2, G)
    gid = np.repeat(np.arange(G), np.diff(group_off))
    return base[gid] * np.exp(per_cand)


def uniform_task_off(T: int, per_task: int) -> np.ndarray:
    return (np.arange(T + 1, dtype=np.int64) * per_task)


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32/fp64 values to the nearest bf16-representable value (RNE).
    Used only to make synthetic weights bf16-representable."""
    f = np.asarray(x, np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = ((u + 0x7FFF + lsb) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).astype(np.float64)


def init_params(seed: int, shapes: Sequence[Tuple[str, Tuple[int, ...]]],
                bf16: bool = True, scale: float = 1.0) -> List[np.ndarray]:
    """Seeded Kaiming-uniform-style init for a list of (name, shape) entries.
    Weights [in,out] get U(-1/sqrt(in), 1/sqrt(in)); biases likewise with fan_in
    of the preceding weight."""
    rng = np.random.default_rng(seed)
    out = []
    fan = 1
    for name, shp in shapes:
        if len(shp) == 2:
            fan = shp[0]
        b = scale / np.sqrt(max(fan, 1))
        v = rng.uniform(-b, b, shp)
        out.append(bf16_round(v) if bf16 else v)
    return out


# ----------------------------------------------------------------------------
# Search-space templates for the synthetic Ansor-style round driver (SURVEY
# §8(f) NEXT-1; "SyntheticSubgraph" / "SyntheticOracle").
# Plumbing only: a template is a fixed skeleton sequence (the "sketch" Ansor
# derives for a subgraph by predefined rules) whose tunable arguments
# ("knobs": split factors, annotation enums, pragma strings) each take one
# value of a small domain.  A candidate is one domain index per knob (a gene
# vector).  The latency function stands in for the target hardware (P:558
# "measure the latency"); it is the SPEC's log-linear form with pairwise terms.
# ----------------------------------------------------------------------------

FACTOR_DOMAIN = tuple(float(2 ** i) for i in range(7))   # split factors 1..64
ANNOT_DOMAIN = tuple(float(i) for i in range(6))          # annotation enum
MAX_KNOBS = 64                                            # gene row width cap


@dataclass
class Template:
    """One subgraph's search space.  ``prims`` is the skeleton in the abstract
    form [(type, [num | name, ...])]; knob g replaces ``prims[knob_prim[g]]``'s
    argument ``knob_arg[g]`` by ``domains[g][gene]``."""
    prims: List[Prim]
    knob_prim: List[int]
    knob_arg: List[int]
    domains: List[Tuple[Arg, ...]]

    @property
    def G(self) -> int:
        return len(self.knob_prim)

    def dom_sizes(self) -> np.ndarray:
        return np.array([len(d) for d in self.domains], np.int64)

    def knob_groups(self) -> np.ndarray:
        """Ordinal of each knob's primitive among the knob-bearing primitives
        (the crossover unit: whole primitives)."""
        order = {p: i for i, p in enumerate(sorted(set(self.knob_prim)))}
        return np.array([order[p] for p in self.knob_prim], np.int64)


def make_template(seed: int, subgraph: int, min_len: int = 12, max_knobs: int = MAX_KNOBS) -> Template:
    """A seeded TenSet-shaped skeleton whose SP split factors, AN annotations
    and PR pragma strings are knobs."""
    rng = np.random.default_rng([seed, subgraph])
    L = int(np.clip(draw_lengths(rng, 1)[0], min_len, 54))
    seq = generate(int(rng.integers(0, 2 ** 31)), 1, unseen_rate=0.0, lengths=[L]).to_lists()[0]
    kp: List[int] = []
    ka: List[int] = []
    dom: List[Tuple[Arg, ...]] = []
    for p, (t, args) in enumerate(seq):
        slots: List[Tuple[int, Tuple[Arg, ...]]] = []
        if t == SP:
            slots = [(i, FACTOR_DOMAIN) for i in range(3, len(args) - 1)]
        elif t == AN:
            slots = [(2, ANNOT_DOMAIN)]
        elif t == PR:
            slots = [(2, PRAGMAS)]
        for i, d in slots:
            if len(kp) < max_knobs:
                kp.append(p); ka.append(i); dom.append(d)
    return Template(seq, kp, ka, dom)


def small_template(domain_sizes: Sequence[int]) -> Template:
    """A hand-built template with one SP factor knob per entry (domain = the
    first ``d`` split factors), e.g. (4, 4, 4) = a 64-point search space."""
    prims: List[Prim] = [(CHW, [0.0, "local"])]
    kp, ka, dom = [], [], []
    for d in domain_sizes:
        assert 1 <= d <= len(FACTOR_DOMAIN)
        kp.append(len(prims)); ka.append(3); dom.append(FACTOR_DOMAIN[:d])
        prims.append((SP, [float(len(prims)), 1.0, 64.0, 1.0, 0.0]))  # distinct stages: rows differ
    prims.append((AN, [0.0, 1.0, 2.0]))
    return Template(prims, kp, ka, dom)


def template_weights(seed: int, subgraph: int, G: int) -> Tuple[float, np.ndarray, np.ndarray]:
    """(base, w [G], v [G,G] upper-triangular) of the synthetic latency."""
    rng = np.random.default_rng([seed, subgraph, 7])
    base = float(10.0 ** rng.uniform(-4, -2))
    w = rng.normal(0.0, 1.0, G)
    v = np.triu(rng.normal(0.0, 0.5 / np.sqrt(max(G, 1)), (G, G)), 1)
    return base, w, v


def template_latency(tmpl: Template, genes: np.ndarray, seed: int, subgraph: int) -> np.ndarray:
    """Synthetic hardware: base * exp(w.g + sum_{j<l} v_jl g_j g_l)
    with g = gene / (|domain| - 1) in [0, 1].  > 0, deterministic."""
    genes = np.atleast_2d(np.asarray(genes, np.int64))
    base, w, v = template_weights(seed, subgraph, tmpl.G)
    D = tmpl.dom_sizes().astype(np.float64)
    g = genes[:, :tmpl.G] / np.maximum(D - 1.0, 1.0)
    return base * np.exp(g @ w + np.einsum("ni,ij,nj->n", g, v, g))


@dataclass
class PackedSpace:
    """Device layout of ``tlp_ga_space`` (include/tlp.h): S skeletons packed
    as one batch plus flat knob / domain tables.  Host numpy arrays."""
    tmpl: PackedBatch
    knob_off: np.ndarray   # int64 [S+1]
    knob_arg: np.ndarray   # int64 [K]  global argument index into tmpl's args
    knob_grp: np.ndarray   # int32 [K]  crossover group within the subgraph
    dom_off: np.ndarray    # int64 [K+1]
    dom_num: np.ndarray    # float64 [D]
    dom_name: np.ndarray   # int32 [D]  string index, -1 for a number

    @property
    def S(self) -> int:
        return len(self.knob_off) - 1

    @property
    def G(self) -> int:
        return int(np.diff(self.knob_off).max()) if self.S else 0


def pack_space(templates: Sequence[Template]) -> PackedSpace:
    strings: List[str] = []
    for t in templates:  # every domain string enters the batch string table
        for d in t.domains:
            for v in d:
                if isinstance(v, str) and v not in strings:
                    strings.append(v)
    b = pack([t.prims for t in templates])
    for s in b.strings:
        if s not in strings:
            strings.append(s)
    remap = np.array([strings.index(s) for s in b.strings] or [0], np.int32)
    arg_name = np.where(b.arg_name >= 0, remap[np.maximum(b.arg_name, 0)], -1).astype(np.int32)
    b = PackedBatch(b.seq_off, b.prim_type, b.arg_off, b.arg_kind, b.arg_num, arg_name, strings)
    knob_off = [0]; knob_arg = []; knob_grp = []; dom_off = [0]; dom_num = []; dom_name = []
    for s, t in enumerate(templates):
        grp = t.knob_groups()
        for g in range(t.G):
            p = int(b.seq_off[s]) + t.knob_prim[g]
            knob_arg.append(int(b.arg_off[p]) + t.knob_arg[g])
            knob_grp.append(int(grp[g]))
            for v in t.domains[g]:
                if isinstance(v, str):
                    dom_num.append(0.0); dom_name.append(strings.index(v))
                else:
                    dom_num.append(float(v)); dom_name.append(-1)
            dom_off.append(len(dom_num))
        knob_off.append(len(knob_arg))
    return PackedSpace(b, np.asarray(knob_off, np.int64), np.asarray(knob_arg, np.int64),
                       np.asarray(knob_grp, np.int32), np.asarray(dom_off, np.int64),
                       np.asarray(dom_num, np.float64), np.asarray(dom_name, np.int32))
