"""Pins for oracle O1 (tokenizer), against what the paper and SPEC fix."""
import json
import os

import numpy as np
import pytest

import synth
from oracle import tokenizer as tk

HERE = os.path.dirname(__file__)


def f32bits(x):
    return "0x%08X" % np.float32(x).view(np.uint32)


# --- SPEC worked vectors, cfg num_types=3 [SP,RE,FU], E=8 -------
SP3, RE3, FU3 = 0, 1, 2
TT = {"i0": 2, "i1": 3}


def test_spec_embed_primitive_vectors():
    row = lambda p: tk.extract_rows([p], TT, 1, 8, 3)[0]  # noqa: E731
    assert row((SP3, [4.0, 8.0])).tolist() == [1, 0, 0, 4, 8, 0, 0, 0]
    assert row((RE3, ["i0"])).tolist() == [0, 1, 0, 2, 0, 0, 0, 0]
    assert row((FU3, [1.0, 2.0, 3.0, 4.0, 5.0, 6.0])).tolist() == [0, 0, 1, 1, 2, 3, 4, 5]


def test_spec_extract_features_pad_crop_determinism():
    seq2 = [(SP3, [1.0]), (RE3, [2.0])]
    X = tk.extract_rows(seq2, TT, 4, 8, 3)
    assert X.shape == (4, 8) and not X[2:].any() and X[:2].any()
    seq5 = [(SP3, [float(i)]) for i in range(5)]
    X5 = tk.extract_rows(seq5, TT, 4, 8, 3)
    assert X5[:, 3].tolist() == [0, 1, 2, 3]  # 5th primitive cropped (R4: keep head)
    assert np.array_equal(tk.extract_rows(seq5, TT, 4, 8, 3).view(np.uint32), X5.view(np.uint32))


def test_spec_token_table():
    assert tk.build_token_table(["i0", "i1", "i0"]) == {"i0": 2, "i1": 3}
    assert tk.build_token_table([]) == {}
    assert tk.extract_rows([(RE3, ["zz"])], TT, 1, 8, 3)[0, 3] == 1.0  # unknown -> 1


def test_spec_normalization():
    X = np.zeros((3, 1, 4), np.float32)
    X[:, 0, 1] = [0, 4, 8]
    X[1, 0, 0] = 1.0  # one-hot-like column
    s = tk.fit_scales(X)
    assert s.tolist() == [1.0, 8.0, 1.0, 1.0]
    assert (X[1, 0] / s)[1] == 0.5


def test_derived_worked_example_bits():
    g = json.load(open(os.path.join(HERE, "golden", "tokenizer_worked_example.json")))
    reg = {n: i for i, n in enumerate(g["registry"])}
    seq = [(reg[t], [a if isinstance(a, str) else float(a) for a in args]) for t, args in g["sequence"]]
    tokens = tk.build_token_table([a for _, args in seq for a in args if isinstance(a, str)])
    assert tokens == g["tokens"]
    raw = tk.extract_rows(seq, tokens, 25, 22, 11)
    expect = np.zeros((25, 22), np.float32)
    for r, cols in g["unnormalized_nonzeros"].items():
        for c, v in cols.items():
            expect[int(r), int(c)] = v
    assert np.array_equal(raw, expect)
    scale = tk.fit_scales(raw[None])
    exp_scale = np.ones(22, np.float32)
    for c, v in g["scales_nonunit"].items():
        exp_scale[int(c)] = v
    assert np.array_equal(scale, exp_scale)
    X = tk.encode([seq], tokens, scale)[0]
    for rc, bits in g["normalized_bits_nonunit"].items():
        r, c = map(int, rc.split(","))
        assert f32bits(X[r, c]) == bits
    special = {tuple(map(int, k.split(","))) for k in g["normalized_bits_nonunit"]}
    for r, c in zip(*np.nonzero(X)):
        if (r, c) not in special:
            assert X[r, c] == 1.0
    assert not X[5:].any()


def test_re_crop_keeps_first_11_args():
    # tab 3_1_step_len: RE max embedding 40 = 11 + 29 args.
    seq = [(synth.RE, [float(i + 1) for i in range(29)])]
    X = tk.extract_rows(seq, {}, 25, 22, 11)
    assert X[0, 11:].tolist() == [float(i + 1) for i in range(11)]


def test_table_3_1_max_embedding_reproduced_by_generator():
    # Per-type max (11 + #args) over a large synthetic sample == tab 3_1_step_len.
    b = synth.generate(1, 60000)
    nargs = np.diff(b.arg_off)
    for t, name in enumerate(synth.TYPE_NAMES):
        m = b.prim_type == t
        assert 11 + nargs[m].max() == synth.TABLE_MAX_EMBED[name], name


def test_crop_safe_inverse_map_and_shape():
    rng = np.random.default_rng(3)
    tokens = {"a": 2, "b": 3, "c": 4}
    inv = {v: k for k, v in tokens.items()}
    for _ in range(300):
        n = int(rng.integers(1, 26))
        seq = []
        for _ in range(n):
            t = int(rng.integers(0, 11))
            args = []
            for _ in range(int(rng.integers(0, 12))):
                if rng.random() < 0.3:
                    args.append(["a", "b", "c"][int(rng.integers(0, 3))])
                else:
                    args.append(float(rng.integers(5, 1000)))  # >= 5: never a token value
            seq.append((t, args))
        X = tk.extract_rows(seq, tokens, 25, 22, 11)
        assert X.shape == (25, 22)
        rec = []
        for r in range(25):
            if not X[r].any():
                break
            t = int(np.argmax(X[r, :11]))
            vals = X[r, 11:]
            k = len(vals)
            while k > 0 and vals[k - 1] == 0:
                k -= 1
            rec.append((t, [inv[int(v)] if v < 5 else float(v) for v in vals[:k]]))
        assert rec == [(t, a) for t, a in seq]
    for L in range(1, 101, 9):
        seq = [(0, [1.0])] * L
        assert tk.extract_rows(seq, {}, 25, 22, 11).shape == (25, 22)


def test_errors_and_kept_only_validation():
    with pytest.raises(tk.TokenizeError) as e:
        tk.extract_rows([], {}, 25, 22, 11)
    assert e.value.code == "EMPTY_SEQ"
    with pytest.raises(tk.TokenizeError) as e:
        tk.extract_rows([(11, [])], {}, 25, 22, 11)
    assert e.value.code == "UNKNOWN_TYPE"
    with pytest.raises(tk.TokenizeError) as e:
        tk.extract_rows([(0, [float("nan")])], {}, 25, 22, 11)
    assert e.value.code == "NONFINITE"
    with pytest.raises(tk.TokenizeError):
        tk.extract_rows([(0, [1e300])], {}, 25, 22, 11)  # overflows fp32 -> non-finite
    # Beyond the crop nothing is read (R3/R4 "validation covers kept data only").
    seq = [(0, [1.0] * 11 + [float("nan")])] + [(0, [])] * 24 + [(99, [float("inf")])]
    tk.extract_rows(seq, {}, 25, 22, 11)


def test_synonym_distance_property():
    # same-type primitives with close params are close after normalisation.
    scale = np.full(22, 8.0, np.float32)
    scale[:11] = 1
    a = tk.encode([[(2, [1.0, 2.0, 4.0])]], {}, scale)[0, 0]
    b = tk.encode([[(2, [1.0, 2.0, 6.0])]], {}, scale)[0, 0]
    c = tk.encode([[(3, [1.0, 2.0, 4.0])]], {}, scale)[0, 0]
    assert np.isclose(np.linalg.norm(a - b), 2.0 / 8.0)
    assert (a[:11] != c[:11]).sum() == 2


def test_packed_roundtrip_and_generator_shape():
    b = synth.generate(7, 2000)
    lens = np.diff(b.seq_off)
    assert lens.min() >= 4 and lens.max() <= 54
    assert abs((lens == 21).mean() - 0.209) < 0.03
    assert (lens <= 25).mean() > 0.85
    seqs = b.to_lists()
    b2 = synth.pack(seqs)
    assert b2.to_lists() == seqs
