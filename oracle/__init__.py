"""CPU oracle for the TLP / MTL-TLP hot path (arXiv 2211.03578).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2211_03578_b200``) never imports it and
shares no code with it: no kernels, headers, helpers, tables or constants.

Plain, slow, obviously-correct NumPy, float64 everywhere except where the
contract fixes fp32 (the tokenizer output, P:239 + SURVEY §8(c) R3/R5, and
label rounding, O6).  Each function cites the PAPER.md passage (``P:n``) it
follows and the reading (``R#``, SURVEY.md §8(c) / DESIGN.md "Readings") it
takes where the paper is silent.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``):
  tokenizer  -- SPEC worked vectors, derived worked example with hex bits,
                crop-safety inverse map, shape invariant.
  forward    -- torch fp64 nn.MultiheadAttention / nn.Linear re-implementation,
                permutation invariance, zero weights, Wq=Wk=0 closed form,
                pad-row identity, head-order identity (R13).
  backward   -- central finite differences, torch autograd (fp64).
  lambdarank -- brute-force |dNDCG| by swapping, finite differences, derived
                values, tie / single-pair cases.
  MTL        -- R19 discriminating example, head separation, additivity.
  topk       -- full stable sort by brute force, shard merge.
  labels     -- SPEC example, range (0,1], one label == 1 per group.
  adam       -- torch.optim.Adam.
  dp         -- R-rank emulation equals the unsharded step.
  dataset    -- (NEXT-2) SPEC duplicate-rate / dedup / top-k-score examples,
                brute-force pairwise classes, permutation invariance.
  search     -- (NEXT-1) Philox4x64-10 == numpy's Philox; fitness-proportional
                selection by enumeration; SPEC genetic-operator properties;
                cheating model finds the brute-force optimum; constant model
                == random search; tuner budget / monotonicity invariants.
"""
from .tokenizer import build_token_table, extract_rows, fit_scales, encode  # noqa: F401
from .model import Config, param_shapes, unflatten, flatten, forward, backward  # noqa: F401
from .rank_loss import lambdarank, strict_pair_counts, mtl_lambdarank  # noqa: F401
from .select import topk, normalize_labels  # noqa: F401
from .optim import adam_step, AdamState  # noqa: F401
from .dp import dp_emulate  # noqa: F401
from .dataset import feature_classes, duplicate_rate, dedup_labels, topk_score  # noqa: F401
