"""ORACLE — test infrastructure only.  NOT part of the product path.

A CPU (numpy) restatement of the reference `shardsim` algorithm for the FSDP
sharded-training hot path (flatten/pad/shard, all-gather, reduce-scatter,
hybrid RS->AR, gradient write-back, /W post-divide + accumulation, the sharded
gradient scaler and SGD/Adam on shards).  Every function cites the reference
file:line it restates (paths are relative to the reference's
`pkg/src/shardsim/`).

Who may import this package (and nothing else may):
  * `tests/`                       — as the parity checker;
  * `__graft_entry__.smoke()`      — as the checker of one small invocation;
  * `bench.py`                     — only the `cpu_baseline` leg and the
                                     `--impl reference` arm (CPU timing).
The CUDA product path in `paper_2304_11277_b200/` never imports, calls or
falls back to this package; it fails loudly when its extension is missing.

Parity is PINNED: `tests/golden/make_golden.py` imports the real reference
(`/root/reference/pkg/src`, only available in the build container) and writes
golden vectors under `tests/golden/`; `tests/test_oracle_golden.py` checks this
restatement against them bit-for-bit with the reference's own dtypes
(full = float64, low = float32).  The B200 build runs the same algorithm with
full = float32 (master/optimizer/accumulation) and low = bfloat16 (gathered
parameters, gradient payloads); the restatement is dtype-parameterised so the
identical code defines the GPU's expected outputs.
"""
from .bf16 import bf16_bits_to_f32, f32_to_bf16_bits, round_to_bf16  # noqa: F401
from . import shardsim_port  # noqa: F401
