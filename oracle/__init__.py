"""fp64 CPU oracle for the ragged transformer-encoder layer of CoRa (arXiv 2110.10221).

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import or execute
anything under `oracle/`.  The product path (`paper_2110_10221_b200`) never
imports it, and this package never imports the product path: the two share
no code.  The only shared module is `synth` (seeded input generators, which
hold none of the method's arithmetic).

Everything here is plain, slow, obviously-correct NumPy in float64, written
in the paper's order and notation.  Each function cites the passage it
follows (PAPER.md line numbers, section / equation / table).  Readings where
the paper is silent or garbled are the c1..c18 readings of DESIGN.md.

Pins (tests/test_oracle_*.py, run with `-m "not gpu"`):
  layout     -- SPEC.md worked examples (tests/golden/spec_examples.json),
                brute-force enumeration bijection, B.2 identities.
  tile list  -- brute-force sort of all (b,h,qt) by the stated key.
  attention  -- torch SDPA fp64 (B=1 reduces to textbook SDPA); padded+masked
                dense brute force; invariants (rows sum to 1, L=1 -> O=V);
                the row-at-a-time form (long sequences) against torch SDPA
                per sampled row, bidirectional and causal.
  softmax    -- SPEC example [0,0] -> [0.5,0.5]; shift invariance; sums.
  layernorm  -- torch.nn.functional.layer_norm fp64; closed-form moments.
  linear     -- pure-Python MAC loops on tiny inputs.
  layer      -- torch.nn.TransformerEncoderLayer fp64, per sequence and
                padded with src_key_padding_mask.
  flops      -- instrumented MAC counts == closed form; SPEC [2,4] -> 32/20.
  shard plan -- exhaustive search over all contiguous partitions (tiny B).
  vgemm/trmm -- pure-Python triple loops on tiny problems (row i of trmm
                reduces over k <= i only); identity / zero-padding cases;
                instrumented MAC counts == the FLOP closed forms.
No function here is "parity unpinned".
"""
from .layout import (  # noqa: F401
    row_offsets,
    attn_offsets,
    fusion_maps,
    packed_offset,
    attn_offset,
    attn_total_size,
    tile_list,
    unit_list,
    short_windows,
    packed_tile_list,
    packed_unit_list,
    n_tiles,
    validate_lengths,
    STATUS_OK,
    STATUS_BAD_LENGTH,
    STATUS_SUM_MISMATCH,
)
from .encoder import (  # noqa: F401
    linear,
    layernorm,
    softmax_row,
    ragged_softmax,
    ragged_attention,
    ragged_attention_rows,
    attention_scores_ragged,
    encoder_layer,
    relu,
    gelu_erf,
)
from .flops import useful_flops, padded_flops, useful_macs_bruteforce, padded_macs_bruteforce, qkt_macs, causal_attention_flops  # noqa: F401
from .shard import shard_cost, shard_plan  # noqa: F401
from .matmul import vgemm, trmm, vgemm_flops, vgemm_padded_flops, trmm_flops  # noqa: F401
