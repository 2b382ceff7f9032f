"""CPU oracle for SpecMemo's Medusa tree-verification hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_2506_01986_b200``) never imports it and the
two share no code; the only common module is ``synth`` (seeded inputs, no
method arithmetic).

Plain, slow, obviously-correct numpy (float64) implementation, written from
the paper (``/root/reference/PAPER.md``, cited as P:<line>) and the readings
recorded in DESIGN.md §3.

Modules
  tree    -- Medusa path-list trees: canonical order, ancestor mask, candidate
             paths (Eq. 2), R4 right-to-left pruning.
  model   -- random-init Llama decoder + Medusa-1 heads, one row at a time,
             with an optional bf16 storage-point emulation (rounding contract).
  spec    -- the speculative step: propose / verify / accept / compact
              and vanilla greedy decoding.
  sizing  -- Eq. 1 (KV bytes, with d) and Eq. 3 (runtime buffers).

Parity status per function is listed in DESIGN.md §3.3; functions whose
values are fixed only by invariants say so ("parity unpinned" for the raw
logit values and the typical-acceptance constants eps/alpha/T).
"""
