"""CPU oracle for the HydraInfer hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package, and only as the checker or the timed
CPU baseline; the product path (``paper_2505_12658_b200``) never imports it.

Contents
  batch_log.py   golden scheduler logs captured from the reference epdsim itself
                 (decisions, batch composition, migration jobs)  -- PINNED: the sha of
                 config 1 equals the value in BASELINE.md (033af48c14991898)
  block_alloc.py restatement of CachePool count semantics (engine.py:156-191) plus the
                 builder's lowest-id-first physical block policy -- PINNED on the
                 reference's own pool events
  synth.py       numpy restatement of the counter-hash weight synthesis (bit-exact)
  mllm_fp32.py   fp32 CPU restatement of the executed model (ViT + projector + Llama
                 decoder with chunked prefill over a per-request KV cache).  The
                 reference pins no tensor numerics (it ships no model code),
                 so for logits the parity is UNPINNED against the reference and pinned
                 only against this restatement.
"""
