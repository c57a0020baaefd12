"""Shared parity helpers: replay a GPU run's captured batches through the CPU oracle.

Used by the -m gpu parity tests and by __graft_entry__.smoke().  The oracle is only the
checker here.
"""

from __future__ import annotations

import gzip
import json
import os
from typing import Dict, List, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

# logits tolerance (north_star: "max-abs <= 2e-2"), on the tiny config's logits (std ~0.5)
LOGIT_ATOL = 2e-2


def load_golden(name: str) -> Dict:
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as fh:
        return json.load(fh)


def golden_trace(E, g: Dict):
    slo = E.SloSpec(*g["slo"])
    reqs = tuple(E.RequestSpec(rid, t, tuple(imgs), p, o, slo)
                 for rid, t, imgs, p, o in g["requests"])
    return E.Trace(reqs, name=g["name"])


def normalise(log) -> List:
    return json.loads(json.dumps(log))


def oracle_replay(cluster, shape, seed: int, max_batches: int = None) -> Dict:
    """Replay every captured batch of every instance (in global order) on the oracle.

    Teacher forcing: decode inputs are the GPU's own previous tokens, so both sides stay
    on the same sequence.  Returns per-row logit errors and token agreement stats."""
    from oracle.mllm_fp32 import OracleMLLM
    from paper_2505_12658_b200.inputs import prompt_tokens
    from paper_2505_12658_b200.weights import weight_specs

    oracle = OracleMLLM(shape.asdict(), weight_specs(shape), seed)
    # the runtimes append in global batch order per instance; merge by the global order
    # recorded in cluster.exec_order
    last_tok: Dict[str, int] = {}
    max_err = 0.0
    n_rows = n_tok_equal = n_near_tie = 0
    worst = None
    entries = cluster.exec_order
    if max_batches is not None:
        entries = entries[:max_batches]
    for iid, idx in entries:
        e = cluster.runtimes[iid].exec_log[idx]
        reqs = cluster.reqs
        # encode: each image's rows appended to the request's image rows
        for rid, k, first in e["encode"]:
            counts = reqs[rid].spec.image_token_counts
            for ii in range(first, first + k):
                gh, gw = shape.patch_grid(counts[ii])
                px = cluster.images.request_image(rid, ii, gh, gw)
                oracle.add_image_rows(rid, oracle.encode_image(px, gh, gw))
        outs = {}
        for rid, kv_len in e["decode"]:
            outs[rid] = oracle.decode(rid, last_tok[rid], kv_len)
        for rid, c, o in e["prefill"]:
            r = reqs[rid]
            prompt = prompt_tokens(seed, rid, r.spec.prompt_tokens, shape.vocab)
            lg = oracle.prefill_chunk(rid, prompt, r.plan.visual_tokens, o, c)
            if o + c >= r.plan.prefill_total_tokens:
                outs[rid] = lg
        for j, rid in enumerate(e["out_rids"]):
            ref = outs[rid].numpy()
            got = e["logits"][j]
            err = float(np.abs(ref - got).max())
            if err > max_err:
                max_err, worst = err, (iid, idx, rid)
            tok = int(e["tokens"][j])
            n_rows += 1
            ref_tok = int(ref.argmax())
            if tok == ref_tok:
                n_tok_equal += 1
            elif ref[ref_tok] - ref[tok] <= 2 * LOGIT_ATOL:
                n_near_tie += 1  # documented near-tie: the two candidates are within tolerance
            last_tok[rid] = tok
    return {"max_abs_err": max_err, "rows": n_rows, "tokens_equal": n_tok_equal,
            "near_ties": n_near_tie, "worst": worst}
