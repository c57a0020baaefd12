"""Regenerate the golden fixtures in tests/golden/ from the reference epdsim.

Run in the build container (where /root/reference exists):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py
The fixtures are committed; tests never read /root/reference at run time.

Each fixture holds the reference's own scheduler output for one config -- batch log
(BASELINE.md section 2 recipe), migration jobs, pool events -- plus the reference
aggregates, captured by oracle/batch_log.py.
"""

from __future__ import annotations

import gzip
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import epdsim as E  # noqa: E402
from epdsim.cluster import ClusterSpec, DisaggregationMethod, pool_capacities  # noqa: E402

from oracle.batch_log import capture, digest  # noqa: E402

TRACES = "/root/reference/pkg/traces"
TINY = dict(lang_hidden=512, lang_heads=4, lang_layers=2, vision_hidden=256, vision_heads=4,
            vision_layers=2)
QWEN = dict(lang_hidden=3584, lang_heads=28, lang_layers=28, vision_hidden=1280,
            vision_heads=16, vision_layers=32, kv_head_ratio=4 / 28)
SLO = E.SloSpec(4.0, 0.08)


def hw_b200():
    return E.HardwareProfile(2.25e15, 8.0e12, 160e9, 14e9, 900e9)


def mixed32():
    tr = E.load_trace(os.path.join(TRACES, "mixed_small.jsonl"), default_slo=SLO)
    return E.Trace(tr.requests[:32], name="mixed_small32")


def write(name, obj):
    path = os.path.join(HERE, name + ".json.gz")
    with gzip.open(path, "wt") as fh:
        json.dump(obj, fh, sort_keys=True)
    print(f"wrote {path}")


def config(name, method, model, hw, slo, trace, *, trace_desc, model_desc, policy=None,
           spec_overrides=None):
    spec = ClusterSpec(method=DisaggregationMethod.parse(method),
                       **({"policy": policy} if policy else {}), **(spec_overrides or {}))
    cap = capture(E, spec, model, hw, slo, trace)
    caps = {}
    for itype, count in spec.method.counts:
        kvb, imb = pool_capacities(itype, model, hw, spec.image_pool_fraction)
        for i in range(count):
            caps[f"{itype.name}{i}"] = [kvb, imb]
    out = {
        "name": name, "method": method, "model": model_desc, "trace": trace_desc,
        "policy": spec.policy, "spec_overrides": spec_overrides or {},
        "hw": [hw.peak_flops, hw.mem_bandwidth, hw.gpu_memory_bytes, hw.model_weight_bytes,
               hw.interconnect_bandwidth],
        "slo": [slo.ttft_max, slo.tbt_max],
        "requests": [[r.id, r.arrival_time, list(r.image_token_counts), r.prompt_tokens,
                      r.output_tokens] for r in trace.requests],
        "n_batches": len(cap["batches"]), "sha": digest(cap["batches"]),
        "batches": cap["batches"], "migrations": cap["migrations"],
        "pool_events": cap["pool_events"], "capacities": caps,
        "aggregates": cap["aggregates"],
    }
    write(name, out)
    return out


def main():
    tiny = E.ModelProfile(**TINY)
    base = mixed32()
    fast = E.scale_to_rate(base, 2000.0)
    c1 = config("config1_native", "EPD:1", tiny, E.DEFAULT_HARDWARE, SLO, base,
                trace_desc="mixed_small.jsonl[:32] native rate", model_desc=TINY)
    assert c1["sha"] == "033af48c14991898", c1["sha"]
    config("config1_2000rps", "EPD:1", tiny, E.DEFAULT_HARDWARE, SLO, fast,
           trace_desc="mixed_small.jsonl[:32] scaled to 2000 req/s", model_desc=TINY)
    for method in ("EP:1,D:1", "E:1,P:1,D:1", "E:1,PD:1"):
        config("tiny_" + method.replace(":", "").replace(",", "_"), method, tiny,
               E.DEFAULT_HARDWARE, SLO, fast,
               trace_desc="mixed_small.jsonl[:32] scaled to 2000 req/s", model_desc=TINY)
    qwen = E.ModelProfile(**QWEN)
    dyn = E.synth_trace(seed=5, n_requests=12, rate=50.0, image_count_dist=[0, 1, 2],
                        visual_token_choices=[256, 576, 1024], prompt_dist=[20, 60],
                        output_dist=[8, 16], slo=E.SloSpec(8.0, 0.10))
    config("qwen_EP1_D1", "EP:1,D:1", qwen, hw_b200(), E.SloSpec(8.0, 0.10), dyn,
           trace_desc="synth_trace(seed=5, n=12, rate=50, images [0,1,2] x [256,576,1024], "
                      "prompt [20,60], output [8,16])", model_desc=QWEN)
    # baseline scheduling policies (engine.py:406-497): whole-prompt prefills, decodes
    # first / unbudgeted encodes -- the executor must run their batches too
    # (a burst -- 32 requests in 0.3 ms -- with budget ceilings of 512 tokens / 2 images, so
    # the three policies form different batches: stage-level caps encodes at 2 images,
    # stall-free encodes up to 22 at once, prefill-prioritized runs whole 1242-token prompts)
    burst = E.scale_to_rate(base, 1e5)
    tight = {"token_budget_ceiling": 512, "image_budget_ceiling": 2}
    for pol in ("stage_level", "prefill_prioritized", "stall_free_chunked"):
        config("config1_burst_" + pol, "EPD:1", tiny, E.DEFAULT_HARDWARE, SLO, burst,
               policy=pol, spec_overrides=tight, model_desc=TINY,
               trace_desc="mixed_small.jsonl[:32] scaled to 1e5 req/s; ceilings 512 / 2")
    # the bench config's model (LLaVA-1.5-7B profile, B200 hardware): decisions of the
    # full-size model, executed at full width with reduced depth by the GPU parity tests
    llava = E.MODEL_PRESETS["llava-1.5-7b"]
    cap = E.load_trace(os.path.join(TRACES, "captioning_medium.jsonl"), default_slo=SLO)
    cap24 = E.scale_to_rate(E.Trace(cap.requests[:24], name="captioning_medium24"), 2000.0)
    for method in ("EPD:1", "EP:1,D:1"):
        config("llava_" + method.replace(":", "").replace(",", "_"), method, llava, hw_b200(),
               SLO, cap24, trace_desc="captioning_medium.jsonl[:24] scaled to 2000 req/s",
               model_desc="llava-1.5-7b")
    # multi-image high-resolution stress (BASELINE config 5 shape, workload.py:234-264):
    # 4 images x ~2.9k tokens, prompts 1-2k, contexts to ~14k tokens, PD jobs of ~870 blocks
    stress = E.synth_trace(seed=21, n_requests=3, rate=2.0, image_count_dist=4,
                           visual_token_choices=[2800, 2900, 3000], prompt_dist=[1000, 2000],
                           output_dist=[64, 128], slo=SLO)
    config("llava_stress_EP1_D1", "EP:1,D:1", llava, hw_b200(), SLO, stress,
           trace_desc="synth_trace(seed=21, n=3, rate=2, 4 images x [2800,2900,3000], "
                      "prompt [1000,2000], output [64,128])", model_desc="llava-1.5-7b")
    # known answers from the reference's own tests
    ka = {
        "llava_kv_bytes_per_token": llava.kv_bytes_per_token,           # test_model_cost.py:197
        "llava_image_bytes_576": E.image_cache_bytes(576, llava),         # test_migration.py:28-30
        "llava_kv_bytes_616": E.kv_cache_bytes(616, llava),               # test_migration.py:32-34
        "kv_blocks_needed": {str(t): E.kv_blocks_needed(t) for t in (0, 1, 15, 16, 17, 616, 617)},
        "image_blocks_needed": {str(t): E.image_blocks_needed(t) for t in (0, 1, 576, 577, 2900)},
        "b200_pool_capacities_llava": {
            t: list(pool_capacities(E.InstanceType(t), llava, hw_b200(), 0.1))
            for t in ("E", "P", "D", "EP", "ED", "PD", "EPD")},
    }
    write("known_answers", ka)


if __name__ == "__main__":
    main()
