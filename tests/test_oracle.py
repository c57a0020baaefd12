"""CPU tests of the oracle itself: pinned against the reference's own outputs.

* the golden batch logs re-derive from the reference scheduler (sha of config 1 is the
  value recorded in BASELINE.md section 2);
* the known answers of the reference's tests (test_model_cost.py:196-204,
  test_migration.py:26-35) hold;
* the numpy weight synthesis is deterministic and matches its documented formula;
* the fp32 oracle model is self-consistent: chunked prefill == one-shot prefill, and
  decode-after-prefill == prefill of the longer sequence.
"""

import numpy as np
import pytest
import torch

from oracle import batch_log, synth
from paper_2505_12658_b200._epdsim import C, E
from parity_util import golden_trace, load_golden


@pytest.mark.parametrize("name", ["config1_native", "config1_2000rps", "tiny_EP1_D1",
                                  "tiny_E1_P1_D1", "tiny_E1_PD1", "qwen_EP1_D1"])
def test_golden_logs_rederive_from_reference(name):
    g = load_golden(name)
    prof = E.ModelProfile(**g["model"])
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(g["method"]))
    cap = batch_log.capture(E, spec, prof, E.HardwareProfile(*g["hw"]), E.SloSpec(*g["slo"]),
                            golden_trace(E, g))
    assert batch_log.digest(cap["batches"]) == g["sha"]
    assert [list(m) for m in cap["migrations"]] == g["migrations"]
    assert [list(e) for e in cap["pool_events"]] == g["pool_events"]


def test_config1_sha_is_baseline_value():
    assert load_golden("config1_native")["sha"] == "033af48c14991898"
    assert load_golden("config1_native")["n_batches"] == 3293


def test_known_answers():
    ka = load_golden("known_answers")
    assert ka["llava_kv_bytes_per_token"] == 524288
    assert ka["llava_image_bytes_576"] == 4718592
    assert ka["llava_kv_bytes_616"] == 322961408
    assert ka["kv_blocks_needed"] == {"0": 0, "1": 1, "15": 1, "16": 1, "17": 2, "616": 39,
                                      "617": 39}
    from paper_2505_12658_b200 import get_shape
    s = get_shape("llava-1.5-7b")
    assert s.kv_bytes_per_token == ka["llava_kv_bytes_per_token"]
    assert s.profile() == E.MODEL_PRESETS["llava-1.5-7b"]


def test_synth_formula_and_bf16_rounding():
    a = synth.uniform_tensor(0, 123, 4, 8, 1.0, 0.0)
    b = synth.uniform_tensor(0, 123, 4, 8, 1.0, 0.0)
    assert np.array_equal(a, b)
    assert np.all((a >= -1.0) & (a < 1.0))
    # every value is bf16-representable
    assert np.array_equal(synth.bf16_round(a), a)
    # a different tensor id gives different values
    assert not np.array_equal(a, synth.uniform_tensor(0, 124, 4, 8, 1.0, 0.0))
    # bf16 rounding: ties to even
    x = np.array([1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8], dtype=np.float32)
    assert synth.bf16_round(x).tolist() == [1.0, 1.0 + 2 ** -6]
    # swiglu interleave is a permutation
    rows = synth.swiglu_physical_rows(64)
    assert sorted(rows.tolist()) == list(range(64))
    assert rows[:16].tolist() == list(range(16)) and rows[16:32].tolist() == list(range(32, 48))


def test_oracle_chunked_prefill_and_decode_consistency():
    from oracle.mllm_fp32 import OracleMLLM
    from paper_2505_12658_b200 import get_shape, with_layers
    from paper_2505_12658_b200.weights import weight_specs
    shape = with_layers(get_shape("tiny"), 1, 1)
    o = OracleMLLM(shape.asdict(), weight_specs(shape), seed=3)
    prompt = np.arange(40, dtype=np.int32) * 7 % shape.vocab
    full = o.prefill_chunk("a", prompt, 0, 0, 40)
    o.prefill_chunk("b", prompt, 0, 0, 25)
    part = o.prefill_chunk("b", prompt, 0, 25, 15)
    assert torch.allclose(full, part, atol=1e-4)
    nxt = int(full.argmax())
    dec = o.decode("a", nxt, 40)
    prompt2 = np.concatenate([prompt, [nxt]]).astype(np.int32)
    ref = o.prefill_chunk("c", prompt2, 0, 0, 41)
    assert torch.allclose(dec, ref, atol=1e-4)
