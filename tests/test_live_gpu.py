"""f1: the live asynchronous loop (paper_2505_12658_b200/live.py) on the tiny model.

Wall-clock serving changes which requests share a batch (timing-dependent), so scheduler
decisions are not compared with the golden log; what must hold: every request finishes with
exactly its output tokens, the physical pools stay consistent with the reference's counts
after every event, migrations copy the blocks the reference reserved, and -- on one
instance, where every batch's inputs are fully determined by the batches before it -- the
logits of every emitted token match the fp32 oracle replay of the batches actually run.
"""
import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from parity_util import LOGIT_ATOL, golden_trace, load_golden, oracle_replay  # noqa: E402


def _cluster(name, capture):
    from paper_2505_12658_b200 import get_shape
    from paper_2505_12658_b200._epdsim import C, E
    from paper_2505_12658_b200.cluster import GpuCluster
    g = load_golden(name)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse(g["method"]))
    cl = GpuCluster(spec, get_shape("tiny"), E.HardwareProfile(*g["hw"]), E.SloSpec(*g["slo"]),
                    clock="device", record_batches=True, capture=capture,
                    pool_bytes_limit=4 << 30)
    return g, cl, golden_trace(E, g)


def test_time_scale_validated():
    from paper_2505_12658_b200.live import run_live
    with pytest.raises(ValueError):
        run_live(None, None, time_scale=0.0)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["config1_2000rps", "tiny_E1_P1_D1", "tiny_EP1_D1"])
def test_live_run_completes(name):
    from paper_2505_12658_b200.live import run_live
    g, cl, trace = _cluster(name, capture=False)
    rep = run_live(cl, trace, time_scale=1.0, check_invariants=True, timeout_s=120)
    assert cl.finished == cl.arrived == len(trace.requests)
    for r in trace.requests:
        assert len(cl.generated[r.id]) == r.output_tokens
        assert cl.reqs[r.id].tokens_out == r.output_tokens
    assert rep.aggregates["n_requests"] == len(trace.requests)
    for iid, rt in cl.runtimes.items():
        assert rt.kv_pool.consistent() and rt.image_pool.consistent()
    if len(cl.instances) > 1:
        assert cl.migration_log, "disaggregated run without migrations"
    cl.close()


@pytest.mark.gpu
def test_live_single_instance_logits_match_oracle():
    from paper_2505_12658_b200 import get_shape
    from paper_2505_12658_b200.live import run_live
    g, cl, trace = _cluster("config1_2000rps", capture=True)
    run_live(cl, trace, time_scale=0.5, check_invariants=True, timeout_s=120)
    res = oracle_replay(cl, get_shape("tiny"), seed=0)
    assert res["max_abs_err"] <= LOGIT_ATOL, res
    assert res["tokens_equal"] + res["near_ties"] == res["rows"], res
    cl.close()
