"""Algorithm 2 on measured stage speeds (planner.py): with the reference's
roofline as the timer it must reproduce epdsim.profiler.plan_partition exactly, for several
models, traces and cluster sizes; with slower measured timers the split shifts as expected."""

import os
import sys

import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_12658_b200 import b200_hardware, get_shape  # noqa: E402
from paper_2505_12658_b200._epdsim import E  # noqa: E402
from paper_2505_12658_b200.planner import (measured_plan_partition,  # noqa: E402
                                           roofline_timers)

import epdsim.profiler as P  # noqa: E402


def _trace(seed, tokens):
    return E.synth_trace(seed=seed, n_requests=200, rate=4.0, image_count_dist=1,
                         visual_token_choices=tokens, prompt_dist=[25, 35, 45],
                         output_dist=[90, 110, 130], slo=E.SloSpec(4.0, 0.08))


@pytest.mark.parametrize("name", ["llava-1.5-7b", "qwen2-vl-7b"])
@pytest.mark.parametrize("N", [3, 4, 8])
@pytest.mark.parametrize("seed,tokens", [(7, 576), (3, [256, 576, 1024])])
def test_roofline_timers_reproduce_reference_plan(name, N, seed, tokens):
    model = get_shape(name).profile()
    hw = b200_hardware()
    slo = E.SloSpec(4.0, 0.08)
    tr = _trace(seed, tokens)
    ref = P.plan_partition(tr, N, slo, model, hw)
    got = measured_plan_partition(tr, N, slo, model, hw, *roofline_timers(model, hw))
    assert got == ref


def test_slower_decode_shifts_instances_to_decode():
    model = get_shape("llava-1.5-7b").profile()
    hw = b200_hardware()
    slo = E.SloSpec(4.0, 0.08)
    tr = _trace(7, 576)
    tp, te, td = roofline_timers(model, hw)
    base = measured_plan_partition(tr, 8, slo, model, hw, tp, te, td)
    slow = measured_plan_partition(tr, 8, slo, model, hw, tp, te,
                                   lambda n, ctx: 3.0 * td(n, ctx))
    assert slow.N_d >= base.N_d and slow.t_d > base.t_d
    assert base.N_e + base.N_p + base.N_d == 8 == slow.N_e + slow.N_p + slow.N_d


@pytest.mark.parametrize("N", [3, 4])
def test_measured_selection_reproduces_reference_select_method(N):
    """f3 (profiler.py:216-270): with roofline timers and the reference's own replayed
    goodput as the scorer, measured_select_method picks exactly what select_method picks
    (same partition, same three candidates, same goodput table, same tie rule)."""
    from paper_2505_12658_b200.planner import measured_select_method
    model = get_shape("llava-1.5-7b").profile()
    hw = b200_hardware()
    slo = E.SloSpec(4.0, 0.08)
    tr = E.synth_trace(seed=7, n_requests=60, rate=4.0, image_count_dist=1,
                       visual_token_choices=576, prompt_dist=[25, 35, 45],
                       output_dist=[90, 110, 130], slo=slo)
    bounds = (1.0, 64.0)
    ref = P.select_method(tr, N, slo, model, hw, rate_bounds=bounds, tolerance=0.5)
    got = measured_select_method(
        tr, N, slo, model, hw,
        lambda m: P.method_goodput(m, tr, slo, model, hw, bounds, 0.5))
    assert got.best == ref.best
    assert got.table == ref.table
    assert got.partition == ref.partition
