"""Measured-probe budget search (budgets.py) with an injectable prober:
under the reference's roofline prober it must equal the reference's own
``budgets_for_type`` -> ``search_budgets`` (cluster.py:147-158, engine.py:105-153) for
every instance type, model, SLO and budget ceiling; a slower prober only shrinks budgets."""

import types

import pytest

from paper_2505_12658_b200 import b200_hardware, get_shape
from paper_2505_12658_b200._epdsim import C, EN, E
from paper_2505_12658_b200.budgets import (RooflineProber, measured_budgets,
                                           search_with_prober)

SLOS = [E.SloSpec(4.0, 0.08), E.SloSpec(8.0, 0.10), E.SloSpec(0.5, 0.02), E.SloSpec(0.05, 0.001)]


@pytest.mark.parametrize("name", ["tiny", "llava-1.5-7b", "qwen2-vl-7b"])
@pytest.mark.parametrize("hw", ["default", "b200"])
def test_roofline_prober_equals_reference_search(name, hw):
    model = get_shape(name).profile()
    hwp = E.DEFAULT_HARDWARE if hw == "default" else b200_hardware()
    for slo in SLOS:
        for ceil in ((16384, 128), (512, 2), (100000, 1000)):
            spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("EPD:1"),
                                 token_budget_ceiling=ceil[0], image_budget_ceiling=ceil[1])
            for itype in EN.ALL_INSTANCE_TYPES:
                ref = C.budgets_for_type(itype, slo, model, hwp, spec)
                got = search_with_prober(itype, slo, spec, RooflineProber(model, hwp))
                assert got == ref, (itype, slo, ceil)


def test_measured_budgets_with_injected_prober():
    """measured_budgets drives search_with_prober per instance type of a cluster; with the
    roofline prober injected it installs the reference's budgets unchanged, with a prober
    twice as slow the budgets can only shrink."""
    model = get_shape("llava-1.5-7b").profile()
    hw = b200_hardware()
    slo = E.SloSpec(4.0, 0.08)
    spec = C.ClusterSpec(method=C.DisaggregationMethod.parse("E:1,P:1,D:1,EP:1,EPD:1"))
    ref = C.Cluster(spec, model, hw, slo)
    fake = types.SimpleNamespace(
        spec=spec, model=model, hw=hw, slo=slo, shape=get_shape("llava-1.5-7b"),
        instances=ref.instances, type_budgets=dict(ref.type_budgets),
        runtimes={iid: types.SimpleNamespace(device="cuda:0") for iid in ref.instances})
    want = dict(ref.type_budgets)
    got = measured_budgets(fake, prober_factory=lambda rt, shape: RooflineProber(model, hw))
    assert got == want
    assert all(inst.budgets == want[inst.itype] for inst in ref.instances.values())

    class Slow(RooflineProber):
        def tokens(self, n):
            return 2 * super().tokens(n)

        def images(self, e, t):
            return 2 * super().images(e, t)

    slow = measured_budgets(fake, prober_factory=lambda rt, shape: Slow(model, hw))
    for it, b in slow.items():
        assert b.token_budget <= want[it].token_budget
        assert b.image_budget <= want[it].image_budget
