"""CPU tests of the shared work-sharing engine (SURVEY §8a "Shared engine /
split ratio"): the split formula, WorkShare bounds, the golden-section
calibrate (reference hb/worksharing.py:63-156), gain / idle
(:159-174), and run_workshared + calibrate_measured on a host-only toy
workload — the behaviour pinned by the reference's tests/test_worksharing.py."""

import math

import numpy as np
import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_1303_2171_b200.platform import Accounting, DeviceId, Interval, Platform, Timeline, modeled_compute_time
from paper_1303_2171_b200.worksharing import (
    ShareOrigin,
    WorkShare,
    calibrate,
    calibrate_measured,
    compute_gain,
    compute_idle,
    formula_share,
    run_workshared,
    split_fraction_formula,
)

positive = st.floats(min_value=1e-6, max_value=1e6)


def test_split_formula_values():
    assert split_fraction_formula(12.0, 4.0).fraction_a == 0.25
    assert split_fraction_formula(2.5, 2.5).fraction_a == 0.5
    assert split_fraction_formula(0.82, 0.18).fraction_a == pytest.approx(0.18)
    for bad in ((0.0, 1.0), (1.0, -3.0)):
        with pytest.raises(ValueError):
            split_fraction_formula(*bad)


@given(t_a=positive, t_b=positive)
def test_split_formula_balances_the_two_sides(t_a, t_b):
    f = split_fraction_formula(t_a, t_b).fraction_a
    assert 0.0 <= f <= 1.0
    assert f * t_a == pytest.approx((1.0 - f) * t_b, rel=1e-9, abs=1e-12 * max(t_a, t_b))


def test_manual_share_bounds_and_formula_share(platform13):
    for bad in (-0.01, 1.01, math.nan):
        with pytest.raises(ValueError):
            WorkShare.manual(bad)
    assert formula_share(platform13).fraction_a == 0.25


def _modeled(device, work):
    return modeled_compute_time(device, work)


def test_calibrate_keeps_the_formula_split_under_a_linear_model(platform13):
    share = calibrate(platform13, _modeled, sample=1000.0, max_refinements=12)
    assert share.fraction_a == 0.25 and share.origin is ShareOrigin.CALIBRATED
    first = share.probe.refinement_steps[0][1]
    assert all(t >= first for _, t in share.probe.refinement_steps)
    assert calibrate(Platform.build(1.0, 1.0), _modeled, sample=10.0, max_refinements=6).fraction_a == 0.5
    zero = calibrate(platform13, _modeled, sample=10.0, max_refinements=0)
    assert zero.fraction_a == 0.25 and len(zero.probe.refinement_steps) == 1


def test_calibrate_leaves_the_formula_when_the_host_has_overhead(platform13):
    def probe(device, work):
        t = modeled_compute_time(device, work)
        return t + 5.0 if device.id is DeviceId.A and work > 0 else t

    share = calibrate(platform13, probe, sample=100.0, max_refinements=40)

    def both(f):
        return max(probe(platform13.device_a, f * 100.0), probe(platform13.device_b, (1 - f) * 100.0))

    assert share.fraction_a < 0.25 and both(share.fraction_a) <= both(0.25)


def test_gain_and_idle():
    assert compute_gain(75.0, 100.0, 300.0) == 25.0
    assert compute_gain(100.0, 100.0, 120.0) == 0.0
    assert compute_gain(81.4, 100.0, 250.0) == pytest.approx(18.6)
    assert compute_gain(200.0, 100.0, 150.0) < 0
    for bad in ((0.0, 1.0, 1.0), (1.0, -1.0, 1.0)):
        with pytest.raises(ValueError):
            compute_gain(*bad)
    assert compute_idle(Timeline.build([Interval(0, 10)], [Interval(0, 10)])) == 0.0
    assert compute_idle(Timeline.build([Interval(0, 10)], [])) == 50.0
    assert compute_idle(Timeline.build([Interval(0, 10)], [Interval(0, 8)])) == 10.0
    a, b = [Interval(0, 3), Interval(5, 6)], [Interval(0, 9)]
    assert compute_idle(Timeline.build(a, b)) == compute_idle(Timeline.build(b, a))
    with pytest.raises(ValueError):
        compute_idle(Timeline.build())


class _SumWorkload:
    """Host-only Partitionable: the sum of a float array, index split; both
    'devices' run numpy (so the engine is exercised without a GPU)."""

    name = "toy-sum"
    unit = "elements"

    def __init__(self, data):
        self.data = data

    def partition(self, fraction_a):
        s = int(math.floor(fraction_a * self.data.size))
        return self.data[:s], self.data[s:]

    def work_units(self, part):
        return float(part.size)

    def run_part(self, device, part):
        return float(np.sum(part, dtype=np.float64))

    def merge(self, partials):
        return partials[0] + partials[1]


@pytest.mark.parametrize("f", [0.0, 0.25, 0.6, 1.0])
def test_run_workshared_modeled_report(platform13, f):
    data = np.arange(100_000, dtype=np.float64)
    result, report = run_workshared(platform13, _SumWorkload(data), WorkShare.manual(f))
    assert result == float(data.sum())
    assert report.pure_a_time == pytest.approx(100_000 / 1.0)
    assert report.pure_b_time == pytest.approx(100_000 / 3.0)
    if f == 0.25:  # the formula split: both sides finish together
        assert report.idle_percent == pytest.approx(0.0, abs=1e-9)
        assert report.gain_percent == pytest.approx(25.0, abs=1e-9)
    if f in (0.0, 1.0):  # one side idle the whole run
        assert report.idle_percent == 50.0
    assert report.resource_efficiency_percent == 100.0 - report.idle_percent


def test_calibrate_measured_on_a_host_only_workload():
    p = Platform.build(1.0, 3.0, accounting=Accounting.MEASURED)
    wl = _SumWorkload(np.random.default_rng(0).random(200_000))
    share = calibrate_measured(wl, p, max_refinements=3, repeats=1)
    assert 0.0 <= share.fraction_a <= 1.0 and share.origin is ShareOrigin.CALIBRATED
    assert len(share.probe.refinement_steps) >= 3 + 2  # start, refinements, both ends
    seq = calibrate_measured(wl, p, max_refinements=2, concurrent=False)
    assert 0.0 <= seq.fraction_a <= 1.0


def test_resolve_share_modes(platform13):
    """resolve_share (reference workloads.py:73-79) over every ShareSpec mode,
    and ShareSpec's validation (config.py:91-106)."""
    from paper_1303_2171_b200.errors import ConfigError
    from paper_1303_2171_b200.worksharing import ShareSpec, resolve_share

    assert resolve_share(platform13, ShareSpec(), 100.0).fraction_a == pytest.approx(0.25)
    assert resolve_share(platform13, ShareSpec("manual", 0.4), 100.0).fraction_a == 0.4
    cal = resolve_share(platform13, ShareSpec("calibrated", refinements=6), 0.0)
    assert cal.origin.value == "calibrated" and cal.fraction_a == pytest.approx(0.25)
    assert cal.probe.sample_size == 1.0  # max(total_units, 1)
    with pytest.raises(ConfigError):
        ShareSpec("sometimes")
    with pytest.raises(ConfigError):
        ShareSpec("manual", 1.5)
    with pytest.raises(ConfigError):
        ShareSpec("calibrated", refinements=-1)
    with pytest.raises(ValueError):
        resolve_share(platform13, ShareSpec("measured", refinements=1), 10.0)
