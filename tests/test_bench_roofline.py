"""The roofline arithmetic bench.py reports: the exp capacity of SFU + FMA pipe and
the north-star pair ceilings, pinned to the closed forms DESIGN.md states."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def test_exp_capacity_closed_form(bench):
    # max P s.t. (1 - f) P <= 16 and P (a + 8 f) <= 128: f = (128 - 16 a) / (16 * 8 + 128)
    for a, f, p in [(2.0, 0.375, 25.6), (3.0, 0.3125, 16 / 0.6875)]:
        c = bench.exp_capacity(a)
        assert c["soft_exp_fraction"] == pytest.approx(f)
        assert c["pairs_per_clk_sm"] == pytest.approx(p)
    # an FMA-saturated pass gets no software exponentials
    assert bench.exp_capacity(10.0)["soft_exp_fraction"] == 0.0


def test_pair_ceilings(bench):
    clk = 1965e6 * 148
    tc = bench.pair_ceiling(16, tc=True)
    assert tc["sfu_pairs_per_s"] == pytest.approx(16 * clk)            # one MUFU.EX2 per pair
    assert tc["pipe"] == "sfu" and tc["pairs_per_s"] == tc["sfu_pairs_per_s"]
    assert tc["exp_sfu_plus_fma_pairs_per_s"] == pytest.approx(25.6 * clk)
    ff = bench.pair_ceiling(1)
    assert ff["fp32_pairs_per_s"] == pytest.approx(128 * clk / 3)      # d + 2 FP32 lane-ops per pair
    assert ff["pipe"] == "sfu"                                         # 16 < 128 / 3 pairs/clk/SM
