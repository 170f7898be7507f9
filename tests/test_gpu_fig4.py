"""Fig. 4 claim on the GPU path: for d_in in {768, 2048, 8192} at N = 2048 the
bit-error rate of decrypted dot products is below 1% at every bit position >= 12 (soft pin:
figure-only claim; R12)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_fig4_msb_error_rates_below_one_percent(phe):
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import bit_error_study
    rows = bit_error_study.run(trials=8192)
    for d_in in (768, 2048, 8192):
        assert max(r[2] for r in rows if r[0] == d_in and r[1] >= 12) < 0.01
        # the LSB is essentially a coin flip after the 39 -> 26 switch (Delta_out = 1/2, R11)
        assert 0.3 < [r[2] for r in rows if r[0] == d_in and r[1] == 0][0] < 0.7


def test_fig4_d_in_trend_with_input_noise(phe):
    """P:403 "Higher input dimensions increase LSB error due to noise accumulation": with an input
    noise whose sigma ||w|| / Delta is comparable to the switch error (R25: sigma = 24 in
    Z_Q units; Table 1's sigma rounds to 0), the low-bit error rates grow with d_in while every
    position >= 12 stays below 1%."""
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import bit_error_study
    rows = bit_error_study.run(trials=16384, sigma=24.0)
    low = {d: sum(r[2] for r in rows if r[0] == d and 6 <= r[1] <= 10) for d in (768, 2048, 8192)}
    assert low[768] < low[2048] < low[8192]
    for d_in in (768, 2048, 8192):
        assert max(r[2] for r in rows if r[0] == d_in and r[1] >= 12) < 0.01
