"""tools/example_protocol.py -- the public API end to end on host buffers (client encrypt ->
wire bytes -> server host pipeline -> wire bytes -> client decrypt) with CBD(21) encryption noise:
the decrypted products equal W.x within the gamma-MSB contract, for the LWE outputs
(hot path) and the packed RLWE outputs (NEXT #1), on a ragged shape (d_in, d_out not multiples
of N)."""
import os
import sys

import pytest

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))


@pytest.mark.parametrize("packed", [False, True], ids=["lwe", "packed"])
def test_example_protocol(phe, packed):
    import example_protocol
    r = example_protocol.run(d_out=2500, d_in=3000, tokens=7, packed=packed)
    assert r["ok"], r
    assert r["bytes_up"] == 7 * 2 * 9992                      # two input blocks per token
    if packed:
        assert r["bytes_down"] == 7 * 2 * 13312               # two packed ciphertexts per token
