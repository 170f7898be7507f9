"""Pins for the NEXT #2 oracle (wire format), -m "not gpu": the sizes and expansion factors are
the numbers PAPER.md prints; bit layout checked by hand; round trips."""
import numpy as np
import pytest

from oracle import phe_oracle as O
import synth


def test_paper_wire_sizes_and_factors():
    r = O.expansion_report(O.PAPER)
    assert r["input_bytes"] == 9992          # 8 + 9984
    assert r["output_bytes"] == 13312        # 2 x 6656
    assert abs(r["input_factor"] - 4.88) < 0.01
    assert abs(r["output_factor"] - 4.33) < 0.01


def test_bit_layout_by_hand():
    # two 39-bit values: 1 at bit 0, and 2^38 + 1 at bits 39..77 -> bits 39 and 77 set
    data = O.bitpack([1, 2 ** 38 + 1], 39)
    assert len(data) == 10  # ceil(78 / 8)
    v = int.from_bytes(data, "little")
    assert v == 1 | (1 << 39) | (1 << 77)
    # 26-bit: value 0x3FFFFFF then 0 -> low 26 bits set
    assert int.from_bytes(O.bitpack([2 ** 26 - 1, 0], 26), "little") == 2 ** 26 - 1


def test_roundtrips():
    N = 2048
    body = synth.uniform_u64(N, 3, 39)
    blob = O.serialize_input(0xDEADBEEF12345678, body, 39)
    seed, back = O.deserialize_input(blob, N, 39)
    assert seed == 0xDEADBEEF12345678 and np.array_equal(back, body)
    A, B = synth.uniform_u64(N, 4, 26), synth.uniform_u64(N, 5, 26)
    blob = O.serialize_output(A, B, 26)
    A2, B2 = O.deserialize_output(blob, N, 26)
    assert np.array_equal(A, A2) and np.array_equal(B, B2)
    with pytest.raises(ValueError):
        O.deserialize_output(blob[:-1], N, 26)
    with pytest.raises(ValueError):
        O.deserialize_input(b"", N, 39)
