"""GPU parity of NEXT #2 (wire format) against the oracle's serializers (-m gpu)."""
import numpy as np
import pytest
import torch

import synth
from oracle import phe_oracle as O

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def test_wire_inputs_bytes_match_oracle(phe):
    p = phe.params(phe.PRESET_PAPER)
    S = phe.keygen(p, 1)
    x = synth.activations_int8(3, 3000)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 2 ** 63 + 5)
    wire = phe.wire_serialize_inputs(p, seeds, body)
    assert wire.shape == (3, 2, 9992)
    w = wire.cpu().numpy()
    sd = seeds.cpu().numpy().view(np.uint64)
    bd = body.cpu().numpy().view(np.uint64)
    for t in range(3):
        for i in range(2):
            assert bytes(w[t, i]) == O.serialize_input(int(sd[t, i]), bd[t, i], 39)
    s2, b2 = phe.wire_deserialize_inputs(p, wire)
    assert torch.equal(s2, seeds) and torch.equal(b2, body)


def test_wire_packed_bytes_match_oracle_and_server_wire_path(phe):
    p = phe.params(phe.PRESET_PAPER, N=256)
    W = synth.weights_int8(300, 256)
    x = synth.activations_int8(40, 256)
    S = phe.keygen(p, 3)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 4)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 5))
    opnd = phe.ct_prepare(p, seeds, body)
    packed = phe.matmul_clear_packed(p, w, opnd, 40, K)
    wire = phe.wire_serialize_packed(p, packed)
    assert wire.shape == (40, 2, 2 * 256 * 26 // 8)
    pk = packed.cpu().numpy().astype(np.uint32).astype(np.uint64)
    wn = wire.cpu().numpy()
    for t in [0, 17, 39]:
        for g in range(2):
            assert bytes(wn[t, g]) == O.serialize_output(pk[t, g, 0], pk[t, g, 1], 26)
    assert torch.equal(phe.wire_deserialize_packed(p, wire), packed)
    # the whole server step on wire bytes (host buffers)
    h_in = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()
    h_out = torch.empty((40, 2, wire.shape[2]), dtype=torch.uint8).pin_memory()
    phe.server_wire_host(p, w, K, h_in, h_out, chunk_tokens=16)
    assert torch.equal(h_out, wire.cpu())
