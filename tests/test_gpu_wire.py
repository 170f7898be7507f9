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


def test_lwe_wire_roundtrip_and_bits(phe):
    """LWE outputs at q_out bits: exact round trip, the byte count, and the bit layout of the
    first token checked against a little-endian bitstream built here with Python ints."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(300, 2048)
    x = synth.activations_int8(3, 2048)
    S = phe.keygen(p, 5)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 91)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    m, b = phe.matmul_clear(p, w, phe.ct_prepare(p, seeds, body), 3)
    wire = phe.wire_serialize_lwe(p, m, b)
    assert wire.shape == (3, phe.wire_lwe_bytes(p, 300))
    assert phe.wire_lwe_bytes(p, 300) == 300 * 2048 * 26 // 8 + 8 * ((300 * 26 + 63) // 64)
    m2, b2 = phe.wire_deserialize_lwe(p, wire, 300)
    assert torch.equal(m2, m) and torch.equal(b2, b)
    vals = m[0].cpu().numpy().astype(np.uint64).reshape(-1).tolist()
    acc = 0
    for k, v in enumerate(vals[:4096]):       # first two mask segments, 26 bits each
        acc |= int(v) << (26 * k)
    ref = acc.to_bytes(26 * 4096 // 8, "little")
    assert bytes(wire[0, : len(ref)].cpu().numpy().tobytes()) == ref


def test_server_matvec_wire_host_matches_device(phe):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(256, 2048)
    x = synth.activations_int8(70, 2048)
    S = phe.keygen(p, 6)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 92)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    m, b = phe.matmul_clear(p, w, phe.ct_prepare(p, seeds, body), 70, row_begin=3, row_end=250)
    hi = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()
    ho = torch.empty((70, phe.wire_lwe_bytes(p, 247)), dtype=torch.uint8, pin_memory=True)
    phe.server_matvec_wire_host(p, w, hi, ho, chunk_tokens=32, row_begin=3, row_end=250)
    m2, b2 = phe.wire_deserialize_lwe(p, ho.cuda(), 247)
    assert torch.equal(m2, m) and torch.equal(b2, b)



@pytest.mark.parametrize("d_out,d_in,T,transpose,rows", [
    (300, 2048, 53, False, None),       # R = 300 (even record), ragged token tiles
    (2048, 2048, 60, False, (0, 2048)),  # q_proj shape, 51 + 9 tokens (narrow tail MMA)
    (512, 2048, 9, True, None),         # k^T: d_in = 512 < N, (j, j+1) CTA pairs
    (301, 700, 17, False, (5, 261)),     # partial block, a row range with R = 256
    (301, 700, 1, False, (0, 300)),      # odd rows in the last (j, j+1) pair
    (8192, 2048, 4, True, None),        # gate^T: L = 4
])
def test_matmul_clear_wire_equals_serialized(phe, d_out, d_in, T, transpose, rows):
    """phe_matmul_clear_wire (the mask epilogue bit-packs the switched words into the wire record,
    R22) is byte-identical to wire_serialize_lwe of matmul_clear's uint32 outputs, whose bytes are
    pinned to the oracle's serializer above."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(d_out, d_in, seed=d_out + d_in)
    cols = d_out if transpose else d_in
    x = synth.activations_int8(T, cols, seed=T)
    S = phe.keygen(p, 7)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 93)
    w = phe.Weights(p, torch.from_numpy(W).cuda(), transpose=transpose)
    opnd = phe.ct_prepare(p, seeds, body)
    r0, r1 = rows if rows else (0, w.rows)
    assert phe.wire_lwe_direct_supported(p, r1 - r0)
    f = phe.matmul_clear_T if transpose else phe.matmul_clear
    m, b = f(p, w, opnd, T, row_begin=r0, row_end=r1)
    ref = phe.wire_serialize_lwe(p, m, b)
    got = phe.matmul_clear_wire(p, w, opnd, T, row_begin=r0, row_end=r1)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def test_matmul_clear_wire_unsupported_record_stride(phe):
    """R = 301 gives an odd number of 64-bit words per record (no 16-byte TMA row stride): the fused
    form refuses (EUNSUPPORTED) and the host pipeline falls back to uint32 outputs + serialize."""
    p = phe.params(phe.PRESET_PAPER)
    assert not phe.wire_lwe_direct_supported(p, 301)
    W = synth.weights_int8(301, 2048, seed=3)
    x = synth.activations_int8(5, 2048, seed=4)
    S = phe.keygen(p, 8)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 94)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    with pytest.raises(phe.PheError):
        phe.matmul_clear_wire(p, w, phe.ct_prepare(p, seeds, body), 5)
    m, b = phe.matmul_clear(p, w, phe.ct_prepare(p, seeds, body), 5)
    hi = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()
    ho = torch.empty((5, phe.wire_lwe_bytes(p, 301)), dtype=torch.uint8, pin_memory=True)
    phe.server_matvec_wire_host(p, w, hi, ho, chunk_tokens=2)
    assert torch.equal(ho.cuda(), phe.wire_serialize_lwe(p, m, b))


def test_server_matvec_wire_host_fused_epilogue(phe):
    """The host pipeline with a supported R runs phe_matmul_clear_wire inside: same bytes."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(256, 2048, seed=5)
    x = synth.activations_int8(70, 2048, seed=6)
    S = phe.keygen(p, 9)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 95)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    assert phe.wire_lwe_direct_supported(p, 256)
    m, b = phe.matmul_clear(p, w, phe.ct_prepare(p, seeds, body), 70)
    hi = phe.wire_serialize_inputs(p, seeds, body).cpu().pin_memory()
    ho = torch.empty((70, phe.wire_lwe_bytes(p, 256)), dtype=torch.uint8, pin_memory=True)
    phe.server_matvec_wire_host(p, w, hi, ho, chunk_tokens=32)
    assert torch.equal(ho.cuda(), phe.wire_serialize_lwe(p, m, b))


@pytest.mark.parametrize("over,d_out,d_in,T", [
    (dict(N=512, q_in=39, q_out=26, beta=27), 64, 1100, 9),    # P1-like ring, L = 3
    (dict(N=4096, q_in=39, q_out=26, beta=27), 64, 4096, 3),   # P3 ring
    (dict(N=2048, q_in=32, q_out=24, beta=27), 64, 2048, 70),  # P2: ell = 4, q_out = 24 (generic epilogue)
    (dict(N=2048, q_in=39, q_out=20, beta=27), 64, 2048, 20),  # q_out = 20: 3-coefficient words
    (dict(N=2048, q_in=39, q_out=16, beta=16, gamma=8), 64, 2048, 5),  # q_out = 16 (lower bound)
])
def test_matmul_clear_wire_parameter_sets(phe, over, d_out, d_in, T):
    """The wire-record epilogue on other rings and output widths (16 <= q_out <= 26): byte-identical
    to wire_serialize_lwe(matmul_clear)."""
    p = phe.params(phe.PRESET_PAPER, **over)
    assert phe.wire_lwe_direct_supported(p, d_out)
    W = synth.weights_int8(d_out, d_in, seed=d_out + d_in + p.N)
    x = synth.activations_int8(T, d_in, seed=T + p.N)
    S = phe.keygen(p, 3)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).cuda(), 96)
    w = phe.Weights(p, torch.from_numpy(W).cuda())
    opnd = phe.ct_prepare(p, seeds, body)
    m, b = phe.matmul_clear(p, w, opnd, T)
    got = phe.matmul_clear_wire(p, w, opnd, T)
    torch.cuda.synchronize()
    assert torch.equal(got, phe.wire_serialize_lwe(p, m, b))
