"""GPU parity of NEXT #1 (KeySwitch packing, Eq. 7 + Eq. 8) against the CPU oracle (-m gpu).
KSK generation and every packed ciphertext word are compared bit-exactly; decryption must
recover W.x within the post-switch gamma-MSB contract."""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import phe_oracle as O
from oracle.phe_oracle import Params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("over,d_out,d_in,T,eta", [
    (dict(N=256), 512, 300, 3, 0),          # G = 2 groups, ragged input block
    (dict(N=256), 300, 256, 2, 21),         # rows not a multiple of 256 (padded rows), noisy KSK
    (dict(N=2048), 256, 2048, 2, 0),        # Table 1 ring
])
def test_packed_bit_exact(phe, coracle, over, d_out, d_in, T, eta):
    p = phe.params(phe.PRESET_PAPER, noise_eta=eta, **over)
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma, eta=eta)
    W = synth.weights_int8(d_out, d_in, seed=d_out + d_in)
    x = synth.activations_int8(T, d_in, seed=T + d_in)
    S = phe.keygen(p, 5)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77, 3)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    opnd = phe.ct_prepare(p, seeds, body)
    ksk = phe.ksk_gen(p, S, 1234)
    K = phe.KeySwitchKey(p, ksk)
    packed = phe.matmul_clear_packed(p, w, opnd, T, K)
    torch.cuda.synchronize()
    # oracle: its own key, KSK, encryption, Eq. 6, Eq. 7/8
    So = O.keygen(5, op.N)
    KA, KB = coracle.ksk_gen(op, So, 1234, eta=eta, nthreads=os.cpu_count())
    kk = u64(ksk)
    assert np.array_equal(kk[0], KA) and np.array_equal(kk[1], KB)
    seeds_o = O.block_seeds(77, T, op.L(d_in))
    E = O.noise(op, 3, T, op.L(d_in))
    G = (d_out + op.N - 1) // op.N
    got = packed.cpu().numpy().astype(np.uint32).astype(np.uint64)
    wx = (W.astype(np.int64) @ x.astype(np.int64).T).T
    for tau in range(T):
        A, B = O.encrypt(op, So, x[tau], seeds_o[tau], E[tau])
        m, b = coracle.matmul_clear_literal(op, W, A, B, nthreads=os.cpu_count())
        PA, PB = coracle.pack(op, m, b, KA, KB, nthreads=os.cpu_count())
        assert np.array_equal(got[tau, :, 0], O.modswitch(PA, op.q_in, op.q_out))
        assert np.array_equal(got[tau, :, 1], O.modswitch(PB, op.q_in, op.q_out))
    y = phe.decrypt_packed(p, S, packed, d_out).cpu().numpy().astype(np.int64)
    assert np.all(np.abs(y - wx) < 2 ** 15)  # top gamma = 12 of beta = 27 bits


def test_packed_transpose_backward(phe, coracle):
    p = phe.params(phe.PRESET_PAPER, N=256)
    op = Params(N=256, q_in=39, q_out=26, beta=27, gamma=12)
    W = synth.weights_int8(200, 512)   # backward: rows = d_in = 512, input g in Z^200
    g = synth.gradients_int8(2, 200)
    S = phe.keygen(p, 8)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(g).to(DEV), 9)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=True)
    opnd = phe.ct_prepare(p, seeds, body)
    K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 10))
    packed = phe.matmul_clear_packed(p, w, opnd, 2, K)
    So = O.keygen(8, 256)
    KA, KB = coracle.ksk_gen(op, So, 10, nthreads=os.cpu_count())
    seeds_o = O.block_seeds(9, 2, 1)
    got = packed.cpu().numpy().astype(np.uint32).astype(np.uint64)
    for tau in range(2):
        A, B = O.encrypt(op, So, g[tau], seeds_o[tau])
        m, b = coracle.matmul_clear_literal(op, np.ascontiguousarray(W.T), A, B, nthreads=os.cpu_count())
        PA, PB = coracle.pack(op, m, b, KA, KB, nthreads=os.cpu_count())
        assert np.array_equal(got[tau, :, 0], O.modswitch(PA, 39, 26))
        assert np.array_equal(got[tau, :, 1], O.modswitch(PB, 39, 26))


def test_packed_host_path_and_stages_agree(phe):
    """phe_server_matvec_packed_host (host buffers, chunked) == device call == staged calls."""
    p = phe.params(phe.PRESET_PAPER, N=256)
    W = synth.weights_int8(512, 256)
    x = synth.activations_int8(70, 256)
    S = phe.keygen(p, 3)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 4)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 5))
    opnd = phe.ct_prepare(p, seeds, body)
    ref = phe.matmul_clear_packed(p, w, opnd, 70, K)
    dig, bod = phe.matmul_clear_digits(p, w, opnd, 70)
    staged = phe.pack(p, dig, bod, K)
    assert torch.equal(staged, ref)
    ho = torch.empty((70, 2, 2, 256), dtype=torch.int32).pin_memory()
    phe.server_matvec_packed_host(p, w, K, seeds.cpu().pin_memory(), body.cpu().pin_memory(), ho, chunk_tokens=33)
    assert torch.equal(ho, ref.cpu())
