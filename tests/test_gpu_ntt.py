"""GPU parity tests (-m gpu) for NEXT #4, the NTT-domain mask contraction
(phe_matmul_clear_ntt[_T], paper_2505_07329_b200/csrc/ntt_path.cu).

Bar: bit-exact against the oracle's literal Eq. 6 (C path, oracle/phe_oracle.c) and bit-identical
to the tensor-core limb GEMM on the same inputs — Eq. 6 defines every output word
uniquely, so two correct paths cannot differ in a single bit.  Cases cover every N the kernel
is specialised for (512 ... 8192), ragged rows/blocks/tokens, both output widths, the backward
W^T registration, row sharding, the CRT range at its worst case and the EUNSUPPORTED boundary.
"""
import ctypes
import os

import numpy as np
import pytest
import torch

import synth
from oracle import phe_oracle as O
from oracle.phe_oracle import Params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def oparams(p):
    return Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma, eta=p.noise_eta)


def u64(t):
    return t.cpu().numpy().view(np.uint64)


def encrypt(phe, p, x, sbase=4242, sk_seed=7, noise_seed=0):
    S = phe.keygen(p, sk_seed)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), sbase, noise_seed)
    return S, seeds, body


def oracle_literal(coracle, p, M, seeds, body):
    """Literal Eq. 6 on the oracle side from the same public ciphertext (seeds, bodies): the
    masks are re-expanded by the oracle's own ChaCha20 (oracle/phe_oracle.c)."""
    op = oparams(p)
    sd, bd = u64(seeds), u64(body)
    masks, bodies = [], []
    for tau in range(sd.shape[0]):
        A = np.stack([coracle.expand_mask(int(s), op.N, op.q_in) for s in sd[tau]])
        m, b = coracle.matmul_clear_literal(op, M, A, bd[tau], nthreads=os.cpu_count())
        masks.append(m); bodies.append(b)
    return np.stack(masks), np.stack(bodies)


def ntt_run(phe, p, W, seeds, body, transpose=False, out_bits=None, **kw):
    tabs = phe.NttTables(p)
    w = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=transpose)
    op = phe.ntt_ct_prepare(p, tabs, seeds, body)
    res = phe.matmul_clear_ntt(p, w, op, seeds.shape[0], out_bits=out_bits, **kw)
    torch.cuda.synchronize()
    return w, op, res


@pytest.mark.parametrize("preset,over,d_out,d_in,T", [
    ("TOY", {}, 64, 64, 16),                                  # BASELINE configs[0] shape
    ("PAPER", {}, 200, 4100, 5),                              # ragged rows, L = 3 ragged block
    ("PAPER", {}, 37, 2048, 70),                              # many tokens (several CTAs/row)
    ("PAPER", dict(N=512), 40, 1100, 9),                      # LOGN 9, L = 3
    ("PAPER", dict(N=4096), 5, 4096, 3),                      # LOGN 12
    ("PAPER", dict(N=8192), 3, 8192, 2),                      # LOGN 13 (4th exchange phase)
    ("PAPER", dict(N=2048, q_in=32, q_out=24), 33, 2048, 11),  # P2: q 2^32 -> 2^24
])
def test_ntt_bit_exact_vs_oracle(phe, coracle, preset, over, d_out, d_in, T):
    p = phe.params(getattr(phe, "PRESET_" + preset), **over)
    W = synth.uniform_int8((d_out, d_in), d_in + T, -127, 127)
    x = synth.uniform_int8((T, d_in), d_out + T, -100, 100)
    S, seeds, body = encrypt(phe, p, x)
    w, opnd, (mq, bq) = ntt_run(phe, p, W, seeds, body, out_bits=p.q_in)
    mask_o, body_o = oracle_literal(coracle, p, W, seeds, body)
    assert np.array_equal(u64(mq), mask_o)
    assert np.array_equal(u64(bq), body_o)
    ms, bs = phe.matmul_clear_ntt(p, w, opnd, T)  # switched to q_out in the epilogue
    assert np.array_equal(ms.cpu().numpy().astype(np.uint32).astype(np.uint64),
                          O.modswitch(mask_o, p.q_in, p.q_out))
    assert np.array_equal(bs.cpu().numpy().astype(np.uint32).astype(np.uint64),
                          O.modswitch(body_o, p.q_in, p.q_out))
    y = phe.decrypt_unpack(p, S, mq, bq, p.q_in).cpu().numpy()   # E = 0: exact W x
    assert np.array_equal(y, (W.astype(np.int64) @ x.astype(np.int64).T).T)


def test_ntt_identical_to_tensor_core_path(phe):
    """Same inputs through both contractions: identical words (Eq. 6 is unique)."""
    p = phe.params(phe.PRESET_PAPER, noise_eta=21)
    W = synth.weights_int8(300, 8192, seed=5)   # down_proj-like d_in, L = 4
    x = synth.activations_int8(60, 8192, seed=6)
    S, seeds, body = encrypt(phe, p, x, noise_seed=77)
    _, _, (mn, bn) = ntt_run(phe, p, W, seeds, body)
    wd = phe.Weights(p, torch.from_numpy(W).to(DEV))
    md, bd = phe.matmul_clear(p, wd, phe.ct_prepare(p, seeds, body), 60)
    assert torch.equal(mn, md) and torch.equal(bn, bd)


def test_ntt_backward_transpose(phe, coracle):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(2100, 70, seed=3)    # W^T . g with g in Z^2100: L = 2 ragged
    g = synth.gradients_int8(4, 2100, seed=4)
    S, seeds, body = encrypt(phe, p, g)
    w, opnd, (m, b) = ntt_run(phe, p, W, seeds, body, transpose=True, out_bits=p.q_in)
    assert m.shape == (4, 70, p.N)
    mask_o, body_o = oracle_literal(coracle, p, np.ascontiguousarray(W.T), seeds, body)
    assert np.array_equal(u64(m), mask_o) and np.array_equal(u64(b), body_o)


def test_ntt_row_sharding_and_empty(phe):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(300, 2048)
    x = synth.activations_int8(20, 2048)
    S, seeds, body = encrypt(phe, p, x)
    w, opnd, (m, b) = ntt_run(phe, p, W, seeds, body)
    for r0, r1 in [(0, 128), (128, 300), (17, 18), (5, 5)]:
        ms, bs = phe.matmul_clear_ntt(p, w, opnd, 20, row_begin=r0, row_end=r1)
        assert torch.equal(ms, m[:, r0:r1]) and torch.equal(bs, b[:, r0:r1])
    empty = torch.zeros(phe.load().phe_ntt_operand_bytes(ctypes.byref(p), 0, 1), dtype=torch.uint8, device=DEV)
    m0, b0 = phe.matmul_clear_ntt(p, w, empty, 0)
    assert m0.shape == (0, 300, p.N)
    S1, s1, b1 = encrypt(phe, p, x[:1])
    _, _, (m1, bb1) = ntt_run(phe, p, W, s1, b1)
    assert torch.equal(m1[0], m[0]) and torch.equal(bb1[0], b[0])


def test_ntt_max_blocks_and_refusal(phe, coracle):
    """N = 512, q_in = 39: the CRT allows 27 blocks (centred masks); L = 27 runs bit-exact, one
    block more is refused (EUNSUPPORTED), never silently wrong."""
    p = phe.params(phe.PRESET_PAPER, N=512)
    Lmax = phe.ntt_max_blocks(p)
    assert Lmax == 27
    d_in = Lmax * 512
    W = synth.uniform_int8((2, d_in), 5, -127, 127)
    x = synth.uniform_int8((2, d_in), 11, -3, 3)
    S, seeds, body = encrypt(phe, p, x)
    _, _, (m, b) = ntt_run(phe, p, W, seeds, body, out_bits=39)
    mask_o, body_o = oracle_literal(coracle, p, W, seeds, body)
    assert np.array_equal(u64(m), mask_o) and np.array_equal(u64(b), body_o)
    W2 = np.ones((2, d_in + 512), np.int8)
    tabs = phe.NttTables(p)
    w2 = phe.NttWeights(p, tabs, torch.from_numpy(W2).to(DEV))
    x2 = synth.uniform_int8((1, d_in + 512), 12, -3, 3)
    _, s2, b2 = encrypt(phe, p, x2)
    op2 = phe.ntt_ct_prepare(p, tabs, s2, b2)
    with pytest.raises(phe.PheError, match="unsupported"):
        phe.matmul_clear_ntt(p, w2, op2, 1)


@pytest.mark.parametrize("wval", [-127, 127])
def test_ntt_crt_range_adversarial(phe, coracle, wval):
    """The CRT range at its worst case: every mask word 2^39 - 1 (centred: 2^38 - 1) and every
    weight -127 (or 127; -128 is refused at registration) over L = 27 blocks of N = 512 puts |P'[N-1]| = L N (2^38 - 1) |w| at the
    bound of phe_ntt_max_blocks.  The NTT-domain operand is built on the host by the independent
    Python NTT of tools/ntt_model.py (no seed can produce constant masks); expected values come
    from the oracle's literal Eq. 6."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import ntt_model
    p = phe.params(phe.PRESET_PAPER, N=512)
    N, L, T = 512, phe.ntt_max_blocks(p), 1
    H = 2 ** 38
    A = np.full((L, N), 2 ** 39 - 1, np.uint64)
    W = np.full((2, L * N), wval, np.int8)
    W[1, ::7] = 0  # second row: a different weight sum parity / pattern
    ahat = np.zeros((T, L, 2, N), np.uint32)
    # storage order of NTT-domain vectors (include/phe.h): element k at 4*(((k>>2)&3)*N/16 + (k>>4)) + (k&3)
    pos = np.array([4 * (((k >> 2) & 3) * (N // 16) + (k >> 4)) + (k & 3) for k in range(N)])
    for q, (pr, g) in enumerate(zip(ntt_model.P, ntt_model.GEN)):
        fwd, _ = ntt_model.tables(pr, g, N)
        for i in range(L):
            ahat[0, i, q, pos] = ntt_model.ntt_fwd([(int(a) - H) % pr for a in A[i]], pr, fwd)
    nbytes = phe.load().phe_ntt_operand_bytes(ctypes.byref(p), T, L)
    opnd = np.zeros(nbytes, np.uint8)           # body planes zero: B = 0
    opnd[: ahat.nbytes] = ahat.reshape(-1).view(np.uint8)
    tabs = phe.NttTables(p)
    w = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV))
    m, b = phe.matmul_clear_ntt(p, w, torch.from_numpy(opnd).to(DEV), T, out_bits=39)
    mo, bo = coracle.matmul_clear_literal(oparams(p), W, A, np.zeros((L, N), np.uint64), nthreads=os.cpu_count())
    assert np.array_equal(u64(m[0]), mo) and np.array_equal(u64(b[0]), bo)


def test_ntt_full_size_q_proj_sampled(phe, coracle):
    """configs[1] shape (q_proj 2048x2048, T = 2048) through the NTT path: identical to the
    tensor-core path on every word, plus one full token against the oracle's literal Eq. 6."""
    p = phe.params(phe.PRESET_PAPER)
    d, T = 2048, 2048
    W = synth.weights_int8(d, d)
    x = synth.activations_int8(T, d)
    S, seeds, body = encrypt(phe, p, x)
    w, opnd, (mn, bn) = ntt_run(phe, p, W, seeds, body)
    wd = phe.Weights(p, torch.from_numpy(W).to(DEV))
    md, bd = phe.matmul_clear(p, wd, phe.ct_prepare(p, seeds, body), T)
    assert torch.equal(bn, bd)
    assert torch.equal(mn, md)
    del md
    tau = 777
    mask_o, body_o = oracle_literal(coracle, p, W, seeds[tau:tau + 1], body[tau:tau + 1])
    assert np.array_equal(mn[tau].cpu().numpy().astype(np.uint32).astype(np.uint64), O.modswitch(mask_o[0], 39, 26))


@pytest.mark.parametrize("preset,over,eta,d_in,T", [
    ("TOY", {}, 0, 64, 16), ("PAPER", {}, 0, 4100, 7), ("PAPER", {}, 21, 2048, 5),
    ("PAPER", dict(N=512), 21, 1100, 3), ("PAPER", dict(N=8192), 0, 8192, 2),
])
def test_encrypt_pack_ntt_identical(phe, coracle, preset, over, eta, d_in, T):
    """phe_encrypt_pack_ntt == phe_encrypt_pack word for word (the latter is pinned to the oracle:
    test_gpu_parity.py::test_keygen_and_encrypt_match_oracle); one block also against the oracle."""
    p = phe.params(getattr(phe, "PRESET_" + preset), noise_eta=eta, **over)
    x = torch.from_numpy(synth.uniform_int8((T, d_in), 3 + T, -100, 100)).to(DEV)
    S = phe.keygen(p, 11)
    s1, b1 = phe.encrypt_pack(p, S, x, 777, 99)
    tabs = phe.NttTables(p)
    s2, b2 = phe.encrypt_pack_ntt(p, tabs, S, x, 777, 99)
    assert torch.equal(s1, s2) and torch.equal(b1, b2)
    op = oparams(p)
    So = O.keygen(11, op.N)
    E = O.noise(op, 99, T, op.L(d_in))
    A, B = O.encrypt(op, So, x[0].cpu().numpy(), O.block_seeds(777, T, op.L(d_in))[0], E[0])
    assert np.array_equal(u64(b2[0]), B)


@pytest.mark.parametrize("transpose,d_out,d_in,T", [(False, 300, 2048, 5), (True, 700, 2100, 3), (False, 2048, 8192, 2)])
def test_digits_ntt_identical_to_tensor_core(phe, transpose, d_out, d_in, T):
    """Stage 1 of the packed primitive: NTT digits + bodies == tcgen05 digits + bodies (bitwise),
    and the packed result through phe_pack is the same."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(d_out, d_in, seed=d_out + d_in)
    x = synth.activations_int8(T, d_out if transpose else d_in, seed=T)
    S, seeds, body = encrypt(phe, p, x)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    dg, bd = phe.matmul_clear_digits(p, w, phe.ct_prepare(p, seeds, body), T)
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=transpose)
    dn, bn = phe.matmul_clear_digits_ntt(p, wn, phe.ntt_ct_prepare(p, tabs, seeds, body), T)
    assert torch.equal(bn, bd)
    assert torch.equal(dn, dg)
    if not transpose and d_out <= 2048:
        K = phe.KeySwitchKey(p, phe.ksk_gen(p, S, 3))
        assert torch.equal(phe.pack(p, dn, bn, K), phe.pack(p, dg, bd, K))

