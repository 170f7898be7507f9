"""Every Llama-3.2-1B linear shape at full size (north_star: "bit-exact encrypted W.[x] and
W^T.[g] for every Llama-3.2-1B linear layer"), forward and backward, through both mask
contractions (tcgen05 limb GEMM and the NTT domain), with the Table 1 parameters.

q_proj / o_proj (2048 x 2048) are covered at T = 2048 by test_gpu_parity / test_gpu_ntt; here:
k_proj / v_proj (512 x 2048, GQA), gate_proj / up_proj (8192 x 2048), down_proj (2048 x 8192,
L = 4 blocks), each as W.[x] and W^T.[g].  Per case: 4,000 sampled mask words against the C
oracle's O(d_in) closed form (Eq. 6 with SampleExtract at N-1), computed from the
oracle's own ChaCha20 re-expansion of the seeds; every (tau, j) output through the E = 0
decryption invariant b - <a, S> = Delta (M v)_j; the tc and NTT paths
word-identical; and the fused 39 -> 26 switch against the oracle's modswitch on the
sampled words."""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import phe_oracle as O
from oracle.phe_oracle import Params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

# (name, d_out, d_in) of Llama-3.2-1B (hidden 2048, intermediate 8192, 8 KV heads x 64)
SHAPES = [("k_proj", 512, 2048), ("gate_proj", 8192, 2048), ("down_proj", 2048, 8192)]


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("transpose", [False, True], ids=["fwd", "bwd_T"])
@pytest.mark.parametrize("name,d_out,d_in", SHAPES, ids=[s[0] for s in SHAPES])
def test_llama_linear_full_size(phe, coracle, name, d_out, d_in, transpose):
    p = phe.params(phe.PRESET_PAPER)
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma, eta=p.noise_eta)
    T = 512 if max(d_out, d_in) <= 2048 else 192
    W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED + d_out + 3 * d_in)
    M = np.ascontiguousarray(W.T) if transpose else W          # the matrix the server applies
    v_len, r_out = M.shape[1], M.shape[0]
    v = synth.gradients_int8(T, v_len) if transpose else synth.activations_int8(T, v_len)
    S = phe.keygen(p, 11)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(v).to(DEV), 4242)
    L = op.L(v_len)
    assert seeds.shape == (T, L)

    # tcgen05 path, q_in outputs
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    opnd = phe.ct_prepare(p, seeds, body)
    f = phe.matmul_clear_T if transpose else phe.matmul_clear
    m39, b39 = f(p, w, opnd, T, out_bits=39)
    torch.cuda.synchronize()
    assert m39.shape == (T, r_out, p.N) and b39.shape == (T, r_out)

    # (i) sampled mask words vs the oracle's closed form, masks re-expanded by the oracle
    rng = np.random.default_rng(d_out + d_in + int(transpose))
    n = 4000
    taus, js, ts = rng.integers(0, T, n), rng.integers(0, r_out, n), rng.integers(0, p.N, n)
    idx = [torch.from_numpy(a).to(DEV) for a in (taus, js, ts)]
    got = _u64(m39[idx[0], idx[1], idx[2]].contiguous())
    sd = _u64(seeds)
    for tau in np.unique(taus):
        sel = taus == tau
        A = np.stack([coracle.expand_mask(int(s), op.N, op.q_in) for s in sd[tau]])
        assert np.array_equal(got[sel], coracle.mask_entries(op, M, A, js[sel], ts[sel])), (name, tau)

    # (ii) every output: E = 0 decryption invariant == exact integer M v
    y = phe.decrypt_unpack(p, S, m39, b39, 39)
    mv = torch.from_numpy(v).to(DEV).double() @ torch.from_numpy(M).to(DEV).double().T
    assert torch.equal(y.double(), mv)

    # (iii) the NTT-domain contraction: identical words (switched to q_out in its epilogue) and
    # the tensor-core path's fused switch, both against the oracle's modswitch on the samples
    m26, b26 = f(p, w, opnd, T)
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=transpose)
    on = phe.ntt_ct_prepare(p, tabs, seeds, body)
    mn, bn = phe.matmul_clear_ntt(p, wn, on, T)
    torch.cuda.synchronize()
    assert torch.equal(bn, b26) and torch.equal(mn, m26)
    sw = m26[idx[0], idx[1], idx[2]].cpu().numpy().astype(np.uint32).astype(np.uint64)
    assert np.array_equal(sw, O.modswitch(got, 39, 26))
    y26 = phe.decrypt_unpack(p, S, m26, b26, 26).double()
    assert (y26 - mv).abs().max().item() <= 1 + int(S.sum().item())


@pytest.mark.parametrize("transpose", [False, True], ids=["fwd", "bwd_T"])
@pytest.mark.parametrize("name,d_out,d_in", SHAPES, ids=[s[0] for s in SHAPES])
def test_llama_linear_packed_training_step_config(phe, coracle, name, d_out, d_in, transpose):
    """The packed primitive (Eq. 6 -> Decomp digits -> Eq. 8 KeySwitch -> Eq. 7 rotate-sum ->
    switch; NEXT #1) per linear in bench.py's `stack_packed` launch configuration: T = 16 (the
    paper's training step, B = 1, C = 16), stage 1 in the NTT domain, stage 2 in the NTT
    domain.  Checked: the NTT stages == the tensor-core stages word for word (G = d_out / N groups,
    up to 4); one token against the oracle's own keygen, KSK, literal Eq. 6 and literal Eq. 7/8;
    every output decrypts to M v within the gamma-MSB contract."""
    p = phe.params(phe.PRESET_PAPER)
    T = 16
    W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED + d_out + 3 * d_in)
    M = np.ascontiguousarray(W.T) if transpose else W
    v_len, r_out = M.shape[1], M.shape[0]
    v = synth.gradients_int8(T, v_len) if transpose else synth.activations_int8(T, v_len)
    S = phe.keygen(p, 5)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(v).to(DEV), 77)
    ksk = phe.ksk_gen(p, S, 1234)
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=transpose)
    dig, bod = phe.matmul_clear_digits_ntt(p, wn, phe.ntt_ct_prepare(p, tabs, seeds, body), T)
    got = phe.pack_ntt(p, dig, bod, phe.NttKeySwitchKey(p, ksk))
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    dig_t, bod_t = phe.matmul_clear_digits(p, w, phe.ct_prepare(p, seeds, body), T)
    assert torch.equal(dig, dig_t) and torch.equal(bod, bod_t)
    ref = phe.pack(p, dig_t, bod_t, phe.KeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    G = (r_out + p.N - 1) // p.N
    assert got.shape == (T, G, 2, p.N) and torch.equal(got, ref)
    # one token through the oracle (O(rows L N^2) + O(rows 4 N^2) in C/OpenMP)
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma)
    So = O.keygen(5, op.N)
    KA, KB = coracle.ksk_gen(op, So, 1234, nthreads=os.cpu_count())
    seeds_o = O.block_seeds(77, T, op.L(v_len))
    assert np.array_equal(_u64(seeds), seeds_o)
    g = got.cpu().numpy().astype(np.uint32).astype(np.uint64)
    tau = 11
    A, B = O.encrypt(op, So, v[tau], seeds_o[tau])
    m, b = coracle.matmul_clear_literal(op, M, A, B, nthreads=os.cpu_count())
    PA, PB = coracle.pack(op, m, b, KA, KB, nthreads=os.cpu_count())
    assert np.array_equal(g[tau, :, 0], O.modswitch(PA, op.q_in, op.q_out))
    assert np.array_equal(g[tau, :, 1], O.modswitch(PB, op.q_in, op.q_out))
    y = phe.decrypt_packed(p, S, got, r_out).double()
    mv = torch.from_numpy(v).to(DEV).double() @ torch.from_numpy(M).to(DEV).double().T
    assert (y - mv).abs().max().item() < 2 ** 15
