"""Every output word of every Llama-3.2-1B linear, in bench.py's stack launch configuration,
against the oracle (-m gpu).

bench.py's default workload (BASELINE configs[3]: all linears x 16 layers, forward + W^T backward,
T = 2048 tokens) launches each registered linear on token chunks of 255 tokens (the largest output,
gate_up 16384 x 2048, at <= 34 GB per chunk; 255 = 5 tensor-core tiles of 51 tokens) and one ragged
chunk of 2048 - 8*255 = 8 tokens.  Here each registered shape runs at exactly those two chunk sizes
through the C ABI, with outputs at q_in (no switch) and then switched (the bench's form):

  * masks, ALL T x R x N words: Freivalds projections.  For random r_e in Z_Q^N,
      sum_t a_{tau,j}[t] r_e[t]  ==  oracle_mask_projection (sum_c W[j,c] (A_{tau,i} * r_e)[c mod N],
    the negacyclic product with the oracle's own ChaCha20 masks; derivation in oracle/phe_oracle.c).
    A word error e != 0 escapes one projection with probability <= 1/2 (an error in the top bit
    only), 2^-39 for an odd error; four independent r_e per (tau, j) bound any escape by 1/16 per
    output row, and a kernel fault flips many rows;
  * bodies, all T x R: sum_j rp[j] b_{tau,j} == oracle.body_projection;
  * 2,000 sampled mask words against the O(d_in) closed form (oracle_mask_entries);
  * the fused ModulusSwitch: the switched words of 4 whole tokens == the oracle's
    modswitch of the verified q_in words, plus the sampled words;
  * the NTT-domain contraction (NEXT #4) on the same inputs: identical words.

Inputs are independent of the CUDA path: seeds from the oracle's block_seeds, bodies uniform in
Z_Q from synth (the server cannot tell an encryption from a uniform body), W from synth.
"""
import os

import numpy as np
import pytest
import torch

import synth
from freivalds_util import NR, projections as _projections, r_limbs as _r_limbs
from oracle import phe_oracle as O
from oracle.phe_oracle import Params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"

# (name, d_out, d_in, transpose): the 8 distinct registrations of bench.py's stack workload
# (qkv / gate_up fused forward; q/o share 2048x2048, k/v 512x2048, gate/up 8192x2048 backward)
CASES = [("qkv", 3072, 2048, False), ("o", 2048, 2048, False), ("gate_up", 16384, 2048, False),
         ("down", 2048, 8192, False), ("q_T", 2048, 2048, True), ("k_T", 512, 2048, True),
         ("gate_T", 8192, 2048, True), ("down_T", 2048, 8192, True),
         # bench.py --bwd fused: dx of the fused projections (L = 2 with a half block; L = 8)
         ("qkv_T", 3072, 2048, True), ("gate_up_T", 16384, 2048, True)]


def _u64(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("T", [255, 8], ids=["chunk255", "tail8"])
@pytest.mark.parametrize("name,d_out,d_in,transpose", CASES, ids=[c[0] for c in CASES])
def test_all_outputs_vs_oracle(phe, coracle, name, d_out, d_in, transpose, T):
    p = phe.params(phe.PRESET_PAPER)
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma, eta=p.noise_eta)
    N, Q = op.N, op.Q
    W = synth.weights_int8(d_out, d_in, seed=synth.MASTER_SEED + d_out + 3 * d_in)
    M = np.ascontiguousarray(W.T) if transpose else W
    R, cols = M.shape
    L = op.L(cols)
    sbase = synth.seed_base(R + cols + T)
    seeds = O.block_seeds(sbase, T, L)                               # public seeds
    body = synth.uniform_u64((T, L, N), R + 7 * cols + T, op.q_in)  # bodies: uniform in Z_Q
    A = np.stack([np.stack([coracle.expand_mask(int(s), N, op.q_in) for s in seeds[t]]) for t in range(T)])

    sd = torch.from_numpy(seeds.view(np.int64)).to(DEV)
    bd = torch.from_numpy(body.view(np.int64)).to(DEV)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    opnd = phe.ct_prepare(p, sd, bd)
    f = phe.matmul_clear_T if transpose else phe.matmul_clear
    m39, b39 = f(p, w, opnd, T, out_bits=p.q_in)
    torch.cuda.synchronize()
    assert m39.shape == (T, R, N) and b39.shape == (T, R)

    rng = np.random.default_rng(R * 31 + cols + T)
    r = rng.integers(0, Q, size=(NR, N), dtype=np.uint64)
    got = _projections(m39, _r_limbs(r, DEV)) & np.uint64(Q - 1)
    want = coracle.mask_projection(op, M, A, r, nthreads=os.cpu_count())
    bad = np.argwhere(got != want)
    assert bad.size == 0, f"{name} T={T}: {len(bad)} (tau, j, e) projections differ, first {bad[:5].tolist()}"

    rp = rng.integers(0, Q, size=R, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bproj = (_u64(b39) * rp[None, :]).sum(-1, dtype=np.uint64) & np.uint64(Q - 1)
    assert np.array_equal(bproj, O.body_projection(op, M, body, rp))

    n = 2000
    taus, js, ts = rng.integers(0, T, n), rng.integers(0, R, n), rng.integers(0, N, n)
    idx = [torch.from_numpy(a).to(DEV) for a in (taus, js, ts)]
    words = _u64(m39[idx[0], idx[1], idx[2]].contiguous())
    for tau in np.unique(taus):
        sel = taus == tau
        assert np.array_equal(words[sel], coracle.mask_entries(op, M, A[tau], js[sel], ts[sel]))

    # the bench's form: switched to q_out in the epilogue
    m26, b26 = f(p, w, opnd, T)
    torch.cuda.synchronize()
    for tau in sorted({0, T - 1, T // 2, T // 3}):
        ms = m26[tau].cpu().numpy().astype(np.uint32).astype(np.uint64)
        assert np.array_equal(ms, O.modswitch(_u64(m39[tau]), op.q_in, op.q_out)), (name, tau)
    sw = m26[idx[0], idx[1], idx[2]].cpu().numpy().astype(np.uint32).astype(np.uint64)
    assert np.array_equal(sw, O.modswitch(words, op.q_in, op.q_out))
    assert np.array_equal(b26.cpu().numpy().astype(np.uint32).astype(np.uint64),
                          O.modswitch(_u64(b39), op.q_in, op.q_out))
    del m26, b26

    # NEXT #4: the NTT-domain contraction on the same inputs, identical q_in words (within its
    # CRT range: L <= phe_ntt_max_blocks, R23)
    if L > phe.ntt_max_blocks(p):
        return
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=transpose)
    mn, bn = phe.matmul_clear_ntt(p, wn, phe.ntt_ct_prepare(p, tabs, sd, bd), T, out_bits=p.q_in)
    torch.cuda.synchronize()
    assert torch.equal(mn, m39) and torch.equal(bn, b39)
