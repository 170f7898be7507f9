"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle.

Bar: ciphertext words bit-exact (integer work); decrypted plaintexts equal exact integer W x
(pre-switch, E = 0) or stay inside the post-switch bound 1 + hw(S) (P:198 contract).
Sizes: the oracle finishes in seconds and the shapes span several tiles and ragged tails;
the full-size case (bench launch configuration) is checked on sampled entries by the O(d_in)
closed form, on one full token by the literal path, and on every output by the decryption
invariant.
"""
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


def run_gpu(phe, p, W, x, sk_seed=7, sbase=12345, noise_seed=0, transpose=False, out_bits=None):
    S = phe.keygen(p, sk_seed)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), sbase, noise_seed)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    op = phe.ct_prepare(p, seeds, body)
    T = x.shape[0]
    f = phe.matmul_clear_T if transpose else phe.matmul_clear
    res = f(p, w, op, T, out_bits=out_bits)
    torch.cuda.synchronize()
    return S, seeds, body, w, op, res


def oracle_expect(coracle, p, M, x, sk_seed, sbase, noise_seed=0):
    """Oracle: its own keygen / expansion / encryption / literal Eq. 6 for matrix M."""
    op = oparams(p)
    S = O.keygen(sk_seed, op.N)
    T, d = x.shape
    L = op.L(d)
    seeds = O.block_seeds(sbase, T, L)
    E = O.noise(op, noise_seed, T, L)
    masks, bodies, Bs = [], [], []
    for tau in range(T):
        A, B = O.encrypt(op, S, x[tau], seeds[tau], E[tau])
        m, b = coracle.matmul_clear_literal(op, M, A, B, nthreads=os.cpu_count())
        masks.append(m); bodies.append(b); Bs.append(B)
    return S, seeds, np.stack(Bs), np.stack(masks), np.stack(bodies)


# ----------------------------------------------------------------------------- configs[0]
def test_toy_config_bit_exact(phe, coracle):
    """BASELINE configs[0]: toy RLWE N=1024, q 2^32 -> 2^28, 64x64, 16 tokens."""
    p = phe.params(phe.PRESET_TOY)
    W = synth.weights_int8(64, 64)
    x = synth.activations_int8(16, 64)
    S, seeds, body, w, opnd, (m32, b32) = run_gpu(phe, p, W, x, out_bits=p.q_in)
    So, seeds_o, B_o, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 12345)
    assert np.array_equal(S.cpu().numpy(), So)
    assert np.array_equal(u64(seeds), seeds_o)
    assert np.array_equal(u64(body), B_o)
    assert np.array_equal(u64(m32), mask_o) and np.array_equal(u64(b32), body_o)
    m28, b28 = phe.matmul_clear(p, w, opnd, 16, out_bits=p.q_out)
    assert np.array_equal(m28.cpu().numpy().astype(np.uint64), O.modswitch(mask_o, 32, 28))
    assert np.array_equal(b28.cpu().numpy().astype(np.uint64), O.modswitch(body_o, 32, 28))
    y = phe.decrypt_unpack(p, S, m28, b28, p.q_out).cpu().numpy()
    assert np.array_equal(y, (W.astype(np.int64) @ x.astype(np.int64).T).T)
    y32 = phe.decrypt_unpack(p, S, m32, b32, p.q_in).cpu().numpy()
    assert np.array_equal(y32, (W.astype(np.int64) @ x.astype(np.int64).T).T)


def test_toy_backward_transpose(phe, coracle):
    p = phe.params(phe.PRESET_TOY)
    W = synth.weights_int8(64, 48)           # d_out=64, d_in=48
    g = synth.gradients_int8(9, 64)           # g in Z^{d_out}
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, g, transpose=True, out_bits=p.q_in)
    _, _, _, mask_o, body_o = oracle_expect(coracle, p, np.ascontiguousarray(W.T), g, 7, 12345)
    assert m.shape == (9, 48, p.N)
    assert np.array_equal(u64(m), mask_o) and np.array_equal(u64(b), body_o)
    y = phe.decrypt_unpack(p, S, m, b, p.q_in).cpu().numpy()
    assert np.array_equal(y, (W.T.astype(np.int64) @ g.astype(np.int64).T).T)


# ----------------------------------------------------------------------------- paper params
@pytest.mark.parametrize("d_out,d_in,T", [(40, 3000, 7), (130, 2048, 53), (3, 768, 1), (256, 512, 60)])
def test_paper_params_bit_exact(phe, coracle, d_out, d_in, T):
    """Ragged rows (not a tile multiple), ragged last block, several token tiles."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(d_out, d_in, seed=d_out * 7 + d_in)
    x = synth.activations_int8(T, d_in, seed=T + d_in)
    S, seeds, body, w, opnd, (m39, b39) = run_gpu(phe, p, W, x, sbase=99 + T, out_bits=p.q_in)
    _, _, B_o, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 99 + T)
    assert np.array_equal(u64(body), B_o)
    assert np.array_equal(u64(b39), body_o)
    assert np.array_equal(u64(m39), mask_o)
    m26, b26 = phe.matmul_clear(p, w, opnd, T)
    assert np.array_equal(m26.cpu().numpy().astype(np.uint64), O.modswitch(mask_o, 39, 26))
    assert np.array_equal(b26.cpu().numpy().astype(np.uint64), O.modswitch(body_o, 39, 26))
    wx = (W.astype(np.int64) @ x.astype(np.int64).T).T
    assert np.array_equal(phe.decrypt_unpack(p, S, m39, b39, 39).cpu().numpy(), wx)  # E = 0: exact
    err = phe.decrypt_unpack(p, S, m26, b26, 26).cpu().numpy().astype(np.int64) - wx
    assert np.abs(err).max() <= 1 + int(S.sum().item())
    assert np.all(np.abs(err) < 2 ** 15)  # gamma = 12 MSBs of beta = 27 preserved


def test_row_sharding_equals_slices(phe):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(300, 2048)
    x = synth.activations_int8(20, 2048)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x)
    for r0, r1 in [(0, 128), (128, 300), (17, 18), (5, 5)]:
        ms, bs = phe.matmul_clear(p, w, opnd, 20, row_begin=r0, row_end=r1)
        assert torch.equal(ms, m[:, r0:r1]) and torch.equal(bs, b[:, r0:r1])


def test_row_ranges_partial_block_vs_oracle(phe, coracle):
    """A partial last block (d_in = 700 < N) runs the mask GEMM with CTA pairs over rows (j, j+1):
    odd row counts and row ranges that end inside a pair (the partner row is computed but its
    stores fall outside the range) give exactly the oracle's rows."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(301, 700, seed=4)
    x = synth.activations_int8(9, 700, seed=5)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x, out_bits=p.q_in)
    _, _, _, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 12345)
    assert np.array_equal(u64(m), mask_o) and np.array_equal(u64(b), body_o)
    for r0, r1 in [(17, 18), (5, 128), (0, 301), (299, 301), (100, 233)]:
        ms, bs = phe.matmul_clear(p, w, opnd, 9, out_bits=p.q_in, row_begin=r0, row_end=r1)
        assert np.array_equal(u64(ms), mask_o[:, r0:r1]) and np.array_equal(u64(bs), body_o[:, r0:r1])


def test_multiblock_L4_and_noise(phe, coracle):
    """d_in = 8192 (down_proj, L = 4) with CBD(21) noise in the encryption."""
    p = phe.params(phe.PRESET_PAPER, noise_eta=21)
    W = synth.weights_int8(6, 8192)
    x = synth.activations_int8(3, 8192)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x, noise_seed=55, out_bits=39)
    _, _, B_o, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 12345, noise_seed=55)
    assert np.array_equal(u64(body), B_o)
    assert np.array_equal(u64(m), mask_o) and np.array_equal(u64(b), body_o)


def test_extreme_limbs_and_weights(phe, coracle):
    """All limb bytes at their maxima and |w| = 127 everywhere: largest int32 partial sums."""
    p = phe.params(phe.PRESET_PAPER)
    op = oparams(p)
    d_out, d_in, T = 4, 8192, 3
    W = np.where(synth.uniform_int8((d_out, d_in), 3) >= 0, 127, -127).astype(np.int8)
    W[0] = 127
    W[1] = -127
    L = op.L(d_in)
    # hand-built operand: masks (2^39 - 1 or random) via limb planes, bodies 2^39 - 1
    A = np.full((T, L, op.N), 2 ** 39 - 1, np.uint64)
    A[2] = synth.uniform_u64((L, op.N), 9, 39)
    Bv = np.full((T, L, op.N), 2 ** 39 - 1, np.uint64)
    nbytes = phe.load().phe_ct_operand_bytes(__import__("ctypes").byref(p), T, L)
    rows = nbytes // (2 * L * op.N)
    planes = np.zeros((2, rows, L * op.N), np.uint8)
    for tau in range(T):
        for l in range(5):
            planes[0, tau * 5 + l] = ((A[tau].reshape(-1) >> np.uint64(8 * l)) & np.uint64(255)).astype(np.uint8)
            planes[1, tau * 5 + l] = ((Bv[tau].reshape(-1) >> np.uint64(8 * l)) & np.uint64(255)).astype(np.uint8)
    opnd = torch.from_numpy(planes.reshape(-1)).to(DEV)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    m, b = phe.matmul_clear(p, w, opnd, T, out_bits=39)
    for tau in range(T):
        mo, bo = coracle.matmul_clear_literal(op, W, A[tau], Bv[tau], nthreads=os.cpu_count())
        assert np.array_equal(u64(m[tau]), mo) and np.array_equal(u64(b[tau]), bo)


@pytest.mark.parametrize("pos", ["first", "last", "middle", "unaligned_tail"])
def test_weight_minus_128_refused_on_both_paths(phe, pos):
    """w = -128 lies outside symmetric int8 quantization's [-127, 127] and
    encode_weights refuses out-of-range weights: both registrations (tensor-core and
    NTT, forward and W^T) return PHE_ERANGE instead of computing with it.  Positions cover the
    range kernel's unaligned head, 16-byte body and tail."""
    p = phe.params(phe.PRESET_PAPER)
    d_out, d_in = 37, 2100
    W = synth.weights_int8(d_out, d_in, seed=3)
    flat = torch.from_numpy(W.reshape(-1).copy())
    buf = torch.zeros(flat.numel() + 1, dtype=torch.int8)
    off = 1 if pos == "unaligned_tail" else 0   # W starting 1 byte past a 16-byte boundary
    k = {"first": 0, "last": flat.numel() - 1, "middle": flat.numel() // 2 + 5,
         "unaligned_tail": flat.numel() - 3}[pos]
    flat[k] = -128
    buf[off: off + flat.numel()] = flat
    Wd = buf.to(DEV)[off: off + flat.numel()].view(d_out, d_in)
    tabs = phe.NttTables(p)
    for tr in (False, True):
        with pytest.raises(phe.PheError, match="out of range"):
            phe.Weights(p, Wd, transpose=tr)
        with pytest.raises(phe.PheError, match="out of range"):
            phe.NttWeights(p, tabs, Wd, transpose=tr)
    flat[k] = -127                               # the same matrix inside the range registers
    buf[off: off + flat.numel()] = flat
    Wd = buf.to(DEV)[off: off + flat.numel()].view(d_out, d_in)
    phe.Weights(p, Wd)
    phe.NttWeights(p, tabs, Wd)


def test_full_int8_range_both_paths_vs_oracle(phe, coracle):
    """Every weight value the paths accept, [-127, 127], with the extremes on both halves of the
    Hankel operand (the negacyclic wrap stores -w): tensor-core and NTT paths bit-exact vs the
    oracle's literal Eq. 6, forward and W^T."""
    p = phe.params(phe.PRESET_PAPER)
    op = oparams(p)
    W = synth.uniform_int8((70, 2100), 31, -127, 127)
    W[0, :] = -127
    W[1, :] = 127
    W[2, ::2] = -127
    for tr in (False, True):
        M = np.ascontiguousarray(W.T) if tr else W
        x = synth.uniform_int8((3, M.shape[1]), 5 + tr, -127, 127)
        S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x, transpose=tr, out_bits=39)
        tabs = phe.NttTables(p)
        wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV), transpose=tr)
        mn, bn = phe.matmul_clear_ntt(p, wn, phe.ntt_ct_prepare(p, tabs, seeds, body), 3, out_bits=39)
        sd, bd = u64(seeds), u64(body)
        for tau in range(3):
            A = np.stack([coracle.expand_mask(int(s_), op.N, op.q_in) for s_ in sd[tau]])
            mo, bo = coracle.matmul_clear_literal(op, M, A, bd[tau], nthreads=os.cpu_count())
            assert np.array_equal(u64(m[tau]), mo) and np.array_equal(u64(b[tau]), bo)
            assert np.array_equal(u64(mn[tau]), mo) and np.array_equal(u64(bn[tau]), bo)


def test_matmul_clear_ct_one_call(phe):
    """phe_matmul_clear_ct (north_star's matmul_clear(W, ct)) == ct_prepare + matmul_clear[_T]."""
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(300, 2100)
    x = synth.activations_int8(9, 2100)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x)
    m1, b1 = phe.matmul_clear_ct(p, w, seeds, body, row_begin=7, row_end=299)
    assert torch.equal(m1, m[:, 7:299]) and torch.equal(b1, b[:, 7:299])
    g = synth.gradients_int8(5, 300)
    S, sg, bg, wT, og, (mT, bT) = run_gpu(phe, p, W, g, transpose=True)
    mT1, bT1 = phe.matmul_clear_ct(p, wT, sg, bg)
    assert torch.equal(mT1, mT) and torch.equal(bT1, bT)
    small = torch.empty(16, dtype=torch.uint8, device=DEV)
    with pytest.raises(phe.PheError, match="buffer too small"):
        phe.matmul_clear_ct(p, w, seeds, body, ws=small)


def test_simt_cross_check_matches_tensor_core(phe):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(24, 4100)
    x = synth.activations_int8(70, 4100)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x)
    ms, bs = phe.matmul_clear_simt(p, torch.from_numpy(W).to(DEV), opnd, 70)
    assert torch.equal(ms, m) and torch.equal(bs, b)


def test_empty_and_single_token(phe, coracle):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(8, 2048)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    empty = torch.zeros(phe.load().phe_ct_operand_bytes(__import__("ctypes").byref(p), 0, 1),
                        dtype=torch.uint8, device=DEV)
    m, b = phe.matmul_clear(p, w, empty, 0)
    assert m.shape == (0, 8, 2048)
    x = synth.activations_int8(1, 2048)
    S, seeds, body, w, opnd, (m1, b1) = run_gpu(phe, p, W, x, out_bits=39)
    _, _, _, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 12345)
    assert np.array_equal(u64(m1), mask_o) and np.array_equal(u64(b1), body_o)


# ----------------------------------------------------------------------------- side kernels
def test_modswitch_kernel(phe):
    v = synth.uniform_u64(100003, 4, 39)
    out = phe.modswitch(torch.from_numpy(v.view(np.int64)).to(DEV), 39, 26)
    assert np.array_equal(out.cpu().numpy().astype(np.uint64), O.modswitch(v, 39, 26))
    v2 = synth.uniform_u64(1000, 5, 32)
    out2 = phe.modswitch(torch.from_numpy(v2.view(np.int64)).to(DEV), 32, 28)
    assert np.array_equal(out2.cpu().numpy().astype(np.uint64), O.modswitch(v2, 32, 28))


def test_keygen_and_encrypt_match_oracle(phe):
    p = phe.params(phe.PRESET_PAPER, noise_eta=21)
    op = oparams(p)
    S = phe.keygen(p, 2 ** 64 - 3)
    So = O.keygen(2 ** 64 - 3, op.N)
    assert np.array_equal(S.cpu().numpy(), So)
    x = synth.activations_int8(2, 2500)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 2 ** 63 + 11, 77)
    E = O.noise(op, 77, 2, 2)
    for tau in range(2):
        A, B = O.encrypt(op, So, x[tau], u64(seeds)[tau], E[tau])
        assert np.array_equal(u64(body)[tau], B)
        dec = np.concatenate([O.decrypt_rlwe(A[i], B[i], So, op) for i in range(2)])
        assert np.array_equal(dec[:2500], x[tau].astype(np.int64))


# ----------------------------------------------------------------------------- host path
def test_server_matvec_host_matches_device(phe):
    p = phe.params(phe.PRESET_PAPER)
    W = synth.weights_int8(64, 2048)
    x = synth.activations_int8(100, 2048)
    S, seeds, body, w, opnd, (m, b) = run_gpu(phe, p, W, x)
    hs = seeds.cpu().pin_memory()
    hb = body.cpu().pin_memory()
    hm = torch.empty((100, 64, p.N), dtype=torch.int32).pin_memory()
    hbo = torch.empty((100, 64), dtype=torch.int32).pin_memory()
    phe.server_matvec_host(p, w, hs, hb, hm, hbo, chunk_tokens=33)
    assert torch.equal(hm, m.cpu()) and torch.equal(hbo, b.cpu())


# ----------------------------------------------------------------------------- full size
@pytest.mark.slow
def test_full_size_q_proj_bench_config(phe, coracle):
    """configs[1] in bench.py's launch configuration: q_proj 2048x2048, T = 2048 tokens.
    (i) 10^4 random (tau, j, t) mask entries by the closed form, (ii) one full token by the
    literal path, (iii) all 4.2M (tau, j) outputs through the E = 0 decryption invariant."""
    p = phe.params(phe.PRESET_PAPER)
    op = oparams(p)
    d, T = 2048, 2048
    W = synth.weights_int8(d, d)
    x = synth.activations_int8(T, d)
    S, seeds, body, w, opnd, (m39, b39) = run_gpu(phe, p, W, x, out_bits=39)
    rng = np.random.default_rng(0)
    taus = rng.integers(0, T, 10000)
    js = rng.integers(0, d, 10000)
    ts = rng.integers(0, op.N, 10000)
    sd = u64(seeds)
    got = m39[torch.from_numpy(taus).to(DEV), torch.from_numpy(js).to(DEV), torch.from_numpy(ts).to(DEV)]
    got = got.cpu().numpy().view(np.uint64)
    for tau in np.unique(taus):
        sel = taus == tau
        A = O.expand_mask(int(sd[tau, 0]), op.N, op.q_in)[None]
        ref = coracle.mask_entries(op, W, A, js[sel], ts[sel])
        assert np.array_equal(got[sel], ref)
    tau = 1234
    A = O.expand_mask(int(sd[tau, 0]), op.N, op.q_in)[None]
    mo, bo = coracle.matmul_clear_literal(op, W, A, u64(body)[tau], nthreads=os.cpu_count())
    assert np.array_equal(u64(m39[tau]), mo) and np.array_equal(u64(b39)[tau], bo)
    y = phe.decrypt_unpack(p, S, m39, b39, 39)
    wx = (torch.from_numpy(x).to(DEV).double() @ torch.from_numpy(W).to(DEV).double().T)
    assert torch.equal(y.double(), wx)
    # (iv) all 8.6e9 mask words: NR Freivalds projections per (tau, j) vs the oracle's
    # (A_tau * r) . W with the oracle's own mask expansion (tests/test_gpu_freivalds.py)
    from freivalds_util import NR, projections, r_limbs
    seeds_o = O.block_seeds(12345, T, 1)
    assert np.array_equal(sd, seeds_o)
    A_all = np.stack([coracle.expand_mask(int(s_), op.N, op.q_in)[None] for s_ in seeds_o[:, 0]])
    r = rng.integers(0, op.Q, size=(NR, op.N), dtype=np.uint64)
    got = projections(m39, r_limbs(r, DEV)) & np.uint64(op.Q - 1)
    assert np.array_equal(got, coracle.mask_projection(op, W, A_all, r, nthreads=os.cpu_count()))
    del m39
    m26, b26 = phe.matmul_clear(p, w, opnd, T)
    y26 = phe.decrypt_unpack(p, S, m26, b26, 26).double()
    assert (y26 - wx).abs().max().item() <= 1 + int(S.sum().item())


# ----------------------------------------------------------------------------- other parameter sets
@pytest.mark.parametrize("over,d_out,d_in,T", [
    (dict(N=512, q_in=39, q_out=26, beta=27), 40, 1100, 9),     # P1-like ring, L = 3, 2-CTA path
    (dict(N=4096, q_in=39, q_out=26, beta=27), 5, 4096, 3),     # P3 ring
    (dict(N=2048, q_in=32, q_out=24, beta=27), 33, 2048, 70),   # P2: ell = 4, s = 8 (generic epilogue)
    (dict(N=256, q_in=48, q_out=30, beta=27), 17, 300, 11),     # ell = 6: 1-CTA fallback kernel
    (dict(N=256, q_in=20, q_out=16, beta=12, gamma=8), 9, 256, 100),  # ell = 3, 1-CTA kernel
])
def test_parameter_sets_bit_exact(phe, coracle, over, d_out, d_in, T):
    p = phe.params(phe.PRESET_PAPER, **over)
    W = synth.uniform_int8((d_out, d_in), d_in + T, -127, 127)
    x = synth.uniform_int8((T, d_in), d_out + T, -7, 7)
    S, seeds, body, w, opnd, (mq, bq) = run_gpu(phe, p, W, x, out_bits=p.q_in)
    _, _, B_o, mask_o, body_o = oracle_expect(coracle, p, W, x, 7, 12345)
    assert np.array_equal(u64(body), B_o)
    assert np.array_equal(u64(mq), mask_o) and np.array_equal(u64(bq), body_o)
    ms, bs = phe.matmul_clear(p, w, opnd, T)
    assert np.array_equal(ms.cpu().numpy().astype(np.uint32).astype(np.uint64), O.modswitch(mask_o, p.q_in, p.q_out))
    assert np.array_equal(bs.cpu().numpy().astype(np.uint32).astype(np.uint64), O.modswitch(body_o, p.q_in, p.q_out))
