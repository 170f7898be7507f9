"""GPU parity of stage 2 of the packed primitive in the NTT domain (phe_pack_ntt: Eq. 7 + Eq. 8,
P:187-191, exchanged into sum_{l,i} D_{l,i}(X) * KSK_{l,i}(X)) against the CPU
oracle's literal Eq. 7 and against the tensor-core packing GEMM (phe_pack), bit-exactly."""
import os

import numpy as np
import pytest
import torch

import synth
from oracle import phe_oracle as O
from oracle.phe_oracle import Params

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def _setup(phe, over, d_out, d_in, T, eta, transpose=False, seed=0):
    p = phe.params(phe.PRESET_PAPER, noise_eta=eta, **over)
    W = synth.weights_int8(d_out, d_in, seed=d_out + d_in + seed)
    cols = d_out if transpose else d_in
    x = synth.activations_int8(T, cols, seed=T + cols + seed)
    S = phe.keygen(p, 5)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77, 3)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV), transpose=transpose)
    opnd = phe.ct_prepare(p, seeds, body)
    ksk = phe.ksk_gen(p, S, 1234)
    return p, W, x, S, w, opnd, ksk


@pytest.mark.parametrize("over,d_out,d_in,T,eta", [
    (dict(N=256), 512, 300, 3, 0),          # G = 2 groups, ragged input block
    (dict(N=256), 300, 256, 2, 21),         # rows not a multiple of 256 (zeroed pad rows), noisy KSK
    (dict(N=512), 700, 512, 2, 0),          # G = 2, second group ragged (rows beyond R256)
])
def test_pack_ntt_bit_exact_vs_oracle(phe, coracle, over, d_out, d_in, T, eta):
    p, W, x, S, w, opnd, ksk = _setup(phe, over, d_out, d_in, T, eta)
    dig, bod = phe.matmul_clear_digits(p, w, opnd, T)
    got_t = phe.pack_ntt(p, dig, bod, phe.NttKeySwitchKey(p, ksk))
    ref_t = phe.pack(p, dig, bod, phe.KeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    assert torch.equal(got_t, ref_t)
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma, eta=eta)
    So = O.keygen(5, op.N)
    KA, KB = coracle.ksk_gen(op, So, 1234, eta=eta, nthreads=os.cpu_count())
    seeds_o = O.block_seeds(77, T, op.L(d_in))
    E = O.noise(op, 3, T, op.L(d_in))
    got = got_t.cpu().numpy().astype(np.uint32).astype(np.uint64)
    for tau in range(T):
        A, B = O.encrypt(op, So, x[tau], seeds_o[tau], E[tau])
        m, b = coracle.matmul_clear_literal(op, W, A, B, nthreads=os.cpu_count())
        PA, PB = coracle.pack(op, m, b, KA, KB, nthreads=os.cpu_count())
        assert np.array_equal(got[tau, :, 0], O.modswitch(PA, op.q_in, op.q_out))
        assert np.array_equal(got[tau, :, 1], O.modswitch(PB, op.q_in, op.q_out))
    wx = (W.astype(np.int64) @ x.astype(np.int64).T).T
    y = phe.decrypt_packed(p, S, got_t, d_out).cpu().numpy().astype(np.int64)
    assert np.all(np.abs(y - wx) < 2 ** 15)  # top gamma = 12 of beta = 27 bits


@pytest.mark.parametrize("over,d_out,d_in,T,transpose", [
    (dict(N=1024), 1100, 1024, 3, False),
    (dict(N=2048), 2048, 2048, 3, False),   # Table 1 ring, q_proj rows
    (dict(N=2048), 700, 2100, 2, True),     # W^T (backward), ragged
    (dict(N=4096), 300, 4096, 1, False),
    (dict(N=8192), 256, 8192, 1, False),
])
def test_pack_ntt_identical_to_tensor_core(phe, over, d_out, d_in, T, transpose):
    """Every log2 N the kernel is instantiated for: phe_pack_ntt == phe_pack word for word (Eq. 7
    defines the words uniquely; phe_pack is oracle-pinned in test_gpu_pack.py)."""
    p, W, x, S, w, opnd, ksk = _setup(phe, over, d_out, d_in, T, 0, transpose)
    dig, bod = phe.matmul_clear_digits(p, w, opnd, T)
    got = phe.pack_ntt(p, dig, bod, phe.NttKeySwitchKey(p, ksk))
    ref = phe.pack(p, dig, bod, phe.KeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


@pytest.mark.parametrize("dval,kval", [(-128, 1 << 38), (127, (1 << 38) - 1)])
def test_pack_ntt_crt_range_adversarial(phe, dval, kval):
    """Every digit at an extreme and every KSK word at the largest centred magnitude: the exact
    sums reach 4N * N * 128 * 2^38 in magnitude, the top of the CRT range the launch admits."""
    p = phe.params(phe.PRESET_PAPER, N=256)
    N, T, R = p.N, 2, 256
    dig = torch.full((T, R, 4, N), dval, dtype=torch.int8, device=DEV)
    bod = torch.zeros((T, R), dtype=torch.int64, device=DEV)
    ksk = torch.full((2, 4 * N, N), kval, dtype=torch.int64, device=DEV)
    got = phe.pack_ntt(p, dig, bod, phe.NttKeySwitchKey(p, ksk))
    ref = phe.pack(p, dig, bod, phe.KeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    # closed form: D_{l,i} = d * sum_r X^r and K = k * sum_c X^c for every (l, i), so coefficient
    # c of the negacyclic product is d k (#{r + s = c} - #{r + s = c + N}) = d k (2c + 2 - N)
    c = np.arange(N, dtype=np.int64)
    acc = (4 * N * dval * (2 * c + 2 - N)).astype(object) * ((kval - (1 << 39)) if kval >= 1 << 38 else kval)
    A = np.array([(-v) % (1 << 39) for v in acc], dtype=np.uint64)
    exp = O.modswitch(A, 39, 26)
    assert np.array_equal(got[0, 0, 0].cpu().numpy().astype(np.uint32).astype(np.uint64), exp)


def test_pack_ntt_empty_and_errors(phe):
    p = phe.params(phe.PRESET_PAPER, N=256)
    ksk = torch.zeros((2, 4 * 256, 256), dtype=torch.int64, device=DEV)
    nk = phe.NttKeySwitchKey(p, ksk)
    dig = torch.zeros((0, 256, 4, 256), dtype=torch.int8, device=DEV)
    bod = torch.zeros((0, 256), dtype=torch.int64, device=DEV)
    out = phe.pack_ntt(p, dig, bod, nk)
    assert out.shape == (0, 1, 2, 256)
    with pytest.raises(phe.PheError):
        phe.pack_ntt(p, torch.zeros((1, 256, 4, 256), dtype=torch.int8, device=DEV),
                     torch.zeros((1, 256), dtype=torch.int64, device=DEV), nk,
                     ws=torch.empty(16, dtype=torch.uint8, device=DEV))
    # both stages in the NTT domain (its smallest ring, N = 512): T = 0 is a no-op, a short
    # workspace is refused
    p5 = phe.params(phe.PRESET_PAPER, N=512)
    nk5 = phe.NttKeySwitchKey(p5, torch.zeros((2, 4 * 512, 512), dtype=torch.int64, device=DEV))
    tabs = phe.NttTables(p5)
    wn = phe.NttWeights(p5, tabs, torch.from_numpy(synth.weights_int8(700, 512, seed=9)).to(DEV))
    opnd = torch.empty(phe.load().phe_ntt_operand_bytes(__import__("ctypes").byref(p5), 1, 1), dtype=torch.uint8,
                       device=DEV)
    out0 = phe.matmul_clear_packed_nttw(p5, wn, opnd, 0, nk5)
    assert out0.shape == (0, 2, 2, 512)
    with pytest.raises(phe.PheError):
        phe.matmul_clear_packed_nttw(p5, wn, opnd, 1, nk5, ws=torch.empty(16, dtype=torch.uint8, device=DEV))


def test_packed_ntt_primitive_and_wire_host(phe):
    """phe_matmul_clear_packed_ntt == phe_matmul_clear_packed (whole primitive), and the wire-byte
    host pipeline with the NTT packing stage == the tensor-core one, byte for byte."""
    p, W, x, S, w, opnd, ksk = _setup(phe, dict(N=2048), 2048, 2048, 5, 0)
    K, NK = phe.KeySwitchKey(p, ksk), phe.NttKeySwitchKey(p, ksk)
    ref = phe.matmul_clear_packed(p, w, opnd, 5, K)
    got = phe.matmul_clear_packed_ntt(p, w, opnd, 5, NK)
    assert torch.equal(got, ref)
    T = 5
    s2, b2 = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77, 3)  # the ciphertexts behind opnd
    hi = phe.wire_serialize_inputs(p, s2, b2).cpu().pin_memory()
    ho_ref = torch.empty((T, 1, phe.wire_output_bytes(p)), dtype=torch.uint8).pin_memory()
    ho_ntt = torch.empty_like(ho_ref).pin_memory()
    phe.server_wire_host(p, w, K, hi, ho_ref, chunk_tokens=2)
    phe.server_wire_host_ntt(p, w, NK, hi, ho_ntt, chunk_tokens=2)
    assert torch.equal(ho_ref, ho_ntt)
    assert torch.equal(phe.wire_deserialize_packed(p, ho_ntt.to(DEV)).view(T, 1, 2, p.N), ref)
    # both stages in the NTT domain (NTT weights + NTT operand): the same words and wire bytes
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV))
    got_w = phe.matmul_clear_packed_nttw(p, wn, phe.ntt_ct_prepare(p, tabs, s2, b2), T, NK)
    assert torch.equal(got_w, ref)
    ho_w = torch.empty_like(ho_ref).pin_memory()
    phe.server_wire_host_nttw(p, wn, NK, hi, ho_w, chunk_tokens=2)
    assert torch.equal(ho_w, ho_ref)


def test_wire_host_ragged_last_chunk(phe):
    """the NTT packing workspace is not monotone in T (the K-split follows wave fill;
    q_proj: T = 7 needs more than T = 8), so a host pipeline sized for the full chunk failed with
    ENOMEM on a shorter last chunk.  T = 15 in chunks of 8: all three wire pipelines == the device
    primitive; the workspace query covers both chunk sizes; a short workspace is refused."""
    import ctypes
    p, W, x, S, w, opnd, ksk = _setup(phe, dict(N=2048), 2048, 2048, 15, 0)
    K, NK = phe.KeySwitchKey(p, ksk), phe.NttKeySwitchKey(p, ksk)
    ref = phe.matmul_clear_packed(p, w, opnd, 15, K)
    s2, b2 = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77, 3)
    hi = phe.wire_serialize_inputs(p, s2, b2).cpu().pin_memory()
    tabs = phe.NttTables(p)
    wn = phe.NttWeights(p, tabs, torch.from_numpy(W).to(DEV))
    lib = phe.load()
    for fn, wt, key, api in [(phe.server_wire_host, w, K, "phe_server_wire_host"),
                             (phe.server_wire_host_ntt, w, NK, "phe_server_wire_host_ntt"),
                             (phe.server_wire_host_nttw, wn, NK, "phe_server_wire_host_nttw")]:
        need = getattr(lib, api + "_ws_bytes")(ctypes.byref(p), 2048, 2048, 0, 15, 8)
        ws_fn = lib.phe_packed_ntt_ws_bytes if api != "phe_server_wire_host" else lib.phe_packed_ws_bytes
        assert need >= 2 * max(ws_fn(ctypes.byref(p), 2048, 8), ws_fn(ctypes.byref(p), 2048, 7))
        ho = torch.empty((15, 1, phe.wire_output_bytes(p)), dtype=torch.uint8).pin_memory()
        fn(p, wt, key, hi, ho, chunk_tokens=8)
        assert torch.equal(phe.wire_deserialize_packed(p, ho.to(DEV)).view(15, 1, 2, p.N), ref), api
    # the C ABI refuses a workspace one byte short (ENOMEM), before enqueueing anything
    need = lib.phe_server_wire_host_ntt_ws_bytes(ctypes.byref(p), 2048, 2048, 0, 15, 8)
    ws = torch.empty(need - 1, dtype=torch.uint8, device=DEV)
    ho = torch.empty((15, 1, phe.wire_output_bytes(p)), dtype=torch.uint8).pin_memory()
    rc = lib.phe_server_wire_host_ntt(ctypes.byref(p), w.buf.data_ptr(), 2048, 2048, 0, NK.buf.data_ptr(),
                                      hi.data_ptr(), 15, 8, ho.data_ptr(), ws.data_ptr(), ws.numel(), None)
    assert rc == phe.PHE_ENOMEM


@pytest.mark.slow
def test_full_size_q_proj_packed_bench_config(phe, coracle):
    """bench.py --workload q_proj_packed in its launch configuration (q_proj 2048x2048, T = 2048,
    Table 1): (i) every packed word of all 2048 tokens through phe_matmul_clear_packed_ntt equals
    the tensor-core primitive's; (ii) two sampled tokens against the oracle's own keygen, KSK,
    encryption, literal Eq. 6 and literal Eq. 7/8; (iii) all 4.2M packed outputs decrypt to W.x
    within the gamma-MSB contract."""
    p = phe.params(phe.PRESET_PAPER)
    d, T = 2048, 2048
    W = synth.weights_int8(d, d)
    x = synth.activations_int8(T, d)
    S = phe.keygen(p, 5)
    seeds, body = phe.encrypt_pack(p, S, torch.from_numpy(x).to(DEV), 77)
    w = phe.Weights(p, torch.from_numpy(W).to(DEV))
    opnd = phe.ct_prepare(p, seeds, body)
    ksk = phe.ksk_gen(p, S, 1234)
    got = phe.matmul_clear_packed_ntt(p, w, opnd, T, phe.NttKeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    ref = phe.matmul_clear_packed(p, w, opnd, T, phe.KeySwitchKey(p, ksk))
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    del ref
    phe._ws_cache.clear()
    op = Params(N=p.N, q_in=p.q_in, q_out=p.q_out, beta=p.beta, gamma=p.gamma)
    So = O.keygen(5, op.N)
    KA, KB = coracle.ksk_gen(op, So, 1234, nthreads=os.cpu_count())
    seeds_o = O.block_seeds(77, T, 1)
    g = got.cpu().numpy().astype(np.uint32).astype(np.uint64)
    for tau in (0, 1733):
        A, B = O.encrypt(op, So, x[tau], seeds_o[tau])
        m, b = coracle.matmul_clear_literal(op, W, A, B, nthreads=os.cpu_count())
        PA, PB = coracle.pack(op, m, b, KA, KB, nthreads=os.cpu_count())
        assert np.array_equal(g[tau, :, 0], O.modswitch(PA, op.q_in, op.q_out))
        assert np.array_equal(g[tau, :, 1], O.modswitch(PB, op.q_in, op.q_out))
    y = phe.decrypt_packed(p, S, got, d).double()
    wx = torch.from_numpy(x).to(DEV).double() @ torch.from_numpy(W).to(DEV).double().T
    assert (y - wx).abs().max().item() < 2 ** 15
