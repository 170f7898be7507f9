"""Pins for the NEXT #1 oracle (KeySwitch packing, Eq. 7 + Eq. 8), -m "not gpu".

Key external pin: with an exact gadget decomposition (base_log * levels = q) and noiseless
keys, KeySwitch is an algebraic identity: B' - A'S = b - <a, S'> in coefficient 0 and 0
elsewhere.  So keyswitched / packed ciphertexts must decrypt exactly, whatever the code does
internally.  The paper's (8, 3) decomposition then only adds the bounded rounding term.
"""
import os

import numpy as np
import pytest

from oracle import phe_oracle as O
from oracle.phe_oracle import Params
import synth

U64 = np.uint64


def test_decompose_spec_examples():
    assert O.decompose(0, 39) == [0, 0, 0, 0] and O.decompose(0, 39, 8, 3) == [0, 0, 0]
    assert O.decompose(0x50, 8, 4, 2) == [5, 0]
    d = O.decompose(0x78, 8, 4, 2)
    assert O.recompose(d, 8, 4) == 0x78 and all(-8 <= x < 8 for x in d)


def test_decompose_exhaustive_exact_when_no_tail():
    for v in range(256):                                               # S:67, exhaustive
        d = O.decompose(v, 8, 4, 2)
        assert O.recompose(d, 8, 4) == v and all(-8 <= x < 8 for x in d)


@pytest.mark.parametrize("levels", [3, 4])
def test_decompose_paper_params_error_bound(levels):
    vals = synth.uniform_u64(3000, 41, 39)
    for v in vals:
        d = O.decompose(int(v), 39, 8, levels)
        assert len(d) == levels and all(-128 <= x < 128 for x in d)
        err = (int(v) - O.recompose(d, 39, 8)) % 2 ** 39
        err = err - 2 ** 39 if err >= 2 ** 38 else err
        assert abs(err) <= 2 ** (39 - 8 * levels - 1)                  # S:32 invariant


def _small():
    return Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)


def test_ksk_entries_decrypt_to_scaled_key_bits():
    P = _small()
    S = O.keygen(5, P.N)
    KA, KB = O.ksk_gen(P, S, 99, base_log=13, levels=3)
    for l in range(3):  # exact 39-bit gadget (13 x 3)
        for i in range(P.N):
            r = l * P.N + i
            AS = O.negacyclic_mul(KA[r], S.astype(np.int64), 39)
            phase = (KB[r] - AS) & U64(2 ** 39 - 1)
            exp = np.zeros(P.N, U64)
            exp[0] = int(S[i]) << (39 - (l + 1) * 13)
            assert np.array_equal(phase, exp)


def test_keyswitch_trivial_lwe_is_exact():
    P = _small()
    S = O.keygen(6, P.N)
    KA, KB = O.ksk_gen(P, S, 7)
    A, B = O.keyswitch(P, np.zeros(P.N, U64), P.delta * 1234, KA, KB)
    assert not A.any() and int(B[0]) == P.delta * 1234 and not B[1:].any()


@pytest.mark.parametrize("bl,lv", [(13, 3)])
def test_keyswitch_exact_decomposition_identity(bl, lv):
    """B' - A'S == (b - <a,S'>) X^0 exactly with an exact decomposition and E = 0."""
    P = _small()
    S = O.keygen(8, P.N)
    KA, KB = O.ksk_gen(P, S, 9, base_log=bl, levels=lv)
    for s in range(3):
        a = synth.uniform_u64(P.N, 100 + s, 39)
        b = int(synth.uniform_u64(1, 200 + s, 39)[0])
        A2, B2 = O.keyswitch(P, a, b, KA, KB, base_log=bl, levels=lv)
        AS = O.negacyclic_mul(A2, S.astype(np.int64), 39)
        phase = (B2 - AS) & U64(2 ** 39 - 1)
        exp = np.zeros(P.N, U64)
        exp[0] = O.lwe_phase(a, b, S, 39)
        assert np.array_equal(phase, exp)


def test_keyswitch_batched_equals_sequential():
    P = _small()
    S = O.keygen(10, P.N)
    KA, KB = O.ksk_gen(P, S, 11, eta=3)
    A_lwe = synth.uniform_u64((5, P.N), 12, 39)
    b_lwe = synth.uniform_u64(5, 13, 39)
    Ab, Bb = O.keyswitch_batched(P, A_lwe, b_lwe, KA, KB)
    for j in range(5):
        As, Bs = O.keyswitch(P, A_lwe[j], int(b_lwe[j]), KA, KB)
        assert np.array_equal(As, Ab[j]) and np.array_equal(Bs, Bb[j])


def _lwes(P, d_out, d_in, seed):
    S = O.keygen(seed, P.N)
    W = synth.uniform_int8((d_out, d_in), seed + 1)
    x = synth.uniform_int8(d_in, seed + 2)
    A, B = O.encrypt(P, S, x, O.block_seeds(seed, 1, P.L(d_in))[0])
    m, b = O.matmul_clear_literal(P, W, A, B)
    return S, W, x, m, b


def test_pack_exact_identity_places_every_output():
    """d_out = 2N + 3 -> 3 RLWE ciphertexts; coefficient j mod N of ciphertext j // N decrypts
    to x.w_j exactly (exact decomposition, E = 0); the unused slots of the last one are 0."""
    P = _small()
    N = P.N
    S, W, x, m, b = _lwes(P, 2 * N + 3, 20, 21)
    KA, KB = O.ksk_gen(P, S, 22, base_log=13, levels=3)
    # pack with the exact decomposition (Eq. 7 literally: keyswitch, rotate by j mod N, sum)
    G = 3
    PA = np.zeros((G, N), U64); PB = np.zeros((G, N), U64)
    with np.errstate(over="ignore"):
        for j in range(2 * N + 3):
            A2, B2 = O.keyswitch(P, m[j], int(b[j]), KA, KB, base_log=13, levels=3)
            g, r = divmod(j, N)
            PA[g] = (PA[g] + O.rotate(A2, r, 39)) & U64(2 ** 39 - 1)
            PB[g] = (PB[g] + O.rotate(B2, r, 39)) & U64(2 ** 39 - 1)
    wx = W.astype(np.int64) @ x.astype(np.int64)
    dec = np.concatenate([O.decrypt_packed(P, PA[g], PB[g], S, 39) for g in range(G)])
    assert np.array_equal(dec[:2 * N + 3], wx) and not dec[2 * N + 3:].any()


def test_pack_paper_decomposition_within_bound():
    """Paper (8, 3) decomposition with noisy KSK, then the 39 -> 26 switch: every output
    keeps its top gamma = 12 of beta = 27 bits."""
    P = Params(N=32, q_in=39, q_out=26, beta=27, gamma=12)
    S, W, x, m, b = _lwes(P, 32, 40, 31)
    KA, KB = O.ksk_gen(P, S, 32, eta=21)
    PA, PB = O.pack_lwes(P, m, b, KA, KB, out_bits=26)
    dec = O.decrypt_packed(P, PA[0], PB[0], S, 26)
    wx = W.astype(np.int64) @ x.astype(np.int64)
    assert np.all(np.abs(dec - wx) < 2 ** 15)
    PA2, PB2 = O.pack_lwes(P, m, b, KA, KB, out_bits=None, batched=False)
    PA3, PB3 = O.pack_lwes(P, m, b, KA, KB, out_bits=None, batched=True)
    assert np.array_equal(PA2, PA3) and np.array_equal(PB2, PB3)


def test_c_oracle_ksk_and_pack_match_python(coracle):
    P = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
    S = O.keygen(40, P.N)
    for eta in [0, 5]:
        KA, KB = O.ksk_gen(P, S, 41, eta=eta)
        cA, cB = coracle.ksk_gen(P, S, 41, eta=eta, nthreads=2)
        assert np.array_equal(KA, cA) and np.array_equal(KB, cB)
    A_lwe = synth.uniform_u64((2 * P.N + 5, P.N), 42, 39)
    b_lwe = synth.uniform_u64(2 * P.N + 5, 43, 39)
    PA, PB = O.pack_lwes(P, A_lwe, b_lwe, KA, KB)
    cA, cB = coracle.pack(P, A_lwe, b_lwe, KA, KB, nthreads=3)
    assert np.array_equal(PA, cA) and np.array_equal(PB, cB)
    import ctypes
    for v in synth.uniform_u64(200, 44, 39):
        for lv in (3, 4):
            d = (ctypes.c_int32 * lv)()
            coracle.lib.oracle_decompose(ctypes.c_uint64(int(v)), 39, 8, lv, d)
            assert list(d) == O.decompose(int(v), 39, 8, lv)


@pytest.mark.slow
def test_fig4_claim_on_the_oracle_pipeline(coracle):
    """Fig. 4 on the oracle's own full pipeline (noisy inputs, Eq. 6, Eq. 7/8 packing with
    the 4-level gadget, 39 -> 26 switch): bit-error rate < 1% at every position >= 12 over 512
    random int8 dot products, d_in = 768, N = 2048.  With the 3-level gadget of S:88 the same
    pipeline errs at bit 12 far more often (the reason for R18)."""
    P = O.Params(N=2048, q_in=39, q_out=26, beta=27, gamma=12, eta=21)
    S = O.keygen(3, P.N)
    W = synth.uniform_int8((512, 768), 5)
    x = synth.uniform_int8(768, 6)
    E = O.noise(P, 7, 1, 1)[0]
    A, B = O.encrypt(P, S, x, O.block_seeds(8, 1, 1)[0], E)
    m, b = coracle.matmul_clear_literal(P, W, A, B, nthreads=os.cpu_count())
    truth = W.astype(np.int64) @ x.astype(np.int64)
    rates = {}
    for lv in (4, 3):
        KA, KB = coracle.ksk_gen(P, S, 4, eta=0, levels=lv, nthreads=os.cpu_count())  # sigma_ksk -> 0 (R5)
        PA, PB = coracle.pack(P, m, b, KA, KB, levels=lv, nthreads=os.cpu_count())
        y = O.decrypt_packed(P, O.modswitch(PA[0], 39, 26), O.modswitch(PB[0], 39, 26), S, 26)[:512]
        d = (y ^ truth) & (2 ** 27 - 1)
        rates[lv] = [float(((d >> bb) & 1).mean()) for bb in range(27)]
    assert max(rates[4][12:]) < 0.01
    assert rates[3][12] > rates[4][12]
