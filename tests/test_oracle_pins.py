"""Pins for the CPU oracle (-m "not gpu").

Each test ties oracle/ to something other than itself: RFC 8439 vectors and a third-party
ChaCha20, brute-force convolution, textbook special cases (W = I is SampleExtract, A = 0 is
an integer matvec), the E = 0 decryption invariant of Eq. 6, SPEC/paper worked values and
hand-derived golden vectors (tests/golden/, each with its citation).
"""
import os

import numpy as np
import pytest

from oracle import phe_oracle as O
from oracle.phe_oracle import PAPER, TOY, Params
import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")
U64 = np.uint64


def _golden(name):
    rows = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append(line.split())
    return rows


# ---------------------------------------------------------------- parameters (Table 1)
def test_table1_parameters():
    g = {r[0]: r for r in _golden("spec_examples.txt")}
    beta, gamma, N, q_in, q_out = map(int, g["table1"][2:7])
    assert (PAPER.beta, PAPER.gamma, PAPER.N, PAPER.q_in, PAPER.q_out) == (beta, gamma, N, q_in, q_out)
    assert PAPER.delta == 2 ** 12 and PAPER.t == 2 ** 27  # Delta = q/p, R4
    assert float(g["sigma"][2]) == O.PAPER_SIGMA


# ---------------------------------------------------------------- ChaCha20 (R6)
def test_chacha20_rfc8439_zero_key_vector():
    # RFC 8439 Appendix A.1 test vector #1: all-zero key and nonce, counter 0.
    ks = O.chacha20_block(bytes(32), 0, bytes(12))
    assert ks[:32].hex() == "76b8e0ada0f13d90405d6ae55386bd28bdd219b8a08ded1aa836efcc8b770dc7"


def test_chacha20_rfc8439_232_block():
    # RFC 8439 §2.3.2: key 00..1f, nonce 000000090000004a00000000, counter 1.
    ks = O.chacha20_block(bytes(range(32)), 1, bytes.fromhex("000000090000004a00000000"))
    assert ks[:16].hex() == "10f1e7e4d13b5915500fdd1fa32071c4"


def test_chacha20_rfc8439_242_encryption():
    # RFC 8439 §2.4.2: the sunscreen plaintext, counter 1, nonce 000000000000004a00000000.
    pt = (b"Ladies and Gentlemen of the class of '99: If I could offer you only one tip "
          b"for the future, sunscreen would be it.")
    ks = O.chacha20_keystream(bytes(range(32)), bytes.fromhex("000000000000004a00000000"),
                              len(pt), counter0=1)
    ct = bytes(a ^ b for a, b in zip(pt, ks))
    assert ct[:16].hex() == "6e2e359a2568f98041ba0728dd0d6981"


def test_chacha20_matches_cryptography_package():
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    for seed in [0, 1, 0x250507329, 2 ** 64 - 1]:
        key = O.seed_key(seed)
        for nonce in [O.NONCE_MASK, O.NONCE_SK, O.NONCE_NOISE]:
            # cryptography's ChaCha20 nonce = counter(LE32) || nonce(12)
            enc = Cipher(algorithms.ChaCha20(key, b"\0\0\0\0" + nonce), mode=None).encryptor()
            ref = enc.update(bytes(64 * 5))
            assert O.chacha20_keystream(key, nonce, 64 * 5) == ref


def test_expand_mask_is_masked_le64_words():
    from cryptography.hazmat.primitives.ciphers import Cipher, algorithms
    seed = 0x250507329
    enc = Cipher(algorithms.ChaCha20(O.seed_key(seed), bytes(16)), mode=None).encryptor()
    raw = np.frombuffer(enc.update(bytes(8 * 64)), dtype="<u8")
    A = O.expand_mask(seed, 64, 39)
    assert np.array_equal(A, raw & U64(2 ** 39 - 1))
    assert A.max() < 2 ** 39


def test_c_oracle_chacha_and_expand(coracle):
    for seed in [1, 77, 2 ** 63 + 5]:
        key = O.seed_key(seed)
        assert coracle.chacha20_block(key, 3, O.NONCE_MASK) == O.chacha20_block(key, 3, O.NONCE_MASK)
        for q in [32, 39, 64]:
            assert np.array_equal(coracle.expand_mask(seed, 128, q), O.expand_mask(seed, 128, q))


def test_keygen_binary_deterministic():
    S1 = O.keygen(42, 2048)
    assert set(np.unique(S1)) <= {0, 1}
    assert np.array_equal(S1, O.keygen(42, 2048))
    assert (S1 != O.keygen(43, 2048)).sum() > 2048 // 4
    assert 800 < S1.sum() < 1250


def test_noise_cbd_range():
    P = Params(N=64, q_in=39, q_out=26, beta=27, gamma=12, eta=21)
    E = O.noise(P, 9, 2, 3)
    assert E.shape == (2, 3, 64) and np.abs(E).max() <= 21 and E.std() > 1.0
    assert not O.noise(PAPER, 9, 1, 1).any()  # eta = 0: E == 0 (R5)


# ---------------------------------------------------------------- ring arithmetic
def test_negacyclic_spec_example():
    row = [r for r in _golden("spec_examples.txt") if r[0] == "negacyclic"][0]
    N, q = int(row[2]), int(row[3])
    a = np.array([int(v) for v in row[4].split(",")], dtype=U64)
    w = np.array([int(v) for v in row[5].split(",")])
    exp = [int(v) for v in row[6].split(",")]
    assert [int(v) for v in O.negacyclic_mul(a, w, q)] == exp


@pytest.mark.parametrize("N", [4, 8, 16, 64])
def test_negacyclic_vs_folded_convolution(N):
    """Brute force: numpy full convolution (object ints) folded with X^N = -1."""
    for s in range(4):
        a = synth.uniform_u64(N, 100 + s, 39)
        w = synth.uniform_int8(N, 200 + s).astype(np.int64)
        full = np.convolve(a.astype(object), w.astype(object))
        fold = [(int(full[k]) - (int(full[k + N]) if k + N < len(full) else 0)) % 2 ** 39
                for k in range(N)]
        assert [int(v) for v in O.negacyclic_mul(a, w, 39)] == fold


def test_rotate_is_negacyclic_shift():
    N = 16
    a = synth.uniform_u64(N, 5, 39)
    r = O.rotate(a, 3, 39)
    for k in range(N):
        src = k - 3
        exp = int(a[src]) if src >= 0 else (-int(a[src + N])) % 2 ** 39
        assert int(r[k]) == exp
    # X^N = -1
    assert [int(v) for v in O.rotate(a, N, 39)] == [(-int(v)) % 2 ** 39 for v in a]


def test_negacyclic_linearity():
    N = 32
    a, b = synth.uniform_u64(N, 1, 39), synth.uniform_u64(N, 2, 39)
    w = synth.uniform_int8(N, 3)
    lhs = O.negacyclic_mul((a + b) & U64(2 ** 39 - 1), w, 39)
    rhs = (O.negacyclic_mul(a, w, 39) + O.negacyclic_mul(b, w, 39)) & U64(2 ** 39 - 1)
    assert np.array_equal(lhs, rhs)


# ---------------------------------------------------------------- encryption
@pytest.mark.parametrize("params", [TOY, Params(N=64, q_in=39, q_out=26, beta=27, gamma=12, eta=21)])
def test_encrypt_decrypt_roundtrip(params):
    N = params.N
    S = O.keygen(7, N)
    x = synth.uniform_int8(2 * N - 5, 11)
    seeds = O.block_seeds(99, 1, params.L(len(x)))[0]
    E = O.noise(params, 5, 1, len(seeds))[0]
    A, B = O.encrypt(params, S, x, seeds, E)
    assert np.array_equal(A[0], O.expand_mask(int(seeds[0]), N, params.q_in))
    dec = np.concatenate([O.decrypt_rlwe(A[i], B[i], S, params) for i in range(len(seeds))])
    assert np.array_equal(dec[:len(x)], x.astype(np.int64))
    assert not dec[len(x):].any()


# ---------------------------------------------------------------- SampleExtract (Eq. 2)
def test_sample_extract_h0_spec_example():
    N = 8
    A = synth.uniform_u64(N, 3, 39)
    B = synth.uniform_u64(N, 4, 39)
    a, b = O.sample_extract(A, B, 0, 39)
    assert int(a[0]) == int(A[0]) and b == int(B[0])
    for i in range(1, N):
        assert int(a[i]) == (-int(A[N - i])) % 2 ** 39


def test_sample_extract_decrypts_coefficient():
    P = Params(N=32, q_in=39, q_out=26, beta=27, gamma=12)
    S = O.keygen(3, P.N)
    m = synth.uniform_int8(P.N, 8)
    A, B = O.encrypt(P, S, m, O.block_seeds(5, 1, 1)[0])
    for h in range(P.N):
        a, b = O.sample_extract(A[0], B[0], h, P.q_in)
        assert O.decrypt_lwe(a, b, S, P.q_in, P.beta) == int(m[h])


def test_encode_weights_reverse_spec_example():
    N = 8
    W = np.zeros((1, N), np.int8)
    W[0, 0] = 1  # w_j = e_0 -> w_hat has 1 at N-1
    wh = O.encode_weights(W, N)
    assert wh[0, 0, N - 1] == 1 and wh.sum() == 1


# ---------------------------------------------------------------- Eq. 6
def test_g1_hand_derived_golden():
    P = Params(N=4, q_in=39, q_out=26, beta=27, gamma=12)
    W = np.array([[1, 2, 3, 4], [-1, 0, 1, -2]], np.int8)
    A = np.array([[5, 6, 7, 8]], U64)
    B = np.array([[9, 10, 11, 12]], U64)
    mask, body = O.matmul_clear_literal(P, W, A, B)
    for row in _golden("g1_hand.txt"):
        j = int(row[0])
        vals = [int(v) % 2 ** 39 for v in row[1:]]
        assert [int(v) for v in mask[j]] == vals[:4]
        assert int(body[j]) == vals[4]


def test_identity_weight_is_sample_extract():
    """W = I (d = N): Eq. 6 gives LWE_j = SampleExtract(RLWE(x), j) for every j (textbook)."""
    P = Params(N=32, q_in=39, q_out=26, beta=27, gamma=12)
    W = np.eye(P.N, dtype=np.int8)
    A = synth.uniform_u64((1, P.N), 1, 39)
    B = synth.uniform_u64((1, P.N), 2, 39)
    mask, body = O.matmul_clear_literal(P, W, A, B)
    for j in range(P.N):
        a, b = O.sample_extract(A[0], B[0], j, 39)
        assert np.array_equal(mask[j], a) and int(body[j]) == b


def test_trivial_ciphertext_is_integer_matvec():
    """A = 0: masks vanish and the body is W . B mod Q (plain integer matvec)."""
    P = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
    W = synth.uniform_int8((5, 40), 3)
    L = P.L(40)
    A = np.zeros((L, P.N), U64)
    B = synth.uniform_u64((L, P.N), 4, 39)
    mask, body = O.matmul_clear_literal(P, W, A, B)
    assert not mask.any()
    ref = (W.astype(object) @ B.reshape(-1)[:40].astype(object)) % 2 ** 39
    assert [int(v) for v in body] == [int(v) for v in ref]


@pytest.mark.parametrize("N,d_out,d_in", [(8, 3, 8), (8, 4, 21), (16, 5, 48), (32, 3, 70)])
def test_decryption_invariant_E0(N, d_out, d_in):
    """With E = 0: b_j - <a_j, S> = Delta * (W x)_j mod Q exactly (P:58 + Eq. 6)."""
    P = Params(N=N, q_in=39, q_out=26, beta=27, gamma=12)
    S = O.keygen(1234 + N, N)
    W = synth.uniform_int8((d_out, d_in), N + d_in)
    x = synth.uniform_int8(d_in, 2 * N + d_in)
    seeds = O.block_seeds(777, 1, P.L(d_in))[0]
    A, B = O.encrypt(P, S, x, seeds)
    mask, body = O.matmul_clear_literal(P, W, A, B)
    wx = W.astype(np.int64) @ x.astype(np.int64)
    for j in range(d_out):
        assert O.lwe_phase(mask[j], int(body[j]), S, 39) == (P.delta * int(wx[j])) % P.Q


def test_closed_form_equals_literal():
    P = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
    d_in = 37
    W = synth.uniform_int8((4, d_in), 8)
    A = synth.uniform_u64((P.L(d_in), P.N), 9, 39)
    B = synth.uniform_u64((P.L(d_in), P.N), 10, 39)
    mask, body = O.matmul_clear_literal(P, W, A, B)
    for j in range(4):
        for t in range(P.N):
            assert O.mask_entry_closed_form(P, W, A, j, t) == int(mask[j, t])
    assert np.array_equal(O.body_closed_form(P, W, B), body)


def test_onehot_column_readout():
    """x = e_c => output j decrypts to W[j, c]."""
    P = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
    S = O.keygen(4, P.N)
    W = synth.uniform_int8((6, 20), 21)
    for c in [0, 7, 15, 16, 19]:
        x = np.zeros(20, np.int8)
        x[c] = 1
        A, B = O.encrypt(P, S, x, O.block_seeds(c, 1, 2)[0])
        mask, body = O.matmul_clear_literal(P, W, A, B)
        for j in range(6):
            assert O.decrypt_lwe(mask[j], int(body[j]), S, 39, 27) == int(W[j, c])


def test_linearity_over_weights_and_ciphertexts():
    P = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12)
    W1, W2 = synth.uniform_int8((3, 16), 1, -60, 60), synth.uniform_int8((3, 16), 2, -60, 60)
    A = synth.uniform_u64((1, 16), 3, 39)
    B = synth.uniform_u64((1, 16), 4, 39)
    m1, b1 = O.matmul_clear_literal(P, W1, A, B)
    m2, b2 = O.matmul_clear_literal(P, W2, A, B)
    m3, b3 = O.matmul_clear_literal(P, (W1.astype(np.int16) + W2).astype(np.int8), A, B)
    q = U64(2 ** 39 - 1)
    assert np.array_equal((m1 + m2) & q, m3) and np.array_equal((b1 + b2) & q, b3)
    A2 = synth.uniform_u64((1, 16), 5, 39)
    B2 = synth.uniform_u64((1, 16), 6, 39)
    ma, ba = O.matmul_clear_literal(P, W1, A2, B2)
    ms, bs = O.matmul_clear_literal(P, W1, (A + A2) & q, (B + B2) & q)
    assert np.array_equal((m1 + ma) & q, ms) and np.array_equal((b1 + ba) & q, bs)


# ---------------------------------------------------------------- ModulusSwitch
def test_modswitch_spec_examples():
    for r in _golden("spec_examples.txt"):
        if r[0] == "modswitch":
            v, f, t, exp = map(int, r[2:6])
            assert O.modswitch(v, f, t) == exp


def test_modswitch_half_ulp_bound():
    v = synth.uniform_u64(20000, 17, 39)
    r = O.modswitch(v, 39, 26)
    back = (r.astype(object) * 2 ** 13 - v.astype(object))
    cen = [((int(d) + 2 ** 38) % 2 ** 39) - 2 ** 38 for d in back]
    assert max(abs(c) for c in cen) <= 2 ** 12


def test_post_switch_decrypt_bound():
    """|dec - W x| <= 1 + hw(S) after the 39->26 switch at paper params (P:198 contract)."""
    P = Params(N=64, q_in=39, q_out=26, beta=27, gamma=12)
    S = O.keygen(11, P.N)
    W = synth.uniform_int8((8, 100), 12)
    x = synth.uniform_int8(100, 13)
    A, B = O.encrypt(P, S, x, O.block_seeds(3, 1, 2)[0])
    mask, body = O.matmul_clear_literal(P, W, A, B)
    ms, bs = O.modswitch(mask, 39, 26), O.modswitch(body, 39, 26)
    wx = W.astype(np.int64) @ x.astype(np.int64)
    for j in range(8):
        d = O.decrypt_lwe(ms[j], int(bs[j]), S, 26, 27)
        assert abs(d - int(wx[j])) <= 1 + int(S.sum())
        assert (d - int(wx[j])) >> 15 in (0, -1)  # top gamma=12 of beta=27 bits kept


# ---------------------------------------------------------------- C oracle == Python oracle
@pytest.mark.parametrize("N,d_out,d_in", [(16, 5, 16), (16, 4, 37), (64, 3, 200), (128, 2, 128)])
def test_c_oracle_literal_matches_python(coracle, N, d_out, d_in):
    P = Params(N=N, q_in=39, q_out=26, beta=27, gamma=12)
    W = synth.uniform_int8((d_out, d_in), N * d_in)
    L = P.L(d_in)
    A = synth.uniform_u64((L, N), 1 + N, 39)
    B = synth.uniform_u64((L, N), 2 + N, 39)
    m1, b1 = O.matmul_clear_literal(P, W, A, B)
    m2, b2 = coracle.matmul_clear_literal(P, W, A, B, nthreads=2)
    assert np.array_equal(m1, m2) and np.array_equal(b1, b2)
    js = np.array([0, d_out - 1, d_out // 2]); ts = np.array([0, N - 1, N // 3])
    ent = coracle.mask_entries(P, W, A, js, ts)
    assert [int(e) for e in ent] == [int(m1[j, t]) for j, t in zip(js, ts)]


def test_c_oracle_decryption_invariant_paper_params(coracle):
    """The C literal path at the real ring size N=2048 against the E=0 invariant."""
    P = PAPER
    S = O.keygen(2025, P.N)
    d_in, d_out = 3000, 6  # L = 2, ragged last block
    W = synth.weights_int8(d_out, d_in)
    x = synth.activations_int8(1, d_in)[0]
    A, B = O.encrypt(P, S, x, O.block_seeds(31, 1, P.L(d_in))[0])
    mask, body = coracle.matmul_clear_literal(P, W, A, B, nthreads=4)
    wx = W.astype(np.int64) @ x.astype(np.int64)
    sidx = S.astype(bool)
    for j in range(d_out):
        phase = (int(body[j]) - int(mask[j][sidx].astype(object).sum())) % P.Q
        assert phase == (P.delta * int(wx[j])) % P.Q


def test_c_oracle_modswitch(coracle):
    v = synth.uniform_u64(1000, 3, 39)
    assert np.array_equal(coracle.modswitch(v, 39, 26), O.modswitch(v, 39, 26))


@pytest.mark.parametrize("N,d_out,d_in,q", [(16, 5, 37, 39), (8, 3, 8, 16), (256, 4, 600, 39)])
def test_mask_projection_is_the_literal_masks_projected(coracle, N, d_out, d_in, q):
    """oracle_mask_projection (the Freivalds check the GPU suites run over every output) equals
    sum_t a_j[t] r[t] mod 2^q computed with Python integers from the literal Eq. 6 masks
    (Python oracle for tiny N; the C literal path for N = 256), ragged last block included."""
    prm = Params(N=N, q_in=q, q_out=min(q, 26) - 4, beta=min(q, 26) - 4, gamma=4, eta=0)
    rng = np.random.default_rng(N + d_in)
    W = rng.integers(-127, 128, size=(d_out, d_in)).astype(np.int8)
    T, L = 3, prm.L(d_in)
    A = rng.integers(0, 2 ** 62, size=(T, L, N), dtype=np.uint64) & np.uint64(prm.Q - 1)
    r = rng.integers(0, 2 ** 62, size=(2, N), dtype=np.uint64) & np.uint64(prm.Q - 1)
    got = coracle.mask_projection(prm, W, A, r)
    for tau in range(T):
        if N <= 16:
            mask, _ = O.matmul_clear_literal(prm, W, A[tau], np.zeros((L, N), np.uint64))
        else:
            mask, _ = coracle.matmul_clear_literal(prm, W, A[tau], np.zeros((L, N), np.uint64))
        for j in range(d_out):
            for e in range(2):
                want = sum(int(mask[j, t]) * int(r[e, t]) for t in range(N)) % prm.Q
                assert int(got[tau, j, e]) == want
    # a single flipped top bit in one mask word changes the projection for odd r[t]
    r1 = np.ones((1, N), np.uint64)
    base = coracle.mask_projection(prm, W, A, r1)
    mask, _ = coracle.matmul_clear_literal(prm, W, A[0], np.zeros((L, N), np.uint64))
    assert int(base[0, 0, 0]) == sum(int(v) for v in mask[0]) % prm.Q


def test_body_projection_is_the_closed_form_bodies_projected():
    """body_projection == sum_j rp[j] * body_closed_form(...)[j] mod Q in Python integers."""
    prm = Params(N=16, q_in=39, q_out=26, beta=27, gamma=12, eta=0)
    rng = np.random.default_rng(7)
    W = rng.integers(-127, 128, size=(6, 37)).astype(np.int8)
    B = rng.integers(0, 2 ** 39, size=(4, 3, 16), dtype=np.uint64)
    rp = rng.integers(0, 2 ** 39, size=6, dtype=np.uint64)
    got = O.body_projection(prm, W, B, rp)
    for tau in range(4):
        b = O.body_closed_form(prm, W, B[tau])
        assert int(got[tau]) == sum(int(rp[j]) * int(b[j]) for j in range(6)) % prm.Q
