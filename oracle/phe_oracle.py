"""CPU ORACLE for the encrypted-vector x clear-matrix hot path of arXiv 2505.07329.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import, call, link or execute anything under
oracle/.  The product path (paper_2505_07329_b200/) never does, and shares no code with
this file (it has its own ChaCha20, its own parameters, its own everything).

Plain, slow, obviously correct: every function follows PAPER.md (P:<line>) step by step,
in the paper's order and notation, using Python integers / numpy uint64 wrap-around
arithmetic (all moduli are powers of two <= 2^64, so uint64 wrap then masking is exact;
DESIGN.md reading R3).  Readings of ambiguous passages are DESIGN.md R1..R17.

Pins (tests/test_oracle_pins.py, -m "not gpu"): RFC 8439 ChaCha20 vectors and a
cross-check against the `cryptography` package; brute-force schoolbook vs numpy
polynomial convolution folded mod X^N+1; SPEC worked examples; Eq. 2 special cases;
W = I reduces Eq. 6 to textbook SampleExtract; A = 0 reduces it to a plain integer
matvec; the E = 0 decryption invariant b - <a,S> = Delta*(W x) mod Q exactly; modulus
switch worked examples and the 1/2-ULP bound; hand-derived golden vectors.  NEXT #1
(KeySwitch packing): SPEC decomposition examples + exhaustive recomposition; with an exact
decomposition (B*levels = q) and E = 0 the keyswitch / pack decrypt EXACTLY (algebraic
identity, independent of the implementation); batched (Eq. 8) == sequential (Eq. 4).
No function here is "parity unpinned".
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np

U64 = np.uint64
MASK64 = (1 << 64) - 1


# --------------------------------------------------------------------------------------
# a1: parameters  (Table 1; Delta = q/p)
# --------------------------------------------------------------------------------------
@dataclass(frozen=True)
class Params:
    N: int          # polynomial size
    q_in: int       # input modulus bits      -> Q  = 2^q_in   (R3)
    q_out: int      # output modulus bits     -> Q' = 2^q_out  (R3)
    beta: int       # bits reserved for computation -> t = 2^beta (R4)
    gamma: int      # MSBs unaffected by noise
    eta: int = 0    # noise: 0 = "SPEC" (E == 0, R5), else centered binomial CBD(eta)

    @property
    def Q(self) -> int:
        return 1 << self.q_in

    @property
    def t(self) -> int:
        return 1 << self.beta

    @property
    def delta(self) -> int:  # Delta = q/p
        return 1 << (self.q_in - self.beta)

    def L(self, d_in: int) -> int:  # L = ceil(d_in / N)
        return (d_in + self.N - 1) // self.N


# Table 1.  sigma = 2.845e-15 is recorded but not used numerically (R5).
PAPER = Params(N=2048, q_in=39, q_out=26, beta=27, gamma=12, eta=0)
PAPER_SIGMA = 2.845e-15
# Toy config (BASELINE configs[0]; not in the paper, R16).
TOY = Params(N=1024, q_in=32, q_out=28, beta=21, gamma=12, eta=0)


def mod(v: int, bits: int) -> int:
    return v & ((1 << bits) - 1)


# --------------------------------------------------------------------------------------
# ChaCha20 (RFC 8439 §2.3), the PRNG both parties "agree on" (reading R6)
# --------------------------------------------------------------------------------------
def _rotl32(v: int, c: int) -> int:
    return ((v << c) | (v >> (32 - c))) & 0xFFFFFFFF


def _quarter(s: list, a: int, b: int, c: int, d: int) -> None:
    s[a] = (s[a] + s[b]) & 0xFFFFFFFF; s[d] ^= s[a]; s[d] = _rotl32(s[d], 16)
    s[c] = (s[c] + s[d]) & 0xFFFFFFFF; s[b] ^= s[c]; s[b] = _rotl32(s[b], 12)
    s[a] = (s[a] + s[b]) & 0xFFFFFFFF; s[d] ^= s[a]; s[d] = _rotl32(s[d], 8)
    s[c] = (s[c] + s[d]) & 0xFFFFFFFF; s[b] ^= s[c]; s[b] = _rotl32(s[b], 7)


def chacha20_block(key: bytes, counter: int, nonce: bytes) -> bytes:
    """RFC 8439 §2.3: 64-byte keystream block."""
    assert len(key) == 32 and len(nonce) == 12
    state = [0x61707865, 0x3320646E, 0x79622D32, 0x6B206574]
    state += list(struct.unpack("<8I", key))
    state += [counter & 0xFFFFFFFF]
    state += list(struct.unpack("<3I", nonce))
    w = list(state)
    for _ in range(10):
        _quarter(w, 0, 4, 8, 12); _quarter(w, 1, 5, 9, 13)
        _quarter(w, 2, 6, 10, 14); _quarter(w, 3, 7, 11, 15)
        _quarter(w, 0, 5, 10, 15); _quarter(w, 1, 6, 11, 12)
        _quarter(w, 2, 7, 8, 13); _quarter(w, 3, 4, 9, 14)
    return struct.pack("<16I", *[(w[i] + state[i]) & 0xFFFFFFFF for i in range(16)])


def chacha20_keystream(key: bytes, nonce: bytes, nbytes: int, counter0: int = 0) -> bytes:
    out = bytearray()
    ctr = counter0
    while len(out) < nbytes:
        out += chacha20_block(key, ctr, nonce)
        ctr += 1
    return bytes(out[:nbytes])


def seed_key(seed: int) -> bytes:
    """R6: key = LE64(seed) || 0^24."""
    return struct.pack("<Q", seed & MASK64) + bytes(24)


NONCE_MASK = bytes(12)                       # R6: public mask stream
NONCE_SK = b"phe-sk".ljust(12, b"\0")        # R6: client-only key stream
NONCE_NOISE = b"phe-noise".ljust(12, b"\0")  # R6: client-only noise stream


def keystream_u64(seed: int, nonce: bytes, n_words: int, word0: int = 0) -> np.ndarray:
    """Consecutive little-endian u64 words of the keystream, starting at word `word0`."""
    blk0 = word0 // 8
    skip = word0 - 8 * blk0
    ks = chacha20_keystream(seed_key(seed), nonce, 8 * (n_words + skip), counter0=blk0)
    return np.frombuffer(ks, dtype="<u8")[skip:skip + n_words].astype(U64)


# --------------------------------------------------------------------------------------
# a3: seeded mask expansion A = PRNG(se)
# --------------------------------------------------------------------------------------
def expand_mask(seed: int, N: int, q_in: int) -> np.ndarray:
    """A[k] = LE64(keystream word k) mod 2^q_in, k in [0, N)  (R6)."""
    w = keystream_u64(seed, NONCE_MASK, N)
    return w & U64((1 << q_in) - 1) if q_in < 64 else w


def block_seeds(seed_base: int, T: int, L: int) -> np.ndarray:
    """One fresh public seed per block: seed_{tau,i} = seed_base + tau*L + i (R6)."""
    return (np.arange(T * L, dtype=np.uint64) + U64(seed_base & MASK64)).reshape(T, L)


# --------------------------------------------------------------------------------------
# keygen: S in R_2, LWE key S' = coefficients of S
# --------------------------------------------------------------------------------------
def keygen(master_seed: int, N: int) -> np.ndarray:
    """S[k] = bit (k mod 8) of keystream byte floor(k/8) under nonce "phe-sk" (R6)."""
    ks = chacha20_keystream(seed_key(master_seed), NONCE_SK, (N + 7) // 8)
    return np.array([(ks[k // 8] >> (k % 8)) & 1 for k in range(N)], dtype=np.uint8)


def noise(params: Params, noise_seed: int, T: int, L: int) -> np.ndarray:
    """E_{tau,i}[k] as int64 [T][L][N].  eta = 0: E == 0 (SPEC reading of sigma, R5).
    eta > 0: one keystream u64 word w per coefficient in global order (tau, i, k),
    e = popcount(w & (2^eta-1)) - popcount((w >> eta) & (2^eta-1))  (CBD, R5/R6)."""
    N = params.N
    if params.eta == 0 or T * L == 0:
        return np.zeros((T, L, N), dtype=np.int64)
    eta = params.eta
    w = keystream_u64(noise_seed, NONCE_NOISE, T * L * N)
    m = (1 << eta) - 1
    e = np.array([bin(int(x) & m).count("1") - bin((int(x) >> eta) & m).count("1") for x in w],
                 dtype=np.int64)
    return e.reshape(T, L, N)


# --------------------------------------------------------------------------------------
# ring arithmetic in R_q = Z_q[X]/(X^N + 1)  (negacyclic)
# --------------------------------------------------------------------------------------
def negacyclic_mul(a: np.ndarray, w: np.ndarray, q_bits: int) -> np.ndarray:
    """Schoolbook product in Z_{2^q}[X]/(X^N+1): X^N = -1.
    result[k] = sum_{m+n=k} a_m w_n - sum_{m+n=k+N} a_m w_n  (mod 2^q).
    a: uint64 residues; w: small signed integers (cleartext polynomial) or residues."""
    N = len(a)
    assert len(w) == N
    a = np.asarray(a, dtype=U64)
    wu = np.asarray(w).astype(np.int64).astype(U64)  # two's complement mod 2^64
    acc = np.zeros(N, dtype=U64)
    with np.errstate(over="ignore"):
        for m in range(N):  # term a_m X^m * w(X)
            am = a[m]
            if m == 0:
                acc += am * wu
            else:
                acc[m:] += am * wu[:N - m]          # m + n < N
                acc[:m] -= am * wu[N - m:]          # m + n >= N: X^N = -1
    return acc & U64((1 << q_bits) - 1) if q_bits < 64 else acc


def rotate(p: np.ndarray, k: int, q_bits: int) -> np.ndarray:
    """Multiply by X^k (negacyclic rotation)."""
    N = len(p)
    mono = np.zeros(N, dtype=np.int64)
    kk = k % (2 * N)
    if kk < N:
        mono[kk] = 1
    else:
        mono[kk - N] = -1
    return negacyclic_mul(p, mono, q_bits)


# --------------------------------------------------------------------------------------
# encrypt_pack (client op): x_hat_i[k] = x[iN+k] zero-padded;
# B = A*S + E + Delta*M mod q; one seed per block
# --------------------------------------------------------------------------------------
def split_blocks(x: np.ndarray, N: int) -> np.ndarray:
    """x (length d_in) -> L blocks of N, last block zero padded."""
    d_in = len(x)
    L = (d_in + N - 1) // N
    out = np.zeros((L, N), dtype=np.int64)
    out.reshape(-1)[:d_in] = np.asarray(x, dtype=np.int64)
    return out


def encrypt(params: Params, S: np.ndarray, x: np.ndarray, seeds: np.ndarray,
            E: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Seeded RLWE encryption of each block of one vector x.
    Returns (A [L][N] uint64 (server re-expands these from seeds), B [L][N] uint64)."""
    N, q = params.N, params.q_in
    xs = np.asarray(x, dtype=np.int64)
    assert np.all(np.abs(xs) < (1 << (params.beta - 1))), "message outside +-2^(beta-1) (S:150)"
    blocks = split_blocks(xs, N)
    L = blocks.shape[0]
    A = np.zeros((L, N), dtype=U64)
    B = np.zeros((L, N), dtype=U64)
    for i in range(L):
        A[i] = expand_mask(int(seeds[i]), N, q)
        AS = negacyclic_mul(A[i], S.astype(np.int64), q)
        e = np.zeros(N, np.int64) if E is None else E[i]
        with np.errstate(over="ignore"):
            Bi = AS + e.astype(U64) + U64(params.delta) * blocks[i].astype(U64)
        B[i] = Bi & U64(params.Q - 1)
    return A, B


# --------------------------------------------------------------------------------------
# a2: reversed weight encoding  w_hat_ij[k] = w_j[iN + N - 1 - k]
# --------------------------------------------------------------------------------------
def encode_weights(W: np.ndarray, N: int) -> np.ndarray:
    """w_hat [d_out][L][N] int64; w_j = row j of W (R1); zero where iN+N-1-k >= d_in."""
    d_out, d_in = W.shape
    L = (d_in + N - 1) // N
    out = np.zeros((d_out, L, N), dtype=np.int64)
    for i in range(L):
        for k in range(N):
            c = i * N + N - 1 - k
            if c < d_in:
                out[:, i, k] = W[:, c]
    return out


# --------------------------------------------------------------------------------------
# SampleExtract (Eq. 2)
# --------------------------------------------------------------------------------------
def sample_extract(A: np.ndarray, B: np.ndarray, h: int, q_bits: int) -> tuple[np.ndarray, int]:
    """a'_i = A_{h-i} (0<=i<=h), a'_i = -A_{N+h-i} (h<i<N), b' = B_h."""
    N = len(A)
    assert 0 <= h < N
    a = np.zeros(N, dtype=U64)
    for i in range(N):
        if i <= h:
            a[i] = A[h - i]
        else:
            a[i] = (-int(A[N + h - i])) % (1 << q_bits)
    return a, int(B[h])


# --------------------------------------------------------------------------------------
# a5..a7: Eq. 6, LWE(x.w_j) = sum_i SampleExtract(RLWE(x_hat_i) . w_hat_ij, N-1)
# --------------------------------------------------------------------------------------
def matmul_clear_literal(params: Params, W: np.ndarray, A: np.ndarray, B: np.ndarray,
                         rows: range | None = None) -> tuple[np.ndarray, np.ndarray]:
    """One token: A, B [L][N] uint64 (the expanded input ciphertext).
    Returns (mask [rows][N] uint64, body [rows] uint64) mod 2^q_in, literally:
      for each j: for each i: P = A_i*w_hat_ij, Qp = B_i*w_hat_ij (homomorphic multiplication
      by a cleartext polynomial); (a', b') = SampleExtract((P, Qp), N-1);
      accumulate (LWE addition).  Partial sums are added in LWE space."""
    N, q = params.N, params.q_in
    d_out, d_in = W.shape
    L = params.L(d_in)
    assert A.shape == (L, N) and B.shape == (L, N)
    what = encode_weights(W, N)
    rows = range(d_out) if rows is None else rows
    mask = np.zeros((len(rows), N), dtype=U64)
    body = np.zeros(len(rows), dtype=U64)
    for r, j in enumerate(rows):
        acc_a = np.zeros(N, dtype=U64)
        acc_b = 0
        for i in range(L):
            P = negacyclic_mul(A[i], what[j, i], q)
            Qp = negacyclic_mul(B[i], what[j, i], q)
            a_ext, b_ext = sample_extract(P, Qp, N - 1, q)
            with np.errstate(over="ignore"):
                acc_a = (acc_a + a_ext) & U64(params.Q - 1)
            acc_b = (acc_b + b_ext) % params.Q
        mask[r] = acc_a
        body[r] = acc_b
    return mask, body


def mask_entry_closed_form(params: Params, W: np.ndarray, A: np.ndarray, j: int, t: int) -> int:
    """Closed form of one mask coefficient, O(d_in) (derived from Eq. 2 + Eq. 6 + P:182;
    DESIGN.md §Oracle):  a_j[t] = sum_c W[j,c] * At[c mod N, t] over blocks i = c // N,
    At[m,t] = A_i[m-t] if m >= t else -A_i[m-t+N]."""
    N, Q = params.N, params.Q
    acc = 0
    for c in range(W.shape[1]):
        i, m = divmod(c, N)
        w = int(W[j, c])
        if w == 0:
            continue
        if m >= t:
            acc += w * int(A[i, m - t])
        else:
            acc -= w * int(A[i, m - t + N])
    return acc % Q


def body_closed_form(params: Params, W: np.ndarray, B: np.ndarray) -> np.ndarray:
    """b_j = sum_c W[j,c] * B_{c//N}[c mod N] mod Q: coefficient N-1 of B*w_hat.
    A plain integer matvec (exact in Python ints)."""
    d_out, d_in = W.shape
    flat = [int(v) for v in B.reshape(-1)[:d_in]]
    out = np.zeros(d_out, dtype=U64)
    for j in range(d_out):
        out[j] = sum(int(W[j, c]) * flat[c] for c in range(d_in)) % params.Q
    return out


def body_projection(params: Params, W: np.ndarray, B: np.ndarray, rp: np.ndarray) -> np.ndarray:
    """Freivalds projection of the bodies (a TEST PIN over all outputs, not a method step):
    sum_j rp[j] b_{tau,j} mod Q for B [T][L][N], with b_j = body_closed_form (the N-1 coefficient
    of B*w_hat):  sum_j rp[j] sum_c W[j,c] B[c] = sum_c (sum_j rp[j] W[j,c]) B[c].
    uint64 wrap-around arithmetic is exact mod Q = 2^q (R3).  Returns [T] uint64."""
    d_out, d_in = W.shape
    T = B.shape[0]
    with np.errstate(over="ignore"):
        Wu = W.astype(np.int64).astype(U64)                      # two's complement mod 2^64
        v = np.zeros(d_in, dtype=U64)
        for j in range(d_out):                                   # v = rp^T W
            v += U64(int(rp[j])) * Wu[j]
        flat = B.reshape(T, -1)[:, :d_in].astype(U64)
        out = np.zeros(T, dtype=U64)
        for tau in range(T):
            out[tau] = np.sum(flat[tau] * v, dtype=U64)
    return out & U64(params.Q - 1)


# --------------------------------------------------------------------------------------
# a8: ModulusSwitch q_from -> q_to; round half up (R8)
# --------------------------------------------------------------------------------------
def modswitch(v, q_from: int, q_to: int):
    """r = floor((v + 2^(f-t-1)) / 2^(f-t)) mod 2^t, for v a residue mod 2^f."""
    s = q_from - q_to
    if s == 0:
        return v
    if isinstance(v, np.ndarray):
        with np.errstate(over="ignore"):
            r = (v.astype(U64) + U64(1 << (s - 1))) >> U64(s)
        return r & U64((1 << q_to) - 1)
    return ((int(v) + (1 << (s - 1))) >> s) % (1 << q_to)


# --------------------------------------------------------------------------------------
# decrypt (client op): LWE under S'; decode + centre (R8, R9, R11)
# --------------------------------------------------------------------------------------
def lwe_phase(a: np.ndarray, b: int, S: np.ndarray, q_bits: int) -> int:
    """phi = (b - <a, S'>) mod 2^q."""
    s = sum(int(a[k]) for k in range(len(a)) if S[k])
    return (int(b) - s) % (1 << q_bits)


def decode(phi: int, q_bits: int, beta: int) -> int:
    """q >= beta: m = floor((phi + Delta_q/2) / Delta_q) mod t, Delta_q = 2^(q-beta);
    q < beta: m = phi * 2^(beta-q) mod t.  Centre into [-t/2, t/2)."""
    t = 1 << beta
    if q_bits >= beta:
        dq = 1 << (q_bits - beta)
        m = ((phi + dq // 2) // dq) % t
    else:
        m = (phi << (beta - q_bits)) % t
    return m - t if m >= t // 2 else m


def decrypt_lwe(a: np.ndarray, b: int, S: np.ndarray, q_bits: int, beta: int) -> int:
    return decode(lwe_phase(a, b, S, q_bits), q_bits, beta)


def decrypt_rlwe(A: np.ndarray, B: np.ndarray, S: np.ndarray, params: Params) -> np.ndarray:
    """round((B - A*S)/Delta), centred ("B - A*S ~ Delta M and scaling down")."""
    AS = negacyclic_mul(A, S.astype(np.int64), params.q_in)
    with np.errstate(over="ignore"):
        phi = (B.astype(U64) - AS) & U64(params.Q - 1)
    return np.array([decode(int(p), params.q_in, params.beta) for p in phi], dtype=np.int64)


# --------------------------------------------------------------------------------------
# convenience: the whole server step for T tokens (used by tests and the cpu baseline)
# --------------------------------------------------------------------------------------
def server_matmul(params: Params, W: np.ndarray, seeds: np.ndarray, bodies: np.ndarray,
                  out_bits: int | None = None, lib=None, nthreads: int = 1):
    """seeds [T][L] uint64, bodies [T][L][N] uint64 -> (mask [T][d_out][N], body [T][d_out]).
    Server-side: expand A from the seeds, Eq. 6 literally, then
    ModulusSwitch to q_out if out_bits == q_out.  `lib`: optional ctypes handle to
    the C oracle (oracle/phe_oracle.c) for the same literal path at full size."""
    T, L = seeds.shape
    d_out = W.shape[0]
    N = params.N
    mask = np.zeros((T, d_out, N), dtype=U64)
    body = np.zeros((T, d_out), dtype=U64)
    for tau in range(T):
        A = np.stack([expand_mask(int(seeds[tau, i]), N, params.q_in) for i in range(L)])
        if lib is not None:
            m, b = lib.matmul_clear_literal(params, W, A, bodies[tau], nthreads=nthreads)
        else:
            m, b = matmul_clear_literal(params, W, A, bodies[tau])
        mask[tau], body[tau] = m, b
    if out_bits is not None and out_bits != params.q_in:
        assert out_bits == params.q_out
        mask = modswitch(mask, params.q_in, params.q_out)
        body = modswitch(body, params.q_in, params.q_out)
    return mask, body


# ======================================================================================
# NEXT #1: KeySwitch packing of the LWE outputs into RLWE (Eq. 7; Eq. 8)
# Readings (R18-R21): Decomp = signed balanced base-2^B digits of the top B*levels
# bits after rounding (TFHE), B = 8, levels = 4 (Fig. 4's < 1% error at bit
# positions >= 12 fails with SPEC's 3 levels); KSK_{i,l} = RLWE_S(S'_i *
# 2^(q - (l+1)B)); K-index of the batched form = l*N + i (planar).
# ======================================================================================
KS_BASE_LOG = 8
KS_LEVELS = 4
NONCE_KSK = b"phe-ksk".ljust(12, b"\0")
NONCE_KSK_NOISE = b"phe-ksknoise"  # exactly 12 bytes


def decompose(v: int, q_bits: int, base_log: int = KS_BASE_LOG, levels: int = KS_LEVELS) -> list:
    """Decomp (Eq. 4): signed digits d_0..d_{levels-1} in [-2^(B-1), 2^(B-1)) with
    v ~= sum_l d_l 2^(q - (l+1)B) mod 2^q, |error| <= 2^(q - levels*B - 1).
    Round the discarded tail half up (R8), then peel digits from the least significant one,
    moving d >= 2^(B-1) to d - 2^B with a carry into the next digit; the last carry is mod q."""
    tail = q_bits - base_log * levels
    assert tail >= 0
    vr = (v + ((1 << (tail - 1)) if tail > 0 else 0)) >> tail
    vr %= 1 << (base_log * levels)
    digits = [0] * levels
    for l in range(levels - 1, -1, -1):
        d = vr & ((1 << base_log) - 1)
        vr >>= base_log
        if d >= 1 << (base_log - 1):
            d -= 1 << base_log
            vr += 1
        digits[l] = d
    return digits


def recompose(digits: list, q_bits: int, base_log: int = KS_BASE_LOG) -> int:
    return sum(d << (q_bits - (l + 1) * base_log) for l, d in enumerate(digits)) % (1 << q_bits)


def ksk_gen(params: Params, S: np.ndarray, ksk_seed: int, eta: int = 0,
            base_log: int = KS_BASE_LOG, levels: int = KS_LEVELS):
    """KSK_{i,l} = RLWE_S(S'_i * 2^(q - (l+1)B)) for i in [0,N), l in [0,levels).
    A_{i,l} = ChaCha20 words (nonce "phe-ksk") in order (l, i, k) mod 2^q; E_{i,l} = CBD(eta)
    (nonce "phe-ksk-noise", same order) or 0.  Returns KSK_A, KSK_B as [levels*N][N] uint64
    with row l*N + i (the batched matrices of Eq. 8)."""
    N, q = params.N, params.q_in
    rows = levels * N
    Aall = keystream_u64(ksk_seed, NONCE_KSK, rows * N).reshape(rows, N) & U64(params.Q - 1)
    if eta:
        w = keystream_u64(ksk_seed, NONCE_KSK_NOISE, rows * N)
        m = (1 << eta) - 1
        Eall = np.array([bin(int(x) & m).count("1") - bin((int(x) >> eta) & m).count("1") for x in w],
                        dtype=np.int64).reshape(rows, N)
    else:
        Eall = np.zeros((rows, N), np.int64)
    Ball = np.zeros((rows, N), U64)
    for l in range(levels):
        g = 1 << (q - (l + 1) * base_log)
        for i in range(N):
            r = l * N + i
            AS = negacyclic_mul(Aall[r], S.astype(np.int64), q)
            with np.errstate(over="ignore"):
                Br = AS + Eall[r].astype(U64)
                Br[0] += U64(int(S[i]) * g)
            Ball[r] = Br & U64(params.Q - 1)
    return Aall, Ball


def keyswitch(params: Params, a: np.ndarray, b: int, KA: np.ndarray, KB: np.ndarray,
              base_log: int = KS_BASE_LOG, levels: int = KS_LEVELS):
    """Eq. 4 literally: (A', B') = (0, b) - sum_i Decomp(a_i) . KSK_i."""
    N, q = params.N, params.q_in
    Ap = [0] * N
    Bp = [0] * N
    Bp[0] = int(b)
    for i in range(N):
        ds = decompose(int(a[i]), q, base_log, levels)
        for l, d in enumerate(ds):
            if d == 0:
                continue
            r = l * N + i
            for k in range(N):
                Ap[k] -= d * int(KA[r, k])
                Bp[k] -= d * int(KB[r, k])
    Q = params.Q
    return np.array([x % Q for x in Ap], U64), np.array([x % Q for x in Bp], U64)


def decomp_matrix(params: Params, A_lwe: np.ndarray, base_log: int = KS_BASE_LOG,
                  levels: int = KS_LEVELS) -> np.ndarray:
    """Decomp(A_LWE) of Eq. 8: [d_out][levels*N] int64, column l*N + i = digit l of a_j[i]."""
    d_out, N = A_lwe.shape
    D = np.zeros((d_out, levels * N), np.int64)
    for j in range(d_out):
        for i in range(N):
            ds = decompose(int(A_lwe[j, i]), params.q_in, base_log, levels)
            for l, d in enumerate(ds):
                D[j, l * N + i] = d
    return D


def keyswitch_batched(params: Params, A_lwe: np.ndarray, b_lwe: np.ndarray, KA: np.ndarray,
                      KB: np.ndarray, base_log: int = KS_BASE_LOG, levels: int = KS_LEVELS):
    """Eq. 8: A_RLWE = 0 - Decomp(A_LWE) KSK_A, B_RLWE = b - Decomp(A_LWE) KSK_B.
    Row j of the result is the RLWE ciphertext of keyswitch(LWE_j) with b_j in coefficient 0."""
    D = decomp_matrix(params, A_lwe, base_log, levels).astype(object)
    Q = params.Q
    PA = (D @ KA.astype(object)) % Q
    PB = (D @ KB.astype(object)) % Q
    A_r = np.array((-PA) % Q, dtype=U64)
    B_r = (-PB) % Q
    B_r[:, 0] = (B_r[:, 0] + b_lwe.astype(object)) % Q
    return A_r, np.array(B_r, dtype=U64)


def pack_lwes(params: Params, A_lwe: np.ndarray, b_lwe: np.ndarray, KA: np.ndarray, KB: np.ndarray,
              out_bits: int | None = None, batched: bool = True):
    """Eq. 7: for each group g of up to N consecutive outputs,
    RLWE_g = sum_j Rotate(KeySwitch(LWE_j), j - gN); then ModulusSwitch to q_out.
    Returns (A [G][N], B [G][N]) uint64."""
    d_out, N = A_lwe.shape
    q = params.q_in
    G = (d_out + N - 1) // N
    if batched:
        Ar, Br = keyswitch_batched(params, A_lwe, b_lwe, KA, KB)
    else:
        pairs = [keyswitch(params, A_lwe[j], int(b_lwe[j]), KA, KB) for j in range(d_out)]
        Ar = np.stack([p[0] for p in pairs])
        Br = np.stack([p[1] for p in pairs])
    PA = np.zeros((G, N), U64)
    PB = np.zeros((G, N), U64)
    with np.errstate(over="ignore"):
        for j in range(d_out):
            g, r = divmod(j, N)
            PA[g] = (PA[g] + rotate(Ar[j], r, q)) & U64(params.Q - 1)
            PB[g] = (PB[g] + rotate(Br[j], r, q)) & U64(params.Q - 1)
    if out_bits is not None and out_bits != q:
        PA, PB = modswitch(PA, q, out_bits), modswitch(PB, q, out_bits)
    return PA, PB


def decrypt_packed(params: Params, A: np.ndarray, B: np.ndarray, S: np.ndarray, q_bits: int) -> np.ndarray:
    """RLWE decryption of a packed output: phase = B - A*S, decode per coefficient."""
    AS = negacyclic_mul(A, S.astype(np.int64), q_bits)
    with np.errstate(over="ignore"):
        phi = (B.astype(U64) - AS) & U64((1 << q_bits) - 1)
    return np.array([decode(int(p), q_bits, params.beta) for p in phi], dtype=np.int64)


# ======================================================================================
# NEXT #2: wire format.  Little-endian contiguous bitstream, no
# per-coefficient padding: coefficient k occupies bits [k*b, (k+1)*b) (DESIGN R22).
# ======================================================================================
def bitpack(values, bits: int) -> bytes:
    acc = 0
    for k, v in enumerate(values):
        acc |= (int(v) & ((1 << bits) - 1)) << (k * bits)
    nbytes = (len(values) * bits + 7) // 8
    return acc.to_bytes(nbytes, "little")


def bitunpack(data: bytes, bits: int, count: int) -> np.ndarray:
    acc = int.from_bytes(data, "little")
    m = (1 << bits) - 1
    return np.array([(acc >> (k * bits)) & m for k in range(count)], dtype=U64)


def serialize_input(seed: int, body: np.ndarray, q_bits: int) -> bytes:
    """Seeded RLWE block as sent by the client: 8-byte seed + N coefficients at q_in bits
    (8 + 2048*39/8 = 9992 bytes)."""
    return struct.pack("<Q", seed & MASK64) + bitpack(body, q_bits)


def deserialize_input(data: bytes, N: int, q_bits: int):
    if len(data) != 8 + (N * q_bits + 7) // 8:
        raise ValueError("truncated or oversized input block")
    return struct.unpack("<Q", data[:8])[0], bitunpack(data[8:], q_bits, N)


def serialize_output(A: np.ndarray, B: np.ndarray, q_bits: int) -> bytes:
    """Packed RLWE output (A', B') at q_out bits (2 * 2048*26/8 = 13312 bytes)."""
    return bitpack(A, q_bits) + bitpack(B, q_bits)


def deserialize_output(data: bytes, N: int, q_bits: int):
    half = (N * q_bits + 7) // 8
    if len(data) != 2 * half:
        raise ValueError("truncated or oversized output ciphertext")
    return bitunpack(data[:half], q_bits, N), bitunpack(data[half:], q_bits, N)


def expansion_report(params: Params) -> dict:
    """Expansion factors computed from the serializers: input bytes per N int8
    plaintext bytes; output bytes per N*gamma/8 bytes of guaranteed plaintext."""
    N = params.N
    zi = serialize_input(0, np.zeros(N, U64), params.q_in)
    zo = serialize_output(np.zeros(N, U64), np.zeros(N, U64), params.q_out)
    return {"input_bytes": len(zi), "output_bytes": len(zo),
            "input_factor": len(zi) / N, "output_factor": len(zo) / (N * params.gamma / 8)}
