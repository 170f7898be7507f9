"""Host-side checks (no GPU) for NEXT #4, the NTT-domain contraction: the primes the library
exports, the CRT range rule behind phe_ntt_max_blocks, and the kernel's index scheme (modelled in
tools/ntt_model.py: thread/phase mapping, XOR swizzle, twiddle indices, Shoup/Montgomery/CRT)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))

import ntt_model  # noqa: E402


def is_prime(n: int) -> bool:  # deterministic Miller-Rabin for n < 3.3e24
    if n < 2:
        return False
    small = [2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41]
    for q in small:
        if n % q == 0:
            return n == q
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2; s += 1
    for a in small:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@pytest.fixture(scope="module")
def lib():
    import paper_2505_07329_b200 as phe
    phe.load()
    return phe


def test_ntt_primes(lib):
    p0, p1 = lib.ntt_primes()
    assert (p0, p1) == tuple(ntt_model.P)
    for p in (p0, p1):
        assert is_prime(p) and 4 * p < 2 ** 32       # lazy [0, 2p) arithmetic in 32-bit words
        assert (p - 1) % (2 * 8192) == 0          # primitive 2N-th roots exist for N <= 8192
    assert p0 < p1
    assert p0 * p1 > 2 ** 59


@pytest.mark.parametrize("over", [{}, dict(N=512), dict(N=8192), dict(N=1024, q_in=32, q_out=28, beta=21)])
def test_ntt_max_blocks_is_the_crt_range(lib, over):
    p = lib.params(lib.PRESET_PAPER, **over)
    p0, p1 = lib.ntt_primes()
    L = lib.ntt_max_blocks(p)
    # centred masks |A - 2^(q-1)| <= 2^(q-1), |w| <= 128: |sum_i A'_i * w_i| <= L N 2^(q-1) 128;
    # the CRT offset Z = least multiple of 2^q >= worst + 2 p0 must keep worst + Z < p0 p1
    worst = lambda L: L * p.N * 2 ** (p.q_in - 1) * 128
    g = 2 ** p.q_in
    fits = lambda L: worst(L) + -(-(worst(L) + 2 * p0) // g) * g < p0 * p1
    assert L >= 1
    assert fits(L) and not fits(L + 1)
    assert worst(L) < p0 * p1 // 2                 # implies the centred range rule
    if not over:
        assert L == 6                              # Table 1: d_in up to 12288 (Llama-3.2-1B: 8192)


def test_centring_parity_identity():
    """P = P' + H (1 * w) with A' = A - H, and every coefficient of the negacyclic 1 * w has the
    parity of sum(w): so P = P' + H * (sum(w) mod 2) mod 2^q (R23), brute force."""
    import random
    rng = random.Random(9)
    q, N = 39, 32
    H = 2 ** (q - 1)
    for _ in range(30):
        L = rng.randint(1, 3)
        A = [[rng.randrange(2 ** q) for _ in range(N)] for _ in range(L)]
        W = [[rng.randrange(-128, 128) for _ in range(N)] for _ in range(L)]
        full, cent = [0] * N, [0] * N
        for i in range(L):
            for k, v in enumerate(ntt_model.negacyclic(A[i], W[i])):
                full[k] += v
            for k, v in enumerate(ntt_model.negacyclic([a - H for a in A[i]], W[i])):
                cent[k] += v
        par = sum(map(sum, W)) & 1
        assert all((cent[k] + H * par - full[k]) % 2 ** q == 0 for k in range(N))


def test_ntt_kernel_index_scheme():
    for logN in range(9, 14):
        ntt_model.bank_check(logN)
    # exact negacyclic products through the kernel's phase scheme and the two-prime CRT
    import random
    rng = random.Random(3)
    N, L = 512, 2
    A = [[rng.randrange(2 ** 39) for _ in range(N)] for _ in range(L)]
    W = [[rng.choice([-128, 127, rng.randrange(-128, 128)]) for _ in range(N)] for _ in range(L)]
    exact = [0] * N
    for i in range(L):
        for k, v in enumerate(ntt_model.negacyclic(A[i], W[i])):
            exact[k] += v
    res = []
    for p, g in zip(ntt_model.P, ntt_model.GEN):
        fwd, inv = ntt_model.tables(p, g, N)
        c = pow(N, -1, p) * 2 ** 32 % p
        acc = [0] * N
        for i in range(L):
            Ah = ntt_model.ntt_fwd([a % p for a in A[i]], p, fwd)
            Wh = ntt_model.ntt_fwd([w % p for w in W[i]], p, fwd)
            for k in range(N):
                acc[k] = (acc[k] + ntt_model.mont(Wh[k] * c % p, Ah[k], p)) % p
        res.append(ntt_model.intt_kernel_model(acc, p, inv, 9))
    M = ntt_model.P[0] * ntt_model.P[1]
    cinv = pow(ntt_model.P[0], -1, ntt_model.P[1])
    for k in range(N):
        h = ntt_model.shoup((res[1][k] - res[0][k]) % ntt_model.P[1], cinv, ntt_model.P[1])
        v = res[0][k] + ntt_model.P[0] * h
        assert (v - M if v >= M // 2 else v) == exact[k]


def test_ntt_keyswitch_index_scheme_and_split_crt():
    """tools/ntt_ks_model.py (the NTT-domain KeySwitch kernel's scheme, ntt_keyswitch.cu): every
    exchange and digit-tile access bank-conflict free for log2 N = 8..13, and the kernel-order
    forward NTTs + Montgomery pointwise products + KSK hi/lo split + two-prime CRT reproduce the
    exact negacyclic sum of Eq. 7/8 mod 2^39 on a small ring (brute-force schoolbook reference)."""
    import ntt_ks_model as m
    for logN in range(8, 14):
        assert m.bank_check(logN) is None, logN
    import io, contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        m.main()
    assert "logN=8: kernel-scheme" in buf.getvalue()
