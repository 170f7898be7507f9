"""Integer model of the NTT-domain mask contraction kernels (NEXT #4), used to check the index
scheme of paper_2505_07329_b200/csrc/ntt_path.cu before running it: thread/phase mapping, smem
swizzle (bank-conflict freedom), twiddle indices, Montgomery/Shoup arithmetic and the CRT.
Development tool only (not the oracle, not the product).  Run: python tools/ntt_model.py
"""
import random

P = [998244353, 1004535809]
GEN = [3, 3]


def bitrev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2)


def tables(p, g, N):
    logN = N.bit_length() - 1
    psi = pow(g, (p - 1) // (2 * N), p)
    assert pow(psi, N, p) == p - 1
    fwd = [pow(psi, bitrev(k, logN), p) for k in range(N)]
    inv = [pow(psi, (2 * N - bitrev(k, logN)) % (2 * N), p) for k in range(N)]
    return fwd, inv


def shoup(x, w, p):
    wq = (w << 32) // p
    q = (x * wq) >> 32
    r = (x * w - q * p) & 0xFFFFFFFF
    assert r < 2 * p
    return r - p if r >= p else r


def mont(a, b, p):
    pinv = (-pow(p, -1, 2**32)) % 2**32
    t = a * b
    m = (t * pinv) & 0xFFFFFFFF
    u = (t + m * p) >> 32
    assert u < 2 * p
    return u - p if u >= p else u


def ntt_fwd(a, p, fwd):  # CT, natural in -> bit-reversed out (Longa-Naehrig Alg. 1)
    a = list(a); N = len(a); t = N; m = 1
    while m < N:
        t //= 2
        for i in range(m):
            j1 = 2 * i * t; S = fwd[m + i]
            for j in range(j1, j1 + t):
                U = a[j]; V = shoup(a[j + t], S, p)
                a[j] = (U + V) % p; a[j + t] = (U - V) % p
        m *= 2
    return a


def swz(j):
    h = ((j >> 5) & 15) | (((j >> 8) & 1) << 4)
    return j ^ h


# Per-exchange additive layouts (kernel v2+): exchange x writes with phase x's mapping and reads
# with phase x+1's; each layout is conflict-free for exactly those two patterns and is linear in
# the index bits, so every per-element address is a per-thread base plus an immediate.
def lay(x, j):
    if x == 0:
        return j + (j >> 4)
    if x == 1:
        return j + 16 * (j >> 8)
    return j


def lay_words(x, N):
    return max(lay(x, j) for j in range(N)) + 1


def phases(logN):
    out = []; s0 = 0
    while s0 < logN:
        b = min(4, logN - s0); out.append((s0, b)); s0 += b
    return out


def elem_index(tid, e, s0, b, logN):
    """element j owned by thread tid as its e-th value (e < 16) in phase (s0, b)."""
    el = e & ((1 << b) - 1)
    g = e >> b
    o = tid | (g << (logN - 4))
    return (o & ((1 << s0) - 1)) | (el << s0) | ((o >> s0) << (s0 + b))


def intt_kernel_model(ahat, p, inv, logN):
    """GS inverse NTT (bit-reversed in -> natural out) by the kernel's phase scheme."""
    N = 1 << logN; nthr = N // 16
    regs = [[ahat[elem_index(t, e, 0, 4, logN)] for e in range(16)] for t in range(nthr)]
    smem = [None] * N
    for pi, (s0, b) in enumerate(phases(logN)):
        if pi > 0:
            for t in range(nthr):  # load this phase's mapping
                regs[t] = [smem[lay(pi - 1, elem_index(t, e, s0, b, logN))] for e in range(16)]
        for t in range(nthr):
            r = regs[t]
            for s in range(s0, s0 + b):
                d = 1 << (s - s0)
                for e in range(16):
                    if e & d:
                        continue
                    j = elem_index(t, e, s0, b, logN)
                    jp = elem_index(t, e | d, s0, b, logN)
                    assert jp == j + (1 << s)
                    S = inv[(N >> (s + 1)) + (j >> (s + 1))]
                    U, V = r[e], r[e | d]
                    r[e] = (U + V) % p
                    r[e | d] = shoup((U - V) % p, S, p)
        if pi < len(phases(logN)) - 1:
            smem = [None] * lay_words(pi, N)
            for t in range(nthr):
                for e in range(16):
                    smem[lay(pi, elem_index(t, e, s0, b, logN))] = regs[t][e]
    s0, b = phases(logN)[-1]
    out = [None] * N
    for t in range(nthr):
        for e in range(16):
            out[elem_index(t, e, s0, b, logN)] = regs[t][e]
    return out


def bank_check(logN):
    """every warp-wide access of every exchange (write pattern of phase x, read pattern of phase
    x+1, layout x) hits 32 distinct banks; addresses are additive in (thread bits, element bits)"""
    nthr = (1 << logN) // 16
    ph = phases(logN)
    for x in range(len(ph) - 1):
        for (s0, b) in (ph[x], ph[x + 1]):
            for w in range(0, nthr, 32):
                for e in range(16):
                    banks = [lay(x, elem_index(t, e, s0, b, logN)) % 32 for t in range(w, min(w + 32, nthr))]
                    assert len(set(banks)) == len(banks), (logN, x, s0, b, e, banks)
            for t in range(nthr):
                for e in range(16):
                    assert lay(x, elem_index(t, e, s0, b, logN)) == lay(x, elem_index(t, 0, s0, b, logN)) + \
                        lay(x, elem_index(0, e, s0, b, logN))


def negacyclic(a, b):
    N = len(a); c = [0] * N
    for i in range(N):
        for k in range(N):
            if i + k < N: c[i + k] += a[i] * b[k]
            else: c[i + k - N] -= a[i] * b[k]
    return c


def main():
    for logN in (9, 10, 11, 12, 13):
        bank_check(logN)
        N = 1 << logN
        for t in range(N // 16):
            js = sorted(elem_index(t, e, s0, b, logN) for (s0, b) in phases(logN)[:1] for e in range(16))
            assert js == list(range(16 * t, 16 * t + 16))
    print("bank-conflict-free swizzle for logN 9..13; phase-1 rows contiguous")
    rng = random.Random(1)
    for logN in (9, 10, 11):
        N = 1 << logN
        q_in, L = 39, 3
        A = [[rng.randrange(2**q_in) for _ in range(N)] for _ in range(L)]
        W = [[rng.randrange(-128, 128) for _ in range(N)] for _ in range(L)]
        exact = [0] * N
        for i in range(L):
            for k, v in enumerate(negacyclic(A[i], W[i])): exact[k] += v
        res = []
        for p, g in zip(P, GEN):
            fwd, inv = tables(p, g, N)
            ninv_r = pow(N, -1, p) * 2**32 % p
            acc = [0] * N
            for i in range(L):
                Ah = ntt_fwd([x % p for x in A[i]], p, fwd)
                Wh = ntt_fwd([x % p for x in W[i]], p, fwd)
                Wm = [w * ninv_r % p for w in Wh]  # Montgomery form, N^-1 folded
                for k in range(N): acc[k] = (acc[k] + mont(Wm[k], Ah[k], p)) % p
            res.append(intt_kernel_model(acc, p, inv, logN))
        M = P[0] * P[1]
        c = pow(P[0], -1, P[1])
        for k in range(N):
            r0, r1 = res[0][k], res[1][k]
            h = shoup((r1 - r0) % P[1], c, P[1])
            v = r0 + P[0] * h
            if v >= M // 2: v -= M
            assert v == exact[k], (logN, k)
        print(f"logN={logN}: kernel-scheme NTT product == exact negacyclic sum (L={L})")


if __name__ == "__main__":
    main()
