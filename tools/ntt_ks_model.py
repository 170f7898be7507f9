"""Integer model of the NTT-domain KeySwitch packing kernel (stage 2 of the packed primitive,
ntt_keyswitch.cu), used to check its index scheme on the host before running it: the forward
Cooley-Tukey NTT by reversed 3-bit phases in registers (V = 8 values per thread), 32-bit-word
exchange layouts (bank-conflict freedom), the swizzled digit tile, lazy Harvey/Montgomery
arithmetic bounds, the KSK hi/lo split and the two-prime CRT with an offset Z.  Development tool
only (not the oracle, not the product).  Run: python tools/ntt_ks_model.py
"""
import random

P = [268369921, 268271617]   # the two largest primes < 2^28 with 2^14 | p - 1 (16p < 2^32)
GEN = [23, 5]
VB = 3
V = 1 << VB


def bitrev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def tables(p, g, N):
    logN = N.bit_length() - 1
    psi = pow(g, (p - 1) // (2 * N), p)
    assert pow(psi, N, p) == p - 1
    fwd = [pow(psi, bitrev(k, logN), p) for k in range(N)]
    inv = [pow(psi, (2 * N - bitrev(k, logN)) % (2 * N), p) for k in range(N)]
    return fwd, inv


def shoup_lazy(x, w, p):
    assert 0 <= x < 2**32
    wq = (w << 32) // p
    q = (x * wq) >> 32
    r = (x * w - q * p) & 0xFFFFFFFF
    assert r < 2 * p and r % p == x * w % p
    return r


def mont_lazy(a, b, p):
    pinv = (-pow(p, -1, 2**32)) % 2**32
    t = a * b
    m = (t * pinv) & 0xFFFFFFFF
    assert t + m * p < 2**64
    u = (t + m * p) >> 32
    assert u < 2 * p
    return u


def phases(logN):  # inverse-order phase list (3-bit phases); the forward transform runs it reversed
    out = []; s0 = 0
    while s0 < logN:
        b = min(VB, logN - s0); out.append((s0, b)); s0 += b
    return out


def elem_index(tid, e, s0, b, logN):
    el = e & ((1 << b) - 1)
    g = e >> b
    o = tid | (g << (logN - VB))
    return (o & ((1 << s0) - 1)) | (el << s0) | ((o >> s0) << (s0 + b))


def lay(s0_read, j):
    """word address of element j in the exchange buffer read by the phase starting at stage
    s0_read (found by search: conflict-free for both access patterns of that exchange, 32-bit
    words, logN 8..13; additive in disjoint index bits)"""
    return j + (j >> 3) if s0_read == 0 else j + 4 * (j >> 5) if s0_read == 3 else j


def tile_bytes(logN):
    return 8 if logN >= 13 else 16


def tile_addr(r, c, logN):
    tb = tile_bytes(logN)
    wpr = tb // 4
    sws = 3 if wpr == 4 else 4
    w, byte = c >> 2, c & 3
    return r * tb + 4 * (w ^ ((r >> sws) & (wpr - 1))) + byte


def bank_check(logN):
    nthr = (1 << logN) // V
    rev = phases(logN)[::-1]
    for x in range(len(rev) - 1):
        for (s0, b) in (rev[x], rev[x + 1]):
            for w0 in range(0, nthr, 32):
                for e in range(V):
                    banks = [lay(rev[x + 1][0], elem_index(t, e, s0, b, logN)) % 32 for t in range(w0, min(w0 + 32, nthr))]
                    if len(set(banks)) != len(banks):
                        return f"exchange {x} phase {(s0, b)} e={e}: {len(banks) - len(set(banks))} conflicts"
    s0, b = rev[0]
    for w0 in range(0, nthr, 32):
        for e in range(V):
            for c in range(tile_bytes(logN)):
                banks = [tile_addr(elem_index(t, e, s0, b, logN), c, logN) // 4 % 32
                         for t in range(w0, min(w0 + 32, nthr))]
                if len(set(banks)) != len(banks):
                    return f"tile e={e} c={c} conflicts"
    return None


def fwd_kernel_model(a, p, fwd, logN):
    """CT forward NTT (natural in -> bit-reversed out), values lazily in [0, 4p)."""
    N = 1 << logN; nthr = N // V
    rev = phases(logN)[::-1]
    s0, b = rev[0]
    regs = [[a[elem_index(t, e, s0, b, logN)] for e in range(V)] for t in range(nthr)]
    for pi, (s0, b) in enumerate(rev):
        if pi > 0:
            regs = [[smem[lay(s0, elem_index(t, e, s0, b, logN))] for e in range(V)] for t in range(nthr)]
        for t in range(nthr):
            r = regs[t]
            for s in range(s0 + b - 1, s0 - 1, -1):
                d = 1 << (s - s0)
                for e in range(V):
                    if e & d:
                        continue
                    j = elem_index(t, e, s0, b, logN)
                    assert elem_index(t, e | d, s0, b, logN) == j + (1 << s)
                    w = fwd[(N >> (s + 1)) + (j >> (s + 1))]
                    U, Y = r[e], r[e | d]
                    assert U < 16 * p and Y < 16 * p
                    if logN - 1 - s == 7:   # the kernel's only reduction: U < 16p -> < 4p
                        U = min(U, (U - 8 * p) % 2**32)
                        U = min(U, (U - 4 * p) % 2**32)
                    Vp = shoup_lazy(Y, w, p)
                    r[e] = U + Vp
                    r[e | d] = U - Vp + 2 * p
                    assert r[e] < 16 * p and r[e | d] < 16 * p
        if pi < len(rev) - 1:
            smem = {}
            for t in range(nthr):
                for e in range(V):
                    smem[lay(rev[pi + 1][0], elem_index(t, e, s0, b, logN))] = regs[t][e]
    s0, b = rev[-1]
    assert (s0, b) == (0, VB)
    out = [None] * N
    for t in range(nthr):
        for e in range(V):
            assert elem_index(t, e, 0, VB, logN) == V * t + e
            out[V * t + e] = regs[t][e]
    return out


def ntt_fwd_ref(a, p, fwd):
    a = [x % p for x in a]; N = len(a); t = N; m = 1
    while m < N:
        t //= 2
        for i in range(m):
            j1 = 2 * i * t; S = fwd[m + i]
            for j in range(j1, j1 + t):
                U = a[j]; V = a[j + t] * S % p
                a[j] = (U + V) % p; a[j + t] = (U - V) % p
        m *= 2
    return a


def ntt_inv_ref(a, p, inv):  # GS, bit-reversed in -> natural out, unscaled
    a = list(a); N = len(a); logN = N.bit_length() - 1
    for s in range(logN):
        t = 1 << s; h = N >> (s + 1)
        for i in range(h):
            w = inv[h + i]
            for j in range(2 * i * t, 2 * i * t + t):
                U, V = a[j], a[j + t]
                a[j] = (U + V) % p; a[j + t] = (U - V) * w % p
    return a


def negacyclic(a, b):
    N = len(a); c = [0] * N
    for i in range(N):
        if a[i] == 0:
            continue
        for k in range(N):
            if i + k < N: c[i + k] += a[i] * b[k]
            else: c[i + k - N] -= a[i] * b[k]
    return c


def main():
    for logN in range(8, 14):
        msg = bank_check(logN)
        print(f"logN={logN}: exchanges/tile", "conflict-free" if msg is None else msg)
    for logN in range(8, 14):  # lazy bounds (units of p) of the kernel's reduction schedule
        b = 2
        for k in range(logN):
            if k == 7:
                b = 4
            b += 2
            assert b <= 16, (logN, k)
        assert b <= 16 and 16 * max(P) < 2**32
    print("lazy butterfly bounds < 16p < 2^32 for logN 8..13 (one reduction, at stage 7)")
    rng = random.Random(5)
    q_in = 39
    for logN in (8, 9):
        N = 1 << logN
        rows = 3   # a few (l, i) rows of the KeySwitch sum
        D = [[rng.randrange(-128, 128) for _ in range(N)] for _ in range(rows)]
        D[0] = [-128] * N
        K = [[rng.randrange(2**q_in) for _ in range(N)] for _ in range(rows)]
        Kc = [[k - 2**q_in if k >= 2**(q_in - 1) else k for k in Kr] for Kr in K]
        exact = [0] * N
        for r in range(rows):
            for k, v in enumerate(negacyclic(D[r], K[r])): exact[k] += v
        sp = (q_in + 1) // 2                      # K = K_hi 2^sp + K_lo, centred halves
        lo = [[((k + (1 << (sp - 1))) % (1 << sp)) - (1 << (sp - 1)) for k in Kr] for Kr in Kc]
        hi = [[(k - l) >> sp for k, l in zip(Kr, Lr)] for Kr, Lr in zip(Kc, lo)]
        hb = max(sp - 1, q_in - sp)
        assert all(abs(v) <= 1 << hb for Hr in hi + lo for v in Hr)
        bb = 2 * logN + 9 + hb                    # |half-sum| <= 4N N 2^7 2^hb
        assert 2 ** (bb + 1) < P[0] * P[1]
        Z = 1 << bb
        sums = []
        for half in (hi, lo):
            res = []
            for p, g in zip(P, GEN):
                fwd, inv = tables(p, g, N)
                ninv_r = pow(N, -1, p) * 2**32 % p
                acc = [0] * N
                for r in range(rows):
                    Dh = fwd_kernel_model([d + p for d in D[r]], p, fwd, logN)
                    assert [x % p for x in Dh] == ntt_fwd_ref(D[r], p, fwd)
                    Kh = [x * ninv_r % p for x in ntt_fwd_ref(half[r], p, fwd)]
                    for k in range(N):
                        s_ = acc[k] + mont_lazy(Dh[k], Kh[k], p)
                        acc[k] = min(s_, (s_ - 2 * p) % 2**32)
                res.append([x % p for x in ntt_inv_ref([a % p for a in acc], p, inv)])
            p0, p1 = P
            out = []
            for k in range(N):
                r0, r1 = (res[0][k] + Z) % p0, (res[1][k] + Z) % p1
                h1 = (r1 - r0) * pow(p0, -1, p1) % p1
                out.append(r0 + p0 * h1 - Z)      # the exact half-sum
            sums.append(out)
        for k in range(N):
            v = (sums[0][k] * 2**sp + sums[1][k]) % 2**64
            assert v % 2**q_in == exact[k] % 2**q_in, (logN, k)
        print(f"logN={logN}: kernel-scheme forward NTTs + Montgomery pointwise + hi/lo split + 2-prime CRT "
              f"== exact negacyclic KeySwitch sum mod 2^{q_in}")


if __name__ == "__main__":
    main()
