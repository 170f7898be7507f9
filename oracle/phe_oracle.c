/*
 * CPU ORACLE (C part) for the encrypted-vector x clear-matrix hot path of arXiv 2505.07329.
 *
 * TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code, header,
 * table or constant with the CUDA product path (paper_2505_07329_b200/csrc).
 *
 * Same algorithm as oracle/phe_oracle.py, written in plain C so the literal path runs at
 * Llama shapes (d_out * L * N^2 MACs per token).  Plain uint64_t wrap-around arithmetic:
 * every modulus is a power of two <= 2^64 (R3), so wrap then mask is exact.
 * The only concession to speed is an OpenMP loop over independent output rows j.
 *
 * Pinned by tests/test_oracle_pins.py against the Python oracle (itself pinned to RFC 8439,
 * brute force, closed forms and invariants) and directly to the E=0 decryption invariant.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------- ChaCha20, RFC 8439 §2.3 (the agreed PRNG; reading R6) -------- */
static uint32_t rotl32(uint32_t v, int c) { return (v << c) | (v >> (32 - c)); }
#define QR(a, b, c, d)                                   \
  a += b; d ^= a; d = rotl32(d, 16);                     \
  c += d; b ^= c; b = rotl32(b, 12);                     \
  a += b; d ^= a; d = rotl32(d, 8);                      \
  c += d; b ^= c; b = rotl32(b, 7);

void oracle_chacha20_block(const uint8_t key[32], uint32_t counter, const uint8_t nonce[12],
                           uint8_t out[64]) {
  uint32_t s[16], w[16];
  s[0] = 0x61707865u; s[1] = 0x3320646eu; s[2] = 0x79622d32u; s[3] = 0x6b206574u;
  for (int i = 0; i < 8; i++)
    s[4 + i] = (uint32_t)key[4 * i] | ((uint32_t)key[4 * i + 1] << 8) |
               ((uint32_t)key[4 * i + 2] << 16) | ((uint32_t)key[4 * i + 3] << 24);
  s[12] = counter;
  for (int i = 0; i < 3; i++)
    s[13 + i] = (uint32_t)nonce[4 * i] | ((uint32_t)nonce[4 * i + 1] << 8) |
                ((uint32_t)nonce[4 * i + 2] << 16) | ((uint32_t)nonce[4 * i + 3] << 24);
  memcpy(w, s, sizeof w);
  for (int r = 0; r < 10; r++) {
    QR(w[0], w[4], w[8], w[12]) QR(w[1], w[5], w[9], w[13])
    QR(w[2], w[6], w[10], w[14]) QR(w[3], w[7], w[11], w[15])
    QR(w[0], w[5], w[10], w[15]) QR(w[1], w[6], w[11], w[12])
    QR(w[2], w[7], w[8], w[13]) QR(w[3], w[4], w[9], w[14])
  }
  for (int i = 0; i < 16; i++) {
    uint32_t v = w[i] + s[i];
    out[4 * i] = (uint8_t)v; out[4 * i + 1] = (uint8_t)(v >> 8);
    out[4 * i + 2] = (uint8_t)(v >> 16); out[4 * i + 3] = (uint8_t)(v >> 24);
  }
}

/* a3: A[k] = LE64(keystream word k) mod 2^q_in; key = LE64(seed)||0^24, nonce 0^12 (R6). */
void oracle_expand_mask(uint64_t seed, int N, int q_in, uint64_t *A) {
  uint8_t key[32] = {0}, nonce[12] = {0}, blk[64];
  for (int i = 0; i < 8; i++) key[i] = (uint8_t)(seed >> (8 * i));
  uint64_t m = (q_in >= 64) ? ~0ull : ((1ull << q_in) - 1);
  for (int k = 0; k < N; k++) {
    if (k % 8 == 0) oracle_chacha20_block(key, (uint32_t)(k / 8), nonce, blk);
    uint64_t v = 0;
    for (int b = 0; b < 8; b++) v |= (uint64_t)blk[8 * (k % 8) + b] << (8 * b);
    A[k] = v & m;
  }
}

/* P = a * w in Z_{2^64}[X]/(X^N+1), schoolbook (X^N = -1 per P:90). */
static void negacyclic_mul(const uint64_t *a, const int64_t *w, int N, uint64_t *P) {
  memset(P, 0, sizeof(uint64_t) * (size_t)N);
  for (int m = 0; m < N; m++) {
    uint64_t am = a[m];
    for (int n = 0; n < N - m; n++) P[m + n] += am * (uint64_t)w[n];
    for (int n = N - m; n < N; n++) P[m + n - N] -= am * (uint64_t)w[n];
  }
}

/*
 * a5-a7, one token, literally (Eq. 6):
 *   for each j: for each block i: w_hat_ij[k] = W[j, iN+N-1-k] (P:182, 0 beyond d_in);
 *   P = A_i * w_hat_ij; b' = coefficient N-1 of B_i * w_hat_ij;
 *   SampleExtract at h = N-1 (Eq. 2): a'[t] = P[N-1-t] for every t (all t <= h);
 *   LWE sums over i mod 2^q_in.
 * A, B: [L][N] residues.  out_mask: [d_out][N], out_body: [d_out].  Returns 0.
 */
int oracle_matmul_clear_literal(int N, int q_in, const int8_t *W, int64_t d_out, int64_t d_in,
                                const uint64_t *A, const uint64_t *B, uint64_t *out_mask,
                                uint64_t *out_body, int nthreads) {
  int L = (int)((d_in + N - 1) / N);
  uint64_t qm = (q_in >= 64) ? ~0ull : ((1ull << q_in) - 1);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    int64_t *what = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    uint64_t *P = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)N);
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t j = 0; j < d_out; j++) {
      uint64_t *acc = out_mask + j * (int64_t)N;
      uint64_t accb = 0;
      memset(acc, 0, sizeof(uint64_t) * (size_t)N);
      for (int i = 0; i < L; i++) {
        for (int k = 0; k < N; k++) {
          int64_t c = (int64_t)i * N + N - 1 - k;
          what[k] = (c < d_in) ? (int64_t)W[j * d_in + c] : 0;
        }
        negacyclic_mul(A + (int64_t)i * N, what, N, P);
        uint64_t bq = 0; /* coefficient N-1 of B_i * w_hat: m + n = N-1, no wrap terms */
        for (int m = 0; m < N; m++) bq += B[(int64_t)i * N + m] * (uint64_t)what[N - 1 - m];
        for (int t = 0; t < N; t++) acc[t] += P[N - 1 - t];
        accb += bq;
      }
      for (int t = 0; t < N; t++) acc[t] &= qm;
      out_body[j] = accb & qm;
    }
    free(what);
    free(P);
  }
  return 0;
}

/* Closed form, O(d_in) per mask entry:
 * a_j[t] = sum_c W[j,c] * ( A_i[m-t] if m >= t else -A_i[m-t+N] ),  i = c / N, m = c % N. */
void oracle_mask_entries(int N, int q_in, const int8_t *W, int64_t d_in, const uint64_t *A,
                         const int64_t *js, const int64_t *ts, int64_t n, uint64_t *out) {
  uint64_t qm = (q_in >= 64) ? ~0ull : ((1ull << q_in) - 1);
  for (int64_t e = 0; e < n; e++) {
    int64_t j = js[e], t = ts[e];
    uint64_t acc = 0;
    for (int64_t c = 0; c < d_in; c++) {
      int64_t i = c / N, m = c % N;
      uint64_t w = (uint64_t)(int64_t)W[j * d_in + c];
      if (m >= t) acc += w * A[i * N + (m - t)];
      else acc -= w * A[i * N + (m - t + N)];
    }
    out[e] = acc & qm;
  }
}

/* Freivalds projection of Eq. 6's LWE masks (a TEST PIN over all outputs, not a step of the method).
 * For r in Z_Q^N:  sum_t a_j[t] r[t] = sum_c W[j,c] sum_t At_i[m,t] r[t]   (c = iN + m; the closed
 * form above, At_i[m,t] = A_i[m-t] (m >= t), -A_i[m-t+N] (m < t))
 *                                    = sum_c W[j,c] (A_i * r)[m]            (negacyclic product, P:90:
 * (A*r)[m] = sum_{t<=m} A[m-t] r[t] - sum_{t>m} A[m-t+N] r[t]).  One product per (token, block, r),
 * then a plain matvec, so every output (tau, j) of a full-size run is checked against nr random
 * projections without evaluating the N^2 closed-form entries.
 * A: [T][L][N] residues; r: [nr][N] residues (< 2^63); out: [T][d_out][nr] mod 2^q_in. */
void oracle_mask_projection(int N, int q_in, const int8_t *W, int64_t d_out, int64_t d_in, const uint64_t *A,
                            int64_t T, const uint64_t *r, int nr, uint64_t *out, int nthreads) {
  int L = (int)((d_in + N - 1) / N);
  uint64_t qm = (q_in >= 64) ? ~0ull : ((1ull << q_in) - 1);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
  {
    int64_t *rv = (int64_t *)malloc(sizeof(int64_t) * (size_t)N);
    uint64_t *u = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)L * N * nr); /* [nr][L*N] */
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
    for (int64_t tau = 0; tau < T; tau++) {
      for (int e = 0; e < nr; e++) {
        for (int k = 0; k < N; k++) rv[k] = (int64_t)r[(int64_t)e * N + k];
        for (int i = 0; i < L; i++)
          negacyclic_mul(A + (tau * L + i) * (int64_t)N, rv, N, u + ((int64_t)e * L + i) * N);
      }
      for (int64_t j = 0; j < d_out; j++)
        for (int e = 0; e < nr; e++) {
          const uint64_t *ue = u + (int64_t)e * L * N;
          uint64_t acc = 0;
          for (int64_t c = 0; c < d_in; c++) acc += (uint64_t)(int64_t)W[j * d_in + c] * ue[c];
          out[(tau * d_out + j) * nr + e] = acc & qm;
        }
    }
    free(rv);
    free(u);
  }
}

/* ModulusSwitch, round half up (R8): floor((v + 2^(s-1)) / 2^s) mod 2^q_to. */
void oracle_modswitch(const uint64_t *v, int64_t n, int q_from, int q_to, uint64_t *out) {
  int s = q_from - q_to;
  uint64_t m = (q_to >= 64) ? ~0ull : ((1ull << q_to) - 1);
  for (int64_t k = 0; k < n; k++)
    out[k] = (s == 0) ? v[k] : (((v[k] + (1ull << (s - 1))) >> s) & m);
}

/* ================= NEXT #1: KeySwitch packing (Eq. 7; Eq. 4; Eq. 8) ========= */
static void keystream_words(uint64_t seed, const uint8_t nonce[12], uint64_t word0, int64_t n,
                            uint64_t *out) {
  uint8_t key[32] = {0}, blk[64];
  for (int i = 0; i < 8; i++) key[i] = (uint8_t)(seed >> (8 * i));
  int64_t cur = -1;
  for (int64_t k = 0; k < n; k++) {
    uint64_t w = word0 + (uint64_t)k;
    if ((int64_t)(w / 8) != cur) { cur = (int64_t)(w / 8); oracle_chacha20_block(key, (uint32_t)cur, nonce, blk); }
    uint64_t v = 0;
    for (int b = 0; b < 8; b++) v |= (uint64_t)blk[8 * (w % 8) + b] << (8 * b);
    out[k] = v;
  }
}

/* KSK_{i,l} = RLWE_S(S'_i 2^(q-(l+1)B)), row l*N+i; A from nonce "phe-ksk", noise CBD(eta)
 * from "phe-ksknoise", both in word order (l, i, k) (R18-R20). */
void oracle_ksk_gen(int N, int q, const uint8_t *S, uint64_t ksk_seed, int eta, int base_log,
                    int levels, uint64_t *KA, uint64_t *KB, int nthreads) {
  static const uint8_t n_ksk[12] = {'p', 'h', 'e', '-', 'k', 's', 'k', 0, 0, 0, 0, 0};
  static const uint8_t n_kno[12] = {'p', 'h', 'e', '-', 'k', 's', 'k', 'n', 'o', 'i', 's', 'e'};
  uint64_t qm = (q >= 64) ? ~0ull : ((1ull << q) - 1);
  int64_t rows = (int64_t)levels * N;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
  for (int64_t r = 0; r < rows; r++) {
    uint64_t *A = KA + r * N, *B = KB + r * N;
    keystream_words(ksk_seed, n_ksk, (uint64_t)r * N, N, A);
    for (int k = 0; k < N; k++) A[k] &= qm;
    for (int k = 0; k < N; k++) { /* (A*S)[k] = sum_n S_n (A[k-n] or -A[k-n+N]) */
      uint64_t acc = 0;
      for (int n = 0; n < N; n++)
        if (S[n]) acc += (k >= n) ? A[k - n] : (0ull - A[k - n + N]);
      B[k] = acc;
    }
    if (eta > 0) {
      uint64_t *w = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)N);
      keystream_words(ksk_seed, n_kno, (uint64_t)r * N, N, w);
      uint64_t m = (1ull << eta) - 1;
      for (int k = 0; k < N; k++)
        B[k] += (uint64_t)((int64_t)__builtin_popcountll(w[k] & m) - (int64_t)__builtin_popcountll((w[k] >> eta) & m));
      free(w);
    }
    int l = (int)(r / N), i = (int)(r % N);
    B[0] += (uint64_t)S[i] << (q - (l + 1) * base_log);
    for (int k = 0; k < N; k++) B[k] &= qm;
  }
}

/* Decomp (Eq. 4): signed balanced digits of the top base_log*levels bits, tail rounded half up. */
void oracle_decompose(uint64_t v, int q, int base_log, int levels, int32_t *digits) {
  int tail = q - base_log * levels;
  uint64_t vr = (v + (tail > 0 ? (1ull << (tail - 1)) : 0)) >> tail;
  int bits = base_log * levels;
  if (bits < 64) vr &= (1ull << bits) - 1;
  for (int l = levels - 1; l >= 0; l--) {
    int64_t d = (int64_t)(vr & ((1ull << base_log) - 1));
    vr >>= base_log;
    if (d >= (1ll << (base_log - 1))) { d -= (1ll << base_log); vr += 1; }
    digits[l] = (int32_t)d;
  }
}

/* Eq. 7 literally for one token: every LWE j is keyswitched (Eq. 4), rotated by j mod N
 * (X^N = -1), summed into group j / N.  A_lwe [d_out][N], b_lwe [d_out]; PA, PB [G][N]. */
void oracle_pack(int N, int q, const uint64_t *A_lwe, const uint64_t *b_lwe, int64_t d_out,
                 const uint64_t *KA, const uint64_t *KB, int base_log, int levels, uint64_t *PA,
                 uint64_t *PB, int nthreads) {
  uint64_t qm = (q >= 64) ? ~0ull : ((1ull << q) - 1);
  int64_t G = (d_out + N - 1) / N;
  memset(PA, 0, sizeof(uint64_t) * (size_t)(G * N));
  memset(PB, 0, sizeof(uint64_t) * (size_t)(G * N));
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  for (int64_t g = 0; g < G; g++) {
    const int64_t jend = ((g + 1) * N < d_out) ? (g + 1) * N : d_out;
#ifdef _OPENMP
#pragma omp parallel
#endif
    {
      uint64_t *Ap = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)N);
      uint64_t *Bp = (uint64_t *)malloc(sizeof(uint64_t) * (size_t)N);
      uint64_t *accA = (uint64_t *)calloc((size_t)N, sizeof(uint64_t));
      uint64_t *accB = (uint64_t *)calloc((size_t)N, sizeof(uint64_t));
      int32_t dg[64];
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
      for (int64_t j = g * N; j < jend; j++) {
        memset(Ap, 0, sizeof(uint64_t) * (size_t)N);
        memset(Bp, 0, sizeof(uint64_t) * (size_t)N);
        Bp[0] = b_lwe[j];
        for (int i = 0; i < N; i++) {
          oracle_decompose(A_lwe[j * N + i], q, base_log, levels, dg);
          for (int l = 0; l < levels; l++) {
            if (!dg[l]) continue;
            uint64_t d = (uint64_t)(int64_t)dg[l];
            const uint64_t *ka = KA + ((int64_t)l * N + i) * N, *kb = KB + ((int64_t)l * N + i) * N;
            for (int k = 0; k < N; k++) { Ap[k] -= d * ka[k]; Bp[k] -= d * kb[k]; }
          }
        }
        int r = (int)(j - g * N); /* Rotate by X^r and accumulate */
        for (int k = 0; k < N; k++) {
          int p = k + r;
          if (p < N) { accA[p] += Ap[k]; accB[p] += Bp[k]; }
          else { accA[p - N] -= Ap[k]; accB[p - N] -= Bp[k]; }
        }
      }
#ifdef _OPENMP
#pragma omp critical
#endif
      for (int k = 0; k < N; k++) { PA[g * N + k] += accA[k]; PB[g * N + k] += accB[k]; }
      free(Ap); free(Bp); free(accA); free(accB);
    }
    for (int k = 0; k < N; k++) { PA[g * N + k] &= qm; PB[g * N + k] &= qm; }
  }
}
