// ntt_path.cu — NEXT #4: the mask contraction a5 computed in the NTT domain.
//
// Eq. 6 needs, per token tau and output row j, the mask polynomial
//   P_{tau,j} = sum_i A_{tau,i} * w_hat_ij   in Z[X]/(X^N + 1)          (negacyclic)
// and then SampleExtract at h = N-1 (Eq. 2): a'_t = P[N-1-t].  The paper computes the
// products "coefficient-wise".  Power-of-two moduli have no NTT, so this path
// computes an EXACT integer with negacyclic NTTs modulo two 30-bit primes p0, p1 (p0 p1 ~ 2^59.8)
// and recovers it by CRT.  The masks are centred first, A' = A - H with H = 2^(q_in - 1), so
// |P'| = |sum_i A'_i * w_hat_ij| <= L N H 128 (< 2^59 for Table 1 up to L = 6); since every
// coefficient of 1 * w_hat (negacyclic) has the parity of the weight sum, P = P' + H * par_j
// mod 2^q_in with par_j = (sum_c W[j,c]) mod 2, one bit per row.  The result is bit-identical to
// the dense limb GEMM (limb_gemm.cu): both produce the unique value Eq. 6 defines.
//
// Work per output coefficient: L Montgomery products per prime (pointwise) + (log2 N)/2 GS
// butterflies per prime (inverse NTT) + CRT + ModulusSwitch — O(L + log N) instead of the
// dense path's O(L*N) MACs; it runs on the integer ALUs (CUDA cores), not the tensor cores.
//
// Kernels:
//   ntt_tables_kernel    psi^{bitrev(k)}, psi^{-bitrev(k)} with Shoup companions, both primes, and
//                        the hot kernel's per-thread phase-1 twiddle table
//   ntt_weights_kernel   W_hat_ij = NTT(w_hat_ij) * N^{-1} * 2^32 (Montgomery form)  [server, once]
//   ntt_rowpar_kernel    par_j = (sum_c W[j,c]) mod 2                                  [server, once]
//   ntt_masks_kernel     A_hat_{tau,i} = NTT(PRNG(seed_{tau,i}) - H mod p)             [per batch]
//   ntt_encrypt_kernel   client encrypt_pack with A*S = INTT(NTT(A) o NTT(S)) (phe_encrypt_pack_ntt)
//   ntt_mask_kernel<LOGN, SW, NG, NB, WSM, SHIFT, OUTB>  the hot kernel: NG token groups of N/16
//                        threads (16 values per prime per thread) share the twiddles and W_hat_j
//                        in shared memory; pointwise sum over i, lazy inverse NTT in registers with
//                        4-bit phases and additive bank-conflict-free exchange layouts
//                        (tools/ntt_model.py checks the index scheme), compare-free CRT, parity
//                        correction, SampleExtract reversal, fused ModulusSwitch, coalesced stores.
#include <cstdint>
#include <cstdio>

#include "phe_common.cuh"
#include "side_kernels.cuh"

namespace phe {
namespace ntt {

// ---------------------------------------------------------------- primes and constants
// p0 = 119*2^23 + 1, p1 = 479*2^21 + 1 (generator 3 for both): = 1 mod 2^14 (negacyclic NTTs
// up to N = 8192) and < 2^30, so 4p < 2^32: values are kept lazily in [0, 2p) (Harvey) and
// every butterfly needs one conditional subtraction instead of two.  p0 < p1.
constexpr uint32_t P0 = 998244353u, P1 = 1004535809u;
constexpr uint32_t GEN0 = 3u, GEN1 = 3u;

__host__ __device__ constexpr uint32_t neg_inv32(uint32_t p) {
  uint32_t x = p;  // Newton: x <- x*(2 - p*x) doubles the correct low bits (p odd)
  for (int i = 0; i < 5; i++) x *= 2u - p * x;
  return 0u - x;
}
__host__ __device__ constexpr uint32_t pw(uint64_t b, uint64_t e, uint32_t p) {
  uint64_t r = 1;
  b %= p;
  while (e) {
    if (e & 1) r = r * b % p;
    b = b * b % p;
    e >>= 1;
  }
  return (uint32_t)r;
}
constexpr uint32_t PINV0 = neg_inv32(P0), PINV1 = neg_inv32(P1);
constexpr uint32_t CRT_C = pw(P0, P1 - 2, P1);  // p0^{-1} mod p1
constexpr uint32_t CRT_CQ = (uint32_t)(((uint64_t)CRT_C << 32) / P1);
constexpr uint64_t CRT_M = (uint64_t)P0 * P1;
static_assert((uint32_t)(P0 * (0u - PINV0)) == 1u, "Montgomery constant p0");
static_assert((uint32_t)(P1 * (0u - PINV1)) == 1u, "Montgomery constant p1");
static_assert((uint64_t)P0 * CRT_C % P1 == 1, "CRT constant");

__device__ __forceinline__ uint32_t prime(int pr) { return pr ? P1 : P0; }
__device__ __forceinline__ uint32_t pinv(int pr) { return pr ? PINV1 : PINV0; }

// a, b < p < 2^31
__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t s = a + b;
  return min(s, s - p);
}
// x < 2^32 arbitrary, w < p, wq = floor(w 2^32 / p): x*w mod p (Shoup), result < p
__device__ __forceinline__ uint32_t mul_shoup(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
  const uint32_t q = __umulhi(x, wq);
  const uint32_t r = x * w - q * p;
  return min(r, r - p);
}
// a, b < p: a*b*2^-32 mod p (Montgomery), result < p
__device__ __forceinline__ uint32_t mul_mont(uint32_t a, uint32_t b, uint32_t p, uint32_t pi) {
  const uint64_t t = (uint64_t)a * b;
  const uint32_t m = (uint32_t)t * pi;
  const uint32_t u = (uint32_t)((t + (uint64_t)m * p) >> 32);
  return min(u, u - p);
}
// ---- lazy forms (4p < 2^32): operands and results in [0, 2p)
__device__ __forceinline__ uint32_t add_lazy(uint32_t a, uint32_t b, uint32_t p) {
  const uint32_t s = a + b;
  return min(s, s - 2 * p);
}
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t x, uint32_t w, uint32_t wq, uint32_t p) {
  return x * w - __umulhi(x, wq) * p;  // x < 2^32: result in [0, 2p)
}
__device__ __forceinline__ uint32_t mont_lazy(uint32_t a, uint32_t b, uint32_t p, uint32_t pi) {
  const uint64_t t = (uint64_t)a * b;  // a, b < 2p: t < 4p^2, result (t + m p) / 2^32 < 2p
  const uint32_t m = (uint32_t)t * pi;
  return (uint32_t)((t + (uint64_t)m * p) >> 32);
}

__device__ __forceinline__ uint32_t brev(uint32_t k, int logN) { return __brev(k) >> (32 - logN); }

// Storage order of NTT-domain vectors (W_hat, A_hat; per prime, N words): element k (bit-reversed
// transform order) of thread t = k/16 of the hot kernel, k = 16t + 4v + c, is stored at word
// 4 (v NT + t) + c (NT = N/16), so each of the thread's four 16-byte loads is one contiguous
// 512-byte warp access.
__host__ __device__ __forceinline__ int tpos(int k, int N) {
  return 4 * (((k >> 2) & 3) * (N / 16) + (k >> 4)) + (k & 3);
}

// ---------------------------------------------------------------- tables
// d_tables layout: uint2 [2 dirs][2 primes][N]; dir 0 = psi^{bitrev(k)} (forward CT),
// dir 1 = psi^{-bitrev(k)} (inverse GS); .x = w, .y = floor(w 2^32 / p).  psi = g^((p-1)/2N)
// is a primitive 2N-th root of unity (psi^N = -1: the negacyclic twist, X^N = -1).
// Followed by the phase-1 section used by the hot kernel: uint2 [15][N/16][2 primes], entry
// [P1OFF[s] + m][t][pr] = inverse twiddle (N >> (s+1)) + t 2^(3-s) + m for stages s = 0..3 of
// the inverse NTT (thread t's m-th twiddle of stage s; one 16-byte load serves both primes and a
// warp's loads are contiguous).
__host__ __device__ constexpr int p1off(int s) { return s == 0 ? 0 : s == 1 ? 8 : s == 2 ? 12 : 14; }
__global__ void ntt_tables_kernel(int logN, uint32_t psi0, uint32_t psi1, uint2 *__restrict__ tab) {
  const int N = 1 << logN, NT = N / 16;
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= 4 * N + 2 * 15 * NT) return;
  int k, pr, dir;
  if (idx < 4 * N) {
    k = idx % N; pr = (idx / N) & 1; dir = idx / (2 * N);
  } else {
    const int r = idx - 4 * N;
    pr = r & 1; dir = 1;
    const int t = (r >> 1) % NT, slot = (r >> 1) / NT;
    const int s = slot >= 14 ? 3 : slot >= 12 ? 2 : slot >= 8 ? 1 : 0;
    k = (N >> (s + 1)) + t * (1 << (3 - s)) + (slot - p1off(s));
  }
  const uint32_t p = prime(pr), psi = pr ? psi1 : psi0;
  const uint32_t e = brev((uint32_t)k, logN);
  const uint32_t ex = dir ? (uint32_t)((2 * N - e) % (2 * N)) : e;
  const uint32_t w = pw(psi, ex, p);
  tab[idx] = make_uint2(w, (uint32_t)(((uint64_t)w << 32) / p));
}

// In-place forward negacyclic NTT (Cooley-Tukey, natural order in, bit-reversed out) of the two
// prime residue arrays x[pr][N] in shared memory; all threads of the CTA take part.
__device__ void ntt_forward_smem(uint32_t *x, const uint2 *__restrict__ tab, int logN) {
  const int N = 1 << logN;
  for (int s = logN - 1, m = 1; s >= 0; s--, m <<= 1) {  // half-distance t = 2^s
    const int t = 1 << s;
    for (int b = threadIdx.x; b < 2 * (N / 2); b += blockDim.x) {
      const int pr = b / (N / 2), bb = b % (N / 2);
      const int i = bb >> s, j = 2 * i * t + (bb & (t - 1));
      const uint32_t p = prime(pr);
      const uint2 w = __ldg(&tab[pr * N + m + i]);  // forward slice [pr][N]
      uint32_t *a = x + pr * N;
      const uint32_t U = a[j], V = mul_shoup(a[j + t], w.x, w.y, p);
      a[j] = add_mod(U, V, p);
      a[j + t] = add_mod(U, p - V, p);
    }
    __syncthreads();
  }
}

constexpr int PREP_THREADS = 256;

// In-place inverse negacyclic NTT (Gentleman-Sande, bit-reversed in, natural out, unscaled) of the
// two prime residue arrays x[pr][N] in shared memory; tinv = inverse slice [2][N] of the table.
__device__ void ntt_inverse_smem(uint32_t *x, const uint2 *__restrict__ tinv, int logN) {
  const int N = 1 << logN;
  for (int s = 0; s < logN; s++) {  // half-distance t = 2^s, twiddle (N >> (s+1)) + group
    const int t = 1 << s, h = N >> (s + 1);
    for (int b = threadIdx.x; b < 2 * (N / 2); b += blockDim.x) {
      const int pr = b / (N / 2), bb = b % (N / 2);
      const int i = bb >> s, j = 2 * i * t + (bb & (t - 1));
      const uint32_t p = prime(pr);
      const uint2 w = __ldg(&tinv[pr * N + h + i]);
      uint32_t *a = x + pr * N;
      const uint32_t U = a[j], V = a[j + t];
      a[j] = add_mod(U, V, p);
      a[j + t] = mul_shoup(U - V + p, w.x, w.y, p);
    }
    __syncthreads();
  }
}

// W_hat for row j, block i of the prepared matrix M (= W or W^T):
// w_hat_ij[k] = M[j, iN + N-1-k] (0 beyond cols), then NTT, then * N^{-1} 2^32 mod p.
__global__ void __launch_bounds__(PREP_THREADS)
ntt_weights_kernel(int logN, const int8_t *__restrict__ W, int64_t d_in, int transpose, int64_t cols,
                   int64_t Lc, const uint2 *__restrict__ tab, uint32_t c0, uint32_t c1,
                   uint32_t *__restrict__ out) {
  extern __shared__ uint32_t xs[];
  const int N = 1 << logN;
  const int64_t ji = blockIdx.x, j = ji / Lc, i = ji % Lc;
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const int64_t c = i * N + (N - 1 - k);
    int v = 0;
    if (c < cols) v = transpose ? W[c * d_in + j] : W[j * d_in + c];
    xs[k] = v < 0 ? (uint32_t)((int64_t)P0 + v) : (uint32_t)v;
    xs[N + k] = v < 0 ? (uint32_t)((int64_t)P1 + v) : (uint32_t)v;
  }
  __syncthreads();
  ntt_forward_smem(xs, tab, logN);
  uint32_t *o = out + ji * 2 * N;
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) {
    const int pr = k / N;
    o[pr * N + tpos(k % N, N)] = (uint32_t)((uint64_t)xs[k] * (pr ? c1 : c0) % prime(pr));
  }
}

// A_hat for token tau, block i: A = ChaCha20(seed_{tau,i}) mod 2^q_in (R6), centred
// A' = A - 2^(q_in-1), mod p, NTT.
__global__ void __launch_bounds__(PREP_THREADS)
ntt_masks_kernel(KParams kp, int logN, const uint64_t *__restrict__ seeds,
                 const uint2 *__restrict__ tab, uint32_t *__restrict__ out) {
  extern __shared__ uint32_t xs[];
  const int N = 1 << logN;
  const int64_t blk = blockIdx.x;  // tau * L + i
  const uint64_t seed = seeds[blk];
  const uint64_t H = 1ull << (kp.q_in - 1);
  const uint32_t h0 = (uint32_t)(H % P0), h1 = (uint32_t)(H % P1);
  for (int g = threadIdx.x; g < N / 8; g += blockDim.x) {
    uint64_t w[8];
    chacha20_u64x8(seed, (uint32_t)g, nonce_mask(), w);
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const uint64_t a = w[e] & kp.qmask;
      xs[8 * g + e] = add_mod((uint32_t)(a % P0), P0 - h0, P0);
      xs[N + 8 * g + e] = add_mod((uint32_t)(a % P1), P1 - h1, P1);
    }
  }
  __syncthreads();
  ntt_forward_smem(xs, tab, logN);
  uint32_t *o = out + blk * 2 * N;
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) o[(k / N) * N + tpos(k % N, N)] = xs[k];
}

// par[j] = (sum_c M[j, c]) mod 2 (the centring correction bit of row j); one warp per row
__global__ void ntt_rowpar_kernel(const int8_t *__restrict__ W, int64_t d_in, int transpose, int64_t rows,
                                  int64_t cols, uint8_t *__restrict__ par) {
  const int64_t j = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  if (j >= rows) return;
  int s = 0;
  for (int64_t c = threadIdx.x % 32; c < cols; c += 32) s += transpose ? W[c * d_in + j] : W[j * d_in + c];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (threadIdx.x % 32 == 0) par[j] = (uint8_t)(s & 1);
}

// encrypt_pack through the NTT (client side): B = A*S + E + Delta*x_hat mod 2^q_in (P:58, P:62,
// P:174), with the negacyclic product A*S (|A*S| < N 2^q_in) computed exactly as
// INTT(NTT(A) o NTT(S) N^-1) modulo p0, p1 and recovered by a centred CRT.  One CTA per block;
// bit-identical to encrypt_kernel (side_kernels.cu).
__global__ void __launch_bounds__(PREP_THREADS)
ntt_encrypt_kernel(KParams kp, int logN, const uint8_t *__restrict__ S, const int8_t *__restrict__ x,
                   int64_t d_in, int64_t L, uint64_t seed_base, uint64_t noise_seed,
                   const uint2 *__restrict__ tab, uint32_t c0, uint32_t c1, uint64_t *__restrict__ seeds,
                   uint64_t *__restrict__ body) {
  extern __shared__ uint32_t xs[];  // [2][N] A, then [2][N] S
  const int N = 1 << logN;
  uint32_t *ys = xs + 2 * N;
  const int64_t blk = blockIdx.x;  // tau * L + i
  const int64_t tau = blk / L, i = blk % L;
  const uint64_t seed = seed_base + (uint64_t)blk;
  if (threadIdx.x == 0) seeds[blk] = seed;
  for (int g = threadIdx.x; g < N / 8; g += blockDim.x) {
    uint64_t w[8];
    chacha20_u64x8(seed, (uint32_t)g, nonce_mask(), w);
#pragma unroll
    for (int e = 0; e < 8; e++) {
      const uint64_t a = w[e] & kp.qmask;
      xs[8 * g + e] = (uint32_t)(a % P0);
      xs[N + 8 * g + e] = (uint32_t)(a % P1);
    }
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) ys[k] = ys[N + k] = S[k];
  __syncthreads();
  ntt_forward_smem(xs, tab, logN);
  ntt_forward_smem(ys, tab, logN);
  for (int k = threadIdx.x; k < 2 * N; k += blockDim.x) {
    const int pr = k / N;
    const uint32_t p = prime(pr);
    const uint32_t sm = (uint32_t)((uint64_t)ys[k] * (pr ? c1 : c0) % p);  // S_hat N^-1 2^32
    xs[k] = mul_mont(xs[k], sm, p, pinv(pr));
  }
  __syncthreads();
  ntt_inverse_smem(xs, tab + 2 * N, logN);
  const uint64_t delta = 1ull << (kp.q_in - kp.beta);
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const uint32_t r0 = xs[k], r1 = xs[N + k];
    const uint32_t h = mul_shoup(add_mod(r1, P1 - r0, P1), CRT_C, CRT_CQ, P1);
    uint64_t v = (uint64_t)r0 + (uint64_t)P0 * h;
    if (v >= CRT_M / 2) v -= CRT_M;  // centred A*S; wraps mod 2^64
    const int64_t c = i * (int64_t)N + k;
    const int64_t xv = (c < d_in) ? (int64_t)x[tau * d_in + c] : 0;
    int64_t ev = 0;
    if (kp.eta > 0) {  // as encrypt_kernel: one keystream word per coefficient, order (tau, i, k)
      const uint64_t widx = (uint64_t)blk * (uint64_t)N + (uint64_t)k;
      uint32_t o[16];
      chacha20_block(noise_seed, (uint32_t)(widx >> 3), nonce_noise(), o);
      const int q = (int)(widx & 7);
      const uint64_t wd = (uint64_t)o[2 * q] | ((uint64_t)o[2 * q + 1] << 32);
      const uint64_t m = mask_bits(kp.eta);
      ev = (int64_t)__popcll(wd & m) - (int64_t)__popcll((wd >> kp.eta) & m);
    }
    body[blk * (int64_t)N + k] = (v + (uint64_t)ev + delta * (uint64_t)xv) & kp.qmask;
  }
}

// ---------------------------------------------------------------- the hot kernels
struct MaskArgs {
  const uint2 *tinv;        // inverse twiddles [2][N] (dir-1 slice of the table)
  const uint32_t *what;     // [rows][Lc][2][N]
  const uint8_t *par;       // [rows] centring correction bits
  const uint32_t *ahat;     // [T][Lc][2][N]
  int64_t Lc, row_begin, R, T;
  int tok_per_cta;
  int64_t n_chunks;         // ceil(T / tok_per_cta)
  int q_in, out_bits;
  uint64_t qmask;
  uint32_t crt_k1;          // ((Z mod p1 - Z mod p0) mod p1) + 2 p1, Z the CRT offset (crt_store)
  uint32_t crt_z0;          // Z mod p0
  void *out;                // [T][R][N] uint32 (switched) or uint64; DIG: int8 [T][digit_rows][4][N]
  int64_t digit_rows;       // DIG: row stride of the digit tensor
  int64_t out_rows;         // row stride of the output tensor [T][out_rows][N] (>= R)
  int64_t plane;            // DIG: N (bytes between digit planes)
};

// Thread/element mapping of the inverse NTT: N/16 threads per residue array, 16 values each;
// phase (S0, B) makes index bits [S0, S0+B) thread-local (B <= 4).  Element e of thread tid:
template <int LOGN, int S0, int B>
__device__ __forceinline__ int eidx(int tid, int e) {
  const int el = e & ((1 << B) - 1), g = e >> B;
  const int o = tid | (g << (LOGN - 4));
  return (o & ((1 << S0) - 1)) | (el << S0) | ((o >> S0) << (S0 + B));
}
// The thread bits and element bits of eidx are disjoint, so any function linear in the index
// bits splits into a per-thread base plus a compile-time constant per element (immediate
// offsets in LDS/STS, no per-element address registers).
//
// Shared-memory layout of exchange X (written with phase X's mapping, read with phase X+1's):
// chosen so that both warp-wide access patterns hit 32 distinct banks (tools/ntt_model.py
// checks every N in [512, 8192]); exchange 0: j + j/16, exchange 1: j + 16 (j/256), else j.
template <int X>
__device__ __forceinline__ int lay(int j) { return X == 0 ? j + (j >> 4) : X == 1 ? j + 16 * (j >> 8) : j; }
template <int LOGN>
__host__ __device__ constexpr int xwords() { return (1 << LOGN) + (1 << LOGN) / 16; }  // per prime

// Gentleman-Sande stages S0..S0+B-1 (half-distance 2^s) on NP residue arrays in registers.
// Twiddles in shared memory: tw1 = phase-1 table [NP][15][N/16] (see ntt_tables_kernel), twl =
// inverse-table entries [NP][N/16] (phases >= 2 only index below N/16; their loads are
// broadcasts).  All warp-wide twiddle loads are conflict-free.
template <int LOGN, int S0, int B, int NP>
__device__ __forceinline__ void gs_phase(uint32_t (&r)[NP][16], const uint4 *tw1, const uint4 *twl,
                                         const uint32_t (&p)[NP], int tid) {
  static_assert(NP == 2, "both primes per thread");
  constexpr int N = 1 << LOGN, NT = N / 16;
  const int jt = eidx<LOGN, S0, B>(tid, 0);
#pragma unroll
  for (int s = S0; s < S0 + B; s++) {
    const int d = 1 << (s - S0);
    const int tb = (N >> (s + 1)) + (jt >> (s + 1));
#pragma unroll
    for (int e = 0; e < 16; e++) {
      if (e & d) continue;
      const int ti = tb + (eidx<LOGN, S0, B>(0, e) >> (s + 1));
      const uint4 w4 = S0 == 0 ? tw1[(p1off(s) + (e >> (s + 1))) * NT + tid] : twl[ti];
#pragma unroll
      for (int q = 0; q < NP; q++) {
        const uint32_t w = q ? w4.z : w4.x, wq = q ? w4.w : w4.y;
        const uint32_t U = r[q][e], V = r[q][e | d];  // lazy: in [0, 2p)
        r[q][e] = add_lazy(U, V, p[q]);
        r[q][e | d] = shoup_lazy(U - V + 2 * p[q], w, wq, p[q]);
      }
    }
  }
}
// Both residues of an element travel as one 8-byte word: a half-warp's 16 lanes hit 16
// distinct 8-byte bank pairs (the layouts are distinct mod 16 on every half-warp pattern).
template <int LOGN, int S0, int B, int X, int NP>
__device__ __forceinline__ void xstore(const uint32_t (&r)[NP][16], uint32_t *xb, int tid) {
  const int base = lay<X>(eidx<LOGN, S0, B>(tid, 0));
  uint2 *x2 = reinterpret_cast<uint2 *>(xb);
#pragma unroll
  for (int e = 0; e < 16; e++) x2[base + lay<X>(eidx<LOGN, S0, B>(0, e))] = make_uint2(r[0][e], r[1][e]);
}
template <int LOGN, int S0, int B, int X, int NP>
__device__ __forceinline__ void xload(uint32_t (&r)[NP][16], const uint32_t *xb, int tid) {
  const int base = lay<X>(eidx<LOGN, S0, B>(tid, 0));
  const uint2 *x2 = reinterpret_cast<const uint2 *>(xb);
#pragma unroll
  for (int e = 0; e < 16; e++) {
    const uint2 v = x2[base + lay<X>(eidx<LOGN, S0, B>(0, e))];
    r[0][e] = v.x;
    r[1][e] = v.y;
  }
}

// CRT of (r0 mod p0, r1 mod p1) -> the centred integer mod 2^q_in -> [switch] -> store at a'_t,
// t = N-1-jj (SampleExtract at h = N-1, Eq. 2: a'_t = P[N-1-t]).
// SHIFT > 0: switch by a compile-time SHIFT = q_in - q_out (Table 1: 13) to OUTB = q_out bits.
// Bits [s, q_in) of ((v mod 2^q_in) + 2^(s-1)) equal bits [s, q_in) of (v + 2^(s-1)), so the
// rounding constant rides in the CRT's wide multiply-add and no 64-bit masking is needed.
// CRT without a centring compare.  Z is a multiple of 2^q_in with P' + Z in [2 p0, p0 p1) for
// every P' the launch can produce (host: launch_ntt_mask), so with r0 in [0, 2p0) (lazy),
// r1 reduced, h = (r1 - r0 + Z1 - Z0) p0^-1 mod p1 and v = p0 h + r0 + Z0 in [0, p0 p1 + 2 p0)
// the only representative is v = P' + Z exactly; Z vanishes mod 2^q_in.  kadd = Z0 + H par_j
// (+ the switch's rounding constant) is a per-CTA constant.
template <bool SW, int SHIFT, int OUTB, bool DIG = false>
__device__ __forceinline__ void crt_store(const MaskArgs &a, uint32_t r0, uint32_t r1, uint64_t kadd,
                                          int64_t o, int s_shift, uint32_t omask) {
  r1 = min(r1, r1 - P1);
  const uint32_t h = mul_shoup(r1 - r0 + a.crt_k1, CRT_C, CRT_CQ, P1);  // argument < 4 p1 < 2^32
  const uint64_t x = (uint64_t)P0 * h + r0 + kadd;                       // P + Z [+ 2^(s-1)]
  if constexpr (DIG) {
    // Decomp (Eq. 4 / S:59-67; R18): r = top 32 bits of a'_t after rounding the q_in - 32 bit
    // tail half up; signed base-2^8 digits, least significant first with carry.  o addresses
    // plane 0 (weight 2^(q_in - 8)) of [tau][j][l][t]; plane l is l * N bytes further.
    uint32_t r = (uint32_t)(x >> (SHIFT > 0 ? SHIFT : s_shift));
    int8_t *od = static_cast<int8_t *>(a.out) + o;
#pragma unroll
    for (int l = KS_LEVELS - 1; l >= 0; l--) {
      int dl = (int)(r & 255u);
      r >>= 8;
      if (dl >= 128) { dl -= 256; r += 1; }
      od[(int64_t)l * a.plane] = (int8_t)dl;
    }
    return;
  }
  if constexpr (SW && SHIFT > 0) {
    static_cast<uint32_t *>(a.out)[o] = (uint32_t)(x >> SHIFT) & ((1u << OUTB) - 1u);
  } else if constexpr (SW) {
    static_cast<uint32_t *>(a.out)[o] = (uint32_t)(x >> s_shift) & omask;
  } else {
    static_cast<uint64_t *>(a.out)[o] = x & a.qmask;
  }
}

// Barrier over the N/16 threads of one token group (named barrier 1 + group; NG = 1 uses the
// CTA barrier).
template <int LOGN, int NG>
__device__ __forceinline__ void gsync(int grp) {
  if (NG == 1) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(1 + grp), "r"((1 << LOGN) / 16) : "memory");
  }
}

// The inverse NTT by phases, exchanges through `xb` (NBUF = 2: alternate halves, one barrier
// per exchange; NBUF = 1: a barrier before every store as well).
template <int LOGN, int NP, int NBUF, int NG>
__device__ __forceinline__ void intt(uint32_t (&r)[NP][16], const uint4 *tw1, const uint4 *twl,
                                     const uint32_t (&p)[NP], uint32_t *xb, int tid, int grp) {
  uint32_t *x0 = xb, *x1 = NBUF == 2 ? xb + NP * xwords<LOGN>() : xb;
  gs_phase<LOGN, 0, 4, NP>(r, tw1, twl, p, tid);
  if (NBUF == 1) gsync<LOGN, NG>(grp);
  xstore<LOGN, 0, 4, 0, NP>(r, x0, tid);
  gsync<LOGN, NG>(grp);
  xload<LOGN, 4, 4, 0, NP>(r, x0, tid);
  gs_phase<LOGN, 4, 4, NP>(r, tw1, twl, p, tid);
  constexpr int B2 = LOGN - 8 < 4 ? LOGN - 8 : 4;
  if (NBUF == 1) gsync<LOGN, NG>(grp);
  xstore<LOGN, 4, 4, 1, NP>(r, x1, tid);
  gsync<LOGN, NG>(grp);
  xload<LOGN, 8, B2, 1, NP>(r, x1, tid);
  gs_phase<LOGN, 8, B2, NP>(r, tw1, twl, p, tid);
  if constexpr (LOGN > 12) {  // N = 8192: a fourth (1-bit) phase
    gsync<LOGN, NG>(grp);
    xstore<LOGN, 8, 4, 2, NP>(r, x0, tid);
    gsync<LOGN, NG>(grp);
    xload<LOGN, 12, 1, 2, NP>(r, x0, tid);
    gs_phase<LOGN, 12, 1, NP>(r, tw1, twl, p, tid);
  }
}
template <int LOGN>
struct LastPhase {
  static constexpr int S0 = LOGN > 12 ? 12 : 8;
  static constexpr int B = LOGN > 12 ? 1 : (LOGN - 8 < 4 ? LOGN - 8 : 4);
};

// ---- the hot kernel: NG token groups of N/16 threads per CTA share one twiddle copy; each
// group computes both residues of its (j, tau) polynomials, 16 values per prime per thread.
template <int LOGN>
__host__ __device__ constexpr int tw_smem_entries() { return 2 * 16 * ((1 << LOGN) / 16); }  // tw1 + twl
template <int LOGN, int NG, int NB>
__host__ __device__ constexpr int ntt_smem() {
  return tw_smem_entries<LOGN>() * 8 + NG * NB * 2 * xwords<LOGN>() * 4;
}
// stage the kernel's twiddles (both primes per 16-byte entry): tw1 <- the table's phase-1
// section [15][NT][2], twl[k] <- inverse entries k < NT of both primes
template <int LOGN>
__device__ __forceinline__ void load_twiddles(const uint2 *tinv, uint4 *tw1, uint4 *twl, int t0, int nthr) {
  constexpr int N = 1 << LOGN, NT = N / 16;
  const uint4 *p1 = reinterpret_cast<const uint4 *>(tinv + 2 * N);  // follows the inverse slice
  for (int k = t0; k < 15 * NT; k += nthr) tw1[k] = p1[k];
  for (int k = t0; k < NT; k += nthr) {
    const uint2 a = tinv[k], b = tinv[N + k];
    twl[k] = make_uint4(a.x, a.y, b.x, b.y);
  }
}

template <int LOGN, int NG>
__host__ __device__ constexpr int ntt_min_blocks() {  // target 512 threads / SM: 128 registers
  return 512 / (NG * (1 << LOGN) / 16) > 1 ? 512 / (NG * (1 << LOGN) / 16) : 1;
}

// WSM: W_hat_j (all Lc blocks, 8 N bytes each) staged in shared memory once per CTA and shared
// by the NG token groups; else read through L1/L2.
template <int LOGN, bool SW, int NG, int NB, bool WSM, int SHIFT = 0, int OUTB = 0, bool DIG = false>
__global__ void __launch_bounds__(NG * (1 << LOGN) / 16, ntt_min_blocks<LOGN, NG>())
ntt_mask_kernel(MaskArgs a) {
  constexpr int N = 1 << LOGN, NT = N / 16;
  static_assert(LOGN >= 9 && LOGN <= 13, "N in [512, 8192]");
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint4 *tw1 = reinterpret_cast<uint4 *>(smem_raw);
  uint4 *twl = tw1 + 15 * NT;
  const int grp = threadIdx.x / NT;   // token group (warp-aligned)
  const int tid = threadIdx.x % NT;
  uint32_t *xb = reinterpret_cast<uint32_t *>(tw1 + tw_smem_entries<LOGN>() / 2) + grp * NB * 2 * xwords<LOGN>();
  load_twiddles<LOGN>(a.tinv, tw1, twl, threadIdx.x, NG * NT);
  const uint32_t p[2] = {P0, P1};

  const int64_t cta = blockIdx.x;
  const int64_t jr = cta / a.n_chunks, chunk = cta % a.n_chunks;  // row-major: CTAs of a row adjacent
  const int64_t j = a.row_begin + jr;
  const int64_t t_begin = chunk * a.tok_per_cta;
  const int64_t t_end = min(a.T, t_begin + a.tok_per_cta);
  const uint4 *wrow = reinterpret_cast<const uint4 *>(a.what + j * a.Lc * 2 * N) + tid;
  const int64_t tok4 = a.Lc * 2 * (N / 4);
  if constexpr (WSM) {  // stage W_hat_j after the exchange buffers
    uint4 *wsm = reinterpret_cast<uint4 *>(xb - grp * NB * 2 * xwords<LOGN>() + NG * NB * 2 * xwords<LOGN>());
    const uint4 *src = reinterpret_cast<const uint4 *>(a.what + j * a.Lc * 2 * N);
    for (int64_t k = threadIdx.x; k < tok4; k += NG * NT) wsm[k] = src[k];
    wrow = wsm + tid;
  }
  const int s_shift = a.q_in - a.out_bits;
  const uint64_t rnd = (SW && s_shift) ? (1ull << (s_shift - 1)) : 0ull;
  const uint32_t omask = (uint32_t)mask_bits(a.out_bits);
  const uint64_t kadd = (uint64_t)a.crt_z0 + (a.par[j] ? (1ull << (a.q_in - 1)) : 0ull) + rnd;
  // A_hat_{tau,0} of the next token is prefetched into registers while this one is transformed
  uint4 an[2][4];
  if (t_begin + grp < t_end) {
    const uint4 *a0 = reinterpret_cast<const uint4 *>(a.ahat) + (t_begin + grp) * tok4 + tid;
#pragma unroll
    for (int q = 0; q < 2; q++)
#pragma unroll
      for (int v = 0; v < 4; v++) an[q][v] = __ldg(a0 + q * (N / 4) + v * NT);
  }
  __syncthreads();

  for (int64_t tau = t_begin + grp; tau < t_end; tau += NG) {
    uint32_t r[2][16];
    // ---- pointwise: sum_i W_hat_ij o A_hat_{tau,i} (N^{-1} folded into W_hat), elements 16 tid..+15
    const uint4 *arow = reinterpret_cast<const uint4 *>(a.ahat) + tau * tok4 + tid;
#pragma unroll
    for (int q = 0; q < 2; q++) {
      const uint32_t pi = q ? PINV1 : PINV0;
#pragma unroll
      for (int v = 0; v < 4; v++) {
        const uint4 wv = WSM ? wrow[q * (N / 4) + v * NT] : __ldg(wrow + q * (N / 4) + v * NT), av = an[q][v];
        r[q][4 * v + 0] = mont_lazy(wv.x, av.x, p[q], pi);
        r[q][4 * v + 1] = mont_lazy(wv.y, av.y, p[q], pi);
        r[q][4 * v + 2] = mont_lazy(wv.z, av.z, p[q], pi);
        r[q][4 * v + 3] = mont_lazy(wv.w, av.w, p[q], pi);
      }
    }
    if (tau + NG < t_end) {
      const uint4 *a0 = arow + NG * tok4;
#pragma unroll
      for (int q = 0; q < 2; q++)
#pragma unroll
        for (int v = 0; v < 4; v++) an[q][v] = __ldg(a0 + q * (N / 4) + v * NT);
    }
    for (int64_t i = 1; i < a.Lc; i++) {
#pragma unroll
      for (int q = 0; q < 2; q++) {
        const uint32_t pi = q ? PINV1 : PINV0;
#pragma unroll
        for (int v = 0; v < 4; v++) {
          const int64_t off = (i * 2 + q) * (N / 4) + v * NT;
          const uint4 wv = WSM ? wrow[off] : __ldg(wrow + off), av = __ldg(arow + off);
          const uint32_t m[4] = {mont_lazy(wv.x, av.x, p[q], pi), mont_lazy(wv.y, av.y, p[q], pi),
                                 mont_lazy(wv.z, av.z, p[q], pi), mont_lazy(wv.w, av.w, p[q], pi)};
#pragma unroll
          for (int k = 0; k < 4; k++) r[q][4 * v + k] = add_lazy(r[q][4 * v + k], m[k], p[q]);
        }
      }
    }
    intt<LOGN, 2, NB, NG>(r, tw1, twl, p, xb, tid, grp);
    // ---- CRT, mod 2^q_in, SampleExtract reversal, ModulusSwitch, store
    const int64_t obase = (DIG ? (tau * a.digit_rows + jr) * KS_LEVELS : tau * a.out_rows + jr) * (int64_t)N + (N - 1);
    const int jt = eidx<LOGN, LastPhase<LOGN>::S0, LastPhase<LOGN>::B>(tid, 0);
#pragma unroll
    for (int e = 0; e < 16; e++)
      crt_store<SW, SHIFT, OUTB, DIG>(a, r[0][e], r[1][e], kadd,
                    obase - jt - eidx<LOGN, LastPhase<LOGN>::S0, LastPhase<LOGN>::B>(0, e), s_shift, omask);
  }
}

template <int LOGN, bool SW, int NG, int NB, bool WSM, int SHIFT = 0, int OUTB = 0, bool DIG = false>
int launch_mask_cfg(MaskArgs a, cudaStream_t st) {
  auto kern = ntt_mask_kernel<LOGN, SW, NG, NB, WSM, SHIFT, OUTB, DIG>;
  const int smem = ntt_smem<LOGN, NG, NB>() + (WSM ? (int)(a.Lc * 2 * (1 << LOGN) * 4) : 0);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return phe_set_cuda_error(e);
#ifndef PHE_KERNEL_EXPERIMENTS
#define PHE_KERNEL_EXPERIMENTS 0
#endif
  // 8 tokens per group (PHE_NTT_TOK overrides it in experiment builds only)
  const char *ev = PHE_KERNEL_EXPERIMENTS ? getenv("PHE_NTT_TOK") : nullptr;
  a.tok_per_cta = ev ? atoi(ev) : 8 * NG;
  if (a.tok_per_cta < 1) a.tok_per_cta = 1;
  a.n_chunks = (a.T + a.tok_per_cta - 1) / a.tok_per_cta;
  kern<<<(unsigned)(a.R * a.n_chunks), NG * (1 << LOGN) / 16, smem, st>>>(a);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

// One token group and one exchange buffer per CTA (smallest shared-memory footprint: 4 CTAs /
// 16 warps per SM at N = 2048).  Measured alternatives (2 groups sharing the twiddles, 2
// alternating buffers) were within 2% on q_proj and slower at L = 4.
// Launch policy: NG token groups per CTA so that a CTA has 16 warps (NG = min(8, 512 / (N/16))), all
// sharing one twiddle copy and (if it fits) the shared-memory copy of W_hat_j; at N = 2048 and
// L <= 2, two CTAs of 2 groups instead (83-99 KB each).  Table 1's switch (39 -> 26) is compiled in.
constexpr int SMEM_BUDGET = 200 * 1024;
template <int LOGN, bool SW, int NG, int NB>
int launch_mask_ng(const MaskArgs &a, cudaStream_t st) {
  const bool t1 = SW && a.q_in == 39 && a.out_bits == 26;
  const bool wsm = ntt_smem<LOGN, NG, NB>() + a.Lc * 2 * (1 << LOGN) * 4 <= SMEM_BUDGET;
  if (a.digit_rows > 0) {  // Decomp digits (out_bits = 32): Table 1 shift 7 compiled in
    if constexpr (SW) {
      const bool d1 = a.q_in == 39;
      if (wsm) return d1 ? launch_mask_cfg<LOGN, true, NG, NB, true, 7, 32, true>(a, st)
                         : launch_mask_cfg<LOGN, true, NG, NB, true, 0, 0, true>(a, st);
      return d1 ? launch_mask_cfg<LOGN, true, NG, NB, false, 7, 32, true>(a, st)
                : launch_mask_cfg<LOGN, true, NG, NB, false, 0, 0, true>(a, st);
    }
    return PHE_EINVAL;
  }
  if (wsm) return t1 ? launch_mask_cfg<LOGN, SW, NG, NB, true, 13, 26>(a, st) : launch_mask_cfg<LOGN, SW, NG, NB, true>(a, st);
  return t1 ? launch_mask_cfg<LOGN, SW, NG, NB, false, 13, 26>(a, st) : launch_mask_cfg<LOGN, SW, NG, NB, false>(a, st);
}
template <int LOGN, bool SW>
int launch_mask(const MaskArgs &a, cudaStream_t st) {
  // <= 8 groups: named barriers 1..NG of the 16 hardware barriers
  constexpr int NGF = 512 / ((1 << LOGN) / 16) < 8 ? 512 / ((1 << LOGN) / 16) : 8;
  if constexpr (LOGN == 11) {
    if (a.Lc <= 2) return launch_mask_ng<LOGN, SW, 2, 1>(a, st);
  }
  return launch_mask_ng<LOGN, SW, NGF, 1>(a, st);
}

}  // namespace ntt

// ---------------------------------------------------------------- launchers (host)
static uint32_t host_psi(uint32_t p, uint32_t g, int N) {
  return ntt::pw(g, (p - 1) / (2 * (uint32_t)N), p);
}

int ntt_primes(uint32_t out[2]) {
  out[0] = ntt::P0;
  out[1] = ntt::P1;
  return PHE_OK;
}

int launch_ntt_tables(const KParams &kp, void *tables, cudaStream_t st) {
  const int N = kp.N;
  ntt::ntt_tables_kernel<<<(4 * N + 2 * 15 * (N / 16) + 255) / 256, 256, 0, st>>>(
      kp.log2N, host_psi(ntt::P0, ntt::GEN0, N), host_psi(ntt::P1, ntt::GEN1, N),
      static_cast<uint2 *>(tables));
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ntt_weights(const KParams &kp, const void *tables, const int8_t *W, int64_t d_out,
                       int64_t d_in, int transpose, uint32_t *what, cudaStream_t st) {
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  const int N = kp.N;
  const int64_t Lc = (cols + N - 1) / N;
  // N^{-1} * 2^32 mod p: Montgomery form with the inverse transform's scaling folded in
  const uint32_t c0 = (uint32_t)((uint64_t)ntt::pw(N, ntt::P0 - 2, ntt::P0) * ((1ull << 32) % ntt::P0) % ntt::P0);
  const uint32_t c1 = (uint32_t)((uint64_t)ntt::pw(N, ntt::P1 - 2, ntt::P1) * ((1ull << 32) % ntt::P1) % ntt::P1);
  const size_t smem = 2 * N * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ntt::ntt_weights_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return phe_set_cuda_error(e);
  }
  ntt::ntt_weights_kernel<<<(unsigned)(rows * Lc), ntt::PREP_THREADS, smem, st>>>(
      kp.log2N, W, d_in, transpose, cols, Lc, static_cast<const uint2 *>(tables), c0, c1, what);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ntt_encrypt(const KParams &kp, const void *tables, const uint8_t *S, const int8_t *x, int64_t T,
                       int64_t d_in, int64_t L, uint64_t seed_base, uint64_t noise_seed, uint64_t *seeds,
                       uint64_t *body, cudaStream_t st) {
  if (T * L == 0) return PHE_OK;
  const int N = kp.N;
  const uint32_t c0 = (uint32_t)((uint64_t)ntt::pw(N, ntt::P0 - 2, ntt::P0) * ((1ull << 32) % ntt::P0) % ntt::P0);
  const uint32_t c1 = (uint32_t)((uint64_t)ntt::pw(N, ntt::P1 - 2, ntt::P1) * ((1ull << 32) % ntt::P1) % ntt::P1);
  const size_t smem = 4 * (size_t)N * sizeof(uint32_t);
  cudaError_t e = cudaFuncSetAttribute(ntt::ntt_encrypt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return phe_set_cuda_error(e);
  ntt::ntt_encrypt_kernel<<<(unsigned)(T * L), ntt::PREP_THREADS, smem, st>>>(
      kp, kp.log2N, S, x, d_in, L, seed_base, noise_seed, static_cast<const uint2 *>(tables), c0, c1, seeds, body);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ntt_rowpar(const int8_t *W, int64_t d_out, int64_t d_in, int transpose, uint8_t *par,
                      cudaStream_t st) {
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  ntt::ntt_rowpar_kernel<<<(unsigned)((rows + 7) / 8), 256, 0, st>>>(W, d_in, transpose, rows, cols, par);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ntt_masks(const KParams &kp, const void *tables, const uint64_t *seeds, int64_t T, int64_t L,
                     uint32_t *ahat, cudaStream_t st) {
  if (T * L == 0) return PHE_OK;
  const size_t smem = 2 * kp.N * sizeof(uint32_t);
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(ntt::ntt_masks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return phe_set_cuda_error(e);
  }
  ntt::ntt_masks_kernel<<<(unsigned)(T * L), ntt::PREP_THREADS, smem, st>>>(
      kp, kp.log2N, seeds, static_cast<const uint2 *>(tables), ahat);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ntt_mask(const KParams &kp, const void *tables, const uint32_t *what, const uint8_t *par,
                    int64_t rows, int64_t Lc, int64_t row_begin, int64_t row_end, const uint32_t *ahat,
                    int64_t T, int out_bits, void *out, cudaStream_t st, int64_t digit_rows, int64_t out_rows) {
  ntt::MaskArgs a{};
  a.out_rows = out_rows > 0 ? out_rows : row_end - row_begin;
  a.par = par;
  a.digit_rows = digit_rows;  // > 0: Decomp digits, out_bits must be 32
  a.plane = kp.N;
  a.tinv = static_cast<const uint2 *>(tables) + 2 * kp.N;  // inverse slice [pr][N]
  a.what = what;
  a.ahat = ahat;
  a.Lc = Lc;
  a.row_begin = row_begin;
  a.R = row_end - row_begin;
  a.T = T;
  a.q_in = kp.q_in;
  a.out_bits = out_bits;
  a.qmask = kp.qmask;
  a.out = out;
  if (a.R == 0 || T == 0) return PHE_OK;
  {  // the CRT offset Z (crt_store): multiple of 2^q_in >= max|P'| + 2 p0
    const unsigned __int128 maxP = (unsigned __int128)Lc * kp.N * ((unsigned __int128)1 << (kp.q_in - 1)) * 128;
    const unsigned __int128 g = (unsigned __int128)1 << kp.q_in;
    const unsigned __int128 Z = (maxP + 2 * (unsigned __int128)ntt::P0 + g - 1) / g * g;
    if (Z + maxP >= (unsigned __int128)ntt::CRT_M) return PHE_EUNSUPPORTED;
    const uint32_t z0 = (uint32_t)(Z % ntt::P0), z1 = (uint32_t)(Z % ntt::P1);
    a.crt_z0 = z0;
    a.crt_k1 = (uint32_t)(((uint64_t)z1 + ntt::P1 - (z0 % ntt::P1)) % ntt::P1 + 2ull * ntt::P1);
  }
  const bool sw = digit_rows > 0 || out_bits != kp.q_in;
  switch (kp.log2N) {
    case 9: return sw ? ntt::launch_mask<9, true>(a, st) : ntt::launch_mask<9, false>(a, st);
    case 10: return sw ? ntt::launch_mask<10, true>(a, st) : ntt::launch_mask<10, false>(a, st);
    case 11: return sw ? ntt::launch_mask<11, true>(a, st) : ntt::launch_mask<11, false>(a, st);
    case 12: return sw ? ntt::launch_mask<12, true>(a, st) : ntt::launch_mask<12, false>(a, st);
    case 13: return sw ? ntt::launch_mask<13, true>(a, st) : ntt::launch_mask<13, false>(a, st);
    default: return PHE_EUNSUPPORTED;
  }
}

}  // namespace phe
