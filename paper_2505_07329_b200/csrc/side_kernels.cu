// side_kernels.cu — HBM/ALU-bound kernels around the limb GEMM:
//   keygen, encrypt_pack (client), weights_prepare (a2), ct_prepare (a3+a4),
//   modswitch (a8 standalone), decrypt_unpack (client), and the SIMT cross-check GEMM.
// Every kernel is plain, coalesced CUDA for sm_100a; grids are sized in multiples of the SM
// count where the work allows (148 SMs).
#include <cstdint>

#include "phe_common.cuh"
#include "side_kernels.cuh"

namespace phe {

// ------------------------------------------------------------------ keygen (R6)
__global__ void keygen_kernel(uint64_t master_seed, int N, uint8_t *__restrict__ S) {
  // one thread per 64-byte keystream block = 512 key bits
  int blk = blockIdx.x * blockDim.x + threadIdx.x;
  if (blk * 512 >= N) return;
  uint32_t o[16];
  chacha20_block(master_seed, (uint32_t)blk, nonce_sk(), o);
  for (int b = 0; b < 512 && blk * 512 + b < N; b++) {
    uint32_t byte = (o[(b >> 3) >> 2] >> (8 * ((b >> 3) & 3))) & 0xffu;
    S[blk * 512 + b] = (uint8_t)((byte >> (b & 7)) & 1u);
  }
}

// ------------------------------------------------------------------ encrypt_pack
// One CTA per block (tau, i).  B = A*S + E + Delta*x_hat mod 2^q_in.
// A*S: negacyclic product with the binary key, computed as sum over key bits S[n] = 1 of
// the shifted mask: (A*S)[k] = sum_{n<=k, S_n} A[k-n] - sum_{n>k, S_n} A[k-n+N].
// The loop over n is warp-uniform (S[n] read from shared memory by all lanes).
constexpr int ENC_THREADS = 256;

__global__ void __launch_bounds__(ENC_THREADS)
encrypt_kernel(KParams kp, const uint8_t *__restrict__ S, const int8_t *__restrict__ x, int64_t T,
               int64_t d_in, int64_t L, uint64_t seed_base, uint64_t noise_seed,
               uint64_t *__restrict__ seeds, uint64_t *__restrict__ body) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int N = kp.N;
  uint64_t *A = reinterpret_cast<uint64_t *>(smem);
  uint8_t *Ss = smem + sizeof(uint64_t) * N;
  const int64_t blk = blockIdx.x;  // tau * L + i
  const int64_t tau = blk / L, i = blk % L;
  const uint64_t seed = seed_base + (uint64_t)blk;
  if (threadIdx.x == 0) seeds[blk] = seed;
  for (int b = threadIdx.x; b < N / 8; b += blockDim.x) {
    uint64_t w[8];
    chacha20_u64x8(seed, (uint32_t)b, nonce_mask(), w);
#pragma unroll
    for (int e = 0; e < 8; e++) A[8 * b + e] = w[e] & kp.qmask;
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) Ss[k] = S[k];
  __syncthreads();

  const uint64_t delta = 1ull << (kp.q_in - kp.beta);
  // thread handles k = threadIdx.x + e * ENC_THREADS; the n-loop is warp-uniform
  for (int k = threadIdx.x; k < N; k += ENC_THREADS) {
    uint64_t acc = 0;
    for (int n = 0; n < N; n++) {
      if (!Ss[n]) continue;  // uniform branch
      int d = k - n;
      uint64_t a = A[d & (N - 1)];
      acc += (d >= 0) ? a : (0ull - a);
    }
    int64_t c = i * (int64_t)N + k;
    int64_t xv = (c < d_in) ? (int64_t)x[tau * d_in + c] : 0;
    int64_t ev = 0;
    if (kp.eta > 0) {
      // one keystream u64 word per coefficient in global order (tau, i, k)  (R5/R6)
      uint64_t widx = (uint64_t)blk * (uint64_t)N + (uint64_t)k;
      uint32_t o[16];
      chacha20_block(noise_seed, (uint32_t)(widx >> 3), nonce_noise(), o);
      int q = (int)(widx & 7);
      uint64_t w = (uint64_t)o[2 * q] | ((uint64_t)o[2 * q + 1] << 32);
      uint64_t m = mask_bits(kp.eta);
      ev = (int64_t)__popcll(w & m) - (int64_t)__popcll((w >> kp.eta) & m);
    }
    uint64_t v = acc + (uint64_t)ev + delta * (uint64_t)xv;
    body[blk * (int64_t)N + k] = v & kp.qmask;
  }
}

// ------------------------------------------------------------------ weights_prepare (a2)
// 16-shift expansion of wext (P:182 absorbed):
//   exp[((j*Lc + i)*2N + m)*16 + b] = wext_{j,i}[m + b]
//   wext_{j,i}[u] = M[j, iN+u] (u < N), -M[j, iN+u-N] (N <= u < 2N), 0 otherwise / beyond cols.
__device__ __forceinline__ int8_t mat_at(const int8_t *__restrict__ W, int64_t d_in, int transpose,
                                         int64_t r, int64_t c) {
  // M = W (transpose = 0) or W^T (transpose = 1); W is [d_out][d_in]
  return transpose ? W[c * d_in + r] : W[r * d_in + c];
}

__global__ void weights_expand_kernel(const int8_t *__restrict__ W, int64_t d_in, int transpose,
                                      int64_t rows, int64_t cols, int N, int64_t Lc,
                                      uint4 *__restrict__ exp16) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // (j, i, m)
  int64_t total = rows * Lc * 2 * N;
  if (idx >= total) return;
  int64_t m = idx % (2 * N);
  int64_t ji = idx / (2 * N);
  int64_t i = ji % Lc, j = ji / Lc;
  uint32_t wd[4];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    uint32_t packed = 0;
#pragma unroll
    for (int bb = 0; bb < 4; bb++) {
      int64_t u = m + 4 * q + bb;
      int v = 0;
      if (u < 2 * N) {
        int64_t c = i * N + (u < N ? u : u - N);
        if (c < cols) {
          int w = mat_at(W, d_in, transpose, j, c);
          v = (u < N) ? w : -w;
        }
      }
      packed |= ((uint32_t)(uint8_t)(int8_t)v) << (8 * bb);
    }
    wd[q] = packed;
  }
  exp16[idx] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
}

// Symmetric int8 weights lie in [-127, 127] (symmetric quantization, zero-point 0;
// encode_weights refuses out-of-range weights).  The one int8 value outside that range,
// -128, has no negation in int8 (the Hankel operand stores -w for the negacyclic wrap), so
// registration refuses it: *flag != 0 iff some byte of W is 0x80.  One grid-stride pass with
// 16-byte loads (bytes before a 16-byte boundary / after the last full vector byte-wise).
__global__ void weights_range_kernel(const int8_t *__restrict__ W, int64_t n, unsigned *__restrict__ flag) {
  const uint8_t *b = reinterpret_cast<const uint8_t *>(W);
  const int64_t head = (int64_t)((16 - (reinterpret_cast<uintptr_t>(b) & 15)) & 15);
  const int64_t h = head < n ? head : n;
  const int64_t nvec = (n - h) / 16;
  const uint4 *v = reinterpret_cast<const uint4 *>(b + h);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned bad = 0;
  for (int64_t k = tid; k < nvec; k += stride) {
    uint4 q = v[k];
    uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int c = 0; c < 4; c++) {
      uint32_t x = w[c] ^ 0x80808080u;  // byte == 0x80  <=>  byte of x == 0
      bad |= (x - 0x01010101u) & ~x & 0x80808080u;
    }
  }
  for (int64_t k = tid; k < h; k += stride) bad |= (b[k] == 0x80u);
  for (int64_t k = h + nvec * 16 + tid; k < n; k += stride) bad |= (b[k] == 0x80u);
  if (__any_sync(0xffffffffu, bad != 0) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

__global__ void weights_plain_kernel(const int8_t *__restrict__ W, int64_t d_in, int transpose,
                                     int64_t rows, int64_t rows_pad, int64_t cols, int64_t K,
                                     int8_t *__restrict__ plain) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows_pad * K) return;
  int64_t j = idx / K, c = idx % K;
  plain[idx] = (j < rows && c < cols) ? mat_at(W, d_in, transpose, j, c) : (int8_t)0;
}

// ------------------------------------------------------------------ ct_prepare (a3 + a4)
// Thread per (tau, i, 8-word group): expand 8 mask words with ChaCha20 (R6), reduce
// mod 2^q_in, split into ell byte planes; same limb split for the 8 body words.
__global__ void ct_prepare_kernel(KParams kp, const uint64_t *__restrict__ seeds,
                                  const uint64_t *__restrict__ body, int64_t T, int64_t L,
                                  uint8_t *__restrict__ mask_planes,
                                  uint8_t *__restrict__ body_planes) {
  const int N = kp.N;
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t groups = (int64_t)N / 8;
  if (idx >= T * L * groups) return;
  int64_t g = idx % groups;
  int64_t blk = idx / groups;  // tau * L + i
  int64_t tau = blk / L, i = blk % L;
  const int64_t K = L * N;
  uint64_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (mask_planes) chacha20_u64x8(seeds[blk], (uint32_t)g, nonce_mask(), w);  // NULL: bodies only
  const uint64_t *bsrc = body + blk * (int64_t)N + 8 * g;
  uint64_t bw[8];
  {
    const ulonglong2 *b2 = reinterpret_cast<const ulonglong2 *>(bsrc);
#pragma unroll
    for (int e = 0; e < 4; e++) {
      ulonglong2 v = b2[e];
      bw[2 * e] = v.x; bw[2 * e + 1] = v.y;
    }
  }
  const int64_t col = i * N + 8 * g;
  for (int l = 0; l < kp.ell; l++) {
    uint64_t pm = 0, pb = 0;
#pragma unroll
    for (int e = 0; e < 8; e++) {
      pm |= (((w[e] & kp.qmask) >> (8 * l)) & 0xffull) << (8 * e);
      pb |= (((bw[e] & kp.qmask) >> (8 * l)) & 0xffull) << (8 * e);
    }
    int64_t row = tau * kp.ell + l;
    if (mask_planes) *reinterpret_cast<uint64_t *>(mask_planes + row * K + col) = pm;
    *reinterpret_cast<uint64_t *>(body_planes + row * K + col) = pb;
  }
}

// ------------------------------------------------------------------ modswitch (a8)
__global__ void modswitch_kernel(const uint64_t *__restrict__ in, uint32_t *__restrict__ out,
                                 int64_t count, int shift, uint32_t omask) {
  int64_t i4 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  const uint64_t half = shift > 0 ? (1ull << (shift - 1)) : 0ull;
  if (i4 + 3 < count) {
    const ulonglong2 *p = reinterpret_cast<const ulonglong2 *>(in + i4);
    ulonglong2 a = __ldcs(p), b = __ldcs(p + 1);
    uint4 r;
    r.x = (uint32_t)((a.x + half) >> shift) & omask;
    r.y = (uint32_t)((a.y + half) >> shift) & omask;
    r.z = (uint32_t)((b.x + half) >> shift) & omask;
    r.w = (uint32_t)((b.y + half) >> shift) & omask;
    __stcs(reinterpret_cast<uint4 *>(out + i4), r);
  } else {
    for (int64_t k = i4; k < count; k++) out[k] = (uint32_t)((in[k] + half) >> shift) & omask;
  }
}

// ------------------------------------------------------------------ decrypt_unpack
// Warp per LWE ciphertext (tau, j): phi = b - <a, S'> mod 2^q, decode.
template <typename Word>
__global__ void decrypt_kernel(KParams kp, const uint8_t *__restrict__ S,
                               const Word *__restrict__ mask, const Word *__restrict__ body,
                               int64_t n_ct, int q_bits, int32_t *__restrict__ y) {
  extern __shared__ uint8_t Ss[];
  const int N = kp.N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) Ss[k] = S[k];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int V = 16 / sizeof(Word);  // words per 16-byte load
  for (int64_t ct = warp; ct < n_ct; ct += nwarps) {
    const Word *a = mask + ct * (int64_t)N;
    uint64_t acc = 0;
    for (int t0 = lane * V; t0 < N; t0 += 32 * V) {
      uint4 raw = __ldcs(reinterpret_cast<const uint4 *>(a + t0));
      const Word *wv = reinterpret_cast<const Word *>(&raw);
#pragma unroll
      for (int e = 0; e < V; e++) acc += Ss[t0 + e] ? (uint64_t)wv[e] : 0ull;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) {
      const uint64_t qm = mask_bits(q_bits);
      uint64_t phi = ((uint64_t)body[ct] - acc) & qm;
      const uint64_t tmask = mask_bits(kp.beta);
      uint64_t m;
      if (q_bits >= kp.beta) {
        // floor((phi + 2^(sh-1)) / 2^sh) = (phi >> sh) + bit (sh-1) of phi: no carry-out
        int sh = q_bits - kp.beta;
        m = sh == 0 ? phi : ((phi >> sh) + ((phi >> (sh - 1)) & 1ull));
        m &= tmask;
      } else {
        m = (phi << (kp.beta - q_bits)) & tmask;
      }
      int64_t c = (m >= (1ull << (kp.beta - 1))) ? (int64_t)m - (int64_t)(1ull << kp.beta) : (int64_t)m;
      y[ct] = (int32_t)c;
    }
  }
}

// ------------------------------------------------------------------ SIMT cross-check GEMM
// Reference CUDA-core implementation (64-bit MACs, no limbs in the arithmetic): one CTA per
// (tau, j); threads stride over t.  Reads the same limb-plane operand as the tensor-core
// path and reconstructs each mask word from its limbs.  Test infrastructure on the device.
__device__ __forceinline__ uint64_t limb_word(const uint8_t *__restrict__ planes, int64_t K,
                                              int64_t tau, int ell, int64_t col) {
  uint64_t v = 0;
  for (int l = 0; l < ell; l++) v |= (uint64_t)planes[(tau * ell + l) * K + col] << (8 * l);
  return v;
}

__global__ void simt_matmul_kernel(KParams kp, const int8_t *__restrict__ W, int64_t d_in,
                                   int64_t row_begin, int64_t R, const uint8_t *__restrict__ mplanes,
                                   const uint8_t *__restrict__ bplanes, int64_t L, int out_bits,
                                   void *__restrict__ out_mask, void *__restrict__ out_body) {
  const int N = kp.N;
  const int64_t tau = blockIdx.x / R, jr = blockIdx.x % R, j = row_begin + jr;
  const int64_t K = L * N;
  const int8_t *w = W + j * d_in;
  const int shift = kp.q_in - out_bits;
  const uint64_t half = shift > 0 ? (1ull << (shift - 1)) : 0ull;
  for (int t = threadIdx.x; t < N; t += blockDim.x) {
    uint64_t acc = 0;
    for (int64_t c = 0; c < d_in; c++) {
      int64_t i = c / N, m = c % N;
      int64_t wv = w[c];
      if (wv == 0) continue;
      uint64_t a = (m >= t) ? limb_word(mplanes, K, tau, kp.ell, i * N + (m - t))
                            : (0ull - limb_word(mplanes, K, tau, kp.ell, i * N + (m - t + N)));
      acc += (uint64_t)wv * a;
    }
    acc &= kp.qmask;
    int64_t o = (tau * R + jr) * N + t;
    if (shift == 0) static_cast<uint64_t *>(out_mask)[o] = acc;
    else static_cast<uint32_t *>(out_mask)[o] = (uint32_t)(((acc + half) >> shift) & mask_bits(out_bits));
  }
  if (threadIdx.x == 0) {
    uint64_t acc = 0;
    for (int64_t c = 0; c < d_in; c++)
      acc += (uint64_t)(int64_t)w[c] * limb_word(bplanes, K, tau, kp.ell, c);
    acc &= kp.qmask;
    int64_t o = tau * R + jr;
    if (shift == 0) static_cast<uint64_t *>(out_body)[o] = acc;
    else static_cast<uint32_t *>(out_body)[o] = (uint32_t)(((acc + half) >> shift) & mask_bits(out_bits));
  }
}

// ------------------------------------------------------------------ launchers
int launch_keygen(const KParams &kp, uint64_t seed, uint8_t *S, cudaStream_t st) {
  int nb = (kp.N + 511) / 512;
  keygen_kernel<<<1, nb, 0, st>>>(seed, kp.N, S);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_encrypt(const KParams &kp, const uint8_t *S, const int8_t *x, int64_t T, int64_t d_in,
                   int64_t L, uint64_t seed_base, uint64_t noise_seed, uint64_t *seeds,
                   uint64_t *body, cudaStream_t st) {
  if (T == 0) return PHE_OK;
  size_t smem = sizeof(uint64_t) * kp.N + kp.N;
  static thread_local uint64_t configured = 0;  // per device (a per-device attribute)
  if (!(configured & phe_device_bit())) {
    cudaFuncSetAttribute(encrypt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured |= phe_device_bit();
  }
  encrypt_kernel<<<(unsigned)(T * L), ENC_THREADS, smem, st>>>(kp, S, x, T, d_in, L, seed_base,
                                                              noise_seed, seeds, body);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_weights_prepare(const KParams &kp, const int8_t *W, int64_t d_out, int64_t d_in,
                           int transpose, void *wprep, cudaStream_t st) {
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  const int N = kp.N;
  const int64_t Lc = (cols + N - 1) / N;
  uint8_t *base = static_cast<uint8_t *>(wprep);
  int64_t n_exp = rows * Lc * 2 * N;
  weights_expand_kernel<<<(unsigned)((n_exp + 255) / 256), 256, 0, st>>>(
      W, d_in, transpose, rows, cols, N, Lc, reinterpret_cast<uint4 *>(base));
  PHE_CUDA_CHECK_LAUNCH();
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  int64_t n_plain = rows_pad * Lc * N;
  weights_plain_kernel<<<(unsigned)((n_plain + 255) / 256), 256, 0, st>>>(
      W, d_in, transpose, rows, rows_pad, cols, Lc * N, reinterpret_cast<int8_t *>(base + n_exp * 16));
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

// Device-side check of the symmetric weight range (see weights_range_kernel); synchronises `st`
// (registration is a once-per-model call).  flag: 4 bytes of device scratch (the caller's output
// buffer, overwritten afterwards).  PHE_OK, PHE_ERANGE (some w == -128) or PHE_ECUDA.
int check_weights_range(const int8_t *W, int64_t n, unsigned *flag, cudaStream_t st) {
  if (cudaMemsetAsync(flag, 0, sizeof(unsigned), st) != cudaSuccess) return phe_set_cuda_error(cudaGetLastError());
  int64_t blocks = (n / 16 + 255) / 256;
  blocks = blocks < 1 ? 1 : (blocks > 148 * 8 ? 148 * 8 : blocks);
  weights_range_kernel<<<(unsigned)blocks, 256, 0, st>>>(W, n, flag);
  PHE_CUDA_CHECK_LAUNCH();
  unsigned h = 0;
  cudaError_t e = cudaMemcpyAsync(&h, flag, sizeof(unsigned), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return phe_set_cuda_error(e);
  return h ? PHE_ERANGE : PHE_OK;
}

int launch_weights_plain(const KParams &kp, const int8_t *W, int64_t d_out, int64_t d_in, int transpose,
                         int8_t *plain, cudaStream_t st) {
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  const int64_t K = (cols + kp.N - 1) / kp.N * kp.N;
  const int64_t rows_pad = (rows + 127) / 128 * 128;
  const int64_t n = rows_pad * K;
  weights_plain_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(W, d_in, transpose, rows, rows_pad,
                                                                    cols, K, plain);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ct_prepare(const KParams &kp, const uint64_t *seeds, const uint64_t *body, int64_t T,
                      int64_t L, uint8_t *mask_planes, uint8_t *body_planes, cudaStream_t st) {
  int64_t n = T * L * (kp.N / 8);
  if (n == 0) return PHE_OK;
  ct_prepare_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(kp, seeds, body, T, L,
                                                                 mask_planes, body_planes);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_modswitch(const uint64_t *in, uint32_t *out, int64_t count, int from, int to,
                     cudaStream_t st) {
  if (count == 0) return PHE_OK;
  int64_t threads = (count + 3) / 4;
  modswitch_kernel<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(
      in, out, count, from - to, (uint32_t)mask_bits(to));
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_decrypt(const KParams &kp, const uint8_t *S, const void *mask, const void *body,
                   int64_t n_ct, int q_bits, bool u64words, int32_t *y, cudaStream_t st) {
  if (n_ct == 0) return PHE_OK;
  int64_t warps = n_ct;
  int64_t blocks = (warps * 32 + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (u64words)
    decrypt_kernel<uint64_t><<<(unsigned)blocks, 256, kp.N, st>>>(
        kp, S, (const uint64_t *)mask, (const uint64_t *)body, n_ct, q_bits, y);
  else
    decrypt_kernel<uint32_t><<<(unsigned)blocks, 256, kp.N, st>>>(
        kp, S, (const uint32_t *)mask, (const uint32_t *)body, n_ct, q_bits, y);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_simt_matmul(const KParams &kp, const int8_t *W, int64_t d_in, int64_t row_begin,
                       int64_t R, const uint8_t *mplanes, const uint8_t *bplanes, int64_t L,
                       int64_t T, int out_bits, void *out_mask, void *out_body, cudaStream_t st) {
  if (T == 0 || R == 0) return PHE_OK;
  simt_matmul_kernel<<<(unsigned)(T * R), 256, 0, st>>>(kp, W, d_in, row_begin, R, mplanes,
                                                        bplanes, L, out_bits, out_mask, out_body);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

// ================================================================== NEXT #1: KeySwitch packing
// KSK generation (client): row r = l*N + i is RLWE_S(S'_i * 2^(q - (l+1)*8)):
// A_r = ChaCha20 words (nonce "phe-ksk") r*N + k, B_r = A_r*S + E_r + S'_i 2^(q-(l+1)8) X^0.
__global__ void __launch_bounds__(ENC_THREADS)
ksk_gen_kernel(KParams kp, const uint8_t *__restrict__ S, uint64_t seed, uint64_t *__restrict__ KA,
               uint64_t *__restrict__ KB) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int N = kp.N;
  uint64_t *A = reinterpret_cast<uint64_t *>(smem);
  uint8_t *Ss = smem + sizeof(uint64_t) * N;
  const int64_t r = blockIdx.x;
  const int l = (int)(r / N), i = (int)(r % N);
  for (int b = threadIdx.x; b < N / 8; b += blockDim.x) {
    uint64_t w[8];
    chacha20_u64x8(seed, (uint32_t)(r * (N / 8) + b), nonce_ksk(), w);
#pragma unroll
    for (int e = 0; e < 8; e++) A[8 * b + e] = w[e] & kp.qmask;
  }
  for (int k = threadIdx.x; k < N; k += blockDim.x) Ss[k] = S[k];
  __syncthreads();
  for (int k = threadIdx.x; k < N; k += ENC_THREADS) {
    uint64_t acc = 0;
    for (int n = 0; n < N; n++) {
      if (!Ss[n]) continue;
      int d = k - n;
      uint64_t a = A[d & (N - 1)];
      acc += (d >= 0) ? a : (0ull - a);
    }
    if (kp.eta > 0) {
      uint64_t widx = (uint64_t)r * (uint64_t)N + (uint64_t)k;
      uint32_t o[16];
      chacha20_block(seed, (uint32_t)(widx >> 3), nonce_ksk_noise(), o);
      int q = (int)(widx & 7);
      uint64_t w = (uint64_t)o[2 * q] | ((uint64_t)o[2 * q + 1] << 32);
      uint64_t m = mask_bits(kp.eta);
      acc += (uint64_t)((int64_t)__popcll(w & m) - (int64_t)__popcll((w >> kp.eta) & m));
    }
    if (k == 0) acc += (uint64_t)Ss[i] << (kp.q_in - (l + 1) * KS_BASE_LOG);
    KA[r * N + k] = A[k];
    KB[r * N + k] = acc & kp.qmask;
  }
}

// KSK registration (server): limb planes of the packing GEMM's B operand.  Plane row
// slot*ell + l (slot = part*kpad + k, k < N; zero for padding), column c = l'*N + i holds
// byte l of KSK_part[c][k].  32x32 transpose tiles through shared memory.
__global__ void ksk_planes_kernel(const uint64_t *__restrict__ ksk, int N, int ell, int kpad,
                                  int64_t rows, uint8_t *__restrict__ planes) {
  __shared__ uint64_t tile[32][33];
  const int64_t K3 = KS_LEVELS * (int64_t)N;
  const int part = blockIdx.z;
  const int64_t c0 = (int64_t)blockIdx.y * 32, k0 = (int64_t)blockIdx.x * 32;
  const uint64_t *src = ksk + (int64_t)part * K3 * N;
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t c = c0 + y, k = k0 + threadIdx.x;
    tile[y][threadIdx.x] = (c < K3 && k < N) ? src[c * N + k] : 0ull;
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += blockDim.y) {
    const int64_t k = k0 + y, c = c0 + threadIdx.x;
    if (k >= kpad || c >= K3) continue;
    const uint64_t v = tile[threadIdx.x][y];
    const int64_t slot = (int64_t)part * kpad + k;
    for (int l = 0; l < ell; l++) planes[(slot * ell + l) * K3 + c] = (uint8_t)(v >> (8 * l));
  }
}

// Finalize (Eq. 7/8): A = -acc_A, B = b_j - acc_B at coefficient p = j mod N of group j / N,
// reduce mod 2^q_in, ModulusSwitch to q_out.  out: uint32 [T][G][2][N].
__global__ void pack_finalize_kernel(KParams kp, const unsigned long long *__restrict__ acc,
                                     const uint64_t *__restrict__ body, int64_t T, int64_t R, int G,
                                     uint32_t *__restrict__ out) {
  const int N = kp.N;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= T * G * N) return;
  const int p = (int)(idx % N);
  const int64_t tg = idx / N;
  const int g = (int)(tg % G);
  const int64_t tau = tg / G;
  const int64_t j = (int64_t)g * N + p;
  const uint64_t a = (0ull - acc[(tg * 2 + 0) * N + p]) & kp.qmask;
  const uint64_t b = ((j < R ? body[tau * R + j] : 0ull) - acc[(tg * 2 + 1) * N + p]) & kp.qmask;
  const int s = kp.q_in - kp.q_out;
  const uint64_t half = s > 0 ? (1ull << (s - 1)) : 0ull, om = mask_bits(kp.q_out);
  out[(tg * 2 + 0) * N + p] = (uint32_t)(((a + half) >> s) & om);
  out[(tg * 2 + 1) * N + p] = (uint32_t)(((b + half) >> s) & om);
}

// Decryption of packed RLWE outputs (client): phase = B - A*S, decode per coefficient.
__global__ void __launch_bounds__(ENC_THREADS)
decrypt_packed_kernel(KParams kp, const uint8_t *__restrict__ S, const uint32_t *__restrict__ packed,
                      int64_t R, int G, int q_bits, int32_t *__restrict__ y) {
  extern __shared__ __align__(16) uint8_t smem[];
  const int N = kp.N;
  uint32_t *A = reinterpret_cast<uint32_t *>(smem);
  uint8_t *Ss = smem + sizeof(uint32_t) * N;
  const int64_t tg = blockIdx.x;  // tau * G + g
  const int g = (int)(tg % G);
  const int64_t tau = tg / G;
  const uint32_t *pa = packed + tg * 2 * N, *pb = pa + N;
  for (int k = threadIdx.x; k < N; k += blockDim.x) { A[k] = pa[k]; Ss[k] = S[k]; }
  __syncthreads();
  const uint64_t qm = mask_bits(q_bits), tmask = mask_bits(kp.beta);
  for (int k = threadIdx.x; k < N; k += ENC_THREADS) {
    const int64_t j = (int64_t)g * N + k;
    if (j >= R) continue;
    uint64_t acc = 0;
    for (int n = 0; n < N; n++) {
      if (!Ss[n]) continue;
      int d = k - n;
      uint64_t a = A[d & (N - 1)];
      acc += (d >= 0) ? a : (0ull - a);
    }
    const uint64_t phi = ((uint64_t)pb[k] - acc) & qm;
    uint64_t m;
    if (q_bits >= kp.beta) {
      int sh = q_bits - kp.beta;
      m = sh == 0 ? phi : ((phi >> sh) + ((phi >> (sh - 1)) & 1ull));
      m &= tmask;
    } else {
      m = (phi << (kp.beta - q_bits)) & tmask;
    }
    y[tau * R + j] = (int32_t)((m >= (1ull << (kp.beta - 1))) ? (int64_t)m - (int64_t)(1ull << kp.beta) : (int64_t)m);
  }
}

int launch_ksk_gen(const KParams &kp, const uint8_t *S, uint64_t seed, uint64_t *KA, uint64_t *KB,
                   cudaStream_t st) {
  size_t smem = sizeof(uint64_t) * kp.N + kp.N;
  static thread_local uint64_t configured = 0;  // per device (a per-device attribute)
  if (!(configured & phe_device_bit())) {
    cudaFuncSetAttribute(ksk_gen_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    configured |= phe_device_bit();
  }
  ksk_gen_kernel<<<(unsigned)(KS_LEVELS * kp.N), ENC_THREADS, smem, st>>>(kp, S, seed, KA, KB);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_ksk_planes(const KParams &kp, const uint64_t *ksk, int kpad, int64_t rows, uint8_t *planes,
                      cudaStream_t st) {
  if (cudaMemsetAsync(planes, 0, (size_t)rows * KS_LEVELS * kp.N, st) != cudaSuccess)
    return phe_set_cuda_error(cudaGetLastError());
  dim3 grid((unsigned)((kpad + 31) / 32), (unsigned)((KS_LEVELS * kp.N + 31) / 32), 2);
  ksk_planes_kernel<<<grid, dim3(32, 8), 0, st>>>(ksk, kp.N, kp.ell, kpad, rows, planes);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_pack_finalize(const KParams &kp, const void *acc, const uint64_t *body, int64_t T, int64_t R,
                         int G, uint32_t *out, cudaStream_t st) {
  int64_t n = T * G * kp.N;
  if (n == 0) return PHE_OK;
  pack_finalize_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      kp, static_cast<const unsigned long long *>(acc), body, T, R, G, out);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_decrypt_packed(const KParams &kp, const uint8_t *S, const uint32_t *packed, int64_t T, int64_t R,
                          int G, int q_bits, int32_t *y, cudaStream_t st) {
  if (T * G == 0) return PHE_OK;
  size_t smem = sizeof(uint32_t) * kp.N + kp.N;
  decrypt_packed_kernel<<<(unsigned)(T * G), ENC_THREADS, smem, st>>>(kp, S, packed, R, G, q_bits, y);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

// ================================================================== NEXT #2: wire format
// Little-endian contiguous bitstream (R22).  Every segment (input block: LE64 seed, then
// N coefficients at q_in bits; packed ciphertext: 2N coefficients at q_out bits) is a whole
// number of 64-bit words (N % 64 == 0) and starts 8-byte aligned, so the stream is handled as
// aligned uint64 words: serialize = one thread per stream word, gathering the <= 4 coefficients
// that overlap it; deserialize = one thread per coefficient, reading the <= 2 words that cover
// it.  Both directions are fully coalesced.  bits <= 57.
template <typename WordT>
__device__ __forceinline__ uint64_t gather_word(const WordT *vals, int nvals, int bits, int w) {
  const uint64_t m = mask_bits(bits);
  const int b0 = 64 * w;  // in-segment bit offsets fit 32 bits (N <= 16384, bits <= 57)
  uint64_t out = 0;
#pragma unroll 4
  for (int k = b0 / bits; k < nvals && k * bits < b0 + 64; k++) {
    const int sh = k * bits - b0;  // in (-bits, 64)
    const uint64_t v = (uint64_t)vals[k] & m;
    out |= sh >= 0 ? (v << sh) : (v >> (-sh));
  }
  return out;
}
__device__ __forceinline__ uint64_t extract_bits(const uint64_t *words, int k, int bits) {
  const int b = k * bits;
  const int w = b >> 6, r = b & 63;
  uint64_t v = words[w] >> r;
  if (r + bits > 64) v |= words[w + 1] << (64 - r);
  return v & mask_bits(bits);
}

// 2-D grids: y = segment (grid-strided), x = stream word (serialize) or coefficient (deserialize)
// inputs: block (tau, i) -> [LE64 seed][N coefficients at q_in bits], as 1 + N q/64 words
__global__ void wire_inputs_kernel(int N, int q, uint64_t *__restrict__ seeds, uint64_t *__restrict__ body,
                                   int64_t nblk, uint64_t *__restrict__ wire, int dir) {
  const int nw = N * q / 64;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t blk = blockIdx.y; blk < nblk; blk += gridDim.y) {
    uint64_t *wb = wire + blk * (1 + nw);
    if (dir == 0) {
      if (x <= nw) wb[x] = x == 0 ? seeds[blk] : gather_word<uint64_t>(body + blk * N, N, q, x - 1);
    } else {  // 4 coefficients per thread (16-byte stores)
      if (4 * x < N) {
        ulonglong2 *dst = reinterpret_cast<ulonglong2 *>(body + blk * N + 4 * x);
        dst[0] = make_ulonglong2(extract_bits(wb + 1, 4 * x, q), extract_bits(wb + 1, 4 * x + 1, q));
        dst[1] = make_ulonglong2(extract_bits(wb + 1, 4 * x + 2, q), extract_bits(wb + 1, 4 * x + 3, q));
      } else if (4 * x == N) {
        seeds[blk] = wb[0];
      }
    }
  }
}

// packed outputs: ciphertext (tau, g) -> [A' at q_out bits][B' at q_out bits], 2N q/64 words
__global__ void wire_packed_kernel(int N, int q, uint32_t *__restrict__ packed, int64_t nct,
                                   uint64_t *__restrict__ wire, int dir) {
  const int nw = 2 * N * q / 64;
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t ct = blockIdx.y; ct < nct; ct += gridDim.y) {
    if (dir == 0) {
      if (x < nw) wire[ct * nw + x] = gather_word<uint32_t>(packed + ct * 2 * N, 2 * N, q, x);
    } else {  // 4 coefficients per thread (16-byte stores)
      if (4 * x < 2 * N) {
        const uint64_t *wc = wire + ct * nw;
        *reinterpret_cast<uint4 *>(packed + ct * 2 * N + 4 * x) =
            make_uint4((uint32_t)extract_bits(wc, 4 * x, q), (uint32_t)extract_bits(wc, 4 * x + 1, q),
                       (uint32_t)extract_bits(wc, 4 * x + 2, q), (uint32_t)extract_bits(wc, 4 * x + 3, q));
      }
    }
  }
}

// Generic u32 segments at `bits` bits (LWE outputs at q_out bits): segment s = (group g, index j)
// with g = s / per_group, j = s % per_group starts at word g * group_words + off_words +
// j * seg_words (seg_words = ceil(seglen bits / 64); the tail of the last word is zero).
__global__ void wire_u32_kernel(uint32_t *__restrict__ vals, int64_t nseg, int seglen, int bits,
                                uint64_t *__restrict__ wire, int64_t seg_words, int64_t per_group,
                                int64_t group_words, int64_t off_words, int dir) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  for (int64_t sg = blockIdx.y; sg < nseg; sg += gridDim.y) {
    uint64_t *ws = wire + (sg / per_group) * group_words + off_words + (sg % per_group) * seg_words;
    uint32_t *vs = vals + sg * seglen;
    if (dir == 0) {
      if (x < seg_words) ws[x] = gather_word<uint32_t>(vs, seglen, bits, x);
    } else {
      if (x < seglen) vs[x] = (uint32_t)extract_bits(ws, x, bits);
    }
  }
}

// Staged variants (one CTA per segment, grid-strided; segments up to 48 KB): the segment is first
// copied to shared memory by every thread at once (16-byte loads of the values / 8-byte loads of
// the stream words), so each thread has several independent loads in flight instead of a chain of
// 2-4 overlapping ones; the gather / extract then reads shared memory.  Same words as above.
constexpr int WIRE_THREADS = 256;
constexpr int WIRE_SMEM_MAX = 48 * 1024;
// BITS > 0: the coefficient width as a compile-time constant (Table 1's 39 and 26: the word ->
// coefficient divisions become multiplies); 0: runtime `bits`.
template <typename WordT, int BITS>
__global__ void __launch_bounds__(WIRE_THREADS)
wire_ser_staged_kernel(const WordT *__restrict__ vals, int nvals, int bits_rt, int64_t nseg,
                       const uint64_t *__restrict__ head, uint64_t *__restrict__ wire) {
  const int bits = BITS > 0 ? BITS : bits_rt;
  extern __shared__ __align__(16) uint8_t wsm[];
  WordT *sv = reinterpret_cast<WordT *>(wsm);
  const int hw = head != nullptr, nw = (int)(((int64_t)nvals * bits + 63) / 64);
  const int n16 = nvals * (int)sizeof(WordT) / 16;
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const uint4 *src = reinterpret_cast<const uint4 *>(vals + sg * nvals);
#pragma unroll 4
    for (int i = threadIdx.x; i < n16; i += WIRE_THREADS) reinterpret_cast<uint4 *>(sv)[i] = __ldcs(src + i);
    __syncthreads();
    uint64_t *out = wire + sg * (hw + nw);
    if (hw && threadIdx.x == 0) out[0] = head[sg];
    for (int w = threadIdx.x; w < nw; w += WIRE_THREADS) out[hw + w] = gather_word<WordT>(sv, nvals, bits, w);
    __syncthreads();
  }
}
template <typename WordT, int BITS>
__global__ void __launch_bounds__(WIRE_THREADS)
wire_de_staged_kernel(WordT *__restrict__ vals, int nvals, int bits_rt, int64_t nseg, uint64_t *__restrict__ head,
                      const uint64_t *__restrict__ wire) {
  const int bits = BITS > 0 ? BITS : bits_rt;
  extern __shared__ __align__(16) uint8_t wsm[];
  uint64_t *sw = reinterpret_cast<uint64_t *>(wsm);
  const int hw = head != nullptr, nw = (int)(((int64_t)nvals * bits + 63) / 64);
  for (int64_t sg = blockIdx.x; sg < nseg; sg += gridDim.x) {
    const uint64_t *src = wire + sg * (hw + nw);
#pragma unroll 4
    for (int i = threadIdx.x; i < nw; i += WIRE_THREADS) sw[i] = __ldcs(src + hw + i);
    if (hw && threadIdx.x == 0) head[sg] = src[0];
    __syncthreads();
    WordT *dst = vals + sg * nvals;
    for (int k = 4 * threadIdx.x; k < nvals; k += 4 * WIRE_THREADS) {
      if constexpr (sizeof(WordT) == 8) {
        ulonglong2 *d2 = reinterpret_cast<ulonglong2 *>(dst + k);
        d2[0] = make_ulonglong2(extract_bits(sw, k, bits), extract_bits(sw, k + 1, bits));
        d2[1] = make_ulonglong2(extract_bits(sw, k + 2, bits), extract_bits(sw, k + 3, bits));
      } else {
        *reinterpret_cast<uint4 *>(dst + k) =
            make_uint4((uint32_t)extract_bits(sw, k, bits), (uint32_t)extract_bits(sw, k + 1, bits),
                       (uint32_t)extract_bits(sw, k + 2, bits), (uint32_t)extract_bits(sw, k + 3, bits));
      }
    }
    __syncthreads();
  }
}
// grid: 8 resident 256-thread CTAs per SM x 148 SMs, grid-strided over the segments
template <typename WordT>
static int launch_wire_staged(WordT *vals, int nvals, int bits, int64_t nseg, uint64_t *head, uint64_t *wire,
                              int dir, cudaStream_t st) {
  const int64_t nw = ((int64_t)nvals * bits + 63) / 64;
  const size_t smem = dir == 0 ? (size_t)nvals * sizeof(WordT) : (size_t)nw * 8;
  const unsigned grid = (unsigned)(nseg < 148 * 8 ? nseg : 148 * 8);
#define PHE_WIRE_LAUNCH(B)                                                                             \
  do {                                                                                                 \
    if (dir == 0)                                                                                      \
      wire_ser_staged_kernel<WordT, B><<<grid, WIRE_THREADS, smem, st>>>(vals, nvals, bits, nseg, head, wire); \
    else                                                                                               \
      wire_de_staged_kernel<WordT, B><<<grid, WIRE_THREADS, smem, st>>>(vals, nvals, bits, nseg, head, wire);  \
  } while (0)
  if (bits == 39) PHE_WIRE_LAUNCH(39);
  else if (bits == 26) PHE_WIRE_LAUNCH(26);
  else PHE_WIRE_LAUNCH(0);
#undef PHE_WIRE_LAUNCH
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_wire_u32(uint32_t *vals, int64_t nseg, int seglen, int bits, uint8_t *wire, int64_t seg_words,
                    int64_t per_group, int64_t group_words, int64_t off_words, int dir, cudaStream_t st) {
  if (nseg == 0) return PHE_OK;
  const int64_t nx = dir == 0 ? seg_words : seglen;
  const dim3 grid((unsigned)((nx + 255) / 256), (unsigned)(nseg < 65535 ? nseg : 65535));
  wire_u32_kernel<<<grid, 256, 0, st>>>(vals, nseg, seglen, bits, reinterpret_cast<uint64_t *>(wire), seg_words,
                                        per_group, group_words, off_words, dir);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_wire_inputs(const KParams &kp, uint64_t *seeds, uint64_t *body, int64_t nblk, uint8_t *wire,
                       int dir, cudaStream_t st) {
  if (nblk == 0) return PHE_OK;
  if ((size_t)kp.N * 8 <= WIRE_SMEM_MAX)
    return launch_wire_staged<uint64_t>(body, kp.N, kp.q_in, nblk, seeds, reinterpret_cast<uint64_t *>(wire), dir, st);
  const int nx = dir == 0 ? 1 + kp.N * kp.q_in / 64 : kp.N / 4 + 1;
  const dim3 grid((unsigned)((nx + 255) / 256), (unsigned)(nblk < 65535 ? nblk : 65535));
  wire_inputs_kernel<<<grid, 256, 0, st>>>(kp.N, kp.q_in, seeds, body, nblk, reinterpret_cast<uint64_t *>(wire), dir);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

int launch_wire_packed(const KParams &kp, uint32_t *packed, int64_t nct, uint8_t *wire, int dir, cudaStream_t st) {
  if (nct == 0) return PHE_OK;
  if ((size_t)2 * kp.N * 4 <= WIRE_SMEM_MAX)
    return launch_wire_staged<uint32_t>(packed, 2 * kp.N, kp.q_out, nct, nullptr, reinterpret_cast<uint64_t *>(wire), dir, st);
  const int nx = dir == 0 ? 2 * kp.N * kp.q_out / 64 : 2 * kp.N / 4;
  const dim3 grid((unsigned)((nx + 255) / 256), (unsigned)(nct < 65535 ? nct : 65535));
  wire_packed_kernel<<<grid, 256, 0, st>>>(kp.N, kp.q_out, packed, nct, reinterpret_cast<uint64_t *>(wire), dir);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

}  // namespace phe
