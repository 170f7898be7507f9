// phe_common.cuh — device helpers shared by the product kernels (NOT by the oracle).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/phe.h"

namespace phe {

// Runtime copy of the parameters used by kernels (validated on the host first).
struct KParams {
  int N;          // ring degree
  int log2N;
  int q_in, q_out, beta, eta;
  int ell;        // limbs per word = ceil(q_in/8)
  uint64_t qmask; // 2^q_in - 1
};

__host__ __device__ inline uint64_t mask_bits(int bits) {
  return bits >= 64 ? ~0ull : ((1ull << bits) - 1ull);
}

// ---------------------------------------------------------------------------------------
// ChaCha20 block function (RFC 8439 §2.3), the PRNG the parties agree on (DESIGN R6).
// key = LE64(seed) || 0^24; the nonce is one of three 12-byte domain constants.
// ---------------------------------------------------------------------------------------
struct Nonce { uint32_t w0, w1, w2; };
// R6 nonces as little-endian words: 0^12, "phe-sk"\0.., "phe-noise"\0..
__host__ __device__ constexpr Nonce nonce_mask() { return {0u, 0u, 0u}; }
__host__ __device__ constexpr Nonce nonce_sk() { return {0x2d656870u, 0x00006b73u, 0u}; }
__host__ __device__ constexpr Nonce nonce_noise() { return {0x2d656870u, 0x73696f6eu, 0x00000065u}; }
// NEXT #1 (R18-R20): "phe-ksk" (KSK masks), "phe-ksknoise" (KSK noise)
__host__ __device__ constexpr Nonce nonce_ksk() { return {0x2d656870u, 0x006b736bu, 0u}; }
__host__ __device__ constexpr Nonce nonce_ksk_noise() { return {0x2d656870u, 0x6e6b736bu, 0x6573696fu}; }

// KeySwitch gadget (Decomp) parameters: base 2^8, 4 levels = top 32 bits (R18: P:396's
// Fig. 4 claim, < 1% error at bit positions >= 12, needs the 4th level; 3 levels fail it)
constexpr int KS_BASE_LOG = 8;
constexpr int KS_LEVELS = 4;
constexpr int KS_BITS = KS_BASE_LOG * KS_LEVELS;  // 32

__device__ __forceinline__ uint32_t rotl(uint32_t v, int c) { return __funnelshift_l(v, v, c); }

#define PHE_QR(a, b, c, d)                       \
  a += b; d ^= a; d = rotl(d, 16);               \
  c += d; b ^= c; b = rotl(b, 12);               \
  a += b; d ^= a; d = rotl(d, 8);                \
  c += d; b ^= c; b = rotl(b, 7);

// Writes the 16 little-endian keystream words of block `counter`.
__device__ __forceinline__ void chacha20_block(uint64_t seed, uint32_t counter, Nonce n,
                                               uint32_t out[16]) {
  uint32_t s[16];
  s[0] = 0x61707865u; s[1] = 0x3320646eu; s[2] = 0x79622d32u; s[3] = 0x6b206574u;
  s[4] = (uint32_t)seed; s[5] = (uint32_t)(seed >> 32);
  s[6] = s[7] = s[8] = s[9] = s[10] = s[11] = 0u;
  s[12] = counter; s[13] = n.w0; s[14] = n.w1; s[15] = n.w2;
  uint32_t x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = s[i];
#pragma unroll
  for (int r = 0; r < 10; r++) {
    PHE_QR(x[0], x[4], x[8], x[12]) PHE_QR(x[1], x[5], x[9], x[13])
    PHE_QR(x[2], x[6], x[10], x[14]) PHE_QR(x[3], x[7], x[11], x[15])
    PHE_QR(x[0], x[5], x[10], x[15]) PHE_QR(x[1], x[6], x[11], x[12])
    PHE_QR(x[2], x[7], x[8], x[13]) PHE_QR(x[3], x[4], x[9], x[14])
  }
#pragma unroll
  for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}
#undef PHE_QR

// The 8 consecutive u64 words [8*blk, 8*blk+8) of the keystream.
__device__ __forceinline__ void chacha20_u64x8(uint64_t seed, uint32_t blk, Nonce n,
                                               uint64_t w[8]) {
  uint32_t o[16];
  chacha20_block(seed, blk, n, o);
#pragma unroll
  for (int i = 0; i < 8; i++) w[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
}

}  // namespace phe

// thread-local error plumbing (phe_api.cu)
int phe_set_cuda_error(cudaError_t e);
// Bit of the calling thread's current device, for "once per device" caches of per-device
// settings (cudaFuncSetAttribute is a per-device property: a per-thread flag alone would skip it
// when one thread drives a second GPU).
inline uint64_t phe_device_bit() {
  int dev = 0;
  cudaGetDevice(&dev);
  return 1ull << (dev & 63);
}

#define PHE_CUDA_CHECK_LAUNCH()                                   \
  do {                                                            \
    cudaError_t e__ = cudaGetLastError();                         \
    if (e__ != cudaSuccess) return phe_set_cuda_error(e__);       \
  } while (0)
