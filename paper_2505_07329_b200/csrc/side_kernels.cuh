// side_kernels.cuh — launchers (host) for side_kernels.cu and limb_gemm.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "phe_common.cuh"

namespace phe {

int launch_keygen(const KParams &kp, uint64_t seed, uint8_t *S, cudaStream_t st);
int launch_encrypt(const KParams &kp, const uint8_t *S, const int8_t *x, int64_t T, int64_t d_in,
                   int64_t L, uint64_t seed_base, uint64_t noise_seed, uint64_t *seeds,
                   uint64_t *body, cudaStream_t st);
int launch_weights_prepare(const KParams &kp, const int8_t *W, int64_t d_out, int64_t d_in,
                           int transpose, void *wprep, cudaStream_t st);
int launch_ct_prepare(const KParams &kp, const uint64_t *seeds, const uint64_t *body, int64_t T,
                      int64_t L, uint8_t *mask_planes, uint8_t *body_planes, cudaStream_t st);
int launch_modswitch(const uint64_t *in, uint32_t *out, int64_t count, int from, int to,
                     cudaStream_t st);
int launch_decrypt(const KParams &kp, const uint8_t *S, const void *mask, const void *body,
                   int64_t n_ct, int q_bits, bool u64words, int32_t *y, cudaStream_t st);
int launch_simt_matmul(const KParams &kp, const int8_t *W, int64_t d_in, int64_t row_begin,
                       int64_t R, const uint8_t *mplanes, const uint8_t *bplanes, int64_t L,
                       int64_t T, int out_bits, void *out_mask, void *out_body, cudaStream_t st);

int launch_ksk_gen(const KParams &kp, const uint8_t *S, uint64_t seed, uint64_t *KA, uint64_t *KB,
                   cudaStream_t st);
int launch_ksk_planes(const KParams &kp, const uint64_t *ksk, int kpad, int64_t rows, uint8_t *planes,
                      cudaStream_t st);
int launch_pack_finalize(const KParams &kp, const void *acc, const uint64_t *body, int64_t T, int64_t R,
                         int G, uint32_t *out, cudaStream_t st);
int launch_decrypt_packed(const KParams &kp, const uint8_t *S, const uint32_t *packed, int64_t T, int64_t R,
                          int G, int q_bits, int32_t *y, cudaStream_t st);

int launch_wire_inputs(const KParams &kp, uint64_t *seeds, uint64_t *body, int64_t nblk, uint8_t *wire,
                       int dir, cudaStream_t st);
int launch_wire_packed(const KParams &kp, uint32_t *packed, int64_t nct, uint8_t *wire, int dir, cudaStream_t st);
int launch_wire_u32(uint32_t *vals, int64_t nseg, int seglen, int bits, uint8_t *wire, int64_t seg_words,
                    int64_t per_group, int64_t group_words, int64_t off_words, int dir, cudaStream_t st);

int check_weights_range(const int8_t *W, int64_t n, unsigned *flag, cudaStream_t st);
int launch_weights_plain(const KParams &kp, const int8_t *W, int64_t d_out, int64_t d_in, int transpose,
                         int8_t *plain, cudaStream_t st);

// ntt_path.cu (NEXT #4): the mask contraction in the NTT domain (two 31-bit primes + CRT).
int ntt_primes(uint32_t out[2]);
int launch_ntt_tables(const KParams &kp, void *tables, cudaStream_t st);
int launch_ntt_weights(const KParams &kp, const void *tables, const int8_t *W, int64_t d_out,
                       int64_t d_in, int transpose, uint32_t *what, cudaStream_t st);
int launch_ntt_masks(const KParams &kp, const void *tables, const uint64_t *seeds, int64_t T, int64_t L,
                     uint32_t *ahat, cudaStream_t st);
int launch_ntt_encrypt(const KParams &kp, const void *tables, const uint8_t *S, const int8_t *x, int64_t T,
                       int64_t d_in, int64_t L, uint64_t seed_base, uint64_t noise_seed, uint64_t *seeds,
                       uint64_t *body, cudaStream_t st);
int launch_ntt_rowpar(const int8_t *W, int64_t d_out, int64_t d_in, int transpose, uint8_t *par,
                      cudaStream_t st);
int launch_ntt_mask(const KParams &kp, const void *tables, const uint32_t *what, const uint8_t *par,
                    int64_t rows, int64_t Lc, int64_t row_begin, int64_t row_end, const uint32_t *ahat,
                    int64_t T, int out_bits, void *out, cudaStream_t st, int64_t digit_rows = 0,
                    int64_t out_rows = 0);

// ntt_keyswitch.cu (NEXT #1 stage 2 in the NTT domain): sum_{l,i} D_{l,i} * KSK_{l,i} mod 2^q_in
// through three 30-bit primes + CRT, written as the packing GEMM's accumulator.
size_t ntt_ks_bytes(const KParams &kp);
bool ntt_ks_supported(const KParams &kp);
int launch_ntt_ks_prepare(const KParams &kp, const uint64_t *ksk, void *buf, cudaStream_t st);
int ntt_ks_splits(const KParams &kp, int64_t T, int64_t G);
size_t ntt_ks_ws_bytes(const KParams &kp, int64_t T, int64_t G);
int launch_ntt_ks(const KParams &kp, const void *buf, const int8_t *digits, int64_t T, int64_t R, void *ws,
                  void *acc_out, cudaStream_t st);

// limb_gemm.cu: the tcgen05 int8 limb GEMM (mask = Hankel operand, body = plain operand).
struct GemmArgs {
  KParams kp;
  const uint8_t *wexp;    // [rows][Lc][2N][16] 16-shift expansion
  const int8_t *wplain;   // [wplain_rows][Lc*N] (rows padded to a multiple of 128)
  int64_t rows;           // rows of the prepared matrix M
  int64_t wplain_rows;    // padded row count of wplain
  int64_t op_rows;        // padded row count of each limb-plane matrix (>= T*ell, mult. of 256)
  int64_t Lc;             // blocks along M's columns (= L of the input ciphertext)
  int64_t cols;           // columns of M (the contraction length, unpadded)
  int64_t row_begin, row_end;
  const uint8_t *mplanes; // [T*ell][Lc*N]
  const uint8_t *bplanes; // [T*ell][Lc*N]
  int64_t T;
  int out_bits;
  void *out_mask, *out_body;
  int64_t out_rows;       // row stride of out_mask/out_body ([T][out_rows][N] / [T][out_rows]); 0 = R
  int digits;             // 1: out_mask receives Decomp digits int8 [T][digit_rows][3][N] (Eq. 8)
  int64_t digit_rows;     // row stride of the digit tensor (>= row_end - row_begin)
  int64_t wire_words;     // > 0: out_mask is the LWE wire record [T][wire_words] (uint64 words, R22):
                          // the mask GEMM writes the switched words bit-packed at q_out; out_body
                          // receives uint32 bodies (packed into the record by the caller)
};
int launch_limb_gemm(const GemmArgs &a, cudaStream_t st, int *n_launches);

// KeySwitch packing GEMM (NEXT #1): digits [T*rows_pad][3N] int8 x KSK limb planes.
struct PackArgs {
  int N, ell;
  int64_t T, rows_pad;
  int G;
  const uint8_t *digits;
  const uint8_t *kplanes;
  int64_t kplane_rows;
  void *acc;  // uint64 [T][G][2][N], zeroed by the caller
};
int launch_pack_gemm(const PackArgs &a, cudaStream_t st);

}  // namespace phe
