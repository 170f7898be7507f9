/*
 * phe.h — C ABI of the B200-native encrypted-vector x clear-matrix hot path of
 * arXiv 2505.07329 ("private LoRA fine-tuning with HE"): W . [x]_HE.
 *
 * Citations: P:<n> = /root/reference/PAPER.md line n, S:<n> = SPEC.md line n (the reference
 * tree is not shipped; DESIGN.md restates every passage used).
 *
 * Conventions (all calls):
 *  - Pointers prefixed d_ are DEVICE pointers (cudaMalloc / torch CUDA tensors) owned by the
 *    caller.  The library never allocates device memory: every scratch buffer is a caller
 *    workspace sized by a *_bytes / *_ws_bytes query.  Host pointers are prefixed h_.
 *  - The host-buffer pipelines (phe_server_*_host) take a caller device workspace d_ws of two
 *    chunk slots (their *_ws_bytes query, same shape arguments; ENOMEM if smaller), create two
 *    streams + one event on the current device for the call, order after the caller's stream,
 *    and return only after both streams drained (also on an error: no copy still touches the
 *    caller's host buffers).  They are synchronous, re-entrant and hold no state between calls.
 *  - Every call is asynchronous on the caller's `stream` (a cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Argument validation is synchronous: on a non-zero
 *    return nothing was enqueued.
 *  - Errors are returned as int codes (PHE_*); phe_strerror() names them.  A CUDA launch or
 *    runtime failure returns PHE_ECUDA (the CUDA error is left queryable via
 *    phe_last_cuda_error()).  No exception ever crosses the ABI.
 *  - All functions are re-entrant and thread-safe.
 *  - Privacy rule, structural: no server-side call (phe_weights_prepare,
 *    phe_ct_prepare, phe_matmul_clear[_T], phe_modswitch) takes the secret key.
 *  - Integers: ciphertext words are residues mod 2^q stored in uint64_t (q <= 64) or, after
 *    the fused modulus switch to q_out <= 32, in uint32_t.  Moduli are powers of two
 *    (reading R3): Q = 2^q_in, Q' = 2^q_out, t = 2^beta, Delta = Q/t.
 */
#ifndef PHE_H_
#define PHE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes ------------------------------------------------------------------ */
#define PHE_OK 0
#define PHE_EINVAL 1       /* bad dimension / pointer / parameter   */
#define PHE_ERANGE 2       /* |w| > 127 or message outside +-2^(beta-1)   */
#define PHE_EMODULUS 3     /* modulus mismatch: out_bits not in {q_in, q_out} */
#define PHE_ENOMEM 4       /* caller buffer / workspace too small                          */
#define PHE_ECUDA 5        /* CUDA runtime / launch error                                  */
#define PHE_EUNSUPPORTED 6 /* valid parameters this build does not implement (e.g. N<128) */

const char *phe_strerror(int code);
int phe_last_cuda_error(void);

/* ---- a1: parameters (Table 1) -------------------------------------------
 * N      polynomial size, power of two.          GPU path: 128 <= N <= 16384.
 * q_in   input ciphertext modulus bits.           8 <= q_in <= 64 (GPU: <= 64).
 * q_out  output modulus bits after ModulusSwitch. q_out <= q_in, q_out <= 32.
 * beta   plaintext bits, t = 2^beta (R4).          gamma <= beta <= q_in.
 * gamma  MSBs guaranteed noise-free; informational (decrypt contract).
 * noise_eta  0 = E == 0 ("SPEC" reading of sigma, R5); else CBD(eta), eta <= 32.
 *
 * SECURITY NOTE: both presets set noise_eta = 0, the reading under which Table 1's sigma rounds
 * to zero at q = 2^39 (R5).  With E == 0 every input ciphertext satisfies B - A S == Delta x
 * exactly, so anyone who expands A from the public seed can solve for the binary key S: the
 * presets give NO confidentiality and exist for bit-exact parity and benchmarks (the server-side
 * cost does not depend on E).  Encrypt real data with noise, e.g. noise_eta = 21 (sigma ~ 3.2).
 */
typedef struct phe_params {
  int32_t N;
  int32_t q_in;
  int32_t q_out;
  int32_t beta;
  int32_t gamma;
  int32_t noise_eta;
} phe_params;

#define PHE_PRESET_PAPER 0 /* N=2048, q_in=39, q_out=26, beta=27, gamma=12 (Table 1)       */
#define PHE_PRESET_TOY 1   /* N=1024, q_in=32, q_out=28, beta=21, gamma=12 (DESIGN R16)    */

int phe_params_init(phe_params *p, int preset);
/* PHE_OK if valid: N power of two, q_out <= q_in <= 64, gamma <= beta <= q_in. */
int phe_params_validate(const phe_params *p);
/* ell = ceil(q_in / 8): int8 limbs per Z_Q word. */
int phe_num_limbs(const phe_params *p);
/* L = ceil(d / N) blocks per vector of length d. */
int64_t phe_num_blocks(const phe_params *p, int64_t d);

/* ---- keygen (client): S in R_2, binary, deterministic in master_seed.
 * d_S: [N] uint8 in {0,1}; S' = coefficients of S is the LWE key.
 * S[k] = bit (k mod 8) of ChaCha20 keystream byte k/8, key LE64(master_seed)||0^24,
 * nonce "phe-sk" (R6). */
int phe_keygen(const phe_params *p, uint64_t master_seed, uint8_t *d_S, void *stream);

/* ---- encrypt_pack (client): block split + seeded RLWE.
 * d_x:     [T][d_in] int8 (quantized activations/gradients, symmetric).
 * d_seeds: [T][L] uint64 out: seed_{tau,i} = seed_base + tau*L + i (public, one per block).
 * d_body:  [T][L][N] uint64 out: B = A*S + E + Delta*x_hat mod 2^q_in, A = expand(seed),
 *          x_hat_i[k] = x[iN+k] zero-padded; E from noise_seed per noise_eta (R5).
 * Errors: EINVAL (T < 0, d_in < 1, null pointers), ERANGE if 2^(beta-1) <= 128.      */
int phe_encrypt_pack(const phe_params *p, const uint8_t *d_S, const int8_t *d_x, int64_t T,
                     int64_t d_in, uint64_t seed_base, uint64_t noise_seed, uint64_t *d_seeds,
                     uint64_t *d_body, void *stream);

/* ---- a2: weight registration (server, once per model) --------------------------------
 * Absorbs the reversed encoding w_hat_ij[k] = w_j[iN+N-1-k] into the operand layout
 * of the limb GEMM.  With transpose = 0 the prepared matrix is
 * M = W ([rows=d_out][cols=d_in]); with transpose = 1 it is M = W^T ([rows=d_in][cols=d_out])
 * for the backward W^T . [g].  d_W is always W, row-major [d_out][d_in].
 * Layout of d_wprep (bytes, caller-allocated, size phe_weights_bytes):
 *   [rows][Lc][2N][16] int8  "16-shift expansion" of wext_{j,i}[m] = M[j,iN+m] (m < N),
 *                            -M[j,iN+m-N] (N <= m < 2N), 0 beyond cols/2N; Lc = ceil(cols/N)
 *   [rows][Lc*N]       int8  M, zero-padded to Lc*N columns (body GEMM operand)
 * Errors: EINVAL on dims, ENOMEM if bytes is too small, ERANGE if some weight is -128: symmetric
 *   quantization gives w in [-127, 127], and encode_weights refuses out-of-range
 *   weights.  The range check runs on the device and SYNCHRONISES `stream` (once per
 *   model); on ERANGE nothing else was enqueued and d_wprep's contents are unspecified.       */
size_t phe_weights_bytes(const phe_params *p, int64_t rows, int64_t cols);
int phe_weights_prepare(const phe_params *p, const int8_t *d_W, int64_t d_out, int64_t d_in,
                        int transpose, void *d_wprep, size_t bytes, void *stream);

/* ---- a3+a4: ct_prepare (server) -----------------------------------------------------
 * Expands every mask A_{tau,i} = PRNG(seed_{tau,i}) mod 2^q_in (ChaCha20 per R6) and
 * splits masks and bodies into ell little-endian 8-bit limb planes (the GEMM's B operand):
 *   d_operand = [ mask planes  [T*ell][L*N] uint8 | body planes [T*ell][L*N] uint8 ]
 *   plane row tau*ell + l holds byte l of every word of token tau, column i*N + k.
 * Inputs that several linears share (q/k/v; gate/up) are prepared once.            */
size_t phe_ct_operand_bytes(const phe_params *p, int64_t T, int64_t L);
int phe_ct_prepare(const phe_params *p, const uint64_t *d_seeds, const uint64_t *d_body,
                   int64_t T, int64_t L, void *d_operand, size_t bytes, void *stream);

/* ---- a5-a8: matmul_clear (server): LWE(x.w_j) for j in [row_begin, row_end) ---------
 * Eq. 6: LWE(x.w_j) = sum_i SampleExtract(RLWE(x_hat_i) . w_hat_ij, N-1),
 * computed as an int8 limb GEMM on tcgen05 tensor cores with the limb recombination mod
 * 2^q_in and (if out_bits == q_out) the ModulusSwitch fused in the epilogue.
 *   d_wprep:   from phe_weights_prepare(transpose = 0) of W [d_out][d_in].
 *   d_operand: from phe_ct_prepare with L = ceil(d_in / N) for T tokens.
 *   out_bits:  q_in  -> d_out_mask uint64 [T][R][N], d_out_body uint64 [T][R]  (no switch)
 *              q_out -> d_out_mask uint32 [T][R][N], d_out_body uint32 [T][R]  (switched)
 *              with R = row_end - row_begin (row sharding).
 *   Mask entry [tau][j][t] is a'_t of LWE(x_tau . w_j) (Eq. 2 with h = N-1); body [tau][j] = b'.
 *   Either output pointer may be NULL: that part (a5 mask / a6 body GEMM) is then skipped,
 *   so the two contractions can be launched and timed separately.
 * Errors: EINVAL (row range, T < 0, null), EMODULUS (out_bits not q_in/q_out),
 *         EUNSUPPORTED (N < 128, ell > 8).  T == 0 is a no-op returning PHE_OK.          */
int phe_matmul_clear(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                     int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                     int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream);

/* ---- a9: matmul_clear_T (server, backward): LWE((W^T g)_c), c in [row_begin, row_end) --
 * Same contract with M = W^T: d_wprep from phe_weights_prepare(transpose = 1) of W
 * [d_out][d_in]; the input ciphertext encrypts g in Z^{d_out} (L = ceil(d_out / N)); output
 * rows index c in [0, d_in).                                                */
int phe_matmul_clear_T(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                       int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                       int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream);

/* ---- matmul_clear into a row block of a larger output (row sharding with a fused gather) -----
 * Same contract as phe_matmul_clear (transpose = 0) / phe_matmul_clear_T (transpose = 1), except
 * that the outputs are written with a row stride of out_rows (>= row_end - row_begin): mask word
 * (tau, j, t) goes to d_out_mask[(tau * out_rows + (j - row_begin)) * N + t], body (tau, j) to
 * d_out_body[tau * out_rows + (j - row_begin)].  Point d_out_mask/d_out_body at the rank's row
 * block inside a [T][R_total][N] gather buffer -- also a peer GPU's buffer mapped through CUDA
 * IPC (paper_2505_07329_b200.dist.PeerGather): the epilogue's TMA stores then move the shard
 * over NVLink as it is produced, and no separate gather collective runs.       */
int phe_matmul_clear_into(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T, int32_t out_bits,
                          void *d_out_mask, void *d_out_body, int64_t out_rows, void *stream);

/* ---- matmul_clear(W, ct): the north_star's one-call form on device buffers ------------------
 * phe_ct_prepare of (d_seeds, d_body) into the caller's workspace d_ws (>= phe_ct_operand_bytes(p,
 * T, L), L = blocks of the input length: d_in forward, d_out backward), then phe_matmul_clear
 * (transpose = 0, d_wprep of W) or phe_matmul_clear_T (transpose = 1, d_wprep of W^T).  Same
 * outputs, layouts and errors as those two calls; ENOMEM if ws_bytes is too small.          */
int phe_matmul_clear_ct(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                        int transpose, int64_t row_begin, int64_t row_end, const uint64_t *d_seeds,
                        const uint64_t *d_body, int64_t T, int32_t out_bits, void *d_ws,
                        size_t ws_bytes, void *d_out_mask, void *d_out_body, void *stream);

/* ---- a8 standalone: ModulusSwitch --------------------------
 * d_out[k] = floor((d_in[k] + 2^(f-t-1)) / 2^(f-t)) mod 2^t, f = from_bits, t = to_bits,
 * round half up on the non-negative residue (R8).  Requires 1 <= t <= f <= 64, t <= 32.  */
int phe_modswitch(const uint64_t *d_in, uint32_t *d_out, int64_t count, int32_t from_bits,
                  int32_t to_bits, void *stream);

/* ---- decrypt_unpack (client): LWE decryption under S' ---
 * phi = (b - sum_t a[t] S[t]) mod 2^q_bits; q_bits >= beta: m = round(phi / 2^(q-beta)) mod t;
 * q_bits < beta: m = phi * 2^(beta-q) mod t; centred into [-t/2, t/2).
 * d_mask/d_body: uint64 if q_bits == p->q_in, uint32 if q_bits == p->q_out (matmul outputs);
 * shapes [T][rows][N] and [T][rows].  d_y: [T][rows] int32 out.                          */
int phe_decrypt_unpack(const phe_params *p, const uint8_t *d_S, const void *d_mask,
                       const void *d_body, int64_t T, int64_t rows, int32_t q_bits,
                       int32_t *d_y, void *stream);

/* ---- end to end with HOST buffers (the server step as a client call sees it) ----------
 * h_seeds [T][L] uint64, h_body [T][L][N] uint64 (pinned host memory recommended);
 * result (switched to q_out, uint32) streamed back into h_out_mask [T][R][N], h_out_body
 * [T][R].  Tokens are processed in chunks of `chunk_tokens`: H2D of chunk c+1 and D2H of
 * chunk c-1 overlap the GEMM of chunk c on two per-call streams.  d_wprep is device-resident
 * (registered once).  d_ws: caller workspace of phe_server_matvec_host_ws_bytes(...) bytes
 * (same p, d_out, d_in, transpose, rows, T, chunk_tokens; 0 = invalid arguments).
 * Synchronous: returns after all copies completed.                                        */
size_t phe_server_matvec_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose,
                                       int64_t row_begin, int64_t row_end, int64_t T, int64_t chunk_tokens);
int phe_server_matvec_host(const phe_params *p, const void *d_wprep, int64_t d_out,
                           int64_t d_in, int transpose, int64_t row_begin, int64_t row_end,
                           const uint64_t *h_seeds, const uint64_t *h_body, int64_t T,
                           int64_t chunk_tokens, uint32_t *h_out_mask, uint32_t *h_out_body,
                           void *d_ws, size_t ws_bytes, void *stream);

/* ---- NEXT #1: KeySwitch packing of the LWE outputs into RLWE (Eq. 7; Eq. 8,
 * P:233-249) --------------------------------------------------------------------------------
 * Gadget: Decomp = signed balanced base-2^8 digits of the top 32 bits (4 levels) after rounding
 * the q_in - 32 bit tail half up (R18: 4 levels because P:396's Fig. 4 claim
 * fails with 3).  Requires q_in >= 32.
 * KSK_{i,l} = RLWE_S(S'_i * 2^(q_in - 8(l+1))) for i < N, l < 4.
 *
 * phe_ksk_gen (client): d_ksk = uint64 [2][4N][N]: part 0 = KSK_A, part 1 = KSK_B, row l*N + i
 *   (the batched matrices of Eq. 8).  Masks from ChaCha20(ksk_seed, "phe-ksk"), noise CBD(eta)
 *   from "phe-ksknoise" (R19).  Public key material: the server may hold it.            */
size_t phe_ksk_bytes(const phe_params *p);
int phe_ksk_gen(const phe_params *p, const uint8_t *d_S, uint64_t ksk_seed, void *d_ksk,
                size_t bytes, void *stream);
/* phe_ksk_prepare (server, once per key): KSK limb planes, the B operand of the packing GEMM
 * (uint8 [rows][4N], rows = phe_ksk_prep_bytes / 4N).                                      */
size_t phe_ksk_prep_bytes(const phe_params *p);
int phe_ksk_prepare(const phe_params *p, const void *d_ksk, void *d_kprep, size_t bytes, void *stream);
/* phe_matmul_clear_packed (server): the paper's whole primitive RLWE(Wx) for T tokens:
 *   LWE outputs of Eq. 6 (mask GEMM writing Decomp digits, body GEMM at q_in), then Eq. 8 +
 *   Eq. 7 (packing GEMM: KeySwitch, Rotate by j mod N, sum), then ModulusSwitch to q_out.
 *   d_out_packed: uint32 [T][G][2][N], G = ceil(R / N), R = rows of M (d_out, or d_in with
 *   transpose = 1); [..][0][..] = A', [..][1][..] = B'; output j sits in coefficient j mod N
 *   of ciphertext j / N.  d_ws: workspace of phe_packed_ws_bytes(p, R, T) bytes.
 *   Errors: EUNSUPPORTED unless ell in {4,5}, N % 256 == 0, q_in >= 32.                      */
size_t phe_packed_ws_bytes(const phe_params *p, int64_t rows, int64_t T);
/* The two stages of phe_matmul_clear_packed, callable separately:
 * phe_matmul_clear_digits: Eq. 6 with the LWE masks written as Decomp digits, int8
 *   d_digits [T][R256][4][N] (R256 = R rounded up to 256; pad rows zeroed; plane l = digit of
 *   weight 2^(q_in - 8(l+1))) and bodies d_body uint64 [T][R] at q_in.
 * phe_pack: Eq. 8 + Eq. 7 from those digits/bodies; d_acc: uint64 scratch of
 *   phe_pack_acc_bytes(p, R, T) bytes; output as phe_matmul_clear_packed.                    */
int phe_matmul_clear_digits(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                            int transpose, const void *d_operand, int64_t T, void *d_digits,
                            uint64_t *d_body, void *stream);
size_t phe_pack_acc_bytes(const phe_params *p, int64_t rows, int64_t T);
int phe_pack(const phe_params *p, const void *d_digits, const uint64_t *d_body, int64_t T, int64_t rows,
             const void *d_kprep, void *d_acc, size_t acc_bytes, uint32_t *d_out_packed, void *stream);
int phe_matmul_clear_packed(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                            int transpose, const void *d_operand, int64_t T, const void *d_kprep,
                            void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream);
/* phe_server_matvec_packed_host: phe_server_matvec_host for the packed primitive: host seeds /
 * bodies in, h_out_packed uint32 [T][G][2][N] out (chunked, copies overlapped; caller workspace
 * of phe_server_matvec_packed_host_ws_bytes(...) bytes, sized for the full and the ragged last
 * chunk).                                                                                   */
size_t phe_server_matvec_packed_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose,
                                              int64_t T, int64_t chunk_tokens);
int phe_server_matvec_packed_host(const phe_params *p, const void *d_wprep, int64_t d_out,
                                  int64_t d_in, int transpose, const void *d_kprep,
                                  const uint64_t *h_seeds, const uint64_t *h_body, int64_t T,
                                  int64_t chunk_tokens, uint32_t *h_out_packed, void *d_ws, size_t ws_bytes,
                                  void *stream);
/* phe_decrypt_packed (client): d_y int32 [T][rows] = decode(B' - A'S) coefficient-wise. */
int phe_decrypt_packed(const phe_params *p, const uint8_t *d_S, const uint32_t *d_packed, int64_t T,
                       int64_t rows, int32_t q_bits, int32_t *d_y, void *stream);

/* ---- NEXT #2: wire format ------------------------------------
 * Little-endian contiguous bitstream, no per-coefficient padding (R22).
 * Input block (client -> server): [LE64 seed][N body coefficients at q_in bits]
 *   = 8 + N*q_in/8 bytes (9992 at Table 1).
 * Packed output (server -> client): [A' at q_out bits][B' at q_out bits] = 2*N*q_out/8 bytes
 *   (13312 at Table 1).  Requires q_in <= 57, N % 8 == 0.
 * d_seeds [T][L] / d_body [T][L][N] uint64; d_packed uint32 [n_ct][2][N]; d_wire bytes, 8-byte
 * aligned (else EINVAL); requires N % 64 == 0 and q_in <= 57 (else EUNSUPPORTED).           */
size_t phe_wire_input_bytes(const phe_params *p);
size_t phe_wire_output_bytes(const phe_params *p);
int phe_wire_serialize_inputs(const phe_params *p, const uint64_t *d_seeds, const uint64_t *d_body,
                              int64_t T, int64_t L, uint8_t *d_wire, void *stream);
int phe_wire_deserialize_inputs(const phe_params *p, const uint8_t *d_wire, int64_t T, int64_t L,
                                uint64_t *d_seeds, uint64_t *d_body, void *stream);
int phe_wire_serialize_packed(const phe_params *p, const uint32_t *d_packed, int64_t n_ct,
                              uint8_t *d_wire, void *stream);
int phe_wire_deserialize_packed(const phe_params *p, const uint8_t *d_wire, int64_t n_ct,
                                uint32_t *d_packed, void *stream);
/* The server step as the network sees it: h_wire_in [T][L] input blocks -> h_wire_out [T][G]
 * packed ciphertexts (host buffers; chunked; caller workspace of phe_server_wire_host_ws_bytes
 * bytes, sized for the full and the ragged last chunk: the packing workspace is not monotone
 * in T).                                                                                    */
size_t phe_server_wire_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                     int64_t chunk_tokens);
int phe_server_wire_host(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                         int transpose, const void *d_kprep, const uint8_t *h_wire_in, int64_t T,
                         int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream);

/* ---- NEXT #4: the mask contraction a5 in the NTT domain ---------
 * Same contract and bit-identical results as phe_matmul_clear(_T): Eq. 6 defines the
 * LWE outputs uniquely.  Computed as negacyclic products in Z_p[X]/(X^N + 1) (X^N = -1)
 * for two primes p0 = 15*2^27+1 and p1 = 63*2^25+1 (forward NTT, pointwise sum over blocks i,
 * inverse NTT; CUDA cores, not tensor cores); the exact integer product is recovered by CRT and
 * reduced mod 2^q_in, since power-of-two moduli admit no NTT (R23).
 * Requirements: N a power of two in [512, 8192] and L <= phe_ntt_max_blocks(p) (CRT
 * exactness: L*N*(2^q_in - 1)*128 < p0*p1/2; 14 blocks for Table 1), else PHE_EUNSUPPORTED.
 *   d_tables  phe_ntt_tables_bytes(p): uint2 [2 dirs][2 primes][N] twiddles (w, floor(w 2^32/p)),
 *             dir 0 = psi^bitrev(k), dir 1 = psi^-bitrev(k), then uint2 [15][N/16][2 primes], the
 *             inverse twiddles of stages 0-3 regrouped per thread of the hot kernel; written
 *             once by phe_ntt_tables_init; read-only afterwards; shared by every call with p.
 *   d_nttw    phe_ntt_weights_bytes(p, rows, cols), rows/cols of M = W (transpose 0) or W^T:
 *               [rows][Lc][2][N] uint32  NTT_p(w_hat_ij) * N^-1 * 2^32 mod p (w_hat_ij[k] =
 *                                        M[j, iN+N-1-k])
 *               [round128(rows)][Lc*N] int8  M zero-padded (body GEMM operand)
 *               [round16(rows)] uint8    (sum_c M[j,c]) mod 2, the centring correction (R23)
 *   d_operand phe_ntt_operand_bytes(p, T, L):
 *               [T][L][2][N] uint32  NTT_p(A_{tau,i} - 2^(q_in-1) mod p), A = PRNG(seed) mod 2^q_in
 *                                    (centred, R23)
 *               [op_rows][L*N] uint8 body limb planes (the second half of phe_ct_prepare's layout)
 *             NTT-domain vectors: element k of the bit-reversed transform output is stored at
 *             word 4*(((k>>2)&3)*(N/16) + (k>>4)) + (k&3) (the hot kernel's thread order).
 * Errors as phe_matmul_clear; EUNSUPPORTED for N or L outside the range above; ERANGE (after a
 * synchronising device-side check, as phe_weights_prepare) if some weight is -128 (P:150-164,
 * S:253-255): both contractions accept exactly the same weights.                             */
int phe_ntt_primes(uint32_t *out2);
int64_t phe_ntt_max_blocks(const phe_params *p);
size_t phe_ntt_tables_bytes(const phe_params *p);
int phe_ntt_tables_init(const phe_params *p, void *d_tables, size_t bytes, void *stream);
size_t phe_ntt_weights_bytes(const phe_params *p, int64_t rows, int64_t cols);
int phe_ntt_weights_prepare(const phe_params *p, const void *d_tables, const int8_t *d_W,
                            int64_t d_out, int64_t d_in, int transpose, void *d_nttw, size_t bytes,
                            void *stream);
size_t phe_ntt_operand_bytes(const phe_params *p, int64_t T, int64_t L);
int phe_ntt_ct_prepare(const phe_params *p, const void *d_tables, const uint64_t *d_seeds,
                       const uint64_t *d_body, int64_t T, int64_t L, void *d_operand, size_t bytes,
                       void *stream);
/* encrypt_pack with the product A*S through the NTT (client side): same contract and
 * bit-identical output as phe_encrypt_pack; A*S (|A*S| < N 2^q_in) is computed exactly as
 * INTT(NTT(A) o NTT(S)) mod p0, p1 and a centred CRT -- O(N log N) per block instead of N^2/2.
 * d_tables from phe_ntt_tables_init.  EUNSUPPORTED if N 2^q_in >= p0 p1 / 2.                 */
int phe_encrypt_pack_ntt(const phe_params *p, const void *d_tables, const uint8_t *d_S, const int8_t *d_x,
                         int64_t T, int64_t d_in, uint64_t seed_base, uint64_t noise_seed, uint64_t *d_seeds,
                         uint64_t *d_body, void *stream);
/* Stage 1 of the packed primitive through the NTT path: same contract and bit-identical output
 * as phe_matmul_clear_digits (digits int8 [T][round256(rows)][4][N], bodies uint64 [T][rows] at
 * q_in), mask contraction in the NTT domain; then phe_pack as usual.  Requires q_in >= 32.     */
int phe_matmul_clear_digits_ntt(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                                int64_t d_in, int transpose, const void *d_operand, int64_t T, void *d_digits,
                                uint64_t *d_body, void *stream);
int phe_matmul_clear_ntt(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                         int64_t d_in, int64_t row_begin, int64_t row_end, const void *d_operand,
                         int64_t T, int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream);
int phe_matmul_clear_ntt_into(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                              int64_t d_in, int transpose, int64_t row_begin, int64_t row_end,
                              const void *d_operand, int64_t T, int32_t out_bits, void *d_out_mask,
                              void *d_out_body, int64_t out_rows, void *stream);
int phe_matmul_clear_ntt_T(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                           int64_t d_in, int64_t row_begin, int64_t row_end, const void *d_operand,
                           int64_t T, int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream);

/* ---- LWE outputs on the wire: the switched LWE ciphertexts at q_out bits (R22's bitstream) ----
 * Per token: R mask segments of N coefficients (N q_out / 64 words each), then the R bodies at
 * q_out bits padded to a whole 64-bit word: phe_wire_lwe_bytes(p, R) bytes per token (Table 1,
 * R = 2048: 13,638,144 B = 0.8125 of the uint32 form).  d_mask uint32 [T][R][N], d_body uint32
 * [T][R] (as phe_matmul_clear at out_bits = q_out); d_wire 8-byte aligned.                     */
size_t phe_wire_lwe_bytes(const phe_params *p, int64_t R);
int phe_wire_serialize_lwe(const phe_params *p, const uint32_t *d_mask, const uint32_t *d_body, int64_t T,
                           int64_t R, uint8_t *d_wire, void *stream);
int phe_wire_deserialize_lwe(const phe_params *p, const uint8_t *d_wire, int64_t T, int64_t R,
                             uint32_t *d_mask, uint32_t *d_body, void *stream);
/* phe_matmul_clear_wire: matmul_clear(_T) (by `transpose`) with the fused switch, writing the wire
 * records directly: the mask GEMM's epilogue packs each 128-coefficient block of a row at q_out
 * bits (2 q_out 64-bit words) and TMA-stores it into d_wire [T][phe_wire_lwe_bytes(p, R)], R =
 * row_end - row_begin; the bodies go through d_ws (uint32 [T][R], phe_matmul_clear_wire_ws_bytes)
 * into each record's tail.  Byte-identical to phe_wire_serialize_lwe of phe_matmul_clear's
 * uint32 outputs, with 0.8125 of their HBM writes.  EUNSUPPORTED unless
 * phe_wire_lwe_direct_supported(p, R) (ell in {4, 5}, N a multiple of 256, 16 <= q_out <= 26 < q_in,
 * 16-byte record stride) and d_wire is 16-byte aligned.                                        */
size_t phe_matmul_clear_wire_ws_bytes(const phe_params *p, int64_t T, int64_t R);
int phe_wire_lwe_direct_supported(const phe_params *p, int64_t R);
int phe_matmul_clear_wire(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T, uint8_t *d_wire,
                          void *d_ws, size_t ws_bytes, void *stream);
/* The LWE server step as the network sees it: h_wire_in [T][L] wire input blocks (9992 B each)
 * -> h_wire_out [T][phe_wire_lwe_bytes(p, R)], R = row_end - row_begin; chunked H2D, deserialize,
 * ct_prepare, matmul_clear(_T) with the fused switch (phe_matmul_clear_wire where supported, else
 * uint32 outputs + serialize), D2H on two per-call streams
 * (caller workspace of phe_server_matvec_wire_host_ws_bytes bytes).  Synchronous.           */
size_t phe_server_matvec_wire_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose,
                                            int64_t row_begin, int64_t row_end, int64_t T, int64_t chunk_tokens);
int phe_server_matvec_wire_host(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                                int transpose, int64_t row_begin, int64_t row_end, const uint8_t *h_wire_in,
                                int64_t T, int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes,
                                void *stream);

/* ---- NEXT #1 stage 2 in the NTT domain (Eq. 7 + Eq. 8) ---------------
 * Exchanging Eq. 7's sum over outputs j with Eq. 4's sum over KSK rows gives, for packed
 * ciphertext g,  acc_g = sum_{l,i} D_{l,i}(X) * KSK_{l,i}(X),  D_{l,i}(X) = sum_r d_{gN+r,i,l} X^r
 * (negacyclic, X^N = -1): 4N polynomial products, computed exactly modulo three 30-bit
 * primes (forward NTT of every D_{l,i}, pointwise products with the registered KSK, inverse NTT)
 * and recovered mod 2^q_in by CRT; then (0, b) - acc and the switch as phe_pack.  Same contract
 * and bit-identical output as phe_pack (the value is Eq. 7's, unique); O(log N) work per (l, i,
 * coefficient) instead of the MatMul's O(N).
 * phe_ntt_ksk_prepare (server, once per key): d_nksk (phe_ntt_ksk_bytes(p) bytes, 256-aligned)
 *   <- twiddle tables + NTT(centred KSK rows) N^-1 2^32 mod p for the three primes; d_ksk as
 *   phe_ksk_gen writes it ([2][4N][N] uint64).  Public key material only.
 * phe_pack_ntt: d_digits / d_body / d_out_packed as phe_pack; d_ws scratch of
 *   phe_pack_ntt_ws_bytes(p, rows, T) bytes.
 * Errors: EUNSUPPORTED unless 256 <= N <= 8192, q_in >= 32 and 2^(q_in + 2 log2 N + 9) <
 *   p0 p1 p2 (Table 1: q_in <= 56 at N = 2048); ENOMEM for short buffers.                     */
size_t phe_ntt_ksk_bytes(const phe_params *p);
int phe_ntt_ksk_prepare(const phe_params *p, const void *d_ksk, void *d_nksk, size_t bytes, void *stream);
size_t phe_pack_ntt_ws_bytes(const phe_params *p, int64_t rows, int64_t T);
int phe_pack_ntt(const phe_params *p, const void *d_digits, const uint64_t *d_body, int64_t T, int64_t rows,
                 const void *d_nksk, void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream);
/* phe_matmul_clear_packed_ntt: the whole primitive as phe_matmul_clear_packed (same contract and
 *   output), stage 1 (Eq. 6 -> Decomp digits) on the tensor cores, stage 2 through phe_pack_ntt;
 *   d_nksk from phe_ntt_ksk_prepare, d_ws of phe_packed_ntt_ws_bytes(p, rows, T) bytes.
 * phe_server_wire_host_ntt: phe_server_wire_host with phe_matmul_clear_packed_ntt inside.
 * phe_matmul_clear_packed_nttw: the same primitive with stage 1 in the NTT domain as well
 *   (phe_matmul_clear_digits_ntt on d_nttw from phe_ntt_weights_prepare and d_operand from
 *   phe_ntt_ct_prepare, d_tables from phe_ntt_tables_init), then phe_pack_ntt; same output, d_ws
 *   of phe_packed_ntt_ws_bytes(p, rows, T) bytes; errors as phe_matmul_clear_packed_ntt, and
 *   EUNSUPPORTED where phe_matmul_clear_digits_ntt is (q_in < 32, L above phe_ntt_max_blocks).
 * phe_server_wire_host_nttw: phe_server_wire_host with phe_ntt_ct_prepare +
 *   phe_matmul_clear_packed_nttw inside (NTT weights and tables instead of d_wprep).            */
size_t phe_packed_ntt_ws_bytes(const phe_params *p, int64_t rows, int64_t T);
int phe_matmul_clear_packed_ntt(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                                int transpose, const void *d_operand, int64_t T, const void *d_nksk,
                                void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream);
size_t phe_server_wire_host_ntt_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                         int64_t chunk_tokens);
int phe_server_wire_host_ntt(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                             const void *d_nksk, const uint8_t *h_wire_in, int64_t T, int64_t chunk_tokens,
                             uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream);
int phe_matmul_clear_packed_nttw(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                                 int64_t d_in, int transpose, const void *d_operand, int64_t T, const void *d_nksk,
                                 void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream);
size_t phe_server_wire_host_nttw_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                          int64_t chunk_tokens);
int phe_server_wire_host_nttw(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                              int64_t d_in, int transpose, const void *d_nksk, const uint8_t *h_wire_in, int64_t T,
                              int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream);

/* ---- introspection (tests / bench) -------------------------------------------------- */
/* Number of kernel launches the last phe_matmul_clear[_T] on this thread enqueued. */
int phe_last_launch_count(void);
/* Reference SIMT (CUDA-core, 64-bit) implementation of the same contract as
 * phe_matmul_clear, used only as an on-device cross-check in tests.                      */
int phe_matmul_clear_simt(const phe_params *p, const int8_t *d_W, int64_t d_out, int64_t d_in,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                          int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* PHE_H_ */
