// phe_api.cu — the C ABI declared in include/phe.h: validation, layouts, launches, and the
// host-buffer end-to-end pipeline.  No torch types cross this boundary.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstring>
#include <vector>

#include "phe_common.cuh"
#include "side_kernels.cuh"

using phe::KParams;

static thread_local int g_last_cuda_error = 0;
static thread_local int g_last_launches = 0;

int phe_set_cuda_error(cudaError_t e) {
  g_last_cuda_error = (int)e;
  return PHE_ECUDA;
}

extern "C" {

const char *phe_strerror(int code) {
  switch (code) {
    case PHE_OK: return "ok";
    case PHE_EINVAL: return "invalid argument";
    case PHE_ERANGE: return "value out of range";
    case PHE_EMODULUS: return "modulus mismatch";
    case PHE_ENOMEM: return "buffer too small";
    case PHE_ECUDA: return "CUDA error";
    case PHE_EUNSUPPORTED: return "unsupported parameters";
  }
  return "unknown error";
}

int phe_last_cuda_error(void) { return g_last_cuda_error; }
int phe_last_launch_count(void) { return g_last_launches; }

int phe_params_init(phe_params *p, int preset) {
  if (!p) return PHE_EINVAL;
  if (preset == PHE_PRESET_PAPER) {  // Table 1
    *p = phe_params{2048, 39, 26, 27, 12, 0};
  } else if (preset == PHE_PRESET_TOY) {  // DESIGN.md R16
    *p = phe_params{1024, 32, 28, 21, 12, 0};
  } else {
    return PHE_EINVAL;
  }
  return PHE_OK;
}

int phe_params_validate(const phe_params *p) {
  if (!p) return PHE_EINVAL;
  if (p->N < 2 || (p->N & (p->N - 1))) return PHE_EINVAL;  // power of two
  if (p->q_in < 1 || p->q_in > 64) return PHE_EINVAL;
  if (p->q_out < 1 || p->q_out > p->q_in) return PHE_EINVAL;
  if (p->beta < p->gamma || p->beta > p->q_in || p->gamma < 0) return PHE_EINVAL;
  if (p->noise_eta < 0 || p->noise_eta > 32) return PHE_EINVAL;
  return PHE_OK;
}

int phe_num_limbs(const phe_params *p) { return p ? (p->q_in + 7) / 8 : 0; }

int64_t phe_num_blocks(const phe_params *p, int64_t d) {
  return (p && p->N > 0 && d > 0) ? (d + p->N - 1) / p->N : 0;
}

}  // extern "C"

// GPU-path requirements beyond phe_params_validate
static int check_gpu(const phe_params *p, KParams *kp) {
  int rc = phe_params_validate(p);
  if (rc) return rc;
  if (p->N < 128 || p->N > 16384) return PHE_EUNSUPPORTED;
  if (p->q_out > 32) return PHE_EUNSUPPORTED;
  kp->N = p->N;
  kp->log2N = 0;
  while ((1 << kp->log2N) < p->N) kp->log2N++;
  kp->q_in = p->q_in; kp->q_out = p->q_out; kp->beta = p->beta; kp->eta = p->noise_eta;
  kp->ell = (p->q_in + 7) / 8;
  kp->qmask = phe::mask_bits(p->q_in);
  return PHE_OK;
}

static inline cudaStream_t S(void *s) { return reinterpret_cast<cudaStream_t>(s); }
static inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
static inline int64_t op_rows(int64_t T, int ell) {
  int64_t r = round_up(T * ell, 256);
  return r < 256 ? 256 : r;
}

extern "C" {

int phe_keygen(const phe_params *p, uint64_t master_seed, uint8_t *d_S, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (!d_S) return PHE_EINVAL;
  return phe::launch_keygen(kp, master_seed, d_S, S(stream));
}

int phe_encrypt_pack(const phe_params *p, const uint8_t *d_S, const int8_t *d_x, int64_t T,
                     int64_t d_in, uint64_t seed_base, uint64_t noise_seed, uint64_t *d_seeds,
                     uint64_t *d_body, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (T < 0 || d_in < 1) return PHE_EINVAL;
  if (T > 0 && (!d_S || !d_x || !d_seeds || !d_body)) return PHE_EINVAL;
  if (p->beta < 9) return PHE_ERANGE;  // int8 messages need |m| < 2^(beta-1)
  int64_t L = phe_num_blocks(p, d_in);
  return phe::launch_encrypt(kp, d_S, d_x, T, d_in, L, seed_base, noise_seed, d_seeds, d_body,
                             S(stream));
}

size_t phe_weights_bytes(const phe_params *p, int64_t rows, int64_t cols) {
  if (!p || rows < 1 || cols < 1 || p->N < 1) return 0;
  int64_t Lc = phe_num_blocks(p, cols);
  return (size_t)(rows * Lc * 2 * p->N * 16) + (size_t)(round_up(rows, 128) * Lc * p->N);
}

int phe_weights_prepare(const phe_params *p, const int8_t *d_W, int64_t d_out, int64_t d_in,
                        int transpose, void *d_wprep, size_t bytes, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (!d_W || !d_wprep || d_out < 1 || d_in < 1 || (transpose != 0 && transpose != 1))
    return PHE_EINVAL;
  int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (bytes < phe_weights_bytes(p, rows, cols)) return PHE_ENOMEM;
  rc = phe::check_weights_range(d_W, d_out * d_in, static_cast<unsigned *>(d_wprep), S(stream));
  if (rc) return rc;
  return phe::launch_weights_prepare(kp, d_W, d_out, d_in, transpose, d_wprep, S(stream));
}

size_t phe_ct_operand_bytes(const phe_params *p, int64_t T, int64_t L) {
  if (!p || T < 0 || L < 1 || p->N < 1) return 0;
  int ell = (p->q_in + 7) / 8;
  return (size_t)(2 * op_rows(T, ell) * L * p->N);
}

int phe_ct_prepare(const phe_params *p, const uint64_t *d_seeds, const uint64_t *d_body, int64_t T,
                   int64_t L, void *d_operand, size_t bytes, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (T < 0 || L < 1 || !d_operand) return PHE_EINVAL;
  if (T > 0 && (!d_seeds || !d_body)) return PHE_EINVAL;
  if (bytes < phe_ct_operand_bytes(p, T, L)) return PHE_ENOMEM;
  uint8_t *mp = static_cast<uint8_t *>(d_operand);
  uint8_t *bp = mp + op_rows(T, kp.ell) * L * p->N;
  return phe::launch_ct_prepare(kp, d_seeds, d_body, T, L, mp, bp, S(stream));
}

}  // extern "C"

static int matmul_common(const phe_params *p, const void *d_wprep, int64_t rows, int64_t cols,
                         int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                         int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream,
                         int64_t out_rows = 0) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (rows < 1 || cols < 1 || T < 0) return PHE_EINVAL;
  if (row_begin < 0 || row_end > rows || row_begin > row_end) return PHE_EINVAL;
  if (out_bits != p->q_in && out_bits != p->q_out) return PHE_EMODULUS;
  if (T == 0 || row_end == row_begin) return PHE_OK;
  if (!d_wprep || !d_operand || (!d_out_mask && !d_out_body)) return PHE_EINVAL;
  if (p->N % 128) return PHE_EUNSUPPORTED;
  const int64_t N = p->N, Lc = phe_num_blocks(p, cols);
  phe::GemmArgs a{};
  a.kp = kp;
  a.wexp = static_cast<const uint8_t *>(d_wprep);
  a.wplain = reinterpret_cast<const int8_t *>(a.wexp + rows * Lc * 2 * N * 16);
  a.rows = rows;
  a.wplain_rows = round_up(rows, 128);
  a.op_rows = op_rows(T, kp.ell);
  a.Lc = Lc;
  a.cols = cols;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.mplanes = static_cast<const uint8_t *>(d_operand);
  a.bplanes = a.mplanes + a.op_rows * Lc * N;
  a.T = T;
  a.out_bits = out_bits;
  a.out_mask = d_out_mask;
  a.out_body = d_out_body;
  a.out_rows = out_rows;
  int n = 0;
  rc = phe::launch_limb_gemm(a, S(stream), &n);
  g_last_launches = n;
  return rc;
}

extern "C" {

int phe_matmul_clear(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                     int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                     int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream) {
  return matmul_common(p, d_wprep, d_out, d_in, row_begin, row_end, d_operand, T, out_bits,
                       d_out_mask, d_out_body, stream);
}

int phe_matmul_clear_T(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                       int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                       int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream) {
  // M = W^T: rows = d_in, cols = d_out
  return matmul_common(p, d_wprep, d_in, d_out, row_begin, row_end, d_operand, T, out_bits,
                       d_out_mask, d_out_body, stream);
}

int phe_matmul_clear_into(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T, int32_t out_bits,
                          void *d_out_mask, void *d_out_body, int64_t out_rows, void *stream) {
  if (!p || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (out_rows < row_end - row_begin) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  return matmul_common(p, d_wprep, rows, cols, row_begin, row_end, d_operand, T, out_bits, d_out_mask,
                       d_out_body, stream, out_rows);
}

int phe_matmul_clear_ct(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                        int transpose, int64_t row_begin, int64_t row_end, const uint64_t *d_seeds,
                        const uint64_t *d_body, int64_t T, int32_t out_bits, void *d_ws,
                        size_t ws_bytes, void *d_out_mask, void *d_out_body, void *stream) {
  if (!p || (transpose != 0 && transpose != 1) || d_out < 1 || d_in < 1) return PHE_EINVAL;
  const int64_t L = phe_num_blocks(p, transpose ? d_out : d_in);
  int rc = phe_ct_prepare(p, d_seeds, d_body, T, L, d_ws, ws_bytes, stream);
  if (rc) return rc;
  return transpose ? phe_matmul_clear_T(p, d_wprep, d_out, d_in, row_begin, row_end, d_ws, T, out_bits,
                                        d_out_mask, d_out_body, stream)
                   : phe_matmul_clear(p, d_wprep, d_out, d_in, row_begin, row_end, d_ws, T, out_bits,
                                      d_out_mask, d_out_body, stream);
}

int phe_matmul_clear_simt(const phe_params *p, const int8_t *d_W, int64_t d_out, int64_t d_in,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                          int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (d_out < 1 || d_in < 1 || T < 0 || row_begin < 0 || row_end > d_out || row_begin > row_end)
    return PHE_EINVAL;
  if (out_bits != p->q_in && out_bits != p->q_out) return PHE_EMODULUS;
  if (T == 0 || row_end == row_begin) return PHE_OK;
  const int64_t L = phe_num_blocks(p, d_in);
  const uint8_t *mp = static_cast<const uint8_t *>(d_operand);
  const uint8_t *bp = mp + op_rows(T, kp.ell) * L * p->N;
  return phe::launch_simt_matmul(kp, d_W, d_in, row_begin, row_end - row_begin, mp, bp, L, T,
                                 out_bits, d_out_mask, d_out_body, S(stream));
}

int phe_modswitch(const uint64_t *d_in, uint32_t *d_out, int64_t count, int32_t from_bits,
                  int32_t to_bits, void *stream) {
  if (count < 0 || to_bits < 1 || to_bits > 32 || from_bits < to_bits || from_bits > 64)
    return PHE_EINVAL;
  if (count == 0) return PHE_OK;
  if (!d_in || !d_out) return PHE_EINVAL;
  if ((reinterpret_cast<uintptr_t>(d_in) & 15) || (reinterpret_cast<uintptr_t>(d_out) & 15))
    return PHE_EINVAL;  // 16-byte vector accesses
  return phe::launch_modswitch(d_in, d_out, count, from_bits, to_bits, S(stream));
}

int phe_decrypt_unpack(const phe_params *p, const uint8_t *d_S, const void *d_mask,
                       const void *d_body, int64_t T, int64_t rows, int32_t q_bits, int32_t *d_y,
                       void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (T < 0 || rows < 0) return PHE_EINVAL;
  if (q_bits != p->q_in && q_bits != p->q_out) return PHE_EMODULUS;
  if (T * rows == 0) return PHE_OK;
  if (!d_S || !d_mask || !d_body || !d_y) return PHE_EINVAL;
  const bool u64 = (q_bits == p->q_in);  // matmul_clear writes uint64 iff out_bits == q_in
  return phe::launch_decrypt(kp, d_S, d_mask, d_body, T * rows, q_bits, u64, d_y, S(stream));
}

// ------------------------------------------------------------------ host end-to-end
// Chunked pipelines over two workspace slots and two streams: chunk c runs H2D -> compute -> D2H
// on stream c%2 in slot c%2, so chunk c+1's copies overlap chunk c's kernels.  The device memory
// is the caller's (d_ws: two slots, sized by the matching *_ws_bytes query; SURVEY §8(b)
// ownership rule); the two streams and the ordering event are created per call on the current
// device and destroyed before returning, after both streams drained -- also on an error, so no
// copy touches the caller's host buffers once the call has returned.
struct HostPipe {
  cudaStream_t st[2] = {nullptr, nullptr};
  cudaEvent_t ev = nullptr;
  int start(cudaStream_t caller) {
    for (int s = 0; s < 2; s++)
      if (cudaStreamCreateWithFlags(&st[s], cudaStreamNonBlocking) != cudaSuccess)
        return phe_set_cuda_error(cudaGetLastError());
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
    // order after work already queued on the caller's stream (weight registration, the
    // workspace allocation of a stream-ordered allocator)
    if (cudaEventRecord(ev, caller) != cudaSuccess) return phe_set_cuda_error(cudaGetLastError());
    cudaStreamWaitEvent(st[0], ev, 0);
    cudaStreamWaitEvent(st[1], ev, 0);
    return PHE_OK;
  }
  // drain both streams (always), release them, and report the first failure
  int finish(int rc) {
    cudaError_t e0 = st[0] ? cudaStreamSynchronize(st[0]) : cudaSuccess;
    cudaError_t e1 = st[1] ? cudaStreamSynchronize(st[1]) : cudaSuccess;
    release();
    if (rc) return rc;
    if (e0 != cudaSuccess) return phe_set_cuda_error(e0);
    if (e1 != cudaSuccess) return phe_set_cuda_error(e1);
    cudaError_t e = cudaGetLastError();
    return e != cudaSuccess ? phe_set_cuda_error(e) : PHE_OK;
  }
  void release() {
    for (int s = 0; s < 2; s++)
      if (st[s]) { cudaStreamDestroy(st[s]); st[s] = nullptr; }
    if (ev) { cudaEventDestroy(ev); ev = nullptr; }
  }
  ~HostPipe() { release(); }
};

// sequential carving of one workspace slot
struct Carve {
  uint8_t *base;
  size_t off = 0;
  void *take(size_t bytes) {
    void *r = base + off;
    off += bytes;
    return r;
  }
};

static inline int64_t host_chunk(int64_t T, int64_t chunk_tokens) { return chunk_tokens < T ? chunk_tokens : T; }

// slot of phe_server_matvec_host: seeds, bodies, operand, uint32 mask and body outputs
struct MatvecSlot {
  size_t seeds, body, op, om, ob;
  size_t total() const { return seeds + body + op + om + ob; }
};
static MatvecSlot matvec_slot(const phe_params *p, int64_t L, int64_t R, int64_t C) {
  const int64_t N = p->N;
  return {(size_t)round_up(C * L * 8, 256), (size_t)round_up(C * L * N * 8, 256),
          (size_t)round_up((int64_t)phe_ct_operand_bytes(p, C, L), 256), (size_t)round_up(C * R * N * 4, 256),
          (size_t)round_up(C * R * 4, 256)};
}

size_t phe_server_matvec_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose,
                                       int64_t row_begin, int64_t row_end, int64_t T, int64_t chunk_tokens) {
  if (!p || phe_params_validate(p) || d_out < 1 || d_in < 1 || T < 1 || chunk_tokens < 1) return 0;
  const int64_t cols = transpose ? d_out : d_in, R = row_end - row_begin;
  if (R < 1) return 0;
  return 2 * matvec_slot(p, phe_num_blocks(p, cols), R, host_chunk(T, chunk_tokens)).total();
}

int phe_server_matvec_host(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                           int transpose, int64_t row_begin, int64_t row_end,
                           const uint64_t *h_seeds, const uint64_t *h_body, int64_t T,
                           int64_t chunk_tokens, uint32_t *h_out_mask, uint32_t *h_out_body,
                           void *d_ws, size_t ws_bytes, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (rows < 1 || cols < 1 || T < 0 || chunk_tokens < 1) return PHE_EINVAL;
  if (row_begin < 0 || row_end > rows || row_begin > row_end) return PHE_EINVAL;
  if (T == 0 || row_end == row_begin) return PHE_OK;
  if (!d_wprep || !h_seeds || !h_body || !h_out_mask || !h_out_body || !d_ws) return PHE_EINVAL;
  const int64_t N = p->N, L = phe_num_blocks(p, cols), R = row_end - row_begin;
  const int64_t C = host_chunk(T, chunk_tokens);
  const MatvecSlot sl = matvec_slot(p, L, R, C);
  const size_t slot = sl.total();
  if (ws_bytes < 2 * slot) return PHE_ENOMEM;
  HostPipe pipe;
  rc = pipe.start(S(stream));
  int64_t c = 0;
  for (int64_t t0 = 0; !rc && t0 < T; t0 += C, c++) {
    const int64_t n = (T - t0) < C ? (T - t0) : C;
    cudaStream_t st = pipe.st[c & 1];
    Carve cv{static_cast<uint8_t *>(d_ws) + (c & 1) * slot};
    uint64_t *d_seeds = static_cast<uint64_t *>(cv.take(sl.seeds));
    uint64_t *d_bod = static_cast<uint64_t *>(cv.take(sl.body));
    void *d_op = cv.take(sl.op);
    uint32_t *d_om = static_cast<uint32_t *>(cv.take(sl.om));
    uint32_t *d_ob = static_cast<uint32_t *>(cv.take(sl.ob));
    cudaMemcpyAsync(d_seeds, h_seeds + t0 * L, n * L * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_bod, h_body + t0 * L * N, n * L * N * 8, cudaMemcpyHostToDevice, st);
    rc = phe_ct_prepare(p, d_seeds, d_bod, n, L, d_op, sl.op, st);
    if (!rc) rc = matmul_common(p, d_wprep, rows, cols, row_begin, row_end, d_op, n, p->q_out, d_om, d_ob, st);
    if (rc) break;
    cudaMemcpyAsync(h_out_mask + t0 * R * N, d_om, n * R * N * 4, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(h_out_body + t0 * R, d_ob, n * R * 4, cudaMemcpyDeviceToHost, st);
  }
  return pipe.finish(rc);
}

}  // extern "C"

// ------------------------------------------------------------------ NEXT #1: packing
static inline int ks_spt(int ell) { return 256 / ell; }
static inline int64_t ks_kpad(const phe_params *p) {
  int spt = ks_spt((p->q_in + 7) / 8);
  return (p->N + spt - 1) / spt * spt;
}
static inline int64_t ks_plane_rows(const phe_params *p) {
  int ell = (p->q_in + 7) / 8, spt = ks_spt(ell);
  int64_t n_tiles = 2 * ks_kpad(p) / spt;
  return round_up(n_tiles * spt * ell + 1, 256);
}
static int check_pack(const phe_params *p, KParams *kp) {
  int rc = check_gpu(p, kp);
  if (rc) return rc;
  if (p->q_in < phe::KS_BITS || (kp->ell != 4 && kp->ell != 5) || p->N % 256) return PHE_EUNSUPPORTED;
  return PHE_OK;
}

extern "C" {

size_t phe_ksk_bytes(const phe_params *p) {
  return p ? (size_t)2 * phe::KS_LEVELS * p->N * (size_t)p->N * 8 : 0;
}

int phe_ksk_gen(const phe_params *p, const uint8_t *d_S, uint64_t ksk_seed, void *d_ksk, size_t bytes,
                void *stream) {
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  if (!d_S || !d_ksk) return PHE_EINVAL;
  if (bytes < phe_ksk_bytes(p)) return PHE_ENOMEM;
  uint64_t *KA = static_cast<uint64_t *>(d_ksk), *KB = KA + (int64_t)phe::KS_LEVELS * p->N * p->N;
  return phe::launch_ksk_gen(kp, d_S, ksk_seed, KA, KB, S(stream));
}

size_t phe_ksk_prep_bytes(const phe_params *p) {
  return p ? (size_t)ks_plane_rows(p) * phe::KS_LEVELS * (size_t)p->N : 0;
}

int phe_ksk_prepare(const phe_params *p, const void *d_ksk, void *d_kprep, size_t bytes, void *stream) {
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  if (!d_ksk || !d_kprep) return PHE_EINVAL;
  if (bytes < phe_ksk_prep_bytes(p)) return PHE_ENOMEM;
  return phe::launch_ksk_planes(kp, static_cast<const uint64_t *>(d_ksk), (int)ks_kpad(p), ks_plane_rows(p),
                                static_cast<uint8_t *>(d_kprep), S(stream));
}

size_t phe_packed_ws_bytes(const phe_params *p, int64_t rows, int64_t T) {
  if (!p || rows < 1 || T < 0) return 0;
  const int64_t N = p->N, rp = round_up(rows, 256), G = (rows + N - 1) / N;
  return (size_t)(round_up(T * rp * phe::KS_LEVELS * N, 256) + round_up(T * rows * 8, 256) +
                  round_up(T * G * 2 * N * 8, 256));
}

int phe_matmul_clear_digits(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                            int transpose, const void *d_operand, int64_t T, void *d_digits,
                            uint64_t *d_body, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  if (d_out < 1 || d_in < 1 || T < 0 || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_wprep || !d_operand || !d_digits || !d_body) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  const int64_t N = p->N, rp = round_up(rows, 256);
  uint8_t *digits = static_cast<uint8_t *>(d_digits);
  cudaStream_t st = S(stream);
  int launches = 0;
  rc = matmul_common(p, d_wprep, rows, cols, 0, rows, d_operand, T, p->q_in, nullptr, d_body, stream);
  if (rc) return rc;
  launches += g_last_launches;
  if (rp > rows) {  // zero digit rows of the 256-row padding (they contribute nothing)
    const int64_t KL = phe::KS_LEVELS * N;
    if (cudaMemset2DAsync(digits + rows * KL, (size_t)(rp * KL), 0, (size_t)((rp - rows) * KL),
                          (size_t)T, st) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
  }
  const int64_t Lc = phe_num_blocks(p, cols);
  phe::GemmArgs a{};
  a.kp = kp;
  a.wexp = static_cast<const uint8_t *>(d_wprep);
  a.wplain = reinterpret_cast<const int8_t *>(a.wexp + rows * Lc * 2 * N * 16);
  a.rows = rows; a.wplain_rows = round_up(rows, 128); a.op_rows = op_rows(T, kp.ell);
  a.Lc = Lc; a.cols = cols; a.row_begin = 0; a.row_end = rows;
  a.mplanes = static_cast<const uint8_t *>(d_operand);
  a.bplanes = a.mplanes + a.op_rows * Lc * N;
  a.T = T; a.out_bits = p->q_in; a.out_mask = digits; a.out_body = nullptr;
  a.digits = 1; a.digit_rows = rp;
  int n = 0;
  rc = phe::launch_limb_gemm(a, st, &n);
  if (rc) return rc;
  g_last_launches = launches + n;
  return PHE_OK;
}

size_t phe_pack_acc_bytes(const phe_params *p, int64_t rows, int64_t T) {
  if (!p || rows < 1 || T < 0) return 0;
  const int64_t G = (rows + p->N - 1) / p->N;
  return (size_t)(T * G * 2 * p->N * 8);
}

int phe_pack(const phe_params *p, const void *d_digits, const uint64_t *d_body, int64_t T, int64_t rows,
             const void *d_kprep, void *d_acc, size_t acc_bytes, uint32_t *d_out_packed, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  if (rows < 1 || T < 0) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_digits || !d_body || !d_kprep || !d_acc || !d_out_packed) return PHE_EINVAL;
  if (acc_bytes < phe_pack_acc_bytes(p, rows, T)) return PHE_ENOMEM;
  const int64_t N = p->N, rp = round_up(rows, 256), G = (rows + N - 1) / N;
  cudaStream_t st = S(stream);
  if (cudaMemsetAsync(d_acc, 0, (size_t)(T * G * 2 * N * 8), st) != cudaSuccess)
    return phe_set_cuda_error(cudaGetLastError());
  phe::PackArgs pa{};
  pa.N = (int)N; pa.ell = kp.ell; pa.T = T; pa.rows_pad = rp; pa.G = (int)G;
  pa.digits = static_cast<const uint8_t *>(d_digits);
  pa.kplanes = static_cast<const uint8_t *>(d_kprep);
  pa.kplane_rows = ks_plane_rows(p);
  pa.acc = d_acc;
  rc = phe::launch_pack_gemm(pa, st);
  if (rc) return rc;
  rc = phe::launch_pack_finalize(kp, d_acc, d_body, T, rows, (int)G, d_out_packed, st);
  if (rc) return rc;
  g_last_launches = 2;
  return PHE_OK;
}

int phe_matmul_clear_packed(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                            int transpose, const void *d_operand, int64_t T, const void *d_kprep,
                            void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  if (d_out < 1 || d_in < 1 || T < 0 || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_wprep || !d_operand || !d_kprep || !d_ws || !d_out_packed) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out;
  if (ws_bytes < phe_packed_ws_bytes(p, rows, T)) return PHE_ENOMEM;
  const int64_t N = p->N, rp = round_up(rows, 256);
  uint8_t *digits = static_cast<uint8_t *>(d_ws);
  uint64_t *body = reinterpret_cast<uint64_t *>(digits + round_up(T * rp * phe::KS_LEVELS * N, 256));
  void *acc = reinterpret_cast<uint8_t *>(body) + round_up(T * rows * 8, 256);
  // (1) LWE outputs of Eq. 6: body at q_in, masks as Decomp digits (Eq. 8's left operand)
  rc = phe_matmul_clear_digits(p, d_wprep, d_out, d_in, transpose, d_operand, T, digits, body, stream);
  if (rc) return rc;
  const int l1 = g_last_launches;
  // (2) Eq. 8 + Eq. 7 (KeySwitch GEMM, Rotate, sum), (0, b) - ..., ModulusSwitch to q_out
  rc = phe_pack(p, digits, body, T, rows, d_kprep, acc, phe_pack_acc_bytes(p, rows, T), d_out_packed, stream);
  if (rc) return rc;
  g_last_launches += l1;
  return PHE_OK;
}

int phe_decrypt_packed(const phe_params *p, const uint8_t *d_S, const uint32_t *d_packed, int64_t T,
                       int64_t rows, int32_t q_bits, int32_t *d_y, void *stream) {
  KParams kp;
  int rc = check_gpu(p, &kp);
  if (rc) return rc;
  if (T < 0 || rows < 0 || q_bits < 1 || q_bits > 32) return PHE_EINVAL;
  if (T * rows == 0) return PHE_OK;
  if (!d_S || !d_packed || !d_y) return PHE_EINVAL;
  const int64_t G = (rows + p->N - 1) / p->N;
  return phe::launch_decrypt_packed(kp, d_S, d_packed, T, rows, (int)G, q_bits, d_y, S(stream));
}

}  // extern "C"

// slot of phe_server_matvec_packed_host: seeds, bodies, operand, packing workspace, packed outputs.
// The packing workspace is not monotone in T (the K-split follows wave fill), so it is sized for
// both the full chunk and the ragged last one.
struct PackedSlot {
  size_t seeds, body, op, ws, out;
  size_t total() const { return seeds + body + op + ws + out; }
};
static PackedSlot packed_slot(const phe_params *p, int64_t rows, int64_t L, int64_t C, int64_t tail) {
  const int64_t N = p->N, G = (rows + N - 1) / N;
  int64_t ws = (int64_t)phe_packed_ws_bytes(p, rows, C);
  if (tail > 0 && (int64_t)phe_packed_ws_bytes(p, rows, tail) > ws) ws = (int64_t)phe_packed_ws_bytes(p, rows, tail);
  return {(size_t)round_up(C * L * 8, 256), (size_t)round_up(C * L * N * 8, 256),
          (size_t)round_up((int64_t)phe_ct_operand_bytes(p, C, L), 256), (size_t)round_up(ws, 256),
          (size_t)round_up(C * G * 2 * N * 4, 256)};
}

extern "C" size_t phe_server_matvec_packed_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in,
                                                         int transpose, int64_t T, int64_t chunk_tokens) {
  if (!p || phe_params_validate(p) || d_out < 1 || d_in < 1 || T < 1 || chunk_tokens < 1) return 0;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in, C = host_chunk(T, chunk_tokens);
  return 2 * packed_slot(p, rows, phe_num_blocks(p, cols), C, T % C).total();
}

extern "C" int phe_server_matvec_packed_host(const phe_params *p, const void *d_wprep, int64_t d_out,
                                             int64_t d_in, int transpose, const void *d_kprep,
                                             const uint64_t *h_seeds, const uint64_t *h_body, int64_t T,
                                             int64_t chunk_tokens, uint32_t *h_out_packed, void *d_ws,
                                             size_t ws_bytes, void *stream) {
  KParams kp;
  int rc = check_pack(p, &kp);
  if (rc) return rc;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (rows < 1 || cols < 1 || T < 0 || chunk_tokens < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_wprep || !d_kprep || !h_seeds || !h_body || !h_out_packed || !d_ws) return PHE_EINVAL;
  const int64_t N = p->N, L = phe_num_blocks(p, cols), G = (rows + N - 1) / N;
  const int64_t C = host_chunk(T, chunk_tokens);
  const PackedSlot sl = packed_slot(p, rows, L, C, T % C);
  const size_t slot = sl.total();
  if (ws_bytes < 2 * slot) return PHE_ENOMEM;
  HostPipe pipe;
  rc = pipe.start(S(stream));
  int64_t c = 0;
  for (int64_t t0 = 0; !rc && t0 < T; t0 += C, c++) {
    const int64_t n = (T - t0) < C ? (T - t0) : C;
    cudaStream_t st = pipe.st[c & 1];
    Carve cv{static_cast<uint8_t *>(d_ws) + (c & 1) * slot};
    uint64_t *d_seeds = static_cast<uint64_t *>(cv.take(sl.seeds));
    uint64_t *d_bod = static_cast<uint64_t *>(cv.take(sl.body));
    void *d_op = cv.take(sl.op);
    void *d_wsp = cv.take(sl.ws);
    uint32_t *d_o = static_cast<uint32_t *>(cv.take(sl.out));
    cudaMemcpyAsync(d_seeds, h_seeds + t0 * L, n * L * 8, cudaMemcpyHostToDevice, st);
    cudaMemcpyAsync(d_bod, h_body + t0 * L * N, n * L * N * 8, cudaMemcpyHostToDevice, st);
    rc = phe_ct_prepare(p, d_seeds, d_bod, n, L, d_op, sl.op, st);
    if (!rc) rc = phe_matmul_clear_packed(p, d_wprep, d_out, d_in, transpose, d_op, n, d_kprep, d_wsp, sl.ws, d_o, st);
    if (rc) break;
    cudaMemcpyAsync(h_out_packed + t0 * G * 2 * N, d_o, n * G * 2 * N * 4, cudaMemcpyDeviceToHost, st);
  }
  return pipe.finish(rc);
}

// ------------------------------------------------------------------ NEXT #2: wire format
static int check_wire(const phe_params *p, KParams *kp) {
  int rc = check_gpu(p, kp);
  if (rc) return rc;
  if (p->q_in > 57 || p->N % 64) return PHE_EUNSUPPORTED;  // whole 64-bit stream words per segment
  return PHE_OK;
}

extern "C" {

size_t phe_wire_input_bytes(const phe_params *p) {
  return p ? (size_t)(8 + (int64_t)p->N * p->q_in / 8) : 0;
}
size_t phe_wire_output_bytes(const phe_params *p) {
  return p ? (size_t)(2 * (int64_t)p->N * p->q_out / 8) : 0;
}

int phe_wire_serialize_inputs(const phe_params *p, const uint64_t *d_seeds, const uint64_t *d_body, int64_t T,
                              int64_t L, uint8_t *d_wire, void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (T < 0 || L < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_seeds || !d_body || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  return phe::launch_wire_inputs(kp, const_cast<uint64_t *>(d_seeds), const_cast<uint64_t *>(d_body), T * L, d_wire, 0,
                                 S(stream));
}

int phe_wire_deserialize_inputs(const phe_params *p, const uint8_t *d_wire, int64_t T, int64_t L,
                                uint64_t *d_seeds, uint64_t *d_body, void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (T < 0 || L < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_seeds || !d_body || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  return phe::launch_wire_inputs(kp, d_seeds, d_body, T * L, const_cast<uint8_t *>(d_wire), 1, S(stream));
}

int phe_wire_serialize_packed(const phe_params *p, const uint32_t *d_packed, int64_t n_ct, uint8_t *d_wire,
                              void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (n_ct < 0) return PHE_EINVAL;
  if (n_ct == 0) return PHE_OK;
  if (!d_packed || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  return phe::launch_wire_packed(kp, const_cast<uint32_t *>(d_packed), n_ct, d_wire, 0, S(stream));
}

int phe_wire_deserialize_packed(const phe_params *p, const uint8_t *d_wire, int64_t n_ct, uint32_t *d_packed,
                                void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (n_ct < 0) return PHE_EINVAL;
  if (n_ct == 0) return PHE_OK;
  if (!d_packed || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  return phe::launch_wire_packed(kp, d_packed, n_ct, const_cast<uint8_t *>(d_wire), 1, S(stream));
}

// The server step as the network sees it (Fig. 1): wire-format input blocks in (9992 B each at
// Table 1), wire-format packed ciphertexts out (13312 B each).  Chunked, two streams.
// mode 0: tensor-core stage 1 + packing GEMM; 1: tensor-core stage 1 + NTT-domain packing;
// 2: NTT-domain stage 1 (d_tables, NTT weights, NTT operand) + NTT-domain packing.
struct WireSlot {
  size_t win, seeds, body, op, ws, pk, wout;
  size_t total() const { return win + seeds + body + op + ws + pk + wout; }
};
static size_t wire_pack_ws(const phe_params *p, int64_t rows, int64_t n, int mode) {
  return mode >= 1 ? phe_packed_ntt_ws_bytes(p, rows, n) : phe_packed_ws_bytes(p, rows, n);
}
static WireSlot wire_slot(const phe_params *p, int64_t rows, int64_t L, int64_t C, int64_t tail, int mode) {
  const int64_t N = p->N, G = (rows + N - 1) / N;
  const int64_t bin = (int64_t)phe_wire_input_bytes(p), bout = (int64_t)phe_wire_output_bytes(p);
  const size_t op = mode == 2 ? phe_ntt_operand_bytes(p, C, L) : phe_ct_operand_bytes(p, C, L);
  size_t ws = wire_pack_ws(p, rows, C, mode);  // not monotone in T: full and ragged chunk
  if (tail > 0 && wire_pack_ws(p, rows, tail, mode) > ws) ws = wire_pack_ws(p, rows, tail, mode);
  return {(size_t)round_up(C * L * bin, 256), (size_t)round_up(C * L * 8, 256), (size_t)round_up(C * L * N * 8, 256),
          op ? (size_t)round_up((int64_t)op, 256) : 0, (size_t)round_up((int64_t)ws, 256),
          (size_t)round_up(C * G * 2 * N * 4, 256), (size_t)round_up(C * G * bout, 256)};
}
static size_t server_wire_host_ws(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                  int64_t chunk_tokens, int mode) {
  if (!p || phe_params_validate(p) || d_out < 1 || d_in < 1 || T < 1 || chunk_tokens < 1) return 0;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in, C = host_chunk(T, chunk_tokens);
  const WireSlot sl = wire_slot(p, rows, phe_num_blocks(p, cols), C, T % C, mode);
  return sl.op ? 2 * sl.total() : 0;
}

static int server_wire_host_impl(const phe_params *p, const void *d_tables, const void *d_wprep, int64_t d_out,
                                 int64_t d_in, int transpose, const void *d_kprep, const uint8_t *h_wire_in,
                                 int64_t T, int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes,
                                 void *stream, int mode) {
  const bool ntt_pack = mode >= 1, ntt_s1 = mode == 2;
  if (ntt_s1 && !d_tables) return PHE_EINVAL;
  KParams kp;
  int rc = check_pack(p, &kp);
  if (!rc) rc = check_wire(p, &kp);
  if (!rc && ntt_pack && !phe::ntt_ks_supported(kp)) rc = PHE_EUNSUPPORTED;
  if (rc) return rc;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (rows < 1 || cols < 1 || T < 0 || chunk_tokens < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_wprep || !d_kprep || !h_wire_in || !h_wire_out || !d_ws) return PHE_EINVAL;
  const int64_t L = phe_num_blocks(p, cols), G = (rows + p->N - 1) / p->N;
  const int64_t bin = (int64_t)phe_wire_input_bytes(p), bout = (int64_t)phe_wire_output_bytes(p);
  const int64_t C = host_chunk(T, chunk_tokens);
  const WireSlot sl = wire_slot(p, rows, L, C, T % C, mode);
  if (sl.op == 0) return PHE_EUNSUPPORTED;
  const size_t slot = sl.total();
  if (ws_bytes < 2 * slot) return PHE_ENOMEM;
  HostPipe pipe;
  rc = pipe.start(S(stream));
  int64_t c = 0;
  for (int64_t t0 = 0; !rc && t0 < T; t0 += C, c++) {
    const int64_t n = (T - t0) < C ? (T - t0) : C;
    cudaStream_t st = pipe.st[c & 1];
    Carve cv{static_cast<uint8_t *>(d_ws) + (c & 1) * slot};
    uint8_t *d_win = static_cast<uint8_t *>(cv.take(sl.win));
    uint64_t *d_seeds = static_cast<uint64_t *>(cv.take(sl.seeds));
    uint64_t *d_bod = static_cast<uint64_t *>(cv.take(sl.body));
    void *d_op = cv.take(sl.op);
    void *d_wsp = cv.take(sl.ws);
    uint32_t *d_pk = static_cast<uint32_t *>(cv.take(sl.pk));
    uint8_t *d_wout = static_cast<uint8_t *>(cv.take(sl.wout));
    cudaMemcpyAsync(d_win, h_wire_in + t0 * L * bin, n * L * bin, cudaMemcpyHostToDevice, st);
    rc = phe_wire_deserialize_inputs(p, d_win, n, L, d_seeds, d_bod, st);
    if (!rc)
      rc = ntt_s1 ? phe_ntt_ct_prepare(p, d_tables, d_seeds, d_bod, n, L, d_op, sl.op, st)
                  : phe_ct_prepare(p, d_seeds, d_bod, n, L, d_op, sl.op, st);
    if (!rc)
      rc = ntt_s1 ? phe_matmul_clear_packed_nttw(p, d_tables, d_wprep, d_out, d_in, transpose, d_op, n, d_kprep, d_wsp,
                                                 sl.ws, d_pk, st)
           : ntt_pack ? phe_matmul_clear_packed_ntt(p, d_wprep, d_out, d_in, transpose, d_op, n, d_kprep, d_wsp, sl.ws,
                                                    d_pk, st)
                      : phe_matmul_clear_packed(p, d_wprep, d_out, d_in, transpose, d_op, n, d_kprep, d_wsp, sl.ws,
                                                d_pk, st);
    if (!rc) rc = phe_wire_serialize_packed(p, d_pk, n * G, d_wout, st);
    if (rc) break;
    cudaMemcpyAsync(h_wire_out + t0 * G * bout, d_wout, n * G * bout, cudaMemcpyDeviceToHost, st);
  }
  return pipe.finish(rc);
}

size_t phe_server_wire_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                     int64_t chunk_tokens) {
  return server_wire_host_ws(p, d_out, d_in, transpose, T, chunk_tokens, 0);
}
size_t phe_server_wire_host_ntt_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                         int64_t chunk_tokens) {
  return server_wire_host_ws(p, d_out, d_in, transpose, T, chunk_tokens, 1);
}
size_t phe_server_wire_host_nttw_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose, int64_t T,
                                          int64_t chunk_tokens) {
  return server_wire_host_ws(p, d_out, d_in, transpose, T, chunk_tokens, 2);
}
int phe_server_wire_host(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                         const void *d_kprep, const uint8_t *h_wire_in, int64_t T, int64_t chunk_tokens,
                         uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream) {
  return server_wire_host_impl(p, nullptr, d_wprep, d_out, d_in, transpose, d_kprep, h_wire_in, T, chunk_tokens,
                               h_wire_out, d_ws, ws_bytes, stream, 0);
}
int phe_server_wire_host_ntt(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                             const void *d_nksk, const uint8_t *h_wire_in, int64_t T, int64_t chunk_tokens,
                             uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream) {
  return server_wire_host_impl(p, nullptr, d_wprep, d_out, d_in, transpose, d_nksk, h_wire_in, T, chunk_tokens,
                               h_wire_out, d_ws, ws_bytes, stream, 1);
}
int phe_server_wire_host_nttw(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                              int64_t d_in, int transpose, const void *d_nksk, const uint8_t *h_wire_in, int64_t T,
                              int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes, void *stream) {
  return server_wire_host_impl(p, d_tables, d_nttw, d_out, d_in, transpose, d_nksk, h_wire_in, T, chunk_tokens,
                               h_wire_out, d_ws, ws_bytes, stream, 2);
}

// ================================================================ LWE outputs on the wire
static inline int64_t lwe_seg_words(const phe_params *p) { return (int64_t)p->N * p->q_out / 64; }
static inline int64_t lwe_body_words(const phe_params *p, int64_t R) { return (R * p->q_out + 63) / 64; }

extern "C" {

size_t phe_wire_lwe_bytes(const phe_params *p, int64_t R) {
  if (!p || R < 1 || p->N % 64) return 0;
  return (size_t)(8 * (R * lwe_seg_words(p) + lwe_body_words(p, R)));
}

int phe_wire_serialize_lwe(const phe_params *p, const uint32_t *d_mask, const uint32_t *d_body, int64_t T,
                           int64_t R, uint8_t *d_wire, void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (T < 0 || R < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_mask || !d_body || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  const int64_t tw = (int64_t)phe_wire_lwe_bytes(p, R) / 8, sw = lwe_seg_words(p);
  rc = phe::launch_wire_u32(const_cast<uint32_t *>(d_mask), T * R, p->N, p->q_out, d_wire, sw, R, tw, 0, 0,
                            S(stream));
  if (rc) return rc;
  return phe::launch_wire_u32(const_cast<uint32_t *>(d_body), T, (int)R, p->q_out, d_wire, lwe_body_words(p, R),
                              1, tw, R * sw, 0, S(stream));
}

int phe_wire_deserialize_lwe(const phe_params *p, const uint8_t *d_wire, int64_t T, int64_t R, uint32_t *d_mask,
                             uint32_t *d_body, void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (T < 0 || R < 1) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_mask || !d_body || !d_wire || ((uintptr_t)d_wire & 7)) return PHE_EINVAL;
  const int64_t tw = (int64_t)phe_wire_lwe_bytes(p, R) / 8, sw = lwe_seg_words(p);
  uint8_t *w = const_cast<uint8_t *>(d_wire);
  rc = phe::launch_wire_u32(d_mask, T * R, p->N, p->q_out, w, sw, R, tw, 0, 1, S(stream));
  if (rc) return rc;
  return phe::launch_wire_u32(d_body, T, (int)R, p->q_out, w, lwe_body_words(p, R), 1, tw, R * sw, 1, S(stream));
}

size_t phe_matmul_clear_wire_ws_bytes(const phe_params *p, int64_t T, int64_t R) {
  if (!p || T < 0 || R < 1) return 0;
  return (size_t)round_up(T * R * 4, 256);
}

// the fused wire form is supported iff the 2-CTA mask kernel runs (ell 4/5, N a multiple of 256),
// q_out <= 26 and the per-token record is a whole number of 16-byte units (TMA row stride)
static bool wire_direct_ok(const phe_params *p, int64_t R) {
  const int ell = (p->q_in + 7) / 8;
  if ((ell != 4 && ell != 5) || p->N % 256 || p->q_out > 26 || p->q_out < 16 || p->q_out == p->q_in) return false;
  return (phe_wire_lwe_bytes(p, R) % 16) == 0;
}
int phe_wire_lwe_direct_supported(const phe_params *p, int64_t R) {
  if (!p || phe_params_validate(p) || R < 1 || p->N % 64) return 0;
  return wire_direct_ok(p, R) ? 1 : 0;
}

int phe_matmul_clear_wire(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in, int transpose,
                          int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T, uint8_t *d_wire,
                          void *d_ws, size_t ws_bytes, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  if (transpose != 0 && transpose != 1) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (rows < 1 || cols < 1 || T < 0) return PHE_EINVAL;
  if (row_begin < 0 || row_end > rows || row_begin > row_end) return PHE_EINVAL;
  const int64_t R = row_end - row_begin;
  if (T == 0 || R == 0) return PHE_OK;
  if (!d_wprep || !d_operand || !d_wire || !d_ws) return PHE_EINVAL;
  if (!wire_direct_ok(p, R) || ((uintptr_t)d_wire & 15)) return PHE_EUNSUPPORTED;
  if (ws_bytes < phe_matmul_clear_wire_ws_bytes(p, T, R)) return PHE_ENOMEM;
  const int64_t N = p->N, Lc = phe_num_blocks(p, cols);
  phe::GemmArgs a{};
  a.kp = kp;
  a.wexp = static_cast<const uint8_t *>(d_wprep);
  a.wplain = reinterpret_cast<const int8_t *>(a.wexp + rows * Lc * 2 * N * 16);
  a.rows = rows;
  a.wplain_rows = round_up(rows, 128);
  a.op_rows = op_rows(T, kp.ell);
  a.Lc = Lc;
  a.cols = cols;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.mplanes = static_cast<const uint8_t *>(d_operand);
  a.bplanes = a.mplanes + a.op_rows * Lc * N;
  a.T = T;
  a.out_bits = p->q_out;
  a.out_mask = d_wire;
  a.out_body = d_ws;  // uint32 bodies [T][R], then packed into each record's tail
  a.wire_words = (int64_t)phe_wire_lwe_bytes(p, R) / 8;
  int n = 0;
  rc = phe::launch_limb_gemm(a, S(stream), &n);
  if (rc) return rc;
  rc = phe::launch_wire_u32(static_cast<uint32_t *>(d_ws), T, (int)R, p->q_out, d_wire, lwe_body_words(p, R), 1,
                            a.wire_words, R * lwe_seg_words(p), 0, S(stream));
  g_last_launches = n + 1;
  return rc;
}

// slot of phe_server_matvec_wire_host: wire inputs, seeds, bodies, operand, uint32 outputs, wire outputs
struct LweWireSlot {
  size_t win, seeds, body, op, om, ob, wout;
  size_t total() const { return win + seeds + body + op + om + ob + wout; }
};
// (with the fused wire epilogue -- phe_matmul_clear_wire -- no uint32 mask buffer is needed)
static LweWireSlot lwe_wire_slot(const phe_params *p, int64_t L, int64_t R, int64_t C) {
  const int64_t N = p->N, bin = (int64_t)phe_wire_input_bytes(p), bout = (int64_t)phe_wire_lwe_bytes(p, R);
  const bool direct = wire_direct_ok(p, R);
  return {(size_t)round_up(C * L * bin, 256), (size_t)round_up(C * L * 8, 256), (size_t)round_up(C * L * N * 8, 256),
          (size_t)round_up((int64_t)phe_ct_operand_bytes(p, C, L), 256),
          direct ? (size_t)0 : (size_t)round_up(C * R * N * 4, 256), (size_t)round_up(C * R * 4, 256),
          (size_t)round_up(C * bout, 256)};
}

size_t phe_server_matvec_wire_host_ws_bytes(const phe_params *p, int64_t d_out, int64_t d_in, int transpose,
                                            int64_t row_begin, int64_t row_end, int64_t T, int64_t chunk_tokens) {
  if (!p || phe_params_validate(p) || p->N % 64 || d_out < 1 || d_in < 1 || T < 1 || chunk_tokens < 1) return 0;
  const int64_t cols = transpose ? d_out : d_in, R = row_end - row_begin;
  if (R < 1) return 0;
  return 2 * lwe_wire_slot(p, phe_num_blocks(p, cols), R, host_chunk(T, chunk_tokens)).total();
}

int phe_server_matvec_wire_host(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                                int transpose, int64_t row_begin, int64_t row_end, const uint8_t *h_wire_in,
                                int64_t T, int64_t chunk_tokens, uint8_t *h_wire_out, void *d_ws, size_t ws_bytes,
                                void *stream) {
  KParams kp;
  int rc = check_wire(p, &kp);
  if (rc) return rc;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (rows < 1 || cols < 1 || T < 0 || chunk_tokens < 1) return PHE_EINVAL;
  if (row_begin < 0 || row_end > rows || row_begin > row_end) return PHE_EINVAL;
  if (T == 0 || row_end == row_begin) return PHE_OK;
  if (!d_wprep || !h_wire_in || !h_wire_out || !d_ws) return PHE_EINVAL;
  const int64_t L = phe_num_blocks(p, cols), R = row_end - row_begin;
  const int64_t C = host_chunk(T, chunk_tokens);
  const int64_t bin = (int64_t)phe_wire_input_bytes(p), bout = (int64_t)phe_wire_lwe_bytes(p, R);
  const LweWireSlot sl = lwe_wire_slot(p, L, R, C);
  const size_t slot = sl.total();
  if (ws_bytes < 2 * slot) return PHE_ENOMEM;
  HostPipe pipe;
  rc = pipe.start(S(stream));
  int64_t c = 0;
  for (int64_t t0 = 0; !rc && t0 < T; t0 += C, c++) {
    const int64_t n = (T - t0) < C ? (T - t0) : C;
    cudaStream_t st = pipe.st[c & 1];
    Carve cv{static_cast<uint8_t *>(d_ws) + (c & 1) * slot};
    uint8_t *d_win = static_cast<uint8_t *>(cv.take(sl.win));
    uint64_t *d_seeds = static_cast<uint64_t *>(cv.take(sl.seeds));
    uint64_t *d_bod = static_cast<uint64_t *>(cv.take(sl.body));
    void *d_op = cv.take(sl.op);
    uint32_t *d_om = static_cast<uint32_t *>(cv.take(sl.om));
    uint32_t *d_ob = static_cast<uint32_t *>(cv.take(sl.ob));
    uint8_t *d_wout = static_cast<uint8_t *>(cv.take(sl.wout));
    cudaMemcpyAsync(d_win, h_wire_in + t0 * L * bin, n * L * bin, cudaMemcpyHostToDevice, st);
    rc = phe_wire_deserialize_inputs(p, d_win, n, L, d_seeds, d_bod, st);
    if (!rc) rc = phe_ct_prepare(p, d_seeds, d_bod, n, L, d_op, sl.op, st);
    if (sl.om == 0) {  // the mask GEMM writes the wire record itself
      if (!rc) rc = phe_matmul_clear_wire(p, d_wprep, d_out, d_in, transpose, row_begin, row_end, d_op, n, d_wout, d_ob,
                                          sl.ob, st);
    } else {
      if (!rc) rc = matmul_common(p, d_wprep, rows, cols, row_begin, row_end, d_op, n, p->q_out, d_om, d_ob, st);
      if (!rc) rc = phe_wire_serialize_lwe(p, d_om, d_ob, n, R, d_wout, st);
    }
    if (rc) break;
    cudaMemcpyAsync(h_wire_out + t0 * bout, d_wout, n * bout, cudaMemcpyDeviceToHost, st);
  }
  return pipe.finish(rc);
}

}  // extern "C"

// ================================================================ NEXT #4: NTT-domain contraction
static int check_ntt(const phe_params *p, KParams *kp) {
  int rc = check_gpu(p, kp);
  if (rc) return rc;
  if (p->N < 512 || p->N > 8192) return PHE_EUNSUPPORTED;
  if (phe_ntt_max_blocks(p) < 1) return PHE_EUNSUPPORTED;
  return PHE_OK;
}

int phe_ntt_primes(uint32_t *out2) {
  if (!out2) return PHE_EINVAL;
  return phe::ntt_primes(out2);
}

int64_t phe_ntt_max_blocks(const phe_params *p) {
  if (phe_params_validate(p)) return 0;
  uint32_t pr[2];
  phe::ntt_primes(pr);
  // centred masks: |P'| <= maxP(L) = L N 2^(q_in-1) 128; the CRT needs Z(L) + maxP(L) < p0 p1 with
  // Z(L) = the least multiple of 2^q_in >= maxP(L) + 2 p0 (R23, ntt_path.cu crt_store)
  const unsigned __int128 M = (unsigned __int128)pr[0] * pr[1];
  const unsigned __int128 per = (unsigned __int128)p->N * ((unsigned __int128)1 << (p->q_in - 1)) * 128;
  const unsigned __int128 g = (unsigned __int128)1 << p->q_in;
  auto fits = [&](unsigned __int128 L) {
    const unsigned __int128 mp = L * per, Z = (mp + 2 * (unsigned __int128)pr[0] + g - 1) / g * g;
    return Z + mp < M;
  };
  unsigned __int128 L = M / (2 * per) + 1;
  if (L > 1000000) L = 1000000;
  while (L > 0 && !fits(L)) L--;
  return (int64_t)L;
}

size_t phe_ntt_tables_bytes(const phe_params *p) {
  if (!p || p->N < 16) return 0;
  return (size_t)(4 * p->N + 2 * 15 * (p->N / 16)) * 8;
}

int phe_ntt_tables_init(const phe_params *p, void *d_tables, size_t bytes, void *stream) {
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (!d_tables) return PHE_EINVAL;
  if (bytes < phe_ntt_tables_bytes(p)) return PHE_ENOMEM;
  return phe::launch_ntt_tables(kp, d_tables, S(stream));
}

size_t phe_ntt_weights_bytes(const phe_params *p, int64_t rows, int64_t cols) {
  if (!p || rows < 1 || cols < 1 || p->N < 1) return 0;
  const int64_t Lc = phe_num_blocks(p, cols);
  return (size_t)(rows * Lc * 2 * p->N * 4) + (size_t)(round_up(rows, 128) * Lc * p->N) +
         (size_t)round_up(rows, 16);
}

int phe_ntt_weights_prepare(const phe_params *p, const void *d_tables, const int8_t *d_W,
                            int64_t d_out, int64_t d_in, int transpose, void *d_nttw, size_t bytes,
                            void *stream) {
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (!d_tables || !d_W || !d_nttw || d_out < 1 || d_in < 1 || (transpose != 0 && transpose != 1))
    return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  if (bytes < phe_ntt_weights_bytes(p, rows, cols)) return PHE_ENOMEM;
  rc = phe::check_weights_range(d_W, d_out * d_in, static_cast<unsigned *>(d_nttw), S(stream));
  if (rc) return rc;
  const int64_t Lc = phe_num_blocks(p, cols);
  uint32_t *what = static_cast<uint32_t *>(d_nttw);
  rc = phe::launch_ntt_weights(kp, d_tables, d_W, d_out, d_in, transpose, what, S(stream));
  if (rc) return rc;
  int8_t *plain = reinterpret_cast<int8_t *>(what + rows * Lc * 2 * p->N);
  rc = phe::launch_weights_plain(kp, d_W, d_out, d_in, transpose, plain, S(stream));
  if (rc) return rc;
  uint8_t *par = reinterpret_cast<uint8_t *>(plain) + round_up(rows, 128) * Lc * p->N;
  return phe::launch_ntt_rowpar(d_W, d_out, d_in, transpose, par, S(stream));
}

size_t phe_ntt_operand_bytes(const phe_params *p, int64_t T, int64_t L) {
  if (!p || T < 0 || L < 1 || p->N < 1) return 0;
  const int ell = (p->q_in + 7) / 8;
  return (size_t)(T * L * 2 * p->N * 4) + (size_t)(op_rows(T, ell) * L * p->N);
}

int phe_ntt_ct_prepare(const phe_params *p, const void *d_tables, const uint64_t *d_seeds,
                       const uint64_t *d_body, int64_t T, int64_t L, void *d_operand, size_t bytes,
                       void *stream) {
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (T < 0 || L < 1 || !d_operand || !d_tables) return PHE_EINVAL;
  if (T > 0 && (!d_seeds || !d_body)) return PHE_EINVAL;
  if (bytes < phe_ntt_operand_bytes(p, T, L)) return PHE_ENOMEM;
  if (T == 0) return PHE_OK;
  uint32_t *ahat = static_cast<uint32_t *>(d_operand);
  rc = phe::launch_ntt_masks(kp, d_tables, d_seeds, T, L, ahat, S(stream));
  if (rc) return rc;
  uint8_t *bp = reinterpret_cast<uint8_t *>(ahat + T * L * 2 * p->N);
  return phe::launch_ct_prepare(kp, d_seeds, d_body, T, L, nullptr, bp, S(stream));
}

int phe_encrypt_pack_ntt(const phe_params *p, const void *d_tables, const uint8_t *d_S, const int8_t *d_x,
                         int64_t T, int64_t d_in, uint64_t seed_base, uint64_t noise_seed, uint64_t *d_seeds,
                         uint64_t *d_body, void *stream) {
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (T < 0 || d_in < 1) return PHE_EINVAL;
  if (T > 0 && (!d_tables || !d_S || !d_x || !d_seeds || !d_body)) return PHE_EINVAL;
  if (p->beta < 9) return PHE_ERANGE;
  // |A*S| < N 2^q_in must stay below p0 p1 / 2 for the centred CRT
  uint32_t pr[2];
  phe::ntt_primes(pr);
  if ((unsigned __int128)p->N << p->q_in >= ((unsigned __int128)pr[0] * pr[1]) / 2) return PHE_EUNSUPPORTED;
  return phe::launch_ntt_encrypt(kp, d_tables, d_S, d_x, T, d_in, phe_num_blocks(p, d_in), seed_base, noise_seed,
                                 d_seeds, d_body, S(stream));
}

static int ntt_common(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t rows,
                      int64_t cols, int64_t row_begin, int64_t row_end, const void *d_operand, int64_t T,
                      int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream,
                      int64_t out_rows = 0) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (rows < 1 || cols < 1 || T < 0) return PHE_EINVAL;
  if (row_begin < 0 || row_end > rows || row_begin > row_end) return PHE_EINVAL;
  if (out_bits != p->q_in && out_bits != p->q_out) return PHE_EMODULUS;
  const int64_t N = p->N, Lc = phe_num_blocks(p, cols);
  if (Lc > phe_ntt_max_blocks(p)) return PHE_EUNSUPPORTED;
  if (T == 0 || row_end == row_begin) return PHE_OK;
  if (!d_tables || !d_nttw || !d_operand || (!d_out_mask && !d_out_body)) return PHE_EINVAL;
  const uint32_t *what = static_cast<const uint32_t *>(d_nttw);
  const uint32_t *ahat = static_cast<const uint32_t *>(d_operand);
  int n = 0;
  if (d_out_body) {
    phe::GemmArgs a{};
    a.kp = kp;
    a.wexp = nullptr;
    a.wplain = reinterpret_cast<const int8_t *>(what + rows * Lc * 2 * N);
    a.rows = rows;
    a.wplain_rows = round_up(rows, 128);
    a.op_rows = op_rows(T, kp.ell);
    a.Lc = Lc;
    a.cols = cols;
    a.row_begin = row_begin;
    a.row_end = row_end;
    a.mplanes = nullptr;
    a.bplanes = reinterpret_cast<const uint8_t *>(ahat + T * Lc * 2 * N);
    a.T = T;
    a.out_bits = out_bits;
    a.out_mask = nullptr;
    a.out_body = d_out_body;
    a.out_rows = out_rows;
    rc = phe::launch_limb_gemm(a, S(stream), &n);
    if (rc) return rc;
  }
  if (d_out_mask) {
    const uint8_t *par = reinterpret_cast<const uint8_t *>(what + rows * Lc * 2 * N) +
                         round_up(rows, 128) * Lc * N;
    rc = phe::launch_ntt_mask(kp, d_tables, what, par, rows, Lc, row_begin, row_end, ahat, T, out_bits,
                              d_out_mask, S(stream), 0, out_rows);
    if (rc) return rc;
    n++;
  }
  g_last_launches = n;
  return PHE_OK;
}

int phe_matmul_clear_digits_ntt(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                                int64_t d_in, int transpose, const void *d_operand, int64_t T, void *d_digits,
                                uint64_t *d_body, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_ntt(p, &kp);
  if (rc) return rc;
  if (p->q_in < 32) return PHE_EUNSUPPORTED;  // Decomp keeps the top 32 bits (R18)
  if (d_out < 1 || d_in < 1 || T < 0 || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_tables || !d_nttw || !d_operand || !d_digits || !d_body) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  const int64_t N = p->N, rp = round_up(rows, 256), Lc = phe_num_blocks(p, cols);
  if (Lc > phe_ntt_max_blocks(p)) return PHE_EUNSUPPORTED;
  // bodies at q_in (the tcgen05 body GEMM, as phe_matmul_clear_digits)
  rc = ntt_common(p, d_tables, d_nttw, rows, cols, 0, rows, d_operand, T, p->q_in, nullptr, d_body, stream);
  if (rc) return rc;
  int launches = g_last_launches;
  uint8_t *digits = static_cast<uint8_t *>(d_digits);
  if (rp > rows) {  // zero digit rows of the 256-row padding (they contribute nothing)
    const int64_t KL = phe::KS_LEVELS * N;
    if (cudaMemset2DAsync(digits + rows * KL, (size_t)(rp * KL), 0, (size_t)((rp - rows) * KL), (size_t)T,
                          S(stream)) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
  }
  const uint32_t *what = static_cast<const uint32_t *>(d_nttw);
  const uint8_t *par = reinterpret_cast<const uint8_t *>(what + rows * Lc * 2 * N) + round_up(rows, 128) * Lc * N;
  rc = phe::launch_ntt_mask(kp, d_tables, what, par, rows, Lc, 0, rows, static_cast<const uint32_t *>(d_operand), T,
                            phe::KS_BITS, d_digits, S(stream), rp);
  if (rc) return rc;
  g_last_launches = launches + 1;
  return PHE_OK;
}

// NEXT #1 stage 2 in the NTT domain (ntt_keyswitch.cu)
static int check_ntt_ks(const phe_params *p, KParams *kp) {
  int rc = check_pack(p, kp);
  if (rc) return rc;
  return phe::ntt_ks_supported(*kp) ? PHE_OK : PHE_EUNSUPPORTED;
}

size_t phe_ntt_ksk_bytes(const phe_params *p) {
  KParams kp;
  if (!p || check_ntt_ks(p, &kp)) return 0;
  return phe::ntt_ks_bytes(kp);
}

int phe_ntt_ksk_prepare(const phe_params *p, const void *d_ksk, void *d_nksk, size_t bytes, void *stream) {
  KParams kp;
  int rc = check_ntt_ks(p, &kp);
  if (rc) return rc;
  if (!d_ksk || !d_nksk) return PHE_EINVAL;
  if (bytes < phe::ntt_ks_bytes(kp)) return PHE_ENOMEM;
  return phe::launch_ntt_ks_prepare(kp, static_cast<const uint64_t *>(d_ksk), d_nksk, S(stream));
}

size_t phe_pack_ntt_ws_bytes(const phe_params *p, int64_t rows, int64_t T) {
  KParams kp;
  if (!p || rows < 1 || T < 0 || check_ntt_ks(p, &kp)) return 0;
  return phe::ntt_ks_ws_bytes(kp, T, (rows + p->N - 1) / p->N);
}

int phe_pack_ntt(const phe_params *p, const void *d_digits, const uint64_t *d_body, int64_t T, int64_t rows,
                 const void *d_nksk, void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_ntt_ks(p, &kp);
  if (rc) return rc;
  if (rows < 1 || T < 0) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_digits || !d_body || !d_nksk || !d_ws || !d_out_packed) return PHE_EINVAL;
  if (ws_bytes < phe_pack_ntt_ws_bytes(p, rows, T)) return PHE_ENOMEM;
  const int64_t G = (rows + p->N - 1) / p->N;
  // the CRT-recovered sum, then the packing GEMM path's own finish ((0, b) - acc, switch)
  const size_t partb = phe::ntt_ks_ws_bytes(kp, T, G) - (size_t)T * G * 2 * p->N * 8;
  void *acc = static_cast<uint8_t *>(d_ws) + partb;
  rc = phe::launch_ntt_ks(kp, d_nksk, static_cast<const int8_t *>(d_digits), T, rows, d_ws, acc, S(stream));
  if (rc) return rc;
  rc = phe::launch_pack_finalize(kp, acc, d_body, T, rows, (int)G, d_out_packed, S(stream));
  if (rc) return rc;
  g_last_launches = 3;
  return PHE_OK;
}

size_t phe_packed_ntt_ws_bytes(const phe_params *p, int64_t rows, int64_t T) {
  KParams kp;
  if (!p || rows < 1 || T < 0 || check_ntt_ks(p, &kp)) return 0;
  const int64_t N = p->N, rp = round_up(rows, 256);
  return (size_t)(round_up(T * rp * phe::KS_LEVELS * N, 256) + round_up(T * rows * 8, 256)) +
         phe_pack_ntt_ws_bytes(p, rows, T);
}

int phe_matmul_clear_packed_ntt(const phe_params *p, const void *d_wprep, int64_t d_out, int64_t d_in,
                                int transpose, const void *d_operand, int64_t T, const void *d_nksk,
                                void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_ntt_ks(p, &kp);
  if (rc) return rc;
  if (d_out < 1 || d_in < 1 || T < 0 || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_wprep || !d_operand || !d_nksk || !d_ws || !d_out_packed) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out;
  if (ws_bytes < phe_packed_ntt_ws_bytes(p, rows, T)) return PHE_ENOMEM;
  const int64_t N = p->N, rp = round_up(rows, 256);
  uint8_t *digits = static_cast<uint8_t *>(d_ws);
  uint64_t *body = reinterpret_cast<uint64_t *>(digits + round_up(T * rp * phe::KS_LEVELS * N, 256));
  void *ws2 = reinterpret_cast<uint8_t *>(body) + round_up(T * rows * 8, 256);
  // (1) Eq. 6 on the tensor cores, masks written as Decomp digits; (2) Eq. 7/8 in the NTT domain
  rc = phe_matmul_clear_digits(p, d_wprep, d_out, d_in, transpose, d_operand, T, digits, body, stream);
  if (rc) return rc;
  const int l1 = g_last_launches;
  rc = phe_pack_ntt(p, digits, body, T, rows, d_nksk, ws2, phe_pack_ntt_ws_bytes(p, rows, T), d_out_packed, stream);
  if (rc) return rc;
  g_last_launches += l1;
  return PHE_OK;
}

int phe_matmul_clear_packed_nttw(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                                 int64_t d_in, int transpose, const void *d_operand, int64_t T, const void *d_nksk,
                                 void *d_ws, size_t ws_bytes, uint32_t *d_out_packed, void *stream) {
  g_last_launches = 0;
  KParams kp;
  int rc = check_ntt_ks(p, &kp);
  if (rc) return rc;
  if (d_out < 1 || d_in < 1 || T < 0 || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (T == 0) return PHE_OK;
  if (!d_tables || !d_nttw || !d_operand || !d_nksk || !d_ws || !d_out_packed) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out;
  if (ws_bytes < phe_packed_ntt_ws_bytes(p, rows, T)) return PHE_ENOMEM;
  const int64_t N = p->N, rp = round_up(rows, 256);
  uint8_t *digits = static_cast<uint8_t *>(d_ws);
  uint64_t *body = reinterpret_cast<uint64_t *>(digits + round_up(T * rp * phe::KS_LEVELS * N, 256));
  void *ws2 = reinterpret_cast<uint8_t *>(body) + round_up(T * rows * 8, 256);
  // (1) Eq. 6 in the NTT domain, masks written as Decomp digits; (2) Eq. 7/8 in the NTT domain
  rc = phe_matmul_clear_digits_ntt(p, d_tables, d_nttw, d_out, d_in, transpose, d_operand, T, digits, body, stream);
  if (rc) return rc;
  const int l1 = g_last_launches;
  rc = phe_pack_ntt(p, digits, body, T, rows, d_nksk, ws2, phe_pack_ntt_ws_bytes(p, rows, T), d_out_packed, stream);
  if (rc) return rc;
  g_last_launches += l1;
  return PHE_OK;
}

int phe_matmul_clear_ntt(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                         int64_t d_in, int64_t row_begin, int64_t row_end, const void *d_operand,
                         int64_t T, int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream) {
  return ntt_common(p, d_tables, d_nttw, d_out, d_in, row_begin, row_end, d_operand, T, out_bits,
                    d_out_mask, d_out_body, stream);
}

int phe_matmul_clear_ntt_into(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                              int64_t d_in, int transpose, int64_t row_begin, int64_t row_end,
                              const void *d_operand, int64_t T, int32_t out_bits, void *d_out_mask,
                              void *d_out_body, int64_t out_rows, void *stream) {
  if (!p || (transpose != 0 && transpose != 1)) return PHE_EINVAL;
  if (out_rows < row_end - row_begin) return PHE_EINVAL;
  const int64_t rows = transpose ? d_in : d_out, cols = transpose ? d_out : d_in;
  return ntt_common(p, d_tables, d_nttw, rows, cols, row_begin, row_end, d_operand, T, out_bits, d_out_mask,
                    d_out_body, stream, out_rows);
}

int phe_matmul_clear_ntt_T(const phe_params *p, const void *d_tables, const void *d_nttw, int64_t d_out,
                           int64_t d_in, int64_t row_begin, int64_t row_end, const void *d_operand,
                           int64_t T, int32_t out_bits, void *d_out_mask, void *d_out_body, void *stream) {
  return ntt_common(p, d_tables, d_nttw, d_in, d_out, row_begin, row_end, d_operand, T, out_bits,
                    d_out_mask, d_out_body, stream);
}

}  // extern "C"
