// limb_gemm.cu — the hot path: Eq. 6 + SampleExtract(N-1) + block sum + limb recombination
// + ModulusSwitch as ONE int8 GEMM on tcgen05 tensor cores (sm_100a), per DESIGN.md.
//
// Formulation ("Hankel form").  For one token tau and output row j
// (P:176-182 with Eq. 2 at h = N-1):
//     a_{tau,j}[t] = sum_i sum_{k<N} A_{tau,i}[k] * wext_{j,i}[k + t]   (mod 2^q_in)
//     wext_{j,i}[u] = W[j, iN+u] (u < N),  -W[j, iN+u-N] (N <= u < 2N)
// Split every 39-bit mask word into ell little-endian u8 limbs A = sum_l 2^(8l) A_l.  Then
//     D[(j,t), (tau,l)] = sum_{(i,k)} Hankel(wext)[(j,t), (i,k)] * A_l[tau][(i,k)]
// is a plain int8 x uint8 -> int32 GEMM:  M = rows*N (row = (j,t)), N_gemm = T*ell (column =
// (tau,l)), K = L*N.  The epilogue recombines v = sum_l D[.,(tau,l)] << 8l mod 2^q_in and
// applies the modulus switch, writing one word per (tau, j, t).
// The body b_{tau,j} = sum_c W[j,c] B_tau[c] (coefficient N-1 of B*w_hat) is the same GEMM
// with a plain W operand ("PLAIN" mode, M = rows).
//
// The Hankel A operand is never materialised.  Its tile (128 rows t x 128 bytes of k) holds
// only 240 distinct 16-byte rows R[p] = wext[s+p .. s+p+16) (s = k0 + t0): core matrix (g,h)
// (8 rows x 16 B, K-major, no swizzle) equals R[8(g+2h) .. +8), so a UMMA smem descriptor with
// SBO = 128 B and LBO = 256 B walks a compact 3840-byte buffer.  That buffer is a plain TMA
// box of the weight's 16-shift expansion (phe_weights_prepare).
//
// Pipeline (per CTA, persistent over tiles, 1 CTA per SM):
//   warps 0-7  epilogue      (tcgen05.ld -> recombine -> modswitch -> HBM); warp w reads TMEM
//                            lane quarter w % 4 (= its SM sub-partition)
//   warp 8     TMA producer  (A box + B box per K-stage, mbarrier complete_tx)
//   warp 9     MMA issuer    (tcgen05.mma kind::i8: M=128 N=256 K=32, or the CTA-pair M=256)
//   warp 10    TMEM allocator (512 columns = 2 accumulator stages of 256)
// The role warps have the HIGHEST warp ids on purpose: the sub-partition scheduler picks the
// highest eligible warp id first, so the single MMA-issuing thread is never starved by the
// epilogue warps that share its sub-partition (measured: ~10% of tensor-pipe cycles).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>

#include "phe_common.cuh"
#include "side_kernels.cuh"

namespace phe {
namespace tc {

constexpr int BM = 128;   // rows per tile (TMEM lanes)
constexpr int BN = 256;   // GEMM columns per tile: tokens*ell (+ pad)
constexpr int BK = 128;   // bytes of K per pipeline stage
constexpr int UK = 32;    // K of one tcgen05.mma kind::i8
constexpr int NUM_THREADS = 384;  // 8 epilogue warps (0-7) + producer 8, MMA 9, TMEM 10, spare 11
constexpr int W_PROD = 8, W_MMA = 9, W_TMEM = 10;
constexpr int NUM_EPI = 256;
// The 2-CTA mask kernel's epilogue groups (4 warps each, one per TMEM lane quarter): EG = 3 gives
// 12 epilogue warps (0-11) + producer 12, MMA 13, TMEM 14, spare 15 (512 threads).
#ifndef PHE_EPI_GROUPS
#define PHE_EPI_GROUPS 2
#endif
constexpr int EG = PHE_EPI_GROUPS;
constexpr int NT2 = (4 * EG + 4) * 32;
constexpr int W2_PROD = 4 * EG, W2_MMA = 4 * EG + 1, W2_TMEM = 4 * EG + 2;
constexpr int NUM_EPI2 = 128 * EG;
constexpr int A_ROWS_HANKEL = BM + BK - 16;            // 240 compact rows
constexpr int A_BYTES_HANKEL = A_ROWS_HANKEL * 16;     // 3840
constexpr int A_BYTES_PLAIN = BM * BK;                 // 16384
constexpr int B_BYTES = BN * BK;                       // 32768

template <bool HANKEL> struct Cfg;
template <> struct Cfg<true> {
  static constexpr int STAGES = 5;
  static constexpr int A_BYTES = A_BYTES_HANKEL;
  static constexpr int A_SLOT = 4096;  // 1024-aligned slot
};
template <> struct Cfg<false> {
  static constexpr int STAGES = 4;
  static constexpr int A_BYTES = A_BYTES_PLAIN;
  static constexpr int A_SLOT = A_BYTES_PLAIN;
};
template <bool HANKEL>
constexpr int smem_bytes() {
  return 1024 /*align slack*/ + Cfg<HANKEL>::STAGES * (B_BYTES + Cfg<HANKEL>::A_SLOT) + 256;
}

struct KArgs {
  int N;
  int tpt;            // tokens per tile
  int n_mma;          // MMA N = round16(tpt * ell) (2-CTA kernel)
  int n_mma_tail;     // MMA N of the last token tile (T % tpt tokens; == n_mma when it is full):
                      // the ragged tile runs a narrower MMA instead of a full-width one
  int n_tiles;        // token tiles
  int tb_per_row;     // N / BM (HANKEL) or 1
  int64_t m_tiles;    // rows*tb_per_row (HANKEL) or ceil(rows/BM)
  int64_t total_tiles;
  int k_blocks;       // Lc*N / BK
  int kb_per_block;   // N / BK
  int64_t Lc;
  int64_t cols;       // columns of the prepared matrix (d_in of the contraction)
  int full_k;         // no zero-padded K-blocks (or more than 64): no skipping
  int jpair;          // 2-CTA mask kernel: the pair's CTAs take rows j, j+1 over the same 128 t
                      // (tile = 128 t x 2 j) instead of 256 consecutive t of one j: the Hankel
                      // K-window of a partial block is then V + 127 wide instead of V + 255
  int64_t row_begin;  // absolute first row
  int64_t R;          // rows in range
  int64_t out_rows;   // row stride of the output tensor [T][out_rows][N] (>= R; > R when the
                      // output is a row block of a larger, possibly peer-mapped, gather buffer)
  int64_t T;
  int q_in, out_bits;
  int dbg;            // experiments only (PHE_DEBUG_EPI): 1 = no TMEM loads/stores, 2 = no stores
  void *out;
};

// Experiment knobs (PHE_DEBUG_EPI: skip TMEM loads / stores / operand loads, clock64 pipeline
// counters) exist only in builds with -DPHE_KERNEL_EXPERIMENTS=1; in production kdbg() is the
// constant 0 and every instrumentation branch folds away.
#ifndef PHE_KERNEL_EXPERIMENTS
#define PHE_KERNEL_EXPERIMENTS 0
#endif
__host__ __device__ __forceinline__ int kdbg(const KArgs &ka) { return PHE_KERNEL_EXPERIMENTS ? ka.dbg : 0; }

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap *map, int x, int y,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t *v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptors (sm_100 format: version 1 at bit 46).
// Hankel: K-major, SWIZZLE_NONE, core matrix 8 rows x 16 B; LBO (next 16 B of K) = 256 B,
// SBO (next 8 rows) = 128 B  ->  core (g,h) at start + 128*(g + 2h) (compact buffer).
__device__ __forceinline__ uint64_t desc_hankel(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(256 >> 4) << 16) |
         ((uint64_t)(128 >> 4) << 32) | (1ull << 46);
}
// Dense K-major tile written by TMA with 128-byte swizzle: SBO = 1024 B (8 rows x 128 B).
__device__ __forceinline__ uint64_t desc_sw128(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) |
         (1ull << 46) | (2ull << 61);
}
// Instruction descriptor: D = S32, A = s8 (weights), B = u8 (limbs), both K-major.
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (0u << 10) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(m >> 4) << 24);
}

// Persistent tile walk: tile = cid, cid + ncl, ... decoded incrementally (no 64-bit divides
// per tile): tile = m * n_tiles + n.
struct TileIter {
  int64_t tile, m;
  int n;
  int64_t step_m;
  int step_n;
  __device__ __forceinline__ TileIter(int64_t cid, int64_t ncl, int n_tiles) {
    tile = cid; m = cid / n_tiles; n = (int)(cid % n_tiles);
    step_m = ncl / n_tiles; step_n = (int)(ncl % n_tiles);
  }
  __device__ __forceinline__ void next(int64_t ncl, int n_tiles) {
    tile += ncl; m += step_m; n += step_n;
    if (n >= n_tiles) { n -= n_tiles; m++; }
  }
};

// One lane of a fully active warp (the issuing loops run warp-wide so that descriptors and
// loop state stay warp-uniform, i.e. in uniform registers; only the elected lane issues).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

// Limb recombination mod 2^q_in (a7) + ModulusSwitch (a8), one output word:
//   x = half + sum_l acc_l * 2^(8l)  (two's complement in 64 bits; 2^q_in | 2^64)
//   SW:  r = (x >> (q_in - q_out)) mod 2^q_out   (round half up: half = 2^(q_in-q_out-1))
//   !SW: r = x mod 2^q_in
// acc_l * 2^(8l) for 8l < 32 is one IMAD.WIDE; for 8l >= 32 only the high word moves.
template <int ELL, bool SW, typename OutT>
__device__ __forceinline__ OutT finish(const uint32_t *acc, int64_t half, int shift, uint64_t omask) {
  int64_t x = half + (int64_t)(int32_t)acc[0];
#pragma unroll
  for (int l = 1; l < ELL; l++) {
    if (8 * l < 32) x += (int64_t)(int32_t)acc[l] * (int64_t)(1ll << (8 * l));
    else x += (int64_t)((uint64_t)(uint32_t)acc[l] << (8 * l));
  }
  if (SW) return (OutT)(((uint64_t)x >> shift) & omask);
  return (OutT)((uint64_t)x & omask);
}

// Same result for SW with s = q_in - q_out known at compile time, in 32-bit integer ALU ops
// only (no wide multiplies).  With M = floor(s/8):
//   c_0 = acc_0 + 2^(s-1);  c_l = acc_l + (c_(l-1) >> 8)  (l = 1..M, arithmetic shifts)
//   r   = (c_M >> (s - 8M)) + sum_{l > M} acc_l << (8l - s)   (mod 2^q_out)
// Exact: floor((sum_l acc_l 2^(8l) + 2^(s-1)) / 2^s) splits into the exact multiples of 2^s
// (limbs l > M) plus a floor over the low limbs, and floor((2^8 Y + r)/2^s) = floor(Y / 2^(s-8))
// for 0 <= r < 2^8 <= 2^s.  |c_l| < 2^29 for K <= 8192 (|acc| <= 8192*127*255 < 2^28).
template <int ELL, int SH>
__device__ __forceinline__ uint32_t finish_sw(const uint32_t *acc, uint32_t omask) {
  constexpr int M = SH / 8;
  int32_t c = (int32_t)acc[0] + (1 << (SH - 1));
#pragma unroll
  for (int l = 1; l <= M && l < ELL; l++) c = (int32_t)acc[l] + (c >> 8);
  uint32_t r = (uint32_t)(c >> (SH - 8 * M));
#pragma unroll
  for (int l = M + 1; l < ELL; l++)
    if (8 * l - SH < 32) r += acc[l] << (8 * l - SH);
  return r & omask;
}

// ------------------------------------------------------------------ the kernel
template <int ELL, bool HANKEL, bool SW>
__global__ void __launch_bounds__(NUM_THREADS, 1)
limb_gemm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 KArgs ka) {
  using C = Cfg<HANKEL>;
  using OutT = typename std::conditional<SW, uint32_t, unsigned long long>::type;
  constexpr int S = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sB = smem;                          // S x 32 KB (1024-aligned)
  uint8_t *sA = smem + S * B_BYTES;            // S x A_SLOT
  uint64_t *bars = reinterpret_cast<uint64_t *>(sA + S * C::A_SLOT);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], NUM_EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_PROD && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == W_TMEM) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int64_t total = ka.total_tiles;
  if (warp == W_PROD) {
    // ===== TMA producer (warp-wide loop, elected lane issues) =====
    int s = 0; uint32_t ph = 0;
    for (TileIter it(blockIdx.x, gridDim.x, ka.n_tiles); it.tile < total; it.next(gridDim.x, ka.n_tiles)) {
      const int64_t m_tile = it.m;
      const int brow = it.n * ka.tpt * ELL;
      int64_t jrow; int t0;
      if (HANKEL) { jrow = ka.row_begin + m_tile / ka.tb_per_row; t0 = (int)(m_tile % ka.tb_per_row) * BM; }
      else { jrow = ka.row_begin + m_tile * BM; t0 = 0; }
      int i = 0, kk = 0;
      for (int kb = 0; kb < ka.k_blocks; kb++) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          mbar_expect_tx(&full[s], (uint32_t)(C::A_BYTES + B_BYTES));
          if (HANKEL) {
            const int64_t arow = (jrow * ka.Lc + i) * (2 * (int64_t)ka.N) + kk * BK + t0;
            tma_load_2d(smem_u32(sA + s * C::A_SLOT), &map_a, 0, (int)arow, &full[s]);
          } else {
            tma_load_2d(smem_u32(sA + s * C::A_SLOT), &map_a, kb * BK, (int)jrow, &full[s]);
          }
          tma_load_2d(smem_u32(sB + s * B_BYTES), &map_b, kb * BK, brow, &full[s]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
        if (++kk == ka.kb_per_block) { kk = 0; i++; }
      }
    }
  } else if (warp == W_MMA) {
    // ===== MMA issuer (warp-wide loop, elected lane issues + commits) =====
    constexpr uint32_t idesc = idesc_i8(BM, BN);
    int s = 0; uint32_t ph = 0; int acc = 0; uint32_t aph = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      mbar_wait(&tempty[acc], aph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
      for (int kb = 0; kb < ka.k_blocks; kb++) {
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * C::A_SLOT);
        const uint32_t b_addr = smem_u32(sB + s * B_BYTES);
        if (elect_one()) {
#pragma unroll
          for (int q = 0; q < BK / UK; q++) {
            const uint64_t adesc = HANKEL ? desc_hankel(a_addr + 512 * q) : desc_sw128(a_addr + 32 * q);
            mma_i8(d_tmem, adesc, desc_sw128(b_addr + 32 * q), idesc, (kb | q) != 0 ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
      if (elect_one()) tc_commit(&tfull[acc]);
      __syncwarp();
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  } else if (warp < 8) {
    // ===== epilogue: TMEM -> registers -> recombine limbs -> modswitch -> HBM =====
    // 8 warps (0-7): two per TMEM lane quarter; group g = 0/1 takes the even/odd 16-token chunks.
    const int q4 = warp & 3;  // TMEM lane quarter this warp may access
    const int grp = warp >> 2;
    const int row = q4 * 32 + lane;
    const int shift = ka.q_in - ka.out_bits;
    const int64_t half = SW ? (1ll << (shift - 1)) : 0;
    const uint64_t omask = mask_bits(ka.out_bits);
    const int64_t N = ka.N;
    OutT *const out = static_cast<OutT *>(ka.out);
    int acc = 0; uint32_t aph = 0;
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
      const int64_t m_tile = tile / ka.n_tiles;
      const int n_tile = (int)(tile % ka.n_tiles);
      const int64_t tau0 = (int64_t)n_tile * ka.tpt;
      const int ntok = (int)min((int64_t)ka.tpt, ka.T - tau0);
      int64_t obase;    // output index of (tau0, this row)
      int64_t tstride;  // index stride between consecutive tokens
      bool valid = true;
      if (HANKEL) {
        const int64_t jr = m_tile / ka.tb_per_row;
        const int64_t t = (m_tile % ka.tb_per_row) * BM + row;
        tstride = ka.out_rows * N;
        obase = tau0 * tstride + jr * N + t;
      } else {
        const int64_t jr = m_tile * BM + row;
        valid = jr < ka.R;
        tstride = ka.out_rows;
        obase = tau0 * tstride + jr;
      }
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN);
      for (int c0 = 16 * grp; c0 < ntok; c0 += 32) {
        const int nt = min(16, ntok - c0);
        const int nloads = (nt * ELL + 15) / 16;
        uint32_t v[16 * ELL];
#pragma unroll
        for (int q = 0; q < ELL; q++)
          if (q < nloads) tmem_ld16(tbase + (uint32_t)(c0 * ELL + 16 * q), &v[16 * q]);
        tmem_wait_ld();
        OutT *o = out + obase + (int64_t)c0 * tstride;
        if (nt == 16 && valid) {
#pragma unroll
          for (int tk = 0; tk < 16; tk++) {
            __stcs(o, finish<ELL, SW, OutT>(&v[tk * ELL], half, shift, omask));
            o += tstride;
          }
        } else if (valid) {
#pragma unroll
          for (int tk = 0; tk < 16; tk++) {
            if (tk < nt) __stcs(o, finish<ELL, SW, OutT>(&v[tk * ELL], half, shift, omask));
            o += tstride;
          }
        }
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == W_TMEM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// Experiment-only pipeline counters (PHE_DEBUG_EPI=4): cycles spent in each wait, summed over CTAs.
__device__ unsigned long long g_dbg_cnt[8];
__device__ __forceinline__ void dbg_add(int i, long long v) { atomicAdd(&g_dbg_cnt[i], (unsigned long long)v); }

// ------------------------------------------------------------------ 2-CTA (CTA pair) kernel
// Same contraction on a CTA pair (cluster of 2 on one TPC): tcgen05.mma.cta_group::2 with
// M = 256 (CTA r holds Hankel rows t0 + 128r .. +128 of the same j) and N = n_mma <= 256
// (CTA r holds B rows n_mma/2 * r .. +n_mma/2).  Per SM this halves the B (limb-plane) bytes
// moved through TMA, L2 and shared memory per MAC.  Only the leader CTA issues MMAs; both
// CTAs run TMA and the epilogue.  Epilogue: TMEM -> registers (recombine + switch) -> shared
// memory -> TMA bulk-tensor store of a [16 tokens][1 row j][128 t] box, double-buffered.
constexpr int B_HALF_MAX = (BN / 2) * BK;     // 16 KB per stage per CTA
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;   // clears the peer bit: addresses CTA 0's barrier
constexpr int EPI_TOK = 16;                   // tokens per epilogue chunk
// Output modes of the 2-CTA mask kernel.
constexpr int OUT_U64 = 0;  // raw LWE masks mod 2^q_in (uint64)
constexpr int OUT_U32 = 1;  // modulus-switched to q_out (uint32), the hot-path product
constexpr int OUT_DIG = 2;  // Decomp(A_LWE) digits for KeySwitch packing (Eq. 8): 3 int8 planes
constexpr int OUT_WIRE = 3; // switched to q_out and packed into the wire bitstream (R22): a CTA's
                            // 128 coefficients of one row are 2 q_out consecutive 64-bit words
constexpr int WIRE_QMAX = 26;  // q_out bound of OUT_WIRE (shared-memory budget)
template <int MODE> struct Cfg2 {
  using OutT = typename std::conditional<MODE == OUT_U64, unsigned long long,
               typename std::conditional<MODE == OUT_U32 || MODE == OUT_WIRE, uint32_t, uint8_t>::type>::type;
  static constexpr int STAGES = MODE == OUT_U64 ? 6 : (EG > 2 && MODE == OUT_WIRE) ? 7 : 8;
  static constexpr int OUT_BUF = EPI_TOK * BM * (MODE == OUT_DIG ? KS_LEVELS : (int)sizeof(OutT));  // 8/16/8 KB
  static constexpr int WIRE_BUF = MODE == OUT_WIRE ? EPI_TOK * 2 * WIRE_QMAX * 8 : 0;              // 6.5 KB
  static constexpr int SMEM = 1024 + STAGES * (B_HALF_MAX + 4096) + 2 * EG * (OUT_BUF + WIRE_BUF) + 256;
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_2sm(uint32_t dst, const CUtensorMap *map, int x, int y,
                                                uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster)
      : "memory");
}
// Same with an L2 eviction-priority hint (createpolicy: evict_first for streamed operands,
// evict_last for operands re-read by many tiles)
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_load_2d_2sm_hint(uint32_t dst, const CUtensorMap *map, int x, int y,
                                                     uint32_t bar_cluster, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(bar_cluster), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, uint32_t src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "r"(z)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *map, uint32_t src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tma_store_4d(const CUtensorMap *map, uint32_t src, int x, int y, int z, int w) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.tile.bulk_group [%0, {%2, %3, %4, %5}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_read_1() {
  asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_commit_mc2(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void mma_i8_2sm(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc,
                                           uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Epilogue -> MMA "accumulator drained" signal.  Relaxed: what must be ordered before it is
// only the TMEM reads, which tcgen05.wait::ld + tcgen05.fence::before_thread_sync completed.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

// K-block skipping for zero-padded blocks: the pair tile (rows tp .. tp+255) reads
// wext[u], u in [k0 + tp, k0 + tp + 383) for K-block k0 of block i; wext is zero outside
// [0, V) U [N, N+V), V = min(N, cols - iN).  Full blocks are never skipped; the tile's mask
// (bit kb = issue) is computed once per tile, identically by the producer and MMA warps, so
// the smem ring stays in step.  Never empty for V >= 1.  Blocks kb >= 64 are never skipped.
__device__ __forceinline__ uint64_t kblock_mask(const KArgs &ka, int tp) {
  const int span = ka.jpair ? BM : 2 * BM;  // rows t of the tile: tp .. tp + span - 1
  if (ka.full_k || kdbg(ka) == 9) return ~0ull;
  // Closed form (checked against the per-block definition above for N in 256..4096, all
  // cols, all tp): only the last block il = Lc-1 can be partial (V < N); its needed kk are
  // [0, lo_end) U [hi_start, hi_end) with a = kk*BK + tp:
  //   a < V               <=> kk < ceil((V - tp) / BK)
  //   a + span+127 > N    <=> kk >= floor((N - tp - span - 127) / BK) + 1   (all kk if < 0)
  //   a < N + V           <=> kk < ceil((N + V - tp) / BK)
  const int kbpb = ka.kb_per_block, N = ka.N, il = (int)ka.Lc - 1;
  const int V = (int)(ka.cols - (int64_t)il * N);
  auto cl = [kbpb](int v) { return v < 0 ? 0 : (v > kbpb ? kbpb : v); };
  auto rng = [](int a, int b) -> uint64_t { return b > a ? (((1ull << b) - 1ull) & ~((1ull << a) - 1ull)) : 0ull; };
  const int lo_end = V - tp > 0 ? cl((V - tp + BK - 1) / BK) : 0;
  const int x = N - tp - (span + BK - 1);
  const int hi_start = x >= 0 ? cl(x / BK + 1) : 0;
  const int hi_end = cl((N + V - tp + BK - 1) / BK);
  const uint64_t full_bits = il * kbpb >= 64 ? ~0ull : ((1ull << (il * kbpb)) - 1ull);
  return full_bits | ((rng(0, lo_end) | rng(hi_start, hi_end)) << (il * kbpb));
}
__device__ __forceinline__ bool kb_issue(uint64_t m, int kb) { return kb >= 64 || ((m >> kb) & 1ull); }

template <int ELL, int MODE, int SH>
__global__ void __launch_bounds__(NT2, 1)
limb_gemm_2sm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     const __grid_constant__ CUtensorMap map_b_tail, const __grid_constant__ CUtensorMap map_out,
                     const __grid_constant__ CUtensorMap map_out_tail, KArgs ka) {
  using C2 = Cfg2<MODE>;
  using OutT = typename C2::OutT;
  constexpr bool SW = MODE != OUT_U64;  // OUT_DIG shifts by q_in - 32 (ka.out_bits = 32)
  constexpr int S = C2::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sB = smem;                                // S x 16 KB (1024-aligned)
  uint8_t *sA = smem + S * B_HALF_MAX;               // S x 4 KB
  uint8_t *sO = sA + S * 4096;                       // EG groups x 2 buffers x OUT_BUF
  uint64_t *sW = reinterpret_cast<uint64_t *>(sO + 2 * EG * C2::OUT_BUF);  // OUT_WIRE: EG x 2 x WIRE_BUF
  uint64_t *bars = reinterpret_cast<uint64_t *>(sO + 2 * EG * C2::OUT_BUF + 2 * EG * C2::WIRE_BUF);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int n_mma = ka.n_mma;                 // MMA N = round16(tpt * ELL)
  const int b_half = (n_mma / 2) * BK;        // B bytes per CTA per stage

  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * NUM_EPI2); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W2_PROD && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_out)) : "memory");
  }
  if (warp == W2_TMEM) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  const int64_t total = ka.total_tiles;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  if (warp == W2_PROD) {
    // ===== TMA producer (both CTAs, warp-wide loop, elected lane issues): own Hankel rows +
    // own half of B, bytes land on CTA 0's barrier =====
    int s = 0; uint32_t ph = 0;
    long long pw = 0;
    const int a_tx = kdbg(ka) == 5 ? 0 : A_BYTES_HANKEL;
    const uint32_t tx_full = (uint32_t)(2 * (a_tx + (kdbg(ka) == 6 ? 0 : b_half)));
    const uint32_t tx_tail = (uint32_t)(2 * (a_tx + (kdbg(ka) == 6 ? 0 : (ka.n_mma_tail / 2) * BK)));
    for (TileIter it(cid, ncl, ka.n_tiles); it.tile < total; it.next(ncl, ka.n_tiles)) {
      const int64_t m_tile = it.m;
      const int n_tile = it.n;
      const bool tl = n_tile == ka.n_tiles - 1;  // ragged last token tile: narrower B box
      const uint32_t tx = tl ? tx_tail : tx_full;
      const CUtensorMap *mbp = tl ? &map_b_tail : &map_b;
      const int brow = n_tile * ka.tpt * ELL + (int)crank * ((tl ? ka.n_mma_tail : n_mma) / 2);
      const int jr_ = (int)((uint32_t)m_tile / (uint32_t)ka.tb_per_row);
      int64_t jrow, abase;
      int tp;  // the tile's first row t
      if (ka.jpair) {  // CTA r: row j = 2 jr_ + r, rows t tp .. tp + 127
        tp = ((int)m_tile - jr_ * ka.tb_per_row) * BM;
        jrow = ka.row_begin + 2 * (int64_t)jr_ + (int)crank;
        abase = jrow * ka.Lc * (2 * (int64_t)ka.N) + tp;
      } else {         // CTA r: row j = jr_, rows t tp + 128 r .. + 127
        tp = ((int)m_tile - jr_ * ka.tb_per_row) * (2 * BM);
        jrow = ka.row_begin + jr_;
        abase = jrow * ka.Lc * (2 * (int64_t)ka.N) + tp + (int)crank * BM;
      }
      const uint64_t km = kblock_mask(ka, tp);
      int i = 0, kk = 0;
      for (int kb = 0; kb < ka.k_blocks; kb++) {
        if (kb_issue(km, kb)) {
          long long w0 = kdbg(ka) == 4 ? clock64() : 0;
          mbar_wait(&empty[s], ph ^ 1);
          if (kdbg(ka) == 4) pw += clock64() - w0;
          if (elect_one()) {
            if (leader) mbar_expect_tx(&full[s], tx);
            const uint32_t fb = smem_u32(&full[s]) & PEER_MASK;
            const int64_t arow = abase + (int64_t)i * (2 * (int64_t)ka.N) + kk * BK;
            if (kdbg(ka) != 5) tma_load_2d_2sm(smem_u32(sA + s * 4096), &map_a, 0, (int)arow, fb);
            if (kdbg(ka) != 6) tma_load_2d_2sm(smem_u32(sB + s * B_HALF_MAX), mbp, kb * BK, brow, fb);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (++kk == ka.kb_per_block) { kk = 0; i++; }
      }
    }
    if (kdbg(ka) == 4 && lane == 0) dbg_add(5, pw);
  } else if (warp == W2_MMA) {
    // ===== MMA issuer (leader CTA only; warp-wide loop, elected lane issues + commits) =====
    if (leader) {
      const uint32_t idesc_full = idesc_i8(2 * BM, n_mma), idesc_tail = idesc_i8(2 * BM, ka.n_mma_tail);
      int s = 0; uint32_t ph = 0; int acc = 0; uint32_t aph = 0;
      long long t_start = kdbg(ka) == 4 ? clock64() : 0, wt = 0, wf = 0;
      for (TileIter it(cid, ncl, ka.n_tiles); it.tile < total; it.next(ncl, ka.n_tiles)) {
        const uint32_t idesc = it.n == ka.n_tiles - 1 ? idesc_tail : idesc_full;
        long long w0 = kdbg(ka) == 4 ? clock64() : 0;
        mbar_wait(&tempty[acc], aph ^ 1);
        if (kdbg(ka) == 4) wt += clock64() - w0;
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        const int tp = (int)((uint32_t)it.m % (uint32_t)ka.tb_per_row) * (ka.jpair ? BM : 2 * BM);
        const uint64_t km = kblock_mask(ka, tp);
        uint32_t acc_flag = 0;  // first issued MMA of the tile overwrites the accumulator
        for (int kb = 0; kb < ka.k_blocks; kb++) {
          if (!kb_issue(km, kb)) continue;
          long long w1 = kdbg(ka) == 4 ? clock64() : 0;
          mbar_wait(&full[s], ph);
          if (kdbg(ka) == 4) wf += clock64() - w1;
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * 4096);
          const uint32_t b_addr = smem_u32(sB + s * B_HALF_MAX);
          if (elect_one()) {
#pragma unroll
            for (int q = 0; q < BK / UK; q++)
              mma_i8_2sm(d_tmem, desc_hankel(a_addr + 512 * q), desc_sw128(b_addr + 32 * q), idesc,
                         (acc_flag | (uint32_t)q) ? 1u : 0u);
            tc_commit_mc2(&empty[s]);
          }
          __syncwarp();
          acc_flag = 1u;
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (elect_one()) tc_commit_mc2(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
      if (kdbg(ka) == 4 && lane == 0) { dbg_add(0, wt); dbg_add(1, wf); dbg_add(2, clock64() - t_start); }
    }
  } else if (warp < 4 * EG) {
    // ===== epilogue (both CTAs): own 128 TMEM lanes = own 128 rows t =====
    // Group g (warps 0-3 / 4-7) takes every other 16-token chunk (alternating per tile).
    const int q4 = warp & 3;
    const int grp = warp >> 2;
    const int row = q4 * 32 + lane;
    const bool issuer = (warp & 3) == 0 && lane == 0;
    const int shift = ka.q_in - ka.out_bits;
    const int64_t half = SW ? (1ll << (shift - 1)) : 0;
    const uint64_t omask = mask_bits(ka.out_bits);
    const uint32_t tempty_c0 = smem_u32(&tempty[0]) & PEER_MASK;
    OutT *const obuf = reinterpret_cast<OutT *>(sO + grp * 2 * C2::OUT_BUF);  // grp < EG
    constexpr int OB_ELEMS = C2::OUT_BUF / (int)sizeof(OutT);
    int acc = 0; uint32_t aph = 0; int nbuf = 0; int64_t iter = 0;
    for (TileIter it(cid, ncl, ka.n_tiles); it.tile < total; it.next(ncl, ka.n_tiles), iter++) {
      const int n_tile = it.n;
      const int tau0 = n_tile * ka.tpt;
      const int ntok = (int)min((int64_t)ka.tpt, ka.T - tau0);
      const int jq = (int)((uint32_t)it.m / (uint32_t)ka.tb_per_row);
      const int jr = ka.jpair ? 2 * jq + (int)crank : jq;
      const int tb = ka.jpair ? ((int)it.m - jq * ka.tb_per_row) * BM
                              : ((int)it.m - jq * ka.tb_per_row) * (2 * BM) + (int)crank * BM;
      const int nchunks = (ntok + EPI_TOK - 1) / EPI_TOK;
      const int first = (grp + (int)(iter % EG)) % EG;
      long long e0 = (kdbg(ka) == 4 && warp == 0 && lane == 0) ? clock64() : 0;
      mbar_wait(&tfull[acc], aph);
      long long e1 = (kdbg(ka) == 4 && warp == 0 && lane == 0) ? clock64() : 0;
      if (kdbg(ka) == 4 && warp == 0 && lane == 0) dbg_add(4, e1 - e0);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN);
      bool arrived = false;
      for (int c = first; c < nchunks; c += EG) {
        const int c0 = c * EPI_TOK;
        const int nt = min(EPI_TOK, ntok - c0);
        const int nloads = (nt * ELL + 15) / 16;
        uint32_t v[EPI_TOK * ELL];
#pragma unroll
        for (int q = 0; q < ELL; q++)
          if (q < nloads) tmem_ld16(tbase + (uint32_t)(c0 * ELL + 16 * q), &v[16 * q]);
        tmem_wait_ld();
        if (c + EG >= nchunks) {  // last TMEM read of this tile by this thread: release the buffer
          tc_fence_before();
          mbar_arrive_cluster(tempty_c0 + 8u * (uint32_t)acc);
          arrived = true;
        }
        OutT *ob = obuf + nbuf * OB_ELEMS;
        named_bar(1 + grp, 128);  // the store that last read buffer nbuf has drained
        if constexpr (MODE == OUT_WIRE) {
          // the warp's 32 consecutive coefficients (t = 32 q4 + lane) of one token are 32 q bits =
          // q 32-bit words of the wire bitstream (R22): lane k < q assembles word k from the (up
          // to three) coefficients it overlaps, taken from their lanes by shuffles, and stores it
          // at u32 word 4 q tk + q q4 + k of the chunk's [16 tokens][128 coefficients] block
          const int qb = ka.out_bits;
          const int c0 = (32 * lane) / qb, s0 = 32 * lane - qb * c0;
          const int l0 = min(c0, 31), l1 = min(c0 + 1, 31), l2 = min(c0 + 2, 31);
          uint32_t *wb32 = reinterpret_cast<uint32_t *>(sW + (grp * 2 + nbuf) * (C2::WIRE_BUF / 8));
#pragma unroll
          for (int tk = 0; tk < EPI_TOK; tk++) {
            uint32_t val;
            if constexpr (SH > 0) val = finish_sw<ELL, SH>(&v[tk * ELL], (uint32_t)omask);
            else val = (uint32_t)finish<ELL, true, uint32_t>(&v[tk * ELL], half, shift, omask);
            const uint64_t a0 = __shfl_sync(0xffffffffu, val, l0);
            const uint64_t a1 = __shfl_sync(0xffffffffu, val, l1);
            const uint64_t a2 = __shfl_sync(0xffffffffu, val, l2);
            const uint64_t cat = a0 | (a1 << qb) | (a2 << (2 * qb));
            if (lane < qb && tk < nt) wb32[tk * 4 * qb + q4 * qb + lane] = (uint32_t)(cat >> s0);
          }
        } else if (kdbg(ka) != 1) {
          if constexpr (MODE == OUT_DIG) {
            // r = top 32 bits of v after rounding the q_in - 32 bit tail half up; signed base-2^8
            // digits, least significant first with carry (Decomp, Eq. 4 / S:59-67; R18);
            // planes [tk][l][t], plane l has weight 2^(q_in - 8(l+1))
            uint8_t *od = reinterpret_cast<uint8_t *>(ob);
#pragma unroll
            for (int tk = 0; tk < EPI_TOK; tk++) {
              uint32_t r;
              if constexpr (SH > 0) r = finish_sw<ELL, SH>(&v[tk * ELL], 0xFFFFFFFFu);
              else if (shift == 0) r = (uint32_t)finish<ELL, false, uint64_t>(&v[tk * ELL], 0, 0, ~0ull);
              else r = (uint32_t)finish<ELL, true, uint64_t>(&v[tk * ELL], half, shift, 0xFFFFFFFFull);
              int d[KS_LEVELS];
#pragma unroll
              for (int l = KS_LEVELS - 1; l >= 0; l--) {
                int dl = (int)(r & 255u);
                r >>= 8;
                if (dl >= 128) { dl -= 256; r += 1; }
                d[l] = dl;
              }
#pragma unroll
              for (int l = 0; l < KS_LEVELS; l++) od[(tk * KS_LEVELS + l) * BM + row] = (uint8_t)d[l];
            }
          } else {
#pragma unroll
            for (int tk = 0; tk < EPI_TOK; tk++) {
              if constexpr (SW && SH > 0) ob[tk * BM + row] = (OutT)finish_sw<ELL, SH>(&v[tk * ELL], (uint32_t)omask);
              else ob[tk * BM + row] = finish<ELL, SW, OutT>(&v[tk * ELL], half, shift, omask);
            }
          }
        }
        fence_proxy_async_smem();
        named_bar(1 + grp, 128);  // chunk staged
        if (MODE == OUT_WIRE && issuer && jr < ka.R) {
          // [tokens][words] box: the row's segment word jr * N q / 64 + the block's first word
          const CUtensorMap *mo = (c0 + EPI_TOK <= ka.tpt) ? &map_out : &map_out_tail;
          const int qw = 2 * ka.out_bits;
          uint64_t *wb = sW + (grp * 2 + nbuf) * (C2::WIRE_BUF / 8);
          if (kdbg(ka) == 0 || kdbg(ka) == 4)
            tma_store_2d(mo, smem_u32(wb), (int)((int64_t)jr * (ka.N / BM) * qw + (tb / BM) * qw), tau0 + c0);
          bulk_wait_read_1();
        } else if (MODE != OUT_WIRE && issuer) {
          // a full 16-token box, or the tpt % 16 tail box of this tile (never past the tile)
          const CUtensorMap *mo = (c0 + EPI_TOK <= ka.tpt) ? &map_out : &map_out_tail;
          if (kdbg(ka) == 0 || kdbg(ka) == 4) {
            if constexpr (MODE == OUT_DIG) tma_store_4d(mo, smem_u32(ob), tb, 0, jr, tau0 + c0);
            else tma_store_3d(mo, smem_u32(ob), tb, jr, tau0 + c0);
          }
          bulk_wait_read_1();
        }
        nbuf ^= 1;
      }
      if (!arrived) {
        tc_fence_before();
        mbar_arrive_cluster(tempty_c0 + 8u * (uint32_t)acc);
      }
      if (kdbg(ka) == 4 && warp == 0 && lane == 0) { dbg_add(3, clock64() - e1); dbg_add(6, 1); }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
    if (issuer) bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == W2_TMEM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ------------------------------------------------------------------ KeySwitch packing GEMM (NEXT #1)
// Eq. 8 + the rotate-and-sum of Eq. 7 for T tokens at once:
//   C[(tau,j), (part,k)] = sum_{(l,i)} Decomp(a_{tau,j})[l*N+i] * KSK_part[l*N+i][k]   (mod 2^q)
// as an int8 (digits) x u8 (KSK limbs) GEMM on tcgen05 cta_group::2: M = rows (tau, j) (256
// per pair), N = 51 coefficient slots x 5 limbs, K = KS_LEVELS*N.  The epilogue recombines limbs and
// applies Rotate(., j mod N) + the sum over j of Eq. 7 in shared-memory bins (a CTA's 128 rows
// and 51 slots land on 178 consecutive output coefficients), then reduces the bins into the
// packed accumulator [T][G][part][N] (uint64, mod 2^64) with global atomics.
struct PArgs {
  int N;
  int kpad;           // coefficient slots per part = ceil(N / spt) * spt
  int spt;            // slots per tile = floor(256 / ell)
  int n_tiles;        // 2 * kpad / spt
  int tpt_rows;       // 256-row tiles per token = rows_pad / 256
  int64_t rows_pad;   // digit rows per token (multiple of 256)
  int G;              // output RLWE groups per token = ceil(R / N)
  int64_t total_tiles;
  int64_t m_tiles;    // T * tpt_rows
  int ng;             // N-tile group width of the rasterization (pack_tile)
  int hints;          // L2 eviction hints on the operand loads
  int k_blocks;       // KS_LEVELS*N / BK
  unsigned long long *acc;
};

// Grouped rasterization: tiles sweep every M-tile (token rows) inside a group of `ng` N-tiles
// (KSK coefficient slots), so the group's KSK limb planes (ng x 2 MB) stay L2-resident while
// the digits stream through once per group.  (m-major order over all 82 N-tiles re-streamed the
// whole 168 MB KSK -- more than L2 -- from HBM for every wave of 74 tiles.)
__device__ __forceinline__ void pack_tile(const PArgs &pa, int64_t t, int64_t &m, int &n) {
  const int64_t gsz = pa.m_tiles * pa.ng;
  const int64_t g = t / gsz;
  const int64_t r = t - g * gsz;
  const int n0 = (int)g * pa.ng;
  const int w = min(pa.ng, pa.n_tiles - n0);
  m = r / w;
  n = n0 + (int)(r - m * w);
}
constexpr int PK_STAGES = 6;
constexpr int PK_A_BYTES = BM * BK;            // 16 KB per CTA per stage (digit rows)
constexpr int PK_B_BYTES = (BN / 2) * BK;      // 16 KB per CTA per stage (KSK limb rows)
constexpr int PK_BINS = 184;                   // >= spt + BM - 1
constexpr int PK_SMEM = 1024 + PK_STAGES * (PK_A_BYTES + PK_B_BYTES) + 2 * PK_BINS * 8 + 256;

template <int ELL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
pack_gemm_2sm_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                     PArgs pa) {
  constexpr int S = PK_STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  uint8_t *sB = smem;
  uint8_t *sA = smem + S * PK_B_BYTES;
  unsigned long long *bins = reinterpret_cast<unsigned long long *>(sA + S * PK_A_BYTES);  // [2][PK_BINS]
  uint64_t *bars = reinterpret_cast<uint64_t *>(bins + 2 * PK_BINS);
  uint64_t *full = bars, *empty = bars + S, *tfull = bars + 2 * S, *tempty = bars + 2 * S + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(bars + 2 * S + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;

  for (int i = threadIdx.x; i < 2 * PK_BINS; i += blockDim.x) bins[i] = 0ull;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; s++) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; a++) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 2 * NUM_EPI); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == W_PROD && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == W_TMEM) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     smem_u32(tmem_holder))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  const int64_t total = pa.total_tiles;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

  if (warp == W_PROD) {
    int s = 0; uint32_t ph = 0;
    const uint32_t tx = (uint32_t)(2 * (PK_A_BYTES + PK_B_BYTES));
    const uint64_t pol_a = l2_policy_evict_first(), pol_b = l2_policy_evict_last();
    for (int64_t tile = cid; tile < total; tile += ncl) {
      int64_t tm; int tn;
      pack_tile(pa, tile, tm, tn);
      const int tau = (int)((uint64_t)tm / (uint64_t)pa.tpt_rows);
      const int64_t j0 = (tm - (int64_t)tau * pa.tpt_rows) * (2 * BM);
      const int64_t arow = (int64_t)tau * pa.rows_pad + j0 + (int)crank * BM;
      const int brow = tn * pa.spt * ELL + (int)crank * (BN / 2);
      for (int kb = 0; kb < pa.k_blocks; kb++) {
        mbar_wait(&empty[s], ph ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&full[s], tx);
          const uint32_t fb = smem_u32(&full[s]) & PEER_MASK;
          if (pa.hints) {  // digits stream (evict_first); the KSK group is re-read (evict_last)
            tma_load_2d_2sm_hint(smem_u32(sA + s * PK_A_BYTES), &map_a, kb * BK, (int)arow, fb, pol_a);
            tma_load_2d_2sm_hint(smem_u32(sB + s * PK_B_BYTES), &map_b, kb * BK, brow, fb, pol_b);
          } else {
            tma_load_2d_2sm(smem_u32(sA + s * PK_A_BYTES), &map_a, kb * BK, (int)arow, fb);
            tma_load_2d_2sm(smem_u32(sB + s * PK_B_BYTES), &map_b, kb * BK, brow, fb);
          }
        }
        __syncwarp();
        if (++s == S) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == W_MMA) {
    if (leader) {
      const uint32_t idesc = idesc_i8(2 * BM, BN);
      int s = 0; uint32_t ph = 0; int acc = 0; uint32_t aph = 0;
      for (int64_t tile = cid; tile < total; tile += ncl) {
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < pa.k_blocks; kb++) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * PK_A_BYTES);
          const uint32_t b_addr = smem_u32(sB + s * PK_B_BYTES);
          if (elect_one()) {
#pragma unroll
            for (int q = 0; q < BK / UK; q++)
              mma_i8_2sm(d_tmem, desc_sw128(a_addr + 32 * q), desc_sw128(b_addr + 32 * q), idesc,
                         (kb | q) != 0 ? 1u : 0u);
            tc_commit_mc2(&empty[s]);
          }
          __syncwarp();
          if (++s == S) { s = 0; ph ^= 1; }
        }
        if (elect_one()) tc_commit_mc2(&tfull[acc]);
        __syncwarp();
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
  } else if (warp < 8) {
    // ===== epilogue: recombine limbs, Rotate(., j mod N) + sum over j into bins, reduce =====
    const int q4 = warp & 3, grp = warp >> 2;
    const int row = q4 * 32 + lane;  // this CTA's row = TMEM lane
    const int etid = threadIdx.x;    // 0..255 (epilogue warps are 0-7)
    const uint32_t tempty_c0 = smem_u32(&tempty[0]) & PEER_MASK;
    const int nchunks = (pa.spt + EPI_TOK - 1) / EPI_TOK;
    int acc = 0; uint32_t aph = 0; int64_t iter = 0;
    for (int64_t tile = cid; tile < total; tile += ncl, iter++) {
      int64_t tm; int tn;
      pack_tile(pa, tile, tm, tn);
      const int tau = (int)((uint64_t)tm / (uint64_t)pa.tpt_rows);
      const int64_t jc = (tm - (int64_t)tau * pa.tpt_rows) * (2 * BM) + (int)crank * BM;
      const int g = (int)(jc / pa.N);
      const int r_c0 = (int)(jc - (int64_t)g * pa.N);  // rotation of this CTA's first row
      const int slot0 = tn * pa.spt;
      const int part = slot0 / pa.kpad;
      const int k0 = slot0 - part * pa.kpad;
      unsigned long long *bn = bins + acc * PK_BINS;
      const int first = (grp + (int)(iter & 1)) & 1;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(acc * BN);
      bool arrived = false;
      for (int c = first; c < nchunks; c += 2) {
        const int c0 = c * EPI_TOK;
        const int nt = min(EPI_TOK, pa.spt - c0);
        const int nloads = (nt * ELL + 15) / 16;
        uint32_t v[EPI_TOK * ELL];
#pragma unroll
        for (int q = 0; q < ELL; q++)
          if (q < nloads) tmem_ld16(tbase + (uint32_t)(c0 * ELL + 16 * q), &v[16 * q]);
        tmem_wait_ld();
        if (c + 2 >= nchunks) {
          tc_fence_before();
          mbar_arrive_cluster(tempty_c0 + 8u * (uint32_t)acc);
          arrived = true;
        }
#pragma unroll
        for (int tk = 0; tk < EPI_TOK; tk++) {
          if (tk < nt && k0 + c0 + tk < pa.N) {
            uint64_t x = 0;
#pragma unroll
            for (int l = 0; l < ELL; l++) x += (uint64_t)(int64_t)(int32_t)v[tk * ELL + l] << (8 * l);
            if (x) atomicAdd(&bn[c0 + tk + row], (unsigned long long)x);  // p = k + r, unwrapped
          }
        }
      }
      if (!arrived) {
        tc_fence_before();
        mbar_arrive_cluster(tempty_c0 + 8u * (uint32_t)acc);
      }
      named_bar(1, NUM_EPI);  // all slots of this tile are in the bins
      for (int t = etid; t < pa.spt + BM - 1; t += NUM_EPI) {
        unsigned long long val = bn[t];
        if (val) {
          bn[t] = 0ull;
          int p = k0 + r_c0 + t;                 // X^N = -1: p >= N wraps with a sign flip
          if (p >= pa.N) { p -= pa.N; val = 0ull - val; }
          atomicAdd(pa.acc + (((int64_t)tau * pa.G + g) * 2 + part) * pa.N + p, val);
        }
      }
      // bins[acc] is reused two tiles later, after the next tile's named barrier
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == W_TMEM) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem_base) : "memory");
  }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

static int make_map_2d(CUtensorMap *m, const void *base, uint64_t dim0, uint64_t dim1,
                       uint64_t stride1, uint32_t box0, uint32_t box1, CUtensorMapSwizzle sw) {
  auto enc = get_encode();
  if (!enc) return PHE_ECUDA;
  cuuint64_t dims[2] = {dim0, dim1};
  cuuint64_t strides[1] = {stride1};
  cuuint32_t box[2] = {box0, box1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PHE_OK : PHE_EINVAL;
}

static int num_sms() {  // per device (a process may drive several GPUs)
  static int cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &n = cache[dev & 63];
  if (!n) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n = v > 0 ? v : 148;
  }
  return n;
}

template <int ELL, bool HANKEL, bool SW>
static int launch_one(const CUtensorMap &ma, const CUtensorMap &mb, const KArgs &ka, cudaStream_t st) {
  auto kern = limb_gemm_kernel<ELL, HANKEL, SW>;
  constexpr int smem = smem_bytes<HANKEL>();
  static thread_local uint64_t set = 0;  // devices this thread configured the kernel on
  if (!(set & phe_device_bit())) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
    set |= phe_device_bit();
  }
  int64_t grid = ka.total_tiles < num_sms() ? ka.total_tiles : num_sms();
  kern<<<(unsigned)grid, NUM_THREADS, smem, st>>>(ma, mb, ka);
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

template <bool HANKEL, bool SW>
static int dispatch_ell(int ell, const CUtensorMap &ma, const CUtensorMap &mb, const KArgs &ka,
                        cudaStream_t st) {
  switch (ell) {
    case 1: return launch_one<1, HANKEL, SW>(ma, mb, ka, st);
    case 2: return launch_one<2, HANKEL, SW>(ma, mb, ka, st);
    case 3: return launch_one<3, HANKEL, SW>(ma, mb, ka, st);
    case 4: return launch_one<4, HANKEL, SW>(ma, mb, ka, st);
    case 5: return launch_one<5, HANKEL, SW>(ma, mb, ka, st);
    case 6: return launch_one<6, HANKEL, SW>(ma, mb, ka, st);
    case 7: return launch_one<7, HANKEL, SW>(ma, mb, ka, st);
    case 8: return launch_one<8, HANKEL, SW>(ma, mb, ka, st);
  }
  return PHE_EUNSUPPORTED;
}


template <int ELL, int MODE, int SH>
static int launch_2sm(const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbt, const CUtensorMap &mo,
                      const CUtensorMap &mot, const KArgs &ka, cudaStream_t st) {
  auto kern = limb_gemm_2sm_kernel<ELL, MODE, SH>;
  constexpr int smem = Cfg2<MODE>::SMEM;
  static thread_local uint64_t set = 0;  // devices this thread configured the kernel on
  if (!(set & phe_device_bit())) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
    set |= phe_device_bit();
  }
  int64_t pairs = num_sms() / 2;
  if (ka.total_tiles < pairs) pairs = ka.total_tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(NT2);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, mbt, mo, mot, ka) != cudaSuccess)
    return phe_set_cuda_error(cudaGetLastError());
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

template <int MODE>
static int dispatch_2sm(int ell, const CUtensorMap &ma, const CUtensorMap &mb, const CUtensorMap &mbt, const CUtensorMap &mo,
                        const CUtensorMap &mot, const KArgs &ka, cudaStream_t st) {
  const int sh = ka.q_in - ka.out_bits;
  if (MODE != OUT_U64 && ell == 5 && sh == 13) return launch_2sm<5, MODE, 13>(ma, mb, mbt, mo, mot, ka, st);  // Table 1
  if (MODE != OUT_U64 && ell == 5 && sh == 7) return launch_2sm<5, MODE, 7>(ma, mb, mbt, mo, mot, ka, st);  // digits, q=39
  if (MODE != OUT_U64 && ell == 4 && sh == 4) return launch_2sm<4, MODE, 4>(ma, mb, mbt, mo, mot, ka, st);    // toy
  switch (ell) {
    case 4: return launch_2sm<4, MODE, 0>(ma, mb, mbt, mo, mot, ka, st);
    case 5: return launch_2sm<5, MODE, 0>(ma, mb, mbt, mo, mot, ka, st);
  }
  return PHE_EUNSUPPORTED;
}

// Tokens per tile for the 2-CTA kernel: floor(256/ell) (MMA N = 256: N = 240 runs at the
// N = 256 rate on the tensor core, so fewer, fuller tiles win), fewer when T is small.
static int choose_tpt(int64_t T, int ell, int *n_mma) {
  int tpt = BN / ell;
  if (T < tpt) tpt = (int)T;
  int n = ((tpt * ell + 15) / 16) * 16;
  if (n < 32) n = 32;
  *n_mma = n;
  return tpt;
}

static int make_map_digits(CUtensorMap *m, void *base, int64_t N, int64_t Rpad, int64_t T, int box_tok) {
  auto enc = get_encode();
  if (!enc) return PHE_ECUDA;
  cuuint64_t dims[4] = {(cuuint64_t)N, KS_LEVELS, (cuuint64_t)Rpad, (cuuint64_t)T};
  cuuint64_t strides[3] = {(cuuint64_t)N, (cuuint64_t)(KS_LEVELS * N), (cuuint64_t)(KS_LEVELS * N * Rpad)};
  cuuint32_t box[4] = {(cuuint32_t)BM, KS_LEVELS, 1, (cuuint32_t)box_tok};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, base, dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PHE_OK : PHE_EINVAL;
}

// LWE wire records [T][tw] uint64 words; box = one row's 128-coefficient block (2 q words) x tokens
static int make_map_wire(CUtensorMap *m, void *base, int64_t tw, int64_t T, int qw, int box_tok) {
  auto enc = get_encode();
  if (!enc) return PHE_ECUDA;
  cuuint64_t dims[2] = {(cuuint64_t)tw, (cuuint64_t)T};
  cuuint64_t strides[1] = {(cuuint64_t)(tw * 8)};
  cuuint32_t box[2] = {(cuuint32_t)qw, (cuuint32_t)box_tok};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PHE_OK : PHE_EINVAL;
}

static int make_map_out(CUtensorMap *m, void *base, bool sw, int64_t N, int64_t R, int64_t T, int box_tok,
                        int64_t out_rows) {
  auto enc = get_encode();
  if (!enc) return PHE_ECUDA;
  const uint64_t es = sw ? 4 : 8;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)R, (cuuint64_t)T};
  cuuint64_t strides[2] = {(cuuint64_t)(N * es), (cuuint64_t)(out_rows * N * es)};
  cuuint32_t box[3] = {(cuuint32_t)BM, 1, (cuuint32_t)box_tok};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, sw ? CU_TENSOR_MAP_DATA_TYPE_UINT32 : CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, base, dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? PHE_OK : PHE_EINVAL;
}

template <bool HANKEL>
static int dispatch(int ell, bool sw, const CUtensorMap &ma, const CUtensorMap &mb, const KArgs &ka,
                    cudaStream_t st) {
  return sw ? dispatch_ell<HANKEL, true>(ell, ma, mb, ka, st) : dispatch_ell<HANKEL, false>(ell, ma, mb, ka, st);
}

}  // namespace tc

int launch_limb_gemm(const GemmArgs &a, cudaStream_t st, int *n_launches) {
  using namespace tc;
  const int N = a.kp.N, ell = a.kp.ell;
  *n_launches = 0;
  const int64_t R = a.row_end - a.row_begin;
  if (a.T == 0 || R == 0) return PHE_OK;
  if (N % BM != 0 || N % BK != 0) return PHE_EUNSUPPORTED;
  const int64_t K = a.Lc * N;
  const int tpt = BN / ell;
  const int n_tiles = (int)((a.T + tpt - 1) / tpt);
  const uint64_t brows = (uint64_t)a.op_rows;  // padded: boxes never leave the allocation
  KArgs ka{};
  ka.N = N; ka.tpt = tpt; ka.n_tiles = n_tiles; ka.k_blocks = (int)(K / BK);
  ka.kb_per_block = N / BK; ka.Lc = a.Lc; ka.cols = a.cols; ka.row_begin = a.row_begin; ka.R = R; ka.T = a.T;
  ka.out_rows = a.out_rows > 0 ? a.out_rows : R;
  ka.full_k = (a.cols == a.Lc * N) || (K / BK > 64);
  ka.q_in = a.kp.q_in; ka.out_bits = a.out_bits;
  ka.dbg = (PHE_KERNEL_EXPERIMENTS && getenv("PHE_DEBUG_EPI")) ? atoi(getenv("PHE_DEBUG_EPI")) : 0;
  // ---- body: plain W operand, M = rows in range (skipped when out_body == NULL)
  if (a.out_body) {
    CUtensorMap ma, mb;
    int rc = make_map_2d(&ma, a.wplain, (uint64_t)K, (uint64_t)a.wplain_rows, (uint64_t)K, BK, BM,
                         CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_map_2d(&mb, a.bplanes, (uint64_t)K, brows, (uint64_t)K, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    KArgs kb = ka;
    kb.tb_per_row = 1;
    kb.m_tiles = (R + BM - 1) / BM;
    kb.total_tiles = kb.m_tiles * n_tiles;
    kb.out = a.out_body;
    rc = dispatch<false>(ell, a.out_bits != a.kp.q_in, ma, mb, kb, st);
    if (rc) return rc;
    (*n_launches)++;
  }
  // ---- mask: Hankel operand, M = R * N (skipped when out_mask == NULL)
  if (a.out_mask) {
    const bool two_sm = (ell == 4 || ell == 5) && (N % (2 * BM) == 0) && !(PHE_KERNEL_EXPERIMENTS && getenv("PHE_FORCE_1SM"));
    const bool sw = a.out_bits != a.kp.q_in;
    KArgs km = ka;
    if (two_sm) km.tpt = choose_tpt(a.T, ell, &km.n_mma);
    km.n_tiles = (int)((a.T + km.tpt - 1) / km.tpt);
    {  // the last token tile holds T - (n_tiles - 1) tpt tokens: MMA N = round16 of their limb columns
      const int tail_tok = (int)(a.T - (int64_t)(km.n_tiles - 1) * km.tpt);
      int nt = ((tail_tok * ell + 15) / 16) * 16;
      if (nt < 32) nt = 32;
      km.n_mma_tail = nt < km.n_mma ? nt : km.n_mma;
    }
    CUtensorMap ma, mb, mbt, mo;
    int rc = make_map_2d(&ma, a.wexp, 16, (uint64_t)(a.rows * a.Lc * 2 * N), 16, 16, A_ROWS_HANKEL,
                         CU_TENSOR_MAP_SWIZZLE_NONE);
    if (rc) return rc;
    rc = make_map_2d(&mb, a.mplanes, (uint64_t)K, brows, (uint64_t)K, BK, two_sm ? km.n_mma / 2 : BN,
                     CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    rc = make_map_2d(&mbt, a.mplanes, (uint64_t)K, brows, (uint64_t)K, BK, two_sm ? km.n_mma_tail / 2 : BN,
                     CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    // pairs over (j, j+1) when the last block is partial (a K-window V + 127 instead of V + 255
    // wide: k/v^T at d_in = 512 issue 5 of 16 K-blocks per tile instead of 7)
    km.jpair = two_sm && !ka.full_k && R >= 2 && !(PHE_KERNEL_EXPERIMENTS && getenv("PHE_NO_JPAIR"));
    km.tb_per_row = N / (two_sm && !km.jpair ? 2 * BM : BM);
    km.m_tiles = (km.jpair ? (R + 1) / 2 : R) * km.tb_per_row;
    km.total_tiles = km.m_tiles * km.n_tiles;
    km.out = a.out_mask;
    if (a.digits && !two_sm) return PHE_EUNSUPPORTED;
    if (a.wire_words > 0 && (!two_sm || !sw || a.out_bits > WIRE_QMAX || (a.wire_words & 1) ||
                             (reinterpret_cast<uintptr_t>(a.out_mask) & 15)))
      return PHE_EUNSUPPORTED;
    if (two_sm) {
      const int tail = km.tpt % EPI_TOK ? km.tpt % EPI_TOK : EPI_TOK;
      CUtensorMap mot;
      if (a.digits) {
        rc = make_map_digits(&mo, a.out_mask, N, a.digit_rows, a.T, EPI_TOK);
        if (!rc) rc = make_map_digits(&mot, a.out_mask, N, a.digit_rows, a.T, tail);
      } else if (a.wire_words > 0) {
        rc = make_map_wire(&mo, a.out_mask, a.wire_words, a.T, 2 * a.out_bits, EPI_TOK);
        if (!rc) rc = make_map_wire(&mot, a.out_mask, a.wire_words, a.T, 2 * a.out_bits, tail);
      } else {
        rc = make_map_out(&mo, a.out_mask, sw, N, R, a.T, EPI_TOK, ka.out_rows);
        if (!rc) rc = make_map_out(&mot, a.out_mask, sw, N, R, a.T, tail, ka.out_rows);
      }
      if (rc) return rc;
      unsigned long long zero[8] = {0};
      if (km.dbg == 4) cudaMemcpyToSymbolAsync(g_dbg_cnt, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
      if (a.digits) {
        km.out_bits = KS_BITS;  // digits keep the top 32 bits (q_in >= 32)
        rc = dispatch_2sm<OUT_DIG>(ell, ma, mb, mbt, mo, mot, km, st);
      } else if (a.wire_words > 0) {
        rc = dispatch_2sm<OUT_WIRE>(ell, ma, mb, mbt, mo, mot, km, st);
      } else {
        rc = sw ? dispatch_2sm<OUT_U32>(ell, ma, mb, mbt, mo, mot, km, st)
                : dispatch_2sm<OUT_U64>(ell, ma, mb, mbt, mo, mot, km, st);
      }
      if (km.dbg == 4) {
        unsigned long long c[8];
        cudaMemcpyFromSymbolAsync(c, g_dbg_cnt, sizeof(c), 0, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st);
        const double pairs = (double)(num_sms() / 2), ntiles = (double)c[6] / (2.0 * pairs);
        fprintf(stderr, "[phe dbg] per leader: mma_total %.1fM wait_tempty %.1fM wait_full %.1fM | "
                "per CTA: producer_wait_empty %.1fM | epi(warp4): busy/tile %.0f wait/tile %.0f tiles %.0f\n",
                c[2] / pairs / 1e6, c[0] / pairs / 1e6, c[1] / pairs / 1e6, c[5] / (2 * pairs) / 1e6,
                (double)c[3] / c[6], (double)c[4] / c[6], ntiles);
      }
    } else {
      rc = dispatch<true>(ell, sw, ma, mb, km, st);
    }
    if (rc) return rc;
    (*n_launches)++;
  }
  return PHE_OK;
}

// ------------------------------------------------------------------ packing GEMM launcher
int launch_pack_gemm(const PackArgs &a, cudaStream_t st) {
  using namespace tc;
  const int N = a.N, ell = a.ell;
  if (a.T == 0) return PHE_OK;
  if (ell != 5 && ell != 4) return PHE_EUNSUPPORTED;
  if (N % (2 * BM) != 0 || a.rows_pad % (2 * BM) != 0) return PHE_EUNSUPPORTED;
  PArgs pa{};
  pa.N = N;
  pa.spt = BN / ell;
  pa.kpad = (N + pa.spt - 1) / pa.spt * pa.spt;
  pa.n_tiles = 2 * pa.kpad / pa.spt;
  pa.rows_pad = a.rows_pad;
  pa.tpt_rows = (int)(a.rows_pad / (2 * BM));
  pa.G = a.G;
  pa.total_tiles = (int64_t)a.T * pa.tpt_rows * pa.n_tiles;
  pa.m_tiles = (int64_t)a.T * pa.tpt_rows;
  // groups of 21 N-tiles (~42 MB of KSK limb planes at N = 2048) + L2 hints: measured best of
  // {11, 14, 16, 21, 28, 41, 82 (= the plain m-major order)} (profiles/r1_summary.md)
  pa.ng = 21;
  pa.hints = 1;
  if (PHE_KERNEL_EXPERIMENTS) {
    if (const char *ev = getenv("PHE_PACK_NG")) pa.ng = atoi(ev);
    if (const char *eh = getenv("PHE_PACK_HINTS")) pa.hints = atoi(eh);
  }
  if (pa.ng < 1 || pa.ng > pa.n_tiles) pa.ng = pa.n_tiles;
  pa.k_blocks = KS_LEVELS * N / BK;
  pa.acc = static_cast<unsigned long long *>(a.acc);
  CUtensorMap ma, mb;
  int rc = make_map_2d(&ma, a.digits, (uint64_t)(KS_LEVELS * N), (uint64_t)(a.T * a.rows_pad), (uint64_t)(KS_LEVELS * N), BK, BM,
                       CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_map_2d(&mb, a.kplanes, (uint64_t)(KS_LEVELS * N), (uint64_t)a.kplane_rows, (uint64_t)(KS_LEVELS * N), BK, BN / 2,
                   CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  auto kern = ell == 5 ? pack_gemm_2sm_kernel<5> : pack_gemm_2sm_kernel<4>;
  static thread_local uint64_t set5 = 0, set4 = 0;  // devices configured, per instantiation
  uint64_t &set = ell == 5 ? set5 : set4;
  if (!(set & phe_device_bit())) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, PK_SMEM) != cudaSuccess)
      return phe_set_cuda_error(cudaGetLastError());
    set |= phe_device_bit();
  }
  int64_t pairs = num_sms() / 2;
  if (pa.total_tiles < pairs) pairs = pa.total_tiles;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((unsigned)(2 * pairs));
  cfg.blockDim = dim3(NUM_THREADS);
  cfg.dynamicSmemBytes = PK_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (cudaLaunchKernelEx(&cfg, kern, ma, mb, pa) != cudaSuccess) return phe_set_cuda_error(cudaGetLastError());
  PHE_CUDA_CHECK_LAUNCH();
  return PHE_OK;
}

}  // namespace phe
