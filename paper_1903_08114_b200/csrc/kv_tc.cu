// tcgen05 (5th-generation tensor core) fused K·V kernel for sm_100a.
//
// out[i, :] = s2 * sum_j kappa(r2_ij) V[j, :]  for 128-row tiles, streaming
// 64-column tiles; the n x n kernel matrix never leaves TMEM.
//
// Per column tile j of a row tile (one CTA per SM, persistent over items):
//   1. TMA warp   : cp.async.bulk the pre-tiled column image (X_c hi/lo, with
//                   the squared norm folded in as an extra K column) and the
//                   V image [V_hi | V_lo] (tf32, 32 rows) into a 4-stage ring.
//   2. MMA thread : S = A . B^T on tcgen05 (kind::tf32, M=128, N=64), where
//                   a_i = [c x_i, -c|x_i|^2/2, -c/2], b_j = [x_j, 1, |x_j|^2]
//                   so S = -(c/2) r2 exactly in the expansion of
//                   kernels.py:216-222; 3xTF32 (hi.hi + hi.lo + lo.hi) keeps
//                   fp32 accuracy. S lands in TMEM (double buffered).
//   3. 8 epilogue warps: tcgen05.ld S, kappa on the SFU (RBF: 1 ex2;
//                   Matern: sqrt + ex2), split K = K_hi + K_lo (tf32), and
//                   tcgen05.st both back into TMEM as the A operand.
//   4. MMA thread : O = K_hi.[V_hi | V_lo] (N = 32) + K_lo.V_hi (N = 16,
//                   accumulated into the first half), A from TMEM, M=128,
//                   K=64; a fresh accumulator every tile, folded into fp32
//                   registers one tile later. Merging two 3xTF32 passes into
//                   one N = 32 instruction matters: a small-N tcgen05.mma
//                   costs ~30 cycles of issue (measured), and the 24 N = 16
//                   instructions of the unmerged contraction bound the tile.
//                   (A 2-term fp16 split halves the count again but its
//                   F2FP conversions run on the XU pipe the SFU epilogue
//                   saturates; measured slower for Matern-3/2.)
// Reference semantics: kernels.py:225-244 (kappa), :293-316 (rows of K̂),
// partition.py:224-241 (row-block product). Per-row column order is fixed by
// the column count, so row sharding across GPUs is bitwise neutral.
#include "tc_common.cuh"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>

namespace gp {
namespace tc {

constexpr int BM = 128;   // rows per tile (UMMA M)
constexpr int BN = 64;    // columns per tile (distance N, contraction K)
constexpr int TN = 16;    // right-hand sides (contraction N)
constexpr int CHUNK = 1;  // column tiles per O-accumulator flush: TMEM fp32 accumulation
                          // is lossy over long K (measured: 64 tiles -> 4e-5 rel error,
                          // 1 tile -> 5e-7), and the lagged flush hides its latency
// contraction operand format: fp16 2-term split (kind::f16, K = 16 per MMA)
// or tf32 hi/lo (kind::tf32, K = 8 per MMA); the kernel is bound by the
// single MMA-issuing thread, so halving the instruction count matters
constexpr bool KV_F16 = true;
constexpr uint32_t V_TILE = KV_F16 ? 2u * TN * BN * 2u : 2u * TN * BN * 4u;   // [V1 | V2] of one column tile
constexpr int NUM_EPI_WARPS = 16;                   // 4 per TMEM lane quarter (SMSP)
constexpr int EPI_COLS = BN / (NUM_EPI_WARPS / 4);   // columns of a tile per epilogue warp
constexpr int NTHREADS = 32 * (4 + NUM_EPI_WARPS);
constexpr int EPI_WARP0 = 4;


struct Args {
  const float* row_img;   // [row tiles][2][BM*DK]
  const float* col_img;   // [col tiles][2][BN*DK]
  const void* v_img;      // [col tiles][32 x 64] [V1 | V2] (fp16 or tf32)
  const float* inv_vscale; // [TN] 2^-s_c (fp16 image scaling)
  const float* dscale;    // TS: S = S' dscale (fp16 distance images, points_image16_kernel)
  int DK;
  int64_t n_rows, n_cols;
  int row_tiles, col_tiles, splits, tiles_per_split;
  int nstages;
  int fam;
  int t;
  float s2, noise;
  int64_t diag_offset;
  int64_t self_offset;
  const float* V; int64_t ldv;
  float* out; int64_t ldo;
  int64_t split_stride;   // 0 = final output
  int chunk;              // column tiles per O flush
  int lookahead;          // distance MMAs issued this many tiles ahead (<= nstages - 1)
  long long* prof;        // optional per-warp wait counters (GP_TC_PROF=1, diagnostic)
};

#define TC_T(slot, ...)                                   \
  do {                                                    \
    const long long _t0 = a.prof ? clock64() : 0;         \
    __VA_ARGS__;                                          \
    if (a.prof) tacc[slot] += clock64() - _t0;            \
  } while (0)

// ---------------------------------------------------------------------------
// image preparation (fp64 arithmetic, tf32 hi/lo split)
// ---------------------------------------------------------------------------
// role 0: row image a_i = [c x_i, -c |x_i|^2 / 2, -c/2]   (R = BM)
// role 1: col image b_j = [x_j, 1, |x_j|^2]               (R = BN)
// column means (fp64) of the prescaled points: both sides are shifted by the
// same vector (translation invariance of r2), which shrinks |x|^2 and with it
// the cancellation of the expansion |a|^2 + |b|^2 - 2ab in fp32.
// per-column mean of X (n x d, d <= 1024): an 8-CTA cluster splits the rows,
// each CTA reduces its rows in a fixed thread order, and CTA 0 adds the
// CTAs' partials through distributed shared memory in rank order, so the
// result is deterministic without a global workspace (one CTA per column
// read the column with an ldx stride and took ~0.5 ms at n = 10^6)
constexpr int kColClusterCtas = 8;
__global__ void __cluster_dims__(kColClusterCtas, 1, 1) __launch_bounds__(1024)
    column_mean_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int d, double* mean) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  __shared__ double red[1024];
  __shared__ double part[1024];
  const int rank = (int)cl.block_rank(), nb = (int)cl.num_blocks();
  const int64_t per = (n + nb - 1) / nb;
  const int64_t r0 = min(n, (int64_t)rank * per), r1 = min(n, r0 + per);
  const int rpp = (int)blockDim.x / d;
  const int tr = (int)threadIdx.x / d, tc = (int)threadIdx.x - tr * d;
  double acc = 0.0;
  if (tr < rpp)
#pragma unroll 8  // loads of later rows issue ahead of the dependent adds
    for (int64_t r = r0 + tr; r < r1; r += rpp) acc += (double)X[r * ldx + tc];
  red[threadIdx.x] = acc;
  __syncthreads();
  if ((int)threadIdx.x < d) {
    double sum = 0.0;
    for (int q = 0; q < rpp; ++q) sum += red[q * d + threadIdx.x];
    part[threadIdx.x] = sum;
  }
  cl.sync();
  if (rank == 0 && (int)threadIdx.x < d) {
    double tot = 0.0;
    for (int b = 0; b < nb; ++b) tot += *cl.map_shared_rank(&part[threadIdx.x], b);
    mean[threadIdx.x] = n > 0 ? tot / (double)n : 0.0;
  }
  cl.sync();   // peers' shared memory stays alive until CTA 0 has read it
}

// role 0: row image a_i = [c y_i, -c |y_i|^2 / 2, -c/2]   (R = BM)
// role 1: col image b_j = [y_j, 1, |y_j|^2]               (R = BN)
// with y = x - mean (fp64), split into tf32 hi + lo.
__global__ void points_image_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int d, int DK,
                                    int R, int role, double c, const double* __restrict__ mean,
                                    float* img, int64_t ntiles) {
  int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= ntiles * R) return;
  int64_t tile = row / R;
  int r = (int)(row - tile * R);
  float* hi = img + tile * 2 * (int64_t)R * DK;
  float* lo = hi + (int64_t)R * DK;
  double nrm = 0.0;
  bool valid = row < n;
  if (valid)
    for (int k = 0; k < d; ++k) {
      double x = (double)X[row * ldx + k] - mean[k];
      nrm += x * x;
    }
  for (int k = 0; k < DK; ++k) {
    double v = 0.0;
    if (valid) {
      if (k < d) v = ((double)X[row * ldx + k] - mean[k]) * (role == 0 ? c : 1.0);
      else if (k == d) v = role == 0 ? -0.5 * c * nrm : 1.0;
      else if (k == d + 1) v = role == 0 ? -0.5 * c : nrm;
    }
    float h = tf32_rna((float)v);
    float l = (float)(v - (double)h);
    hi[canon(r, k, R)] = h;
    lo[canon(r, k, R)] = l;
  }
}

// Large d (TS mode): the augmented points as fp16 hi + lo (22 significant
// bits, like tf32 hi + lo) in the 16-bit canonical layout, so the distance
// product runs at the f16 rate and a column tile takes half the SMEM. fp16
// needs a range: each side is scaled by one power of two 2^-e chosen from the
// largest |value| of that side (|value| 2^-e <= 2^14), and the epilogue
// multiplies S by 2^(e_row + e_col) (`dscale`).
// rng[0..1] = max |y_k|, max |y|^2 over the points (y = x - mean), as fp32
// bits (non-negative floats order as integers: atomicMax)
__global__ void points_range_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int d,
                                    const double* __restrict__ mean, unsigned* rng) {
  float m1 = 0.f, m2 = 0.f;
  for (int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; row < n;
       row += (int64_t)gridDim.x * blockDim.x) {
    double nrm = 0.0, mx = 0.0;
    for (int k = 0; k < d; ++k) {
      const double y = (double)X[row * ldx + k] - mean[k];
      nrm += y * y;
      mx = fmax(mx, fabs(y));
    }
    m1 = fmaxf(m1, (float)mx);
    m2 = fmaxf(m2, (float)nrm);
  }
  for (int o = 16; o > 0; o >>= 1) {
    m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, o));
    m2 = fmaxf(m2, __shfl_xor_sync(0xffffffffu, m2, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&rng[0], __float_as_uint(m1));
    atomicMax(&rng[1], __float_as_uint(m2));
  }
}

// exponent e of one side: the largest |value| of its image times 2^-e is <= 2^14
__device__ __forceinline__ int image_exp16(int role, double c, const unsigned* rng) {
  const double m1 = __uint_as_float(rng[0]), m2 = __uint_as_float(rng[1]);
  const double M = role == 0 ? fmax(fabs(c) * m1, fmax(0.5 * fabs(c) * m2, 0.5 * fabs(c))) : fmax(fmax(m1, m2), 1.0);
  int ex;
  frexp(M, &ex);   // M < 2^ex
  return ex - 14;
}

__global__ void points_image16_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int d, int DK, int R,
                                      int role, double c, const double* __restrict__ mean, const unsigned* rng,
                                      const unsigned* rng_other, __half* img, int64_t ntiles, float* dscale) {
  const int e = image_exp16(role, c, rng);
  if (dscale && blockIdx.x == 0 && threadIdx.x == 0)   // S = S' 2^(e_row + e_col)
    *dscale = ldexpf(1.f, e + image_exp16(1 - role, role == 0 ? 1.0 : c, rng_other));
  int64_t row = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= ntiles * R) return;
  int64_t tile = row / R;
  int r = (int)(row - tile * R);
  __half* hi = img + tile * 2 * (int64_t)R * DK;
  __half* lo = hi + (int64_t)R * DK;
  double nrm = 0.0;
  bool valid = row < n;
  if (valid)
    for (int k = 0; k < d; ++k) {
      double x = (double)X[row * ldx + k] - mean[k];
      nrm += x * x;
    }
  for (int k = 0; k < DK; ++k) {
    double v = 0.0;
    if (valid) {
      if (k < d) v = ((double)X[row * ldx + k] - mean[k]) * (role == 0 ? c : 1.0);
      else if (k == d) v = role == 0 ? -0.5 * c * nrm : 1.0;
      else if (k == d + 1) v = role == 0 ? -0.5 * c : nrm;
    }
    v = ldexp(v, -e);
    const __half h = __double2half(v);
    hi[canon16(r, k, R)] = h;
    lo[canon16(r, k, R)] = __double2half(v - (double)__half2float(h));
  }
}

// ---------------------------------------------------------------------------
// the fused kernel
//   TMEM: S_0..2 (3 x 64 cols, distance accumulators, 2 tiles of look-ahead),
//         K_0..1 (hi 64 + lo 64 cols each, contraction A operand),
//         O_0..1 (32 cols each = [K_hi V_hi + K_lo V_hi | K_hi V_lo]).
//   Barriers: full/empty (SMEM ring), s_full[3] (MMA -> epilogue),
//   k_full[2] (epilogue -> MMA), k_empty[2] (MMA -> epilogue, contraction
//   done reading K), o_full/o_empty[2], xr_full/xr_empty (row image).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t TMS(uint32_t b) { return b * 64; }           // 0, 64, 128
// TS mode: S buffers 0, 1 at [0, 128) and the third past the fp16 row image
// (DK <= 96 columns from TMXA = 320), at [416, 480)
__device__ __forceinline__ uint32_t TMS_TS(uint32_t b) { return b < 2 ? b * 64 : 416u; }
// TMEM layouts (columns):            S            K (x2)       O (x2)     row image
//   SS distance (3 S buffers):   [0, 192)     192 + 128b   [448, 512)   -
//   TS distance (3 S buffers):   [0, 128) + [416, 480)   [128, 256)   [256, 320)   [320, 320 + DK) (fp16 pairs)
// K buffer b, fp16 pairs: K1 [tm_k + 64b, +32) | K2 [+32, +64); tf32 (SS only): hi 64 | lo 64
#define TMKH(b) ((TS ? 128u : 192u) + (uint32_t)(b) * (TS ? 64u : 128u))
#define TMKL(b) (TMKH(b) + (KV_F16 ? 32u : 64u))
#define TMO(c) ((TS ? 256u : 448u) + (uint32_t)(c) * 32u)
#define TMXA 320u

template <int FAM, bool TS>
__global__ void __launch_bounds__(NTHREADS, 1) kv_tc_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int DK = a.DK;
  constexpr uint32_t EB = TS ? 2u : 4u;   // bytes per image element (TS: fp16, else tf32)
  const uint32_t row_bytes = 2u * BM * DK * EB;
  const uint32_t col_bytes = 2u * BN * DK * EB;
  const uint32_t v_bytes = V_TILE;
  const uint32_t stage_bytes = col_bytes + v_bytes;
  const int NS = a.nstages;
  uint8_t* xr_s = smem;                          // SS only: the row image (TS: TMEM, copied from global)
  uint8_t* stages = smem + (TS ? 0u : row_bytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * stage_bytes);
  uint64_t* full = bars;             // [NS]
  uint64_t* empty = bars + NS;       // [NS]
  uint64_t* s_full = bars + 2 * NS;  // [3]
  uint64_t* k_full = s_full + 3;     // [2]
  uint64_t* k_empty = k_full + 2;    // [2]
  uint64_t* o_full = k_empty + 2;    // [2]
  uint64_t* o_empty = o_full + 2;    // [2]
  uint64_t* xr_full = o_empty + 2;   // [1]
  uint64_t* xr_empty = xr_full + 1;  // [1]
  uint64_t* xa_full = xr_empty + 1;  // [1] row image copied into TMEM (TS mode)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xa_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 3; ++b) mbar_init(smem_u32(&s_full[b]), 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&k_full[b]), NUM_EPI_WARPS / 2);
      mbar_init(smem_u32(&k_empty[b]), 1);
      mbar_init(smem_u32(&o_full[b]), 1);
      mbar_init(smem_u32(&o_empty[b]), 4);
    }
    mbar_init(smem_u32(xr_full), 1);
    mbar_init(smem_u32(xr_empty), 1);
    mbar_init(smem_u32(xa_full), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();

  const int n_items = a.row_tiles * a.splits;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0, itc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
        const int rt = it / a.splits, sp = it - rt * a.splits;
        const int ct0 = sp * a.tiles_per_split;
        const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
        if (!TS) {   // TS: the epilogue copies the row image from global memory into TMEM
          mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
          mbar_expect_tx(smem_u32(xr_full), row_bytes);
          bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)rt * (row_bytes / 4), row_bytes, smem_u32(xr_full));
        }
        const float* cimg = a.col_img + (int64_t)ct0 * (col_bytes / 4);
        const uint8_t* vimg = static_cast<const uint8_t*>(a.v_img) + (int64_t)ct0 * v_bytes;
        for (int ct = ct0; ct < ct1; ++ct) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          uint8_t* st = stages + s * stage_bytes;
          mbar_expect_tx(smem_u32(&full[s]), stage_bytes);
          bulk_g2s(smem_u32(st), cimg, col_bytes, smem_u32(&full[s]));
          bulk_g2s(smem_u32(st + col_bytes), vimg, v_bytes, smem_u32(&full[s]));
          cimg += col_bytes / 4;
          vimg += v_bytes;
          if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // The whole warp runs the (warp-uniform) control flow so bookkeeping
    // lives in uniform registers; one elected lane issues tcgen05 ops.
    // Descriptors are built once; per-MMA work is a 32-bit add on the
    // start-address field (addresses advance in 16-byte units).
    const uint32_t idesc_d = TS ? idesc_f16(BM, BN) : make_idesc(BM, BN);
    const uint32_t idesc_c32 = KV_F16 ? idesc_f16(BM, 2 * TN) : make_idesc(BM, 2 * TN);
    const uint32_t idesc_c16 = KV_F16 ? idesc_f16(BM, TN) : make_idesc(BM, TN);
    const uint32_t lbo_a = (BM / 8) * 128, lbo_b = (BN / 8) * 128, lbo_v = (2 * TN / 8) * 128;
    const uint32_t a_half16 = (BM * DK * EB) >> 4, b_half16 = (BN * DK * EB) >> 4;
    const int ksteps = TS ? DK / 16 : DK / 8;   // K per MMA: 16 fp16 / 8 tf32 (both 32 B per row)
    const uint64_t da0 = make_desc(smem_u32(xr_s), lbo_a, 128);
    const uint64_t db0 = make_desc(smem_u32(stages), lbo_b, 128);
    const uint64_t dv0 = make_desc(smem_u32(stages + col_bytes), lbo_v, 128);
    const uint32_t stage16 = stage_bytes >> 4;
    const uint32_t kstep_a16 = (2 * lbo_a) >> 4, kstep_b16 = (2 * lbo_b) >> 4, kstep_v16 = (2 * lbo_v) >> 4;
    const bool leader = elect_one();
    // distance-stage ring position (ahead of the contraction by LA tiles)
    uint32_t ds = 0, dph = 0;      // stage / phase for the next dist()
    uint32_t cs = 0;               // stage of the next contraction
    uint32_t sb_next = 0, sph_unused = 0;
    (void)sph_unused;
    uint32_t kb = 0, kph = 0;      // K buffer / phase of the next contraction
    uint32_t oc = 0, oph = 0;      // O buffer / phase
    uint32_t itc = 0;
    const int LA = a.lookahead;    // 1 or 2; the SMEM ring needs LA + 1 stages
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      const int sp = it % a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      const int J = ct1 - ct0;
      if (TS) mbar_wait(smem_u32(xa_full), itc & 1);
      else mbar_wait(smem_u32(xr_full), itc & 1);
      tc_fence_after();
      auto dist = [&]() {
        TC_T(0, mbar_wait(smem_u32(&full[ds]), dph));
        tc_fence_after();
        const uint32_t d_tm = tmem + (TS ? TMS_TS(sb_next) : TMS(sb_next));
        const uint64_t db = db0 + (uint64_t)(ds * stage16);
        if (leader) {
          if (TS) {
#pragma unroll
            // fp16 pairs: hi at TMXA, lo at TMXA + DK/2 (one kstep = 8 columns)
            for (int pass = 0; pass < 3; ++pass) {
              const uint32_t a_t = tmem + TMXA + (pass == 0 ? (uint32_t)(DK / 2) : 0u);
              const uint64_t b_p = db + (pass == 1 ? b_half16 : 0u);
              for (int ks = 0; ks < ksteps; ++ks)
                mma16_ts(d_tm, a_t + ks * 8, b_p + (uint64_t)(ks * kstep_b16), idesc_d, (pass | ks) != 0);
            }
          } else {
#pragma unroll
            for (int pass = 0; pass < 3; ++pass) {
              const uint64_t a_p = da0 + (pass == 0 ? a_half16 : 0u);
              const uint64_t b_p = db + (pass == 1 ? b_half16 : 0u);
              for (int ks = 0; ks < ksteps; ++ks)
                mma_ss(d_tm, a_p + (uint64_t)(ks * kstep_a16), b_p + (uint64_t)(ks * kstep_b16), idesc_d,
                       (pass | ks) != 0);
            }
          }
        }
        if (leader) {
          tc_commit(smem_u32(&s_full[sb_next]));
        }
        __syncwarp();
        if (++ds == (uint32_t)NS) { ds = 0; dph ^= 1; }
        if (++sb_next == 3u) sb_next = 0;
      };
      for (int jj = 0; jj < LA && jj < J; ++jj) dist();
      for (int jj = 0; jj < J; ++jj) {
        // S buffer of tile jj+LA was last read by the epilogue for tile
        // jj+LA-3 <= jj-1, whose k_full we waited for already
        if (jj + LA < J) dist();
        TC_T(1, mbar_wait(smem_u32(&k_full[kb]), kph));
        tacc[7] += 1;
        tc_fence_after();
        TC_T(2, mbar_wait(smem_u32(&o_empty[oc]), oph ^ 1));  // chunk = 1 tile
        tc_fence_after();
        const uint64_t vb = dv0 + (uint64_t)(cs * stage16);
        const uint32_t o_tm = tmem + TMO(oc);
        const uint32_t khi = tmem + TMKH(kb), klo = tmem + TMKL(kb);
        if (leader) {
          // O = K_hi.[V_hi | V_lo];  O[:, 0:16] += K_lo.V_hi  (fresh accumulator every tile)
          if constexpr (KV_F16) {
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks)
              mma16_ts(o_tm, khi + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c32, ks != 0);
#pragma unroll
            for (int ks = 0; ks < BN / 16; ++ks)
              mma16_ts(o_tm, klo + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c16, 1);
          } else {
#pragma unroll
            for (int ks = 0; ks < BN / 8; ++ks)
              mma_ts(o_tm, khi + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c32, ks != 0);
#pragma unroll
            for (int ks = 0; ks < BN / 8; ++ks)
              mma_ts(o_tm, klo + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c16, 1);
          }
        }
        if (leader) {
          tc_commit(smem_u32(&empty[cs]));
          tc_commit(smem_u32(&k_empty[kb]));
          tc_commit(smem_u32(&o_full[oc]));
        }
        __syncwarp();
        if (++cs == (uint32_t)NS) cs = 0;
        if (++kb == 2) { kb = 0; kph ^= 1; }
        if (++oc == 2) { oc = 0; oph ^= 1; }
      }
      if (leader) tc_commit(smem_u32(xr_empty));
      __syncwarp();
    }
  } else if (warp >= EPI_WARP0) {
    // ===================== epilogue (16 warps, two groups) =====================
    // Group g = (warp - 4) / 8 takes the tiles of parity g (global tile count
    // of this CTA), so one group's SFU phase overlaps the other's TMEM store /
    // barrier tail; tile parity also selects the K and O buffers, so each
    // group owns K[g], O[g]. Within a group two warps per TMEM lane quarter
    // cover 32 columns each, in two 16-column chunks (register budget).
    const int e = warp - EPI_WARP0;
    const int g = e >> 3;                      // tile parity group
    const int q = warp & 3;                    // TMEM lane quarter
    const int half = (e >> 2) & 1;             // column half of the 64-col tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t T = 0;                            // tiles seen by this CTA (both groups)
    uint32_t kuse = 0, ouse = 0;               // uses of K[g] / O[g] by this group
    float acc[TN];
    float* comb = reinterpret_cast<float*>(tmem_slot + 4);   // [BM][TN] group-1 partials
    // Every tile's product lands in a fresh TMEM accumulator (tensor-core fp32
    // accumulation over long K is lossy); slice-0 warps fold it into fp32
    // registers one group-tile later, when it is long complete.
    int pending = 0;
    auto flush = [&]() {
      TC_T(2, mbar_wait(smem_u32(&o_full[g]), (ouse - 1) & 1));
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + TMO(g), o);
      tmem_wait_ld();
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[c] += __uint_as_float(o[c]) + __uint_as_float(o[c + TN]);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&o_empty[g]));
      pending = 0;
    };
    uint32_t itc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      const int rt = it / a.splits, sp = it - rt * a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      const int J = ct1 - ct0;
      const int64_t my_row = (int64_t)rt * BM + q * 32 + lane;
      const int64_t diag_col = (a.self_offset >= 0 && my_row < a.n_rows) ? my_row + a.self_offset : -1000;
      if (TS && g == 0 && half == 0) {
        // TS mode: row image hi | lo -> TMEM (A operand of the distance
        // product), read straight from global memory (once per row item; the
        // SMEM it would take holds two more column stages instead).
        // xr_empty of the previous item: its MMAs have completed.
        mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
        const __half* xr = reinterpret_cast<const __half*>(a.row_img) + (int64_t)rt * (2 * BM * DK);
        const int i_loc = q * 32 + lane;
        for (int part = 0; part < 2; ++part)
          for (int k0 = 0; k0 < DK; k0 += 16) {
            uint32_t w[8];   // 16 fp16 along K = 8 TMEM columns (one kstep)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              w[kk] = *reinterpret_cast<const uint32_t*>(xr + part * BM * DK + canon16(i_loc, k0 + 2 * kk, BM));
            tmem_st8(tmem + lane_base + TMXA + part * (DK / 2) + k0 / 2, w);
          }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(xa_full));
      }
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[c] = 0.f;
      for (int jj = 0; jj < J; ++jj, ++T) {
        if ((int)(T & 1) != g) continue;
        const uint32_t sb = T % 3u, sph = (T / 3u) & 1;
        TC_T(0, mbar_wait(smem_u32(&s_full[sb]), sph));
        tacc[7] += 1;
        tc_fence_after();
        // this warp's 32 columns in one TMEM load (one round trip per tile)
        const int c0 = half * 32;
        uint32_t v[32];
        TC_T(3, tmem_ld32(tmem + lane_base + (TS ? TMS_TS(sb) : TMS(sb)) + c0, v); tmem_wait_ld());
        {
          const int64_t e_diag = diag_col - ((int64_t)(ct0 + jj) * BN + c0);
          // self-diagonal entry (same point on both sides): r2 = 0 exactly
          if (__any_sync(0xffffffffu, e_diag >= 0 && e_diag < 32)) {
#pragma unroll
            for (int k = 0; k < 32; ++k)
              if (k == e_diag) v[k] = 0u;
          }
        }
        const long long tk0 = a.prof ? clock64() : 0;
        {
          const float dsc = TS ? *a.dscale : 1.f;
#pragma unroll
          for (int k = 0; k < 32; ++k) {
            float sv = TS ? __uint_as_float(v[k]) * dsc : __uint_as_float(v[k]);
            float kap;
            // clamps written as selects so NaN inputs propagate (the
            // reference raises on non-finite blocks, partition.py:231-236)
            if (KV_F16) {
              kap = kappa_split_scaled<FAM>(sv);   // x 2^12, divided out by inv_vscale
            } else if (FAM == GP_FAMILY_RBF) {
              kap = ex2_approx(min0_nan(sv));  // S = -log2(e) r2 / 2
            } else {
              float u = sqrt_approx(max0_nan(sv));  // S = 3 r2, u = sqrt(3) r
              float ex = ex2_approx(u * -kLog2e);
              kap = fmaf(u, ex, ex);                       // (1 + sqrt3 r) e^{-sqrt3 r}
            }
            v[k] = __float_as_uint(kap);
          }
        }
        if (a.prof) { v[0] |= (uint32_t)(clock64() == 0); tacc[4] += clock64() - tk0; }
        // K[g] was last read by this group's previous contraction
        TC_T(1, mbar_wait(smem_u32(&k_empty[g]), (kuse & 1) ^ 1));
        ++kuse;
        tc_fence_after();
        if constexpr (KV_F16) {
#pragma unroll
          for (int s16 = 0; s16 < 2; ++s16) {
            uint32_t p1[8], p2[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
              split_pair(__uint_as_float(v[16 * s16 + 2 * k]), __uint_as_float(v[16 * s16 + 2 * k + 1]), p1[k], p2[k]);
            tmem_st8(tmem + lane_base + TMKH(g) + c0 / 2 + 8 * s16, p1);
            tmem_st8(tmem + lane_base + TMKL(g) + c0 / 2 + 8 * s16, p2);
          }
        } else {
#pragma unroll
          for (int s16 = 0; s16 < 2; ++s16) {
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              hi[k] = v[16 * s16 + k] & 0xFFFFE000u;
              lo[k] = __float_as_uint(__uint_as_float(v[16 * s16 + k]) - __uint_as_float(hi[k]));
            }
            tmem_st16(tmem + lane_base + TMKH(g) + c0 + 16 * s16, hi);
            tmem_st16(tmem + lane_base + TMKL(g) + c0 + 16 * s16, lo);
          }
        }
        TC_T(5, tmem_wait_st());
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&k_full[g]));
        if (half == 0) {
          if (pending) flush();
          pending = 1;
          ++ouse;
        }
      }
      if (half == 0) {
        if (pending) flush();
        // combine the two groups' partial row sums (named barrier over the 8
        // slice-0 warps of both groups)
        if (g == 1) {
#pragma unroll
          for (int c = 0; c < TN; ++c) comb[(q * 32 + lane) * TN + c] = acc[c];
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (g == 0) {
#pragma unroll
          for (int c = 0; c < TN; ++c) acc[c] += comb[(q * 32 + lane) * TN + c];
          const int64_t row = my_row;
          if (row < a.n_rows) {
            float* dst = a.split_stride ? a.out + (int64_t)sp * a.split_stride + row * a.t
                                        : a.out + row * a.ldo;
#pragma unroll
            for (int c = 0; c < TN; ++c) {
              if (c < a.t) {
                float r = KV_F16 ? acc[c] * __ldg(&a.inv_vscale[c]) : acc[c];
                if (!a.split_stride) {
                  r *= a.s2;
                  if (a.diag_offset >= 0) r = fmaf(a.noise, a.V[(row + a.diag_offset) * a.ldv + c], r);
                }
                dst[c] = r;
              }
            }
          }
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
    }
  }

  if (a.prof && lane == 0) {
    tacc[6] = clock64() - t_start;
    for (int k = 0; k < 8; ++k) a.prof[((int64_t)blockIdx.x * (NTHREADS / 32) + warp) * 8 + k] = tacc[k];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// Row and column images of the augmented points for the distance MMA
// (shared by the K·V and gradient kernels): c = -6 gives S = 3 r2 (Matern),
// c = log2(e) gives S = -log2(e) r2 / 2 (RBF).
int distance_images(const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
                    int d, int DK, int BMr, int BNc, double c, double* mean, float* row_img,
                    float* col_img, cudaStream_t st) {
  column_mean_kernel<<<kColClusterCtas, 1024, 0, st>>>(Xc, ldc, nc, d, mean);
  GP_LAUNCH_CHECK();
  int64_t row_tiles = (nr + BMr - 1) / BMr, col_tiles = (nc + BNc - 1) / BNc;
  int64_t rows = row_tiles * BMr;
  points_image_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(Xr, ldr, nr, d, DK, BMr, 0, c, mean,
                                                                     row_img, row_tiles);
  GP_LAUNCH_CHECK();
  int64_t cols = col_tiles * BNc;
  points_image_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(Xc, ldc, nc, d, DK, BNc, 1, 1.0, mean,
                                                                     col_img, col_tiles);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

// fp16 images of the large-d path: column means, the two sides' ranges,
// then the scaled hi | lo images; dscale = 2^(e_row + e_col)
int distance_images16(const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
                      int d, int DK, int BMr, int BNc, double c, double* mean, unsigned* rng, __half* row_img,
                      __half* col_img, float* dscale, cudaStream_t st) {
  column_mean_kernel<<<kColClusterCtas, 1024, 0, st>>>(Xc, ldc, nc, d, mean);
  GP_LAUNCH_CHECK();
  GP_CUDA_TRY(cudaMemsetAsync(rng, 0, 4 * sizeof(unsigned), st));
  const bool same = Xr == Xc && ldr == ldc && nr == nc;
  auto range = [&](const float* X, int64_t ld, int64_t n, unsigned* out) -> int {
    if (n <= 0) return GP_OK;
    const unsigned nb = (unsigned)std::min<int64_t>((n + 255) / 256, 4LL * num_sms());
    points_range_kernel<<<nb, 256, 0, st>>>(X, ld, n, d, mean, out);
    GP_LAUNCH_CHECK();
    return GP_OK;
  };
  if (int rc = range(Xc, ldc, nc, rng + 2)) return rc;
  if (same) GP_CUDA_TRY(cudaMemcpyAsync(rng, rng + 2, 2 * sizeof(unsigned), cudaMemcpyDeviceToDevice, st));
  else if (int rc = range(Xr, ldr, nr, rng)) return rc;
  int64_t row_tiles = (nr + BMr - 1) / BMr, col_tiles = (nc + BNc - 1) / BNc;
  int64_t rows = row_tiles * BMr, cols = col_tiles * BNc;
  points_image16_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, st>>>(Xr, ldr, nr, d, DK, BMr, 0, c, mean, rng,
                                                                       rng + 2, row_img, row_tiles, dscale);
  GP_LAUNCH_CHECK();
  points_image16_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(Xc, ldc, nc, d, DK, BNc, 1, 1.0, mean,
                                                                       rng + 2, rng, col_img, col_tiles, nullptr);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

// V image: per 64-point tile a 32-row K-major fp16 operand (canonical
// no-swizzle layout, core = 8 rows x 8 halves): rows 0-15 V1 = fp16(2^s V),
// rows 16-31 V2 = fp16(2^s V - V1), so one N = 32 MMA forms K1.V1 and K1.V2
__global__ void v_image16_kernel(const float* __restrict__ V, int64_t ldv, int t, int64_t ncols,
                                 const float* __restrict__ vscale, __half* img, int64_t ntiles) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * BN * TN) return;
  int64_t tile = idx / (BN * TN);
  int rem = (int)(idx - tile * BN * TN);
  int k = rem / TN, nn = rem - k * TN;
  int64_t col = tile * BN + k;
  float v = (col < ncols && nn < t) ? V[col * ldv + nn] * vscale[nn] : 0.f;
  __half h1 = __float2half_rn(v);
  __half h2 = __float2half_rn(v - __half2float(h1));
  __half* base = img + tile * (2 * TN * BN);
  base[canon16(nn, k, 2 * TN)] = h1;
  base[canon16(TN + nn, k, 2 * TN)] = h2;
}

// V image for the contraction: per column tile a 32-row K-major tf32 operand,
// rows 0-15 V_hi, rows 16-31 V_lo, so one N = 32 MMA forms K_hi.V_hi and K_hi.V_lo
__global__ void v_image32_kernel(const float* __restrict__ V, int64_t ldv, int t, int64_t ncols, float* img,
                                 int64_t ntiles) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * BN * TN) return;
  int64_t tile = idx / (BN * TN);
  int rem = (int)(idx - tile * BN * TN);
  int k = rem / TN, nn = rem - k * TN;
  int64_t col = tile * BN + k;
  float v = (col < ncols && nn < t) ? V[col * ldv + nn] : 0.f;
  float h = tf32_rna(v);
  float* base = img + tile * 2 * BN * TN;
  base[canon(nn, k, 2 * TN)] = h;
  base[canon(TN + nn, k, 2 * TN)] = v - h;
}

int v_images32(const float* V, int64_t ldv, int t, int64_t ncols, float* img, int64_t ntiles, cudaStream_t st) {
  int64_t tot = ntiles * BN * TN;
  v_image32_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, ldv, t, ncols, img, ntiles);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int v_images16(const float* V, int64_t ldv, int t, int64_t ncols, const float* vscale, __half* img,
               int64_t ntiles, cudaStream_t st) {
  int64_t tot = ntiles * BN * TN;
  v_image16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, ldv, t, ncols, vscale, img, ntiles);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

__global__ void v_colscale_kernel(const float* __restrict__ V, int64_t ldv, int64_t n, int t, float* vscale,
                                  float* inv_vscale) {
  __shared__ float mx[256];
  const int c = blockIdx.x;
  float m = 0.f;
  if (c < t)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) m = fmaxf(m, fabsf(V[i * ldv + c]));
  mx[threadIdx.x] = m;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) mx[threadIdx.x] = fmaxf(mx[threadIdx.x], mx[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int S = 0;
    if (mx[0] > 0.f && mx[0] < INFINITY) {
      int ex;
      frexpf(mx[0], &ex);   // max < 2^ex
      S = max(-100, min(100, 14 - ex));
    }
    vscale[c] = ldexpf(1.0f, S);
    inv_vscale[c] = ldexpf(1.0f, -S - kKScaleLog2);   // also undoes the 2^12 K scaling of the fp16 split
  }
}

// V image for the wide kernel: rows 0..NW-1 V1, NW..2NW-1 V2 (canonical, 2NW rows)
__global__ void v_image16w_kernel(const float* __restrict__ V, int64_t ldv, int t, int NW, int64_t ncols,
                                  const float* __restrict__ vscale, __half* img, int64_t ntiles, int TP) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * TP * NW) return;
  int64_t tile = idx / (TP * NW);
  int rem = (int)(idx - tile * TP * NW);
  int k = rem / NW, nn = rem - k * NW;
  int64_t col = tile * TP + k;
  float v = (col < ncols && nn < t) ? V[col * ldv + nn] * vscale[nn] : 0.f;
  __half h1 = __float2half_rn(v);
  __half h2 = __float2half_rn(v - __half2float(h1));
  __half* base = img + tile * (2 * NW * TP);
  base[canon16(nn, k, 2 * NW)] = h1;
  base[canon16(NW + nn, k, 2 * NW)] = h2;
}

int v_images16_wide(const float* V, int64_t ldv, int t, int NW, int64_t ncols, const float* vscale, __half* img,
                    int64_t ntiles, cudaStream_t st, int tile_points) {
  int64_t tot = ntiles * tile_points * NW;
  v_image16w_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, ldv, t, NW, ncols, vscale, img, ntiles,
                                                                   tile_points);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int v_colscale(const float* V, int64_t ldv, int64_t n, int t, float* vscale, float* inv_vscale, cudaStream_t st) {
  v_colscale_kernel<<<std::max(t, TN), 256, 0, st>>>(V, ldv, n, t, vscale, inv_vscale);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

struct Plan {
  int DK, row_tiles, col_tiles, splits, tiles_per_split, nstages;
  size_t row_img_bytes, col_img_bytes, v_img_bytes, split_bytes, smem;
};

static Plan make_plan(const gp_kv_desc* d, int t) {
  Plan p;
  p.DK = (d->d + 2 + 7) / 8 * 8;
  p.row_tiles = (int)((d->n_rows + BM - 1) / BM);
  p.col_tiles = (int)((d->n_cols + BN - 1) / BN);
  // column splits depend on the column count only for the square training
  // operator (bitwise-identical rows under any row sharding)
  int64_t hint_rows = (d->diag_offset >= 0 || d->self_offset >= 0 || d->Xr == d->Xc) ? d->n_cols : d->n_rows;
  int64_t hint_tiles = (hint_rows + BM - 1) / BM;
  int64_t target = 2LL * num_sms();
  int64_t s = (target + hint_tiles - 1) / hint_tiles;
  s = std::max<int64_t>(1, std::min<int64_t>({s, 64, (int64_t)p.col_tiles}));
  p.tiles_per_split = (int)((p.col_tiles + s - 1) / s);
  p.splits = (p.col_tiles + p.tiles_per_split - 1) / p.tiles_per_split;
  p.row_img_bytes = (size_t)p.row_tiles * 2 * BM * p.DK * 4;
  p.col_img_bytes = (size_t)p.col_tiles * 2 * BN * p.DK * 4;
  p.v_img_bytes = (size_t)p.col_tiles * V_TILE;
  p.split_bytes = (p.splits > 1 ? (size_t)p.splits * d->n_rows * t * 4 : 0) + 256 * sizeof(double) +
                  2 * TN * sizeof(float) + 8 * sizeof(float);
  // TS mode (KV_F16, DK >= 48): the row image lives in TMEM, copied there
  // from global memory, so its SMEM goes to the column ring
  const bool ts = KV_F16 && p.DK >= 48;
  size_t row_b = ts ? 0 : 2u * BM * p.DK * 4, stage_b = 2u * BN * p.DK * (ts ? 2 : 4) + V_TILE;
  size_t budget = 220 * 1024 - row_b - 256 - BM * TN * 4;
  p.nstages = (int)std::min<size_t>(ts ? 6 : 4, budget / stage_b);
  p.smem = row_b + p.nstages * stage_b + 256 + BM * TN * 4;
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace tc

bool kv_tc_supported(const gp_kv_desc* d, int t) {
  if (t < 1 || t > tc::TN) return false;
  if (d->d < 1 || d->d + 2 > 96) return false;
  return tc::make_plan(d, t).nstages >= 2;
}

size_t kv_tc_workspace(const gp_kv_desc* d, int t) {
  if (!kv_tc_supported(d, t)) return 0;
  tc::Plan p = tc::make_plan(d, t);
  return tc::align256(p.row_img_bytes) + tc::align256(p.col_img_bytes) + tc::align256(p.v_img_bytes) +
         tc::align256(p.split_bytes);
}

int kv_tc(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo, void* ws,
          size_t ws_bytes, cudaStream_t st) {
  using namespace tc;
  Plan p = make_plan(desc, t);
  size_t need = kv_tc_workspace(desc, t);
  GP_REQUIRE(ws != nullptr && ws_bytes >= need, "gp_kv(tcgen05): workspace of %zu bytes required, %zu given",
             need, ws_bytes);
  char* w = static_cast<char*>(ws);
  float* row_img = reinterpret_cast<float*>(w); w += align256(p.row_img_bytes);
  float* col_img = reinterpret_cast<float*>(w); w += align256(p.col_img_bytes);
  void* v_img = w; w += align256(p.v_img_bytes);
  double* mean = reinterpret_cast<double*>(w); w += 256 * sizeof(double);
  float* vscale = reinterpret_cast<float*>(w); w += TN * sizeof(float);
  float* inv_vscale = reinterpret_cast<float*>(w); w += TN * sizeof(float);
  unsigned* rng = reinterpret_cast<unsigned*>(w); w += 4 * sizeof(unsigned);   // TS: row, col ranges
  float* dscale = reinterpret_cast<float*>(w); w += 4 * sizeof(float);
  float* split_ws = reinterpret_cast<float*>(w);
  const double c = desc->family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  const bool ts = KV_F16 && p.DK >= 48;   // large d: fp16 distance images, row image in TMEM
  {
    if (!kv_images_current) {
      if (ts) {
        if (int rc = distance_images16(desc->Xr, desc->ldr, desc->n_rows, desc->Xc, desc->ldc, desc->n_cols,
                                       desc->d, p.DK, BM, BN, c, mean, rng, reinterpret_cast<__half*>(row_img),
                                       reinterpret_cast<__half*>(col_img), dscale, st))
          return rc;
      } else if (int rc = distance_images(desc->Xr, desc->ldr, desc->n_rows, desc->Xc, desc->ldc, desc->n_cols,
                                          desc->d, p.DK, BM, BN, c, mean, row_img, col_img, st)) {
        return rc;
      }
    }
    if (KV_F16) {
      if (int rc = v_colscale(V, ldv, desc->n_cols, t, vscale, inv_vscale, st)) return rc;
      if (int rc = v_images16(V, ldv, t, desc->n_cols, vscale, static_cast<__half*>(v_img), p.col_tiles, st))
        return rc;
    } else if (int rc = v_images32(V, ldv, t, desc->n_cols, static_cast<float*>(v_img), p.col_tiles, st)) {
      return rc;
    }
  }
  Args a;
  a.row_img = row_img; a.col_img = col_img; a.v_img = v_img; a.inv_vscale = inv_vscale; a.DK = p.DK;
  a.dscale = dscale;
  a.n_rows = desc->n_rows; a.n_cols = desc->n_cols;
  a.row_tiles = p.row_tiles; a.col_tiles = p.col_tiles; a.splits = p.splits;
  a.tiles_per_split = p.tiles_per_split; a.nstages = p.nstages; a.fam = desc->family; a.t = t;
  a.s2 = (float)desc->outputscale; a.noise = (float)desc->noise; a.diag_offset = desc->diag_offset;
  a.self_offset = desc->self_offset;
  a.V = V; a.ldv = ldv;
  // large d: row image TMEM-resident (TS distance MMA on fp16 images, 3 S buffers, look-ahead 2)
  a.lookahead = std::min(2, p.nstages - 1);   // 3 S buffers in both modes
  a.chunk = CHUNK;
  if (p.splits > 1) {
    a.out = split_ws; a.ldo = t; a.split_stride = desc->n_rows * (int64_t)t;
  } else {
    a.out = out; a.ldo = ldo; a.split_stride = 0;
  }
  int items = p.row_tiles * p.splits;
  int grid = std::min(items, num_sms());
  auto kern = desc->family == GP_FAMILY_RBF ? (ts ? kv_tc_kernel<GP_FAMILY_RBF, true> : kv_tc_kernel<GP_FAMILY_RBF, false>)
                                            : (ts ? kv_tc_kernel<GP_FAMILY_MATERN32, true>
                                                  : kv_tc_kernel<GP_FAMILY_MATERN32, false>);
  GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  a.prof = nullptr;
  const char* pe = getenv("GP_TC_PROF");
  if (pe && *pe == '1') GP_CUDA_TRY(cudaMalloc(&a.prof, (size_t)grid * (NTHREADS / 32) * 8 * sizeof(long long)));
  kern<<<grid, NTHREADS, p.smem, st>>>(a);
  GP_LAUNCH_CHECK();
  if (a.prof) {   // diagnostic only: per-role average wait cycles per tile
    std::vector<long long> h((size_t)grid * (NTHREADS / 32) * 8);
    GP_CUDA_TRY(cudaStreamSynchronize(st));
    GP_CUDA_TRY(cudaMemcpy(h.data(), a.prof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(a.prof);
    for (int wi : {1, 4, 5, 8, 12}) {
      double s[8] = {0};
      for (int cta = 0; cta < grid; ++cta)
        for (int k = 0; k < 8; ++k) s[k] += (double)h[((size_t)cta * (NTHREADS / 32) + wi) * 8 + k];
      fprintf(stderr, "[tc prof] warp %d:", wi);
      for (int k = 0; k < 8; ++k) fprintf(stderr, " w%d=%.0f", k, k == 7 ? s[7] / grid : s[k] / std::max(1.0, s[7]));
      fprintf(stderr, "\n");
    }
  }
  if (p.splits > 1) {
    return launch_split_reduce(split_ws, p.splits, a.split_stride, desc->n_rows, t, out, ldo, a.s2,
                               a.noise, V, ldv, desc->diag_offset, st);
  }
  return GP_OK;
}

}  // namespace gp

extern "C" int gp_has_tcgen05(void) { return 1; }
