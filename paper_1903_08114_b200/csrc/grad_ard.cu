// tcgen05 fused gradient forms for ARD lengthscales (sm_100a):
//   out[0]   = sum_ij kappa_ij H_ij
//   out[1+k] = sum_ij eps_ij (x_ik - x_jk)^2 H_ij,   H = Y R^T (never materialised)
// (same outputs as grad.cu / grad_tc.cu; likelihood.py:166-216 via the
// identity in grad.cu).
//
// The per-dimension sums are moved onto the tensor core. With
// W_ij = eps_ij H_ij,
//   sum_j W_ij (x_ik - x_jk)^2 = x_ik^2 sum_j W_ij - 2 x_ik (W X)_ik + (W X^2)_ik,
// so per 128 x 64 tile the epilogue only forms W (one product per entry,
// instead of 3 d flops) and the tensor core accumulates G = W [X | X^2]
// (N = 2 d) in TMEM across the item; the d sums are formed once per row and
// item. Coordinates are centred (the distance images' column mean), which
// keeps the expansion's cancellation small.
//
// Per tile on the tensor core (one elected thread issues):
//   S = A.B^T        3xTF32 (kind::tf32, SS), as in grad_tc.cu
//   H = Y.R^T        bf16 two-term split: Y1.R1 + Y1.R2 + Y2.R1 (A = Y in TMEM)
//   G += W.[X | X^2] bf16 two-term split (A = W in TMEM, written by the epilogue)
// bf16 keeps fp32's range, so no operand needs scaling; the two-term split
// carries 16 significant bits (the gradients' tolerance is 1e-3).
#include "tc_common.cuh"

#include <cuda_bf16.h>

#include <algorithm>

namespace gp {
namespace ga {

using namespace gp::tc;

constexpr int BM = 128;         // rows per tile; columns per tile BN = 64 (d + 2 <= 32) or 32 (larger d)
constexpr int NTHREADS = 384;   // 0 TMA, 1 MMA, 2 TMEM alloc, 3 idle, 4-11 epilogue
constexpr int EPI0 = 4, NEPI = 8;
constexpr int MAXNL = 32;       // ARD dimensions per launch (G = 2 nl <= 64 TMEM columns)
constexpr int MAXWP = 56;       // bf16 pairs of Y per row (w <= 112)

struct Args {
  const float* row_img;   // [row tiles][2][BM*DK] tf32 (distance A)
  const float* col_img;   // [col tiles][2][BN*DK] tf32 (distance B)
  const __nv_bfloat16* r_img;   // [col tiles][2][BN*WK] bf16 R1 | R2 (K-major, K = w)
  const __nv_bfloat16* xx_img;  // [col tiles][2][GN*BN] bf16 XX1 | XX2 (K-major, K = j)
  const uint32_t* y_rows;       // [rows][2*WP] bf16 pairs: Y1 then Y2
  const float* Xr; int64_t ldr;
  const double* mean;
  const float* dscale;    // large d: fp16 hi | lo distance images, S = S' dscale (null: tf32)
  int DK, WK, WP, GN, d, p0, nl;
  int64_t n_rows, n_cols;
  int row_tiles, col_tiles, splits, tiles_per_split, nstages;
  int64_t self_offset;
  double* partials;       // [gridDim.x][1 + MAXNL]
};

// TMEM columns (BN = 64: S_b 64b | H_b 128 + 64b | Y 256 | W1 368 | W2 400 | G 432;
// BN = 32 halves the S, H and W blocks): S_b, H_b double buffered, Y1 | Y2
// resident per row tile (<= 2 x 56 bf16-pair columns), W1 | W2 (the G
// product's A operand), G = [W X | W X^2] (<= 64 columns)
template <int BN> struct Tm {
  __host__ __device__ static constexpr uint32_t S(uint32_t b) { return (uint32_t)BN * b; }
  __host__ __device__ static constexpr uint32_t H(uint32_t b) { return 2u * BN + (uint32_t)BN * b; }
  static constexpr uint32_t Y = 4u * BN;
  static constexpr uint32_t W1 = Y + 2u * MAXWP;
  static constexpr uint32_t W2 = W1 + BN / 2;
  static constexpr uint32_t G = W2 + BN / 2;
  static_assert(G + 64 <= 512, "TMEM plan");
};

__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void split_bf16(float a, float b, uint32_t& p1, uint32_t& p2) {
  const __nv_bfloat162 h1 = __floats2bfloat162_rn(a, b);
  const float2 f1 = __bfloat1622float2(h1);
  const __nv_bfloat162 h2 = __floats2bfloat162_rn(a - f1.x, b - f1.y);
  p1 = *reinterpret_cast<const uint32_t*>(&h1);
  p2 = *reinterpret_cast<const uint32_t*>(&h2);
}

template <int FAM, int BN>
__global__ void __launch_bounds__(NTHREADS, 1) grad_ard_kernel(const Args a) {
  using TM = Tm<BN>;
  constexpr int CW = BN / 2;   // columns of a tile per epilogue warp
  extern __shared__ __align__(1024) uint8_t smem[];
  const int DK = a.DK, WK = a.WK, GN = a.GN;
  const bool F16I = a.dscale != nullptr;   // fp16 hi | lo distance images (large d)
  const uint32_t EB = F16I ? 2u : 4u;
  const uint32_t row_bytes = 2u * BM * DK * EB;
  const uint32_t col_bytes = 2u * BN * DK * EB;
  const uint32_t r_bytes = 2u * BN * WK * 2u;
  const uint32_t xx_bytes = 2u * GN * BN * 2u;
  const uint32_t stage_bytes = col_bytes + r_bytes + xx_bytes;
  const int NS = a.nstages;
  uint8_t* xr_s = smem;
  uint8_t* stages = smem + row_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * stage_bytes);
  uint64_t* full = bars;             // [NS] stage landed                     TMA -> MMA
  uint64_t* empty = bars + NS;       // [NS] G of the stage's tile done       MMA -> TMA
  uint64_t* s_full = bars + 2 * NS;  // [2]  S, H in TMEM buffer b            MMA -> epi
  uint64_t* s_empty = s_full + 2;    // [2]  S, H of buffer b loaded          epi -> MMA
  uint64_t* w_full = s_empty + 2;    //      W of the tile in TMEM            epi -> MMA
  uint64_t* w_empty = w_full + 1;    //      G of the tile done with W        MMA -> epi
  uint64_t* g_full = w_empty + 1;    //      item's G complete                MMA -> epi
  uint64_t* g_empty = g_full + 1;    //      G read                           epi -> MMA
  uint64_t* y_full = g_empty + 1;    //      Y rows in TMEM                   epi -> MMA
  uint64_t* y_empty = y_full + 1;    //      item's H products done           MMA -> epi
  uint64_t* xr_full = y_empty + 1;   //      row image landed                 TMA -> MMA
  uint64_t* xr_empty = xr_full + 1;  //      item's distance products done    MMA -> TMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xr_empty + 1);
  __shared__ double red[NEPI][1 + MAXNL];
  __shared__ float mean_s[MAXNL];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < MAXNL) mean_s[threadIdx.x] = threadIdx.x < a.nl ? (float)a.mean[a.p0 + threadIdx.x] : 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&s_full[b]), 1);
      mbar_init(smem_u32(&s_empty[b]), NEPI);
    }
    mbar_init(smem_u32(w_full), NEPI);
    mbar_init(smem_u32(w_empty), 1);
    mbar_init(smem_u32(g_full), 1);
    mbar_init(smem_u32(g_empty), NEPI);
    mbar_init(smem_u32(y_full), NEPI);
    mbar_init(smem_u32(y_empty), 1);
    mbar_init(smem_u32(xr_full), 1);
    mbar_init(smem_u32(xr_empty), 1);
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
  const int n_items = a.row_tiles * a.splits;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0, itc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
        const int rt = it / a.splits, sp = it - rt * a.splits;
        const int ct0 = sp * a.tiles_per_split;
        const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
        mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
        mbar_expect_tx(smem_u32(xr_full), row_bytes);
        bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)rt * (row_bytes / 4), row_bytes, smem_u32(xr_full));
        for (int ct = ct0; ct < ct1; ++ct) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          uint8_t* st = stages + s * stage_bytes;
          mbar_expect_tx(smem_u32(&full[s]), stage_bytes);
          bulk_g2s(smem_u32(st), a.col_img + (int64_t)ct * (col_bytes / 4), col_bytes, smem_u32(&full[s]));
          bulk_g2s(smem_u32(st + col_bytes), a.r_img + (int64_t)ct * (r_bytes / 2), r_bytes, smem_u32(&full[s]));
          bulk_g2s(smem_u32(st + col_bytes + r_bytes), a.xx_img + (int64_t)ct * (xx_bytes / 2), xx_bytes,
                   smem_u32(&full[s]));
          if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (warp-uniform) =====================
    // per tile T: S and H of T, then G of T - 1 (its W is being written by
    // the epilogue while S, H of T run)
    const uint32_t idesc_d = F16I ? idesc_f16(BM, BN) : make_idesc(BM, BN);
    const uint32_t idesc_h = idesc_bf16(BM, BN), idesc_g = idesc_bf16(BM, GN);
    const uint32_t lbo_a = (BM / 8) * 128, lbo_b = (BN / 8) * 128;
    const uint32_t lbo_r = (BN / 8) * 128, lbo_x = (GN / 8) * 128;
    const uint64_t da0 = make_desc(smem_u32(xr_s), lbo_a, 128);
    const uint64_t db0 = make_desc(smem_u32(stages), lbo_b, 128);
    const uint64_t dr0 = make_desc(smem_u32(stages + col_bytes), lbo_r, 128);
    const uint64_t dx0 = make_desc(smem_u32(stages + col_bytes + r_bytes), lbo_x, 128);
    const uint32_t a_half16 = (BM * DK * EB) >> 4, b_half16 = (BN * DK * EB) >> 4;
    const uint32_t r_half16 = (BN * WK * 2) >> 4, x_half16 = (GN * BN * 2) >> 4;
    const uint32_t stage16 = stage_bytes >> 4;
    const uint32_t ka16 = (2 * lbo_a) >> 4, kb16 = (2 * lbo_b) >> 4;
    const uint32_t kr16 = (2 * lbo_r) >> 4, kx16 = (2 * lbo_x) >> 4;
    const int dsteps = F16I ? DK / 16 : DK / 8, hsteps = WK / 16;   // 32 B of K per row and MMA
    const uint32_t ty1 = tmem + TM::Y, ty2 = tmem + TM::Y + (uint32_t)a.WP;
    const bool leader = elect_one();
    uint32_t s = 0, ph = 0, T = 0, itc = 0;
    auto issue_g = [&](uint32_t Tg, uint32_t sg, bool fresh, bool last) {
      mbar_wait(smem_u32(w_full), Tg & 1);
      if (fresh && itc >= 1) mbar_wait(smem_u32(g_empty), (itc - 1) & 1);
      tc_fence_after();
      if (leader) {
        const uint64_t dx = dx0 + (uint64_t)(sg * stage16);
        const uint32_t g = tmem + TM::G;
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {   // W1.XX1 + W1.XX2 + W2.XX1
          const uint32_t wa = tmem + (pass == 2 ? TM::W2 : TM::W1);
          const uint64_t xb = dx + (pass == 1 ? x_half16 : 0u);
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks)
            mma16_ts(g, wa + ks * 8, xb + (uint64_t)(ks * kx16), idesc_g, !(fresh && pass == 0 && ks == 0));
        }
        tc_commit(smem_u32(&empty[sg]));
        tc_commit(smem_u32(w_empty));
        if (last) tc_commit(smem_u32(g_full));
      }
      __syncwarp();
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int sp = it % a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      mbar_wait(smem_u32(xr_full), itc & 1);
      mbar_wait(smem_u32(y_full), itc & 1);
      tc_fence_after();
      uint32_t s_prev = 0;
      for (int ct = ct0; ct < ct1; ++ct) {
        const uint32_t b = T & 1;
        if (T >= 2) mbar_wait(smem_u32(&s_empty[b]), ((T >> 1) - 1) & 1);
        mbar_wait(smem_u32(&full[s]), ph);
        tc_fence_after();
        if (leader) {
          const uint32_t d_s = tmem + TM::S(b), d_h = tmem + TM::H(b);
          const uint64_t db = db0 + (uint64_t)(s * stage16);
          const uint64_t dr = dr0 + (uint64_t)(s * stage16);
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint64_t ap = da0 + (pass == 0 ? a_half16 : 0u);
            const uint64_t bp = db + (pass == 1 ? b_half16 : 0u);
            for (int ks = 0; ks < dsteps; ++ks) {
              if (F16I)
                mma16_ss(d_s, ap + (uint64_t)(ks * ka16), bp + (uint64_t)(ks * kb16), idesc_d, (pass | ks) != 0);
              else
                mma_ss(d_s, ap + (uint64_t)(ks * ka16), bp + (uint64_t)(ks * kb16), idesc_d, (pass | ks) != 0);
            }
          }
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {   // Y1.R1 + Y1.R2 + Y2.R1
            const uint32_t ya = pass == 2 ? ty2 : ty1;
            const uint64_t rb = dr + (pass == 1 ? r_half16 : 0u);
            for (int ks = 0; ks < hsteps; ++ks)
              mma16_ts(d_h, ya + ks * 8, rb + (uint64_t)(ks * kr16), idesc_h, (pass | ks) != 0);
          }
          tc_commit(smem_u32(&s_full[b]));
        }
        __syncwarp();
        if (ct > ct0) issue_g(T - 1, s_prev, ct - 1 == ct0, false);
        s_prev = s;
        if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        ++T;
      }
      if (leader) {
        tc_commit(smem_u32(y_empty));
        tc_commit(smem_u32(xr_empty));
      }
      __syncwarp();
      issue_g(T - 1, s_prev, ct1 - 1 == ct0, true);
      ++itc;
    }
  } else if (warp >= EPI0) {
    // ===================== epilogue (8 warps) =====================
    const int q = warp & 3, half = (warp - EPI0) >> 2, ew = warp - EPI0;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    double acc0 = 0.0;   // sum kappa H (this thread's entries)
    double acck = 0.0;   // sum for dimension k = lane (after the per-item warp reductions)
    uint32_t T = 0, itc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      const int rt = it / a.splits, sp = it - rt * a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      const int64_t row = (int64_t)rt * BM + q * 32 + lane;
      // ---- Y rows -> TMEM (half 0: Y1, half 1: Y2) once the previous item's H is done
      mbar_wait(smem_u32(y_empty), (itc & 1) ^ 1);
      tc_fence_after();
      {
        const uint32_t* src = a.y_rows + row * (2 * (int64_t)a.WP) + half * a.WP;
        const uint32_t dst = tmem + lane_base + TM::Y + (uint32_t)(half * a.WP);
        for (int c0 = 0; c0 < a.WP; c0 += 8) {
          uint32_t v[8];
#pragma unroll
          for (int e = 0; e < 8; e += 4) {
            const uint4 f = *reinterpret_cast<const uint4*>(src + c0 + e);
            v[e] = f.x; v[e + 1] = f.y; v[e + 2] = f.z; v[e + 3] = f.w;
          }
          tmem_st8(dst + c0, v);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(y_full));
      }
      const int64_t diag_col = (a.self_offset >= 0 && row < a.n_rows) ? row + a.self_offset : -1000;
      int64_t e_diag = diag_col - ((int64_t)ct0 * BN + half * CW);
      float rs = 0.f;   // sum_j W_ij over this warp's columns of the item
      for (int ct = ct0; ct < ct1; ++ct, e_diag -= BN, ++T) {
        const uint32_t b = T & 1;
        mbar_wait(smem_u32(&s_full[b]), (T >> 1) & 1);
        tc_fence_after();
        uint32_t sv[CW], hv[CW];
        if constexpr (CW == 32) {
          tmem_ld32(tmem + lane_base + TM::S(b) + half * CW, reinterpret_cast<uint32_t (&)[32]>(sv));
          tmem_ld32(tmem + lane_base + TM::H(b) + half * CW, reinterpret_cast<uint32_t (&)[32]>(hv));
        } else {
          tmem_ld16(tmem + lane_base + TM::S(b) + half * CW, reinterpret_cast<uint32_t (&)[16]>(sv));
          tmem_ld16(tmem + lane_base + TM::H(b) + half * CW, reinterpret_cast<uint32_t (&)[16]>(hv));
        }
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s_empty[b]));
        if (__any_sync(0xffffffffu, e_diag >= 0 && e_diag < CW)) {
#pragma unroll
          for (int e = 0; e < CW; ++e)
            if (e == e_diag) sv[e] = 0u;
        }
        float a0 = 0.f;
        const float dsc = F16I ? *a.dscale : 1.f;
#pragma unroll
        for (int e = 0; e < CW; ++e) {
          const float S = __uint_as_float(sv[e]) * dsc;
          const float h = __uint_as_float(hv[e]);
          float kap, eps;
          if (FAM == GP_FAMILY_RBF) {
            kap = ex2_approx(min0_nan(S));          // S = -log2(e) r2 / 2
            eps = kap;
          } else {
            const float u = sqrt_approx(max0_nan(S));   // S = 3 r2
            const float ex = ex2_approx(u * -kLog2e);
            kap = fmaf(u, ex, ex);
            eps = 3.0f * ex;
          }
          a0 = fmaf(kap, h, a0);
          const float wv = eps * h;
          rs += wv;
          hv[e] = __float_as_uint(wv);
        }
        acc0 += (double)a0;
        uint32_t p1[CW / 2], p2[CW / 2];
#pragma unroll
        for (int k = 0; k < CW / 2; ++k)
          split_bf16(__uint_as_float(hv[2 * k]), __uint_as_float(hv[2 * k + 1]), p1[k], p2[k]);
        // W (this warp's CW columns = CW / 2 pair columns) once G of the previous tile is done with it
        if (T >= 1) mbar_wait(smem_u32(w_empty), (T - 1) & 1);
        tc_fence_after();
        if constexpr (CW == 32) {
          tmem_st16(tmem + lane_base + TM::W1 + half * 16, reinterpret_cast<const uint32_t (&)[16]>(p1));
          tmem_st16(tmem + lane_base + TM::W2 + half * 16, reinterpret_cast<const uint32_t (&)[16]>(p2));
        } else {
          tmem_st8(tmem + lane_base + TM::W1 + half * 8, p1);
          tmem_st8(tmem + lane_base + TM::W2 + half * 8, p2);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(w_full));
      }
      // ---- item done: sum_j W_ij (x_ik - x_jk)^2 = x_ik^2 rs_i - 2 x_ik G_ik + G'_ik
      // (half 0 adds the G terms, both halves their own row-sum term)
      mbar_wait(smem_u32(g_full), itc & 1);
      tc_fence_after();
      const bool in = row < a.n_rows;
      for (int k0 = 0; k0 < a.nl; k0 += 16) {
        uint32_t gx[16], gq[16];
        if (half == 0) {
          tmem_ld16(tmem + lane_base + TM::G + k0, gx);
          tmem_ld16(tmem + lane_base + TM::G + a.nl + k0, gq);
          tmem_wait_ld();
        }
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
          const int k = k0 + kk;
          if (k < a.nl) {
            const float x = in ? a.Xr[row * a.ldr + a.p0 + k] - mean_s[k] : 0.f;
            float v = x * x * rs;
            if (half == 0) v += fmaf(-2.f * x, __uint_as_float(gx[kk]), __uint_as_float(gq[kk]));
            const double tot = warp_sum((double)(in ? v : 0.f));
            if (lane == k) acck += tot;
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(g_empty));
    }
    // fixed-order reduction: warp butterfly, then warps in index order
    const double s0 = warp_sum(acc0);
    if (lane == 0) red[ew][0] = s0;
    if (lane < MAXNL) red[ew][1 + lane] = acck;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 1 + MAXNL) {
    double v = 0.0;
    for (int w = 0; w < NEPI; ++w) v += red[w][threadIdx.x];
    a.partials[(int64_t)blockIdx.x * (1 + MAXNL) + threadIdx.x] = v;
  }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---- operand preparation -------------------------------------------------
// Y rows as bf16 pairs: [rows][Y1 (WP pairs) | Y2 (WP pairs)], zero padded
__global__ void y_bf16_kernel(const float* __restrict__ Y, int64_t ldy, int64_t n, int w, int WP, int64_t rows_pad,
                              uint32_t* out) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows_pad * WP) return;
  const int64_t r = idx / WP;
  const int pr = (int)(idx - r * WP);
  const int k = 2 * pr;
  const float a = (r < n && k < w) ? Y[r * ldy + k] : 0.f;
  const float b = (r < n && k + 1 < w) ? Y[r * ldy + k + 1] : 0.f;
  uint32_t p1, p2;
  split_bf16(a, b, p1, p2);
  out[r * 2 * WP + pr] = p1;
  out[r * 2 * WP + WP + pr] = p2;
}

// R image per 64-column tile: bf16 K-major (rows = columns j, K = w), R1 then R2
__global__ void r_bf16_kernel(const float* __restrict__ R, int64_t ldr, int64_t n, int w, int WK, int BN,
                              int64_t ntiles, __nv_bfloat16* img) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * BN * WK) return;
  const int64_t tile = idx / (BN * WK);
  const int rem = (int)(idx - tile * BN * WK);
  const int r = rem / WK, k = rem - r * WK;
  const int64_t col = tile * BN + r;
  const float v = (col < n && k < w) ? R[col * ldr + k] : 0.f;
  const __nv_bfloat16 h1 = __float2bfloat16_rn(v);
  const __nv_bfloat16 h2 = __float2bfloat16_rn(v - __bfloat162float(h1));
  __nv_bfloat16* base = img + tile * 2 * BN * WK;
  base[canon16(r, k, BN)] = h1;
  base[BN * WK + canon16(r, k, BN)] = h2;
}

// [X | X^2] image per 64-column tile (centred coordinates of dims p0..p0+nl):
// bf16 K-major with rows = the GN outputs (x_k, then x_k^2), K = the 64 columns
__global__ void xx_bf16_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, const double* __restrict__ mean,
                               int p0, int nl, int GN, int BN, int64_t ntiles, __nv_bfloat16* img) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * BN * GN) return;
  const int64_t tile = idx / (BN * GN);
  const int rem = (int)(idx - tile * BN * GN);
  const int j = rem / GN, o = rem - j * GN;
  const int64_t col = tile * BN + j;
  float v = 0.f;
  if (col < n && o < 2 * nl) {
    const int k = o < nl ? o : o - nl;
    const float x = (float)((double)X[col * ldx + p0 + k] - mean[p0 + k]);
    v = o < nl ? x : x * x;
  }
  const __nv_bfloat16 h1 = __float2bfloat16_rn(v);
  const __nv_bfloat16 h2 = __float2bfloat16_rn(v - __bfloat162float(h1));
  __nv_bfloat16* base = img + tile * 2 * GN * BN;
  base[canon16(o, j, GN)] = h1;
  base[GN * BN + canon16(o, j, GN)] = h2;
}

__global__ void grad_ard_finalize(const double* __restrict__ partials, int nblocks, int p0, int nl, int with_s2,
                                  double* out) {
  const int p = threadIdx.x;
  if (p > nl || (p == 0 && !with_s2)) return;
  double acc = 0.0;
  for (int b = 0; b < nblocks; ++b) acc += partials[(int64_t)b * (1 + MAXNL) + p];
  out[p == 0 ? 0 : 1 + p0 + (p - 1)] = acc;
}

struct Plan {
  int BN, DK, WK, WP, row_tiles, col_tiles, splits, tiles_per_split, nstages, grid;
  int eb;   // distance-image element bytes: 2 (fp16 hi | lo, DK >= 48) or 4 (tf32)
  size_t row_img, col_img, r_img, xx_img, y_rows, partials, smem;
};

static int gn_for(int nl) { return std::max(16, (2 * nl + 15) / 16 * 16); }

static Plan make_plan(int64_t nr, int64_t nc, int d, int w) {
  Plan p;
  p.DK = (d + 2 + 7) / 8 * 8;
  p.eb = p.DK >= 48 ? 2 : 4;
  const int BN = p.DK <= 32 ? 64 : 32;   // large d: narrower tiles keep two SMEM stages
  p.BN = BN;
  p.WK = (w + 15) / 16 * 16;
  p.WP = p.WK / 2;
  p.row_tiles = (int)((nr + BM - 1) / BM);
  p.col_tiles = (int)((nc + BN - 1) / BN);
  const int64_t target = 2LL * num_sms();
  const int64_t s = std::max<int64_t>(1, std::min<int64_t>({(target + p.row_tiles - 1) / p.row_tiles, 64,
                                                            (int64_t)p.col_tiles}));
  p.tiles_per_split = (int)((p.col_tiles + s - 1) / s);
  p.splits = (p.col_tiles + p.tiles_per_split - 1) / p.tiles_per_split;
  p.grid = std::min(p.row_tiles * p.splits, num_sms());
  const int GNmax = gn_for(std::min(d, MAXNL));
  p.row_img = (size_t)p.row_tiles * 2 * BM * p.DK * 4;
  p.col_img = (size_t)p.col_tiles * 2 * BN * p.DK * 4;
  p.r_img = (size_t)p.col_tiles * 2 * BN * p.WK * 2;
  p.xx_img = (size_t)p.col_tiles * 2 * GNmax * BN * 2;
  p.y_rows = (size_t)p.row_tiles * BM * 2 * p.WP * 4;
  p.partials = (size_t)num_sms() * (1 + MAXNL) * 8;
  const size_t row_b = 2u * BM * p.DK * p.eb;
  const size_t stage_b = 2u * BN * p.DK * p.eb + 2u * BN * p.WK * 2 + 2u * GNmax * BN * 2;
  const size_t budget = 225 * 1024 - row_b - 512;
  p.nstages = (int)std::min<size_t>(3, budget / stage_b);
  p.smem = row_b + p.nstages * stage_b + 256;
  return p;
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace ga

// ARD gradients on the tensor core: dims up to 94 (64-column tiles up to
// d = 30, 32-column tiles beyond, for the SMEM plan), w <= 112 (Y resident in
// TMEM as bf16 pairs)
bool grad_ard_supported(int64_t nr, int64_t nc, int d, int w) {
  if (d < 1 || d + 2 > 96 || w < 1 || w > 2 * ga::MAXWP || nr < 1 || nc < 1) return false;
  return ga::make_plan(nr, nc, d, w).nstages >= 2;
}

size_t grad_ard_workspace(int64_t nr, int64_t nc, int d, int w) {
  ga::Plan p = ga::make_plan(nr, nc, d, w);
  using ga::al256;
  return al256(p.row_img) + al256(p.col_img) + al256(p.r_img) + al256(p.xx_img) + al256(p.y_rows) +
         al256(p.partials) + 256 * sizeof(double) + 8 * sizeof(float);
}

int grad_ard(int family, int d, const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
             const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w, int64_t self_offset, double* out,
             void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace ga;
  Plan p = make_plan(nr, nc, d, w);
  GP_REQUIRE(ws_bytes >= grad_ard_workspace(nr, nc, d, w), "gp_grad_forms(tcgen05 ARD): workspace too small");
  char* wp = static_cast<char*>(ws);
  float* row_img = reinterpret_cast<float*>(wp); wp += al256(p.row_img);
  float* col_img = reinterpret_cast<float*>(wp); wp += al256(p.col_img);
  __nv_bfloat16* r_img = reinterpret_cast<__nv_bfloat16*>(wp); wp += al256(p.r_img);
  __nv_bfloat16* xx_img = reinterpret_cast<__nv_bfloat16*>(wp); wp += al256(p.xx_img);
  uint32_t* y_rows = reinterpret_cast<uint32_t*>(wp); wp += al256(p.y_rows);
  double* partials = reinterpret_cast<double*>(wp); wp += al256(p.partials);
  double* mean = reinterpret_cast<double*>(wp); wp += 256 * sizeof(double);
  unsigned* rng = reinterpret_cast<unsigned*>(wp); wp += 4 * sizeof(unsigned);
  float* dscale = reinterpret_cast<float*>(wp);
  const double c = family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  const int BN = p.BN;
  if (p.eb == 2) {
    if (int rc = tc::distance_images16(Xr, ldr, nr, Xc, ldc, nc, d, p.DK, BM, BN, c, mean, rng,
                                       reinterpret_cast<__half*>(row_img), reinterpret_cast<__half*>(col_img),
                                       dscale, st))
      return rc;
  } else if (int rc = tc::distance_images(Xr, ldr, nr, Xc, ldc, nc, d, p.DK, BM, BN, c, mean, row_img, col_img,
                                          st)) {
    return rc;
  }
  {
    const int64_t rows_pad = (int64_t)p.row_tiles * BM;
    int64_t tot = rows_pad * p.WP;
    y_bf16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Y, ldy, nr, w, p.WP, rows_pad, y_rows);
    GP_LAUNCH_CHECK();
    tot = (int64_t)p.col_tiles * BN * p.WK;
    r_bf16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(R, ldrr, nc, w, p.WK, BN, p.col_tiles, r_img);
    GP_LAUNCH_CHECK();
  }
  Args a;
  a.row_img = row_img; a.col_img = col_img; a.r_img = r_img; a.xx_img = xx_img; a.y_rows = y_rows;
  a.Xr = Xr; a.ldr = ldr; a.mean = mean; a.DK = p.DK;
  a.dscale = p.eb == 2 ? dscale : nullptr; a.WK = p.WK; a.WP = p.WP; a.d = d;
  a.n_rows = nr; a.n_cols = nc; a.row_tiles = p.row_tiles; a.col_tiles = p.col_tiles;
  a.splits = p.splits; a.tiles_per_split = p.tiles_per_split; a.nstages = p.nstages;
  a.self_offset = self_offset; a.partials = partials;
  auto kern = family == GP_FAMILY_RBF
                  ? (BN == 64 ? grad_ard_kernel<GP_FAMILY_RBF, 64> : grad_ard_kernel<GP_FAMILY_RBF, 32>)
                  : (BN == 64 ? grad_ard_kernel<GP_FAMILY_MATERN32, 64> : grad_ard_kernel<GP_FAMILY_MATERN32, 32>);
  GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const int nchunks = (d + MAXNL - 1) / MAXNL;
  for (int ch = 0; ch < nchunks; ++ch) {
    a.p0 = ch * MAXNL;
    a.nl = std::min(MAXNL, d - a.p0);
    a.GN = gn_for(a.nl);
    const int64_t tot = (int64_t)p.col_tiles * BN * a.GN;
    xx_bf16_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Xc, ldc, nc, mean, a.p0, a.nl, a.GN, BN,
                                                                  p.col_tiles, xx_img);
    GP_LAUNCH_CHECK();
    kern<<<p.grid, NTHREADS, p.smem, st>>>(a);
    GP_LAUNCH_CHECK();
    grad_ard_finalize<<<1, 64, 0, st>>>(partials, p.grid, a.p0, a.nl, ch == 0, out);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

}  // namespace gp
