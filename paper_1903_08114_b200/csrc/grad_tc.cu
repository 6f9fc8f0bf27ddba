// tcgen05 fused gradient forms (sm_100a):
//   g_p = sum_ij (dK/dtheta_p)_ij H_ij,  H = Y R^T  (n x n, never materialised)
// for p = outputscale, shared lengthscale or ARD lengthscales (see grad.cu
// for the identity with likelihood.py:166-216 and the output convention).
//
// Per 128x64 tile (one persistent CTA per SM):
//   MMA thread : S = A.B^T (distance, 3xTF32, as in kv_tc.cu) and
//                H = Y.R^T (3xTF32, K = w = 1 + t + k) with Y resident in
//                TMEM as the A operand (loaded once per row tile by the
//                epilogue warps), R tiles streamed by bulk TMA.
//   8 epilogue warps: tcgen05.ld S and H, kappa / eps on the SFU, and
//                per-entry accumulation sum kappa H, sum eps r2 H, or
//                sum eps (x_k - x'_k)^2 H (ARD, column coordinates from the
//                SMEM stage), fp32 per tile then fp64.
// The fp64 per-CTA partials are reduced in a fixed order (deterministic).
#include "tc_common.cuh"

#include <algorithm>

namespace gp {
namespace tc {

constexpr int GBM = 128, GBN = 64;
constexpr int G_NTHREADS = 384;
constexpr int G_EPI0 = 4;
constexpr int G_NEPI = 8;
constexpr int G_MAXNL = 16;  // ARD dims handled per launch

struct GArgs {
  const float* row_img;   // [row tiles][2][GBM*DK]  distance A operand
  const float* col_img;   // [col tiles][2][GBN*DK]  distance B operand
  const float* r_img;     // [col tiles][2][GBN*WK]  H B operand (canonical, hi/lo)
  const float* y_rows;    // [rows][2*WKP] plain fp32: hi (WKP) then lo (WKP)
  const float* col_xy;    // [col tiles][GBN*DP]     column coordinates (ARD), plain fp32
  const float* Xr; int64_t ldr;  // row coordinates (ARD)
  int DK, WK, WKP, DP, d, p0, nl;
  int64_t n_rows, n_cols;
  int row_tiles, col_tiles, splits, tiles_per_split, nstages;
  int64_t self_offset;
  double* partials;       // [gridDim.x][1 + G_MAXNL]
  // symmetric schedule (square operator, Y R^T symmetric): items are
  // (row tile, first column tile) pairs over the upper triangle of 128 x 128
  // blocks (column tiles ct >= 2 rt); tiles off the diagonal block count twice
  const int2* items;      // [n_items] or nullptr (rectangular: rt = it / splits)
  int n_items;
};

// item -> row tile and column-tile range
__device__ __forceinline__ void g_item(const GArgs& a, int it, int& rt, int& ct0, int& ct1) {
  if (a.items) {
    const int2 e = a.items[it];
    rt = e.x;
    ct0 = e.y;
  } else {
    rt = it / a.splits;
    ct0 = (it - rt * a.splits) * a.tiles_per_split;
  }
  ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
}

// TMEM map: S_b at 64b, H_b at 128 + 64b, Y_hi at 256, Y_lo at 256 + WKP
__device__ __forceinline__ uint32_t G_TS(uint32_t b) { return b * 64; }
__device__ __forceinline__ uint32_t G_TH(uint32_t b) { return 128 + b * 64; }

template <int FAM, bool ARD>
__global__ void __launch_bounds__(G_NTHREADS, 1) grad_tc_kernel(const GArgs a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int DK = a.DK, WK = a.WK, DP = a.DP;
  const uint32_t row_bytes = 2u * GBM * DK * 4u;
  const uint32_t col_bytes = 2u * GBN * DK * 4u;
  const uint32_t r_bytes = 2u * GBN * WK * 4u;
  const uint32_t xy_bytes = ARD ? GBN * DP * 4u : 0u;
  const uint32_t stage_bytes = col_bytes + r_bytes + xy_bytes;
  const int NS = a.nstages;
  uint8_t* xr_s = smem;
  uint8_t* stages = smem + row_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * stage_bytes);
  uint64_t* full = bars;             // [NS]
  uint64_t* empty = bars + NS;       // [NS]
  uint64_t* s_full = bars + 2 * NS;  // [2]
  uint64_t* s_empty = s_full + 2;    // [2]
  uint64_t* y_full = s_empty + 2;    // [1]
  uint64_t* y_empty = y_full + 1;    // [1]
  uint64_t* xr_full = y_empty + 1;   // [1]
  uint64_t* xr_empty = xr_full + 1;  // [1]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xr_empty + 1);
  __shared__ double red[G_NEPI][1 + G_MAXNL];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      // ARD: the epilogue reads column coordinates from the stage too
      mbar_init(smem_u32(&empty[s]), ARD ? 1 + G_NEPI : 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&s_full[b]), 1);
      mbar_init(smem_u32(&s_empty[b]), G_NEPI);
    }
    mbar_init(smem_u32(y_full), G_NEPI);
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
  const uint32_t TY_HI = 256, TY_LO = 256 + a.WKP;
  const int n_items = a.n_items;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0, itc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
        int rt, ct0, ct1;
        g_item(a, it, rt, ct0, ct1);
        mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
        mbar_expect_tx(smem_u32(xr_full), row_bytes);
        bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)rt * (row_bytes / 4), row_bytes, smem_u32(xr_full));
        for (int ct = ct0; ct < ct1; ++ct) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          uint8_t* st = stages + s * stage_bytes;
          mbar_expect_tx(smem_u32(&full[s]), stage_bytes);
          bulk_g2s(smem_u32(st), a.col_img + (int64_t)ct * (col_bytes / 4), col_bytes, smem_u32(&full[s]));
          bulk_g2s(smem_u32(st + col_bytes), a.r_img + (int64_t)ct * (r_bytes / 4), r_bytes,
                   smem_u32(&full[s]));
          if (ARD)
            bulk_g2s(smem_u32(st + col_bytes + r_bytes), a.col_xy + (int64_t)ct * (xy_bytes / 4), xy_bytes,
                     smem_u32(&full[s]));
          if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (warp-uniform) =====================
    const uint32_t idesc = make_idesc(GBM, GBN);
    const uint32_t lbo_a = (GBM / 8) * 128, lbo_b = (GBN / 8) * 128;
    const uint64_t da0 = make_desc(smem_u32(xr_s), lbo_a, 128);
    const uint64_t db0 = make_desc(smem_u32(stages), lbo_b, 128);
    const uint64_t dr0 = make_desc(smem_u32(stages + col_bytes), lbo_b, 128);
    const uint32_t a_half16 = (GBM * DK * 4) >> 4, b_half16 = (GBN * DK * 4) >> 4;
    const uint32_t r_half16 = (GBN * WK * 4) >> 4;
    const uint32_t stage16 = stage_bytes >> 4;
    const uint32_t ka16 = (2 * lbo_a) >> 4, kb16 = (2 * lbo_b) >> 4;
    const int dsteps = DK / 8, hsteps = WK / 8;
    const bool leader = elect_one();
    uint32_t s = 0, ph = 0, b = 0, bph = 0, itc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      int rt, ct0, ct1;
      g_item(a, it, rt, ct0, ct1);
      mbar_wait(smem_u32(xr_full), itc & 1);
      mbar_wait(smem_u32(y_full), itc & 1);
      tc_fence_after();
      for (int ct = ct0; ct < ct1; ++ct) {
        mbar_wait(smem_u32(&s_empty[b]), bph ^ 1);  // epilogue done with this S/H buffer
        mbar_wait(smem_u32(&full[s]), ph);
        tc_fence_after();
        if (leader) {
          const uint32_t d_s = tmem + G_TS(b), d_h = tmem + G_TH(b);
          const uint64_t db = db0 + (uint64_t)(s * stage16);
          const uint64_t dr = dr0 + (uint64_t)(s * stage16);
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint64_t ap = da0 + (pass == 0 ? a_half16 : 0u);
            const uint64_t bp = db + (pass == 1 ? b_half16 : 0u);
            for (int ks = 0; ks < dsteps; ++ks)
              mma_ss(d_s, ap + (uint64_t)(ks * ka16), bp + (uint64_t)(ks * kb16), idesc, (pass | ks) != 0);
          }
          // H = Ylo.Rhi + Yhi.Rlo + Yhi.Rhi
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint32_t ya = tmem + (pass == 0 ? TY_LO : TY_HI);
            const uint64_t rp = dr + (pass == 1 ? r_half16 : 0u);
            for (int ks = 0; ks < hsteps; ++ks)
              mma_ts(d_h, ya + ks * 8, rp + (uint64_t)(ks * kb16), idesc, (pass | ks) != 0);
          }
          tc_commit(smem_u32(&empty[s]));
          tc_commit(smem_u32(&s_full[b]));
        }
        __syncwarp();
        if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        if (++b == 2) { b = 0; bph ^= 1; }
      }
      if (leader) {
        tc_commit(smem_u32(y_empty));
        tc_commit(smem_u32(xr_empty));
      }
      __syncwarp();
    }
  } else if (warp >= G_EPI0) {
    // ===================== epilogue (8 warps) =====================
    const int q = warp & 3, half = (warp - G_EPI0) >> 2, ew = warp - G_EPI0;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    constexpr int NP = 1 + (ARD ? G_MAXNL : 1);
    double acc64[NP];
#pragma unroll
    for (int p = 0; p < NP; ++p) acc64[p] = 0.0;
    uint32_t s = 0, ph = 0, b = 0, bph = 0, itc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      int rt, ct0, ct1;
      g_item(a, it, rt, ct0, ct1);
      const int64_t row = (int64_t)rt * GBM + q * 32 + lane;
      // ---- Y rows -> TMEM (half 0: hi, half 1: lo); previous item's H MMAs must be done
      mbar_wait(smem_u32(y_empty), (itc & 1) ^ 1);
      tc_fence_after();
      {
        const float* src = a.y_rows + row * (2 * (int64_t)a.WKP) + half * a.WKP;
        const uint32_t dst = tmem + lane_base + (half ? TY_LO : TY_HI);
        for (int c0 = 0; c0 < a.WKP; c0 += 32) {
          uint32_t v[32];
#pragma unroll
          for (int e = 0; e < 32; e += 4) {
            float4 f = *reinterpret_cast<const float4*>(src + c0 + e);
            v[e] = __float_as_uint(f.x); v[e + 1] = __float_as_uint(f.y);
            v[e + 2] = __float_as_uint(f.z); v[e + 3] = __float_as_uint(f.w);
          }
          tmem_st32(dst + c0, v);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(y_full));
      }
      float xr[ARD ? G_MAXNL : 1];
      if (ARD) {
#pragma unroll
        for (int k = 0; k < G_MAXNL; ++k)
          xr[k] = (k < a.nl && row < a.n_rows) ? a.Xr[row * a.ldr + a.p0 + k] : 0.f;
      }
      const int64_t diag_col = (a.self_offset >= 0 && row < a.n_rows) ? row + a.self_offset : -1000;
      int64_t e_diag = diag_col - ((int64_t)ct0 * GBN + half * 32);
      for (int ct = ct0; ct < ct1; ++ct, e_diag -= GBN) {
        mbar_wait(smem_u32(&s_full[b]), bph);
        tc_fence_after();
        uint32_t sv[32], hv[32];
        tmem_ld32(tmem + lane_base + G_TS(b) + half * 32, sv);
        tmem_ld32(tmem + lane_base + G_TH(b) + half * 32, hv);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&s_empty[b]));
        if (__any_sync(0xffffffffu, e_diag >= 0 && e_diag < 32)) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e == e_diag) sv[e] = 0u;
        }
        float acc[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) acc[p] = 0.f;
        const float* xy = ARD ? reinterpret_cast<const float*>(stages + s * stage_bytes + col_bytes + r_bytes) +
                                    (half * 32) * DP
                              : nullptr;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float S = __uint_as_float(sv[e]);
          const float h = __uint_as_float(hv[e]);
          float kap, eps, r2;
          if (FAM == GP_FAMILY_RBF) {
            const float Sc = S > 0.f ? 0.f : S;           // S = -log2(e) r2 / 2
            kap = ex2_approx(Sc);
            eps = kap;
            r2 = Sc * (-2.0f / kLog2e);
          } else {
            const float Sc = S < 0.f ? 0.f : S;           // S = 3 r2
            const float u = sqrt_approx(Sc);
            const float ex = ex2_approx(u * -kLog2e);
            kap = fmaf(u, ex, ex);
            eps = 3.0f * ex;
            r2 = Sc * (1.0f / 3.0f);
          }
          acc[0] = fmaf(kap, h, acc[0]);
          const float eh = eps * h;
          if (!ARD) {
            acc[1] = fmaf(eh, r2, acc[1]);
          } else {
            const float* xc = xy + e * DP + a.p0;
#pragma unroll
            for (int k = 0; k < G_MAXNL; k += 4) {
              if (k < a.nl) {
                const float4 c4 = *reinterpret_cast<const float4*>(xc + k);
                const float d0 = xr[k] - c4.x, d1 = xr[k + 1] - c4.y, d2 = xr[k + 2] - c4.z,
                            d3 = xr[k + 3] - c4.w;
                acc[1 + k] = fmaf(eh * d0, d0, acc[1 + k]);
                acc[2 + k] = fmaf(eh * d1, d1, acc[2 + k]);
                acc[3 + k] = fmaf(eh * d2, d2, acc[3 + k]);
                acc[4 + k] = fmaf(eh * d3, d3, acc[4 + k]);
              }
            }
          }
        }
        if (ARD) {  // done with this stage's column coordinates
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(&empty[s]));
        }
        // symmetric schedule: a tile outside the diagonal 128 x 128 block
        // stands for itself and its mirror
        const double wt = (a.items && ct >= 2 * rt + 2) ? 2.0 : 1.0;
#pragma unroll
        for (int p = 0; p < NP; ++p) acc64[p] += wt * (double)acc[p];
        if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        if (++b == 2) { b = 0; bph ^= 1; }
      }
    }
    (void)ph;
    // fixed-order reduction: warp butterfly, then warps in index order
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      double v = warp_sum(acc64[p]);
      if (lane == 0) red[ew][p] = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 1 + G_MAXNL) {
    const int np = 1 + (ARD ? G_MAXNL : 1);
    double v = 0.0;
    if ((int)threadIdx.x < np)
      for (int w = 0; w < G_NEPI; ++w) v += red[w][threadIdx.x];
    a.partials[(int64_t)blockIdx.x * (1 + G_MAXNL) + threadIdx.x] = v;
  }
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// ---- operand preparation -------------------------------------------------
// Y rows: [rows][hi WKP | lo WKP], zero padded beyond w and n
__global__ void y_rows_kernel(const float* __restrict__ Y, int64_t ldy, int64_t n, int w, int WKP,
                              int64_t rows_pad, float* out) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows_pad * WKP) return;
  int64_t r = idx / WKP;
  int k = (int)(idx - r * WKP);
  float v = (r < n && k < w) ? Y[r * ldy + k] : 0.f;
  float h = tf32_rna(v);
  out[r * 2 * WKP + k] = h;
  out[r * 2 * WKP + WKP + k] = v - h;
}

// R image: per 64-column tile, canonical K-major (rows = columns j, K = w)
__global__ void r_image_kernel(const float* __restrict__ R, int64_t ldr, int64_t n, int w, int WK,
                               int64_t ntiles, float* img) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * GBN * WK) return;
  int64_t tile = idx / (GBN * WK);
  int rem = (int)(idx - tile * GBN * WK);
  int r = rem / WK, k = rem - r * WK;
  int64_t col = tile * GBN + r;
  float v = (col < n && k < w) ? R[col * ldr + k] : 0.f;
  float h = tf32_rna(v);
  float* base = img + tile * 2 * GBN * WK;
  base[canon(r, k, GBN)] = h;
  base[GBN * WK + canon(r, k, GBN)] = v - h;
}

// column coordinates per tile [64][DP]
__global__ void col_xy_kernel(const float* __restrict__ X, int64_t ldx, int64_t n, int d, int DP,
                              int64_t ntiles, float* img) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= ntiles * GBN * DP) return;
  int64_t row = idx / DP;
  int k = (int)(idx - row * DP);
  img[idx] = (row < n && k < d) ? X[row * ldx + k] : 0.f;
}

// the symmetric schedule's item table, in row-tile order: row tile rt owns
// ceil((col_tiles - 2 rt) / tps) items starting at column tiles 2 rt + k tps
// (one block: per-thread row ranges, then an exclusive scan of their counts)
__global__ void sym_items_kernel(int row_tiles, int col_tiles, int tps, int2* items) {
  __shared__ int cnt[1024];
  const int per = (row_tiles + blockDim.x - 1) / blockDim.x;
  const int r0 = min(row_tiles, (int)threadIdx.x * per), r1 = min(row_tiles, r0 + per);
  int c = 0;
  for (int rt = r0; rt < r1; ++rt) c += (col_tiles - 2 * rt + tps - 1) / tps;
  cnt[threadIdx.x] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) {
      const int v = cnt[t];
      cnt[t] = acc;
      acc += v;
    }
  }
  __syncthreads();
  int k = cnt[threadIdx.x];
  for (int rt = r0; rt < r1; ++rt)
    for (int ct = 2 * rt; ct < col_tiles; ct += tps) items[k++] = make_int2(rt, ct);
}

__global__ void grad_tc_finalize(const double* __restrict__ partials, int nblocks, int p0, int nl,
                                 int with_s2, double* out) {
  int p = threadIdx.x;
  if (p > nl) return;
  if (p == 0 && !with_s2) return;
  double acc = 0.0;
  for (int b = 0; b < nblocks; ++b) acc += partials[(int64_t)b * (1 + G_MAXNL) + p];
  out[p == 0 ? 0 : 1 + p0 + (p - 1)] = acc;
}

struct GPlan {
  int DK, WK, WKP, DP, row_tiles, col_tiles, splits, tiles_per_split, nstages, grid, n_items;
  size_t row_img, col_img, r_img, y_rows, col_xy, partials, items, smem;
};

static GPlan gplan(int64_t nr, int64_t nc, int d, int ard, int w, bool sym = false) {
  GPlan p;
  p.DK = (d + 2 + 7) / 8 * 8;
  p.WK = (w + 7) / 8 * 8;
  p.WKP = (w + 31) / 32 * 32;
  p.DP = ard ? (std::min(d, G_MAXNL) + 3) / 4 * 4 : 0;
  if (ard) p.DP = (d + 3) / 4 * 4;
  p.row_tiles = (int)((nr + GBM - 1) / GBM);
  p.col_tiles = (int)((nc + GBN - 1) / GBN);
  int64_t target = 2LL * num_sms();
  int64_t s = std::max<int64_t>(1, std::min<int64_t>({(target + p.row_tiles - 1) / p.row_tiles, 64,
                                                      (int64_t)p.col_tiles}));
  p.tiles_per_split = (int)((p.col_tiles + s - 1) / s);
  p.splits = (p.col_tiles + p.tiles_per_split - 1) / p.tiles_per_split;
  p.n_items = p.row_tiles * p.splits;
  p.items = 0;
  if (sym) {
    // upper triangle: row tile rt takes column tiles [2 rt, col_tiles), in
    // pieces of tiles_per_split (about 4 items per SM in total)
    int64_t total = 0;
    for (int rt = 0; rt < p.row_tiles; ++rt) total += p.col_tiles - 2 * rt;
    p.tiles_per_split = (int)std::max<int64_t>(1, std::min<int64_t>(p.col_tiles, total / (4LL * num_sms())));
    int64_t ni = 0;
    for (int rt = 0; rt < p.row_tiles; ++rt) ni += (p.col_tiles - 2 * rt + p.tiles_per_split - 1) / p.tiles_per_split;
    p.n_items = (int)ni;
    p.splits = 0;
    p.items = (size_t)ni * sizeof(int2);
  }
  p.grid = std::min(p.n_items, num_sms());
  p.row_img = (size_t)p.row_tiles * 2 * GBM * p.DK * 4;
  p.col_img = (size_t)p.col_tiles * 2 * GBN * p.DK * 4;
  p.r_img = (size_t)p.col_tiles * 2 * GBN * p.WK * 4;
  p.y_rows = (size_t)p.row_tiles * GBM * 2 * p.WKP * 4;
  p.col_xy = ard ? (size_t)p.col_tiles * GBN * p.DP * 4 : 0;
  p.partials = (size_t)num_sms() * (1 + G_MAXNL) * 8;
  size_t row_b = 2u * GBM * p.DK * 4;
  size_t stage_b = 2u * GBN * p.DK * 4 + 2u * GBN * p.WK * 4 + (ard ? GBN * p.DP * 4u : 0u);
  size_t budget = 225 * 1024 - row_b - 512;
  p.nstages = (int)std::min<size_t>(3, budget / stage_b);
  p.smem = row_b + p.nstages * stage_b + 256;
  return p;
}

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace tc

bool grad_tc_supported(int64_t nr, int64_t nc, int d, int ard, int w) {
  if (d < 1 || d + 2 > 32 || w < 1 || w > 128) return false;
  tc::GPlan p = tc::gplan(nr, nc, d, ard, w);
  return p.nstages >= 2 && 2 * p.WKP <= 256;
}

size_t grad_tc_workspace(int64_t nr, int64_t nc, int d, int ard, int w, bool sym) {
  tc::GPlan p = tc::gplan(nr, nc, d, ard, w, sym);
  return tc::al256(p.row_img) + tc::al256(p.col_img) + tc::al256(p.r_img) + tc::al256(p.y_rows) +
         tc::al256(p.col_xy) + tc::al256(p.partials) + tc::al256(p.items) + 256 * sizeof(double);
}

// sym: the square operator (Xr = Xc, self_offset 0) with Y R^T symmetric;
// only the upper triangle of 128 x 128 blocks is evaluated (half the entries)
int grad_tc(int family, int d, int ard, const float* Xr, int64_t ldr, int64_t nr, const float* Xc,
            int64_t ldc, int64_t nc, const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w,
            int64_t self_offset, double* out, void* ws, size_t ws_bytes, cudaStream_t st, bool sym) {
  using namespace tc;
  GP_REQUIRE(!sym || (nr == nc && self_offset == 0), "gp_grad_forms_sym: square operator only");
  GPlan p = gplan(nr, nc, d, ard, w, sym);
  GP_REQUIRE(ws_bytes >= grad_tc_workspace(nr, nc, d, ard, w, sym), "gp_grad_forms(tcgen05): workspace too small");
  char* wp = static_cast<char*>(ws);
  float* row_img = reinterpret_cast<float*>(wp); wp += al256(p.row_img);
  float* col_img = reinterpret_cast<float*>(wp); wp += al256(p.col_img);
  float* r_img = reinterpret_cast<float*>(wp); wp += al256(p.r_img);
  float* y_rows = reinterpret_cast<float*>(wp); wp += al256(p.y_rows);
  float* col_xy = reinterpret_cast<float*>(wp); wp += al256(p.col_xy);
  double* partials = reinterpret_cast<double*>(wp); wp += al256(p.partials);
  int2* items = reinterpret_cast<int2*>(wp); wp += al256(p.items);
  double* mean = reinterpret_cast<double*>(wp);
  if (sym) {
    sym_items_kernel<<<1, 1024, 0, st>>>(p.row_tiles, p.col_tiles, p.tiles_per_split, items);
    GP_LAUNCH_CHECK();
  }
  const double c = family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  if (int rc = distance_images(Xr, ldr, nr, Xc, ldc, nc, d, p.DK, GBM, GBN, c, mean, row_img, col_img, st))
    return rc;
  {
    int64_t rows_pad = (int64_t)p.row_tiles * GBM;
    int64_t tot = rows_pad * p.WKP;
    y_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Y, ldy, nr, w, p.WKP, rows_pad, y_rows);
    GP_LAUNCH_CHECK();
    tot = (int64_t)p.col_tiles * GBN * p.WK;
    r_image_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(R, ldrr, nc, w, p.WK, p.col_tiles, r_img);
    GP_LAUNCH_CHECK();
    if (ard) {
      tot = (int64_t)p.col_tiles * GBN * p.DP;
      col_xy_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Xc, ldc, nc, d, p.DP, p.col_tiles, col_xy);
      GP_LAUNCH_CHECK();
    }
  }
  GArgs a;
  a.row_img = row_img; a.col_img = col_img; a.r_img = r_img; a.y_rows = y_rows; a.col_xy = col_xy;
  a.Xr = Xr; a.ldr = ldr; a.DK = p.DK; a.WK = p.WK; a.WKP = p.WKP; a.DP = p.DP; a.d = d;
  a.n_rows = nr; a.n_cols = nc; a.row_tiles = p.row_tiles; a.col_tiles = p.col_tiles;
  a.splits = p.splits; a.tiles_per_split = p.tiles_per_split; a.nstages = p.nstages;
  a.self_offset = self_offset; a.partials = partials;
  a.items = sym ? items : nullptr;
  a.n_items = p.n_items;
  const int nchunks = ard ? (d + G_MAXNL - 1) / G_MAXNL : 1;
  for (int ch = 0; ch < nchunks; ++ch) {
    a.p0 = ch * G_MAXNL;
    a.nl = ard ? std::min(G_MAXNL, d - a.p0) : 1;
    void (*kern)(GArgs);
    if (family == GP_FAMILY_RBF) kern = ard ? grad_tc_kernel<GP_FAMILY_RBF, true> : grad_tc_kernel<GP_FAMILY_RBF, false>;
    else kern = ard ? grad_tc_kernel<GP_FAMILY_MATERN32, true> : grad_tc_kernel<GP_FAMILY_MATERN32, false>;
    GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
    kern<<<p.grid, G_NTHREADS, p.smem, st>>>(a);
    GP_LAUNCH_CHECK();
    grad_tc_finalize<<<1, 32, 0, st>>>(partials, p.grid, a.p0, a.nl, ch == 0, out);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

}  // namespace gp
