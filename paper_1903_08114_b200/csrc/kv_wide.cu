// Wide-RHS tcgen05 K·V kernel (16 < t <= 256) for sm_100a: the predictive-
// variance solves (predictor.py:135-182 batches 256 test points per chunk)
// and any caller with many right-hand sides.
//
// Same tile pipeline as kv_tc.cu (persistent CTA per SM, TMA producer warp,
// one elected MMA-issuing thread, epilogue warps computing kappa on the SFU),
// but the contraction has N = t_pad (up to 256) and is tensor-bound rather
// than SFU-bound: per 128 x 64 tile, O += K1.V1 + K1.V2 + K2.V1 (kind::f16,
// 2-term fp16 splits of K and of the column-scaled V, fp32 accumulation in
// TMEM), 12 MMAs of N = t_pad. O (t_pad TMEM columns) accumulates over CH
// column tiles and is then folded into an fp32 accumulator in global memory by
// TMA bulk reduce-adds (cp.reduce.async.bulk, 2 KB per warp block, issued in a
// fixed order per element: deterministic),
// bounding the length of any TMEM accumulation chain (long TMEM accumulation
// loses precision, measured in kv_tc.cu).
//
// Reference semantics: kernels.py:225-244 (kappa), :293-316 / :319-325 (rows
// of K̂ / cross blocks), partition.py:224-241 (row-block products).
#include "tc_common.cuh"

#include <algorithm>

namespace gp {
namespace tw {

using namespace gp::tc;

constexpr int BM = 128;
constexpr int TMAX = 256;          // widest right-hand-side block
constexpr int CH = 32;             // column tiles per TMEM accumulation chain
constexpr int NUM_EPI_WARPS = 8;   // two per TMEM lane quarter, 32 columns of a tile each
constexpr int NTHREADS = 32 * (4 + NUM_EPI_WARPS);

struct Args {
  const float* row_img;   // [row tiles][2][BM*DK]
  const float* col_img;   // [col tiles][2][BN*DK]
  const __half* v_img;    // [col tiles][2*NW x 64] fp16 [V1 | V2]
  const float* inv_vscale;  // [t] 2^-s_c
  const float* dscale;    // large d: fp16 distance images, S = S' dscale (null: tf32 images)
  int DK, NW;             // NW = t rounded up to 16
  int64_t n_rows, n_cols;
  int row_tiles, col_tiles, splits, tiles_per_split;
  int nsc, nsv;           // column-image ring and V ring depths
  int t;
  float s2, noise;
  int64_t diag_offset, self_offset;
  float* accw;            // [splits][NW][rows_pad] column-major fp32 partial sums
  int64_t rows_pad;
  int nfold;              // fold staging buffers per epilogue warp (2, or 1 when SMEM is tight)
};

// accumulator layout (fp32): [split][row tile][lane quarter q][column][32 rows],
// so one epilogue warp's 32 rows x 16 columns block is 2 KB contiguous and is
// folded with a single TMA bulk reduce-add (cp.reduce.async.bulk .add.f32)
__host__ __device__ __forceinline__ int64_t accw_index(int64_t sp, int64_t rt, int row_tiles, int q, int NW, int col,
                                                       int l) {
  return ((((sp * row_tiles + rt) * 4 + q) * NW + col) * 32) + l;
}
constexpr uint32_t STAGE_FOLD_BYTES = 32u * 16u * 4u;   // one warp's 32 x 16 fp32 block

__device__ __forceinline__ void bulk_reduce_add_f32(const void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// TMEM: S 2 x 64 | K1 32 + K2 32 (x2 buffers) | O NW (<= 256)
__device__ __forceinline__ uint32_t TMS(uint32_t b) { return b * 64; }
__device__ __forceinline__ uint32_t TMK1(uint32_t b) { return 128 + b * 64; }
__device__ __forceinline__ uint32_t TMK2(uint32_t b) { return 160 + b * 64; }
constexpr uint32_t TMO = 256;

// BNT: column tile width (64, or 32 when the augmented width DK > 32: the
// d <= 94 images of C4-shaped inputs, whose 96-wide row image alone takes
// 96 KB of SMEM). Each of the 8 epilogue warps covers CW = BNT / 2 columns.
template <int FAM, int BNT>
__global__ void __launch_bounds__(NTHREADS, 1) kv_wide_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int BN = BNT;
  constexpr int CW = BNT / 2;
  const int DK = a.DK, NW = a.NW;
  const bool F16I = a.dscale != nullptr;   // fp16 hi | lo distance images (large d)
  const uint32_t EB = F16I ? 2u : 4u;
  const uint32_t row_bytes = 2u * BM * DK * EB;
  const uint32_t col_bytes = 2u * BN * DK * EB;
  const uint32_t v_bytes = 2u * NW * BN * 2u;
  const int NSC = a.nsc, NSV = a.nsv;
  uint8_t* xr_s = smem;
  uint8_t* cring = smem + row_bytes;           // [NSC] column images (distance B operand)
  uint8_t* vring = cring + NSC * col_bytes;    // [NSV] V images (contraction B operand)
  uint64_t* bars = reinterpret_cast<uint64_t*>(vring + NSV * v_bytes);
  // separate rings: the small column images run far ahead of the 64 KB V
  // tiles, so the distance product of the next tile never waits on a V load
  uint64_t* cfull = bars;                 // [NSC]
  uint64_t* cempty = cfull + NSC;         // [NSC]
  uint64_t* vfull = cempty + NSC;         // [NSV]
  uint64_t* vempty = vfull + NSV;         // [NSV]
  uint64_t* s_full = vempty + NSV;        // [2]
  uint64_t* k_full = s_full + 2;     // [2]
  uint64_t* k_empty = k_full + 2;    // [2]
  uint64_t* o_full = k_empty + 2;    // chunk accumulated
  uint64_t* o_empty = o_full + 1;    // chunk folded into the destination
  uint64_t* xr_full = o_empty + 1;
  uint64_t* xr_empty = xr_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xr_empty + 1);
  float* fold_s = reinterpret_cast<float*>(vring + NSV * v_bytes + 512);   // [8 warps][nfold][32 x 16]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSC; ++s) {
      mbar_init(smem_u32(&cfull[s]), 1);
      mbar_init(smem_u32(&cempty[s]), 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(smem_u32(&vfull[s]), 1);
      mbar_init(smem_u32(&vempty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&s_full[b]), 1);
      mbar_init(smem_u32(&k_full[b]), NUM_EPI_WARPS);
      mbar_init(smem_u32(&k_empty[b]), 1);
    }
    mbar_init(smem_u32(o_full), 1);
    mbar_init(smem_u32(o_empty), NUM_EPI_WARPS);
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
    // ===================== TMA producer: row and column images =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0, itc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
        const int rt = it / a.splits, sp = it - rt * a.splits;
        const int ct0 = sp * a.tiles_per_split;
        const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
        mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
        mbar_expect_tx(smem_u32(xr_full), row_bytes);
        bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)rt * (row_bytes / 4), row_bytes, smem_u32(xr_full));
        const float* cimg = a.col_img + (int64_t)ct0 * (col_bytes / 4);
        for (int ct = ct0; ct < ct1; ++ct) {
          mbar_wait(smem_u32(&cempty[s]), ph ^ 1);
          mbar_expect_tx(smem_u32(&cfull[s]), col_bytes);
          bulk_g2s(smem_u32(cring + s * col_bytes), cimg, col_bytes, smem_u32(&cfull[s]));
          cimg += col_bytes / 4;
          if (++s == (uint32_t)NSC) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 3) {
    // ===================== TMA producer: V tiles =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const int sp = it % a.splits;
        const int ct0 = sp * a.tiles_per_split;
        const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
        const uint8_t* vimg = reinterpret_cast<const uint8_t*>(a.v_img) + (int64_t)ct0 * v_bytes;
        for (int ct = ct0; ct < ct1; ++ct) {
          mbar_wait(smem_u32(&vempty[s]), ph ^ 1);
          mbar_expect_tx(smem_u32(&vfull[s]), v_bytes);
          bulk_g2s(smem_u32(vring + s * v_bytes), vimg, v_bytes, smem_u32(&vfull[s]));
          vimg += v_bytes;
          if (++s == (uint32_t)NSV) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    const uint32_t idesc_d = F16I ? idesc_f16(BM, BN) : make_idesc(BM, BN);
    const uint32_t idesc_c = idesc_f16(BM, NW);
    const uint32_t lbo_a = (BM / 8) * 128, lbo_b = (BN / 8) * 128, lbo_v = (2 * NW / 8) * 128;
    const uint32_t a_half16 = (BM * DK * EB) >> 4, b_half16 = (BN * DK * EB) >> 4;
    const uint32_t v2_16 = ((NW / 8) * 128) >> 4;   // V2 rows start NW/8 core rows down
    const int ksteps = F16I ? DK / 16 : DK / 8;   // 32 B of K per row and MMA either way
    const uint64_t da0 = make_desc(smem_u32(xr_s), lbo_a, 128);
    const uint64_t db0 = make_desc(smem_u32(cring), lbo_b, 128);
    const uint64_t dv0 = make_desc(smem_u32(vring), lbo_v, 128);
    const uint32_t col16 = col_bytes >> 4, v16 = v_bytes >> 4;
    const uint32_t kstep_a16 = (2 * lbo_a) >> 4, kstep_b16 = (2 * lbo_b) >> 4, kstep_v16 = (2 * lbo_v) >> 4;
    const bool leader = elect_one();
    uint32_t ds = 0, dph = 0, vs = 0, vph = 0, sbn = 0, kb = 0, kph = 0, oph = 0;
    uint32_t itc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++itc) {
      const int sp = it % a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      const int J = ct1 - ct0;
      mbar_wait(smem_u32(xr_full), itc & 1);
      tc_fence_after();
      auto dist = [&]() {
        mbar_wait(smem_u32(&cfull[ds]), dph);
        tc_fence_after();
        const uint32_t d_tm = tmem + TMS(sbn);
        const uint64_t db = db0 + (uint64_t)(ds * col16);
        if (leader) {
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint64_t a_p = da0 + (pass == 0 ? a_half16 : 0u);
            const uint64_t b_p = db + (pass == 1 ? b_half16 : 0u);
            for (int ks = 0; ks < ksteps; ++ks) {
              if (F16I)
                mma16_ss(d_tm, a_p + (uint64_t)(ks * kstep_a16), b_p + (uint64_t)(ks * kstep_b16), idesc_d,
                         (pass | ks) != 0);
              else
                mma_ss(d_tm, a_p + (uint64_t)(ks * kstep_a16), b_p + (uint64_t)(ks * kstep_b16), idesc_d,
                       (pass | ks) != 0);
            }
          }
          tc_commit(smem_u32(&s_full[sbn]));
          tc_commit(smem_u32(&cempty[ds]));
        }
        __syncwarp();
        if (++ds == (uint32_t)NSC) { ds = 0; dph ^= 1; }
        sbn ^= 1;
      };
      dist();
      for (int jj = 0; jj < J; ++jj) {
        if (jj + 1 < J) dist();   // S buffer of tile jj+1 was read by the epilogue of tile jj-1 (k_full seen)
        mbar_wait(smem_u32(&k_full[kb]), kph);
        tc_fence_after();
        const bool chunk_start = (jj % CH) == 0;
        if (chunk_start) {   // the previous chunk's O has been folded
          mbar_wait(smem_u32(o_empty), oph ^ 1);
          tc_fence_after();
        }
        mbar_wait(smem_u32(&vfull[vs]), vph);
        tc_fence_after();
        const uint64_t vb = dv0 + (uint64_t)(vs * v16);
        const uint32_t k1 = tmem + TMK1(kb), k2 = tmem + TMK2(kb);
        if (leader) {
          // O += K1.V1 + K1.V2 + K2.V1  (K = 64 = 4 x 16, N = NW)
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks)
            mma16_ts(tmem + TMO, k1 + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c, !(chunk_start && ks == 0));
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks)
            mma16_ts(tmem + TMO, k1 + ks * 8, vb + (uint64_t)(v2_16 + ks * kstep_v16), idesc_c, 1);
#pragma unroll
          for (int ks = 0; ks < BN / 16; ++ks)
            mma16_ts(tmem + TMO, k2 + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c, 1);
          tc_commit(smem_u32(&vempty[vs]));
          tc_commit(smem_u32(&k_empty[kb]));
          if ((jj % CH) == CH - 1 || jj == J - 1) tc_commit(smem_u32(o_full));
        }
        __syncwarp();
        if ((jj % CH) == CH - 1 || jj == J - 1) oph ^= 1;
        if (++vs == (uint32_t)NSV) { vs = 0; vph ^= 1; }
        if (++kb == 2) { kb = 0; kph ^= 1; }
      }
      if (leader) tc_commit(smem_u32(xr_empty));
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ===================== epilogue (8 warps) =====================
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    uint32_t sb = 0, sph = 0, kb = 0, kph = 0, oph = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const int rt = it / a.splits, sp = it - rt * a.splits;
      const int ct0 = sp * a.tiles_per_split;
      const int ct1 = min(a.col_tiles, ct0 + a.tiles_per_split);
      const int J = ct1 - ct0;
      const int64_t row = (int64_t)rt * BM + q * 32 + lane;
      const int64_t diag_col = (a.self_offset >= 0 && row < a.n_rows) ? row + a.self_offset : -1000;
      float* dst = a.accw + accw_index(sp, rt, a.row_tiles, q, NW, 0, 0);   // this warp's [col][32] slab
      for (int jj = 0; jj < J; ++jj) {
        mbar_wait(smem_u32(&s_full[sb]), sph);
        tc_fence_after();
        uint32_t v[32];
        if constexpr (CW == 32) {
          tmem_ld32(tmem + lane_base + TMS(sb) + half * CW, v);
        } else {
          tmem_ld16(tmem + lane_base + TMS(sb) + half * CW, *reinterpret_cast<uint32_t(*)[16]>(v));
        }
        tmem_wait_ld();
        const int64_t e_diag = diag_col - ((int64_t)(ct0 + jj) * BN + half * CW);
        if (__any_sync(0xffffffffu, e_diag >= 0 && e_diag < CW)) {
#pragma unroll
          for (int e = 0; e < CW; ++e)
            if (e == e_diag) v[e] = 0u;   // same point on both sides: r2 = 0 exactly
        }
        const float dsc = F16I ? *a.dscale : 1.f;
#pragma unroll
        for (int e = 0; e < CW; ++e) {
          // x 2^12 for the fp16 split; the finalize's inv_vscale divides it out
          v[e] = __float_as_uint(kappa_split_scaled<FAM>(__uint_as_float(v[e]) * dsc));
        }
        mbar_wait(smem_u32(&k_empty[kb]), kph ^ 1);   // K[kb] was read two tiles ago
        tc_fence_after();
#pragma unroll
        for (int s16 = 0; s16 < CW / 16; ++s16) {
          uint32_t p1[8], p2[8];
#pragma unroll
          for (int k = 0; k < 8; ++k)
            split_pair(__uint_as_float(v[16 * s16 + 2 * k]), __uint_as_float(v[16 * s16 + 2 * k + 1]), p1[k], p2[k]);
          tmem_st8(tmem + lane_base + TMK1(kb) + half * (CW / 2) + 8 * s16, p1);
          tmem_st8(tmem + lane_base + TMK2(kb) + half * (CW / 2) + 8 * s16, p2);
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&k_full[kb]));
        if (++sb == 2) { sb = 0; sph ^= 1; }
        if (++kb == 2) { kb = 0; kph ^= 1; }
        if ((jj % CH) == CH - 1 || jj == J - 1) {
          // fold the chunk: this warp's lane quarter, alternate 16-column blocks per half
          mbar_wait(smem_u32(o_full), oph);
          oph ^= 1;
          tc_fence_after();
          // the previous fold's bulk reductions into this slab must be complete
          // (keeps the per-element addition order fixed: deterministic)
          if (lane == 0) bulk_wait_all();
          __syncwarp();
          float* stg0 = fold_s + (warp - 4) * a.nfold * (32 * 16);
          int buf = 0;
          for (int c0 = half * 16; c0 < NW; c0 += 32, buf = a.nfold == 2 ? buf ^ 1 : 0) {
            uint32_t o[16];
            tmem_ld16(tmem + lane_base + TMO + c0, o);
            if (lane == 0) {   // staging buffer `buf` free again
              if (a.nfold == 2) bulk_wait_read1(); else asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
            __syncwarp();
            tmem_wait_ld();
            float* stg = stg0 + buf * (32 * 16);
#pragma unroll
            for (int c = 0; c < 16; ++c) stg[c * 32 + lane] = __uint_as_float(o[c]);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              bulk_reduce_add_f32(dst + (int64_t)c0 * 32, smem_u32(stg), STAGE_FOLD_BYTES);
              bulk_commit();
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(o_empty));
        }
      }
    }
  }

  if (warp >= 4 && lane == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// out[i, c] = s2 2^-s_c sum_splits accw[sp][c][i] (+ noise V[i + diag_offset, c])
__global__ void kv_wide_finalize(const float* __restrict__ accw, int splits, int NW, int row_tiles,
                                 int64_t nr, int t, const float* __restrict__ inv_vscale, float* out, int64_t ldo,
                                 float s2, float noise, const float* __restrict__ V, int64_t ldv,
                                 int64_t diag_offset) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr * t) return;
  const int c = (int)(idx / nr);
  const int64_t i = idx - (int64_t)c * nr;   // consecutive threads: consecutive rows (coalesced reads)
  const int64_t rt = i / 128;
  const int q = (int)((i / 32) & 3), l = (int)(i & 31);
  float acc = 0.f;
  for (int sp = 0; sp < splits; ++sp) acc += accw[accw_index(sp, rt, row_tiles, q, NW, c, l)];
  float r = s2 * acc * inv_vscale[c];
  if (diag_offset >= 0) r = fmaf(noise, V[(i + diag_offset) * ldv + c], r);
  out[i * ldo + c] = r;
}

struct Plan {
  int DK, NW, BN, nfold, row_tiles, col_tiles, splits, tiles_per_split, nsc, nsv;
  int eb;   // bytes per distance-image element: 2 (fp16 hi | lo, DK >= 48) or 4 (tf32)
  int64_t rows_pad;
  size_t row_img_bytes, col_img_bytes, v_img_bytes, split_bytes, smem;
};

// SMEM rings for column tile width bn with nfold staging buffers per
// epilogue warp; false when a 2-deep column ring and 2-deep V ring do not fit
static bool fit_rings(Plan& p, int bn, int nfold, size_t cap) {
  const size_t row_b = 2u * BM * p.DK * p.eb, col_b = 2u * bn * p.DK * p.eb, v_b = 2u * p.NW * bn * 2;
  const size_t fold_b = (size_t)NUM_EPI_WARPS * nfold * STAGE_FOLD_BYTES;
  if (row_b + 512 + fold_b + 2 * col_b + 2 * v_b > cap) return false;
  const size_t budget = cap - row_b - 512 - fold_b;
  // V ring as deep as fits next to a 2-deep column ring (at most 4), then the
  // column ring takes the rest (at most 8)
  p.nsv = (int)std::min<size_t>(4, (budget - 2 * col_b) / v_b);
  p.nsc = (int)std::min<size_t>(8, (budget - p.nsv * v_b) / col_b);
  p.BN = bn;
  p.nfold = nfold;
  p.smem = row_b + p.nsc * col_b + p.nsv * v_b + 512 + fold_b;
  return true;
}

static Plan make_plan(const gp_kv_desc* d, int t) {
  Plan p;
  p.DK = (d->d + 2 + 7) / 8 * 8;
  p.NW = (t + 15) / 16 * 16;
  p.eb = p.DK >= 48 ? 2 : 4;
  // 64-point column tiles with double-buffered fold staging (the tuned
  // d <= 30 configuration); for large d (C4: DK = 96, a 96 KB row image)
  // 32-point tiles and single-buffered staging in the full 227 KB
  p.nsv = p.nsc = 0;
  if (!fit_rings(p, 64, 2, 224 * 1024) && !fit_rings(p, 32, 2, 227 * 1024 - 1024) &&
      !fit_rings(p, 32, 1, 227 * 1024 - 1024)) {
    p.BN = 32;
    p.nfold = 1;
  }
  const int BN = p.BN;
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
  p.v_img_bytes = (size_t)p.col_tiles * 2 * p.NW * BN * 2;
  p.rows_pad = (int64_t)p.row_tiles * BM;
  p.split_bytes = (size_t)p.splits * p.NW * p.rows_pad * 4 + 256 * sizeof(double) + 2 * TMAX * sizeof(float) +
                  8 * sizeof(float);
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace tw

bool kv_wide_supported(const gp_kv_desc* d, int t) {
  if (t <= 16 || t > tw::TMAX) return false;
  if (d->d < 1 || d->d + 2 > 96) return false;   // DK <= 96 (d <= 94, the kv_tc limit)
  const tw::Plan p = tw::make_plan(d, t);
  return p.nsv >= 2 && p.nsc >= 2;
}

size_t kv_wide_workspace(const gp_kv_desc* d, int t) {
  if (!kv_wide_supported(d, t)) return 0;
  tw::Plan p = tw::make_plan(d, t);
  using tw::align256;
  return align256(p.row_img_bytes) + align256(p.col_img_bytes) + align256(p.v_img_bytes) + align256(p.split_bytes);
}

int kv_wide(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo, void* ws,
            size_t ws_bytes, cudaStream_t st) {
  using namespace tw;
  Plan p = make_plan(desc, t);
  size_t need = kv_wide_workspace(desc, t);
  GP_REQUIRE(ws != nullptr && ws_bytes >= need, "gp_kv(wide): workspace of %zu bytes required, %zu given", need,
             ws_bytes);
  char* w = static_cast<char*>(ws);
  float* row_img = reinterpret_cast<float*>(w); w += align256(p.row_img_bytes);
  float* col_img = reinterpret_cast<float*>(w); w += align256(p.col_img_bytes);
  __half* v_img = reinterpret_cast<__half*>(w); w += align256(p.v_img_bytes);
  double* mean = reinterpret_cast<double*>(w); w += 256 * sizeof(double);
  float* vscale = reinterpret_cast<float*>(w); w += TMAX * sizeof(float);
  float* inv_vscale = reinterpret_cast<float*>(w); w += TMAX * sizeof(float);
  unsigned* rng = reinterpret_cast<unsigned*>(w); w += 4 * sizeof(unsigned);
  float* dscale = reinterpret_cast<float*>(w); w += 4 * sizeof(float);
  float* accw = reinterpret_cast<float*>(w);
  const double c = desc->family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  if (p.eb == 2) {
    if (int rc = tc::distance_images16(desc->Xr, desc->ldr, desc->n_rows, desc->Xc, desc->ldc, desc->n_cols,
                                       desc->d, p.DK, BM, p.BN, c, mean, rng, reinterpret_cast<__half*>(row_img),
                                       reinterpret_cast<__half*>(col_img), dscale, st))
      return rc;
  } else if (int rc = tc::distance_images(desc->Xr, desc->ldr, desc->n_rows, desc->Xc, desc->ldc, desc->n_cols,
                                          desc->d, p.DK, BM, p.BN, c, mean, row_img, col_img, st)) {
    return rc;
  }
  if (int rc = tc::v_colscale(V, ldv, desc->n_cols, t, vscale, inv_vscale, st)) return rc;
  if (int rc = tc::v_images16_wide(V, ldv, t, p.NW, desc->n_cols, vscale, v_img, p.col_tiles, st, p.BN)) return rc;
  Args a;
  a.row_img = row_img; a.col_img = col_img; a.v_img = v_img; a.inv_vscale = inv_vscale;
  a.dscale = p.eb == 2 ? dscale : nullptr;
  a.DK = p.DK; a.NW = p.NW;
  a.n_rows = desc->n_rows; a.n_cols = desc->n_cols;
  a.row_tiles = p.row_tiles; a.col_tiles = p.col_tiles; a.splits = p.splits;
  a.tiles_per_split = p.tiles_per_split; a.nsc = p.nsc; a.nsv = p.nsv; a.t = t;
  a.s2 = (float)desc->outputscale; a.noise = (float)desc->noise; a.diag_offset = desc->diag_offset;
  a.self_offset = desc->self_offset;
  a.accw = accw; a.rows_pad = p.rows_pad; a.nfold = p.nfold;
  GP_CUDA_TRY(cudaMemsetAsync(accw, 0, (size_t)p.splits * p.NW * p.rows_pad * 4, st));
  int items = p.row_tiles * p.splits;
  int grid = std::min(items, num_sms());
  auto kern = desc->family == GP_FAMILY_RBF
                  ? (p.BN == 64 ? kv_wide_kernel<GP_FAMILY_RBF, 64> : kv_wide_kernel<GP_FAMILY_RBF, 32>)
                  : (p.BN == 64 ? kv_wide_kernel<GP_FAMILY_MATERN32, 64> : kv_wide_kernel<GP_FAMILY_MATERN32, 32>);
  GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  kern<<<grid, NTHREADS, p.smem, st>>>(a);
  GP_LAUNCH_CHECK();
  const int64_t tot = desc->n_rows * (int64_t)t;
  kv_wide_finalize<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(accw, p.splits, p.NW, p.row_tiles, desc->n_rows, t,
                                                                  inv_vscale, out, ldo, a.s2, a.noise, V, ldv,
                                                                  desc->diag_offset);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

}  // namespace gp
