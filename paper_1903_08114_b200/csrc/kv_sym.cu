// Symmetric tcgen05 K·V kernel for the square training operator (sm_100a).
//
// out = s2 * kappa(X, X) V (+ noise V), evaluating every unordered pair of
// points ONCE: K is symmetric, so the tile K_IJ (row tile I, column tile J
// strictly above the 128 x 128 diagonal block) serves both
//     out_I += K_IJ   V_J      (direct:  A = K from TMEM, as in kv_tc.cu)
//     out_J += K_IJ^T V_I      (mirror:  A = K^T from TMEM, M = 64)
// which halves the transcendental (SFU) work that bounds the kernel at CG
// width. Diagonal blocks are evaluated in full, direct only.
//
// The mirror product needs K^T with j in TMEM lanes while the distance tile
// lands with i in lanes, so each mirrored tile is transposed once through a
// double-buffered fp32 SMEM tile (producers store kappa, one 4-byte store per
// entry; consumers load 8-byte pairs, split tf32 hi/lo and write the M = 64
// TMEM operand with 16x256b stores: hi in lanes 0-15, lo in lanes 16-31).
// Reading K^T from TMEM rather than SMEM keeps the tensor core off the SMEM
// port (an SS-form mirror was measured 0.74x of the row-tiled kernel); the
// row image is TMEM-resident too (TS-form distance product).
//
// Contributions to one output row come from many CTAs, so they are summed in
// 64-bit FIXED POINT (red.global.add.u64, per-column scale 2^E_c chosen from
// ||V_c||_1 so no partial can overflow): integer addition is associative, so
// the result is bitwise reproducible run to run and independent of the CTA
// schedule, like the reference's partition-count independence
// (test_partition.py:92-102). Quantisation error per partial is
// <= ||V_c||_1 2^-62 (~1e-13 relative at n = 10^6), far below fp32 round-off.
//
// Reference semantics: kernels.py:225-244 (kappa), :293-316 (rows of K̂ incl.
// the sigma^2 diagonal), partition.py:224-241 (row-block products).
#include "tc_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace gp {
namespace tcs {

using namespace gp::tc;

constexpr int BM = 128;   // rows per tile (UMMA M of the direct product)
constexpr int BN = 64;    // columns per tile (UMMA M of the mirror product)
constexpr int TN = 16;    // right-hand sides
constexpr int NTHREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int NUM_EPI_WARPS = 8;
// fp32 kappa^T staging tile in SMEM (double buffered): element (j, i) at
// j * KT_LD + i. Producers (lane = i) store conflict-free; the row stride of
// 136 floats (8 banks) makes the consumers' 8-byte loads (16x256b fragment:
// rows j = lane/4, columns 2(lane%4)) conflict-free as well.
constexpr int KT_LD = 136;
constexpr uint32_t KT32_BYTES = 64u * KT_LD * 4u;
constexpr uint32_t V_TILE_BYTES = 2u * TN * BN * 4u;  // hi + lo image of one 64-column V tile

struct Args {
  const float* row_img;   // [row tiles][2][BM*DK]
  const float* col_img;   // [col tiles][2][BN*DK]
  const float* v_img;     // [col tiles][2][TN*BN]
  int DK;
  int64_t n;
  int row_tiles, col_tiles, splits, n_items;
  int nstages, lookahead;
  int t;
  const int* expo;                  // [TN] E_c: partials are summed as round(v 2^E_c)
  unsigned long long* acc;          // [TN][acc_ld] fixed-point sums (column-major)
  int64_t acc_ld;
  int* bad;                         // [acc_ld] non-finite partial seen for the row
  long long* prof;                  // optional per-warp phase cycle counters (GP_SYM_PROF=1)
  int atom_mode;                    // diagnostic: 0 fixed-point u64, 1 none, 2 f32, 3 convert only
};

// phase timing for the GP_SYM_PROF diagnostic (lane counters, no effect when a.prof == nullptr)
#define SYM_T(slot, ...)                                  \
  do {                                                    \
    const long long _t0 = a.prof ? clock64() : 0;         \
    __VA_ARGS__;                                          \
    if (a.prof) tacc[slot] += clock64() - _t0;            \
  } while (0)

// TMEM columns (512):
//   SK 2 x 128: the distance tile S lands in [0, 64) of buffer b and the
//     epilogue overwrites it in place with K_hi, K_lo going to [64, 128)
//   K^T 128 (M = 64 layout: hi in lanes 0-15, lo in lanes 16-31 of each
//     sub-partition) | row image hi|lo 2 x DK (DK <= 16)
//   O_I 32 = [K_hi V_hi + K_lo V_hi | K_hi V_lo]
//   O_J 2 x 32 (lanes 0-15 [KT_hi V_hi | KT_hi V_lo], lanes 16-31 [KT_lo V_hi | -])
__device__ __forceinline__ uint32_t TMSK(uint32_t b) { return b * 128; }
constexpr uint32_t TMKT = 256, TMXA = 384, TMO = 448;
__device__ __forceinline__ uint32_t TMOJ(uint32_t b) { return b ? 416 : 480; }
__device__ __forceinline__ void red_add_u64(unsigned long long* p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// row-tile items: item L = I * splits + sp covers column tiles
// [2I + sp*C, min(col_tiles, 2I + (sp+1)*C)), C = ceil((col_tiles - 2I) / splits)
struct Item {
  int rt, ct0, ct1;
};
__device__ __forceinline__ Item item_of(const Args& a, int L) {
  Item it;
  it.rt = L / a.splits;
  const int sp = L - it.rt * a.splits;
  const int lo = 2 * it.rt;
  const int m = a.col_tiles - lo;
  const int C = (m + a.splits - 1) / a.splits;
  it.ct0 = lo + sp * C;
  it.ct1 = min(a.col_tiles, it.ct0 + C);
  return it;
}
// boustrophedon assignment of items to persistent CTAs: item sizes fall
// linearly with the row tile, so alternating the direction each round
// balances the per-CTA totals
__device__ __forceinline__ int item_index(int r, int b, int G) {
  return r * G + ((r & 1) ? (G - 1 - b) : b);
}

// v * 2^E as a (truncated) signed 64-bit integer, on the integer pipes: the
// F2I.S64 conversion runs on the SFU's XU pipe, which the kappa epilogue
// saturates. Exact for |v| 2^E >= 2^23; smaller magnitudes lose their
// sub-unit fraction (<= 2^-E absolute, i.e. <= ||V_c||_1 2^-61).
__device__ __forceinline__ long long fixed_point(float v, int E) {
  const uint32_t bits = __float_as_uint(v);
  const int sh = (int)((bits >> 23) & 0xFFu) - 150 + E;      // |v| 2^E = m 2^sh
  const uint64_t m = (uint64_t)((bits & 0x7FFFFFu) | 0x800000u);
  uint64_t mag = sh >= 0 ? (m << min(sh, 39)) : (sh > -24 ? (m >> -sh) : 0ull);
  if (((bits >> 23) & 0xFFu) == 0u) mag = 0ull;                 // zero / denormal
  return (bits >> 31) ? -(long long)mag : (long long)mag;
}

// one fixed-point contribution (lane-parallel)
__device__ __forceinline__ void contribute(const Args& a, int64_t row, int c, float v, int E) {
  if (!(fabsf(v) < INFINITY)) {
    a.bad[row] = 1;
    return;
  }
  if (a.atom_mode == 1) return;
  if (a.atom_mode == 2) {
    atomicAdd(reinterpret_cast<float*>(a.acc + (int64_t)c * a.acc_ld + row), v);
    return;
  }
  const long long q = fixed_point(v, E);
  if (a.atom_mode == 3) {
    if (q == 0x7fffffffffffffffLL) a.bad[row] = 2;
    return;
  }
  red_add_u64(a.acc + (int64_t)c * a.acc_ld + row, q);
}

template <int FAM>
__global__ void __launch_bounds__(NTHREADS, 1) kv_sym_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const int DK = a.DK;
  const uint32_t row_bytes = 2u * BM * DK * 4u;
  const uint32_t col_bytes = 2u * BN * DK * 4u;
  const uint32_t v_bytes = V_TILE_BYTES;
  const uint32_t stage_bytes = col_bytes + v_bytes;
  const int NS = a.nstages;
  float* kt32 = reinterpret_cast<float*>(smem);                   // [2][64][KT_LD] fp32 kappa^T
  uint8_t* xr_s = smem + 2 * KT32_BYTES;                          // row image (TMA)
  uint8_t* vi_s = xr_s + row_bytes;                               // V image of the row tile
  uint8_t* stages = vi_s + 2 * v_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(stages + NS * stage_bytes);
  uint64_t* full = bars;             // [NS]  TMA -> MMA
  uint64_t* empty = bars + NS;       // [NS]  MMA -> TMA
  uint64_t* s_full = bars + 2 * NS;  // [2]   distance tile landed in SK buffer b
  uint64_t* k_empty = s_full + 2;    // [2]   direct product done reading K in SK buffer b
  uint64_t* k_full = k_empty + 2;    // K written over S (+ O_I drained)
  uint64_t* o_full = k_full + 1;     // direct product done
  uint64_t* o_empty = o_full + 1;    // O_I read
  uint64_t* kt_full = o_empty + 1;   // K^T written (+ O_J drained)
  uint64_t* kt_empty = kt_full + 1;  // mirror product done reading K^T
  uint64_t* oj_full = kt_empty + 1;  // [2] mirror product done
  uint64_t* oj_empty = oj_full + 2;  // [2] O_J read
  uint64_t* xr_full = oj_empty + 2;  // row image + V_I landed
  uint64_t* xr_empty = xr_full + 1;  // item's products done with them
  uint64_t* xa_full = xr_empty + 1;  // row image copied into TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xa_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), 1);
    }
    mbar_init(smem_u32(&s_full[0]), 1);
    mbar_init(smem_u32(&s_full[1]), 1);
    mbar_init(smem_u32(&k_empty[0]), 1);
    mbar_init(smem_u32(&k_empty[1]), 1);
    mbar_init(smem_u32(k_full), NUM_EPI_WARPS);
    mbar_init(smem_u32(o_full), 1);
    mbar_init(smem_u32(o_empty), 4);
    mbar_init(smem_u32(kt_full), NUM_EPI_WARPS);
    mbar_init(smem_u32(kt_empty), 1);
    for (int q = 0; q < 2; ++q) {
      mbar_init(smem_u32(&oj_full[q]), 1);
      mbar_init(smem_u32(&oj_empty[q]), 4);
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
  const int G = gridDim.x, b = blockIdx.x;
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      uint32_t s = 0, ph = 0, itc = 0;
      for (int r = 0;; ++r) {
        const int L = item_index(r, b, G);
        if (L >= a.n_items) break;
        const Item it = item_of(a, L);
        if (it.ct1 <= it.ct0) continue;
        mbar_wait(smem_u32(xr_empty), (itc & 1) ^ 1);
        const int vt = min(2, a.col_tiles - 2 * it.rt);  // V tiles of this row tile
        mbar_expect_tx(smem_u32(xr_full), row_bytes + vt * v_bytes);
        bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)it.rt * (row_bytes / 4), row_bytes, smem_u32(xr_full));
        bulk_g2s(smem_u32(vi_s), a.v_img + (int64_t)(2 * it.rt) * (v_bytes / 4), vt * v_bytes,
                 smem_u32(xr_full));
        ++itc;
        const float* cimg = a.col_img + (int64_t)it.ct0 * (col_bytes / 4);
        const float* vimg = a.v_img + (int64_t)it.ct0 * (v_bytes / 4);
        for (int ct = it.ct0; ct < it.ct1; ++ct) {
          mbar_wait(smem_u32(&empty[s]), ph ^ 1);
          uint8_t* st = stages + s * stage_bytes;
          mbar_expect_tx(smem_u32(&full[s]), stage_bytes);
          bulk_g2s(smem_u32(st), cimg, col_bytes, smem_u32(&full[s]));
          bulk_g2s(smem_u32(st + col_bytes), vimg, v_bytes, smem_u32(&full[s]));
          cimg += col_bytes / 4;
          vimg += v_bytes / 4;
          if (++s == (uint32_t)NS) { s = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // per tile, in tensor-pipe order: direct(jj), mirror(jj), dist(jj+2) --
    // dist(jj+2) overwrites the SK buffer direct(jj) just consumed
    const uint32_t idesc_d = make_idesc(BM, BN);
    const uint32_t idesc_c32 = make_idesc(BM, 2 * TN), idesc_c16 = make_idesc(BM, TN);
    const uint32_t idesc_m32 = make_idesc(BN, 2 * TN), idesc_m16 = make_idesc(BN, TN);
    const uint32_t lbo_b = (BN / 8) * 128, lbo_v = (2 * TN / 8) * 128;
    const uint32_t b_half16 = (BN * DK * 4) >> 4;
    const int ksteps = DK / 8;
    const uint64_t db0 = make_desc(smem_u32(stages), lbo_b, 128);
    const uint64_t dv0 = make_desc(smem_u32(stages + col_bytes), lbo_v, 128);
    const uint64_t dvi = make_desc(smem_u32(vi_s), lbo_v, 128);
    const uint32_t vtile16 = v_bytes >> 4;
    const uint32_t stage16 = stage_bytes >> 4;
    const uint32_t kstep_b16 = (2 * lbo_b) >> 4, kstep_v16 = (2 * lbo_v) >> 4;
    const uint32_t xa_hi = tmem + TMXA, xa_lo = tmem + TMXA + (uint32_t)DK;
    const uint32_t kt_hi = tmem + TMKT, kt_lo = tmem + (16u << 16) + TMKT;
    const bool leader = elect_one();
    uint32_t ds = 0, dph = 0, cs = 0, dbuf = 0, keph0 = 0, keph1 = 0;
    uint32_t kph = 0, oph = 0, ktph = 0, ob = 0, ojph = 0;
    uint32_t itc = 0;
    for (int r = 0;; ++r) {
      const int L = item_index(r, b, G);
      if (L >= a.n_items) break;
      const Item it = item_of(a, L);
      if (it.ct1 <= it.ct0) continue;
      const int J = it.ct1 - it.ct0;
      const int first_mirror = 2 * it.rt + 2 - it.ct0;   // tiles jj >= this are mirrored
      mbar_wait(smem_u32(xr_full), itc & 1);
      SYM_T(0, mbar_wait(smem_u32(xa_full), itc & 1));
      ++itc;
      tc_fence_after();
      auto dist = [&]() {   // S = A.B^T into SK[dbuf], A (row image) from TMEM, 3xTF32
        // the previous direct product reading K from this buffer must be complete:
        // the tensor pipe does not order an MMA's TMEM-A reads against a later MMA's D writes
        uint32_t& keph = dbuf ? keph1 : keph0;
        mbar_wait(smem_u32(&k_empty[dbuf]), keph ^ 1);
        keph ^= 1;
        SYM_T(5, mbar_wait(smem_u32(&full[ds]), dph));
        tc_fence_after();
        const uint32_t d_tm = tmem + TMSK(dbuf);
        const uint64_t db = db0 + (uint64_t)(ds * stage16);
        if (leader) {
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint32_t a_p = pass == 0 ? xa_lo : xa_hi;
            const uint64_t b_p = db + (pass == 1 ? b_half16 : 0u);
            for (int ks = 0; ks < ksteps; ++ks)
              mma_ts(d_tm, a_p + ks * 8, b_p + (uint64_t)(ks * kstep_b16), idesc_d, (pass | ks) != 0);
          }
          tc_commit(smem_u32(&s_full[dbuf]));
        }
        __syncwarp();
        if (++ds == (uint32_t)NS) { ds = 0; dph ^= 1; }
        dbuf ^= 1;
      };
      uint32_t kbuf = dbuf;   // SK buffer of tile 0
      dist();
      if (J > 1) dist();
      for (int jj = 0; jj < J; ++jj) {
        SYM_T(1, mbar_wait(smem_u32(k_full), kph));
        tc_fence_after();
        SYM_T(2, mbar_wait(smem_u32(o_empty), oph ^ 1));
        tc_fence_after();
        kph ^= 1;
        oph ^= 1;
        const uint64_t vb = dv0 + (uint64_t)(cs * stage16);
        const uint32_t khi = tmem + TMSK(kbuf), klo = khi + 64;
        if (leader) {
          // direct: O_I[:, 0:32] = Khi.[Vhi | Vlo];  O_I[:, 0:16] += Klo.Vhi
#pragma unroll
          for (int ks = 0; ks < BN / 8; ++ks)
            mma_ts(tmem + TMO, khi + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c32, ks != 0);
#pragma unroll
          for (int ks = 0; ks < BN / 8; ++ks)
            mma_ts(tmem + TMO, klo + ks * 8, vb + (uint64_t)(ks * kstep_v16), idesc_c16, 1);
          tc_commit(smem_u32(&empty[cs]));
          tc_commit(smem_u32(o_full));
          tc_commit(smem_u32(&k_empty[kbuf]));
        }
        __syncwarp();
        if (jj >= first_mirror) {
          // mirror (M = 64, K = 128 rows of I): lanes 0-15 O_J[:, 0:32] = KThi.[VIhi | VIlo],
          // lanes 16-31 O_J[:, 0:16] = KTlo.VIhi (summed by the reader)
          SYM_T(3, mbar_wait(smem_u32(kt_full), ktph));
          tc_fence_after();
          SYM_T(4, mbar_wait(smem_u32(&oj_empty[ob]), ojph ^ 1));
          tc_fence_after();
          ktph ^= 1;
          tacc[7] += 1;
          const uint32_t oj_hi = tmem + TMOJ(ob), oj_lo = tmem + (16u << 16) + TMOJ(ob);
          if (leader) {
#pragma unroll
            for (int ks = 0; ks < BM / 8; ++ks)
              mma_ts(oj_hi, kt_hi + ks * 8, dvi + (uint64_t)((ks >> 3) * vtile16 + (ks & 7) * kstep_v16), idesc_m32,
                     ks != 0);
#pragma unroll
            for (int ks = 0; ks < BM / 8; ++ks)
              mma_ts(oj_lo, kt_lo + ks * 8, dvi + (uint64_t)((ks >> 3) * vtile16 + (ks & 7) * kstep_v16), idesc_m16,
                     ks != 0);
            tc_commit(smem_u32(kt_empty));
            tc_commit(smem_u32(&oj_full[ob]));
          }
          __syncwarp();
          ob ^= 1;
          if (ob == 0) ojph ^= 1;
        }
        if (jj + 2 < J) dist();   // into the buffer direct(jj) just read (in-order pipe)
        kbuf ^= 1;
        if (++cs == (uint32_t)NS) cs = 0;
      }
      if (leader) tc_commit(smem_u32(xr_empty));
      __syncwarp();
    }
  } else if (warp >= EPI_WARP0) {
    // ===================== epilogue (8 warps) =====================
    const int q = warp & 3;                    // TMEM lane quarter
    const int half = (warp - EPI_WARP0) >> 2;  // column half of the 64-col tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int i_loc = q * 32 + lane;
    // consumer view of K^T: rows j = 16q + lane/4 (+8), columns i = 64 half + 8g + 2(lane%4) + c
    const int cj = 16 * q + (lane >> 2), ci = 64 * half + 2 * (lane & 3);
    uint32_t sb = 0, sph = 0, oph = 0, ob = 0, ojph = 0, ktph = 0, kbuf = 0;
    uint32_t itc = 0, kf_tiles = 0;
    float acc[TN];
    int pending = 0;   // half 0: a direct product not yet folded into acc
    int pendj = 0;     // half 1: a mirror product not yet drained
    int64_t pendj_row0 = 0;
    auto flush = [&]() {  // half 0: fold the last direct product into registers
      SYM_T(4, mbar_wait(smem_u32(o_full), oph));
      oph ^= 1;
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + TMO, o);
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(o_empty));
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[c] += __uint_as_float(o[c]) + __uint_as_float(o[c + TN]);
      pending = 0;
    };
    auto flushj = [&]() {  // half 1: last mirror product -> fixed-point sums
      mbar_wait(smem_u32(&oj_full[ob]), ojph);
      tc_fence_after();
      uint32_t o[32];
      tmem_ld32(tmem + lane_base + TMOJ(ob), o);   // lanes 0-15: [hi.Vhi | hi.Vlo], 16-31: [lo.Vhi | -]
      tmem_wait_ld();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&oj_empty[ob]));
      ob ^= 1;
      if (ob == 0) ojph ^= 1;
      float v[TN];
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        const float mine = lane < 16 ? __uint_as_float(o[c]) + __uint_as_float(o[c + TN]) : __uint_as_float(o[c]);
        v[c] = mine + __shfl_xor_sync(0xffffffffu, mine, 16);
      }
      const int64_t row = pendj_row0 + q * 16 + (lane & 15);
      if (row < a.n) {
        const int c0 = lane < 16 ? 0 : TN / 2;
#pragma unroll
        for (int c = 0; c < TN / 2; ++c)
          if (c0 + c < a.t)
            contribute(a, row, c0 + c, lane < 16 ? v[c] : v[c + TN / 2], __ldg(&a.expo[c0 + c]));
      }
      pendj = 0;
    };
    for (int r = 0;; ++r) {
      const int L = item_index(r, b, G);
      if (L >= a.n_items) break;
      const Item it = item_of(a, L);
      if (it.ct1 <= it.ct0) continue;
      const int J = it.ct1 - it.ct0;
      const int first_mirror = 2 * it.rt + 2 - it.ct0;
      const int64_t my_row = (int64_t)it.rt * BM + i_loc;
      if (half == 0) {
        // row image -> TMEM (A operand of the distance product)
        mbar_wait(smem_u32(xr_full), itc & 1);
        const float* xr = reinterpret_cast<const float*>(xr_s);
        for (int part = 0; part < 2; ++part)
          for (int k0 = 0; k0 < DK; k0 += 8) {
            uint32_t w[8];
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
              w[kk] = __float_as_uint(xr[part * BM * DK + canon(i_loc, k0 + kk, BM)]);
            tmem_st8(tmem + lane_base + TMXA + part * DK + k0, w);
          }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(xa_full));
      }
      ++itc;
#pragma unroll
      for (int c = 0; c < TN; ++c) acc[c] = 0.f;
      int64_t e_diag = my_row - ((int64_t)it.ct0 * BN + half * 32);
      for (int jj = 0; jj < J; ++jj, e_diag -= BN) {
        const bool mirror = jj >= first_mirror;
        SYM_T(0, mbar_wait(smem_u32(&s_full[sb]), sph));
        tacc[7] += 1;
        tc_fence_after();
        const uint32_t sk = tmem + lane_base + TMSK(sb);
        uint32_t v[32];
        tmem_ld32(sk + half * 32, v);
        tmem_wait_ld();
        if (!mirror && __any_sync(0xffffffffu, e_diag >= 0 && e_diag < 32)) {
#pragma unroll
          for (int e = 0; e < 32; ++e)
            if (e == e_diag) v[e] = 0u;   // same point on both sides: r2 = 0 exactly
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          float sv = __uint_as_float(v[e]);
          float kap;
          if (FAM == GP_FAMILY_RBF) {
            kap = ex2_approx(sv > 0.f ? 0.f : sv);  // S = -log2(e) r2 / 2
          } else {
            float u = sqrt_approx(sv < 0.f ? 0.f : sv);  // S = 3 r2, u = sqrt(3) r
            float ex = ex2_approx(u * -kLog2e);
            kap = fmaf(u, ex, ex);
          }
          v[e] = __float_as_uint(kap);
        }
        float* ktb = kt32 + kbuf * (64 * KT_LD);
        if (mirror) {
          // kappa^T (fp32) for the transposition: element (j, i) at j*KT_LD + i
#pragma unroll
          for (int e = 0; e < 32; ++e) ktb[(32 * half + e) * KT_LD + i_loc] = __uint_as_float(v[e]);
        }
        uint32_t hi[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          uint32_t h = v[e] & 0xFFFFE000u;
          hi[e] = h;
          v[e] = __float_as_uint(__uint_as_float(v[e]) - __uint_as_float(h));
        }
        // K over S in the same buffer (this warp's S reads completed above)
        tmem_st32(sk + half * 32, hi);
        tmem_st32(sk + 64 + half * 32, v);
        if (half == 0 && pending) SYM_T(1, flush());     // drain O_I before direct(jj) reuses it
        tmem_wait_st();
        tc_fence_before();
        // k_full counts 8 arrivals per tile; a warp running a tile ahead must
        // not arrive before the previous tile's phase completed
        if (kf_tiles > 0) mbar_wait(smem_u32(k_full), (kf_tiles - 1) & 1);
        ++kf_tiles;
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(k_full));
        if (half == 0) pending = 1;
        if (mirror) {
          SYM_T(2, asm volatile("bar.sync 1, 256;" ::: "memory"));   // every producer wrote ktb
          SYM_T(3, mbar_wait(smem_u32(kt_empty), ktph ^ 1));        // previous mirror product done with K^T
          ktph ^= 1;
          tc_fence_after();
          uint32_t w[32];
#pragma unroll
          for (int g = 0; g < 8; ++g)
#pragma unroll
            for (int h8 = 0; h8 < 2; ++h8) {
              const float2 x = *reinterpret_cast<const float2*>(&ktb[(cj + 8 * h8) * KT_LD + ci + 8 * g]);
              w[4 * g + 2 * h8] = __float_as_uint(x.x);
              w[4 * g + 2 * h8 + 1] = __float_as_uint(x.y);
            }
          uint32_t wh[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            wh[e] = w[e] & 0xFFFFE000u;
            w[e] = __float_as_uint(__uint_as_float(w[e]) - __uint_as_float(wh[e]));
          }
          tmem_st16x256_x8(tmem + lane_base + TMKT + 64 * half, wh);
          tmem_st16x256_x8(tmem + lane_base + (16u << 16) + TMKT + 64 * half, w);
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(smem_u32(kt_full));
          kbuf ^= 1;
          if (half == 1 && pendj) SYM_T(5, flushj());     // previous mirror product (other O_J buffer)
          if (half == 1) {
            pendj = 1;
            pendj_row0 = (int64_t)(it.ct0 + jj) * BN;
          }
        }
        sb ^= 1;
        if (sb == 0) sph ^= 1;
      }
      if (half == 0) {
        if (pending) flush();
        if (my_row < a.n) {
#pragma unroll
          for (int c = 0; c < TN; ++c)
            if (c < a.t) contribute(a, my_row, c, acc[c], __ldg(&a.expo[c]));
        }
      } else if (pendj) {
        flushj();
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

// V image for the sym kernel: per 64-column tile a 32-row K-major operand
// [V_hi (rows 0-15) | V_lo (rows 16-31)] in the canonical layout, so one
// N = 32 MMA forms both K_hi.V_hi and K_hi.V_lo
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

// per-column scale 2^E_c with 2^E_c ||V_c||_1 <= 2^61: no partial sum of
// kappa (<= 1) times V can overflow the signed 64-bit accumulator
__global__ void sym_scale_kernel(const float* __restrict__ V, int64_t ldv, int64_t n, int t, int* expo,
                                 double* inv_scale) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double s = 0.0;
  if (c < t)
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += fabs((double)V[i * ldv + c]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if ((int)threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int E = 61;
    double l1 = red[0];
    if (l1 > 0.0 && l1 < INFINITY) {
      int ex;
      frexp(l1, &ex);  // l1 < 2^ex
      E = 61 - ex;
    }
    E = max(-120, min(120, E));
    expo[c] = E;
    inv_scale[c] = ldexp(1.0, -E);
  }
}

// out[i, c] = s2 * acc[c][i] 2^-E_c (+ noise V[i + diag_offset, c]); NaN where a
// non-finite partial was seen (the host names the partition, partition.py:231-236)
__global__ void sym_finalize_kernel(const unsigned long long* __restrict__ acc, int64_t acc_ld,
                                    const int* __restrict__ bad, const double* __restrict__ inv_scale, int64_t n,
                                    int t, float* out, int64_t ldo, double s2, double noise, const float* V,
                                    int64_t ldv, int64_t diag_offset) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * t) return;
  const int64_t i = idx / t;
  const int c = (int)(idx - i * t);
  double r = s2 * ((double)(long long)acc[(int64_t)c * acc_ld + i] * inv_scale[c]);
  if (diag_offset >= 0) r += noise * (double)V[(i + diag_offset) * ldv + c];
  out[i * ldo + c] = bad[i] ? __int_as_float(0x7fc00000) : (float)r;
}

struct Plan {
  int DK, row_tiles, col_tiles, splits, n_items, nstages;
  int64_t acc_ld;
  size_t row_img_bytes, col_img_bytes, v_img_bytes, acc_bytes, bad_bytes, smem;
};

static Plan make_plan(const gp_kv_desc* d) {
  Plan p;
  p.DK = (d->d + 2 + 7) / 8 * 8;
  p.row_tiles = (int)((d->n_rows + BM - 1) / BM);
  p.col_tiles = (int)((d->n_cols + BN - 1) / BN);  // row tile I starts at column tile 2I
  p.splits = std::max(1, std::min(64, (8 * num_sms() + p.row_tiles - 1) / p.row_tiles));
  if (const char* e = getenv("GP_SYM_SPLITS")) p.splits = std::max(1, atoi(e));   // diagnostic
  p.n_items = p.row_tiles * p.splits;
  p.acc_ld = (int64_t)p.row_tiles * BM;
  p.row_img_bytes = (size_t)p.row_tiles * 2 * BM * p.DK * 4;
  p.col_img_bytes = (size_t)p.col_tiles * 2 * BN * p.DK * 4;
  p.v_img_bytes = (size_t)p.col_tiles * V_TILE_BYTES;
  p.acc_bytes = (size_t)TN * p.acc_ld * 8;
  p.bad_bytes = (size_t)p.acc_ld * 4;
  const size_t fixed = 2 * KT32_BYTES + 2u * BM * p.DK * 4 + 2 * V_TILE_BYTES + 512;
  const size_t stage_b = 2u * BN * p.DK * 4 + V_TILE_BYTES;
  const size_t budget = 227 * 1024;
  p.nstages = fixed >= budget ? 0 : (int)std::min<size_t>(4, (budget - fixed) / stage_b);
  p.smem = fixed + p.nstages * stage_b;
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace tcs

// the symmetric kernel applies to the whole square training operator:
// the same point set on both sides, every row and column, t <= 16
bool kv_sym_supported(const gp_kv_desc* d, int t) {
  if (t < 1 || t > tcs::TN) return false;
  if (d->d < 1 || d->d + 2 > 16) return false;   // row image hi|lo must fit 32 TMEM columns
  if (d->Xr != d->Xc || d->ldr != d->ldc || d->n_rows != d->n_cols || d->n_rows < 1) return false;
  if (d->self_offset != 0 || (d->diag_offset != 0 && d->diag_offset >= 0)) return false;
  return tcs::make_plan(d).nstages >= 3;
}

size_t kv_sym_workspace(const gp_kv_desc* d, int t) {
  if (!kv_sym_supported(d, t)) return 0;
  tcs::Plan p = tcs::make_plan(d);
  using tcs::align256;
  return align256(p.row_img_bytes) + align256(p.col_img_bytes) + align256(p.v_img_bytes) +
         align256(p.acc_bytes) + align256(p.bad_bytes) + 256 * sizeof(double) + 2 * 64 * sizeof(double);
}

int kv_sym(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo, void* ws,
           size_t ws_bytes, cudaStream_t st) {
  using namespace tcs;
  Plan p = make_plan(desc);
  size_t need = kv_sym_workspace(desc, t);
  GP_REQUIRE(ws != nullptr && ws_bytes >= need, "gp_kv(symmetric): workspace of %zu bytes required, %zu given",
             need, ws_bytes);
  char* w = static_cast<char*>(ws);
  float* row_img = reinterpret_cast<float*>(w); w += align256(p.row_img_bytes);
  float* col_img = reinterpret_cast<float*>(w); w += align256(p.col_img_bytes);
  float* v_img = reinterpret_cast<float*>(w); w += align256(p.v_img_bytes);
  unsigned long long* acc = reinterpret_cast<unsigned long long*>(w); w += align256(p.acc_bytes);
  int* bad = reinterpret_cast<int*>(w); w += align256(p.bad_bytes);
  double* mean = reinterpret_cast<double*>(w); w += 256 * sizeof(double);
  int* expo = reinterpret_cast<int*>(w); w += 64 * sizeof(double);
  double* inv_scale = reinterpret_cast<double*>(w);
  const int64_t n = desc->n_rows;
  const double c = desc->family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  GP_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)t * p.acc_ld * 8, st));
  GP_CUDA_TRY(cudaMemsetAsync(bad, 0, p.bad_bytes, st));
  sym_scale_kernel<<<TN, 256, 0, st>>>(V, ldv, n, t, expo, inv_scale);
  GP_LAUNCH_CHECK();
  if (int rc = tc::distance_images(desc->Xr, desc->ldr, n, desc->Xc, desc->ldc, n, desc->d, p.DK, BM, BN, c,
                                   mean, row_img, col_img, st))
    return rc;
  {
    int64_t tot = (int64_t)p.col_tiles * BN * TN;
    v_image32_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, ldv, t, n, v_img, p.col_tiles);
    GP_LAUNCH_CHECK();
  }
  Args a;
  a.row_img = row_img; a.col_img = col_img; a.v_img = v_img; a.DK = p.DK;
  a.n = n; a.row_tiles = p.row_tiles; a.col_tiles = p.col_tiles; a.splits = p.splits; a.n_items = p.n_items;
  a.nstages = p.nstages; a.lookahead = 1; a.t = t;
  a.expo = expo; a.acc = acc; a.acc_ld = p.acc_ld; a.bad = bad;
  int grid = std::min(p.n_items, num_sms());
  auto kern = desc->family == GP_FAMILY_RBF ? kv_sym_kernel<GP_FAMILY_RBF> : kv_sym_kernel<GP_FAMILY_MATERN32>;
  GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  a.prof = nullptr;
  const char* am = getenv("GP_SYM_ATOM");
  a.atom_mode = am ? atoi(am) : 0;
  const char* pe = getenv("GP_SYM_PROF");
  if (pe && *pe == '1') GP_CUDA_TRY(cudaMalloc(&a.prof, (size_t)grid * (NTHREADS / 32) * 8 * sizeof(long long)));
  kern<<<grid, NTHREADS, p.smem, st>>>(a);
  GP_LAUNCH_CHECK();
  if (a.prof) {   // diagnostic only: per-role average cycles per tile, CTA-averaged
    std::vector<long long> h((size_t)grid * (NTHREADS / 32) * 8);
    GP_CUDA_TRY(cudaStreamSynchronize(st));
    GP_CUDA_TRY(cudaMemcpy(h.data(), a.prof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(a.prof);
    const char* names[8] = {"wait0", "wait1", "wait2", "wait3", "wait4", "wait5", "total", "tiles"};
    for (int w : {1, 4, 5, 6, 8, 9}) {
      double s[8] = {0};
      for (int c = 0; c < grid; ++c)
        for (int k = 0; k < 8; ++k) s[k] += (double)h[((size_t)c * (NTHREADS / 32) + w) * 8 + k];
      fprintf(stderr, "[sym prof] warp %d:", w);
      for (int k = 0; k < 8; ++k) fprintf(stderr, " %s=%.0f", names[k], k == 7 ? s[7] / grid : s[k] / std::max(1.0, s[7]));
      fprintf(stderr, "\n");
    }
  }
  int64_t tot = n * t;
  sym_finalize_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(acc, p.acc_ld, bad, inv_scale, n, t, out, ldo,
                                                                     desc->outputscale, desc->noise, V, ldv,
                                                                     desc->diag_offset);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

}  // namespace gp
