// Symmetric tcgen05 K·V kernel for the square training operator (sm_100a).
//
// out = s2 * kappa(X, X) V (+ noise V), evaluating every unordered pair of
// points ONCE. K is symmetric, so the tile K_IJ (row tile I, column tile J,
// 128 points each, I < J) serves both
//     out_I += K_IJ   V_J      (direct:  A = K   from TMEM,        M = 128 rows i)
//     out_J += K_IJ^T V_I      (mirror:  A = K^T from SMEM, MN-major, M = 128 rows j)
// which halves the transcendental (SFU) work that bounds the kernel at CG
// width. Diagonal tiles (I = J) are evaluated in full and
// used once (direct only).
//
// The transpose costs nothing extra: each kappa lane (point i) writes its 8
// consecutive K_ij (fp16 pairs along j) as one 16-byte store, which is
// exactly a row of a core matrix of the MN-major (M = j contiguous) canonical
// layout the tensor core reads K^T from. The same fp16 values go to TMEM in
// place over S for the direct product.
//
// Per tile, on the tensor core (one elected thread issues):
//   S = A_I . B_J^T                 3xTF32, A (row image) in TMEM, N = 128
//   O_I[r] += K1.V1 + K2.V1 + K1.V2 (kind::f16, A = K from TMEM, N = 16 each)
//   O_J[c] += K1^T.[V1|V2] + K2^T.V1 (kind::f16, A = K^T from SMEM)
// with the fp16 split K = K1 + K2 (K1 = K truncated to 11 bits) and V scaled
// per column by 2^s into fp16 range (V = V1 + V2): as accurate as 3xTF32.
//
// Work items are 4 x 4 blocks of tiles (block pairs P <= Q, row-major
// upper-triangular order, round-robin over persistent CTAs; with item
// sharding, rank `part` of `nparts` takes the items L = part (mod nparts)).
// O_I (per item row) and O_J[0..3] accumulate in TMEM over 4 tiles of K,
// short enough for the tensor core's fp32 accumulation, and every such
// per-item partial leaves the SM as 64-bit FIXED POINT (per-column scale 2^E_c
// chosen from ||V_c||_1 so no partial can overflow), added into the global
// sums with TMA bulk reduce-adds. Integer addition is associative and the
// partials depend only on the item, so the result is bitwise identical run to
// run, for any CTA schedule and for any split of the items across GPUs, like
// the reference's partition-count independence (test_partition.py:92-102).
//
// Warp roles: 0 TMA producer (column tiles), 1 MMA issuer (also copies each
// row image SMEM -> TMEM with tcgen05.cp), 2-5 drain (warp 2 allocates TMEM),
// 6-21 kappa (S -> K, 32 rows x 32 columns each), 22 TMA producer (row tiles).
//
// Reference semantics: kernels.py:225-244 (kappa), :293-316 (rows of K̂ incl.
// the sigma^2 diagonal), partition.py:224-241 (row-block products).
#include "tc_common.cuh"

#include <cooperative_groups.h>
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

namespace gp {
namespace tcs {

using namespace gp::tc;

constexpr int BT = 128;   // points per tile, both sides (UMMA M of both products)
constexpr int TN = 16;    // right-hand sides
constexpr int RB = 4;     // tiles per block side: an item is a 4 x 4 block of tiles
constexpr int DRAIN_WARP0 = 2, KAPPA_WARP0 = 6, NUM_KAPPA_WARPS = 16;
constexpr int ROW_WARP = KAPPA_WARP0 + NUM_KAPPA_WARPS;   // row image + V_I loader
constexpr int NTHREADS = 32 * (ROW_WARP + 1);
constexpr uint32_t KS_HALF = BT * BT * 2;            // K1 (or K2) of one tile, fp16 MN-major
constexpr uint32_t KS_BYTES = 2 * KS_HALF;
constexpr uint32_t V_TILE_BYTES = 2u * TN * BT * 2u;  // [V1 | V2] of one tile, 32 x 128 fp16
constexpr uint32_t STAGE_BYTES = TN * BT * 8u;       // fixed-point sums of one 128-row block
// Items are dealt to CTAs in chunks of `chunk` consecutive items (mostly
// the same row block P); the O_I partials of a chunk's items are summed in
// SMEM (fp32) and leave the SM once per (chunk, row block). The chunk size is
// a function of the item count alone (item_chunk) and the grouping a
// function of the item index, so the fixed-point result does not depend on
// the grid size or on how the chunks are split across devices. Longer chunks
// carry O_I across more items (fewer flushes; n = 10^6: 4 -> 16 items is
// 360 -> 354 ms, 16 -> 32 is 339.4 -> 337.8 ms, 64 no better) but leave
// fewer chunks than CTAs at small n.
static int item_chunk(int n_items) {
  for (int c = 32; c > 4; c >>= 1)
    if (n_items >= 4 * 148 * c) return c;   // at least 4 chunks per SM of a full B200
  return 4;
}
constexpr uint32_t ACCI_BYTES = RB * BT * TN * 4u;
constexpr uint32_t BAR_BYTES = 1024;

// TMEM columns (512): S/K buffers 2 x 128 | O_I 2 x 32 (by row) | O_J 4 x 32 |
// row image 2 x 2 DK (by row, DK <= 16)
// S (fp32) lands in [128b, 128b + 128); the kappa warps overwrite it in place
// with K1 | K2 (fp16 pairs along j): kstep ks (16 points) at 16 ks (K1), 16 ks + 8 (K2)
__device__ __forceinline__ uint32_t TSK(uint32_t b) { return 128u * b; }
__device__ __forceinline__ uint32_t TOI(uint32_t rb) { return 256u + 32u * rb; }
__device__ __forceinline__ uint32_t TOJ(int c) { return 320u + 32u * (uint32_t)c; }
__device__ __forceinline__ uint32_t TXA(uint32_t xb) { return 448u + 32u * xb; }

struct Args {
  const float* row_img;   // [tiles][2][BT*DK] tf32 hi|lo (A of the distance product)
  const float* col_img;   // [tiles][2][BT*DK]
  const __half* v_img;    // [tiles][32 x 128] fp16 [V1 | V2]
  int DK;
  int64_t n;
  int tiles, nblocks, n_items, nsc, nsv, t;
  int part, nparts;                 // item sharding: this launch takes items L = part (mod nparts)
  int chunk;                        // items per chunk (item_chunk)
  const int* expo;                  // [TN] partials (in scaled units) summed as round(v 2^expo_c)
  unsigned long long* acc;          // [tiles][t][BT] fixed-point sums (row-block major: a
                                    // contiguous row range owns a contiguous slice)
  int64_t acc_ld;
  int* bad;                         // [acc_ld] non-finite partial seen for the row
  long long* prof;                  // optional per-warp phase cycle counters (GP_SYM_PROF=1)
};

// per-role wait counters for diagnosis: build with -DGP_SYM_PROF_BUILD=1 and
// run with GP_SYM_PROF=1 (compiled out by default: the counters cost registers)
#ifndef GP_SYM_PROF_BUILD
#define GP_SYM_PROF_BUILD 0
#endif
#if GP_SYM_PROF_BUILD
#define SYM_T(slot, ...)                                  \
  do {                                                    \
    const long long _t0 = a.prof ? clock64() : 0;         \
    __VA_ARGS__;                                          \
    if (a.prof) tacc[slot] += clock64() - _t0;            \
  } while (0)
#define SYM_COUNT() (tacc[7] += 1)
#else
#define SYM_T(slot, ...) do { __VA_ARGS__; } while (0)
#define SYM_COUNT() ((void)0)
#endif

// TMA bulk reduce-add of a contiguous fixed-point block into the global sums
__device__ __forceinline__ void bulk_red_u64(void* gdst, uint32_t ssrc, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(gdst), "r"(ssrc),
               "r"(bytes)
               : "memory");
}
// SMEM (canonical K-major, no swizzle) -> TMEM, 128 lanes x 8 fp32 columns;
// ordered with the tcgen05.mma of the same thread (one pipeline, issue order)
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}
__device__ __forceinline__ void drain_bar() { asm volatile("bar.sync 2, 128;" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z), "r"(w)
               : "memory");
}

// mbarrier waits with a suspend-time hint (ns): the waiting thread sleeps
// until the phase completes (or the hint expires) instead of re-polling,
// which keeps SYNCS traffic out of the MIO queue the kappa warps' MUFU work
// shares. P: producers and drain (off the critical path), C: MMA and kappa.
#ifndef GP_SYM_HINT_P
#define GP_SYM_HINT_P 1000000
#endif
#ifndef GP_SYM_HINT_C
#define GP_SYM_HINT_C 0
#endif
__device__ __forceinline__ void mbar_wait_hint(uint32_t bar, uint32_t parity, uint32_t ns) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity), "r"(ns)
      : "memory");
}
__device__ __forceinline__ void wait_p(uint32_t bar, uint32_t parity) {
  if (GP_SYM_HINT_P) mbar_wait_hint(bar, parity, GP_SYM_HINT_P);
  else mbar_wait(bar, parity);
}
__device__ __forceinline__ void wait_c(uint32_t bar, uint32_t parity) {
  if (GP_SYM_HINT_C) mbar_wait_hint(bar, parity, GP_SYM_HINT_C);
  else mbar_wait(bar, parity);
}

// row-major upper triangle of an m x m block: local index l -> (p, q), p <= q,
// start(p) = p m - p (p - 1) / 2 <= l < start(p + 1)
__device__ __forceinline__ void tri_pair(int l, int m, int& p, int& q) {
  const double b2 = 2.0 * m + 1.0;
  int x = (int)floor((b2 - sqrt(b2 * b2 - 8.0 * (double)l)) * 0.5);
  x = max(0, min(m - 1, x));
  auto start = [&](int y) { return (long long)y * m - (long long)y * (y - 1) / 2; };
  while (x > 0 && start(x) > l) --x;
  while (x + 1 < m && start(x + 1) <= l) ++x;
  p = x;
  q = x + (int)(l - start(x));
}

// Item order: block pairs are grouped into bands of SB = 128 row blocks (SB x SB
// super-items (U, V), U <= V, row-major; inside one, row-major pairs). The
// ~150 chunks in flight then touch two bands of the fixed-point sums and
// one band of column / V images (a few MB, L2-resident) instead of sweeping
// all n columns per row block (which streamed the 88 MB sums and the
// 190 MB images through DRAM: 202 GB per n = 10^6 launch). With NB <= SB
// this is the plain row-major triangle.
#ifndef GP_SYM_SB
#define GP_SYM_SB 128
#endif
constexpr int SB = GP_SYM_SB;
__device__ __forceinline__ void pair_of(int L, int NB, int& P, int& Q) {
  const int nb = (NB + SB - 1) / SB;
  auto rows = [&](int b) { return min(SB, NB - b * SB); };
  long long l = L;
  int U = 0;
  for (; U < nb - 1; ++U) {
    const long long r = rows(U);
    const long long row_items = r * (r + 1) / 2 + r * (long long)(NB - (U + 1) * SB);
    if (l < row_items) break;
    l -= row_items;
  }
  const int ru = rows(U);
  const long long tri = (long long)ru * (ru + 1) / 2;
  if (l < tri) {
    int p, q;
    tri_pair((int)l, ru, p, q);
    P = U * SB + p;
    Q = U * SB + q;
    return;
  }
  l -= tri;
  // off-diagonal super-items (U, V > U): ru x rows(V), all full but the last
  const long long full = (long long)ru * SB;
  int V = U + 1 + (int)(l / full);
  long long lv = l - (long long)(V - U - 1) * full;
  if (V >= nb) { V = nb - 1; lv = l - (long long)(V - U - 1) * full; }
  const int rv = rows(V);
  P = U * SB + (int)(lv / rv);
  Q = V * SB + (int)(lv % rv);
}

// (P, Q) of item L + 1 from that of item L (the order of pair_of)
__device__ __forceinline__ void step_pair(int NB, int& P, int& Q) {
  const int U = P / SB, V = Q / SB;
  const int q_end = min(NB, (V + 1) * SB);
  if (Q + 1 < q_end) { ++Q; return; }
  const int p_end = min(NB, (U + 1) * SB);
  if (P + 1 < p_end) {   // next row of the super-item (on the diagonal one it starts at Q = P)
    ++P;
    Q = U == V ? P : V * SB;
    return;
  }
  if (q_end < NB) {      // next super-item of the band row
    P = U * SB;
    Q = q_end;
    return;
  }
  P = Q = (U + 1) * SB;  // next band row, its diagonal super-item
}

// The tile sequence of one CTA (every role walks the same sequence): chunks
// k = part + nparts (blockIdx.x + j gridDim.x) of `chunk` items each; within an item, rows r then columns c, with
// c >= r on a diagonal item (P = Q), whose tile (r, r) is a diagonal tile.
struct TileSeq {
  int NB, tiles, n_items, G, CH;   // G = chunk stride (grid x parts), CH = items per chunk
  int k, i;                    // chunk, item within the chunk
  int L, P, Q, r, c, rows_in, cols_in;
  bool ok;
  __device__ void set_item() {
    pair_of(L, NB, P, Q);
    set_pair();
  }
  __device__ void set_pair() {
    rows_in = min(RB, tiles - RB * P);
    cols_in = min(RB, tiles - RB * Q);
    r = 0;
    c = c0();
  }
  __device__ void begin(const Args& a) {
    NB = a.nblocks; tiles = a.tiles; n_items = a.n_items; G = gridDim.x * a.nparts; CH = a.chunk;
    k = a.part + a.nparts * blockIdx.x;
    i = 0;
    L = CH * k;
    ok = L < n_items;
    if (ok) set_item();
  }
  // next item of this CTA's sequence (chunk by chunk)
  __device__ void next_item() {
    if (++i < CH && CH * k + i < n_items) {
      ++L;
      step_pair(NB, P, Q);   // the next item of the chunk: O(1), no pair_of
      set_pair();
      return;
    }
    k += G;
    i = 0;
    L = CH * k;
    ok = L < n_items;
    if (ok) set_item();
  }
  __device__ int c0() const { return P == Q ? r : 0; }
  __device__ void next() {
    if (++c < cols_in) return;
    if (++r < rows_in) { c = c0(); return; }
    next_item();
  }
  __device__ bool first_in_row() const { return c == c0(); }
  __device__ bool last_in_row() const { return c == cols_in - 1; }
  __device__ bool first_in_item() const { return r == 0 && c == c0(); }
  __device__ bool last_in_item() const { return last_in_row() && r == rows_in - 1; }
  __device__ bool mirror() const { return !(P == Q && c == r); }
  __device__ int I() const { return RB * P + r; }
  __device__ int J() const { return RB * Q + c; }
};

// DKT: the augmented-point width (8 or 16) as a compile-time constant, so the
// MMA thread's distance products and row-image copies unroll fully
template <int FAM, int DKT>
__global__ void __launch_bounds__(NTHREADS, 1) kv_sym_kernel(const Args a) {
  extern __shared__ __align__(1024) uint8_t smem[];
  constexpr int DK = DKT;
  const uint32_t img_bytes = 2u * BT * DK * 4u;       // row or column image of one tile (hi | lo)
  const int NSC = a.nsc, NSV = a.nsv;
  uint8_t* ks = smem;                                  // K1 | K2 of the current tile (mirror A operand)
  uint8_t* xr_s = ks + KS_BYTES;                       // row image (TMA, copied into TMEM)
  uint8_t* vi_s = xr_s + img_bytes;                    // V_I, double buffered by row
  uint8_t* cring = vi_s + 2 * V_TILE_BYTES;            // [NSC] column images
  uint8_t* vring = cring + NSC * img_bytes;            // [NSV] V_J images
  float* acci = reinterpret_cast<float*>(vring + NSV * V_TILE_BYTES);   // [RB][BT][TN], 16-B chunks swizzled
  unsigned long long* stage = reinterpret_cast<unsigned long long*>(reinterpret_cast<uint8_t*>(acci) + ACCI_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(stage) + 2 * STAGE_BYTES);
  uint64_t* cfull = bars;               // [NSC] column image landed           TMA -> MMA
  uint64_t* cempty = cfull + NSC;       // [NSC] distance product done         MMA -> TMA
  uint64_t* vfull = cempty + NSC;       // [NSV] V_J landed                    TMA -> MMA
  uint64_t* vempty = vfull + NSV;       // [NSV] direct product done           MMA -> TMA
  uint64_t* vi_full = vempty + NSV;     // [2]   V_I landed                    TMA -> MMA
  uint64_t* vi_empty = vi_full + 2;     // [2]   mirrors of the row done       MMA -> TMA
  uint64_t* s_full = vi_empty + 2;      // [2]   S in TMEM buffer b            MMA -> kappa
  uint64_t* k_full = s_full + 2;        // [2]   K written (TMEM + SMEM)       kappa -> MMA
  uint64_t* sk_empty = k_full + 2;      // [2]   products done with buffer b   MMA -> MMA
  uint64_t* ks_empty = sk_empty + 2;    //       mirror products done with the SMEM K  MMA -> kappa
  uint64_t* xr_full = ks_empty + 1;     //       row image landed              TMA -> MMA
  uint64_t* xr_empty = xr_full + 1;     //       row image copied into TMEM    MMA -> TMA
  uint64_t* oi_full = xr_empty + 1;     // [2]   row's direct products done    MMA -> drain
  uint64_t* oi_empty = oi_full + 2;     // [2]   O_I buffer read               drain -> MMA
  uint64_t* oj_full = oi_empty + 2;     //       item's mirror products done   MMA -> drain
  uint64_t* oj_empty = oj_full + 1;     // [RB]  O_J[c] read                   drain -> MMA
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(oj_empty + RB);
  float* scale_s = reinterpret_cast<float*>(tmem_slot + 4);   // [TN] fixed-point scales 2^expo_c

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int x = threadIdx.x; x < (int)(ACCI_BYTES / 4); x += blockDim.x) acci[x] = 0.f;
  if (threadIdx.x < TN) scale_s[threadIdx.x] = ldexpf(1.0f, a.expo[threadIdx.x]);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSC; ++s) {
      mbar_init(smem_u32(&cfull[s]), 1);
      mbar_init(smem_u32(&cempty[s]), 1);
    }
    for (int s = 0; s < NSV; ++s) {
      mbar_init(smem_u32(&vfull[s]), 1);
      mbar_init(smem_u32(&vempty[s]), 1);
    }
    for (int q = 0; q < 2; ++q) {
      mbar_init(smem_u32(&vi_full[q]), 1);
      mbar_init(smem_u32(&vi_empty[q]), 1);
      mbar_init(smem_u32(&s_full[q]), 1);
      mbar_init(smem_u32(&k_full[q]), NUM_KAPPA_WARPS);
      mbar_init(smem_u32(&sk_empty[q]), 1);
    }
    mbar_init(smem_u32(ks_empty), 1);
    mbar_init(smem_u32(xr_full), 1);
    mbar_init(smem_u32(xr_empty), 1);
    for (int q = 0; q < 2; ++q) {
      mbar_init(smem_u32(&oi_full[q]), 1);
      mbar_init(smem_u32(&oi_empty[q]), 4);
    }
    mbar_init(smem_u32(oj_full), 1);
    for (int c = 0; c < RB; ++c) mbar_init(smem_u32(&oj_empty[c]), 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == DRAIN_WARP0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();

  if (warp == 0) {
    // ===================== TMA producer: column tiles =====================
    if (lane == 0) {
      TileSeq it;
      it.begin(a);
      uint32_t cs = 0, cph = 0, vs = 0, vph = 0;
      const uint32_t img_f = img_bytes / 4, vt_h = V_TILE_BYTES / 2;
      while (it.ok) {
        const int J = it.J();
        // column slot cs holds tile Tn with Tn & 1 == cs (two slots), and the
        // distance product that reads it commits s_full[cs]: wait on that
        wait_p(smem_u32(NSC == 2 ? &s_full[cs] : &cempty[cs]), cph ^ 1);
        mbar_expect_tx(smem_u32(&cfull[cs]), img_bytes);
        bulk_g2s(smem_u32(cring + cs * img_bytes), a.col_img + (int64_t)J * img_f, img_bytes, smem_u32(&cfull[cs]));
        if (++cs == (uint32_t)NSC) { cs = 0; cph ^= 1; }
        // with a 2-deep V ring, slot vs is freed by the direct product of the
        // tile that used S/K buffer vs: wait on that release, no extra commit
        wait_p(smem_u32(NSV == 2 ? &sk_empty[vs] : &vempty[vs]), vph ^ 1);
        mbar_expect_tx(smem_u32(&vfull[vs]), V_TILE_BYTES);
        bulk_g2s(smem_u32(vring + vs * V_TILE_BYTES), a.v_img + (int64_t)J * vt_h, V_TILE_BYTES,
                 smem_u32(&vfull[vs]));
        if (++vs == (uint32_t)NSV) { vs = 0; vph ^= 1; }
        it.next();
      }
    }
  } else if (warp == ROW_WARP) {
    // ===================== TMA producer: row tiles =====================
    // a separate thread, so the next row image is fetched as soon as the
    // previous one is in TMEM instead of behind the column ring
    if (lane == 0) {
      TileSeq it;
      it.begin(a);
      uint32_t R = 0;
      const uint32_t img_f = img_bytes / 4, vt_h = V_TILE_BYTES / 2;
      while (it.ok) {
        const int I = it.I();
        if (R >= 1) wait_p(smem_u32(xr_empty), (R - 1) & 1);
        mbar_expect_tx(smem_u32(xr_full), img_bytes);
        bulk_g2s(smem_u32(xr_s), a.row_img + (int64_t)I * img_f, img_bytes, smem_u32(xr_full));
        const uint32_t vb = R & 1, u = R >> 1;
        if (u >= 1) wait_p(smem_u32(&vi_empty[vb]), (u - 1) & 1);
        mbar_expect_tx(smem_u32(&vi_full[vb]), V_TILE_BYTES);
        bulk_g2s(smem_u32(vi_s + vb * V_TILE_BYTES), a.v_img + (int64_t)I * vt_h, V_TILE_BYTES,
                 smem_u32(&vi_full[vb]));
        ++R;
        // to the first tile of the next row
        const int r0 = it.r;
        const int L0 = it.L;
        while (it.ok && it.r == r0 && it.L == L0) it.next();
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    // per tile T: dist(T+1) (into the other S/K buffer, once the direct
    // product of T-1 is done with it), then direct(T) and mirror(T) once the
    // kappa warps have written K(T)
    const uint32_t idesc_d = make_idesc(BT, BT);
    const uint32_t idesc_n16 = idesc_f16(BT, TN), idesc_n32 = idesc_f16(BT, 2 * TN);
    const uint32_t idesc_m32 = idesc_f16(BT, 2 * TN) | IDESC_A_MN_MAJOR;
    const uint32_t idesc_m16 = idesc_f16(BT, TN) | IDESC_A_MN_MAJOR;
    const uint32_t lbo_b = (BT / 8) * 128, lbo_v = (2 * TN / 8) * 128;
    const uint32_t half16 = (BT * DK * 4) >> 4;
    constexpr int ksteps = DK / 8;
    const uint64_t dc0 = make_desc(smem_u32(cring), lbo_b, 128);
    const uint64_t dv0 = make_desc(smem_u32(vring), lbo_v, 128);
    const uint64_t dvi0 = make_desc(smem_u32(vi_s), lbo_v, 128);
    // K^T, MN-major: core matrix = 8 points i x 8 points j (16 B rows along j);
    // LBO = 128 B between i-groups (the K direction), SBO = 2 KB between j-groups
    const uint64_t dks = make_desc(smem_u32(ks), 128, 2048);
    const uint64_t dxr0 = make_desc(smem_u32(xr_s), lbo_b, 128);   // row image, K-major like the column image
    const uint32_t img16 = img_bytes >> 4, vt16 = V_TILE_BYTES >> 4;
    const uint32_t kstep_b16 = (2 * lbo_b) >> 4, kstep_v16 = (2 * lbo_v) >> 4;
    const uint32_t ks2_16 = KS_HALF >> 4;          // K2 half of the SMEM K
    const bool leader = elect_one();
    uint32_t cs = 0, cph = 0, vs = 0, vph = 0, R = 0, K = 0, T = 0;
    int rowc = -1;
    TileSeq it;
    it.begin(a);
    auto dist = [&](const TileSeq& tt, uint32_t Tn) {
      const uint32_t b = Tn & 1;
      if (Tn >= 2) SYM_T(0, wait_c(smem_u32(&sk_empty[b]), ((Tn >> 1) - 1) & 1));
      if (tt.first_in_row()) {
        // new row: row image SMEM -> TMEM buffer R & 1 (tcgen05.cp, in the
        // tensor pipe ahead of this row's distance products)
        SYM_T(1, wait_c(smem_u32(xr_full), R & 1));
        tc_fence_after();
        if (leader) {
          for (int part = 0; part < 2; ++part)
#pragma unroll
            for (int kb = 0; kb < ksteps; ++kb)
              tmem_cp_128x256b(tmem + TXA(R & 1) + part * DK + 8 * kb,
                               dxr0 + (uint64_t)((part * BT * DK * 4 + kb * 2 * lbo_b) >> 4));
          tc_commit(smem_u32(xr_empty));
        }
        __syncwarp();
        ++R;
      }
      const uint32_t xb = (R - 1) & 1;
      SYM_T(2, wait_c(smem_u32(&cfull[cs]), cph));
      tc_fence_after();
      if (leader) {
        const uint32_t d_tm = tmem + TSK(b);
        const uint64_t db = dc0 + (uint64_t)(cs * img16);
#pragma unroll
        for (int pass = 0; pass < 3; ++pass) {
          const uint32_t a_t = tmem + TXA(xb) + (pass == 0 ? (uint32_t)DK : 0u);
          const uint64_t b_p = db + (pass == 1 ? half16 : 0u);
#pragma unroll
          for (int k = 0; k < ksteps; ++k)
            mma_ts(d_tm, a_t + k * 8, b_p + (uint64_t)(k * kstep_b16), idesc_d, (pass | k) != 0);
        }
        tc_commit(smem_u32(&s_full[b]));
        if (NSC != 2) tc_commit(smem_u32(&cempty[cs]));   // NSC = 2: s_full[b] above releases the slot
      }
      __syncwarp();
      if (++cs == (uint32_t)NSC) { cs = 0; cph ^= 1; }
    };
    if (it.ok) dist(it, 0);
    while (it.ok) {
      TileSeq nx = it;
      nx.next();
      if (nx.ok) dist(nx, T + 1);
      const uint32_t b = T & 1;
      if (it.first_in_row()) {
        ++rowc;
        // O_I buffer rowc & 1 was last used by row rowc - 2
        if (rowc >= 2) SYM_T(3, wait_c(smem_u32(&oi_empty[rowc & 1]), ((rowc >> 1) - 1) & 1));
      }
      if (K >= 1) {
        // O_J[c] of the previous item must be read before tile (0, c) of this
        // one; columns this item does not have are waited for at its end, so
        // every oj_empty phase is consumed once per item
        if (it.r == 0) SYM_T(3, wait_c(smem_u32(&oj_empty[it.c]), (K - 1) & 1));
        if (it.last_in_item())
          for (int cc = it.cols_in; cc < RB; ++cc) wait_c(smem_u32(&oj_empty[cc]), (K - 1) & 1);
      }
      SYM_T(4, wait_c(smem_u32(&k_full[b]), (T >> 1) & 1));
      SYM_COUNT();
      SYM_T(5, wait_c(smem_u32(&vfull[vs]), vph));
      const bool mir = it.mirror();
      // V_I is loaded for every row; a row of a diagonal item whose only tile
      // is the diagonal one has no mirror product, but its load must still be
      // awaited before vi_empty is committed (no bulk copy may be in flight
      // when the barrier is re-armed or the CTA exits)
      if (mir || (it.first_in_row() && it.last_in_row()))
        SYM_T(5, wait_c(smem_u32(&vi_full[rowc & 1]), (rowc >> 1) & 1));
      tc_fence_after();
      if (leader) {
        // direct first, then release the S/K buffer: the mirror reads only
        // SMEM, so it keeps the tensor pipe busy while this thread wakes up on
        // sk_empty and issues the distance product of tile T + 2 into it (with
        // the release after both products the pipe drained every tile)
        const uint32_t oi = tmem + TOI(rowc & 1), sk = tmem + TSK(b);
        const uint64_t vb = dv0 + (uint64_t)(vs * vt16);
        const uint32_t fresh = it.first_in_row() ? 1u : 0u;
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)   // O_I (+)= K1 . [V1 | V2]
          mma16_ts(oi, sk + 16 * k, vb + (uint64_t)(k * kstep_v16), idesc_n32, !(fresh && k == 0));
#pragma unroll
        for (int k = 0; k < BT / 16; ++k)   // O_I[:, 0:16] += K2 . V1
          mma16_ts(oi, sk + 16 * k + 8, vb + (uint64_t)(k * kstep_v16), idesc_n16, 1);
        if (NSV != 2) tc_commit(smem_u32(&vempty[vs]));   // NSV = 2: sk_empty[b] below releases it
        tc_commit(smem_u32(&sk_empty[b]));
        if (it.last_in_row()) tc_commit(smem_u32(&oi_full[rowc & 1]));
        if (mir) {
          const uint32_t oj = tmem + TOJ(it.c);
          const uint64_t vib = dvi0 + (uint64_t)((rowc & 1) * vt16);
          const uint32_t jfresh = it.r == 0 ? 1u : 0u;
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)   // O_J (+)= K1^T . [V1 | V2]
            mma16_ss(oj, dks + (uint64_t)(16 * k), vib + (uint64_t)(k * kstep_v16), idesc_m32, !(jfresh && k == 0));
#pragma unroll
          for (int k = 0; k < BT / 16; ++k)   // O_J[:, 0:16] += K2^T . V1
            mma16_ss(oj, dks + (uint64_t)(ks2_16 + 16 * k), vib + (uint64_t)(k * kstep_v16), idesc_m16, 1);
          tc_commit(smem_u32(ks_empty));   // one phase per mirror tile: every phase has a waiter
        }
        if (it.last_in_row()) tc_commit(smem_u32(&vi_empty[rowc & 1]));
        if (it.last_in_item()) tc_commit(smem_u32(oj_full));
      }
      __syncwarp();
      if (++vs == (uint32_t)NSV) { vs = 0; vph ^= 1; }
      if (it.last_in_item()) ++K;
      it = nx;
      ++T;
    }
  } else if (warp >= KAPPA_WARP0 && warp < ROW_WARP) {
    // ===================== kappa warps: S -> K =====================
    const int e = warp - KAPPA_WARP0;
    const int q = warp & 3;                        // TMEM lane quarter
    const int ch = e >> 2;                         // 32-column chunk of the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int i_loc = q * 32 + lane;
    const uint32_t ks_row = smem_u32(ks) + 16u * (uint32_t)i_loc + (uint32_t)(4 * ch) * 2048u;
    TileSeq it;
    it.begin(a);
    uint32_t T = 0, Mt = 0;   // tiles, mirror tiles
    while (it.ok) {
      const uint32_t b = T & 1;
      SYM_T(0, wait_c(smem_u32(&s_full[b]), (T >> 1) & 1));
      SYM_COUNT();
      tc_fence_after();
      const uint32_t sk = tmem + lane_base + TSK(b) + 32u * ch;
      uint32_t v[32];
      SYM_T(1, tmem_ld32(sk, v); tmem_wait_ld());
      const bool mir = it.mirror();
      if (!mir) {
        // diagonal tile: the same point on both sides has r2 = 0 exactly
        const int e_diag = i_loc - 32 * ch;
        if (__any_sync(0xffffffffu, e_diag >= 0 && e_diag < 32)) {
#pragma unroll
          for (int k = 0; k < 32; ++k)
            if (k == e_diag) v[k] = 0u;
        }
      }
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const float sv = __uint_as_float(v[k]);
        // x 2^12 for the fp16 split (clamps written as selects so NaN
        // inputs propagate); the fixed-point exponents divide it out
        v[k] = __float_as_uint(kappa_split_scaled<FAM>(sv));
      }
      uint32_t p1[16], p2[16];
#pragma unroll
      for (int k = 0; k < 16; ++k) split_pair(__uint_as_float(v[2 * k]), __uint_as_float(v[2 * k + 1]), p1[k], p2[k]);
      // K in place over this warp's own S columns (kstep 2ch at [32ch, +16),
      // 2ch+1 at [32ch+16, +16)) and the K^T rows for the mirror (8
      // consecutive j of point i = one 16-byte core-matrix row), first half
      // of the columns first: its stores go out while the second half's
      // split is still in flight, which shortens the tile's tail (n = 10^6:
      // 342.0 -> 339.5-340.5 ms; per-8-column stores with the K^T wait
      // before the first were slower, 385 ms: profiles/r02_kv_sym.md)
      tmem_st8(sk, p1);
      tmem_st8(sk + 8, p2);
      if (mir) {
        // the previous mirror tile's products have read the SMEM K
        if (Mt >= 1) SYM_T(2, wait_c(smem_u32(ks_empty), (Mt - 1) & 1));
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          sts128(ks_row + m * 2048u, p1[4 * m], p1[4 * m + 1], p1[4 * m + 2], p1[4 * m + 3]);
          sts128(ks_row + KS_HALF + m * 2048u, p2[4 * m], p2[4 * m + 1], p2[4 * m + 2], p2[4 * m + 3]);
        }
      }
      tmem_st8(sk + 16, p1 + 8);
      tmem_st8(sk + 24, p2 + 8);
      if (mir) {
        ++Mt;
#pragma unroll
        for (int m = 2; m < 4; ++m) {
          sts128(ks_row + m * 2048u, p1[4 * m], p1[4 * m + 1], p1[4 * m + 2], p1[4 * m + 3]);
          sts128(ks_row + KS_HALF + m * 2048u, p2[4 * m], p2[4 * m + 1], p2[4 * m + 2], p2[4 * m + 3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      SYM_T(3, tmem_wait_st());
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&k_full[b]));
      it.next();
      ++T;
    }
  } else if (warp >= DRAIN_WARP0 && warp < KAPPA_WARP0) {
    // ===================== drain warps (4): row image -> TMEM, O_I / O_J -> sums =====================
    const int q = warp & 3;
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int i_loc = q * 32 + lane;
    uint32_t K = 0;
    // 128 output rows x t columns -> fixed point -> SMEM staging (column-major,
    // the global layout) -> one TMA bulk reduce-add per 128-row block, issued by one
    // thread; the L2 does the 64-bit integer adds at line granularity
    const bool issuer = warp == DRAIN_WARP0 && lane == 0;
    uint32_t nflush = 0;
    auto flush = [&](int64_t row0, const float (&v)[TN]) {
      unsigned long long* sb = stage + (nflush & 1) * (STAGE_BYTES / 8);
      if (issuer) SYM_T(4, asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"));   // buffer's last reduce read it
      SYM_T(1, drain_bar());
      const int64_t row = row0 + i_loc;
      const bool in = row < a.n;
#pragma unroll
      for (int c = 0; c < TN; ++c) {
        if (c >= a.t) break;   // only the t live columns are staged and reduced
        long long x = 0;
        if (in) {
          // v 2^E_c truncated toward zero (exact scaling: |v| 2^E_c <= 2^61 by
          // the choice of E_c); one F2I on the XU pipe, which has headroom
          if (fabsf(v[c]) < INFINITY) x = __float2ll_rz(v[c] * scale_s[c]);
          else a.bad[row] = 1;
        }
        sb[c * BT + i_loc] = (unsigned long long)x;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      drain_bar();
      if (issuer) {
        // the t columns of a 128-row block are contiguous in both the staging
        // buffer and the row-block-major sums: ONE reduce-add of t x 1 KB
        // (t separate 1 KB reduce-adds kept the drain's issuer on the
        // critical path: n = 10^6 337.9 -> 328.5 ms)
        bulk_red_u64(a.acc + row0 * a.t, smem_u32(sb), (uint32_t)a.t * BT * 8u);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ++nflush;
    };
    // O_I partials of the current (chunk, row block), fp32; 16-byte chunks
    // swizzled by row so the 128-bit accesses of a warp hit distinct banks
    const int sw = (i_loc >> 1) & 3;
    auto acci_row = [&](int r) { return reinterpret_cast<float4*>(acci + (r * BT + i_loc) * TN); };
    auto flush_acci = [&](int P, int rows) {
      for (int r = 0; r < rows; ++r) {
        float4* ar = acci_row(r);
        float v[TN];
#pragma unroll
        for (int j = 0; j < TN / 4; ++j) {
          const float4 x = ar[j ^ sw];
          v[4 * j] = x.x; v[4 * j + 1] = x.y; v[4 * j + 2] = x.z; v[4 * j + 3] = x.w;
          ar[j ^ sw] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        SYM_T(5, flush((int64_t)(RB * P + r) * BT, v));
      }
    };
    TileSeq itm;
    itm.begin(a);
    uint32_t Rd = 0;
    while (itm.ok) {
      const int P = itm.P, Q = itm.Q, rows_in = itm.rows_in, cols_in = itm.cols_in;
      for (int r = 0; r < rows_in; ++r) {
        SYM_T(2, wait_p(smem_u32(&oi_full[Rd & 1]), (Rd >> 1) & 1));
        tc_fence_after();
        uint32_t o[32];
        tmem_ld32(tmem + lane_base + TOI(Rd & 1), o);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&oi_empty[Rd & 1]));
        ++Rd;
        float4* ar = acci_row(r);
#pragma unroll
        for (int j = 0; j < TN / 4; ++j) {
          float4 x = ar[j ^ sw];
          x.x += __uint_as_float(o[4 * j]) + __uint_as_float(o[4 * j + TN]);
          x.y += __uint_as_float(o[4 * j + 1]) + __uint_as_float(o[4 * j + 1 + TN]);
          x.z += __uint_as_float(o[4 * j + 2]) + __uint_as_float(o[4 * j + 2 + TN]);
          x.w += __uint_as_float(o[4 * j + 3]) + __uint_as_float(o[4 * j + 3 + TN]);
          ar[j ^ sw] = x;
        }
      }
      SYM_T(3, wait_p(smem_u32(oj_full), K & 1));
      SYM_COUNT();
      tc_fence_after();
      for (int cc = 0; cc < RB; ++cc) {
        const bool live = cc < cols_in && !(P == Q && cc == 0);
        uint32_t o[32];
        if (live) {
          tmem_ld32(tmem + lane_base + TOJ(cc), o);
          tmem_wait_ld();
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&oj_empty[cc]));
        if (live) {
          float v[TN];
#pragma unroll
          for (int c = 0; c < TN; ++c) v[c] = __uint_as_float(o[c]) + __uint_as_float(o[c + TN]);
          SYM_T(5, flush((int64_t)(RB * Q + cc) * BT, v));
        }
      }
      ++K;
      const int k_now = itm.k;
      itm.next_item();
      // leaving the chunk or the row block: the carried O_I partials go out
      if (!itm.ok || itm.k != k_now || itm.P != P) flush_acci(P, rows_in);
    }
    if (issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }

  if (GP_SYM_PROF_BUILD && a.prof && lane == 0) {
    tacc[6] = clock64() - t_start;
    for (int k = 0; k < 8; ++k) a.prof[((int64_t)blockIdx.x * (NTHREADS / 32) + warp) * 8 + k] = tacc[k];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == DRAIN_WARP0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

// per column: E_c with 2^E_c ||V_c||_1 <= 2^61 (no fixed-point overflow: kappa
// <= 1), s_c with 2^s_c max|V_c| <= 2^14 (fp16 range); partial sums arrive in
// units of 2^s_c, so they are converted with exponent E_c - s_c
// the per-column sums run on an 8-CTA cluster (rows split across the CTAs,
// partials combined by CTA 0 over distributed shared memory in rank order:
// deterministic, no workspace; one CTA per column took ~0.5 ms at n = 10^6)
constexpr int kScaleCtas = 8;
__global__ void __cluster_dims__(kScaleCtas, 1, 1) __launch_bounds__(1024)
    sym_scale_kernel(const float* __restrict__ V, int64_t ldv, int64_t n, int t, int* expo, float* vscale,
                     double* inv_scale) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  __shared__ double red[1024];
  __shared__ float mxr[1024];
  __shared__ double psum[TN];
  __shared__ float pmax[TN];
  const int rank = (int)cl.block_rank(), nb = (int)cl.num_blocks();
  const int64_t per = (n + nb - 1) / nb;
  const int64_t r0 = min(n, (int64_t)rank * per), r1 = min(n, r0 + per);
  const int tw = max(t, 1), rpp = (int)blockDim.x / tw;
  const int tr = (int)threadIdx.x / tw, tc = (int)threadIdx.x - tr * tw;
  double s = 0.0;
  float m = 0.f;
  if (tr < rpp && tc < t)
#pragma unroll 8  // loads of later rows issue ahead of the dependent adds
    for (int64_t i = r0 + tr; i < r1; i += rpp) {
      const float x = fabsf(V[i * ldv + tc]);
      s += (double)x;
      m = fmaxf(m, x);
    }
  red[threadIdx.x] = s;
  mxr[threadIdx.x] = m;
  __syncthreads();
  if ((int)threadIdx.x < t) {
    double ss = 0.0;
    float mm = 0.f;
    for (int q = 0; q < rpp; ++q) {
      ss += red[q * tw + threadIdx.x];
      mm = fmaxf(mm, mxr[q * tw + threadIdx.x]);
    }
    psum[threadIdx.x] = ss;
    pmax[threadIdx.x] = mm;
  }
  cl.sync();
  if (rank == 0 && (int)threadIdx.x < TN) {
    const int c = threadIdx.x;
    double l1 = 0.0;
    float mx = 0.f;
    if (c < t)
      for (int b = 0; b < nb; ++b) {
        l1 += *cl.map_shared_rank(&psum[c], b);
        mx = fmaxf(mx, *cl.map_shared_rank(&pmax[c], b));
      }
    // partials carry the 2^kKScaleLog2 K scaling: |partial| <= 2^(S+12) ||V_c||_1
    int E = 61 - kKScaleLog2, S = 0;
    if (l1 > 0.0 && l1 < INFINITY) {
      int ex;
      frexp(l1, &ex);  // l1 < 2^ex
      E = 61 - kKScaleLog2 - ex;
      frexp((double)mx, &ex);
      S = 14 - ex;
    }
    E = max(-100, min(100, E));
    S = max(-100, min(100, S));
    expo[c] = E - S;
    vscale[c] = ldexpf(1.0f, S);
    inv_scale[c] = ldexp(1.0, -E - kKScaleLog2);
  }
  cl.sync();
}

// out[i, c] = s2 * acc[i][c] 2^-E_c (+ noise V[i + diag_offset, c]); NaN where a
// non-finite partial was seen (the host names the partition, partition.py:231-236)
// rows [row0, row1) of the operator: out[i - row0, c]. acc / bad hold the rows
// from acc_row0 on (a multiple of BT: a rank's reduce-scattered slice)
__global__ void sym_finalize_kernel(const long long* __restrict__ acc, int64_t acc_row0,
                                    const int* __restrict__ bad, const double* __restrict__ inv_scale,
                                    int64_t row0, int64_t row1, int t, float* out, int64_t ldo, double s2,
                                    double noise, const float* V, int64_t ldv, int64_t diag_offset) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (row1 - row0) * t) return;
  const int64_t i = row0 + idx / t;
  const int c = (int)(idx % t);
  const int64_t li = i - acc_row0;
  double r = s2 * ((double)acc[((li / BT) * t + c) * BT + (li % BT)] * inv_scale[c]);
  if (diag_offset >= 0) r += noise * (double)V[(i + diag_offset) * ldv + c];
  out[(i - row0) * ldo + c] = bad[li] ? __int_as_float(0x7fc00000) : (float)r;
}

struct Plan {
  int DK, tiles, nblocks, n_items, nsc, nsv;
  int64_t acc_ld;
  size_t img_bytes_all, v_img_bytes, acc_bytes, bad_bytes, smem;
};

static Plan make_plan(const gp_kv_desc* d) {
  Plan p;
  p.DK = (d->d + 2 + 7) / 8 * 8;
  p.tiles = (int)((d->n_rows + BT - 1) / BT);
  p.nblocks = (p.tiles + RB - 1) / RB;
  p.n_items = p.nblocks * (p.nblocks + 1) / 2;
  p.acc_ld = (int64_t)p.tiles * BT;
  const size_t img = 2u * BT * p.DK * 4u;
  p.img_bytes_all = (size_t)p.tiles * img;
  p.v_img_bytes = (size_t)p.tiles * V_TILE_BYTES;
  p.acc_bytes = (size_t)TN * p.acc_ld * 8;
  p.bad_bytes = (size_t)p.acc_ld * 4;
  const size_t budget = 227 * 1024;
  const size_t fixed = KS_BYTES + img + 2 * V_TILE_BYTES + ACCI_BYTES + 2 * STAGE_BYTES + BAR_BYTES;
  p.nsc = 2;
  p.nsv = 0;
  // a 2-deep V_J ring, released by sk_empty (one commit less per tile on the
  // MMA thread than a 3-deep ring with its own barrier: n = 10^6 354 -> 350 ms)
  if (fixed + p.nsc * img + 2 * V_TILE_BYTES <= budget) p.nsv = 2;
  p.smem = fixed + p.nsc * img + p.nsv * V_TILE_BYTES;
  return p;
}

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace tcs

// the symmetric kernel applies to the whole square training operator:
// the same point set on both sides, every row and column, t <= 16
bool kv_sym_supported(const gp_kv_desc* d, int t) {
  if (t < 1 || t > tcs::TN) return false;
  if (d->d < 1 || d->d + 2 > 16) return false;   // DK <= 16: the SMEM plan (d <= 14)
  if (d->Xr != d->Xc || d->ldr != d->ldc || d->n_rows != d->n_cols || d->n_rows < 1) return false;
  if (d->self_offset != 0 || (d->diag_offset != 0 && d->diag_offset >= 0)) return false;
  return tcs::make_plan(d).nsv >= 2;
}

size_t kv_sym_workspace(const gp_kv_desc* d, int t) {
  if (!kv_sym_supported(d, t)) return 0;
  tcs::Plan p = tcs::make_plan(d);
  using tcs::align256;
  return 2 * align256(p.img_bytes_all) + align256(p.v_img_bytes) + align256(p.acc_bytes) +
         align256(p.bad_bytes) + 256 * sizeof(double) + 3 * 64 * sizeof(double);
}

namespace tcs {
struct WsView {
  float* row_img; float* col_img; __half* v_img;
  long long* acc; int* bad; double* mean; int* expo; float* vscale; double* inv_scale;
};
static WsView carve(const Plan& p, void* ws) {
  WsView v;
  char* w = static_cast<char*>(ws);
  v.row_img = reinterpret_cast<float*>(w); w += align256(p.img_bytes_all);
  v.col_img = reinterpret_cast<float*>(w); w += align256(p.img_bytes_all);
  v.v_img = reinterpret_cast<__half*>(w); w += align256(p.v_img_bytes);
  v.acc = reinterpret_cast<long long*>(w); w += align256(p.acc_bytes);
  v.bad = reinterpret_cast<int*>(w); w += align256(p.bad_bytes);
  v.mean = reinterpret_cast<double*>(w); w += 256 * sizeof(double);
  v.expo = reinterpret_cast<int*>(w); w += 64 * sizeof(double);
  v.vscale = reinterpret_cast<float*>(w); w += 64 * sizeof(double);
  v.inv_scale = reinterpret_cast<double*>(w);
  return v;
}
}  // namespace tcs

int64_t kv_sym_acc_ld(const gp_kv_desc* desc) { return tcs::make_plan(desc).acc_ld; }

// fixed-point sums (tiles x t x 128, row-block major) of the items L = part (mod
// nparts) of the symmetric schedule, written into acc / bad (zeroed here);
// partial sums of disjoint item sets add up (int64) to the full product
int kv_sym_partial(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, int part, int nparts,
                   long long* acc, int* bad, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace tcs;
  GP_REQUIRE(kv_sym_supported(desc, t), "gp_kv_sym: shape unsupported by the symmetric kernel");
  GP_REQUIRE(nparts >= 1 && part >= 0 && part < nparts, "gp_kv_sym: part %d of %d", part, nparts);
  Plan p = make_plan(desc);
  size_t need = kv_sym_workspace(desc, t);
  GP_REQUIRE(ws != nullptr && ws_bytes >= need, "gp_kv(symmetric): workspace of %zu bytes required, %zu given",
             need, ws_bytes);
  WsView w = carve(p, ws);
  const int64_t n = desc->n_rows;
  const double c = desc->family == GP_FAMILY_RBF ? 1.4426950408889634 : -6.0;
  GP_CUDA_TRY(cudaMemsetAsync(acc, 0, (size_t)t * p.acc_ld * 8, st));
  GP_CUDA_TRY(cudaMemsetAsync(bad, 0, p.bad_bytes, st));
  sym_scale_kernel<<<kScaleCtas, 1024, 0, st>>>(V, ldv, n, t, w.expo, w.vscale, w.inv_scale);
  GP_LAUNCH_CHECK();
  if (!kv_images_current)
    if (int rc = tc::distance_images(desc->Xr, desc->ldr, n, desc->Xc, desc->ldc, n, desc->d, p.DK, BT, BT, c,
                                     w.mean, w.row_img, w.col_img, st))
      return rc;
  // the 128-point V image is two consecutive 64-point tile images
  if (int rc = tc::v_images16(V, ldv, t, n, w.vscale, w.v_img, 2 * (int64_t)p.tiles, st)) return rc;
  Args a;
  a.row_img = w.row_img; a.col_img = w.col_img; a.v_img = w.v_img; a.DK = p.DK;
  a.n = n; a.tiles = p.tiles; a.nblocks = p.nblocks; a.n_items = p.n_items;
  a.nsc = p.nsc; a.nsv = p.nsv; a.t = t; a.part = part; a.nparts = nparts;
  a.expo = w.expo; a.acc = reinterpret_cast<unsigned long long*>(acc); a.acc_ld = p.acc_ld; a.bad = bad;
  a.prof = nullptr;
  a.chunk = item_chunk(p.n_items);
  const int chunks = (p.n_items + a.chunk - 1) / a.chunk;
  const int my_chunks = (chunks - part + nparts - 1) / nparts;
  if (my_chunks < 1) return GP_OK;
  int grid = std::min(my_chunks, num_sms());
  auto kern = desc->family == GP_FAMILY_RBF
                  ? (p.DK == 8 ? kv_sym_kernel<GP_FAMILY_RBF, 8> : kv_sym_kernel<GP_FAMILY_RBF, 16>)
                  : (p.DK == 8 ? kv_sym_kernel<GP_FAMILY_MATERN32, 8> : kv_sym_kernel<GP_FAMILY_MATERN32, 16>);
  GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem));
  const char* pe = getenv("GP_SYM_PROF");
  if (GP_SYM_PROF_BUILD && pe && *pe == '1') GP_CUDA_TRY(cudaMalloc(&a.prof, (size_t)grid * (NTHREADS / 32) * 8 * sizeof(long long)));
  kern<<<grid, NTHREADS, p.smem, st>>>(a);
  GP_LAUNCH_CHECK();
  if (a.prof) {   // diagnostic only: per-role average cycles per event, CTA-averaged
    std::vector<long long> h((size_t)grid * (NTHREADS / 32) * 8);
    GP_CUDA_TRY(cudaStreamSynchronize(st));
    GP_CUDA_TRY(cudaMemcpy(h.data(), a.prof, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
    cudaFree(a.prof);
    for (int wi : {1, DRAIN_WARP0, KAPPA_WARP0, KAPPA_WARP0 + 15}) {
      double s[8] = {0};
      for (int cta = 0; cta < grid; ++cta)
        for (int k = 0; k < 8; ++k) s[k] += (double)h[((size_t)cta * (NTHREADS / 32) + wi) * 8 + k];
      fprintf(stderr, "[sym prof] warp %d:", wi);
      for (int k = 0; k < 8; ++k) fprintf(stderr, " w%d=%.0f", k, k == 7 ? s[7] / grid : s[k] / std::max(1.0, s[7]));
      fprintf(stderr, "\n");
    }
  }
  return GP_OK;
}

namespace tcs {
// rows [row0, row1) of s2 * K V (+ noise V) from the (summed) fixed-point
// accumulator; the scales are recomputed from V (the same V as the partials)
// unless this workspace already holds them (the single-device product)
static int finalize_rows(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, const long long* acc,
                         const int* bad, int64_t acc_row0, int64_t row0, int64_t row1, float* out, int64_t ldo,
                         void* ws, size_t ws_bytes, cudaStream_t st, bool scales_ready) {
  using namespace tcs;
  GP_REQUIRE(kv_sym_supported(desc, t), "gp_kv_sym: shape unsupported by the symmetric kernel");
  GP_REQUIRE(0 <= row0 && row0 <= row1 && row1 <= desc->n_rows, "gp_kv_sym_finalize: rows [%lld, %lld)",
             (long long)row0, (long long)row1);
  GP_REQUIRE(acc_row0 >= 0 && acc_row0 % BT == 0 && acc_row0 <= row0,
             "gp_kv_sym_finalize: acc_row0=%lld must be a multiple of %d and <= row0", (long long)acc_row0, BT);
  Plan p = make_plan(desc);
  size_t need = kv_sym_workspace(desc, t);
  GP_REQUIRE(ws != nullptr && ws_bytes >= need, "gp_kv(symmetric): workspace of %zu bytes required, %zu given",
             need, ws_bytes);
  WsView w = carve(p, ws);
  if (!scales_ready) {
    sym_scale_kernel<<<kScaleCtas, 1024, 0, st>>>(V, ldv, desc->n_rows, t, w.expo, w.vscale, w.inv_scale);
    GP_LAUNCH_CHECK();
  }
  const int64_t tot = (row1 - row0) * t;
  if (tot == 0) return GP_OK;
  sym_finalize_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(acc, acc_row0, bad, w.inv_scale, row0, row1, t,
                                                                     out, ldo, desc->outputscale, desc->noise, V,
                                                                     ldv, desc->diag_offset);
  GP_LAUNCH_CHECK();
  return GP_OK;
}
}  // namespace tcs

int kv_sym_finalize(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, const long long* acc,
                    const int* bad, int64_t acc_row0, int64_t row0, int64_t row1, float* out, int64_t ldo, void* ws,
                    size_t ws_bytes, cudaStream_t st) {
  return tcs::finalize_rows(desc, V, ldv, t, acc, bad, acc_row0, row0, row1, out, ldo, ws, ws_bytes, st, false);
}

int kv_sym(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo, void* ws,
           size_t ws_bytes, cudaStream_t st) {
  using namespace tcs;
  GP_REQUIRE(ws != nullptr && ws_bytes >= kv_sym_workspace(desc, t),
             "gp_kv(symmetric): workspace of %zu bytes required, %zu given", kv_sym_workspace(desc, t), ws_bytes);
  WsView w = carve(make_plan(desc), ws);
  if (int rc = kv_sym_partial(desc, V, ldv, t, 0, 1, w.acc, w.bad, ws, ws_bytes, st)) return rc;
  // kv_sym_partial left this V's scales in the workspace
  return finalize_rows(desc, V, ldv, t, w.acc, w.bad, 0, 0, desc->n_rows, out, ldo, ws, ws_bytes, st, true);
}

}  // namespace gp
