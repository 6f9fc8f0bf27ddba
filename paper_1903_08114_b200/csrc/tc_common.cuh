// tcgen05 / TMEM / bulk-TMA / mbarrier helpers shared by the sm_100a
// tensor-core kernels (kv_tc.cu, grad_tc.cu). Inline PTX only.
#pragma once

#include "gp_common.cuh"

#include <cuda_fp16.h>

namespace gp {
namespace tc {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}
// D[tmem] (+)= A[smem desc] . B[smem desc]
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[tmem] . B[smem desc]
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

#define GP_R32(a) "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]), "=r"(a[4]), "=r"(a[5]), "=r"(a[6]), \
    "=r"(a[7]), "=r"(a[8]), "=r"(a[9]), "=r"(a[10]), "=r"(a[11]), "=r"(a[12]), "=r"(a[13]),          \
    "=r"(a[14]), "=r"(a[15]), "=r"(a[16]), "=r"(a[17]), "=r"(a[18]), "=r"(a[19]), "=r"(a[20]),       \
    "=r"(a[21]), "=r"(a[22]), "=r"(a[23]), "=r"(a[24]), "=r"(a[25]), "=r"(a[26]), "=r"(a[27]),       \
    "=r"(a[28]), "=r"(a[29]), "=r"(a[30]), "=r"(a[31])
#define GP_W32(a) "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]),         \
    "r"(a[7]), "r"(a[8]), "r"(a[9]), "r"(a[10]), "r"(a[11]), "r"(a[12]), "r"(a[13]), "r"(a[14]),      \
    "r"(a[15]), "r"(a[16]), "r"(a[17]), "r"(a[18]), "r"(a[19]), "r"(a[20]), "r"(a[21]), "r"(a[22]),   \
    "r"(a[23]), "r"(a[24]), "r"(a[25]), "r"(a[26]), "r"(a[27]), "r"(a[28]), "r"(a[29]), "r"(a[30]),   \
    "r"(a[31])

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : GP_R32(v)
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      GP_W32(v)
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
// 16 lanes x 256 bits, x8 (64 columns): register r of thread t lands in lane
// t/4 + 8*((r>>1)&1), column 8*(r>>2) + 2*(t%4) + (r&1)
__device__ __forceinline__ void tmem_st16x256_x8(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      GP_W32(v)
      : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// SMEM matrix descriptor, K-major, no swizzle (canonical 8-row x 16-byte core
// matrices): LBO = byte distance between K-adjacent core matrices, SBO =
// byte distance between M/N-adjacent core matrices. Bits: start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version 1 [46,48), layout 0 [61,64).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// instruction descriptor: D f32, A/B tf32, K-major both, N>>3 at [17,23), M>>4 at [24,29)
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// canonical K-major no-swizzle offset (floats) of element (r, k) in an R-row tile
__host__ __device__ __forceinline__ int canon(int r, int k, int R) {
  return (((k >> 2) * (R >> 3) + (r >> 3)) << 5) + ((r & 7) << 2) + (k & 3);
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.b32 %0, 1, 0, P;\n}"
      : "=r"(pred));
  return pred != 0;
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t y;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(y) : "f"(x));
  return __uint_as_float(y);
}

// instruction descriptor, kind::f16 with fp16 A/B, fp32 D, K-major both
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma16_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// D[tmem] (+)= A[smem desc] . B[smem desc], kind::f16
__device__ __forceinline__ void mma16_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// instruction-descriptor bit selecting an MN-major A operand (SMEM only)
constexpr uint32_t IDESC_A_MN_MAJOR = 1u << 15;
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// 16 lanes x 256 bits, x4 (32 columns): register r of thread t lands in lane
// t/4 + 8((r>>1)&1), column 8(r>>2) + 2(t%4) + (r&1)
__device__ __forceinline__ void tmem_st16x256_x4(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x256b.x4.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
      "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
// kappa / s2 scaled by 2^kKScaleLog2 for the fp16 split below: K1 and the
// residual K2 = K - K1 (~2^-11 K) then stay in fp16's normal range down to
// K ~ 2^-15 instead of 2^-3, so small kernel values keep their relative
// precision (the scale folds into the ex2 argument: free for Matérn, one
// FADD for RBF; the consumers divide it out with the V column scales)
constexpr int kKScaleLog2 = 12;
template <int FAM>
__device__ __forceinline__ float kappa_split_scaled(float sv) {
  if (FAM == GP_FAMILY_RBF) {
    return ex2_approx(min0_nan(sv) + (float)kKScaleLog2);          // S = -log2(e) r2 / 2
  } else {
    const float u = sqrt_approx(max0_nan(sv));                       // S = 3 r2, u = sqrt(3) r
    const float ex = ex2_approx(fmaf(u, -kLog2e, (float)kKScaleLog2));
    return fmaf(u, ex, ex);                                          // 2^12 (1 + sqrt3 r) e^{-sqrt3 r}
  }
}
// fp16 split of a pair: K1 = K truncated to 11 significant bits, K2 = fp16(K - K1)
__device__ __forceinline__ void split_pair(float a, float b, uint32_t& k1, uint32_t& k2) {
  const float a1 = __uint_as_float(__float_as_uint(a) & 0xFFFFE000u);
  const float b1 = __uint_as_float(__float_as_uint(b) & 0xFFFFE000u);
  __half2 h1 = __floats2half2_rn(a1, b1);
  __half2 h2 = __floats2half2_rn(a - a1, b - b1);
  k1 = *reinterpret_cast<uint32_t*>(&h1);
  k2 = *reinterpret_cast<uint32_t*>(&h2);
}

// canonical K-major no-swizzle offset (halves) of element (r, k) in an R-row
// 16-bit tile: core matrix = 8 rows x 8 halves (16 B)
__host__ __device__ __forceinline__ int canon16(int r, int k, int R) {
  return (((k >> 3) * (R >> 3) + (r >> 3)) << 6) + ((r & 7) << 3) + (k & 7);
}

int distance_images(const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
                    int d, int DK, int BMr, int BNc, double c, double* mean, float* row_img,
                    float* col_img, cudaStream_t st);
// fp16 hi | lo images for large d (DK >= 48): one power-of-two scale per side
// (|value| <= 2^14), *dscale = 2^(e_row + e_col) multiplies S back; rng: 4
// words of scratch
int distance_images16(const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
                      int d, int DK, int BMr, int BNc, double c, double* mean, unsigned* rng, __half* row_img,
                      __half* col_img, float* dscale, cudaStream_t st);
// fp16 V image for the contraction: per 64-point tile a 32-row K-major operand,
// rows 0-15 V1 = fp16(2^s_c V), rows 16-31 V2 = fp16(2^s_c V - V1)
int v_images16(const float* V, int64_t ldv, int t, int64_t ncols, const float* vscale, __half* img,
               int64_t ntiles, cudaStream_t st);
// tf32 V image: per 64-point tile a 32-row K-major operand [V_hi | V_lo]
int v_images32(const float* V, int64_t ldv, int t, int64_t ncols, float* img, int64_t ntiles, cudaStream_t st);
// fp16 V image for the wide kernel: rows 0..NW-1 V1, NW..2NW-1 V2 per tile of tile_points points
int v_images16_wide(const float* V, int64_t ldv, int t, int NW, int64_t ncols, const float* vscale, __half* img,
                    int64_t ntiles, cudaStream_t st, int tile_points = 64);
// per-column power-of-two scales 2^s_c with 2^s_c max|V_c| <= 2^14 (fp16 range) and their inverses
int v_colscale(const float* V, int64_t ldv, int64_t n, int t, float* vscale, float* inv_vscale, cudaStream_t st);

}  // namespace tc
}  // namespace gp
