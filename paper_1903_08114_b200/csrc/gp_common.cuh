// Shared helpers for the gpbbmm CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/gpbbmm.h"

namespace gp {

int set_error(int code, const char* fmt, ...);

// Set by a caller that applies the same operator (same points, same
// workspace) repeatedly — the mBCG loop of gp_mbcg_solve_kv from its second
// iteration on: the K·V kernels then keep the distance images already in the
// workspace instead of rebuilding them from the points.
extern thread_local bool kv_images_current;

#define GP_CUDA_TRY(expr)                                                        \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      return ::gp::set_error(GP_ECUDA, "%s failed: %s (%s:%d)", #expr,           \
                             cudaGetErrorString(_e), __FILE__, __LINE__);        \
  } while (0)

// every kernel launch site is followed by GP_LAUNCH_CHECK(), which also
// counts launches (gp_launch_count) so benchmarks can report how many of
// this library's kernels ran inside a timed region
void note_launch();
#define GP_LAUNCH_CHECK()          \
  do {                             \
    ::gp::note_launch();           \
    GP_CUDA_TRY(cudaGetLastError()); \
  } while (0)

#define GP_REQUIRE(cond, ...)                                                    \
  do {                                                                           \
    if (!(cond)) return ::gp::set_error(GP_EINVAL, __VA_ARGS__);                 \
  } while (0)

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSqrt3 = 1.7320508075688772f;
constexpr double kSqrt3d = 1.7320508075688772935;

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// clamps that propagate NaN in one FMNMX.NAN (the reference raises on
// non-finite kernel blocks, partition.py:231-236, so NaN must survive)
__device__ __forceinline__ float max0_nan(float x) {
  float y;
  asm("max.NaN.f32 %0, %1, 0f00000000;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float min0_nan(float x) {
  float y;
  asm("min.NaN.f32 %0, %1, 0f00000000;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// kappa(r^2) / s2 in fp32 (kernels.py:225-244)
template <int FAM>
__device__ __forceinline__ float kappa_f32(float r2) {
  if (FAM == GP_FAMILY_RBF) {
    return ex2_approx(r2 * (-0.5f * kLog2e));
  } else {
    float r = sqrt_approx(r2);
    return fmaf(kSqrt3, r, 1.0f) * ex2_approx(r * (-kSqrt3 * kLog2e));
  }
}

__device__ __forceinline__ double kappa_f64(int fam, double r2) {
  if (fam == GP_FAMILY_RBF) return exp(-0.5 * r2);
  double r = sqrt(r2);
  return (1.0 + kSqrt3d * r) * exp(-kSqrt3d * r);
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

int num_sms();

// out[row, c] = s2 * sum_s ws[s, row, c] (+ noise V[row + diag_offset, c])
int launch_split_reduce(const float* ws, int S, int64_t stride, int64_t nr, int t, float* out,
                        int64_t ldo, float s2, float noise, const float* V, int64_t ldv,
                        int64_t diag_offset, cudaStream_t st);

}  // namespace gp
