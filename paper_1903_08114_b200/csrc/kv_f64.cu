// fp64 fused K(X_rows, X_cols)·V — the precision of the reference's own
// partitioned_mvm / predict_mean / verify_cache (everything float64,
// partition.py:206-207, kernels.py:216-244, predictor.py:100-132), without
// materialising the block.
//
// The training mBCG keeps its fp32 tcgen05 operator (north_star tolerance);
// this kernel serves the reference-facing entry points whose contract is
// fp64 (the shipped tests compare partitioned_mvm with a dense fp64 product
// at 1e-12, test_partition.py:71-90).
//
// Bound: the FP64 pipe (one DFMA per (entry, dimension) for the direct
// difference form, ~25 DFMA-equivalents for exp/sqrt, one DFMA per
// (entry, RHS column)). Layout per CTA (256 threads): 64 rows × all
// columns in 32-column chunks staged in SMEM; phase 1 writes the 64 × 32
// kappa tile to SMEM (8 entries per thread), phase 2 contracts it against the
// staged V chunk (thread = row × column group, ≤ 16 fp64 accumulators).
// Columns split across gridDim.y with per-split partials reduced in a fixed
// order, so the result is deterministic.

#include <algorithm>

#include "gp_common.cuh"

namespace gp {
namespace {

constexpr int kBR = 64;      // rows per CTA
constexpr int kBC = 32;      // columns per chunk
constexpr int kTC = 64;      // RHS columns per pass
constexpr int kThreads = 256;

struct KvF64Args {
  int fam, d, dp;            // dp = SMEM row stride of the point tiles (odd)
  const double* Xr; int64_t ldr; int64_t nr;
  const double* Xc; int64_t ldc; int64_t nc;
  double s2;
  const double* V; int64_t ldv; int t;
  int t0, tw;                // RHS columns [t0, t0 + tw) of this pass
  int S;                     // column splits
  double* part;              // S x nr x tw partials (S > 1)
  double* out; int64_t ldo;  // S == 1: final (before noise)
};

__global__ void __launch_bounds__(kThreads) kv_f64_kernel(KvF64Args a) {
  extern __shared__ double sm[];
  double* xr = sm;                       // kBR x dp
  double* xc = xr + kBR * a.dp;          // kBC x dp
  double* kt = xc + kBC * a.dp;          // kBR x (kBC + 1)
  double* vt = kt + kBR * (kBC + 1);     // kBC x kTC
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * kBR;
  const int split = blockIdx.y;
  const int64_t cpb = (a.nc + a.S - 1) / a.S;
  const int64_t c_lo = min(a.nc, (int64_t)split * cpb);
  const int64_t c_hi = min(a.nc, c_lo + cpb);

  for (int e = tid; e < kBR * a.d; e += kThreads) {
    int r = e / a.d, k = e - r * a.d;
    xr[r * a.dp + k] = (r0 + r < a.nr) ? a.Xr[(r0 + r) * a.ldr + k] : 0.0;
  }
  const int crow = tid >> 2, cgrp = tid & 3;  // contraction: row, column group
  double acc[kTC / 4];
#pragma unroll
  for (int q = 0; q < kTC / 4; ++q) acc[q] = 0.0;

  for (int64_t c0 = c_lo; c0 < c_hi; c0 += kBC) {
    const int cw = (int)min((int64_t)kBC, c_hi - c0);
    __syncthreads();  // previous chunk fully consumed
    for (int e = tid; e < kBC * a.d; e += kThreads) {
      int c = e / a.d, k = e - c * a.d;
      xc[c * a.dp + k] = (c < cw) ? a.Xc[(c0 + c) * a.ldc + k] : 0.0;
    }
    for (int e = tid; e < kBC * a.tw; e += kThreads) {
      int c = e / a.tw, q = e - c * a.tw;
      vt[c * kTC + q] = (c < cw) ? a.V[(c0 + c) * a.ldv + a.t0 + q] : 0.0;
    }
    __syncthreads();
    // phase 1: kappa tile (warp = one row x 32 columns)
#pragma unroll 1
    for (int e = tid; e < kBR * kBC; e += kThreads) {
      int r = e >> 5, c = e & 31;
      const double* xa = xr + r * a.dp;
      const double* xb = xc + c * a.dp;
      double r2 = 0.0;
      for (int k = 0; k < a.d; ++k) {
        double df = xa[k] - xb[k];
        r2 = fma(df, df, r2);
      }
      kt[r * (kBC + 1) + c] = (c < cw) ? kappa_f64(a.fam, r2) : 0.0;
    }
    __syncthreads();
    // phase 2: acc[row, cgrp + 4 q] += sum_c kt[row, c] vt[c, cgrp + 4 q]
    const double* krow = kt + crow * (kBC + 1);
#pragma unroll 4
    for (int c = 0; c < kBC; ++c) {
      double kv = krow[c];
      const double* vr = vt + c * kTC + cgrp;
#pragma unroll
      for (int q = 0; q < kTC / 4; ++q) acc[q] = fma(kv, vr[4 * q], acc[q]);
    }
  }
  const int64_t row = r0 + crow;
  if (row >= a.nr) return;
#pragma unroll
  for (int q = 0; q < kTC / 4; ++q) {
    int col = cgrp + 4 * q;
    if (col >= a.tw) continue;
    if (a.S == 1)
      a.out[row * a.ldo + a.t0 + col] = a.s2 * acc[q];
    else
      a.part[((int64_t)split * a.nr + row) * a.tw + col] = acc[q];
  }
}

// fixed-order sum of the column-split partials, noise on the diagonal, and
// the first row holding a non-finite value (partition.py:231-236)
__global__ void kv_f64_finish(const double* __restrict__ part, int S, int64_t nr, int t0, int tw,
                              double s2, double noise, const double* __restrict__ V, int64_t ldv,
                              int64_t diag_offset, int64_t nc, double* out, int64_t ldo,
                              int32_t* first_bad) {
  int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nr * tw) return;
  int64_t row = e / tw;
  int col = (int)(e - row * tw);
  double v;
  if (S > 1) {
    double s = 0.0;
    for (int k = 0; k < S; ++k) s += part[((int64_t)k * nr + row) * tw + col];
    v = s2 * s;
  } else {
    v = out[row * ldo + t0 + col];
  }
  if (diag_offset >= 0 && row + diag_offset < nc) v = fma(noise, V[(row + diag_offset) * ldv + t0 + col], v);
  out[row * ldo + t0 + col] = v;
  if (first_bad && !isfinite(v)) atomicMin(first_bad, (int32_t)row);
}

size_t smem_bytes(int d) {
  int dp = d | 1;
  return sizeof(double) * ((size_t)(kBR + kBC) * dp + (size_t)kBR * (kBC + 1) + (size_t)kBC * kTC);
}

int splits_for(int64_t nr, int64_t nc) {
  int tiles = ceil_div(nr, kBR);
  int want = (4 * num_sms() + tiles - 1) / tiles;  // >= 4 CTAs per SM in flight
  int64_t max_by_cols = std::max<int64_t>(1, nc / (4 * kBC));
  return (int)std::max<int64_t>(1, std::min<int64_t>(std::min<int64_t>(want, 64), max_by_cols));
}

}  // namespace
}  // namespace gp

using namespace gp;

extern "C" {

size_t gp_kv_f64_workspace_bytes(int64_t n_rows, int64_t n_cols, int t) {
  if (n_rows <= 0 || n_cols <= 0 || t < 1) return 0;
  int S = splits_for(n_rows, n_cols);
  return S > 1 ? sizeof(double) * (size_t)S * (size_t)n_rows * (size_t)std::min(t, kTC) : 0;
}

int gp_kv_f64(int family, int d, const double* Xr, int64_t ldr, int64_t n_rows, const double* Xc,
              int64_t ldc, int64_t n_cols, double outputscale, double noise, int64_t diag_offset,
              const double* V, int64_t ldv, int t, double* out, int64_t ldo, int32_t* first_bad_row_dev,
              void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(family == GP_FAMILY_RBF || family == GP_FAMILY_MATERN32, "gp_kv_f64: unknown kernel family %d",
             family);
  GP_REQUIRE(d >= 1 && ldr >= d && ldc >= d, "gp_kv_f64: d=%d ldr=%lld ldc=%lld", d, (long long)ldr,
             (long long)ldc);
  GP_REQUIRE(t >= 1 && ldv >= t && ldo >= t, "gp_kv_f64: t=%d ldv=%lld ldo=%lld", t, (long long)ldv,
             (long long)ldo);
  GP_REQUIRE(n_rows >= 0 && n_cols >= 0, "gp_kv_f64: negative shape");
  GP_REQUIRE(diag_offset < 0 || diag_offset + n_rows <= n_cols,
             "gp_kv_f64: diagonal offset outside the column range");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_rows == 0) return GP_OK;
  if (n_cols == 0) {
    for (int64_t r = 0; r < n_rows; ++r) GP_CUDA_TRY(cudaMemsetAsync(out + r * ldo, 0, sizeof(double) * t, st));
    return GP_OK;
  }
  const size_t smem = smem_bytes(d);
  GP_REQUIRE(smem <= 227 * 1024, "gp_kv_f64: d=%d too large for the SMEM tiles", d);
  GP_CUDA_TRY(cudaFuncSetAttribute(kv_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int S = splits_for(n_rows, n_cols);
  const size_t need = gp_kv_f64_workspace_bytes(n_rows, n_cols, t);
  GP_REQUIRE(workspace_bytes >= need && (need == 0 || workspace != nullptr),
             "gp_kv_f64: workspace of %zu bytes, need %zu", workspace_bytes, need);
  for (int t0 = 0; t0 < t; t0 += kTC) {
    KvF64Args a;
    a.fam = family; a.d = d; a.dp = d | 1;
    a.Xr = Xr; a.ldr = ldr; a.nr = n_rows;
    a.Xc = Xc; a.ldc = ldc; a.nc = n_cols;
    a.s2 = outputscale;
    a.V = V; a.ldv = ldv; a.t = t;
    a.t0 = t0; a.tw = std::min(kTC, t - t0);
    a.S = S; a.part = (double*)workspace; a.out = out; a.ldo = ldo;
    dim3 grid((unsigned)ceil_div(n_rows, kBR), (unsigned)S);
    kv_f64_kernel<<<grid, kThreads, smem, st>>>(a);
    GP_LAUNCH_CHECK();
    int64_t tot = n_rows * a.tw;
    kv_f64_finish<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        (const double*)workspace, S, n_rows, t0, a.tw, outputscale, noise, V, ldv, diag_offset, n_cols, out, ldo,
        first_bad_row_dev);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

}  // extern "C"
