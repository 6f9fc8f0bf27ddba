// Fused gradient forms: for every geometric hyperparameter p,
//   g_p = sum_ij (dK/dtheta_p)_ij H_ij,   H = Y R^T  (never materialised).
//
// Reference: likelihood.py:166-216 applies each dK/dtheta (kernels.py:332-371)
// to R = [a | W | L] and contracts with [a | S-W | ...]. Every term there is a
// bilinear form in dK/dtheta, so with
//   Y = [a/2 | -(S-W)/(2t) | L B^{-1}/(2 noise)],  R = [a | W | L]
// the reference gradient equals g_p - tr(dK/dtheta_p)/(2 noise) (the trace is
// n for the outputscale, 0 for lengthscales). One K=w product per tile plus a
// per-parameter epilogue replaces (1+n_l) x w column products.
//
// Kernel outputs (host applies the constant factors):
//   out[0]    = sum kappa_ij H_ij                 (kappa = k/s2)
//   out[1]    = sum eps_ij D_ij H_ij              (shared lengthscale)
//   out[1+i]  = sum eps_ij (xs_i - xs'_i)^2 H_ij  (ARD lengthscale i)
// eps = e^{-D/2} (RBF) or 3 e^{-sqrt3 r} (Matern-3/2); D = scaled sq. distance.
#include "gp_common.cuh"

#include <algorithm>

namespace gp {

struct GradArgs {
  const float* Xr; int64_t ldr; int64_t nr;
  const float* Xc; int64_t ldc; int64_t nc;
  int d; int ard;
  const float* Y; int64_t ldy;
  const float* R; int64_t ldrr;
  int w;
  int p0, nlc;            // lengthscale dims [p0, p0+nlc) handled by this launch
  int with_s2;            // accumulate out[0] in this launch
  int64_t cols_per_split;
  double* partials;       // [blocks][1 + NLC]
};

constexpr int gBM = 64, gBN = 64;

template <int FAM, int NLC>
__global__ void __launch_bounds__(256, 1) grad_forms_kernel(GradArgs a) {
  extern __shared__ __align__(16) float smem[];
  const int d = a.d, w = a.w;
  const int wp = (w + 3) & ~3;
  float* sXr = smem;               // [d][64]
  float* sXc = sXr + d * gBM;      // [d][64]
  float* sY = sXc + d * gBN;       // [wp][64]
  float* sR = sY + wp * gBM;       // [wp][64]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * gBM;
  const int64_t cbeg = (int64_t)blockIdx.y * a.cols_per_split;
  const int64_t cend = min(a.nc, cbeg + a.cols_per_split);

  for (int idx = tid; idx < gBM * d; idx += 256) {
    int r = idx / d, k = idx - r * d;
    int64_t g = row0 + r;
    sXr[k * gBM + r] = g < a.nr ? a.Xr[g * a.ldr + k] : 0.f;
  }
  for (int idx = tid; idx < gBM * wp; idx += 256) {
    int r = idx / wp, q = idx - r * wp;
    int64_t g = row0 + r;
    sY[q * gBM + r] = (g < a.nr && q < w) ? a.Y[g * a.ldy + q] : 0.f;
  }

  double acc64[1 + NLC];
#pragma unroll
  for (int p = 0; p <= NLC; ++p) acc64[p] = 0.0;

  for (int64_t c0 = cbeg; c0 < cend; c0 += gBN) {
    __syncthreads();
    for (int idx = tid; idx < gBN * d; idx += 256) {
      int c = idx / d, k = idx - c * d;
      int64_t g = c0 + c;
      sXc[k * gBN + c] = g < cend ? a.Xc[g * a.ldc + k] : 0.f;
    }
    for (int idx = tid; idx < gBN * wp; idx += 256) {
      int c = idx / wp, q = idx - c * wp;
      int64_t g = c0 + c;
      sR[q * gBN + c] = (g < cend && q < w) ? a.R[g * a.ldrr + q] : 0.f;
    }
    __syncthreads();

    float h[4][4], dd[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) { h[i][j] = 0.f; dd[i][j] = 0.f; }
#pragma unroll 4
    for (int q = 0; q < wp; ++q) {
      float4 y = *reinterpret_cast<const float4*>(&sY[q * gBM + ty * 4]);
      float4 r = *reinterpret_cast<const float4*>(&sR[q * gBN + tx * 4]);
      float yy[4] = {y.x, y.y, y.z, y.w}, rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) h[i][j] = fmaf(yy[i], rr[j], h[i][j]);
    }
#pragma unroll 4
    for (int k = 0; k < d; ++k) {
      float4 xr = *reinterpret_cast<const float4*>(&sXr[k * gBM + ty * 4]);
      float4 xc = *reinterpret_cast<const float4*>(&sXc[k * gBN + tx * 4]);
      float a4[4] = {xr.x, xr.y, xr.z, xr.w}, b4[4] = {xc.x, xc.y, xc.z, xc.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float df = a4[i] - b4[j];
          dd[i][j] = fmaf(df, df, dd[i][j]);
        }
    }
    float acc32[1 + NLC];
#pragma unroll
    for (int p = 0; p <= NLC; ++p) acc32[p] = 0.f;
    float eh[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        float D = dd[i][j];
        float kap, eps;
        if (FAM == GP_FAMILY_RBF) {
          kap = ex2_approx(D * (-0.5f * kLog2e));
          eps = kap;
        } else {
          float r = sqrt_approx(D);
          float e = ex2_approx(r * (-kSqrt3 * kLog2e));
          kap = fmaf(kSqrt3, r, 1.0f) * e;
          eps = 3.0f * e;
        }
        float hv = h[i][j];
        acc32[0] = fmaf(kap, hv, acc32[0]);
        eh[i][j] = eps * hv;
        if (!a.ard) acc32[1] = fmaf(eh[i][j], D, acc32[1]);
      }
    if (a.ard) {
#pragma unroll
      for (int p = 0; p < NLC; ++p) {
        if (p < a.nlc) {
          const int k = a.p0 + p;
          float4 xr = *reinterpret_cast<const float4*>(&sXr[k * gBM + ty * 4]);
          float4 xc = *reinterpret_cast<const float4*>(&sXc[k * gBN + tx * 4]);
          float a4[4] = {xr.x, xr.y, xr.z, xr.w}, b4[4] = {xc.x, xc.y, xc.z, xc.w};
          float s = 0.f;
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              float df = a4[i] - b4[j];
              s = fmaf(eh[i][j] * df, df, s);
            }
          acc32[1 + p] += s;
        }
      }
    }
#pragma unroll
    for (int p = 0; p <= NLC; ++p) acc64[p] += (double)acc32[p];
  }

  // block reduction, fixed order
  __shared__ double sred[8][1 + 16];
  const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
  for (int p = 0; p <= NLC; ++p) {
    double v = warp_sum(acc64[p]);
    if (lane == 0) sred[wid][p] = v;
  }
  __syncthreads();
  if (tid <= NLC) {
    double s = 0.0;
    for (int q = 0; q < 8; ++q) s += sred[q][tid];
    int64_t b = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    a.partials[b * (1 + NLC) + tid] = s;
  }
}

__global__ void grad_finalize(const double* __restrict__ partials, int nblocks, int W, int p0,
                              int nlc, int with_s2, double* out) {
  int s = threadIdx.x;
  if (s >= W) return;
  if (s == 0 && !with_s2) return;
  if (s >= 1 + nlc) return;
  double acc = 0.0;
  for (int b = 0; b < nblocks; ++b) acc += partials[(int64_t)b * W + s];
  out[s == 0 ? 0 : 1 + p0 + (s - 1)] = acc;
}

bool grad_tc_supported(int64_t nr, int64_t nc, int d, int ard, int w);
bool grad_ard_supported(int64_t nr, int64_t nc, int d, int w);
size_t grad_ard_workspace(int64_t nr, int64_t nc, int d, int w);
int grad_ard(int family, int d, const float* Xr, int64_t ldr, int64_t nr, const float* Xc, int64_t ldc, int64_t nc,
             const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w, int64_t self_offset, double* out,
             void* ws, size_t ws_bytes, cudaStream_t st);
size_t grad_tc_workspace(int64_t nr, int64_t nc, int d, int ard, int w, bool sym = false);
int grad_tc(int family, int d, int ard, const float* Xr, int64_t ldr, int64_t nr, const float* Xc,
            int64_t ldc, int64_t nc, const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w,
            int64_t self_offset, double* out, void* ws, size_t ws_bytes, cudaStream_t st, bool sym = false);

static int grad_splits(int64_t nr, int64_t nc) {
  int64_t row_tiles = (nr + gBM - 1) / gBM;
  int64_t col_tiles = (nc + gBN - 1) / gBN;
  int64_t target = 2LL * num_sms();
  int64_t s = (target + row_tiles - 1) / row_tiles;
  s = std::min<int64_t>(s, 256);
  s = std::min<int64_t>(s, col_tiles);
  return (int)std::max<int64_t>(s, 1);
}

}  // namespace gp

using namespace gp;

extern "C" {

size_t gp_grad_forms_workspace_bytes(int64_t n_rows, int64_t n_cols, int d, int ard, int w) {
  // SIMT: blocks = row_tiles * S with S <= ceil(2*SMs / row_tiles)
  int64_t row_tiles = (n_rows + gBM - 1) / gBM;
  size_t simt = (size_t)((row_tiles + 2LL * num_sms() + 1) * 17) * sizeof(double);
  size_t tcw = grad_tc_supported(n_rows, n_cols, d, ard, w) ? grad_tc_workspace(n_rows, n_cols, d, ard, w, false) : 0;
  size_t gaw = ard && grad_ard_supported(n_rows, n_cols, d, w) ? grad_ard_workspace(n_rows, n_cols, d, w) : 0;
  simt = simt > tcw ? simt : tcw;
  return simt > gaw ? simt : gaw;
}

int gp_grad_forms(int family, int d, int ard, const float* Xr, int64_t ldr, int64_t n_rows,
                  const float* Xc, int64_t ldc, int64_t n_cols, double outputscale,
                  const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w,
                  int64_t self_offset, int algo, double* out, void* workspace,
                  size_t workspace_bytes, void* stream) {
  (void)outputscale;
  GP_REQUIRE(family == 0 || family == 1, "gp_grad_forms: family %d", family);
  GP_REQUIRE(d >= 1 && d <= 256 && w >= 1 && w <= 1024, "gp_grad_forms: d=%d w=%d", d, w);
  cudaStream_t st = (cudaStream_t)stream;
  int nparams = 1 + (ard ? d : 1);
  if (n_rows == 0 || n_cols == 0) {
    GP_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * nparams, st));
    return GP_OK;
  }
  // default: the per-entry tcgen05 epilogue (grad_tc.cu, fp32 differences);
  // ARD beyond its d + 2 <= 32 reach uses the tensor-core per-dimension sums
  // (grad_ard.cu: the expansion x_i^2 - 2 x_i x_j + x_j^2 in bf16 two-term
  // products loses digits to cancellation when lengthscales are short
  // relative to the data spread: 5.5e-3 of max|g| at C2,
  // scripts/c2_grad_check.py). algo 1 SIMT, 2 grad_tc, 3 grad_ard.
  const bool tc_ok = grad_tc_supported(n_rows, n_cols, d, ard, w);
  if (ard && (algo == 3 || (algo == 0 && !tc_ok)) && grad_ard_supported(n_rows, n_cols, d, w))
    return grad_ard(family, d, Xr, ldr, n_rows, Xc, ldc, n_cols, Y, ldy, R, ldrr, w, self_offset, out, workspace,
                    workspace_bytes, st);
  if (algo == 2 || (algo == 0 && tc_ok)) {
    GP_REQUIRE(tc_ok, "gp_grad_forms: shape unsupported by the tcgen05 kernel (d=%d w=%d)", d, w);
    return grad_tc(family, d, ard, Xr, ldr, n_rows, Xc, ldc, n_cols, Y, ldy, R, ldrr, w, self_offset, out,
                   workspace, workspace_bytes, st);
  }
  int S = grad_splits(n_rows, n_cols);
  int64_t col_tiles = (n_cols + gBN - 1) / gBN;
  int64_t tps = (col_tiles + S - 1) / S;
  S = (int)((col_tiles + tps - 1) / tps);
  unsigned gx = (unsigned)((n_rows + gBM - 1) / gBM);
  int64_t nblocks = (int64_t)gx * S;
  GP_REQUIRE(workspace_bytes >= (size_t)nblocks * 17 * sizeof(double),
             "gp_grad_forms: workspace too small (%zu < %zu)", workspace_bytes,
             (size_t)nblocks * 17 * sizeof(double));
  GradArgs a;
  a.Xr = Xr; a.ldr = ldr; a.nr = n_rows; a.Xc = Xc; a.ldc = ldc; a.nc = n_cols;
  a.d = d; a.ard = ard; a.Y = Y; a.ldy = ldy; a.R = R; a.ldrr = ldrr; a.w = w;
  a.cols_per_split = tps * gBN;
  a.partials = static_cast<double*>(workspace);
  int wp = (w + 3) & ~3;
  size_t smem = (size_t)(2 * d * 64 + 2 * wp * 64) * sizeof(float);
  int nchunks = ard ? (d + 15) / 16 : 1;
  for (int ch = 0; ch < nchunks; ++ch) {
    a.p0 = ch * 16;
    a.nlc = ard ? std::min(16, d - a.p0) : 1;
    a.with_s2 = ch == 0;
    int W;
    if (ard) {
      W = 17;
      auto kern = family == 0 ? grad_forms_kernel<0, 16> : grad_forms_kernel<1, 16>;
      GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3(gx, S), 256, smem, st>>>(a);
    } else {
      W = 2;
      auto kern = family == 0 ? grad_forms_kernel<0, 1> : grad_forms_kernel<1, 1>;
      GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      kern<<<dim3(gx, S), 256, smem, st>>>(a);
    }
    GP_LAUNCH_CHECK();
    grad_finalize<<<1, 32, 0, st>>>(a.partials, (int)nblocks, W, a.p0, a.nlc, a.with_s2, out);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

size_t gp_grad_forms_sym_workspace_bytes(int64_t n, int d, int ard, int w) {
  if (grad_tc_supported(n, n, d, ard, w)) return grad_tc_workspace(n, n, d, ard, w, true);
  return gp_grad_forms_workspace_bytes(n, n, d, ard, w);
}

int gp_grad_forms_sym_supported(int64_t n, int d, int ard, int w) {
  return n > 0 && grad_tc_supported(n, n, d, ard, w) ? 1 : 0;
}

int gp_grad_forms_sym(int family, int d, int ard, const float* X, int64_t ldx, int64_t n, double outputscale,
                      const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w, double* out,
                      void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(family == 0 || family == 1, "gp_grad_forms_sym: family %d", family);
  GP_REQUIRE(d >= 1 && d <= 256 && w >= 1 && w <= 1024, "gp_grad_forms_sym: d=%d w=%d", d, w);
  cudaStream_t st = (cudaStream_t)stream;
  if (n > 0 && grad_tc_supported(n, n, d, ard, w))
    return grad_tc(family, d, ard, X, ldx, n, X, ldx, n, Y, ldy, R, ldrr, w, 0, out, workspace, workspace_bytes, st,
                   true);
  // beyond the per-entry kernel's reach: the full square (same sum)
  return gp_grad_forms(family, d, ard, X, ldx, n, X, ldx, n, outputscale, Y, ldy, R, ldrr, w, 0, 0, out,
                       workspace, workspace_bytes, stream);
}

}  // extern "C"
