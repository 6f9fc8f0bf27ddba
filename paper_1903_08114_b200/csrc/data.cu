// Device-side data preparation for the training protocol (sm_100a):
// column moments over a row subset, standardisation, row gathers.
//
// Reference: data.py:163-196 (split_and_whiten: feature / target mean and
// population std over the TRAINING rows, zero std -> 1, every row
// standardised), trainer.py:323-330 (the pretraining subset X[idx], y[idx]).
// HBM-bound byte work: one coalesced pass per moment, fixed-order block
// partials (deterministic run to run), fp64 throughout like numpy.
#include "gp_common.cuh"

#include <algorithm>

namespace gp {

constexpr int kDT = 256;

// rows of this block: [r0, r1) of the m selected rows (row i of the subset is
// X row rows[i], or i itself when rows == nullptr)
__device__ __forceinline__ int64_t sel_row(const int64_t* rows, int64_t i) { return rows ? rows[i] : i; }

// pass 0: partial column sums of x; pass 1: partial sums of (x - mean)^2
// layout: thread = (row lane, column) with consecutive threads on consecutive
// columns of a row, so a warp reads contiguous row segments
__global__ void __launch_bounds__(kDT) col_moment_kernel(const double* __restrict__ X, int64_t ldx,
                                                         const int64_t* __restrict__ rows, int64_t m, int d,
                                                         const double* __restrict__ mean, double* partials) {
  __shared__ double sred[kDT];
  const int64_t per = (m + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = min(m, (int64_t)blockIdx.x * per), r1 = min(m, r0 + per);
  for (int c0 = 0; c0 < d; c0 += kDT) {
    const int tw = min(kDT, d - c0);
    const int rpp = kDT / tw;
    const int tc = threadIdx.x % tw, tr = threadIdx.x / tw;
    double acc = 0.0;
    if (tr < rpp) {
      const double mu = mean ? mean[c0 + tc] : 0.0;
      for (int64_t i = r0 + tr; i < r1; i += rpp) {
        const double x = X[sel_row(rows, i) * ldx + c0 + tc];
        if (mean) {
          const double dx = x - mu;
          acc = fma(dx, dx, acc);
        } else {
          acc += x;
        }
      }
    }
    sred[threadIdx.x] = acc;
    __syncthreads();
    if ((int)threadIdx.x < tw) {
      double s = 0.0;
      for (int q = 0; q < rpp; ++q) s += sred[threadIdx.x + q * tw];
      partials[(int64_t)blockIdx.x * d + c0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// out[c] = sum_b partials[b][c] / m (pass 0: mean); pass 1: sqrt(. / m), and
// a zero std becomes 1 when unit_if_zero (data.py:184-189)
__global__ void col_moment_finish(const double* __restrict__ partials, int nb, int d, int64_t m, int pass,
                                  int unit_if_zero, double* out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= d) return;
  double s = 0.0;
  for (int b = 0; b < nb; ++b) s += partials[(int64_t)b * d + c];
  double v = s / (double)m;
  if (pass == 1) {
    v = sqrt(v);
    if (unit_if_zero && v == 0.0) v = 1.0;
  }
  out[c] = v;
}

__global__ void standardize_kernel(const double* __restrict__ X, int64_t ldx, int64_t n, int d,
                                   const double* __restrict__ mean, const double* __restrict__ std_,
                                   double* out, int64_t ldo) {
  const int64_t tot = n * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / d;
    const int c = (int)(e - r * d);
    out[r * ldo + c] = (X[r * ldx + c] - mean[c]) / std_[c];
  }
}

__global__ void gather_kernel(const double* __restrict__ X, int64_t ldx, const int64_t* __restrict__ idx,
                              int64_t m, int d, int64_t n_src, double* out, int64_t ldo, int* bad) {
  const int64_t tot = m * d;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / d;
    const int c = (int)(e - i * d);
    const int64_t r = idx[i];
    if (r < 0 || r >= n_src) {
      *bad = 1;
      continue;
    }
    out[i * ldo + c] = X[r * ldx + c];
  }
}

static int moment_blocks(int64_t m) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(2LL * num_sms(), (m + 255) / 256));
}

}  // namespace gp

using namespace gp;

extern "C" {

int64_t gp_column_moments_workspace_len(int64_t m, int d) { return (int64_t)moment_blocks(m) * d; }

int gp_column_moments(const double* X, int64_t ldx, int64_t m, int d, const int64_t* rows, double* mean,
                      double* std_out, int unit_if_zero, double* workspace, int64_t workspace_len, void* stream) {
  GP_REQUIRE(m >= 1 && d >= 1 && ldx >= d, "gp_column_moments: m=%lld d=%d ldx=%lld", (long long)m, d,
             (long long)ldx);
  const int nb = moment_blocks(m);
  GP_REQUIRE(workspace_len >= (int64_t)nb * d, "gp_column_moments: workspace %lld < %lld",
             (long long)workspace_len, (long long)nb * d);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned fb = (unsigned)((d + 127) / 128);
  col_moment_kernel<<<nb, kDT, 0, st>>>(X, ldx, rows, m, d, nullptr, workspace);
  GP_LAUNCH_CHECK();
  col_moment_finish<<<fb, 128, 0, st>>>(workspace, nb, d, m, 0, 0, mean);
  GP_LAUNCH_CHECK();
  if (std_out) {
    col_moment_kernel<<<nb, kDT, 0, st>>>(X, ldx, rows, m, d, mean, workspace);
    GP_LAUNCH_CHECK();
    col_moment_finish<<<fb, 128, 0, st>>>(workspace, nb, d, m, 1, unit_if_zero, std_out);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

int gp_standardize(const double* X, int64_t ldx, int64_t n, int d, const double* mean, const double* std_in,
                   double* out, int64_t ldo, void* stream) {
  GP_REQUIRE(n >= 0 && d >= 1 && ldx >= d && ldo >= d, "gp_standardize: n=%lld d=%d", (long long)n, d);
  if (n == 0) return GP_OK;
  const int64_t tot = n * d;
  const int nb = (int)std::min<int64_t>((tot + 255) / 256, 8LL * num_sms());
  standardize_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(X, ldx, n, d, mean, std_in, out, ldo);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int gp_gather_rows(const double* X, int64_t ldx, int64_t n_src, const int64_t* idx, int64_t m, int d, double* out,
                   int64_t ldo, int* bad_dev, void* stream) {
  GP_REQUIRE(m >= 0 && d >= 1 && ldx >= d && ldo >= d, "gp_gather_rows: m=%lld d=%d", (long long)m, d);
  if (m == 0) return GP_OK;
  const int64_t tot = m * d;
  const int nb = (int)std::min<int64_t>((tot + 255) / 256, 8LL * num_sms());
  gather_kernel<<<nb, 256, 0, (cudaStream_t)stream>>>(X, ldx, idx, m, d, n_src, out, ldo, bad_dev);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

}  // extern "C"
