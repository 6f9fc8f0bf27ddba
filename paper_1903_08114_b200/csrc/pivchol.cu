// Greedy rank-k pivoted Cholesky of the noiseless kernel matrix, fp64.
//
// Reference: precond.py:58-98 (partial_pivoted_cholesky) driven by
// likelihood.py:74-91 (row oracle = noiseless kernel row, diagonal = s2).
//   i = argmax d (first index on ties); stop if d_i <= 0
//   col = (k(x_i, X) - L[:, :j] L[i, :j]) / sqrt(d_i); L[:, j] = col
//   d -= col^2; d = max(d, 0); d_i = 0
// Every step runs as two stream-ordered launches (select, step) that read the
// pivot from device memory: no host synchronisation inside the factorisation.
#include "gp_common.cuh"

#include <algorithm>

namespace gp {

struct PivArgs {
  int fam; int d; const double* X; int64_t ldx; int64_t n; double s2; int k;
  double* L; int64_t ldl; int64_t* piv; double* dres; int* info;
  double* pval; int64_t* pidx; double* pinfo; int* stop; int nb;
};

__device__ __forceinline__ void better(double& bv, int64_t& bi, double v, int64_t i) {
  // larger value wins; equal values -> lower index (np.argmax semantics);
  // NaN never wins
  if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
}

__device__ void block_argmax_store(double bv, int64_t bi, double* pval, int64_t* pidx) {
  __shared__ double sv[32];
  __shared__ int64_t si[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double v = -INFINITY; int64_t i = INT64_MAX;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) better(v, i, sv[q], si[q]);
    pval[blockIdx.x] = v;
    pidx[blockIdx.x] = i;
  }
}

__global__ void pivchol_init(PivArgs a) {
  int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(a.n, r0 + per);
  double bv = -INFINITY; int64_t bi = INT64_MAX;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
    a.dres[i] = a.s2;
    for (int m = 0; m < a.k; ++m) a.L[i * a.ldl + m] = 0.0;
    better(bv, bi, a.s2, i);
  }
  block_argmax_store(bv, bi, a.pval, a.pidx);
  if (blockIdx.x == 0 && threadIdx.x == 0) { *a.stop = 0; a.info[0] = 0; }
}

// choose pivot j from the block partials and stage its data
// argmax of the per-block partials (largest residual, lowest index on ties:
// an associative choice, so the tree order cannot change the pivot), then the
// pivot's point and L row into pinfo for the step kernel
__global__ void pivchol_select(PivArgs a, int j) {
  if (*a.stop) return;
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t s_piv;
  __shared__ int s_stop;
  double bv = -INFINITY; int64_t bi = INT64_MAX;
  for (int b = threadIdx.x; b < a.nb; b += blockDim.x) better(bv, bi, a.pval[b], a.pidx[b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, ov, oi);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { sv[w] = bv; si[w] = bi; }
  __syncthreads();
  if (w == 0) {
    const int nw = (int)(blockDim.x >> 5);
    bv = lane < nw ? sv[lane] : -INFINITY;
    bi = lane < nw ? si[lane] : INT64_MAX;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      better(bv, bi, ov, oi);
    }
    if (lane == 0) {
      if (!(bv > 0.0)) {  // residual mass exhausted: stop at rank j
        *a.stop = 1;
        a.info[0] = j;
        s_stop = 1;
      } else {
        a.piv[j] = bi;
        a.pinfo[0] = bv;
        s_stop = 0;
      }
      s_piv = bi;
    }
  }
  __syncthreads();
  if (s_stop) return;
  const int64_t p = s_piv;
  for (int q = threadIdx.x; q < a.d; q += blockDim.x) a.pinfo[1 + q] = a.X[p * a.ldx + q];
  for (int m = threadIdx.x; m < j; m += blockDim.x) a.pinfo[1 + a.d + m] = a.L[p * a.ldl + m];
}

// one step of the greedy factorisation over this block's rows. L is n x k
// row-major, so a thread per row would read its row with a 8*ldl-byte stride
// across the warp; instead 8 lanes share a row (coalesced 64-byte reads of
// L[i, :j] and X[i, :]) and combine their partial sums with shuffles.
__global__ void pivchol_step(PivArgs a, int j) {
  if (*a.stop) return;
  extern __shared__ double sp[];  // pinfo copy: 1 + d + j
  for (int q = threadIdx.x; q < 1 + a.d + j; q += blockDim.x) sp[q] = a.pinfo[q];
  __syncthreads();
  const double inv_sq = 1.0 / sqrt(sp[0]);
  const double* xp = sp + 1;
  const double* lp = sp + 1 + a.d;
  const int64_t pj = a.piv[j];
  int64_t per = (a.n + gridDim.x - 1) / gridDim.x;
  int64_t r0 = (int64_t)blockIdx.x * per, r1 = min(a.n, r0 + per);
  const int g = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
  double bv = -INFINITY; int64_t bi = INT64_MAX;
  for (int64_t i0 = r0; i0 < r1; i0 += ngrp) {   // warp-uniform trip count (shuffles below)
    const int64_t i = i0 + grp;
    const bool in = i < r1;
    double r2 = 0.0, dot = 0.0;
    if (in) {
      const double* xi = a.X + i * a.ldx;
      for (int q = g; q < a.d; q += 8) {
        double df = xi[q] - xp[q];
        r2 = fma(df, df, r2);
      }
      const double* li = a.L + i * a.ldl;
      for (int m = g; m < j; m += 8) dot = fma(li[m], lp[m], dot);
    }
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) {
      r2 += __shfl_xor_sync(0xffffffffu, r2, o);
      dot += __shfl_xor_sync(0xffffffffu, dot, o);
    }
    if (in && g == 0) {
      double row = a.s2 * kappa_f64(a.fam, r2);
      double col = (row - dot) * inv_sq;
      a.L[i * a.ldl + j] = col;
      double di = a.dres[i] - col * col;
      di = di > 0.0 ? di : 0.0;
      if (i == pj) di = 0.0;
      a.dres[i] = di;
      better(bv, bi, di, i);
    }
  }
  block_argmax_store(bv, bi, a.pval, a.pidx);
}

__global__ void pivchol_finish(PivArgs a) {
  if (!*a.stop) a.info[0] = a.k;
}

// row blocks of >= 64 rows (two passes of the 32 row groups of a block), at
// most 1024 of them (the select kernel's single block reduces their partials):
// small n spreads over many SMs instead of a few long blocks
static int piv_nb(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(1024, (n + 63) / 64));
}

}  // namespace gp

using namespace gp;

extern "C" {

size_t gp_pivchol_workspace_bytes(int64_t n, int k) {
  int nb = piv_nb(n);
  return (size_t)nb * (sizeof(double) + sizeof(int64_t)) + (size_t)(1 + 256 + k) * sizeof(double) + 64;
}

int gp_pivchol(int family, int d, const double* Xs64, int64_t ldx, int64_t n, double outputscale,
               int k, double* L, int64_t ldl, int64_t* pivots_dev, double* resid_diag,
               int32_t* info_dev, void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(family == 0 || family == 1, "gp_pivchol: family %d", family);
  GP_REQUIRE(n >= 1 && k >= 1 && k <= n, "rank must satisfy 1 <= k <= %lld, got %d", (long long)n, k);
  GP_REQUIRE(d >= 1 && d <= 256, "gp_pivchol: d=%d", d);
  GP_REQUIRE(ldl >= k, "gp_pivchol: ldl < k");
  GP_REQUIRE(workspace_bytes >= gp_pivchol_workspace_bytes(n, k), "gp_pivchol: workspace too small");
  cudaStream_t st = (cudaStream_t)stream;
  PivArgs a;
  a.fam = family; a.d = d; a.X = Xs64; a.ldx = ldx; a.n = n; a.s2 = outputscale; a.k = k;
  a.L = L; a.ldl = ldl; a.piv = pivots_dev; a.dres = resid_diag; a.info = info_dev;
  a.nb = piv_nb(n);
  char* w = static_cast<char*>(workspace);
  a.pval = reinterpret_cast<double*>(w); w += sizeof(double) * a.nb;
  a.pidx = reinterpret_cast<int64_t*>(w); w += sizeof(int64_t) * a.nb;
  a.pinfo = reinterpret_cast<double*>(w); w += sizeof(double) * (1 + 256 + k);
  a.stop = reinterpret_cast<int*>(w);
  pivchol_init<<<a.nb, 256, 0, st>>>(a);
  GP_LAUNCH_CHECK();
  size_t smem_max = sizeof(double) * (1 + d + k);
  if (smem_max > 48 * 1024)
    GP_CUDA_TRY(cudaFuncSetAttribute(pivchol_step, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
  for (int j = 0; j < k; ++j) {
    pivchol_select<<<1, 1024, 0, st>>>(a, j);
    GP_LAUNCH_CHECK();
    pivchol_step<<<a.nb, 256, sizeof(double) * (1 + d + j), st>>>(a, j);
    GP_LAUNCH_CHECK();
  }
  pivchol_finish<<<1, 1, 0, st>>>(a);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

}  // extern "C"
