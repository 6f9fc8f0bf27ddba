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

#include <cooperative_groups.h>

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
  // two rows per 8-lane group and pass (rows i and i + ngrp), their global
  // loads and FMA chains interleaved: twice the loads in flight per lane (the
  // one-row form reached ~34 % of HBM at n = 10^6)
  for (int64_t i0 = r0; i0 < r1; i0 += 2 * ngrp) {   // warp-uniform trip count (shuffles below)
    double r2[2] = {0.0, 0.0}, dot[2] = {0.0, 0.0};
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + grp + u * ngrp;
      if (i < r1) {
        const double* xi = a.X + i * a.ldx;
        for (int q = g; q < a.d; q += 8) {
          double df = xi[q] - xp[q];
          r2[u] = fma(df, df, r2[u]);
        }
      }
    }
    {
      const int64_t ia = i0 + grp, ib = ia + ngrp;
      const bool ina = ia < r1, inb = ib < r1;
      const double* la = a.L + (ina ? ia : r0) * a.ldl;
      const double* lb = a.L + (inb ? ib : r0) * a.ldl;
      for (int m = g; m < j; m += 8) {
        const double pm = lp[m];
        if (ina) dot[0] = fma(la[m], pm, dot[0]);
        if (inb) dot[1] = fma(lb[m], pm, dot[1]);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
#pragma unroll
      for (int o = 1; o < 8; o <<= 1) {
        r2[u] += __shfl_xor_sync(0xffffffffu, r2[u], o);
        dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int64_t i = i0 + grp + u * ngrp;
      if (i < r1 && g == 0) {
        double row = a.s2 * kappa_f64(a.fam, r2[u]);
        double col = (row - dot[u]) * inv_sq;
        a.L[i * a.ldl + j] = col;
        double di = a.dres[i] - col * col;
        di = di > 0.0 ? di : 0.0;
        if (i == pj) di = 0.0;
        a.dres[i] = di;
        better(bv, bi, di, i);
      }
    }
  }
  block_argmax_store(bv, bi, a.pval, a.pidx);
}

__global__ void pivchol_finish(PivArgs a) {
  if (!*a.stop) a.info[0] = a.k;
}

// ---------------------------------------------------------------------------
// Small n: the whole factorisation in ONE launch on an 8-CTA cluster. Each
// step's argmax is combined over distributed shared memory (every CTA reads
// the 8 partials in rank order: the same pivot everywhere) and one cluster
// barrier (release / acquire, also ordering the global L writes) separates
// the steps, instead of two kernel launches per step (C1: 200 launches,
// ~1.9 ms). Per-row arithmetic is that of pivchol_step (8 lanes per row, same
// accumulation and shuffle order), so pivots and factor are identical.
// ---------------------------------------------------------------------------
constexpr int kPivCl = 8;
constexpr int kPivThreads = 1024;
constexpr int64_t kPivClusterMaxN = 65536;

__global__ void __cluster_dims__(kPivCl, 1, 1) __launch_bounds__(kPivThreads)
    pivchol_cluster(PivArgs a) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  extern __shared__ double sp[];           // 1 + d + k: pivot residual | x_p | L[p, :j]
  __shared__ double slot_v[2];
  __shared__ int64_t slot_i[2];
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t s_piv;
  __shared__ int s_stop;
  const int rank = (int)cl.block_rank();
  const int64_t per = (a.n + kPivCl - 1) / kPivCl;
  const int64_t r0 = min(a.n, (int64_t)rank * per), r1 = min(a.n, r0 + per);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
  auto reduce_store = [&](double bv, int64_t bi, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      better(bv, bi, ov, oi);
    }
    if (lane == 0) { sv[w] = bv; si[w] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double v = -INFINITY; int64_t i = INT64_MAX;
      for (int q = 0; q < (int)(blockDim.x >> 5); ++q) better(v, i, sv[q], si[q]);
      slot_v[slot] = v;
      slot_i[slot] = i;
    }
  };
  // init: residual diagonal s2, L zero; every row is a candidate
  {
    double bv = -INFINITY; int64_t bi = INT64_MAX;
    for (int64_t i = r0 + threadIdx.x; i < r1; i += blockDim.x) {
      a.dres[i] = a.s2;
      for (int m = 0; m < a.k; ++m) a.L[i * a.ldl + m] = 0.0;
      better(bv, bi, a.s2, i);
    }
    reduce_store(bv, bi, 1);
  }
  cl.sync();
  int j = 0;
  for (; j < a.k; ++j) {
    const int prev = (j + 1) & 1;   // slot written by the previous step (init: 1)
    if (w == 0) {
      // lane b reads CTA b's partial over DSMEM; the choice (largest, then
      // lowest index) is associative, so the shuffle tree gives the same pivot
      double v = -INFINITY; int64_t i = INT64_MAX;
      if (lane < kPivCl) {
        v = *cl.map_shared_rank(&slot_v[prev], lane);
        i = *cl.map_shared_rank(&slot_i[prev], lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
      }
      if (lane == 0) {
        s_stop = !(v > 0.0);
        s_piv = i;
        sp[0] = v;
        if (rank == 0 && !s_stop) a.piv[j] = i;
      }
    }
    __syncthreads();
    if (s_stop) break;   // uniform over the cluster: every CTA read the same partials
    const int64_t p = s_piv;
    for (int q = threadIdx.x; q < a.d; q += blockDim.x) sp[1 + q] = a.X[p * a.ldx + q];
    for (int m = threadIdx.x; m < j; m += blockDim.x) sp[1 + a.d + m] = a.L[p * a.ldl + m];
    __syncthreads();
    const double inv_sq = 1.0 / sqrt(sp[0]);
    const double* xp = sp + 1;
    const double* lp = sp + 1 + a.d;
    double bv = -INFINITY; int64_t bi = INT64_MAX;
    // RPG rows per 8-lane group and pass: their loads are independent and
    // issue together (the step is load-latency bound at small n)
    constexpr int RPG = 4;
    for (int64_t i0 = r0; i0 < r1; i0 += (int64_t)ngrp * RPG) {
      double r2[RPG], dot[RPG];
#pragma unroll
      for (int u = 0; u < RPG; ++u) {
        const int64_t i = i0 + grp + (int64_t)u * ngrp;
        r2[u] = 0.0;
        dot[u] = 0.0;
        if (i < r1) {
          const double* xi = a.X + i * a.ldx;
          for (int q = g; q < a.d; q += 8) {
            double df = xi[q] - xp[q];
            r2[u] = fma(df, df, r2[u]);
          }
          const double* li = a.L + i * a.ldl;
          for (int m = g; m < j; m += 8) dot[u] = fma(li[m], lp[m], dot[u]);
        }
      }
#pragma unroll
      for (int u = 0; u < RPG; ++u) {
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          r2[u] += __shfl_xor_sync(0xffffffffu, r2[u], o);
          dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
        }
        const int64_t i = i0 + grp + (int64_t)u * ngrp;
        if (i < r1 && g == 0) {
          double row = a.s2 * kappa_f64(a.fam, r2[u]);
          double col = (row - dot[u]) * inv_sq;
          a.L[i * a.ldl + j] = col;
          double di = a.dres[i] - col * col;
          di = di > 0.0 ? di : 0.0;
          if (i == p) di = 0.0;
          a.dres[i] = di;
          better(bv, bi, di, i);
        }
      }
    }
    reduce_store(bv, bi, j & 1);
    cl.sync();   // release / acquire: L[:, j], dres and the slots visible cluster-wide
  }
  if (rank == 0 && threadIdx.x == 0) a.info[0] = j;
}

// Smaller still (rows per CTA x (k + d + 1) doubles within SMEM): a 16-CTA
// cluster keeps its rows of L, X and the residual diagonal in shared memory
// for the whole factorisation; the pivot's point and L row come from the
// owning CTA over DSMEM. Same per-row arithmetic as pivchol_step.
constexpr int kPivCl16 = 16;

__host__ __device__ inline int piv_lds(int k) { return k | 1; }   // odd row stride: fewer bank conflicts

__global__ void __launch_bounds__(kPivThreads) pivchol_cluster_smem(PivArgs a, int rpc) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  extern __shared__ __align__(16) double smd[];
  const int lds = piv_lds(a.k);
  double* Ls = smd;                                // [rpc][lds]
  double* Xs = Ls + (size_t)rpc * lds;             // [rpc][d]
  double* ds = Xs + (size_t)rpc * a.d;             // [rpc]
  double* sp = ds + rpc;                           // 1 + d + k
  __shared__ double slot_v[2];
  __shared__ int64_t slot_i[2];
  __shared__ double sv[32];
  __shared__ int64_t si[32];
  __shared__ int64_t s_piv;
  __shared__ int s_stop;
  const int rank = (int)cl.block_rank(), ncl = (int)cl.num_blocks();
  const int64_t r0 = min(a.n, (int64_t)rank * rpc), r1 = min(a.n, r0 + rpc);
  const int nr = (int)(r1 - r0);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int g = threadIdx.x & 7, grp = threadIdx.x >> 3, ngrp = blockDim.x >> 3;
  for (int p = threadIdx.x; p < rpc * lds; p += blockDim.x) Ls[p] = 0.0;
  for (int p = threadIdx.x; p < nr * a.d; p += blockDim.x) {
    const int r = p / a.d, q = p - r * a.d;
    Xs[p] = a.X[(r0 + r) * a.ldx + q];
  }
  double bv = -INFINITY; int64_t bi = INT64_MAX;
  for (int r = threadIdx.x; r < rpc; r += blockDim.x) {
    ds[r] = a.s2;
    if (r < nr) better(bv, bi, a.s2, r0 + r);
  }
  auto reduce_store = [&](double v, int64_t i, int slot) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, v, o);
      int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
      better(v, i, ov, oi);
    }
    if (lane == 0) { sv[w] = v; si[w] = i; }
    __syncthreads();
    if (w == 0) {   // the warp partials, reduced by warp 0 (same choice in any order)
      double x = lane < (int)(blockDim.x >> 5) ? sv[lane] : -INFINITY;
      int64_t y = lane < (int)(blockDim.x >> 5) ? si[lane] : INT64_MAX;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ox = __shfl_xor_sync(0xffffffffu, x, o);
        int64_t oy = __shfl_xor_sync(0xffffffffu, y, o);
        better(x, y, ox, oy);
      }
      if (lane == 0) {
        slot_v[slot] = x;
        slot_i[slot] = y;
      }
    }
  };
  reduce_store(bv, bi, 1);
  cl.sync();
  int j = 0;
  for (; j < a.k; ++j) {
    const int prev = (j + 1) & 1;
    if (w == 0) {
      double v = -INFINITY; int64_t i = INT64_MAX;
      if (lane < ncl) {
        v = *cl.map_shared_rank(&slot_v[prev], lane);
        i = *cl.map_shared_rank(&slot_i[prev], lane);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        double ov = __shfl_xor_sync(0xffffffffu, v, o);
        int64_t oi = __shfl_xor_sync(0xffffffffu, i, o);
        better(v, i, ov, oi);
      }
      // every lane holds the choice: warp 0 also fetches the pivot's point
      // and L row from the owning CTA, so one block barrier serves both
      if (v > 0.0) {
        const int owner = (int)(i / rpc), lr = (int)(i - (int64_t)owner * rpc);
        const double* xo = cl.map_shared_rank(Xs, owner) + (size_t)lr * a.d;
        const double* lo = cl.map_shared_rank(Ls, owner) + (size_t)lr * lds;
        // up to 4 x 32 values: the remote loads issue together, then the stores
        double pv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = lane + 32 * u;
          pv[u] = q < a.d + j ? (q < a.d ? xo[q] : lo[q - a.d]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (lane + 32 * u < a.d + j) sp[1 + lane + 32 * u] = pv[u];
        for (int q = lane + 128; q < a.d + j; q += 32) sp[1 + q] = q < a.d ? xo[q] : lo[q - a.d];
      }
      if (lane == 0) {
        s_stop = !(v > 0.0);
        s_piv = i;
        sp[0] = v;
        if (rank == 0 && !s_stop) a.piv[j] = i;
      }
    }
    __syncthreads();
    if (s_stop) break;
    const int64_t p = s_piv;
    const double inv_sq = 1.0 / sqrt(sp[0]);
    const double* xp = sp + 1;
    const double* lp = sp + 1 + a.d;
    bv = -INFINITY; bi = INT64_MAX;
    // two rows per 8-lane group and pass, their SMEM loads and FMA chains
    // interleaved (the step is latency bound at small n)
    for (int r = grp; r - grp < nr; r += 2 * ngrp) {   // warp-uniform trip count (shuffles)
      double r2[2] = {0.0, 0.0}, dot[2] = {0.0, 0.0};
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ru = r + u * ngrp;
        if (ru < nr) {
          const double* xi = Xs + (size_t)ru * a.d;
          for (int q = g; q < a.d; q += 8) {
            double df = xi[q] - xp[q];
            r2[u] = fma(df, df, r2[u]);
          }
        }
      }
      {
        const bool in0 = r < nr, in1 = r + ngrp < nr;
        const double* l0 = Ls + (size_t)r * lds;
        const double* l1 = Ls + (size_t)(r + ngrp) * lds;
        for (int m = g; m < j; m += 8) {
          const double pm = lp[m];
          if (in0) dot[0] = fma(l0[m], pm, dot[0]);
          if (in1) dot[1] = fma(l1[m], pm, dot[1]);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
#pragma unroll
        for (int o = 1; o < 8; o <<= 1) {
          r2[u] += __shfl_xor_sync(0xffffffffu, r2[u], o);
          dot[u] += __shfl_xor_sync(0xffffffffu, dot[u], o);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int ru = r + u * ngrp;
        if (ru < nr && g == 0) {
          const int64_t i = r0 + ru;
          double row = a.s2 * kappa_f64(a.fam, r2[u]);
          double col = (row - dot[u]) * inv_sq;
          Ls[(size_t)ru * lds + j] = col;
          double di = ds[ru] - col * col;
          di = di > 0.0 ? di : 0.0;
          if (i == p) di = 0.0;
          ds[ru] = di;
          better(bv, bi, di, i);
        }
      }
    }
    reduce_store(bv, bi, j & 1);
    cl.sync();   // the step's L column, residuals and argmax slots visible cluster-wide
  }
  // the factor and residual diagonal out to global memory (coalesced)
  for (int p = threadIdx.x; p < nr * a.k; p += blockDim.x) {
    const int r = p / a.k, m = p - r * a.k;
    a.L[(r0 + r) * a.ldl + m] = Ls[(size_t)r * lds + m];
  }
  for (int r = threadIdx.x; r < nr; r += blockDim.x) a.dres[r0 + r] = ds[r];
  if (rank == 0 && threadIdx.x == 0) a.info[0] = j;
  cl.sync();   // no CTA exits while another may still read its SMEM
}

static size_t piv_smem16(int64_t n, int d, int k) {
  const int64_t rpc = (n + kPivCl16 - 1) / kPivCl16;
  return (size_t)(rpc * (piv_lds(k) + d + 1) + 1 + d + k) * sizeof(double);
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
  // small n x k: the SMEM-resident 16-CTA cluster (non-portable size; if the
  // launch is refused the 8-CTA global-memory cluster below takes it)
  const size_t smem16 = piv_smem16(n, d, k);
  if (smem16 + 1024 <= 227 * 1024) {
    cudaFuncSetAttribute(pivchol_cluster_smem, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(pivchol_cluster_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem16);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kPivCl16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.gridDim = dim3(kPivCl16); cfg.blockDim = dim3(kPivThreads);
    cfg.dynamicSmemBytes = smem16; cfg.stream = st; cfg.attrs = at; cfg.numAttrs = 1;
    const int rpc = (int)((n + kPivCl16 - 1) / kPivCl16);
    if (cudaLaunchKernelEx(&cfg, pivchol_cluster_smem, a, rpc) == cudaSuccess) {
      GP_LAUNCH_CHECK();
      return GP_OK;
    }
    cudaGetLastError();
  }
  if (n <= kPivClusterMaxN) {
    const size_t smem = sizeof(double) * (1 + d + k);
    if (smem > 48 * 1024)
      GP_CUDA_TRY(cudaFuncSetAttribute(pivchol_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    pivchol_cluster<<<kPivCl, kPivThreads, smem, st>>>(a);
    GP_LAUNCH_CHECK();
    return GP_OK;
  }
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
