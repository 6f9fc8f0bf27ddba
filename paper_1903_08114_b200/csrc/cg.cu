// mBCG phases, deterministic column reductions, low-rank products, and the
// preconditioner's inner factorisation.
//
// Reference semantics: cg.py:84-164 (mbcg_solve: per-column freeze on the
// recurrence residual ||r||/||b||, alpha/beta recorded per active column),
// precond.py:101-139 (Woodbury apply), :165-174 (tr P^{-1}).
//
// All reductions are fixed-order: every block reduces a contiguous row range
// in a fixed thread order into partials[block][slot]; a finalize kernel sums
// the blocks in index order. Results are therefore run-to-run deterministic.
#include "tc_common.cuh"

#include <algorithm>

namespace gp {

constexpr int kRT = 256;  // threads per row-block kernel

__device__ __forceinline__ void row_range(int64_t n, int64_t& r0, int64_t& r1) {
  int64_t per = (n + gridDim.x - 1) / gridDim.x;
  r0 = (int64_t)blockIdx.x * per;
  r1 = min(n, r0 + per);
}

// Per-column sums over this block's rows of f(row, col); writes
// out[c] for c < t. Thread layout: consecutive threads = consecutive columns
// of a row (coalesced on row-major blocks).
template <class F>
__device__ void block_colsum(int64_t r0, int64_t r1, int t, F f, double* out, double* sred) {
  for (int c0 = 0; c0 < t; c0 += kRT) {
    int tw = min(kRT, t - c0);
    int rpp = kRT / tw;
    int tc = threadIdx.x % tw, tr = threadIdx.x / tw;
    double acc = 0.0;
    if (tr < rpp)
      for (int64_t r = r0 + tr; r < r1; r += rpp) acc += f(r, c0 + tc);
    sred[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x < tw) {
      double s = 0.0;
      for (int q = 0; q < rpp; ++q) s += sred[threadIdx.x + q * tw];
      out[c0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
}

// rows [rc, rc + R) x columns [0, CP) of a row-major global matrix into SMEM
// (zero outside nr x cols): warp w takes rows w, w + nwarps, ..., lane l the
// columns l, l + 32, ...: coalesced loads, no index division, several loads
// in flight per thread. transpose: dst[c * dld + r], else dst[r * dld + c].
template <bool TRANSPOSE>
__device__ __forceinline__ void stage_rows(const double* __restrict__ M, int64_t ld, int64_t rc, int nr, int cols,
                                           int R, int CP, double* dst, int dld) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
#pragma unroll 4
  for (int r = w; r < R; r += nw) {
    for (int c = l; c < CP; c += 32) {
      const double v = (r < nr && c < cols) ? M[(rc + r) * ld + c] : 0.0;
      dst[TRANSPOSE ? c * dld + r : r * dld + c] = v;
    }
  }
}

// out[kk*t + c] (per block) = sum_{rows} L[r,kk] * A[r,c]
// Narrow blocks (k <= 128, t <= 16, the CG width): 32-row chunks of L and A
// staged in SMEM with coalesced loads, each thread accumulating a 4 x 4
// (kk x c) register tile over its row group, groups combined in a fixed
// order: every L row is read once per product and the FMA:SMEM-load ratio is
// 2:1 (the one-output-per-thread form re-read L per output and ran at ~10 %
// of HBM). Other shapes: the generic form. `sm` is a scratch of
// ltmul_scratch(k, t) doubles.
constexpr int kLtCR = 32;
__host__ __device__ inline bool ltmul_tiled(int k, int t) { return k <= 128 && t <= 16; }
__host__ __device__ inline int ltmul_scratch(int k, int t) {
  if (ltmul_tiled(k, t)) {
    const int KP = (k + 3) / 4 * 4, TP = (t + 3) / 4 * 4;
    const int stage = 2 * kLtCR * (KP + TP), red = 256 * 16;
    return (stage > red ? stage : red) + 2;   // + the two chunk mbarriers
  }
  return 16 * (k > 1 ? k : 1) + 16 * t;
}
__device__ __forceinline__ void cp_async8z(uint32_t dst, const void* src, bool in) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(in ? 8u : 0u) : "memory");
}
__device__ void block_ltmul(int64_t r0, int64_t r1, int k, int t, const double* __restrict__ L,
                            int64_t ldl, const double* __restrict__ A, int64_t lda, double* out,
                            double* sm, const int* colmask) {
  if (ltmul_tiled(k, t)) {
    const int KQ = (k + 3) / 4, TQ = (t + 3) / 4, KP = 4 * KQ, TP = 4 * TQ;
    const int units = KQ * TQ;                 // <= 128
    const int G = kRT / units;                 // row groups (>= 2)
    const int u = threadIdx.x % units, g = threadIdx.x / units;
    const int kq = u / TQ, tq = u - (u / TQ) * TQ;
    const int stage = kLtCR * (KP + TP);       // one buffer: [kLtCR][KP] L rows, [kLtCR][TP] A rows
    const int w = threadIdx.x >> 5, ln = threadIdx.x & 31, nw = kRT >> 5;
    // chunk copies (8-byte cp.async, zero-filled outside the rows / columns),
    // double buffered so the next chunk streams in during this one's FMAs
    // contiguous L with k % 4 == 0 (rows of KP = k doubles, 32-byte aligned
    // chunks): each chunk of L rows is ONE cp.async.bulk (TMA) issued by
    // thread 0 and completed on an mbarrier, instead of 8-byte copies by
    // every thread; rows past the end are never read, so no zero fill
    const bool bulk = ldl == k && KP == k;
    const int mb_off = 2 * stage > 256 * 16 ? 2 * stage : 256 * 16;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + mb_off);
    if (bulk && threadIdx.x == 0) {
      tc::mbar_init(tc::smem_u32(&bar[0]), 1);
      tc::mbar_init(tc::smem_u32(&bar[1]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    auto issue = [&](int64_t rc, int b) {
      const int nr = (int)min((int64_t)kLtCR, r1 - rc);
      const uint32_t bl = (uint32_t)__cvta_generic_to_shared(sm + (size_t)b * stage);
      const uint32_t ba = bl + (uint32_t)(kLtCR * KP * 8);
      if (bulk) {
        if (threadIdx.x == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          const uint32_t bytes = (uint32_t)(nr * k * 8);
          tc::mbar_expect_tx(tc::smem_u32(&bar[b]), bytes);
          tc::bulk_g2s(bl, L + rc * k, bytes, tc::smem_u32(&bar[b]));
        }
      }
      for (int r = w; r < kLtCR; r += nw) {
        const bool rin = r < nr;
        const double* lr = L + (rin ? (rc + r) * ldl : 0);
        const double* ar = A + (rin ? (rc + r) * lda : 0);
        if (!bulk)
          for (int c = ln; c < KP; c += 32) cp_async8z(bl + (uint32_t)((r * KP + c) * 8), lr + (rin && c < k ? c : 0), rin && c < k);
        for (int c = ln; c < TP; c += 32) cp_async8z(ba + (uint32_t)((r * TP + c) * 8), ar + (rin && c < t ? c : 0), rin && c < t);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    __syncthreads();   // the caller's writes of A (and prior use of sm) are complete
    int b = 0, ci = 0;
    if (bulk) __syncthreads();   // barriers initialised before the first copy completes on them
    if (r0 < r1) issue(r0, 0);
    for (int64_t rc = r0; rc < r1; rc += kLtCR, b ^= 1, ++ci) {
      const int nr = (int)min((int64_t)kLtCR, r1 - rc);
      if (rc + kLtCR < r1) {
        issue(rc + kLtCR, b ^ 1);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
      if (bulk) tc::mbar_wait(tc::smem_u32(&bar[b]), (ci >> 1) & 1);
      __syncthreads();
      const double* sLc = sm + (size_t)b * stage;
      const double* sAc = sLc + kLtCR * KP;
      if (g < G) {
        for (int r = g; r < nr; r += G) {
          const double2 la = *reinterpret_cast<const double2*>(sLc + r * KP + 4 * kq);
          const double2 lb = *reinterpret_cast<const double2*>(sLc + r * KP + 4 * kq + 2);
          const double2 aa = *reinterpret_cast<const double2*>(sAc + r * TP + 4 * tq);
          const double2 ab = *reinterpret_cast<const double2*>(sAc + r * TP + 4 * tq + 2);
          const double l[4] = {la.x, la.y, lb.x, lb.y}, a[4] = {aa.x, aa.y, ab.x, ab.y};
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fma(l[i], a[j], acc[i][j]);
        }
      }
      __syncthreads();   // buffer b is refilled by the issue two chunks on
    }
    // groups in index order (deterministic): red[g][u][16]
    if (g < G) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) sm[((size_t)g * units + u) * 16 + 4 * i + j] = acc[i][j];
    }
    __syncthreads();
    for (int p = threadIdx.x; p < k * t; p += kRT) {
      const int kk = p / t, c = p - kk * t;
      const int uu = (kk >> 2) * TQ + (c >> 2), slot = 4 * (kk & 3) + (c & 3);
      double v = 0.0;
      for (int q = 0; q < G; ++q) v += sm[((size_t)q * units + uu) * 16 + slot];
      out[p] = (colmask && !colmask[c]) ? 0.0 : v;
    }
    __syncthreads();
    return;
  }
  constexpr int CR = 16, PPT = 8;
  double* sL = sm;
  double* sA = sm + 16 * (k > 1 ? k : 1);
  const int KT = k * t;
  for (int p0 = 0; p0 < KT; p0 += kRT * PPT) {
    double acc[PPT];
#pragma unroll
    for (int m = 0; m < PPT; ++m) acc[m] = 0.0;
    for (int64_t rc = r0; rc < r1; rc += CR) {
      int nr = (int)min((int64_t)CR, r1 - rc);
      __syncthreads();
      for (int idx = threadIdx.x; idx < nr * k; idx += kRT) {
        int r = idx / k, kk = idx - r * k;
        sL[r * k + kk] = L[(rc + r) * ldl + kk];
      }
      for (int idx = threadIdx.x; idx < nr * t; idx += kRT) {
        int r = idx / t, c = idx - r * t;
        sA[r * t + c] = A[(rc + r) * lda + c];
      }
      __syncthreads();
#pragma unroll
      for (int m = 0; m < PPT; ++m) {
        int p = p0 + threadIdx.x + m * kRT;
        if (p < KT) {
          int kk = p / t, c = p - kk * t;
          double s = acc[m];
          for (int r = 0; r < nr; ++r) s = fma(sL[r * k + kk], sA[r * t + c], s);
          acc[m] = s;
        }
      }
    }
#pragma unroll
    for (int m = 0; m < PPT; ++m) {
      int p = p0 + threadIdx.x + m * kRT;
      if (p < KT) out[p] = (colmask && !colmask[p % t]) ? 0.0 : acc[m];
    }
    __syncthreads();
  }
}

// out[s] = sum_b partials[b*W + s] for s in [s0, s1), blocks in index order
// one warp per slot: lane l sums blocks l, l + 32, ... in order, then a fixed
// shuffle tree — deterministic, and ~30x shorter than one thread walking all
// the blocks (the mBCG grid is 3 blocks per SM)
__global__ void finalize_partials(const double* __restrict__ partials, int nblocks, int W,
                                  int s0, int s1, double* out) {
  const int s = s0 + (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (s >= s1) return;
  double acc = 0.0;
  for (int b = lane; b < nblocks; b += 32) acc += partials[(int64_t)b * W + s];
  acc = warp_sum(acc);
  if (lane == 0) out[s] = acc;
}

static int finalize(const double* partials, int nb, int W, int s0, int s1, double* out,
                    cudaStream_t st) {
  if (s1 <= s0) return GP_OK;
  const int64_t threads = (int64_t)(s1 - s0) * 32;
  finalize_partials<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(partials, nb, W, s0, s1, out);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

// ---------------------------------------------------------------------------
// mBCG kernels
// ---------------------------------------------------------------------------
struct CgK {  // by-value kernel view of gp_mbcg
  int64_t n; int t; int k; int64_t ld; int64_t ld32;
  double* U; double* R; double* P; double* Z; float* P32;
  double noise;
  const double* L; int64_t ldl; const double* Binv; double pc_noise;
  double* bnorm; double* gamma; double* red; double* cbuf;
  double* alpha_hist; double* beta_hist; double* rel; double* rel_hist;
  int* active; int* converged; int* status; double* partials;
};

static CgK view(const gp_mbcg* s) {
  CgK v;
  v.n = s->n; v.t = s->t; v.k = s->k; v.ld = s->ld; v.ld32 = s->ld32;
  v.U = s->U; v.R = s->R; v.P = s->P; v.Z = s->Z; v.P32 = s->P32; v.noise = s->noise;
  v.L = s->L; v.ldl = s->ldl; v.Binv = s->Binv; v.pc_noise = s->pc_noise;
  v.bnorm = s->bnorm; v.gamma = s->gamma; v.red = s->red; v.cbuf = s->cbuf;
  v.alpha_hist = s->alpha_hist; v.beta_hist = s->beta_hist; v.rel = s->rel;
  v.rel_hist = s->rel_hist; v.active = s->active; v.converged = s->converged;
  v.status = s->status; v.partials = s->partials;
  return v;
}

// red layout offsets
__host__ __device__ inline int off_pv(int) { return 0; }
__host__ __device__ inline int off_rn2(int t) { return t; }
__host__ __device__ inline int off_ltr(int t) { return 2 * t; }
__host__ __device__ inline int off_gam(int t, int k) { return 2 * t + k * t; }

// init_a: R = B, U = 0; partial rn2 = ||B_j||^2 and L^T B
__global__ void __launch_bounds__(kRT) cg_init_a(CgK s, const double* __restrict__ B, int64_t ldb) {
  extern __shared__ __align__(16) double dsm[];
  double* sred = dsm;
  double* sL = sred + kRT;   // block_ltmul scratch
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int t = s.t;
  const int W = 3 * t + s.k * t;
  double* part = s.partials + (int64_t)blockIdx.x * W;
  block_colsum(r0, r1, t, [&](int64_t r, int c) {
    double b = B[r * ldb + c];
    s.R[r * s.ld + c] = b;
    s.U[r * s.ld + c] = 0.0;
    return b * b;
  }, part + t, sred);
  if (s.k > 0) {
    __syncthreads();
    block_ltmul(r0, r1, s.k, t, s.L, s.ldl, s.R, s.ld, part + 2 * t, sL, nullptr);
  }
}

// c = B^{-1} (L^T R) for the given columns (one output per thread, k-long dots)
// C = B^{-1} (L^T R): one warp per output (kk, c), the length-k dot split
// over the lanes and reduced by shuffles (fixed order)
__global__ void cg_cvec(CgK s, int use_active) {
  const int t = s.t, k = s.k;
  const double* ltr = s.red + off_ltr(t);
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t p = w0; p < (int64_t)k * t; p += nw) {
    const int kk = (int)(p / t), c = (int)(p - (int64_t)kk * t);
    double acc = 0.0;
    if (!use_active || s.active[c])
      for (int l = lane; l < k; l += 32) acc = fma(s.Binv[kk * k + l], ltr[l * t + c], acc);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) s.cbuf[p] = acc;
  }
}

static unsigned cvec_blocks(int k, int t) {   // 8 warps per block, one warp per output
  return (unsigned)std::max(1, std::min((k * t + 7) / 8, 4 * num_sms()));
}

// Z = P^{-1} R on (active) columns; partial gam = sum R o Z.
// pc_noise <= 0: no preconditioner (Z = R, cg.py:360, :401);
// k == 0: Z = R / pc_noise (precond.py:131-132).
template <bool INIT>
__global__ void __launch_bounds__(kRT) cg_precond_z(CgK s) {
  extern __shared__ __align__(16) double dsm[];
  double* sred = dsm;
  double* sc = sred + kRT;  // k * t
  const int t = s.t, k = s.k;
  for (int p = threadIdx.x; p < k * t; p += kRT) sc[p] = s.cbuf[p];
  __syncthreads();
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int W = 3 * t + k * t;
  double* part = s.partials + (int64_t)blockIdx.x * W;
  block_colsum(r0, r1, t, [&](int64_t r, int c) {
    if (!INIT && !s.active[c]) return 0.0;
    double rv = s.R[r * s.ld + c];
    double z;
    if (s.pc_noise <= 0.0) {
      z = rv;
    } else {
      double lc = 0.0;
      const double* lr = s.L + r * s.ldl;
      for (int kk = 0; kk < k; ++kk) lc = fma(lr[kk], sc[kk * t + c], lc);
      z = (rv - lc) / s.pc_noise;
    }
    s.Z[r * s.ld + c] = z;
    if (INIT) {
      s.P[r * s.ld + c] = z;
      s.P32[r * s.ld32 + c] = (float)z;
    }
    return rv * z;
  }, part + off_gam(t, k), sred);
}

// Narrow blocks (t <= 16, the CG width, with a rank-k preconditioner): the
// block's rows in 64-row chunks, each chunk's L rows staged in SMEM with
// coalesced loads and C = B^{-1} L^T R resident; a thread owns one row and
// four columns, so each L row is read from HBM once per application (the
// one-output-per-thread form above re-read it t times through L1). Same kk
// order as cg_precond_z, hence the same z; fixed-order column sums.
constexpr int kZR = 32;          // rows per chunk
constexpr int kZLD = kZR + 1;    // transposed chunk [kk][row]: odd stride, conflict-free reads
constexpr int kZT = 128;         // threads: a thread owns one row and four columns
static size_t pz_narrow_smem(int k) {
  return ((size_t)k * 16 + 2 * ((size_t)k * kZLD + kZR * 16) + 16 * kZR) * sizeof(double);
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
template <bool INIT>
__global__ void __launch_bounds__(kZT) cg_precond_z_narrow(CgK s) {
  extern __shared__ __align__(16) double dsm[];
  const int t = s.t, k = s.k, TQ = (t + 3) / 4, TP = 4 * TQ;
  double* sC = dsm;                          // [k][TP]
  const size_t bstride = (size_t)k * kZLD + kZR * 16;
  double* sLb = sC + (size_t)k * 16;         // [2] x ([k][kZLD] L rows transposed | [kZR][16] R rows)
  double* sred = sLb + 2 * bstride;          // [TP][kZR]
  for (int p = threadIdx.x; p < k * TP; p += blockDim.x) {
    const int kk = p / TP, c = p - kk * TP;
    sC[p] = c < t ? s.cbuf[kk * t + c] : 0.0;
  }
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int rl = threadIdx.x % kZR, tq = threadIdx.x / kZR;   // row of the chunk, column quad
  const bool worker = tq < TQ;
  bool live[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = 4 * tq + j;
    live[j] = worker && c < t && (INIT || s.active[c]);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  // chunk c's copies (8-byte cp.async, zero-filled past the block's rows):
  // warp w rows w, w + nw, ..., lane l columns l, l + 32, ...
  auto issue = [&](int64_t rc, int buf) {
    const int nr = (int)min((int64_t)kZR, r1 - rc);
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(sLb + (size_t)buf * bstride);
    const uint32_t rbase = base + (uint32_t)((size_t)k * kZLD * 8);
    for (int r = w; r < kZR; r += nw) {
      const double* src = s.L + (r < nr ? (rc + r) * s.ldl : 0);
      for (int kk = l; kk < k; kk += 32)
        cp_async8(base + (uint32_t)((kk * kZLD + r) * 8), src + (r < nr ? kk : 0), r < nr ? 8u : 0u);
      // the chunk's R rows too: z needs them right after the FMAs
      const double* rsrc = s.R + (r < nr ? (rc + r) * s.ld : 0);
      if (l < 16) cp_async8(rbase + (uint32_t)((r * 16 + l) * 8), rsrc + (r < nr && l < t ? l : 0),
                            r < nr && l < t ? 8u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double gam[4] = {0.0, 0.0, 0.0, 0.0};
  int buf = 0;
  if (r0 < r1) issue(r0, 0);
  for (int64_t rc = r0; rc < r1; rc += kZR, buf ^= 1) {
    const int nr = (int)min((int64_t)kZR, r1 - rc);
    if (rc + kZR < r1) {
      issue(rc + kZR, buf ^ 1);   // the next chunk streams in while this one is used
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* sL = sLb + (size_t)buf * bstride;
    const double* sR = sL + (size_t)k * kZLD;
    if (worker && rl < nr) {
      double lc[4] = {0.0, 0.0, 0.0, 0.0};
      const double* cq = sC + 4 * tq;
      for (int kk = 0; kk < k; ++kk) {
        const double lv = sL[kk * kZLD + rl];
        const double2 ca = *reinterpret_cast<const double2*>(cq + kk * TP);
        const double2 cb = *reinterpret_cast<const double2*>(cq + kk * TP + 2);
        lc[0] = fma(lv, ca.x, lc[0]);
        lc[1] = fma(lv, ca.y, lc[1]);
        lc[2] = fma(lv, cb.x, lc[2]);
        lc[3] = fma(lv, cb.y, lc[3]);
      }
      const int64_t r = rc + rl;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!live[j]) continue;
        const int c = 4 * tq + j;
        const double rv = sR[rl * 16 + c];
        const double z = (rv - lc[j]) / s.pc_noise;
        s.Z[r * s.ld + c] = z;
        if (INIT) {
          s.P[r * s.ld + c] = z;
          s.P32[r * s.ld32 + c] = (float)z;
        }
        gam[j] += rv * z;
      }
    }
    __syncthreads();   // buffer `buf` is refilled by the issue two chunks on
  }
  if (worker) {
#pragma unroll
    for (int j = 0; j < 4; ++j) sred[(4 * tq + j) * kZR + rl] = gam[j];
  }
  __syncthreads();
  if ((int)threadIdx.x < t) {
    double v = 0.0;
    for (int q = 0; q < kZR; ++q) v += sred[threadIdx.x * kZR + q];
    s.partials[(int64_t)blockIdx.x * (3 * t + k * t) + off_gam(t, k) + threadIdx.x] = v;
  }
}

// The same with whole chunks moved by the TMA: when L is contiguous (ld = k)
// and k is even (16-byte aligned chunk starts and sizes), thread 0 copies each
// 32-row chunk of L (25.6 KB at k = 100) with one cp.async.bulk into a
// double-buffered row-major tile; the R rows follow by cp.async. A lane owns
// 2 rows x 4 columns (one C load serves both rows: the one-row form was bound
// by SMEM wavefronts, 5 LDS per 8 DFMA; 0.49 -> 0.35 ms at n = 10^6, k = 100)
// and the k range is split between warp pairs (warps 0-1 kk < k/2, warps 2-3
// the rest, partials added through SMEM), so every warp still covers 16 rows
// of the 32-row chunk. (Three k ranges over 6 warps with R read from global
// memory in the epilogue measured slower: 0.42 ms.) Even / odd kk accumulate
// separately (z differs from the forms above in the last bits).
constexpr int kZB = 32;           // rows per chunk
static size_t pz_bulk_smem(int k) {
  return ((size_t)k * 16 + 2 * ((size_t)kZB * k + kZB * 16) + 16 * kZB) * sizeof(double) + 64;
}
template <bool INIT>
__global__ void __launch_bounds__(128) cg_precond_z_bulk(CgK s) {
  extern __shared__ __align__(128) double dsm[];
  const int t = s.t, k = s.k, TQ = (t + 3) / 4, TP = 4 * TQ;
  double* sC = dsm;                               // [k][TP]
  const size_t bstride = (size_t)kZB * k + kZB * 16;
  double* sB = sC + (size_t)k * 16;               // [2] x ([kZB][k] L rows | [kZB][16] R rows)
  double* sred = sB + 2 * bstride;                // [TP][kZB]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sred + 16 * kZB);   // [2]
  for (int p = threadIdx.x; p < k * TP; p += blockDim.x) {
    const int kk = p / TP, c = p - kk * TP;
    sC[p] = c < t ? s.cbuf[kk * t + c] : 0.0;
  }
  if (threadIdx.x == 0) {
    tc::mbar_init(tc::smem_u32(&bar[0]), 1);
    tc::mbar_init(tc::smem_u32(&bar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int w = threadIdx.x >> 5, ln = threadIdx.x & 31;
  const int rl = 8 * w + (ln >> 2), tq = ln & 3;  // reduction slot, column quad
  const int kh = w >> 1;                           // k half of this warp
  const int ra = 16 * (w & 1) + (ln >> 2), rb = ra + 8;   // the lane's two rows of the chunk
  const int khalf = ((k >> 1) + 1) & ~1;           // even split point
  const int k0 = kh ? khalf : 0, k1 = kh ? k : khalf;
  double* xch = sred;                              // [kZB][16] k-half partials (sred is free in the loop)
  const bool worker = tq < TQ;
  bool live[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = 4 * tq + j;
    live[j] = worker && c < t && (INIT || s.active[c]);
  }
  auto issue = [&](int64_t rc, int b) {
    const int nr = (int)min((int64_t)kZB, r1 - rc);
    double* dst = sB + (size_t)b * bstride;
    if (threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      const uint32_t bytes = (uint32_t)(nr * k * 8);
      tc::mbar_expect_tx(tc::smem_u32(&bar[b]), bytes);
      tc::bulk_g2s(tc::smem_u32(dst), s.L + rc * k, bytes, tc::smem_u32(&bar[b]));
    }
    const uint32_t rb = tc::smem_u32(dst + (size_t)kZB * k);
    for (int e = threadIdx.x; e < kZB * 16; e += blockDim.x) {
      const int r = e >> 4, c = e & 15;
      const bool in = r < nr && c < t;
      cp_async8(rb + (uint32_t)(e * 8), s.R + (in ? (rc + r) * s.ld + c : 0), in ? 8u : 0u);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double gam[4] = {0.0, 0.0, 0.0, 0.0};
  if (r0 < r1) issue(r0, 0);
  int i = 0;
  for (int64_t rc = r0; rc < r1; rc += kZB, ++i) {
    const int b = i & 1;
    const int nr = (int)min((int64_t)kZB, r1 - rc);
    if (rc + kZB < r1) {
      issue(rc + kZB, b ^ 1);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    tc::mbar_wait(tc::smem_u32(&bar[b]), (i >> 1) & 1);
    __syncthreads();
    const double* sL = sB + (size_t)b * bstride;
    const double* sR = sL + (size_t)kZB * k;
    const bool va = worker && ra < nr, vb = worker && rb < nr;
    double sa[4] = {0.0, 0.0, 0.0, 0.0}, sb[4] = {0.0, 0.0, 0.0, 0.0};
    if (va) {
      // even and odd kk in separate accumulators (k is even here): twice
      // the independent DFMA chains, the loop is latency-bound otherwise
      double ea[4] = {0.0, 0.0, 0.0, 0.0}, oa[4] = {0.0, 0.0, 0.0, 0.0};
      double eb[4] = {0.0, 0.0, 0.0, 0.0}, ob[4] = {0.0, 0.0, 0.0, 0.0};
      const double* pa = sL + (size_t)ra * k;
      const double* pb = sL + (size_t)(vb ? rb : ra) * k;
      const double* cq = sC + 4 * tq;
      for (int kk = k0; kk < k1; kk += 2) {
        const double2 la = *reinterpret_cast<const double2*>(pa + kk);
        const double2 lb = *reinterpret_cast<const double2*>(pb + kk);
        const double2 ca = *reinterpret_cast<const double2*>(cq + kk * TP);
        const double2 cb = *reinterpret_cast<const double2*>(cq + kk * TP + 2);
        const double2 da = *reinterpret_cast<const double2*>(cq + (kk + 1) * TP);
        const double2 db = *reinterpret_cast<const double2*>(cq + (kk + 1) * TP + 2);
        ea[0] = fma(la.x, ca.x, ea[0]);
        ea[1] = fma(la.x, ca.y, ea[1]);
        ea[2] = fma(la.x, cb.x, ea[2]);
        ea[3] = fma(la.x, cb.y, ea[3]);
        oa[0] = fma(la.y, da.x, oa[0]);
        oa[1] = fma(la.y, da.y, oa[1]);
        oa[2] = fma(la.y, db.x, oa[2]);
        oa[3] = fma(la.y, db.y, oa[3]);
        eb[0] = fma(lb.x, ca.x, eb[0]);
        eb[1] = fma(lb.x, ca.y, eb[1]);
        eb[2] = fma(lb.x, cb.x, eb[2]);
        eb[3] = fma(lb.x, cb.y, eb[3]);
        ob[0] = fma(lb.y, da.x, ob[0]);
        ob[1] = fma(lb.y, da.y, ob[1]);
        ob[2] = fma(lb.y, db.x, ob[2]);
        ob[3] = fma(lb.y, db.y, ob[3]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        sa[j] = ea[j] + oa[j];
        sb[j] = eb[j] + ob[j];
      }
      if (kh == 1) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          xch[ra * 16 + 4 * tq + j] = sa[j];
          if (vb) xch[rb * 16 + 4 * tq + j] = sb[j];
        }
      }
    }
    __syncthreads();   // the second k half's partials are in xch
    if (kh == 0) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int rr = h ? rb : ra;
        if (!(h ? vb : va)) continue;
        const int64_t r = rc + rr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!live[j]) continue;
          const int c = 4 * tq + j;
          const double lc = (h ? sb[j] : sa[j]) + xch[rr * 16 + c];
          const double rv = sR[rr * 16 + c];
          const double z = (rv - lc) / s.pc_noise;
          s.Z[r * s.ld + c] = z;
          if (INIT) {
            s.P[r * s.ld + c] = z;
            s.P32[r * s.ld32 + c] = (float)z;
          }
          gam[j] += rv * z;
        }
      }
    }
    __syncthreads();   // xch is rewritten and buffer b refilled by the next chunks
  }
  // warps 2-3 hold zero gam: their slots (16-31) add nothing
  if (worker) {
#pragma unroll
    for (int j = 0; j < 4; ++j) sred[(4 * tq + j) * kZB + rl] = gam[j];
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (4 * tq + j < TP) sred[(4 * tq + j) * kZB + rl] = 0.0;
  }
  __syncthreads();
  if ((int)threadIdx.x < t) {
    double v = 0.0;
    for (int q = 0; q < kZB; ++q) v += sred[threadIdx.x * kZB + q];
    s.partials[(int64_t)blockIdx.x * (3 * t + k * t) + off_gam(t, k) + threadIdx.x] = v;
  }
}

// ---------------------------------------------------------------------------
// Wide right-hand-side blocks (t >= kWideT: the 256-column variance solves).
// The Woodbury terms are GEMM-shaped there (n x k by k x t, k x n by n x t)
// and the one-output-per-thread forms above re-read L and C k times per
// element; these register-tiled forms (64 x 64 output tile per block, 4 x 4
// per thread, operands staged in SMEM, 16 DFMA per 4 LDS.128) keep the fp64
// pipe busy instead. Grid (nb, ceil(t / 64)): blockIdx.x owns the same row
// range as the narrow kernels (row_range), so partials stay per row block.
// ---------------------------------------------------------------------------
constexpr int kWideT = 32;
constexpr int kWT = 64;        // output tile edge
constexpr int kWLS = kWT + 4;  // padded SMEM row (keeps 16-byte alignment)

// Z = (R - L C) / pc_noise on (active) columns, C = s.cbuf (k x t);
// partial gam = sum R o Z (cg_precond_z semantics, k > 0 and pc_noise > 0)
template <bool INIT>
__global__ void __launch_bounds__(256) cg_precond_z_wide(CgK s) {
  extern __shared__ __align__(16) double dsm[];
  const int t = s.t, k = s.k;
  const int c0 = blockIdx.y * kWT;
  double* sC = dsm;                    // [k][kWT]
  double* sL = sC + (size_t)k * kWT;   // [k][kWLS]: L^T of the current 64-row tile
  double* sred = sL + (size_t)k * kWLS;  // [16][kWT]
  for (int p = threadIdx.x; p < k * kWT; p += 256) {
    const int kk = p / kWT, c = p - kk * kWT;
    sC[p] = c0 + c < t ? s.cbuf[kk * t + c0 + c] : 0.0;
  }
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  bool live[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = c0 + 4 * tx + j;
    live[j] = c < t && (INIT || s.active[c]);
  }
  double colacc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t rb = r0; rb < r1; rb += kWT) {
    const int nr = (int)min((int64_t)kWT, r1 - rb);
    __syncthreads();
    for (int p = threadIdx.x; p < kWT * k; p += 256) {
      const int r = p / k, kk = p - r * k;
      sL[kk * kWLS + r] = r < nr ? s.L[(rb + r) * s.ldl + kk] : 0.0;
    }
    __syncthreads();
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int kk = 0; kk < k; ++kk) {
      const double2 la = *reinterpret_cast<const double2*>(sL + kk * kWLS + 4 * ty);
      const double2 lb = *reinterpret_cast<const double2*>(sL + kk * kWLS + 4 * ty + 2);
      const double2 ca = *reinterpret_cast<const double2*>(sC + kk * kWT + 4 * tx);
      const double2 cb = *reinterpret_cast<const double2*>(sC + kk * kWT + 4 * tx + 2);
      const double l[4] = {la.x, la.y, lb.x, lb.y}, c[4] = {ca.x, ca.y, cb.x, cb.y};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(l[i], c[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = 4 * ty + i;
      if (rl >= nr) continue;
      const int64_t r = rb + rl;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!live[j]) continue;
        const int c = c0 + 4 * tx + j;
        const double rv = s.R[r * s.ld + c];
        const double z = (rv - acc[i][j]) / s.pc_noise;   // same kk order as cg_precond_z: same z
        s.Z[r * s.ld + c] = z;
        if (INIT) {
          s.P[r * s.ld + c] = z;
          s.P32[r * s.ld32 + c] = (float)z;
        }
        colacc[j] += rv * z;
      }
    }
  }
  // per-column partials: threads of equal tx summed in ty order (deterministic)
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) sred[ty * kWT + 4 * tx + j] = colacc[j];
  __syncthreads();
  if (threadIdx.x < kWT && c0 + (int)threadIdx.x < t) {
    double v = 0.0;
    for (int q = 0; q < 16; ++q) v += sred[q * kWT + threadIdx.x];
    s.partials[(int64_t)blockIdx.x * (3 * t + k * t) + off_gam(t, k) + c0 + threadIdx.x] = v;
  }
}

// partial L^T A over this block's rows into part[kk * t + c] (columns with
// colmask[c] == 0 get 0): the block_ltmul product for wide t
__global__ void __launch_bounds__(256) ltr_wide(int64_t n, int k, int t, const double* __restrict__ L,
                                                int64_t ldl, const double* __restrict__ A, int64_t lda,
                                                double* partials, int W, int slot, const int* colmask) {
  __shared__ __align__(16) double sL[32 * kWLS];
  __shared__ __align__(16) double sA[32 * kWLS];
  int64_t r0, r1;
  row_range(n, r0, r1);
  const int c0 = blockIdx.y * kWT;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double* part = partials + (int64_t)blockIdx.x * W + slot;
  for (int k0 = 0; k0 < k; k0 += kWT) {
    double acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
    for (int64_t rb = r0; rb < r1; rb += 32) {
      const int nr = (int)min((int64_t)32, r1 - rb);
      __syncthreads();
      for (int p = threadIdx.x; p < 32 * kWT; p += 256) {
        const int r = p / kWT, q = p - r * kWT;
        const bool in = r < nr;
        sL[r * kWLS + q] = in && k0 + q < k ? L[(rb + r) * ldl + k0 + q] : 0.0;
        sA[r * kWLS + q] = in && c0 + q < t ? A[(rb + r) * lda + c0 + q] : 0.0;
      }
      __syncthreads();
      for (int r = 0; r < nr; ++r) {
        const double2 la = *reinterpret_cast<const double2*>(sL + r * kWLS + 4 * ty);
        const double2 lb = *reinterpret_cast<const double2*>(sL + r * kWLS + 4 * ty + 2);
        const double2 aa = *reinterpret_cast<const double2*>(sA + r * kWLS + 4 * tx);
        const double2 ab = *reinterpret_cast<const double2*>(sA + r * kWLS + 4 * tx + 2);
        const double l[4] = {la.x, la.y, lb.x, lb.y}, a[4] = {aa.x, aa.y, ab.x, ab.y};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fma(l[i], a[j], acc[i][j]);
      }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int kk = k0 + 4 * ty + i;
      if (kk >= k) continue;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int c = c0 + 4 * tx + j;
        if (c < t) part[kk * t + c] = (colmask && !colmask[c]) ? 0.0 : acc[i][j];
      }
    }
  }
}

__global__ void cg_init_c(CgK s) {
  for (int c = threadIdx.x; c < s.t; c += blockDim.x) {
    s.gamma[c] = s.red[off_gam(s.t, s.k) + c];
    s.active[c] = 1;
    s.converged[c] = 0;
    s.rel[c] = 1.0;
  }
  if (threadIdx.x == 0) {
    s.status[0] = s.t;
    s.status[1] = 0x7fffffff;  // no non-PD column seen
    s.status[2] = 0;
  }
}

__global__ void cg_bnorm(CgK s) {
  for (int c = threadIdx.x; c < s.t; c += blockDim.x) s.bnorm[c] = sqrt(s.red[off_rn2(s.t) + c]);
}

// pv partial = sum P o (Q + noise P) over active columns
template <typename QT>
__global__ void __launch_bounds__(kRT) cg_pv(CgK s, const QT* __restrict__ Q, int64_t ldq) {
  __shared__ double sred[kRT];
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int t = s.t;
  double* part = s.partials + (int64_t)blockIdx.x * (3 * t + s.k * t);
  block_colsum(r0, r1, t, [&](int64_t r, int c) {
    if (!s.active[c]) return 0.0;
    double p = s.P[r * s.ld + c];
    double q = (double)Q[r * ldq + c] + s.noise * p;
    return p * q;
  }, part, sred);
}

// alpha = gamma / pv on active columns + PD check (cg.py:120-128)
__global__ void cg_alpha(CgK s, int it) {
  for (int c = threadIdx.x; c < s.t; c += blockDim.x) {
    double a = 0.0;
    if (s.active[c]) {
      double pv = s.red[off_pv(s.t) + c];
      if (!(pv > 0.0) || !isfinite(pv)) {
        atomicMin(&s.status[1], c);  // lowest offending column
        s.status[2] = it;
      }
      a = s.gamma[c] / pv;
    }
    s.alpha_hist[(int64_t)(it - 1) * s.t + c] = a;
  }
}

// U += alpha P; R -= alpha (Q + noise P); partial rn2; partial L^T R
template <typename QT>
__global__ void __launch_bounds__(kRT) cg_update(CgK s, const QT* __restrict__ Q, int64_t ldq, int it,
                                                 int with_ltr) {
  extern __shared__ __align__(16) double dsm[];
  double* sred = dsm;
  double* sal = sred + kRT;               // t
  double* sL = sal + ((s.t + 1) & ~1);   // block_ltmul scratch, 16-byte aligned
  const int t = s.t, k = s.k;
  for (int c = threadIdx.x; c < t; c += kRT)
    sal[c] = s.active[c] ? s.alpha_hist[(int64_t)(it - 1) * t + c] : 0.0;
  __syncthreads();
  int64_t r0, r1;
  row_range(s.n, r0, r1);
  const int W = 3 * t + k * t;
  double* part = s.partials + (int64_t)blockIdx.x * W;
  block_colsum(r0, r1, t, [&](int64_t r, int c) {
    double rv = s.R[r * s.ld + c];
    if (s.active[c]) {
      double a = sal[c];
      double p = s.P[r * s.ld + c];
      double q = (double)Q[r * ldq + c] + s.noise * p;
      s.U[r * s.ld + c] += a * p;
      rv -= a * q;
      s.R[r * s.ld + c] = rv;
    }
    return rv * rv;
  }, part + t, sred);
  if (with_ltr && k > 0 && s.pc_noise > 0.0) {
    __syncthreads();
    block_ltmul(r0, r1, k, t, s.L, s.ldl, s.R, s.ld, part + 2 * t, sL, s.active);
  }
}

// rel, freeze (cg.py:133-143); c = B^{-1} L^T R for the columns kept
__global__ void cg_freeze(CgK s, int it, double tol) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < s.t; c += blockDim.x) {
    if (s.active[c]) {
      double rel = sqrt(s.red[off_rn2(s.t) + c]) / s.bnorm[c];
      s.rel[c] = rel;
      if (rel <= tol) {
        s.converged[c] = 1;
        s.active[c] = 0;
      }
    }
    s.rel_hist[(int64_t)(it - 1) * s.t + c] = s.rel[c];
    if (s.active[c]) atomicAdd(&cnt, 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) s.status[0] = cnt;
}

// beta = gam / gamma on active columns (cg.py:145-152)
__global__ void cg_beta(CgK s, int it) {
  const double* gam = s.red + off_gam(s.t, s.k);
  for (int c = threadIdx.x; c < s.t; c += blockDim.x) {
    double b = 0.0;
    if (s.active[c]) {
      b = gam[c] / s.gamma[c];
      s.gamma[c] = gam[c];
    }
    s.beta_hist[(int64_t)(it - 1) * s.t + c] = b;
  }
}

__global__ void cg_direction(CgK s, int it) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t tot = s.n * s.t;
  for (; idx < tot; idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx / s.t;
    int c = (int)(idx - r * s.t);
    if (!s.active[c]) continue;
    double b = s.beta_hist[(int64_t)(it - 1) * s.t + c];
    double p = s.Z[r * s.ld + c] + b * s.P[r * s.ld + c];
    s.P[r * s.ld + c] = p;
    s.P32[r * s.ld32 + c] = (float)p;
  }
}


// ---------------------------------------------------------------------------
// generic column reductions / low-rank products
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kRT) coldot_kernel(int64_t n, int t, const double* __restrict__ A,
                                                     int64_t lda, const double* __restrict__ B,
                                                     int64_t ldb, double* partials) {
  __shared__ double sred[kRT];
  int64_t r0, r1;
  row_range(n, r0, r1);
  block_colsum(r0, r1, t, [&](int64_t r, int c) { return A[r * lda + c] * B[r * ldb + c]; },
               partials + (int64_t)blockIdx.x * t, sred);
}

__global__ void __launch_bounds__(kRT) ltmul_kernel(int64_t n, int k, const double* __restrict__ L,
                                                    int64_t ldl, const double* __restrict__ V,
                                                    int64_t ldv, int t, double* partials) {
  extern __shared__ __align__(16) double dsm[];
  int64_t r0, r1;
  row_range(n, r0, r1);
  block_ltmul(r0, r1, k, t, L, ldl, V, ldv, partials + (int64_t)blockIdx.x * k * t, dsm, nullptr);
}

// Y = beta Y + alpha L M
__global__ void lowrank_kernel(int64_t n, int k, const double* __restrict__ L, int64_t ldl,
                               const double* __restrict__ M, int64_t ldm, int t, double alpha,
                               double beta, double* Y, int64_t ldy) {
  extern __shared__ double sM[];  // k x t
  for (int p = threadIdx.x; p < k * t; p += blockDim.x) {
    int kk = p / t, c = p - kk * t;
    sM[p] = M[kk * ldm + c];
  }
  __syncthreads();
  int64_t tot = n * t;
  for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx / t;
    int c = (int)(idx - r * t);
    const double* lr = L + r * ldl;
    double acc = 0.0;
    for (int kk = 0; kk < k; ++kk) acc = fma(lr[kk], sM[kk * t + c], acc);
    double y = beta == 0.0 ? 0.0 : beta * Y[r * ldy + c];
    Y[r * ldy + c] = y + alpha * acc;
  }
}

// Y = beta Y + alpha L M for wide M (t >= 32): 64 x 64 output tile per block,
// 4 x 4 per thread, the tile's L rows (transposed) and M columns staged in
// SMEM (the GEMM-shaped Woodbury products of the 256-column variance solves
// and of the gradient operands L B^-1)
__global__ void __launch_bounds__(256) lowrank_wide(int64_t n, int k, const double* __restrict__ L, int64_t ldl,
                                                    const double* __restrict__ M, int64_t ldm, int t, double alpha,
                                                    double beta, double* Y, int64_t ldy) {
  extern __shared__ __align__(16) double dsm[];
  double* sM = dsm;                    // [k][kWT]
  double* sL = sM + (size_t)k * kWT;   // [k][kWLS]
  const int c0 = blockIdx.y * kWT;
  const int64_t rb = (int64_t)blockIdx.x * kWT;
  const int nr = (int)min((int64_t)kWT, n - rb);
  for (int p = threadIdx.x; p < k * kWT; p += 256) {
    const int kk = p / kWT, c = p - kk * kWT;
    sM[p] = c0 + c < t ? M[kk * ldm + c0 + c] : 0.0;
  }
  for (int p = threadIdx.x; p < kWT * k; p += 256) {
    const int r = p / k, kk = p - r * k;
    sL[kk * kWLS + r] = r < nr ? L[(rb + r) * ldl + kk] : 0.0;
  }
  __syncthreads();
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int kk = 0; kk < k; ++kk) {
    const double2 la = *reinterpret_cast<const double2*>(sL + kk * kWLS + 4 * ty);
    const double2 lb = *reinterpret_cast<const double2*>(sL + kk * kWLS + 4 * ty + 2);
    const double2 ma = *reinterpret_cast<const double2*>(sM + kk * kWT + 4 * tx);
    const double2 mb = *reinterpret_cast<const double2*>(sM + kk * kWT + 4 * tx + 2);
    const double l[4] = {la.x, la.y, lb.x, lb.y}, m[4] = {ma.x, ma.y, mb.x, mb.y};
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = fma(l[i], m[j], acc[i][j]);
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int rl = 4 * ty + i;
    if (rl >= nr) continue;
    const int64_t r = rb + rl;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = c0 + 4 * tx + j;
      if (c >= t) continue;
      const double y = beta == 0.0 ? 0.0 : beta * Y[r * ldy + c];
      Y[r * ldy + c] = y + alpha * acc[i][j];
    }
  }
}

// In-place Cholesky of B = noise I + G (G = L^T L, k x k, row-major, lower
// result), then X = C^{-1} (lower) into Binv (xtx_kernel forms B^{-1} =
// X^T X); out[0] = 2 sum log C_jj, out[1] = tr(B^{-1}) = ||X||_F^2
// (precond.py:114-122, :165-174). Single block, the k x k matrix in shared
// memory (k <= 160), so the k column steps and the substitution run at SMEM
// latency; C is written back for the caller.
__device__ __forceinline__ double block_sum_1024(double v, double* sred) {
  // fixed-order tree: warp shuffles, then warp 0 over the 32 warp sums
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? sred[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  __syncthreads();
  return s;   // valid in warp 0
}

__global__ void __launch_bounds__(1024) precond_factor_kernel(int k, double noise, double* C, double* Binv,
                                                              double* out, int* info) {
  extern __shared__ double Cs[];   // [k][k]: lower = factor, strict upper (transposed) = inverse work
  __shared__ int fail;
  __shared__ double sred[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) fail = 0;
  for (int p = tid; p < k * k; p += nt) {
    const int i = p / k, j = p - i * k;
    Cs[p] = C[p] + (i == j ? noise : 0.0);
  }
  __syncthreads();
  // right-looking Cholesky with one barrier per column: step j updates the
  // trailing square (both triangles, so the column j a thread needs is read
  // as row j: contiguous, conflict-free) with the unscaled column j over
  // d_jj and scales column j - 1 (which no thread reads in step j). Threads
  // form a 32 x 32 grid over (row i, column l): no index division.
  // The pivot's 1 / d_jj, sqrt(d_jj) and 1 / sqrt(d_jj) are formed ONCE, by
  // the thread that wrote d_jj last (thread 0 updates (j, j) in step j - 1),
  // into per-column slots: fp64 division and square root in all 1024 threads
  // every step cost more than the update itself.
  double* s_inv = Cs + (size_t)k * k;   // [k]
  double* s_sq = s_inv + k;             // [k]
  double* s_rs = s_sq + k;              // [k]
  const int tx = tid & 31, ty = tid >> 5, nty = nt >> 5;
  auto pivot_terms = [&](int j) {
    const double d = Cs[j * k + j];
    if (!(d > 0.0) || !isfinite(d)) fail = 1;
    s_inv[j] = 1.0 / d;
    s_sq[j] = sqrt(d);
    s_rs[j] = 1.0 / sqrt(d);
  };
  if (tid == 0) pivot_terms(0);
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (j >= 1) {
      const double rs = s_rs[j - 1];
      for (int i = j + tid; i < k; i += nt) Cs[i * k + j - 1] *= rs;
      if (tid == 0) Cs[(j - 1) * k + j - 1] = s_sq[j - 1];
    }
    const double inv = s_inv[j];
    for (int i = j + 1 + ty; i < k; i += nty) {
      const double a = Cs[i * k + j];
      for (int l = j + 1 + tx; l < k; l += 32) Cs[i * k + l] -= a * Cs[j * k + l] * inv;
    }
    if (tid == 0 && j + 1 < k) pivot_terms(j + 1);   // (j + 1, j + 1) was this thread's first update
    __syncthreads();
  }
  if (tid == 0) Cs[(k - 1) * k + k - 1] = s_sq[k - 1];
  __syncthreads();
  if (fail) {
    if (tid == 0) info[0] = 1;
    return;
  }
  // X = C^{-1} (lower), right-looking: W starts as I; step i finalises row i
  // (X[i][c] = W[i][c] / C_ii) and subtracts C[r][i] X[i][:] from every row
  // r > i. W[r][c] (c < r) lives at Cs[c k + r], the strict upper triangle;
  // consecutive threads take consecutive r (conflict-free stores)
  for (int p = tid; p < k * k; p += nt) {
    const int c = p / k, r = p - c * k;
    if (r > c) Cs[p] = 0.0;
  }
  __syncthreads();
  for (int i = 0; i + 1 < k; ++i) {
    const double rinv = s_rs[i];   // 1 / C_ii
    for (int c = ty; c <= i; c += nty) {
      const double xic = (c == i ? 1.0 : Cs[c * k + i]) * rinv;
      for (int r = i + 1 + tx; r < k; r += 32) Cs[c * k + r] -= Cs[r * k + i] * xic;
    }
    __syncthreads();
  }
  // X out (scaled rows) to Binv, tr(B^{-1}) = ||X||_F^2, logdet = 2 sum log C_jj
  double tr = 0.0, ld = 0.0;
  for (int p = tid; p < k * k; p += nt) {
    const int i = p / k, c = p - i * k;
    const double cii = Cs[i * k + i];
    const double x = c > i ? 0.0 : (c == i ? 1.0 / cii : Cs[c * k + i] / cii);
    Binv[p] = x;
    C[p] = c > i ? 0.0 : Cs[p];
    tr += x * x;
  }
  for (int j = tid; j < k; j += nt) ld += log(Cs[j * k + j]);
  const double trs = block_sum_1024(tr, sred);
  const double lds = block_sum_1024(ld, sred);
  if (tid == 0) {
    out[1] = trs;
    out[0] = 2.0 * lds;
    info[0] = 0;
  }
}

// global-memory form for k > 160 (the k x k matrix exceeds shared memory)
__global__ void precond_factor_global(int k, double noise, double* C, double* Binv, double* out, int* info) {
  __shared__ int fail;
  if (threadIdx.x == 0) fail = 0;
  __syncthreads();
  for (int p = threadIdx.x; p < k * k; p += blockDim.x) {
    int i = p / k, j = p - i * k;
    if (i == j) C[p] += noise;
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    if (threadIdx.x == 0) {
      double djj = C[j * k + j];
      if (!(djj > 0.0) || !isfinite(djj)) fail = 1;
      C[j * k + j] = sqrt(fmax(djj, 0.0));
    }
    __syncthreads();
    if (fail) break;
    double cjj = C[j * k + j];
    for (int i = j + 1 + threadIdx.x; i < k; i += blockDim.x) C[i * k + j] /= cjj;
    __syncthreads();
    int m = k - j - 1;
    for (int p = threadIdx.x; p < m * m; p += blockDim.x) {
      int i = j + 1 + p / m, l = j + 1 + p % m;
      if (l <= i) C[i * k + l] -= C[i * k + j] * C[l * k + j];
    }
    __syncthreads();
  }
  if (fail) {
    if (threadIdx.x == 0) info[0] = 1;
    return;
  }
  for (int p = threadIdx.x; p < k * k; p += blockDim.x) {
    int i = p / k, j = p - i * k;
    if (j > i) C[p] = 0.0;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    for (int i = 0; i < k; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (int l = c; l < i; ++l) s -= C[i * k + l] * Binv[l * k + c];
      Binv[i * k + c] = (i < c) ? 0.0 : s / C[i * k + i];
    }
  }
  __syncthreads();
  __shared__ double sred[1024];
  double tr = 0.0, ld = 0.0;
  for (int p = threadIdx.x; p < k * k; p += blockDim.x) tr += Binv[p] * Binv[p];
  for (int j = threadIdx.x; j < k; j += blockDim.x) ld += log(C[j * k + j]);
  sred[threadIdx.x] = tr;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)blockDim.x; ++q) s += sred[q];
    out[1] = s;
  }
  __syncthreads();
  sred[threadIdx.x] = ld;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int q = 0; q < (int)blockDim.x; ++q) s += sred[q];
    out[0] = 2.0 * s;
    info[0] = 0;
  }
}

// Binv = X^T X given X (lower) in Xs; separate kernel to avoid aliasing
__global__ void xtx_kernel(int k, const double* __restrict__ X, double* out) {
  int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= k * k) return;
  int i = p / k, j = p - i * k;
  int l0 = max(i, j);
  double s = 0.0;
  for (int l = l0; l < k; ++l) s = fma(X[l * k + i], X[l * k + j], s);
  out[p] = s;
}

static int cg_nblocks(const gp_mbcg* s) {
  if (s->nblocks > 0) return s->nblocks;
  int64_t nb = std::min<int64_t>(3 * num_sms(), (s->n + 31) / 32);   // 3 resident blocks per SM, >= 32 rows each
  return (int)std::max<int64_t>(nb, 1);
}

static int check_state(const gp_mbcg* s) {
  GP_REQUIRE(s && s->n >= 0 && s->t >= 1, "gp_mbcg: bad state");
  GP_REQUIRE(s->ld >= s->t && s->ld32 >= s->t, "gp_mbcg: leading dimension < t");
  GP_REQUIRE(s->k >= 0 && s->k <= 1024, "gp_mbcg: k=%d", s->k);
  GP_REQUIRE(s->k == 0 || (s->L && s->Binv), "gp_mbcg: k>0 needs L and Binv");
  int64_t need = (int64_t)cg_nblocks(s) * (3 * s->t + s->k * s->t);
  GP_REQUIRE(s->partials_len >= need, "gp_mbcg: partials workspace %lld < %lld",
             (long long)s->partials_len, (long long)need);
  return GP_OK;
}

static size_t ltmul_smem(int k, int t) { return (size_t)ltmul_scratch(k, t) * sizeof(double); }

// the preconditioner application has a form for every (t, k) whose working
// set fits shared memory: narrow (t <= 16, k <= ~340), wide (t >= 32, k <= 212)
// or the per-element one ((256 + k t) doubles); beyond that the caller must
// split the right-hand sides (predictor.py does, in blocks of 16)

static size_t pz_wide_smem(int k) { return ((size_t)k * (kWT + kWLS) + 16 * kWT) * sizeof(double); }
// the register-tiled Woodbury forms apply to wide blocks with a preconditioner
// whose C tile and L^T tile fit in SMEM (k <= ~200)
static bool use_wide(const gp_mbcg* s) {
  return s->t >= kWideT && s->k > 0 && s->pc_noise > 0.0 && pz_wide_smem(s->k) <= 227 * 1024;
}

// the staged narrow Woodbury form: t <= 16 with a preconditioner whose L
// chunk and C fit in SMEM (k <= ~340)
static bool use_narrow(const gp_mbcg* s) {
  return s->t <= 16 && s->k > 0 && s->pc_noise > 0.0 && pz_narrow_smem(s->k) <= 227 * 1024;
}

// whole-chunk TMA copies of L: contiguous L, even k (16-byte aligned chunks)
static bool use_bulk(const gp_mbcg* s) {
  return use_narrow(s) && s->ldl == s->k && s->k % 2 == 0 && pz_bulk_smem(s->k) <= 227 * 1024;
}

static int check_precond_fits(const gp_mbcg* s) {
  if (s->k == 0 || s->pc_noise <= 0.0 || use_narrow(s) || use_wide(s)) return GP_OK;
  GP_REQUIRE((kRT + (size_t)s->k * s->t) * sizeof(double) <= 227 * 1024,
             "preconditioner rank %d with %d right-hand sides exceeds the device's shared memory; "
             "solve in blocks of at most 16 columns or use a rank of at most 212", s->k, s->t);
  return GP_OK;
}

template <class K>
static int set_smem(K kern, size_t bytes) {
  if (bytes > 48 * 1024)
    GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return GP_OK;
}

}  // namespace gp

using namespace gp;

namespace gp {
thread_local bool kv_images_current = false;
}

extern "C" {

int64_t gp_mbcg_partials_len(int64_t n, int t, int k) {
  int64_t nb = std::min<int64_t>(3 * num_sms(), (n + 31) / 32);
  nb = std::max<int64_t>(nb, 1);
  return nb * (3 * (int64_t)t + (int64_t)k * t);
}

int gp_mbcg_init_a(gp_mbcg* s, const double* B, int64_t ldb, void* stream) {
  if (int rc = check_state(s)) return rc;
  if (int rc = check_precond_fits(s)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int t = s->t, k = s->k, W = 3 * t + k * t, nb = cg_nblocks(s);
  if (s->n > 0) {
    size_t smem = kRT * sizeof(double) + ltmul_smem(k, t);
    if (int rc = set_smem(cg_init_a, smem)) return rc;
    cg_init_a<<<nb, kRT, smem, st>>>(view(s), B, ldb);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_rn2(t), off_ltr(t) + (k > 0 ? k * t : 0), s->red, st);
  }
  GP_CUDA_TRY(cudaMemsetAsync(s->red + off_rn2(t), 0, sizeof(double) * (t + k * t), st));
  return GP_OK;
}

int gp_mbcg_init_b(gp_mbcg* s, void* stream) {
  if (int rc = check_state(s)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CgK v = view(s);
  const int t = s->t, k = s->k, W = 3 * t + k * t, nb = cg_nblocks(s);
  cg_bnorm<<<1, 256, 0, st>>>(v);
  GP_LAUNCH_CHECK();
  if (k > 0 && s->pc_noise > 0.0) {
    cg_cvec<<<cvec_blocks(k, t), 256, 0, st>>>(v, 0);
    GP_LAUNCH_CHECK();
  }
  if (s->n > 0 && use_wide(s)) {
    const size_t smem = pz_wide_smem(k);
    if (int rc = set_smem(cg_precond_z_wide<true>, smem)) return rc;
    cg_precond_z_wide<true><<<dim3(nb, (t + kWT - 1) / kWT), 256, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0 && use_bulk(s)) {
    const size_t smem = pz_bulk_smem(k);
    if (int rc = set_smem(cg_precond_z_bulk<true>, smem)) return rc;
    cg_precond_z_bulk<true><<<nb, 128, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0 && use_narrow(s)) {
    const size_t smem = pz_narrow_smem(k);
    if (int rc = set_smem(cg_precond_z_narrow<true>, smem)) return rc;
    cg_precond_z_narrow<true><<<nb, kZT, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0) {
    size_t smem = (kRT + (size_t)k * t) * sizeof(double);
    if (int rc = set_smem(cg_precond_z<true>, smem)) return rc;
    cg_precond_z<true><<<nb, kRT, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  GP_CUDA_TRY(cudaMemsetAsync(s->red + off_gam(t, k), 0, sizeof(double) * t, st));
  return GP_OK;
}

int gp_mbcg_init_c(gp_mbcg* s, void* stream) {
  if (int rc = check_state(s)) return rc;
  cg_init_c<<<1, 256, 0, (cudaStream_t)stream>>>(view(s));
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int gp_mbcg_pv(gp_mbcg* s, const void* Q, int64_t ldq, int q_is_f64, void* stream) {
  if (int rc = check_state(s)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int t = s->t, k = s->k, W = 3 * t + k * t, nb = cg_nblocks(s);
  if (s->n > 0) {
    if (q_is_f64)
      cg_pv<double><<<nb, kRT, 0, st>>>(view(s), static_cast<const double*>(Q), ldq);
    else
      cg_pv<float><<<nb, kRT, 0, st>>>(view(s), static_cast<const float*>(Q), ldq);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_pv(t), off_pv(t) + t, s->red, st);
  }
  GP_CUDA_TRY(cudaMemsetAsync(s->red, 0, sizeof(double) * t, st));
  return GP_OK;
}

int gp_mbcg_update(gp_mbcg* s, const void* Q, int64_t ldq, int q_is_f64, int iteration,
                   void* stream) {
  if (int rc = check_state(s)) return rc;
  GP_REQUIRE(iteration >= 1 && iteration <= s->max_iters, "gp_mbcg_update: iteration %d", iteration);
  cudaStream_t st = (cudaStream_t)stream;
  CgK v = view(s);
  const int t = s->t, k = s->k, W = 3 * t + k * t, nb = cg_nblocks(s);
  cg_alpha<<<1, 256, 0, st>>>(v, iteration);
  GP_LAUNCH_CHECK();
  if (s->n > 0) {
    size_t smem = (kRT + ((t + 1) & ~1)) * sizeof(double) + ltmul_smem(k, t);
    const int in_kernel_ltr = use_wide(s) ? 0 : 1;
    if (q_is_f64) {
      if (int rc = set_smem(cg_update<double>, smem)) return rc;
      cg_update<double><<<nb, kRT, smem, st>>>(v, static_cast<const double*>(Q), ldq, iteration, in_kernel_ltr);
    } else {
      if (int rc = set_smem(cg_update<float>, smem)) return rc;
      cg_update<float><<<nb, kRT, smem, st>>>(v, static_cast<const float*>(Q), ldq, iteration, in_kernel_ltr);
    }
    GP_LAUNCH_CHECK();
    if (!in_kernel_ltr) {
      ltr_wide<<<dim3(nb, (t + kWT - 1) / kWT), 256, 0, st>>>(s->n, k, t, s->L, s->ldl, s->R, s->ld, s->partials, W,
                                                             off_ltr(t), s->active);
      GP_LAUNCH_CHECK();
    }
    int s1 = (k > 0 && s->pc_noise > 0.0) ? off_ltr(t) + k * t : off_ltr(t);
    return finalize(s->partials, nb, W, off_rn2(t), s1, s->red, st);
  }
  GP_CUDA_TRY(cudaMemsetAsync(s->red + off_rn2(t), 0, sizeof(double) * (t + k * t), st));
  return GP_OK;
}

int gp_mbcg_precond(gp_mbcg* s, int iteration, double tolerance, void* stream) {
  if (int rc = check_state(s)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CgK v = view(s);
  const int t = s->t, k = s->k, W = 3 * t + k * t, nb = cg_nblocks(s);
  cg_freeze<<<1, 256, 0, st>>>(v, iteration, tolerance);
  GP_LAUNCH_CHECK();
  if (k > 0 && s->pc_noise > 0.0) {
    cg_cvec<<<cvec_blocks(k, t), 256, 0, st>>>(v, 1);
    GP_LAUNCH_CHECK();
  }
  if (s->n > 0 && use_wide(s)) {
    const size_t smem = pz_wide_smem(k);
    if (int rc = set_smem(cg_precond_z_wide<false>, smem)) return rc;
    cg_precond_z_wide<false><<<dim3(nb, (t + kWT - 1) / kWT), 256, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0 && use_bulk(s)) {
    const size_t smem = pz_bulk_smem(k);
    if (int rc = set_smem(cg_precond_z_bulk<false>, smem)) return rc;
    cg_precond_z_bulk<false><<<nb, 128, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0 && use_narrow(s)) {
    const size_t smem = pz_narrow_smem(k);
    if (int rc = set_smem(cg_precond_z_narrow<false>, smem)) return rc;
    cg_precond_z_narrow<false><<<nb, kZT, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  if (s->n > 0) {
    size_t smem = (kRT + (size_t)k * t) * sizeof(double);
    if (int rc = set_smem(cg_precond_z<false>, smem)) return rc;
    cg_precond_z<false><<<nb, kRT, smem, st>>>(v);
    GP_LAUNCH_CHECK();
    return finalize(s->partials, nb, W, off_gam(t, k), off_gam(t, k) + t, s->red, st);
  }
  GP_CUDA_TRY(cudaMemsetAsync(s->red + off_gam(t, k), 0, sizeof(double) * t, st));
  return GP_OK;
}

/* The whole single-device solve in one call (iterations after init_a/b/c):
 * per iteration gp_kv (P32 -> Q32) and the four phases, with one 16-byte
 * status read; the host loop stays in C, so a small-n solve pays ~10 kernel
 * launches per iteration instead of five Python round trips. */
int gp_mbcg_solve_kv(gp_mbcg* s, const gp_kv_desc* desc, float* Q32, int64_t ldq, void* kv_ws, size_t kv_ws_bytes,
                     double tolerance, int32_t* iterations_out, void* stream) {
  if (int rc = check_state(s)) return rc;
  GP_REQUIRE(desc != nullptr && iterations_out != nullptr, "gp_mbcg_solve_kv: null argument");
  GP_REQUIRE(desc->n_rows == s->n && desc->n_cols == s->n, "gp_mbcg_solve_kv: operator is %lld x %lld, state n=%lld",
             (long long)desc->n_rows, (long long)desc->n_cols, (long long)s->n);
  cudaStream_t st = (cudaStream_t)stream;
  static thread_local int32_t* hstat = nullptr;
  if (!hstat) GP_CUDA_TRY(cudaMallocHost(&hstat, 8 * sizeof(int32_t)));
  int it = 0;
  *iterations_out = 0;
  struct ImagesScope {   // the flag never outlives this call
    ~ImagesScope() { kv_images_current = false; }
  } images_scope;
  while (it < s->max_iters) {
    ++it;
    // iterations after the first reuse the distance images in kv_ws
    kv_images_current = it > 1;
    if (int rc = gp_kv(desc, s->P32, s->ld32, s->t, Q32, ldq, kv_ws, kv_ws_bytes, stream)) return rc;
    kv_images_current = false;
    if (int rc = gp_mbcg_pv(s, Q32, ldq, 0, stream)) return rc;
    if (int rc = gp_mbcg_update(s, Q32, ldq, 0, it, stream)) return rc;
    if (int rc = gp_mbcg_precond(s, it, tolerance, stream)) return rc;
    GP_CUDA_TRY(cudaMemcpyAsync(hstat, s->status, 4 * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GP_CUDA_TRY(cudaStreamSynchronize(st));
    *iterations_out = it;
    if (hstat[1] < s->t)
      return set_error(GP_ENOTPD, "operator is not positive definite: p^T A p <= 0 for column %d at iteration %d",
                       hstat[1], hstat[2]);
    if (hstat[0] == 0) break;
    if (int rc = gp_mbcg_direction(s, it, stream)) return rc;
  }
  return GP_OK;
}

int gp_mbcg_direction(gp_mbcg* s, int iteration, void* stream) {
  if (int rc = check_state(s)) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  CgK v = view(s);
  cg_beta<<<1, 256, 0, st>>>(v, iteration);
  GP_LAUNCH_CHECK();
  if (s->n > 0) {
    int64_t tot = s->n * s->t;
    int nb = (int)std::min<int64_t>((tot + 255) / 256, 8LL * num_sms());
    cg_direction<<<nb, 256, 0, st>>>(v, iteration);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}


static int nb_rows(int64_t n) {
  int64_t nb = std::min<int64_t>(2 * num_sms(), (n + 63) / 64);
  return (int)std::max<int64_t>(nb, 1);
}

int gp_coldot(int64_t n, int t, const double* A, int64_t lda, const double* B, int64_t ldb,
              double* out, double* partials, int64_t partials_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  GP_REQUIRE(t >= 1, "gp_coldot: t=%d", t);
  if (n == 0) {
    GP_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * t, st));
    return GP_OK;
  }
  int nb = nb_rows(n);
  GP_REQUIRE(partials_len >= (int64_t)nb * t, "gp_coldot: partials %lld < %lld",
             (long long)partials_len, (long long)nb * t);
  coldot_kernel<<<nb, kRT, 0, st>>>(n, t, A, lda, B, ldb, partials);
  GP_LAUNCH_CHECK();
  return finalize(partials, nb, t, 0, t, out, st);
}

int gp_lt_mul(int64_t n, int k, const double* L, int64_t ldl, const double* V, int64_t ldv, int t,
              double* out, double* partials, int64_t partials_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  GP_REQUIRE(t >= 1 && k >= 1, "gp_lt_mul: k=%d t=%d", k, t);
  if (n == 0) {
    GP_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * k * t, st));
    return GP_OK;
  }
  int nb = nb_rows(n);
  GP_REQUIRE(partials_len >= (int64_t)nb * k * t, "gp_lt_mul: partials too small");
  if (t >= kWideT) {   // GEMM-shaped (L^T L of the preconditioner factor, wide blocks)
    ltr_wide<<<dim3(nb, (t + kWT - 1) / kWT), 256, 0, st>>>(n, k, t, L, ldl, V, ldv, partials, k * t, 0, nullptr);
    GP_LAUNCH_CHECK();
    return finalize(partials, nb, k * t, 0, k * t, out, st);
  }
  size_t smem = ltmul_smem(k, t);
  if (int rc = set_smem(ltmul_kernel, smem)) return rc;
  ltmul_kernel<<<nb, kRT, smem, st>>>(n, k, L, ldl, V, ldv, t, partials);
  GP_LAUNCH_CHECK();
  return finalize(partials, nb, k * t, 0, k * t, out, st);
}

int gp_lowrank_mul(int64_t n, int k, const double* L, int64_t ldl, const double* M, int64_t ldm,
                   int t, double alpha, double beta, double* Y, int64_t ldy, void* stream) {
  GP_REQUIRE(t >= 1 && k >= 0, "gp_lowrank_mul: k=%d t=%d", k, t);
  if (n == 0) return GP_OK;
  const size_t wsm = (size_t)k * (kWT + kWLS) * sizeof(double);
  if (t >= kWideT && k > 0 && wsm <= 227 * 1024) {
    if (int rc = set_smem(lowrank_wide, wsm)) return rc;
    lowrank_wide<<<dim3((unsigned)((n + kWT - 1) / kWT), (t + kWT - 1) / kWT), 256, wsm, (cudaStream_t)stream>>>(
        n, k, L, ldl, M, ldm, t, alpha, beta, Y, ldy);
    GP_LAUNCH_CHECK();
    return GP_OK;
  }
  size_t smem = (size_t)k * t * sizeof(double);
  if (int rc = set_smem(lowrank_kernel, smem)) return rc;
  int64_t tot = n * t;
  int nb = (int)std::min<int64_t>((tot + 255) / 256, 8LL * num_sms());
  lowrank_kernel<<<nb, 256, smem, (cudaStream_t)stream>>>(n, k, L, ldl, M, ldm, t, alpha, beta, Y, ldy);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int gp_precond_factor(int64_t n, int k, const double* L, int64_t ldl, double noise, double* chol,
                      double* Binv, double* logdet_tr_dev, int32_t* info_dev, double* partials,
                      int64_t partials_len, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  GP_REQUIRE(k >= 1 && noise > 0.0, "gp_precond_factor: k=%d noise=%g", k, noise);
  // chol <- L^T L
  if (int rc = gp_lt_mul(n, k, L, ldl, L, ldl, k, chol, partials, partials_len, stream)) return rc;
  const size_t fsm = ((size_t)k * k + 3 * (size_t)k) * sizeof(double);   // matrix + pivot terms
  if (k <= 160) {
    if (int rc = set_smem(precond_factor_kernel, fsm)) return rc;
    precond_factor_kernel<<<1, 1024, fsm, st>>>(k, noise, chol, Binv, logdet_tr_dev, info_dev);
  } else {
    precond_factor_global<<<1, 1024, 0, st>>>(k, noise, chol, Binv, logdet_tr_dev, info_dev);
  }
  GP_LAUNCH_CHECK();
  // Binv currently holds X = C^{-1}; form X^T X into partials then copy
  GP_REQUIRE(partials_len >= (int64_t)k * k, "gp_precond_factor: partials too small");
  xtx_kernel<<<(k * k + 255) / 256, 256, 0, st>>>(k, Binv, partials);
  GP_LAUNCH_CHECK();
  GP_CUDA_TRY(cudaMemcpyAsync(Binv, partials, sizeof(double) * k * k, cudaMemcpyDeviceToDevice, st));
  return GP_OK;
}

}  // extern "C"
