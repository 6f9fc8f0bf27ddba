// SIMT (FFMA) fused K·V kernel, fp64 dense kernel blocks, point preparation,
// and the materialised-block product. The tcgen05 K·V kernel lives in
// kv_tc.cu; gp_kv dispatches between them.
//
// Reference semantics: kernels.py:216-308 (distances, kappa, noise on the
// global diagonal), partition.py:186-241 (row-block product, finiteness).
#include "gp_common.cuh"

#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <mutex>

namespace gp {

static thread_local char g_err[1024];
static std::atomic<unsigned long long> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int set_error(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  });
  return sms;
}

// ---------------------------------------------------------------------------
// point preparation
// ---------------------------------------------------------------------------
__global__ void prescale_kernel(const double* __restrict__ X, int64_t n, int d, int64_t ldx,
                                const double* __restrict__ ls, int n_ls, float* Xs32,
                                int64_t ld32, double* Xs64, int64_t ld64, float* norms) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float nrm = 0.f;
  int wmax = 0;
  if (Xs32) wmax = (int)ld32;
  if (Xs64 && (int)ld64 > wmax) wmax = (int)ld64;
  for (int k = 0; k < wmax; ++k) {
    double v = 0.0;
    if (k < d) v = X[i * ldx + k] / ls[n_ls == 1 ? 0 : k];
    if (Xs32 && k < ld32) {
      float f = (float)v;
      Xs32[i * ld32 + k] = f;
      nrm = fmaf(f, f, nrm);
    }
    if (Xs64 && k < ld64) Xs64[i * ld64 + k] = v;
  }
  if (norms) norms[i] = nrm;
}

// ---------------------------------------------------------------------------
// SIMT fused K·V
//   block = 256 threads, tile = 64 rows x 64 columns, thread micro-tile 4x4
//   (rows ty*4+i, columns tx*4+j); distances by direct differences
//   sum_k (xr_k - xc_k)^2 in fp32 (exact zero on the diagonal), kappa on the
//   SFU, contraction against TC right-hand sides by FFMA.
// ---------------------------------------------------------------------------
struct KvSimtArgs {
  const float* Xr; int64_t ldr; int64_t nr;
  const float* Xc; int64_t ldc; int64_t nc;
  int d;
  const float* V; int64_t ldv; int t;
  float* out; int64_t ldo;     // final output or split partials
  int64_t split_stride;        // elements between split partial buffers (0 = final)
  int64_t cols_per_split;      // multiple of 64
  float s2;
  float noise;
  int64_t diag_offset;
};

constexpr int kBM = 64, kBN = 64;

template <int TC> struct TcPad { static constexpr int v = TC <= 2 ? TC : (TC <= 4 ? 4 : (TC <= 12 ? 12 : 20)); };

template <int FAM, int TC>
__global__ void __launch_bounds__(256, 2) kv_simt_kernel(KvSimtArgs a) {
  constexpr int TCP = TcPad<TC>::v;
  extern __shared__ __align__(16) float smem[];
  const int d = a.d;
  float* sXr = smem;              // [d][64]
  float* sXc = sXr + d * kBM;     // [d][64]
  float* sV = sXc + d * kBN;      // [64 slots][TCP]
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t row0 = (int64_t)blockIdx.x * kBM;
  const int tc0 = blockIdx.z * TC;
  const int64_t cbeg = (int64_t)blockIdx.y * a.cols_per_split;
  const int64_t cend = min(a.nc, cbeg + a.cols_per_split);

  for (int idx = tid; idx < kBM * d; idx += 256) {
    int r = idx / d, k = idx - r * d;
    int64_t g = row0 + r;
    sXr[k * kBM + r] = g < a.nr ? a.Xr[g * a.ldr + k] : 0.f;
  }

  float acc[4][TC];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int c = 0; c < TC; ++c) acc[i][c] = 0.f;

  for (int64_t c0 = cbeg; c0 < cend; c0 += kBN) {
    __syncthreads();
    for (int idx = tid; idx < kBN * d; idx += 256) {
      int c = idx / d, k = idx - c * d;
      int64_t g = c0 + c;
      sXc[k * kBN + c] = g < cend ? a.Xc[g * a.ldc + k] : 0.f;
    }
    for (int idx = tid; idx < kBN * TC; idx += 256) {
      int c = idx / TC, q = idx - c * TC;
      int64_t g = c0 + c;
      int col = tc0 + q;
      float v = (g < cend && col < a.t) ? a.V[g * a.ldv + col] : 0.f;
      sV[((c & 3) * 16 + (c >> 2)) * TCP + q] = v;
    }
    __syncthreads();

    float dd[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) dd[i][j] = 0.f;
#pragma unroll 4
    for (int k = 0; k < d; ++k) {
      float4 xr = *reinterpret_cast<const float4*>(&sXr[k * kBM + ty * 4]);
      float4 xc = *reinterpret_cast<const float4*>(&sXc[k * kBN + tx * 4]);
      float rr[4] = {xr.x, xr.y, xr.z, xr.w};
      float cc[4] = {xc.x, xc.y, xc.z, xc.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float df = rr[i] - cc[j];
          dd[i][j] = fmaf(df, df, dd[i][j]);
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float* vp = &sV[(j * 16 + tx) * TCP];
      float v[TC];
      if (TC % 4 == 0) {
#pragma unroll
        for (int q = 0; q < TC; q += 4) {
          float4 t4 = *reinterpret_cast<const float4*>(vp + q);
          v[q] = t4.x; v[(q + 1) % TC] = t4.y; v[(q + 2) % TC] = t4.z; v[(q + 3) % TC] = t4.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < TC; ++q) v[q] = vp[q];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float kv = kappa_f32<FAM>(dd[i][j]);
#pragma unroll
        for (int q = 0; q < TC; ++q) acc[i][q] = fmaf(kv, v[q], acc[i][q]);
      }
    }
  }

  // fixed-order butterfly across the 16 column-threads sharing these rows
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int q = 0; q < TC; ++q) {
      float v = acc[i][q];
      v += __shfl_xor_sync(0xffffffffu, v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      acc[i][q] = v;
    }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t row = row0 + ty * 4 + i;
    if (row >= a.nr) continue;
#pragma unroll
    for (int q = 0; q < TC; ++q) {
      if ((q & 15) != tx) continue;
      int col = tc0 + q;
      if (col >= a.t) continue;
      if (a.split_stride) {
        a.out[(int64_t)blockIdx.y * a.split_stride + row * a.ldo + col] = acc[i][q];
      } else {
        float r = a.s2 * acc[i][q];
        if (a.diag_offset >= 0) r = fmaf(a.noise, a.V[(row + a.diag_offset) * a.ldv + col], r);
        a.out[row * a.ldo + col] = r;
      }
    }
  }
}

__global__ void kv_split_reduce(const float* __restrict__ ws, int S, int64_t stride, int64_t nr,
                                int t, float* out, int64_t ldo, float s2, float noise,
                                const float* __restrict__ V, int64_t ldv, int64_t diag_offset) {
  int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= nr * t) return;
  int64_t row = idx / t;
  int col = (int)(idx - row * t);
  float acc = 0.f;
  for (int s = 0; s < S; ++s) acc += ws[s * stride + row * t + col];
  float r = s2 * acc;
  if (diag_offset >= 0) r = fmaf(noise, V[(row + diag_offset) * ldv + col], r);
  out[row * ldo + col] = r;
}

int launch_split_reduce(const float* ws, int S, int64_t stride, int64_t nr, int t, float* out,
                        int64_t ldo, float s2, float noise, const float* V, int64_t ldv,
                        int64_t diag_offset, cudaStream_t st) {
  int64_t tot = nr * (int64_t)t;
  kv_split_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(ws, S, stride, nr, t, out, ldo, s2,
                                                                 noise, V, ldv, diag_offset);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

// number of column splits: a function of the COLUMN count only (so the per
// row summation order does not depend on how rows are sharded) unless the
// caller is a cross block where determinism across shards is moot.
static int kv_splits(int64_t n_rows_total_hint, int64_t nc) {
  int64_t row_tiles = (n_rows_total_hint + kBM - 1) / kBM;
  int64_t col_tiles = (nc + kBN - 1) / kBN;
  int64_t target = 4LL * num_sms();
  int64_t s = (target + row_tiles - 1) / row_tiles;
  s = std::min<int64_t>(s, 64);
  s = std::min<int64_t>(s, col_tiles);
  return (int)std::max<int64_t>(s, 1);
}

static int pick_tc(int t) {
  if (t <= 1) return 1;
  if (t <= 2) return 2;
  if (t <= 4) return 4;
  if (t <= 8) return 8;
  if (t <= 12) return 12;
  return 16;
}

static int64_t split_hint_rows(const gp_kv_desc* d) {
  // training operator (square): use the column count so every shard splits
  // identically; cross blocks: the actual rows
  return d->diag_offset >= 0 || d->Xr == d->Xc ? d->n_cols : d->n_rows;
}

size_t kv_simt_workspace(const gp_kv_desc* d, int t) {
  int S = kv_splits(split_hint_rows(d), d->n_cols);
  if (S <= 1) return 0;
  return (size_t)S * (size_t)d->n_rows * (size_t)t * sizeof(float);
}

template <int FAM, int TC>
static int launch_simt_tc(const KvSimtArgs& a, int S, cudaStream_t st) {
  size_t smem = (size_t)(2 * a.d * 64 + 64 * TcPad<TC>::v) * sizeof(float);
  auto kern = kv_simt_kernel<FAM, TC>;
  if (smem > 48 * 1024) GP_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)((a.nr + kBM - 1) / kBM), (unsigned)S, (unsigned)((a.t + TC - 1) / TC));
  kern<<<grid, 256, smem, st>>>(a);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

template <int FAM>
static int launch_simt_fam(const KvSimtArgs& a, int S, int tc, cudaStream_t st) {
  switch (tc) {
    case 1: return launch_simt_tc<FAM, 1>(a, S, st);
    case 2: return launch_simt_tc<FAM, 2>(a, S, st);
    case 4: return launch_simt_tc<FAM, 4>(a, S, st);
    case 8: return launch_simt_tc<FAM, 8>(a, S, st);
    case 12: return launch_simt_tc<FAM, 12>(a, S, st);
    default: return launch_simt_tc<FAM, 16>(a, S, st);
  }
}

int kv_simt(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo,
            void* ws, size_t ws_bytes, cudaStream_t st) {
  GP_REQUIRE(desc->d >= 1 && desc->d <= 256, "gp_kv: d=%d outside [1, 256]", desc->d);
  int S = kv_splits(split_hint_rows(desc), desc->n_cols);
  size_t need = kv_simt_workspace(desc, t);
  GP_REQUIRE(ws_bytes >= need && (need == 0 || ws != nullptr),
             "gp_kv: workspace of %zu bytes required, %zu given", need, ws_bytes);
  KvSimtArgs a;
  a.Xr = desc->Xr; a.ldr = desc->ldr; a.nr = desc->n_rows;
  a.Xc = desc->Xc; a.ldc = desc->ldc; a.nc = desc->n_cols;
  a.d = desc->d; a.V = V; a.ldv = ldv; a.t = t;
  a.s2 = (float)desc->outputscale; a.noise = (float)desc->noise; a.diag_offset = desc->diag_offset;
  int64_t col_tiles = (desc->n_cols + kBN - 1) / kBN;
  int64_t tiles_per_split = (col_tiles + S - 1) / S;
  a.cols_per_split = tiles_per_split * kBN;
  S = (int)((col_tiles + tiles_per_split - 1) / tiles_per_split);
  if (S > 1) {
    a.out = static_cast<float*>(ws);
    a.ldo = t;
    a.split_stride = desc->n_rows * (int64_t)t;
  } else {
    a.out = out; a.ldo = ldo; a.split_stride = 0;
  }
  int tc = pick_tc(t);
  int rc = desc->family == GP_FAMILY_RBF ? launch_simt_fam<GP_FAMILY_RBF>(a, S, tc, st)
                                         : launch_simt_fam<GP_FAMILY_MATERN32>(a, S, tc, st);
  if (rc) return rc;
  if (S > 1) {
    int64_t tot = desc->n_rows * (int64_t)t;
    kv_split_reduce<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        static_cast<const float*>(ws), S, a.split_stride, desc->n_rows, t, out, ldo, a.s2, a.noise, V,
        ldv, desc->diag_offset);
    GP_LAUNCH_CHECK();
  }
  return GP_OK;
}

// ---------------------------------------------------------------------------
// fp64 dense kernel block
// ---------------------------------------------------------------------------
__global__ void kernel_block_kernel(int fam, int d, const double* __restrict__ Xr, int64_t ldr,
                                    int64_t nr, const double* __restrict__ Xc, int64_t ldc,
                                    int64_t nc, double s2, double noise, int64_t diag_offset,
                                    double* out, int64_t ldo) {
  int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int64_t i = blockIdx.y + (int64_t)blockIdx.z * 65535;
  if (i >= nr || j >= nc) return;
  double r2 = 0.0;
  for (int k = 0; k < d; ++k) {
    double df = Xr[i * ldr + k] - Xc[j * ldc + k];
    r2 = fma(df, df, r2);
  }
  double v = s2 * kappa_f64(fam, r2);
  if (diag_offset >= 0 && j == i + diag_offset) v += noise;
  out[i * ldo + j] = v;
}

// ---------------------------------------------------------------------------
// materialised row block x V (fp64) with non-finite detection
// ---------------------------------------------------------------------------
__global__ void block_mvm_kernel(const double* __restrict__ B, int64_t nr, int64_t nc, int64_t ldb,
                                 const double* __restrict__ V, int64_t ldv, int t, double* out,
                                 int64_t ldo, int32_t* first_bad) {
  int64_t row = blockIdx.x;
  __shared__ double red[8][32];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const double* brow = B + row * ldb;
  for (int c0 = 0; c0 < t; c0 += 32) {
    int cw = min(32, t - c0);
    double acc[32];
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[q] = 0.0;
    for (int64_t j = threadIdx.x; j < nc; j += blockDim.x) {
      double b = brow[j];
      if (c0 == 0 && !isfinite(b)) bad = 1;
#pragma unroll
      for (int q = 0; q < 32; ++q)
        if (q < cw) acc[q] = fma(b, V[j * ldv + c0 + q], acc[q]);
    }
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 32; ++q) {
      double v = warp_sum(acc[q]);
      if (lane == q) red[w][q] = v;
    }
    __syncthreads();
    if (threadIdx.x < cw) {
      double s = 0.0;
      for (int ww = 0; ww < (int)(blockDim.x >> 5); ++ww) s += red[ww][threadIdx.x];
      out[row * ldo + c0 + threadIdx.x] = s;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && bad) atomicMin(first_bad, (int32_t)row);
}

}  // namespace gp

using namespace gp;

extern "C" {

const char* gp_last_error(void) { return gp::g_err; }
int gp_version(void) { return 1; }
uint64_t gp_launch_count(void) { return gp::g_launches.load(std::memory_order_relaxed); }

int gp_prescale(const double* X, int64_t n, int d, int64_t ldx, const double* ls, int n_ls,
                float* Xs32, int64_t ld32, double* Xs64, int64_t ld64, float* norms32,
                void* stream) {
  GP_REQUIRE(n >= 0 && d >= 1, "gp_prescale: bad shape n=%lld d=%d", (long long)n, d);
  GP_REQUIRE(n_ls == 1 || n_ls == d, "gp_prescale: %d lengthscales for d=%d", n_ls, d);
  GP_REQUIRE(!Xs32 || ld32 >= d, "gp_prescale: ld32 < d");
  GP_REQUIRE(!Xs64 || ld64 >= d, "gp_prescale: ld64 < d");
  if (n == 0) return GP_OK;
  prescale_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      X, n, d, ldx, ls, n_ls, Xs32, ld32, Xs64, ld64, norms32);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int gp_kernel_block(int family, int d, const double* Xr, int64_t ldr, int64_t n_rows,
                    const double* Xc, int64_t ldc, int64_t n_cols, double outputscale,
                    double noise, int64_t diag_offset, double* out, int64_t ldo, void* stream) {
  GP_REQUIRE(family == 0 || family == 1, "gp_kernel_block: unknown family %d", family);
  if (n_rows == 0 || n_cols == 0) return GP_OK;
  int64_t zb = (n_rows + 65534) / 65535;
  dim3 grid((unsigned)((n_cols + 127) / 128), (unsigned)std::min<int64_t>(n_rows, 65535), (unsigned)zb);
  kernel_block_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(family, d, Xr, ldr, n_rows, Xc, ldc,
                                                             n_cols, outputscale, noise,
                                                             diag_offset, out, ldo);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

int gp_block_mvm(const double* block, int64_t n_rows, int64_t n_cols, int64_t ldb, const double* V,
                 int64_t ldv, int t, double* out, int64_t ldo, int32_t* first_bad_row_dev,
                 void* stream) {
  GP_REQUIRE(t >= 1, "gp_block_mvm: t=%d", t);
  if (n_rows == 0) return GP_OK;
  block_mvm_kernel<<<(unsigned)n_rows, 256, 0, (cudaStream_t)stream>>>(
      block, n_rows, n_cols, ldb, V, ldv, t, out, ldo, first_bad_row_dev);
  GP_LAUNCH_CHECK();
  return GP_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// gp_kv dispatcher (SIMT / tcgen05)
// ---------------------------------------------------------------------------
namespace gp {
int kv_tc(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo,
          void* ws, size_t ws_bytes, cudaStream_t st);
size_t kv_tc_workspace(const gp_kv_desc* desc, int t);
bool kv_tc_supported(const gp_kv_desc* desc, int t);
int kv_sym(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo,
           void* ws, size_t ws_bytes, cudaStream_t st);
size_t kv_sym_workspace(const gp_kv_desc* desc, int t);
bool kv_sym_supported(const gp_kv_desc* desc, int t);
int64_t kv_sym_acc_ld(const gp_kv_desc* desc);
int kv_sym_partial(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, int part, int nparts,
                   long long* acc, int* bad, void* ws, size_t ws_bytes, cudaStream_t st);
int kv_sym_finalize(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, const long long* acc,
                    const int* bad, int64_t acc_row0, int64_t row0, int64_t row1, float* out, int64_t ldo, void* ws,
                    size_t ws_bytes, cudaStream_t st);
int kv_wide(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo,
            void* ws, size_t ws_bytes, cudaStream_t st);
size_t kv_wide_workspace(const gp_kv_desc* desc, int t);
bool kv_wide_supported(const gp_kv_desc* desc, int t);
}  // namespace gp

extern "C" {

static bool use_tc(const gp_kv_desc* d, int t) {
  if (d->algo == 1) return false;
  if (d->algo == 2 || d->algo == 3) return true;
  return gp_has_tcgen05() && gp::kv_tc_supported(d, t);
}
// auto: the symmetric kernel whenever the call is the whole square training
// operator (each unordered pair evaluated once) with enough work items to
// fill the SMs: below ~12k points its 4 x 4-tile items leave most SMs idle and
// the row-tiled kernel is faster (n = 8192: 0.11 vs 0.18 ms; n = 16384: 0.24
// vs 0.19 ms, profiles/r01d_small_n.md). GP_KV_NO_SYM=1 opts out.
constexpr int64_t kSymAutoMinPoints = 12288;
static bool use_sym(const gp_kv_desc* d, int t) {
  if (d->algo == 3) return true;
  if (d->algo != 0 || !gp_has_tcgen05() || !gp::kv_sym_supported(d, t)) return false;
  if (d->n_rows < kSymAutoMinPoints) return false;
  const char* e = getenv("GP_KV_NO_SYM");
  return !(e && *e == '1');
}

size_t gp_kv_workspace_bytes(const gp_kv_desc* desc, int t) {
  if (!desc || t < 1) return 0;
  size_t a = gp::kv_simt_workspace(desc, t);
  size_t b = gp_has_tcgen05() ? gp::kv_tc_workspace(desc, t) : 0;
  size_t c = gp_has_tcgen05() ? gp::kv_sym_workspace(desc, t) : 0;
  size_t w = gp_has_tcgen05() ? gp::kv_wide_workspace(desc, t) : 0;
  a = a > b ? a : b;
  a = a > c ? a : c;
  return a > w ? a : w;
}

int gp_kv(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, float* out, int64_t ldo,
          void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(desc != nullptr, "gp_kv: null descriptor");
  GP_REQUIRE(desc->family == GP_FAMILY_RBF || desc->family == GP_FAMILY_MATERN32,
             "gp_kv: unknown kernel family %d", desc->family);
  GP_REQUIRE(t >= 1 && ldv >= t && ldo >= t, "gp_kv: t=%d ldv=%lld ldo=%lld", t, (long long)ldv,
             (long long)ldo);
  GP_REQUIRE(desc->n_rows >= 0 && desc->n_cols >= 0, "gp_kv: negative shape");
  GP_REQUIRE(desc->ldr >= desc->d && desc->ldc >= desc->d, "gp_kv: point leading dim < d");
  GP_REQUIRE(desc->diag_offset < 0 || desc->diag_offset + desc->n_rows <= desc->n_cols,
             "gp_kv: diagonal offset outside the column range");
  cudaStream_t st = (cudaStream_t)stream;
  if (desc->n_rows == 0) return GP_OK;
  if (desc->n_cols == 0) {
    for (int64_t r = 0; r < desc->n_rows; ++r)
      GP_CUDA_TRY(cudaMemsetAsync(out + r * ldo, 0, sizeof(float) * t, st));
    return GP_OK;
  }
  if (use_sym(desc, t)) {
    GP_REQUIRE(gp::kv_sym_supported(desc, t), "gp_kv: shape unsupported by the symmetric tcgen05 kernel");
    return gp::kv_sym(desc, V, ldv, t, out, ldo, workspace, workspace_bytes, st);
  }
  if (desc->algo != 1 && t > 16 && gp_has_tcgen05() && gp::kv_wide_supported(desc, t))
    return gp::kv_wide(desc, V, ldv, t, out, ldo, workspace, workspace_bytes, st);
  if (use_tc(desc, t)) {
    GP_REQUIRE(gp_has_tcgen05(), "gp_kv: tcgen05 kernel requested but not compiled in");
    GP_REQUIRE(gp::kv_tc_supported(desc, t), "gp_kv: shape unsupported by the tcgen05 kernel");
    return gp::kv_tc(desc, V, ldv, t, out, ldo, workspace, workspace_bytes, st);
  }
  return gp::kv_simt(desc, V, ldv, t, out, ldo, workspace, workspace_bytes, st);
}

int gp_kv_sym_supported(const gp_kv_desc* desc, int t) {
  return desc != nullptr && gp_has_tcgen05() && gp::kv_sym_supported(desc, t) ? 1 : 0;
}

int gp_kv_sym_auto(const gp_kv_desc* desc, int t) {
  if (desc == nullptr || t < 1) return 0;
  gp_kv_desc d = *desc;
  d.algo = 0;
  return use_sym(&d, t) ? 1 : 0;
}

int64_t gp_kv_sym_acc_ld(const gp_kv_desc* desc) {
  return desc != nullptr && desc->n_rows > 0 ? gp::kv_sym_acc_ld(desc) : 0;
}

int gp_kv_sym_partial(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, int part, int nparts,
                      int64_t* acc, int32_t* bad, void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(desc != nullptr && V != nullptr && acc != nullptr && bad != nullptr, "gp_kv_sym_partial: null argument");
  GP_REQUIRE(gp_has_tcgen05(), "gp_kv_sym_partial: tcgen05 kernel not compiled in");
  GP_REQUIRE(t >= 1 && ldv >= t, "gp_kv_sym_partial: t=%d ldv=%lld", t, (long long)ldv);
  return gp::kv_sym_partial(desc, V, ldv, t, part, nparts, reinterpret_cast<long long*>(acc),
                            reinterpret_cast<int*>(bad), workspace, workspace_bytes, (cudaStream_t)stream);
}

int gp_kv_sym_finalize(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, const int64_t* acc,
                       const int32_t* bad, int64_t acc_row0, int64_t row0, int64_t row1, float* out, int64_t ldo,
                       void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(desc != nullptr && V != nullptr && acc != nullptr && bad != nullptr && out != nullptr,
             "gp_kv_sym_finalize: null argument");
  GP_REQUIRE(t >= 1 && ldv >= t && ldo >= t, "gp_kv_sym_finalize: t=%d ldv=%lld ldo=%lld", t, (long long)ldv,
             (long long)ldo);
  return gp::kv_sym_finalize(desc, V, ldv, t, reinterpret_cast<const long long*>(acc),
                             reinterpret_cast<const int*>(bad), acc_row0, row0, row1, out, ldo, workspace, workspace_bytes,
                             (cudaStream_t)stream);
}

}  // extern "C"
