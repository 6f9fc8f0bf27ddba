/*
 * gpbbmm.h — C ABI of the B200-native exact-GP BBMM hot path.
 *
 * Drop-in boundary for the reference package blockgp 0.1.0
 * (/root/reference/pkg/src/blockgp). The reference is pure Python, so it has
 * no FFI of its own; each entry point below replaces one operator seam of the
 * reference (cited file:line) and is bound from the Python host mirror
 * (paper_1903_08114_b200/_lib.py) through ctypes. INTEGRATION.md shows the
 * binding a blockgp maintainer would add.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the name ends in _host.
 *   - Matrices are row-major with an explicit leading dimension (elements).
 *   - `stream` is a cudaStream_t passed as void*; every call is stream-ordered
 *     and asynchronous unless documented otherwise.
 *   - The library allocates nothing that outlives a call: callers own every
 *     buffer, including workspaces sized by the *_workspace_bytes queries.
 *   - Every entry point returns a status (GP_OK = 0). gp_last_error() returns
 *     a thread-local message for the last failure on the calling thread.
 */
#ifndef GPBBMM_H
#define GPBBMM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (mapped to ValueError / NumericError / ConvergenceError
 *      by the host mirror; errors.py:4-15 of the reference) ---------------- */
#define GP_OK 0
#define GP_EINVAL 1      /* invalid argument            -> ValueError        */
#define GP_ENONFINITE 2  /* non-finite kernel entry     -> NumericError      */
#define GP_ENOTPD 3      /* p^T A p <= 0 / failed chol  -> NumericError      */
#define GP_ECUDA 4       /* CUDA runtime failure        -> RuntimeError      */
#define GP_EUNSUPPORTED 5 /* shape outside compiled kernels -> ValueError    */
#define GP_ENCCL 6       /* NCCL failure                -> RuntimeError      */

#define GP_FAMILY_RBF 0
#define GP_FAMILY_MATERN32 1

const char* gp_last_error(void);
int gp_version(void);
/* number of kernels this library has launched since it was loaded */
uint64_t gp_launch_count(void);
/* 1 if the tcgen05 (sm_100a tensor-core) K·V kernel is compiled in. */
int gp_has_tcgen05(void);

/* ---- point preparation -------------------------------------------------
 * Xs = X / lengthscale (per column when n_ls == d, shared when n_ls == 1),
 * written as fp32 (ld32 >= d, zero padded) and/or fp64 (ld64 >= d).
 * Replaces the per-call rescaling of kernels.py:266 and :301-302.
 * Either output may be NULL. norms32 (optional) = ||Xs_i||^2 in fp32. */
int gp_prescale(const double* X, int64_t n, int d, int64_t ldx,
                const double* lengthscales, int n_ls,
                float* Xs32, int64_t ld32, double* Xs64, int64_t ld64,
                float* norms32, void* stream);

/* ---- fused on-the-fly kernel-matrix multiply ---------------------------
 * out[i, :] = s2 * sum_j kappa(||xr_i - xc_j||^2) V[j, :]
 *             (+ noise * V[i + diag_offset, :] when diag_offset >= 0)
 * for i < n_rows, j < n_cols, t right-hand sides. The n_rows x n_cols kernel
 * block is never materialised (tiles live in registers / SMEM / TMEM).
 * Replaces kernels.training_mvm_oracle + partition.partitioned_mvm
 * (kernels.py:293-316, partition.py:186-241) and, with diag_offset = -1,
 * kernels.cross_mvm_oracle (kernels.py:319-325, predictor.py:130-131).
 * Xr/Xc are prescaled fp32 points (gp_prescale). The row-tiled kernels' per-row
 * reduction order is fixed by n_cols alone, so their results are bitwise
 * independent of how rows are sharded across devices (test_partition.py:92-102).
 * `algo`: 0 = auto, 1 = SIMT FFMA kernel, 2 = tcgen05 kernel, 3 = symmetric
 * tcgen05 kernel (whole square operator only: Xr == Xc, all rows, self_offset
 * 0; each unordered pair evaluated once, contributions summed in 64-bit fixed
 * point, so the result is bitwise reproducible but not bitwise equal to
 * algo 2). Auto picks 3 for the whole square operator when d <= 14 and
 * t <= 16 (GP_KV_NO_SYM=1 opts out), else 2 (t <= 16) or the wide kernel. */
typedef struct gp_kv_desc {
  int32_t family;        /* GP_FAMILY_* */
  int32_t d;             /* input dimension */
  const float* Xr; int64_t ldr; int64_t n_rows;
  const float* Xc; int64_t ldc; int64_t n_cols;
  double outputscale;    /* s^2 */
  double noise;          /* sigma^2 */
  int64_t diag_offset;   /* global column of row 0 for the noise term, -1 = none */
  int32_t algo;
  int32_t reserved;
  int64_t self_offset;   /* row i of Xr IS column i + self_offset of Xc (-1 = unrelated):
                            that entry is evaluated at r2 = 0 exactly, as the
                            reference's clamp does (kernels.py:216-222) */
} gp_kv_desc;

size_t gp_kv_workspace_bytes(const gp_kv_desc* desc, int t);
int gp_kv(const gp_kv_desc* desc, const float* V, int64_t ldv, int t,
          float* out, int64_t ldo, void* workspace, size_t workspace_bytes,
          void* stream);

/* Symmetric schedule split across devices (multi-GPU row-sharded solver,
 * partition.py:155-183 / PAPER:196-212 shard rows; here the unordered tile
 * pairs are sharded instead, so every device does half the transcendental
 * work of its share):
 *   gp_kv_sym_partial  — 64-bit fixed-point sums of the work items
 *                        L = part (mod nparts) of the whole square operator
 *                        (Xr == Xc, all n rows, V = all n rows) into
 *                        acc (t * acc_ld int64, acc_ld = gp_kv_sym_acc_ld =
 *                        n rounded up to 128; row-block major: element
 *                        (row i, column c) at ((i / 128) t + c) 128 + i % 128,
 *                        so the rows [128 a, 128 b) are the contiguous slice
 *                        [128 a t, 128 b t)) and per-row non-finite flags bad
 *                        (acc_ld int32); both are overwritten.
 *   (caller)           — element-wise integer sums of acc / bad over the parts,
 *                        e.g. an NCCL int64 reduce-scatter that leaves each rank
 *                        the slice of its own 128-aligned rows: deterministic,
 *                        and bitwise equal to the single-device gp_kv result.
 *   gp_kv_sym_finalize — rows [row0, row1) of s2 K V (+ noise V[i + diag_offset])
 *                        from the summed accumulator, NaN rows where bad != 0;
 *                        acc / bad hold the rows from acc_row0 on (a multiple
 *                        of 128, <= row0: 0 for the whole accumulator, the
 *                        rank's first row for its reduce-scattered slice).
 * Workspace: gp_kv_workspace_bytes(desc, t). gp_kv_sym_supported tells
 * whether the descriptor qualifies (d <= 14, t <= 16, whole square operator). */
int gp_kv_sym_supported(const gp_kv_desc* desc, int t);
/* 1 when gp_kv with algo 0 picks the symmetric kernel for this descriptor
 * (supported and at least ~12k points, where its work items fill the SMs);
 * a multi-device caller uses it to make the same choice as one device. */
int gp_kv_sym_auto(const gp_kv_desc* desc, int t);
int64_t gp_kv_sym_acc_ld(const gp_kv_desc* desc);
int gp_kv_sym_partial(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, int part, int nparts,
                      int64_t* acc, int32_t* bad, void* workspace, size_t workspace_bytes, void* stream);
int gp_kv_sym_finalize(const gp_kv_desc* desc, const float* V, int64_t ldv, int t, const int64_t* acc,
                       const int32_t* bad, int64_t acc_row0, int64_t row0, int64_t row1, float* out,
                       int64_t ldo, void* workspace, size_t workspace_bytes, void* stream);

/* Dense fp64 kernel block (kernels.py:247-270 kernel_block, :293-308
 * kernel_rows): out[i,j] = s2 kappa(xr_i, xc_j) (+ noise where
 * j == i + diag_offset, diag_offset >= 0). Xr/Xc are prescaled fp64. */
int gp_kernel_block(int family, int d, const double* Xr, int64_t ldr, int64_t n_rows,
                    const double* Xc, int64_t ldc, int64_t n_cols, double outputscale,
                    double noise, int64_t diag_offset, double* out, int64_t ldo,
                    void* stream);

/* Row-block product for arbitrary (materialised) row blocks — the path of
 * partitioned_mvm with a user row oracle (partition.py:224-237):
 * out = block @ V (fp64); *first_bad_row_dev receives the first row holding a
 * non-finite entry, or n_rows if all are finite. */
int gp_block_mvm(const double* block, int64_t n_rows, int64_t n_cols, int64_t ldb,
                 const double* V, int64_t ldv, int t, double* out, int64_t ldo,
                 int32_t* first_bad_row_dev, void* stream);

/* fp64 fused K̂·V without materialising the block: the precision of the
 * reference's partitioned_mvm(training_mvm_oracle / cross_mvm_oracle),
 * predict_mean and verify_cache (partition.py:186-241, kernels.py:293-325,
 * predictor.py:100-132; all float64). Xr / Xc are prescaled fp64 points
 * (x / lengthscale); out = s2 kappa(Xr, Xc) V (+ noise V[row + diag_offset]
 * when diag_offset >= 0). *first_bad_row_dev (if non-NULL, initialised by
 * the caller to n_rows) receives the first row with a non-finite value.
 * Deterministic (fixed-order column-split reduction). Workspace:
 * gp_kv_f64_workspace_bytes(n_rows, n_cols, t). */
size_t gp_kv_f64_workspace_bytes(int64_t n_rows, int64_t n_cols, int t);
int gp_kv_f64(int family, int d, const double* Xr, int64_t ldr, int64_t n_rows,
              const double* Xc, int64_t ldc, int64_t n_cols, double outputscale,
              double noise, int64_t diag_offset, const double* V, int64_t ldv, int t,
              double* out, int64_t ldo, int32_t* first_bad_row_dev, void* workspace,
              size_t workspace_bytes, void* stream);

/* ---- mBCG (cg.py:84-164) ------------------------------------------------
 * Device-resident batched PCG. The host drives iterations phase by phase so
 * a sharded (multi-GPU) caller can all-reduce the `red` payload between
 * phases:  red = [pv : t | rn2 : t | LtR : k*t | gam : t]  (fp64).
 * Per iteration:
 *   gp_kv(P32 gathered)            Q32 = K P      (rows of this shard)
 *   gp_mbcg_pv(Q)                  red.pv        -> all-reduce
 *   gp_mbcg_update(Q, it)          alpha, U, R, red.rn2, red.LtR -> all-reduce
 *   gp_mbcg_precond(it, tol)       rel, freeze, Z, red.gam        -> all-reduce
 *   gp_mbcg_direction(it)          beta, P, P32
 * status[0] = active columns after the freeze, status[1] = first column
 * with p^T A p <= 0 or non-finite (INT32_MAX if none), status[2] = the
 * iteration at which it happened. */
typedef struct gp_mbcg {
  int64_t n;             /* rows on this shard */
  int32_t t;             /* right-hand sides */
  int32_t k;             /* preconditioner rank (0 = none) */
  int64_t ld;            /* leading dim of U, R, P, Z (>= t) */
  int64_t ld32;          /* leading dim of P32 (>= t) */
  double* U; double* R; double* P; double* Z;
  float* P32;            /* fp32 copy of P: the K·V operand */
  double noise;          /* operator K + noise I */
  const double* L; int64_t ldl;   /* this shard's rows of the n x k factor */
  const double* Binv;    /* k x k, (pc_noise I + L^T L)^{-1}, row-major */
  double pc_noise;       /* preconditioner diagonal */
  double* bnorm;         /* [t] */
  double* gamma;         /* [t] */
  double* red;           /* [3t + k t] reduction payload */
  double* cbuf;          /* [k t] B^{-1} L^T R */
  double* alpha_hist;    /* [max_iters t] */
  double* beta_hist;     /* [max_iters t] */
  double* rel;           /* [t] */
  double* rel_hist;      /* [max_iters t] */
  int32_t* active;       /* [t] */
  int32_t* converged;    /* [t] */
  int32_t* status;       /* [4] */
  double* partials;      /* block partial sums */
  int64_t partials_len;  /* doubles available in `partials` */
  int32_t max_iters;
  int32_t nblocks;       /* 0 = library default */
} gp_mbcg;

int64_t gp_mbcg_partials_len(int64_t n, int t, int k);
/* init: R = B, U = 0, red.rn2 = ||B_j||^2, red.LtR = L^T B (local) */
int gp_mbcg_init_a(gp_mbcg* s, const double* B, int64_t ldb, void* stream);
/* after all-reduce of red: bnorm, Z = P^{-1} R, P = Z, P32, red.gam = r^T z */
int gp_mbcg_init_b(gp_mbcg* s, void* stream);
/* after all-reduce of red.gam: gamma = gam, active = 1 */
int gp_mbcg_init_c(gp_mbcg* s, void* stream);
/* Q = K P for this shard's rows: fp32 from gp_kv (q_is_f64 = 0; the
 * noise * P term is added in fp64 inside the CG kernels) or an fp64 result of
 * a user operator that already includes any diagonal (q_is_f64 = 1, and the
 * state's `noise` should then be 0). */
int gp_mbcg_pv(gp_mbcg* s, const void* Q, int64_t ldq, int q_is_f64, void* stream);
int gp_mbcg_update(gp_mbcg* s, const void* Q, int64_t ldq, int q_is_f64, int iteration,
                   void* stream);
int gp_mbcg_precond(gp_mbcg* s, int iteration, double tolerance, void* stream);
int gp_mbcg_direction(gp_mbcg* s, int iteration, void* stream);
/* The complete single-device solve after gp_mbcg_init_{a,b,c}: iterations of
 * gp_kv (desc applied to P32 into Q32; desc must be the square operator of
 * this state's n rows, noise added by the phases) and the four phases until
 * every column is frozen or max_iters; *iterations_out = iterations run.
 * The reference's mbcg_solve (cg.py:84-164) with a kernel operator. */
int gp_mbcg_solve_kv(gp_mbcg* s, const gp_kv_desc* desc, float* Q32, int64_t ldq, void* kv_ws, size_t kv_ws_bytes,
                     double tolerance, int32_t* iterations_out, void* stream);

/* ---- column reductions / low-rank products (fp64) ----------------------- */
/* out[j] = sum_i A[i,j] * B[i,j], deterministic fixed-order reduction */
int gp_coldot(int64_t n, int t, const double* A, int64_t lda, const double* B,
              int64_t ldb, double* out, double* partials, int64_t partials_len,
              void* stream);
/* out (k x t) = L^T V */
int gp_lt_mul(int64_t n, int k, const double* L, int64_t ldl, const double* V,
              int64_t ldv, int t, double* out, double* partials, int64_t partials_len,
              void* stream);
/* Y = beta * Y + alpha * L M,  L n x k, M k x t (row-major, ldm) */
int gp_lowrank_mul(int64_t n, int k, const double* L, int64_t ldl, const double* M,
                   int64_t ldm, int t, double alpha, double beta, double* Y,
                   int64_t ldy, void* stream);

/* ---- preconditioner (precond.py:58-174, likelihood.py:74-91) ------------
 * Greedy rank-k pivoted Cholesky of the NOISELESS kernel matrix with
 * constant diagonal s2: argmax pivot (lowest index on ties), early stop when
 * the residual diagonal is <= 0, clamp at 0. fp64 throughout.
 * Xs64 are prescaled fp64 points. Outputs: L (n x ldl), pivots_dev (k),
 * resid_diag (n), info_dev[0] = achieved rank. */
size_t gp_pivchol_workspace_bytes(int64_t n, int k);
int gp_pivchol(int family, int d, const double* Xs64, int64_t ldx, int64_t n,
               double outputscale, int k, double* L, int64_t ldl,
               int64_t* pivots_dev, double* resid_diag, int32_t* info_dev,
               void* workspace, size_t workspace_bytes, void* stream);
/* B = noise I + L^T L; chol (lower) ; Binv = B^{-1}; logdet_tr_dev[0] =
 * 2 sum log diag(chol), [1] = tr(B^{-1}); info_dev[0] != 0 on failure. */
int gp_precond_factor(int64_t n, int k, const double* L, int64_t ldl, double noise,
                      double* chol, double* Binv, double* logdet_tr_dev,
                      int32_t* info_dev, double* partials, int64_t partials_len,
                      void* stream);

/* ---- gradient forms (likelihood.py:166-216, kernels.py:332-410) ---------
 * For every geometric hyperparameter p returns sum_ij (dK/dtheta_p)_ij H_ij
 * with H = Y R^T (Y, R: n x w fp32), using prescaled fp32 points:
 *   out[0]     : p = outputscale   (dK/ds2 = kappa)
 *   out[1]     : shared lengthscale: sum eps * D * H
 *   out[1 + i] : ARD lengthscale i:  sum eps * (xs_i - xs'_i)^2 * H
 * with eps = e^{-D/2} (RBF) or 3 e^{-sqrt3 r} (Matern) (the host multiplies by
 * s2 and divides by l). fp64 output, deterministic fixed-order reduction. */
size_t gp_grad_forms_workspace_bytes(int64_t n_rows, int64_t n_cols, int d, int ard, int w);
/* self_offset: row i of Xr is column i + self_offset of Xc (-1 = unrelated);
 * algo: 0 = auto (tcgen05 per-entry epilogue, grad_tc.cu, when d + 2 <= 32 and
 *       w <= 128; ARD beyond that: per-dimension sums on the tensor core, grad_ard.cu;
 *       else SIMT), 1 = SIMT, 2 = tcgen05 per-entry epilogue, 3 = tcgen05 ARD sums */
int gp_grad_forms(int family, int d, int ard, const float* Xr, int64_t ldr, int64_t n_rows,
                  const float* Xc, int64_t ldc, int64_t n_cols, double outputscale,
                  const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w,
                  int64_t self_offset, int algo, double* out, void* workspace,
                  size_t workspace_bytes, void* stream);

/* ---- data preparation for the training protocol ---------------------------
 * data.py:163-196 (split_and_whiten), trainer.py:323-330 (pretraining subset).
 * Column mean and population std (ddof 0, two-pass, fp64, fixed-order
 * reductions) over the m rows `rows` (nullptr: rows 0..m-1) of X; with
 * unit_if_zero a zero std is reported as 1; std_out may be nullptr. */
int64_t gp_column_moments_workspace_len(int64_t m, int d);
int gp_column_moments(const double* X, int64_t ldx, int64_t m, int d, const int64_t* rows, double* mean,
                      double* std_out, int unit_if_zero, double* workspace, int64_t workspace_len, void* stream);
/* out = (X - mean) / std row-wise (the whitening of data.py:191-194) */
int gp_standardize(const double* X, int64_t ldx, int64_t n, int d, const double* mean, const double* std_in,
                   double* out, int64_t ldo, void* stream);
/* out[i, :] = X[idx[i], :]; *bad_dev = 1 if an index is outside [0, n_src) */
int gp_gather_rows(const double* X, int64_t ldx, int64_t n_src, const int64_t* idx, int64_t m, int d, double* out,
                   int64_t ldo, int* bad_dev, void* stream);

/* Symmetric schedule of the same forms for the square training operator
 * (rows = columns = X, likelihood.py:166-216): the caller passes Y, R with
 * Y R^T SYMMETRIC (e.g. Y_s = [a/2 | -(S-W)/(4t) | -W/(4t) | L B^-1/(2 noise)],
 * R_s = [a | W | S-W | L], so Y_s R_s^T = (H + H^T)/2 has the same sums
 * against every symmetric dK/dtheta as H); each unordered 128 x 128 block
 * pair is evaluated once, halving the kernel-entry work. Replaces the
 * reference's run_row_blocks(grad_row_products) pass (likelihood.py:182-189). */
/* 1 if the symmetric per-entry tcgen05 kernel takes the shape (d + 2 <= 32,
 * w <= 128); otherwise gp_grad_forms_sym evaluates the full square through
 * gp_grad_forms, and the caller does better with the (narrower) non-symmetric
 * operands Y = [a/2, -(S-W)/(2t), L B^-1/(2 noise)], R = [a, W, L] there. */
int gp_grad_forms_sym_supported(int64_t n, int d, int ard, int w);
size_t gp_grad_forms_sym_workspace_bytes(int64_t n, int d, int ard, int w);
int gp_grad_forms_sym(int family, int d, int ard, const float* X, int64_t ldx, int64_t n, double outputscale,
                      const float* Y, int64_t ldy, const float* R, int64_t ldrr, int w, double* out,
                      void* workspace, size_t workspace_bytes, void* stream);

/* ---- single-process multi-GPU collectives (NCCL) ------------------------
 * One host thread drives every device with NCCL group calls (SURVEY §8(b)
 * "Collectives"; the reference's equivalent is the thread WorkerPool that
 * runs the row blocks of one MVM in parallel, partition.py:46-57, :155-183).
 * The work items of gp_kv_sym_partial are split over the devices and the
 * fixed-point partial sums reduce-scattered by row, so the product is
 * bitwise that of one device. NCCL is resolved at run time (libnccl.so.2);
 * gp_comm_available() reports whether it was found. Array arguments hold one
 * entry per device of the communicator, in its device order (HOST arrays of
 * device pointers / cudaStream_t). */
typedef struct gp_comm gp_comm;
int gp_comm_available(void);
int gp_comm_init(int ndev, const int* devices_host, gp_comm** out);
int gp_comm_destroy(gp_comm* comm);
int gp_comm_size(const gp_comm* comm);
int gp_comm_broadcast(gp_comm* comm, void* const* bufs, int64_t bytes, int root, void* const* streams);
int gp_comm_allgather(gp_comm* comm, const void* const* send, void* const* recv, int64_t bytes_per_rank,
                      void* const* streams);
int gp_comm_reduce_scatter_i64(gp_comm* comm, const int64_t* const* send, int64_t* const* recv,
                               int64_t count_per_rank, void* const* streams);
int gp_comm_reduce_scatter_i32(gp_comm* comm, const int32_t* const* send, int32_t* const* recv,
                               int64_t count_per_rank, void* const* streams);
int gp_comm_allreduce_f64(gp_comm* comm, double* const* bufs, int64_t count, void* const* streams);

#ifdef __cplusplus
}
#endif
#endif /* GPBBMM_H */
