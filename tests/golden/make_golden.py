"""Generate golden vectors by RUNNING THE REFERENCE (blockgp 0.1.0).

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Everything below calls the reference's own public/internal API from
/root/reference/pkg/src/blockgp; the outputs are committed as small .npz
fixtures that pin both the oracle restatement (oracle/) and the CUDA path.
Large-n inputs are NOT stored: they are regenerated from seeds by
paper_1903_08114_b200.synthetic (numpy PCG64, bit-reproducible).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)

import blockgp  # noqa: E402  (the reference)
from blockgp import kernels as rk, likelihood as rl, cg as rcg, precond as rpc  # noqa: E402
from blockgp import predictor as rpr  # noqa: E402
from blockgp.data import sample_prior  # noqa: E402

from paper_1903_08114_b200 import synthetic as syn  # noqa: E402


def make_instance(n, d, family="rbf", ard=False, seed=0, lengthscale=0.4,
                  outputscale=1.0, noise=0.5, mean=0.0):
    """The reference test-suite recipe (pkg/tests/conftest.py:10-21)."""
    rng = np.random.default_rng(seed)
    X = rng.uniform(0.0, 1.0, size=(n, d))
    ls = lengthscale * np.linspace(0.75, 1.5, d) if ard else np.array([lengthscale])
    model = blockgp.KernelModel(family, outputscale, ls, noise, mean=mean)
    y = sample_prior(model, X, rng)
    return X, y, model


def hp_of(model):
    return dict(family=model.family, s2=model.outputscale, ls=np.asarray(model.lengthscales),
                noise=model.noise, mean=model.mean)


def save(name, **arrs):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrs)
    print(f"  wrote {name}.npz ({os.path.getsize(path) / 1e6:.2f} MB)")


def known_answers():
    m32 = blockgp.KernelModel("matern32", 1.0, np.array([1.0]), 0.1)
    rbf = blockgp.KernelModel("rbf", 1.0, np.array([1.0]), 0.1)
    rep = rcg.mbcg_solve(lambda V: np.array([[4.0, 1.0], [1.0, 3.0]]) @ V,
                         rcg.SolveRequest(rhs=np.array([1.0, 2.0]), tolerance=1e-12))
    two = rcg.mbcg_solve(lambda V: 2.0 * V,
                         rcg.SolveRequest(rhs=np.random.default_rng(0).standard_normal((3, 1)),
                                          tolerance=1e-12))
    fac = rpc.partial_pivoted_cholesky(lambda i: np.diag([4.0, 1.0])[i], np.array([4.0, 1.0]), 1)
    one = blockgp.KernelModel("rbf", 0.5, np.array([1.0]), 0.5)
    mll1 = rl.mll_value_and_grad(one, np.zeros((1, 1)), np.array([0.5]),
                                 blockgp.plan_partitions(1, 1), blockgp.WorkerPool(),
                                 rl.CgConfig(tolerance=1e-10, precond_rank=0, probes=1), 0)
    save("known",
         matern_at_1=rk.kernel_eval(m32, [0.0], [1.0]),
         rbf_at_1=rk.kernel_eval(rbf, [0.0], [1.0]),
         cg2_solution=rep.solutions[:, 0], cg2_iterations=rep.iterations,
         slq_2I3=rcg.slq_logdet(two), pivchol_L=fac.factor, pivchol_piv=fac.pivots,
         pivchol_resid=fac.residual_diag,
         precond_k0_logdet=rpc.build_preconditioner(np.zeros((5, 0)), 0.3).logdet,
         mll_n1=mll1.value)


def kv_small():
    cases = [  # (n, d, family, ard, seed, v_seed, t) from test_partition.py + ARD
        (50, 3, "rbf", False, 1, 2, 4),
        (37, 2, "matern32", False, 3, 4, 3),
        (200, 2, "matern32", False, 3, 4, 3),
        (120, 4, "rbf", False, 5, 6, 5),
        (300, 5, "matern32", True, 7, 8, 11),
        (257, 9, "rbf", True, 9, 10, 16),
    ]
    out = {}
    for c, (n, d, fam, ard, seed, vs, t) in enumerate(cases):
        X, _, model = make_instance(n, d, family=fam, ard=ard, seed=seed)
        V = np.random.default_rng(vs).standard_normal((n, t))
        dense = rk.kernel_block(model, X, X, add_noise=True)
        Xt = np.random.default_rng(vs + 100).uniform(0, 1, (33, d))
        out.update({f"c{c}_X": X, f"c{c}_V": V, f"c{c}_KV": dense @ V,
                    f"c{c}_Xt": Xt, f"c{c}_Kxv": rk.kernel_block(model, Xt, X) @ V[:, 0],
                    f"c{c}_family": fam, f"c{c}_s2": model.outputscale,
                    f"c{c}_ls": model.lengthscales, f"c{c}_noise": model.noise,
                    f"c{c}_block": dense[:7, :9]})
    out["ncases"] = len(cases)
    save("kv_small", **out)


def full_case(name, n, d, family, ard, seed, rank, tol=1.0, probes=10,
              lengthscale=0.4, noise=0.5, mean=0.0, n_pred=200, n_var=64,
              with_prediction=True):
    X, y, model = make_instance(n, d, family=family, ard=ard, seed=seed,
                                lengthscale=lengthscale, noise=noise, mean=mean)
    plan = blockgp.plan_partitions(n, 1024)
    pool = blockgp.WorkerPool(workers=4)
    cfg = rl.CgConfig(tolerance=tol, probes=probes, precond_rank=rank)
    t0 = time.perf_counter()
    res = rl.mll_value_and_grad(model, X, y, plan, pool, cfg, probe_seed=0)
    secs = time.perf_counter() - t0
    # replay the reference's internal stages through its own functions to
    # expose the intermediate objects mll_value_and_grad does not return
    cache = rl.build_kernel_preconditioner(model, X, rank)
    Z = rl.draw_probes(n, probes, 0, cache)
    oracle = rk.training_mvm_oracle(model)
    rep = rcg.mbcg_solve(lambda V: blockgp.partitioned_mvm(oracle, X, V, plan, pool),
                         rcg.SolveRequest(rhs=np.hstack([(y - model.mean)[:, None], Z]),
                                          tolerance=tol, preconditioner=cache))
    arrs = dict(X=X, y=y, family=family, s2=model.outputscale, ls=model.lengthscales,
                noise=model.noise, mean=model.mean, rank=rank, tol=tol, probes=probes,
                value=res.value, grad_keys=np.array(list(res.gradients.keys())),
                grad_vals=np.array(list(res.gradients.values())),
                iterations=res.diagnostics.iterations,
                final_residuals=res.diagnostics.final_residuals,
                logdet=res.diagnostics.logdet_estimate, quad=res.diagnostics.quad_term,
                Z=Z, solutions=rep.solutions, rep_iterations=rep.iterations,
                residual_history=rep.residual_history,
                diag_lens=np.array([T.order for T in rep.tridiagonals]),
                tri_diag=np.concatenate([T.diag for T in rep.tridiagonals]),
                tri_off=np.concatenate([T.offdiag for T in rep.tridiagonals]),
                ref_seconds=secs)
    if cache is not None:
        fac = rpc.partial_pivoted_cholesky(
            lambda i: rk.kernel_rows(model, X, i, i + 1, noise=False)[0],
            np.full(n, model.outputscale), min(rank, n))
        arrs.update(pivots=fac.pivots, L_rows=fac.factor[:16], precond_logdet=cache.logdet,
                    resid_diag_sum=float(fac.residual_diag.sum()))
    if with_prediction:
        pcache = rpr.build_cache(model, X, y, plan, pool, precond_rank=rank)
        Xs = np.random.default_rng(3).uniform(0, 1, (n_pred, d))
        mean_pred = rpr.predict_mean(pcache, Xs, pool=pool)
        var, clamped = rpr.predict_variance(pcache, Xs[:n_var], pool=pool, precond_rank=rank)
        arrs.update(cache_weights=pcache.weights,
                    cache_iterations=pcache.diagnostics["iterations"],
                    cache_residual=pcache.diagnostics["residual"],
                    X_test=Xs, pred_mean=mean_pred, pred_var=var, pred_clamped=clamped)
    save(name, **arrs)
    print(f"  {name}: value={res.value!r} iters={res.diagnostics.iterations} ({secs:.2f}s)")


def row_subsets():
    """K̂[rows,:]·V at the large configs, rows from three places; inputs are
    regenerated from seeds by paper_1903_08114_b200.synthetic."""
    out = {}
    for key in ("C2", "C3", "C4", "C5", "M1e6"):
        w = syn.WORKLOADS[key]
        X = syn.whitened_inputs(w.n, w.d, seed=0)
        V = syn.rhs_block(w.n, 11, seed=2)
        model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
        rows = 16 if w.n > 500_000 else 32
        starts = [0, w.n // 2 - rows // 2, w.n - rows]
        t0 = time.perf_counter()
        got = [rk.kernel_rows(model, X, s, s + rows) @ V for s in starts]
        out[f"{key}_starts"] = np.array(starts)
        out[f"{key}_rows"] = rows
        out[f"{key}_KV"] = np.stack(got)
        out[f"{key}_X_checksum"] = np.array([X.sum(), (X * X).sum(), X[17].sum()])
        print(f"  {key}: {3 * rows} rows x {w.n} in {time.perf_counter() - t0:.1f}s")
    # pivoted-Cholesky pivots at C2 (rank 5) and C3 (rank 100)
    for key in ("C2", "C3"):
        w = syn.WORKLOADS[key]
        X = syn.whitened_inputs(w.n, w.d, seed=0)
        model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
        t0 = time.perf_counter()
        fac = rpc.partial_pivoted_cholesky(
            lambda i: rk.kernel_rows(model, X, i, i + 1, noise=False)[0],
            np.full(w.n, model.outputscale), w.rank)
        pc = rpc.build_preconditioner(fac, model.noise)
        out[f"{key}_pivots"] = fac.pivots
        out[f"{key}_L_rows"] = fac.factor[:8]
        out[f"{key}_precond_logdet"] = pc.logdet
        out[f"{key}_resid_diag_sum"] = float(fac.residual_diag.sum())
        print(f"  {key}: pivchol rank {w.rank} in {time.perf_counter() - t0:.1f}s")
    save("row_subsets", **out)


def large_pivots():
    """Pivoted-Cholesky pivots (rank 100) at C5 and at the bench workload
    M1e6 (precond.py:58-98 through likelihood.py:74-91)."""
    out = {}
    for key in ("C5", "M1e6"):
        w = syn.WORKLOADS[key]
        X = syn.whitened_inputs(w.n, w.d, seed=0)
        model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
        t0 = time.perf_counter()
        fac = rpc.partial_pivoted_cholesky(
            lambda i: rk.kernel_rows(model, X, i, i + 1, noise=False)[0],
            np.full(w.n, model.outputscale), w.rank)
        pc = rpc.build_preconditioner(fac, model.noise)
        out[f"{key}_pivots"] = fac.pivots
        out[f"{key}_L_rows"] = fac.factor[:8]
        out[f"{key}_precond_logdet"] = pc.logdet
        out[f"{key}_resid_diag_sum"] = float(fac.residual_diag.sum())
        print(f"  {key}: pivchol rank {w.rank} in {time.perf_counter() - t0:.1f}s")
    save("large_pivots", **out)


def c4_grad():
    """(dK/dtheta)[rows, :] @ R at C4 (d = 90, Matern-3/2 ARD) for every
    geometric hyperparameter, from the reference's grad_row_products
    (kernels.py:396-410). The GPU test contracts these with a seeded Y on the
    same rows and compares with the fused gradient pass."""
    w = syn.WORKLOADS["C4"]
    X = syn.whitened_inputs(w.n, w.d, seed=0)
    model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    rows, width = 32, 8
    start = w.n // 2 - rows // 2
    R = np.random.default_rng(5).standard_normal((w.n, width))
    pids = [p for p in rk.param_ids(model) if p not in ("noise", "mean")]
    t0 = time.perf_counter()
    prods = rk.grad_row_products(model, X, start, start + rows, R, pids)
    print(f"  C4 grad rows: {len(pids)} params x {rows} rows in {time.perf_counter() - t0:.1f}s")
    save("c4_grad", start=start, rows=rows, width=width, r_seed=5, pids=np.array(pids),
         products=np.stack([prods[p] for p in pids]))


def c2_mll():
    """A full MLL + gradients at C2 (n = 65,536, d = 8, Matern-3/2 ARD,
    rank-5 preconditioner, eps = 1, t = 10) through the reference's
    mll_value_and_grad on all host cores (~12 min)."""
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, seed=0)
    y = syn.rff_target(X, seed=1)
    model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    plan = blockgp.plan_from_budget(w.n)
    pool = blockgp.WorkerPool(workers=os.cpu_count())
    cfg = rl.CgConfig(tolerance=1.0, probes=10, precond_rank=w.rank)
    t0 = time.perf_counter()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        res = rl.mll_value_and_grad(model, X, y, plan, pool, cfg, probe_seed=0)
    secs = time.perf_counter() - t0
    # replay the solve through the reference's own stages to expose the
    # per-column recurrence (residual history, tridiagonal orders)
    cache = rl.build_kernel_preconditioner(model, X, w.rank)
    Z = rl.draw_probes(w.n, 10, 0, cache)
    oracle = rk.training_mvm_oracle(model)
    with threadpool_limits(1):
        rep = rcg.mbcg_solve(lambda V: blockgp.partitioned_mvm(oracle, X, V, plan, pool),
                             rcg.SolveRequest(rhs=np.hstack([(y - model.mean)[:, None], Z]),
                                              tolerance=1.0, preconditioner=cache))
    save("c2_mll", y_checksum=np.array([y.sum(), (y * y).sum(), y[5]]),
         residual_history=rep.residual_history, diag_lens=np.array([T.order for T in rep.tridiagonals]),
         rep_iterations=rep.iterations, Z_checksum=np.array([Z.sum(), (Z * Z).sum()]),
         value=res.value, grad_keys=np.array(list(res.gradients.keys())),
         grad_vals=np.array(list(res.gradients.values())),
         iterations=res.diagnostics.iterations, final_residuals=res.diagnostics.final_residuals,
         logdet=res.diagnostics.logdet_estimate, quad=res.diagnostics.quad_term,
         ref_seconds=secs, workers=os.cpu_count())
    print(f"  C2 MLL: value={res.value!r} iters={res.diagnostics.iterations} ({secs:.0f}s)")


def whiten():
    """split_and_whiten (data.py:163-196) on a table with a constant feature
    column and a wide value range, through the reference."""
    from blockgp.data import RawTable, split_and_whiten
    rng = np.random.default_rng(21)
    n, d = 1001, 5
    X = rng.standard_normal((n, d)) * np.array([1.0, 1e3, 1e-3, 0.0, 5.0]) + np.array([0.0, 7.0, -3.0, 2.5, 1e4])
    y = 3.0 * rng.standard_normal(n) + 40.0
    ds = split_and_whiten(RawTable(X, y, [f"x{i}" for i in range(d)], "y"), seed=5, name="w")
    save("whiten", X_raw=X, y_raw=y, seed=np.array(5), X=ds.X, y=ds.y, train_idx=ds.train_idx,
         val_idx=ds.val_idx, test_idx=ds.test_idx, feature_mean=ds.feature_mean, feature_std=ds.feature_std,
         target_mean=np.array(ds.target_mean), target_std=np.array(ds.target_std))


def c2_tight():
    """The C2 MLL + gradients through the reference at eps = 0.01 (converged
    solves: the value and gradients no longer depend on where an eps = 1
    solve happens to stop; ~1 h on 8 cores)."""
    w = syn.WORKLOADS["C2"]
    X = syn.whitened_inputs(w.n, w.d, seed=0)
    y = syn.rff_target(X, seed=1)
    model = blockgp.KernelModel(w.family, syn.OUTPUTSCALE, w.lengthscales(), syn.NOISE)
    plan = blockgp.plan_from_budget(w.n)
    pool = blockgp.WorkerPool(workers=os.cpu_count())
    cfg = rl.CgConfig(tolerance=0.01, probes=10, precond_rank=w.rank)
    t0 = time.perf_counter()
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        res = rl.mll_value_and_grad(model, X, y, plan, pool, cfg, probe_seed=0)
    secs = time.perf_counter() - t0
    save("c2_tight", value=res.value, grad_keys=np.array(list(res.gradients.keys())),
         grad_vals=np.array(list(res.gradients.values())), iterations=res.diagnostics.iterations,
         final_residuals=res.diagnostics.final_residuals, logdet=res.diagnostics.logdet_estimate,
         quad=res.diagnostics.quad_term, ref_seconds=secs, workers=os.cpu_count())
    print(f"  C2 MLL eps=0.01: value={res.value!r} iters={res.diagnostics.iterations} ({secs:.0f}s)")


def main(which=()):
    t0 = time.perf_counter()
    if not which or "base" in which:
        print("known answers"); known_answers()
        print("kv_small"); kv_small()
        print("full cases")
        full_case("c1_full", 4096, 8, "rbf", False, 0, 100)
        full_case("matern_ard", 800, 5, "matern32", True, 11, 30, n_var=48)
        full_case("noprecond", 300, 3, "rbf", False, 12, 0, n_var=32)
        full_case("tight_tol", 500, 4, "matern32", False, 13, 20, tol=1e-6, with_prediction=False)
    if not which or "row_subsets" in which:
        print("row subsets"); row_subsets()
    if not which or "large_pivots" in which:
        print("large pivots"); large_pivots()
    if not which or "c4_grad" in which:
        print("C4 gradient rows"); c4_grad()
    if not which or "whiten" in which:
        print("whiten"); whiten()
    if not which or "c2_mll" in which:
        print("C2 MLL"); c2_mll()
    if "c2_tight" in which:
        print("C2 MLL, eps = 0.01"); c2_tight()
    print(f"done in {time.perf_counter() - t0:.0f}s")


if __name__ == "__main__":
    # python make_golden.py [base] [row_subsets] [large_pivots] [c4_grad] [whiten] [c2_mll] [c2_tight]
    main(tuple(sys.argv[1:]))
