"""Training driver (trainer.py of the reference): the
optimizers against reference trajectories on an analytic objective (CPU),
and a short full-adam run on the C1 instance against the reference's own
training run (GPU)."""

import numpy as np
import pytest

from conftest import load_golden
from paper_1903_08114_b200 import trainer as tr


class Bowl:
    """Same objective as tests/golden/make_trainer_golden.py."""

    def __init__(self, n, base_seed=3, fresh=True):
        self.w = np.linspace(1.0, 4.0, n)
        self.c = np.linspace(-1.0, 1.5, n)
        self.base_seed = base_seed
        self.fresh = fresh
        self.evals = 0

    def probe_seed(self, step):
        return self.base_seed + step if self.fresh else self.base_seed

    def __call__(self, x, step):
        self.evals += 1
        s = self.probe_seed(step) % 7
        f = float(np.sum(self.w * (x - self.c) ** 2) + 0.1 * np.sum(x ** 4) + 1e-3 * s * x[0])
        g = 2.0 * self.w * (x - self.c) + 0.4 * x ** 3
        g[0] += 1e-3 * s
        return f, g


def test_adam_matches_reference_trajectory():
    g = load_golden("trainer")
    x, trace = tr.adam_run(Bowl(4), g["opt_x0"], tr.AdamConfig(lr=0.05, steps=25))
    np.testing.assert_allclose(x, g["adam_x"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose([r.objective_value for r in trace.records], g["adam_f"], rtol=1e-12)
    np.testing.assert_allclose([r.grad_norm for r in trace.records], g["adam_g"], rtol=1e-12)


def test_lbfgs_matches_reference_trajectory():
    g = load_golden("trainer")
    x, trace = tr.lbfgs_run(Bowl(4), g["opt_x0"], tr.LbfgsConfig(steps=8, history=3))
    np.testing.assert_allclose(x, g["lbfgs_x"], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose([r.objective_value for r in trace.records], g["lbfgs_f"], rtol=1e-10)


def test_adam_nonfinite_handling():
    calls = []

    def obj(x, step):
        calls.append(step)
        if step == 3 and len([c for c in calls if c == 3]) == 1:
            return np.inf, np.full_like(x, np.nan)   # first try of step 3 fails, the retry succeeds
        return float(x @ x), 2 * x

    x, trace = tr.adam_run(obj, np.ones(3), tr.AdamConfig(lr=0.1, steps=4))
    assert len(trace.records) == 4 and calls.count(3) == 2
    with pytest.raises(tr.TrainingError, match="starting point"):
        tr.adam_run(lambda x, s: (np.inf, x), np.ones(2), tr.AdamConfig(steps=2))


def test_config_validation():
    with pytest.raises(ValueError):
        tr.AdamConfig(lr=0.0)
    with pytest.raises(ValueError):
        tr.TrainConfig(protocol="sgd")
    with pytest.raises(ValueError):
        tr.TrainConfig(pretrain_subset=0)
    rows = list(tr.TrainTrace(records=[tr.StepRecord("a", 1, -2.0, 0.5, 0.1, 3)]).csv_rows())
    assert rows[0].startswith("phase,step,mll") and rows[1].startswith("a,1,2,")


@pytest.mark.gpu
def test_full_adam_on_c1_matches_reference_run():
    """Three Adam steps on the C1 instance (n = 4,096): per-step MLL and the
    final raw parameters against the reference's own training run."""
    g = load_golden("trainer")
    c1 = load_golden("c1_full")
    X, y = c1["X"], c1["y"]
    cfg = tr.TrainConfig(protocol="full-adam", family="rbf", adam=tr.AdamConfig(lr=0.1, steps=3), seed=0)
    model, trace = tr.train(X, y, cfg)
    mll = np.array([r.mll for r in trace.records])
    np.testing.assert_allclose(mll, g["c1_mll"], rtol=1e-3)
    from paper_1903_08114_b200 import kernels
    np.testing.assert_allclose(kernels.model_to_raw(model), g["c1_raw"], atol=1e-3)


@pytest.mark.gpu
def test_pretrain_finetune_improves_likelihood():
    c1 = load_golden("c1_full")
    X, y = c1["X"], c1["y"]
    cfg = tr.TrainConfig(protocol="pretrain-finetune", family="rbf", pretrain_subset=1000,
                         lbfgs=tr.LbfgsConfig(steps=3), pretrain_adam_steps=2, finetune_steps=2)
    model, trace = tr.train(X, y, cfg)
    phases = [r.phase for r in trace.records]
    assert phases[:3] == ["pretrain-lbfgs"] * 3 and phases[-2:] == ["finetune-adam"] * 2
    assert trace.subset_evals >= 5 and trace.full_evals == 2
    assert all(np.isfinite(r.mll) for r in trace.records)
