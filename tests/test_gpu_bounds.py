"""Out-of-bounds write checks without compute-sanitizer (the GPU pool keeps
the sanitizer closed): every K·V kernel family writes into an output whose
leading dimension and row count exceed what the call covers, pre-filled
with a canary bit pattern. The call must leave every canary element bitwise
intact, leave its inputs untouched, and give the same values as a call into
a tight buffer (test_partition.py:132-158's "no hidden buffers" contract,
restated as "no writes outside the caller's block")."""

import numpy as np
import pytest

import paper_1903_08114_b200 as gp

pytestmark = pytest.mark.gpu

CANARY = np.float32(-1234.5678)

# (n, d, family, t, algo): SIMT, row-tiled tcgen05, symmetric (ragged n),
# wide right-hand sides (auto picks kv_wide), large-d tcgen05
CASES = [(300, 5, "matern32", 11, 1), (300, 5, "rbf", 11, 2), (300, 5, "matern32", 11, 3),
         (257, 3, "rbf", 16, 3), (1100, 6, "matern32", 13, 3), (300, 5, "matern32", 40, 0),
         (200, 50, "matern32", 11, 2), (333, 90, "rbf", 64, 0)]


@pytest.mark.parametrize("n,d,fam,t,algo", CASES)
def test_kv_writes_stay_inside_the_output_block(n, d, fam, t, algo):
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    rng = np.random.default_rng(n + d + t)
    X = rng.uniform(size=(n, d))
    m = gp.KernelModel(fam, 1.0, np.linspace(0.5, 1.5, d) * np.sqrt(d) * 0.3, 0.2)
    Xs32, _ = D.points(X).scaled(m.scale_for(d))
    op = _ops.FusedKernelOperator(m.family_code, d, Xs32, Xs32, 1.0, 0.2, 0, algo=algo, self_offset=0)
    pad_r, pad_c = 70, 9
    Vbig = torch.full((n + pad_r, t + pad_c), float(CANARY), dtype=torch.float32, device="cuda")
    Vbig[:n, :t] = torch.from_numpy(rng.standard_normal((n, t))).float().cuda()
    V_before = Vbig.clone()
    tight = op.apply32(Vbig[:n, :t].contiguous(), t)
    obig = torch.full((n + pad_r, t + pad_c), float(CANARY), dtype=torch.float32, device="cuda")
    op.apply32(Vbig, t, out32=obig)   # ld = t + pad_c on both sides
    torch.cuda.synchronize()
    assert torch.equal(Vbig, V_before), "input V was written"
    o = obig.cpu().numpy()
    assert np.all(o[:n, t:].view(np.uint32) == CANARY.view(np.uint32)), "write past column t"
    assert np.all(o[n:, :].view(np.uint32) == CANARY.view(np.uint32)), "write past row n"
    np.testing.assert_allclose(o[:n, :t], tight.cpu().numpy(), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("n,t", [(129, 1), (300, 11)])
def test_kv_f64_writes_stay_inside_the_output_block(n, t):
    import torch
    from paper_1903_08114_b200 import _device as D, _ops
    rng = np.random.default_rng(7)
    d = 4
    X = rng.uniform(size=(n, d))
    m = gp.KernelModel("matern32", 1.0, np.linspace(0.4, 0.9, d), 0.3)
    X64 = torch.from_numpy(X / 0.6).cuda()   # any prescaled points
    V = torch.from_numpy(rng.standard_normal((n, t))).cuda()
    tight, _ = _ops.kv_f64(m.family_code, d, X64, X64, 1.0, 0.3, 0, V)
    big = torch.full((n + 40, t + 5), float(CANARY), dtype=torch.float64, device="cuda")
    view = big[:n, :t]
    _ops.kv_f64(m.family_code, d, X64, X64, 1.0, 0.3, 0, V, out=view)
    torch.cuda.synchronize()
    b = big.cpu().numpy()
    assert np.all(b[:n, t:] == np.float64(CANARY)) and np.all(b[n:, :] == np.float64(CANARY))
    assert np.array_equal(b[:n, :t], tight.cpu().numpy())
