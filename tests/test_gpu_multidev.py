"""Single-process multi-GPU path (csrc/comm.cu, multidev.py): the library's
own NCCL group calls and the item-split symmetric operator. The test box has
one GPU, so the group here has one device — the NCCL communicator, the group
calls and the partial -> reduce-scatter -> finalize -> gather sequence all run
for real; the split over several devices is the same item partition the
torchrun tests (test_gpu_sharded.py) check at 2 and 3 ranks."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _setup(n=20_000, d=11, t=11, fam="matern32"):
    import torch
    import paper_1903_08114_b200 as gp
    from paper_1903_08114_b200 import _device as D, _ops
    rng = np.random.default_rng(3)
    X = rng.standard_normal((n, d))
    m = gp.KernelModel(fam, 1.3, np.linspace(0.8, 1.6, d), 0.1)
    ps = D.points(X)
    Xs32, _ = ps.scaled(m.scale_for(d))
    V = torch.from_numpy(rng.standard_normal((n, t))).float().cuda()
    return m, ps, Xs32, V, _ops


def test_nccl_group_collectives_single_device():
    import torch
    from paper_1903_08114_b200 import _lib
    from paper_1903_08114_b200.multidev import DeviceGroup
    assert _lib.lib().gp_comm_available() == 1
    g = DeviceGroup([0])
    assert g.world == 1 and _lib.lib().gp_comm_size(g._h) == 1
    a = torch.arange(1000, dtype=torch.int64, device="cuda") * (1 << 40)
    out = torch.empty_like(a)
    g.reduce_scatter_([out], [a])
    assert torch.equal(out, a)
    b = torch.randn(333, device="cuda")
    ref = b.clone()
    g.broadcast_([b], root=0)
    assert torch.equal(b, ref)
    g.close()


def test_duplicate_device_rejected():
    from paper_1903_08114_b200.multidev import DeviceGroup
    with pytest.raises(ValueError, match="listed twice"):
        DeviceGroup([0, 0])


@pytest.mark.parametrize("t", [1, 11, 16])
def test_multidevice_operator_bitwise_equals_single_device(t):
    import torch
    from paper_1903_08114_b200.multidev import DeviceGroup, MultiDeviceKernelOperator
    m, ps, Xs32, V, _ops = _setup(t=16)
    V = V[:, :t].contiguous()
    ref = _ops.FusedKernelOperator(m.family_code, ps.d, Xs32, Xs32, m.outputscale, 0.0, -1, algo=3,
                                   self_offset=0).apply32(V, t)
    op = MultiDeviceKernelOperator(m.family_code, ps.d, Xs32, m.outputscale, 0.0, -1, DeviceGroup([0]))
    assert op.supported(t)
    got = op.apply32(V, t)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    # a second call reuses the buffers (and the acc padding stays zero)
    assert torch.equal(op.apply32(V, t), ref)
    assert op.group.bytes["reduce_scatter"] > 0


def test_workerpool_on_one_gpu_is_the_single_device_path():
    """WorkerPool(workers=4) spans min(4, device_count) GPUs; with one GPU
    the MLL is the single-device one, bitwise (partition.py:46-57 semantics:
    the pool size never changes the result)."""
    import paper_1903_08114_b200 as gp
    from paper_1903_08114_b200 import likelihood, synthetic as syn
    from paper_1903_08114_b200.multidev import usable_devices
    import torch
    assert usable_devices(4) == list(range(min(4, torch.cuda.device_count())))
    X = syn.whitened_inputs(3000, 5, 0)
    y = syn.rff_target(X, seed=1)
    m = gp.KernelModel("rbf", 1.0, 1.2, 0.1)
    cfg = likelihood.CgConfig(tolerance=0.01, probes=10, precond_rank=50)
    plan = gp.plan_partitions(3000, 1000)
    a = gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(workers=1), cfg, 0)
    b = gp.mll_value_and_grad(m, X, y, plan, gp.WorkerPool(workers=4), cfg, 0)
    assert a.value == b.value and a.gradients == b.gradients
