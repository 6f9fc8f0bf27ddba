"""Single-process multi-GPU K̂·V: the GPUs of one host driven by one thread
(SURVEY §8(b) "Collectives", §8(e)).

The reference parallelises each MVM over the threads of a `WorkerPool`
(partition.py:46-57, :155-183) inside one process. The device equivalent
here splits the symmetric kernel's work items over the GPUs of a
`DeviceGroup` (item L goes to device L mod w, gp_kv_sym_partial), combines the
64-bit fixed-point partial sums with one NCCL reduce-scatter (each device
receives the summed slice of its own 128-aligned rows), finalises those rows
on their device and gathers them into the caller's output on the first
device. Integer sums are associative, so the product is bitwise the
single-device gp_kv result for every device count (the reference's
partition-count independence, test_partition.py:92-102). The collectives are
the library's own NCCL group calls (gp_comm_*, csrc/comm.cu); the torchrun
path (one process per GPU, `sharded.py`) uses the same partial / finalize
entry points over torch.distributed.

`WorkerPool(workers=w)` selects this path for the MLL and the cache solve
when the host has at least two GPUs: the operator spans the first
min(w, device_count) devices; the CG vector work stays on the first device,
as the reference keeps its CG on the control thread.
"""

from __future__ import annotations

import ctypes as C
import math

from . import _device as D
from . import _lib


def usable_devices(workers: int) -> list:
    """The devices a WorkerPool of `workers` spans: the first
    min(workers, device_count) GPUs; one device means the ordinary path."""
    T = D.torch()
    n = T.cuda.device_count() if T.cuda.is_available() else 0
    return list(range(min(max(1, int(workers)), n)))


class DeviceGroup:
    """NCCL communicator over `devices` of this process (gp_comm_init ->
    ncclCommInitAll). Collective payloads are counted in `bytes`."""

    def __init__(self, devices):
        devices = [int(x) for x in devices]
        lib = _lib.lib()
        if not lib.gp_comm_available():
            raise RuntimeError("multi-GPU group: libnccl.so.2 is not available in this process")
        arr = (C.c_int * len(devices))(*devices)
        h = C.c_void_p()
        _lib.check(lib.gp_comm_init(len(devices), arr, C.byref(h)), "gp_comm_init")
        self._h = h
        self.devices = devices
        self.world = len(devices)
        self.bytes = {"broadcast": 0, "reduce_scatter": 0}

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.check(_lib.lib().gp_comm_destroy(self._h), "gp_comm_destroy")
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _arr(self, values):
        return (C.c_void_p * self.world)(*[int(v) for v in values])

    def streams(self):
        return self._arr(_lib.stream_handle(D.torch().device("cuda", d)) for d in self.devices)

    def broadcast_(self, bufs, root: int = 0):
        """bufs[r] (one tensor per device, same byte size) = bufs[root]."""
        nbytes = bufs[0].numel() * bufs[0].element_size()
        _lib.check(_lib.lib().gp_comm_broadcast(self._h, self._arr(b.data_ptr() for b in bufs), nbytes, root,
                                                self.streams()), "gp_comm_broadcast")
        self.bytes["broadcast"] += nbytes * (self.world - 1)

    def reduce_scatter_(self, outs, fulls):
        """outs[r] = sum over devices q of fulls[q][r L : (r + 1) L] (int64 or int32)."""
        T = D.torch()
        L = outs[0].numel()
        fn = {T.int64: _lib.lib().gp_comm_reduce_scatter_i64,
              T.int32: _lib.lib().gp_comm_reduce_scatter_i32}[outs[0].dtype]
        _lib.check(fn(self._h, self._arr(f.data_ptr() for f in fulls), self._arr(o.data_ptr() for o in outs),
                      L, self.streams()), "gp_comm_reduce_scatter")
        self.bytes["reduce_scatter"] += L * self.world * outs[0].element_size()   # per device


class MultiDeviceKernelOperator:
    """The square operator s2 kappa(X, X) (+ noise I) over the devices of a
    DeviceGroup; apply32 takes and returns fp32 blocks on the first device.
    Rows [r m, (r + 1) m) (m = ceil(n / w) rounded up to 128) are finalised
    on device r."""

    def __init__(self, family_code: int, d: int, X32, outputscale: float, noise: float, diag_offset: int,
                 group: DeviceGroup):
        T = D.torch()
        self.group = group
        w = group.world
        n = X32.shape[0]
        self.n_rows = self.n_cols = n
        self.rows_per_dev = m = math.ceil(math.ceil(n / w) / 128) * 128
        self.ranges = [(min(n, r * m), min(n, (r + 1) * m)) for r in range(w)]
        self.X = []
        self.desc = []
        for dev in group.devices:
            Xr = X32.to(T.device("cuda", dev)).contiguous()
            self.X.append(Xr)
            self.desc.append(_lib.KvDesc(family=family_code, d=d, Xr=Xr.data_ptr(), ldr=Xr.stride(0), n_rows=n,
                                         Xc=Xr.data_ptr(), ldc=Xr.stride(0), n_cols=n,
                                         outputscale=float(outputscale), noise=float(noise),
                                         diag_offset=int(diag_offset), algo=0, self_offset=0))
        self._bufs = {}

    def supported(self, t: int) -> bool:
        return bool(_lib.lib().gp_kv_sym_supported(self.desc[0], t)) and self.n_rows >= 128 * self.group.world

    def _buffers(self, t: int, ldv: int):
        key = (t, ldv)
        if key not in self._bufs:
            T = D.torch()
            L = _lib.lib()
            n, m, w = self.n_rows, self.rows_per_dev, self.group.world
            ld = int(L.gp_kv_sym_acc_ld(self.desc[0]))
            full = max(ld, m * w)
            nbytes = int(L.gp_kv_workspace_bytes(self.desc[0], t))
            per = []
            for r, dev in enumerate(self.group.devices):
                dv = T.device("cuda", dev)
                per.append(dict(
                    # the first device's V is the caller's block (set per call)
                    V=T.empty((n, ldv), dtype=T.float32, device=dv) if r else None,
                    acc=T.zeros(t * full, dtype=T.int64, device=dv),
                    bad=T.zeros(full, dtype=T.int32, device=dv),
                    acc_l=T.empty(t * m, dtype=T.int64, device=dv),
                    bad_l=T.empty(m, dtype=T.int32, device=dv),
                    out=T.empty((m, t), dtype=T.float32, device=dv),
                    ws=T.empty(max(nbytes, 1), dtype=T.uint8, device=dv), nbytes=nbytes))
            self._bufs[key] = (ld, full, per)
        return self._bufs[key]

    def apply32(self, V32, t: int, out32=None):
        """out32[:, :t] = K V32[:, :t] (V32 and out32 on the first device)."""
        T = D.torch()
        L = _lib.lib()
        g = self.group
        n = self.n_rows
        if out32 is None:
            out32 = T.empty((n, t), dtype=T.float32, device=V32.device)
        V32 = V32[:n].contiguous()
        ld, full, per = self._buffers(t, V32.shape[1])
        per[0]["V"] = V32
        g.broadcast_([p["V"] for p in per], root=0)
        for r, dev in enumerate(g.devices):
            p = per[r]
            with T.cuda.device(dev):
                st = _lib.stream_handle()
                if full > ld:   # padding rows of the last device's slice
                    p["acc"][t * ld:].zero_()
                    p["bad"][ld:].zero_()
                _lib.check(L.gp_kv_sym_partial(self.desc[r], p["V"].data_ptr(), p["V"].stride(0), t, r, g.world,
                                               p["acc"].data_ptr(), p["bad"].data_ptr(), p["ws"].data_ptr(),
                                               p["nbytes"], st), "gp_kv_sym_partial")
        m = self.rows_per_dev
        g.reduce_scatter_([p["acc_l"] for p in per], [p["acc"][: t * m * g.world] for p in per])
        g.reduce_scatter_([p["bad_l"] for p in per], [p["bad"][: m * g.world] for p in per])
        for r, dev in enumerate(g.devices):
            p = per[r]
            r0, r1 = self.ranges[r]
            if r1 <= r0:
                continue
            with T.cuda.device(dev):
                _lib.check(L.gp_kv_sym_finalize(self.desc[r], p["V"].data_ptr(), p["V"].stride(0), t,
                                                p["acc_l"].data_ptr(), p["bad_l"].data_ptr(), r0, r0, r1,
                                                p["out"].data_ptr(), p["out"].stride(0), p["ws"].data_ptr(),
                                                p["nbytes"], _lib.stream_handle()), "gp_kv_sym_finalize")
            # stream-ordered cross-device copy into the caller's block
            out32[r0:r1, :t].copy_(p["out"][: r1 - r0], non_blocking=True)
        return out32


def training_operator(family_code: int, d: int, X32, outputscale: float, noise: float, diag_offset: int,
                      workers: int, t: int, single):
    """The operator a WorkerPool of `workers` runs on: the multi-device one
    when at least two GPUs take part and the symmetric kernel takes the shape
    (t <= 16 right-hand sides, n >= 128 per device), else `single`."""
    devs = usable_devices(workers)
    if len(devs) < 2:
        return single
    op = MultiDeviceKernelOperator(family_code, d, X32, outputscale, noise, diag_offset, DeviceGroup(devs))
    return op if op.supported(t) else single
