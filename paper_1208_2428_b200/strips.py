"""Row-strip decomposition across GPUs (one process per GPU).

The reference's strips backend splits interior rows into balanced strips,
worker 0 also owning wall row 0 and the last worker row H-1
(make_strip_plan backends.cpp:20-36, worker_rows :140-145), and relies on a
shared address space for the rows across strip borders (run_strips
:149-219). Here each strip lives on its own GPU (fhpg_create_strip) and the
one-row halos (pull motion reaches rows r-1 and r+1 only) are
exchanged every step with point-to-point transfers over NVLink
(torch.distributed / NCCL), ordered on the engine's stream. Every random
decision is keyed by global (x, y, step), so any strip count gives the
single-GPU bits exactly.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def strip_rows(height: int, n: int):
    """make_strip_plan + worker_rows: [(row_begin, row_end)] for n strips."""
    interior = height - 2
    if n < 1:
        raise ValueError("strip count must be >= 1")
    if n > interior:
        raise ValueError("strip count exceeds interior row count")
    base, extra = divmod(interior, n)
    rows, r = [], 1
    for i in range(n):
        k = base + (1 if i < extra else 0)
        rows.append([r, r + k])
        r += k
    rows[0][0] = 0
    rows[-1][1] = height
    return [tuple(x) for x in rows]


class _DeviceBytes:
    """__cuda_array_interface__ view of `n` device bytes (no copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_row(ptr: int, n: int, device: int) -> torch.Tensor:
    return torch.as_tensor(_DeviceBytes(ptr, n), device=f"cuda:{device}")


def engine_halo_tensors(engine, device: int):
    """(send_top, send_bottom, recv_top, recv_bottom) uint8 CUDA tensors."""
    (st, sb, rt, rb), n = engine.halo()
    return tuple(device_row(p, n, device) for p in (st, sb, rt, rb))


def exchange_halos(send_top, send_bottom, recv_top, recv_bottom, rank: int, world: int,
                   group=None, wait: bool = True):
    """Send the first/last owned rows to the strips above/below and receive
    their boundary rows into the halo rows (no-op at the global edges).
    With wait=False the pending works are returned (wait() on each makes the
    current stream wait for the transfer)."""
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, send_top, rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_top, rank - 1, group))
    if rank < world - 1:
        ops.append(dist.P2POp(dist.isend, send_bottom, rank + 1, group))
        ops.append(dist.P2POp(dist.irecv, recv_bottom, rank + 1, group))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    if wait:
        for req in reqs:
            req.wait()
        return []
    return reqs


class LocalStrips:
    """Several strip engines driven from one process (one GPU each, or all on
    one GPU to exercise the decomposition): halo rows are moved with
    device-to-device copies ordered on one shared stream before every step."""

    def __init__(self, width: int, height: int, n: int, devices=None):
        from .engine import Engine
        self.W, self.H = width, height
        self.rows = strip_rows(height, n)
        self.devices = list(devices) if devices is not None else [0] * n
        self.engines = [Engine(width, height, rb, re, dev)
                        for (rb, re), dev in zip(self.rows, self.devices)]
        self.streams = {}
        for e, dev in zip(self.engines, self.devices):
            if dev not in self.streams:
                self.streams[dev] = torch.cuda.Stream(device=dev)
            e.set_stream(self.streams[dev].cuda_stream)

    def set_table(self, table):
        for e in self.engines:
            e.set_table(table)

    def set_obstacles(self, mask):
        for e, (rb, re) in zip(self.engines, self.rows):
            e.set_obstacles(mask[rb:re])

    def upload(self, state):
        for e, (rb, re) in zip(self.engines, self.rows):
            e.upload(state[rb:re])

    def init(self, seed: int, density: float):
        for e in self.engines:
            e.init(seed, density)

    def download(self):
        import numpy as np
        return np.concatenate([e.download() for e in self.engines], axis=0)

    def _exchange(self):
        halos = [engine_halo_tensors(e, dev) for e, dev in zip(self.engines, self.devices)]
        for i in range(len(self.engines) - 1):
            up, dn = halos[i], halos[i + 1]
            # A cross-device copy_ runs on the SOURCE device's current stream
            # and fences the destination's current stream: make both engines'
            # streams current so the copies are ordered after the previous
            # step's boundary rows on both sides and before the next launch.
            with torch.cuda.stream(self.streams[self.devices[i]]), \
                    torch.cuda.stream(self.streams[self.devices[i + 1]]):
                dn[2].copy_(up[1], non_blocking=True)  # strip i's last row -> halo above i+1
                up[3].copy_(dn[0], non_blocking=True)  # strip i+1's first row -> halo below i

    def advance(self, seed: int, force_p: float, first_step: int, step_count: int) -> int:
        from .engine import bernoulli_threshold
        thr = bernoulli_threshold(force_p)
        for e in self.engines:
            e.swaps(reset=True)
        for s in range(first_step, first_step + step_count):
            if len(self.engines) == 1:
                self.engines[0].advance_async(seed, thr, s, 1)
                continue
            for e in self.engines:  # interior rows: no halo needed
                e.advance_part(seed, thr, s, 0)
            self._exchange()
            for e in self.engines:  # boundary rows + swap
                e.advance_part(seed, thr, s, 1)
        return sum(e.swaps() for e in self.engines)


class DistStrips:
    """One strip per rank; `engine` is this rank's strip engine (or any
    object with the same halo_tensors()/advance_async()/swaps() methods,
    which the CPU gloo tests use).

    staging="device": the halo rows go straight between the GPUs (NCCL over
    NVLink); the engine is put on torch's current stream, the stream NCCL
    orders its transfers against (ncclSend waits for the rows written by the
    previous step's part 1, req.wait() orders part 1 after the arrival).
    staging="host": the rows are copied through pinned host buffers and
    exchanged with a CPU backend (gloo) — the multi-process path for ranks
    that share one GPU or have no peer path.
    """

    def __init__(self, engine, rank: int, world: int, halo_tensors=None, group=None,
                 staging: str = "device"):
        self.engine, self.rank, self.world, self.group = engine, rank, world, group
        self._halo = halo_tensors
        if staging not in ("device", "host"):
            raise ValueError("staging must be 'device' or 'host'")
        self.staging = staging
        self._host = None
        if halo_tensors is None and hasattr(engine, "set_stream"):
            engine.set_stream(torch.cuda.current_stream().cuda_stream)

    def _halos(self):
        if self._halo is not None:
            return self._halo()
        return engine_halo_tensors(self.engine, torch.cuda.current_device())

    def _host_exchange(self, st, sb, rt, rb):
        """Host-staged exchange: D2H of the boundary rows (ordered on the
        engine stream), CPU-backend P2P, H2D into the halo rows."""
        n = st.numel()
        if self._host is None or self._host[0].numel() != n:
            self._host = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(4)]
        hst, hsb, hrt, hrb = self._host
        hst.copy_(st)
        hsb.copy_(sb)  # blocking copies: the rows of the previous step are final
        exchange_halos(hst, hsb, hrt, hrb, self.rank, self.world, self.group, wait=True)
        if self.rank > 0:
            rt.copy_(hrt)
        if self.rank < self.world - 1:
            rb.copy_(hrb)

    def advance_async(self, seed: int, force_thr: int, first_step: int, step_count: int):
        if self.world == 1:  # no exchange: one call, the step kernels chain the column keys
            self.engine.advance_async(seed, force_thr, first_step, step_count)
            return
        for s in range(first_step, first_step + step_count):
            if self.staging == "host":
                self._host_exchange(*self._halos())
                self.engine.advance_part(seed, force_thr, s, 0)
                self.engine.advance_part(seed, force_thr, s, 1)
                continue
            # The exchange of this step's boundary rows is issued first (NCCL
            # waits for the previous step), the interior rows run while it is
            # in flight, the boundary rows after it lands.
            reqs = exchange_halos(*self._halos(), self.rank, self.world, self.group, wait=False)
            self.engine.advance_part(seed, force_thr, s, 0)
            for req in reqs:
                req.wait()
            self.engine.advance_part(seed, force_thr, s, 1)

    def advance(self, seed: int, force_thr: int, first_step: int, step_count: int) -> int:
        """Like fhp::advance over the whole lattice: returns the global swap count."""
        self.engine.swaps(reset=True)
        self.advance_async(seed, force_thr, first_step, step_count)
        local = self.engine.swaps()
        if self.world == 1:
            return local
        t = torch.tensor([local], dtype=torch.int64,
                         device="cuda" if dist.get_backend(self.group) == "nccl" else "cpu")
        dist.all_reduce(t, group=self.group)
        return int(t.item())
