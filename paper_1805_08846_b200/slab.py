"""Slab decomposition of the time step over a process group.

The reference is single-process; this module adds the
multi-GPU path the north star asks for without changing the arithmetic:

* the slowest axis (y in 2-D, z in 3-D) is split into P contiguous slabs,
  one per rank (one process per GPU, ``torch.distributed``);
* sweeps along the other axes are rank-local -- each pencil lies entirely
  inside one slab;
* before the slow-axis sweep each rank sends its first/last two owned
  rows/planes (m states) to its neighbours and receives their boundary
  rows into its own ghost layers (``CLB_BC_HALO``), a periodic slow axis
  wrapping rank 0 <-> P-1; the global physical boundary on the slow axis
  is synthesised by ranks 0 and P-1 only;
* the exchange overlaps the slow sweep: the sweep's segments that read no
  ghost row are launched while the send/recv are in flight, the edge
  segments after they land (``slow_sweep``);
* the per-sweep (max |s|, non-finite) results are max-allreduced, so every
  rank takes the identical fp64 accept/revert decision.

Max is exact and order independent and each cell's arithmetic is the
single-domain arithmetic (ghost values are the same bytes either way), so
the dt sequence and every state byte are identical to the 1-GPU run for
any P (tests/test_slab.py, tests/test_gpu_slab.py).

Transport: ``"nccl"`` exchanges device tensors that alias the C library's
buffers (zero copy, ordered on the library's stream = torch's current
stream); ``"host"`` stages the halo rows through host memory and is what
the CPU (gloo) tests and the single-GPU multi-process test use.
"""

from __future__ import annotations

import logging
from dataclasses import dataclass

import numpy as np

from .boundary import BC_HALO
from .grid import GridSpec, StateGrid

log = logging.getLogger("clawtile.slab")


def split_counts(n: int, parts: int) -> list[int]:
    """Contiguous near-equal split (the first n % parts slabs get one more)."""
    if parts < 1 or n < 2 * parts:
        raise ValueError(f"cannot split {n} cells into {parts} slabs of >= 2 cells")
    base, extra = divmod(n, parts)
    return [base + (1 if r < extra else 0) for r in range(parts)]


class _CudaBuffer:
    """__cuda_array_interface__ view of a raw device range (for torch.as_tensor)."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
            "strides": None,
        }


@dataclass
class SlabLayout:
    rank: int
    world: int
    axis: int                 # slow axis (ndim - 1)
    counts: list
    offset: int               # first global index owned along `axis`
    count: int                # owned cells along `axis`
    periodic: bool
    # a periodic slow axis wraps through the exchange even on one rank (the
    # rank is its own neighbour): the single-GPU check of the device path
    self_halo: bool = False

    @property
    def _wraps(self):
        return self.periodic and (self.world > 1 or self.self_halo)

    @property
    def lo_nbr(self):
        if self.rank > 0:
            return self.rank - 1
        return self.world - 1 if self._wraps else None

    @property
    def hi_nbr(self):
        if self.rank < self.world - 1:
            return self.rank + 1
        return 0 if self._wraps else None

    @property
    def exchanges(self):
        return self.lo_nbr is not None or self.hi_nbr is not None


class Slab:
    """One rank's share of a global grid, plus the exchange machinery.

    ``global_spec``: the whole grid.  ``bspec``: global boundary spec.
    ``dist``: ``torch.distributed`` (initialised) or None for world 1.
    """

    def __init__(self, global_spec: GridSpec, boundary, rank: int = 0, world: int = 1,
                 dist=None, transport: str = "nccl", group=None, self_halo: bool = False):
        if global_spec.ndim < 2 and world > 1:
            raise ValueError("slab decomposition needs ndim >= 2")
        self.global_spec = global_spec
        self.boundary = boundary
        axis = global_spec.ndim - 1
        counts = split_counts(global_spec.cells[axis], world) if world > 1 else [global_spec.cells[axis]]
        offset = sum(counts[:rank])
        if transport not in ("nccl", "device", "host"):
            raise ValueError(f"unknown halo transport {transport!r}")
        self.layout = SlabLayout(rank, world, axis, counts, offset, counts[rank],
                                 boundary.is_periodic(axis), self_halo)
        self.dist = dist
        self.group = group
        self.transport = transport
        cells = list(global_spec.cells)
        cells[axis] = counts[rank]
        # shapes only: spacing and cell centres always come from the global spec
        self.local_spec = GridSpec(tuple(cells), global_spec.lower, global_spec.upper,
                                   global_spec.num_states)
        self.dev = None
        self._pinned = {}

    # -- construction helpers ------------------------------------------------
    @property
    def global_spacing(self):
        return self.global_spec.spacing

    def local_bc(self, bc):
        """Global (lo, hi) BC ids -> this rank's ids (HALO at inner faces)."""
        L = self.layout
        out = [tuple(p) for p in bc]
        if L.exchanges:
            lo, hi = out[L.axis]
            if L.lo_nbr is not None:
                lo = BC_HALO
            if L.hi_nbr is not None:
                hi = BC_HALO
            out[L.axis] = (lo, hi)
        return out

    def local_slice(self):
        """Index of this rank's interior inside a global interior array."""
        L = self.layout
        nd = self.global_spec.ndim
        sl = [slice(None)] * (nd + 1)
        sl[1 + (nd - 1 - L.axis)] = slice(L.offset, L.offset + L.count)
        return tuple(sl)

    def local_centers(self):
        """Global cell centres of this rank's cells (array order, like
        StateGrid.centers) -- so profiles evaluate bit-identically."""
        spec = self.global_spec
        axes = [spec.axis_centers(ax) for ax in range(spec.ndim)]
        L = self.layout
        axes[L.axis] = axes[L.axis][L.offset:L.offset + L.count]
        mesh = np.meshgrid(*reversed(axes), indexing="ij")
        return tuple(reversed(mesh))

    def fill_initial(self, grid: StateGrid, profile) -> None:
        """fill_initial (grid.py:210-234) on this rank's slab only."""
        target = (grid.spec.num_states,) + grid.spec.interior_array_shape
        vals = np.asarray(profile(*self.local_centers()), dtype=grid.dtype)
        if vals.shape != target:
            if vals.shape == (grid.spec.num_states,):
                vals = vals.reshape((grid.spec.num_states,) + (1,) * grid.spec.ndim)
            vals = np.broadcast_to(vals, target)
        if not np.all(np.isfinite(vals)):
            raise ValueError("initial profile produced non-finite values")
        grid.interior()[...] = vals

    @property
    def device_resident(self) -> bool:
        """The exchange and the max-allreduce run inside the library (so the
        device controller's attempt graph can drive a slab run)."""
        return self.transport == "device"

    def attach(self, dev) -> None:
        self.dev = dev
        L = self.layout
        if self.transport == "device" and L.exchanges:
            # one NCCL communicator owned by the library: rank 0 makes the id
            from ._native import nccl_unique_id
            uid = nccl_unique_id() if L.rank == 0 else None
            if L.world > 1:
                box = [uid]
                self.dist.broadcast_object_list(box, src=0, group=self.group)
                uid = box[0]
            dev.attach_comm(uid, L.world, L.rank, L.lo_nbr, L.hi_nbr)
            # visible in the job log: one line per rank once the communicator exists
            log.info("clb NCCL communicator ready: rank %d of %d, slow axis %d, neighbours "
                     "lo=%s hi=%s, owned %d of %d cells", L.rank, L.world, L.axis, L.lo_nbr,
                     L.hi_nbr, L.count, self.global_spec.cells[L.axis])
        elif self.transport == "nccl" and L.world > 1:
            # one stream for kernels and NCCL: order is implicit
            dev.set_stream(_torch_stream())

    # -- collectives -----------------------------------------------------------
    def allreduce_max(self, values: np.ndarray) -> np.ndarray:
        if self.layout.world == 1 or self.dist is None:
            return values
        import torch
        # host transport: gloo (CPU tensors); nccl/device: an NCCL process group
        dev = "cpu" if self.transport == "host" else "cuda"
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()

    def allreduce_min_int(self, value: int) -> int:
        if self.layout.world == 1 or self.dist is None:
            return value
        import torch
        # host transport: gloo (CPU tensors); nccl/device: an NCCL process group
        dev = "cpu" if self.transport == "host" else "cuda"
        t = torch.tensor([value], dtype=torch.int64, device=dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
        return int(t.item())

    # -- halo exchange -----------------------------------------------------------
    def exchange(self, buf: int) -> None:
        """Fill the slow-axis ghost layers of device buffer `buf` from the
        neighbours' boundary rows/planes (both sides, every state)."""
        self.exchange_end(self.exchange_begin(buf))

    def exchange_begin(self, buf: int):
        """Post the halo exchange of `buf`.  NCCL: the send/recv run on the
        collective stream behind the work already queued (the sweep that
        produced `buf`) and this returns at once; host transport: done on
        return; device transport: the library's exchange, on its stream.
        Pass the result to exchange_end."""
        L = self.layout
        if not L.exchanges:
            return None
        if self.transport == "device":
            self.dev.halo_exchange(buf)
            return ((), None)
        m = self.global_spec.num_states
        self._buf = buf
        sides = []
        for side, nbr in ((0, L.lo_nbr), (1, L.hi_nbr)):
            if nbr is None:
                continue
            if self.transport == "nccl":
                send, recv, nbytes, sstride = self.dev.halo_layout(buf, side)
                sides.append((side, nbr, send, recv, nbytes, sstride))
            else:
                sides.append((side, nbr))
        if self.transport == "nccl":
            return self._exchange_nccl(sides, m)
        self._exchange_host(sides, m)
        return ((), None)   # completed; the split slow sweep still runs (same path as NCCL)

    @staticmethod
    def exchange_end(pending) -> None:
        """Make the library's stream wait for a posted exchange (stream-level
        for NCCL: the host does not block)."""
        if pending is None:
            return
        reqs, _keep = pending
        for req in reqs:
            req.wait()

    def _exchange_nccl(self, sides, m):
        """Zero-copy NCCL send/recv on the library's buffers.  NCCL pairs
        messages between two ranks in posting order, so the order is
        canonical: send hi rows then lo rows; receive into lo ghosts then hi
        ghosts.  That also pairs correctly when both neighbours are the same
        rank (a 2-rank periodic ring)."""
        import torch
        dist = self.dist
        by_side = {sd[0]: sd for sd in sides}
        ops, keep = [], []

        def view(ptr, nbytes):
            t = torch.as_tensor(_CudaBuffer(ptr, nbytes), device="cuda")
            keep.append(t)
            return t

        for side in (1, 0):
            if side in by_side:
                _, nbr, send, _, nbytes, sstride = by_side[side]
                for k in range(m):
                    ops.append(dist.P2POp(dist.isend, view(send + k * sstride, nbytes), nbr,
                                          group=self.group))
        for side in (0, 1):
            if side in by_side:
                _, nbr, _, recv, nbytes, sstride = by_side[side]
                for k in range(m):
                    ops.append(dist.P2POp(dist.irecv, view(recv + k * sstride, nbytes), nbr,
                                          group=self.group))
        return dist.batch_isend_irecv(ops), keep

    def _exchange_host(self, sides, m):
        import torch
        dist = self.dist
        ops, post = [], []
        for side, nbr, *_ in sides:
            sbuf = np.ascontiguousarray(self.dev.halo_read(self._buf, side))
            rbuf = np.empty_like(sbuf)
            # tag by side so a 2-rank periodic ring (same peer both ways) pairs up
            ops.append(dist.isend(torch.from_numpy(sbuf), nbr, group=self.group, tag=side))
            ops.append(dist.irecv(torch.from_numpy(rbuf), nbr, group=self.group, tag=1 - side))
            post.append((side, rbuf, sbuf))
        for op in ops:
            op.wait()
        for side, rbuf, _ in post:
            self.dev.halo_write(self._buf, side, rbuf)

    # -- the step ------------------------------------------------------------------
    def halo_free_segments(self, axis: int):
        """Segments of the slow-axis sweep that read no ghost row: segment k
        reads rows [k*L - 2, min(n, (k+1)*L) + 2) (clb_sweep_segments)."""
        nseg, seg_len = self.dev.segments(axis)
        n = self.layout.count
        inner = [k for k in range(nseg)
                 if k * seg_len >= 2 and min(n, (k + 1) * seg_len) + 2 <= n]
        return nseg, (inner[0], inner[-1] + 1) if inner else None

    def slow_sweep(self, dt: float, src: int, dst: int, slot: int, literal: bool = False):
        """The slow-axis sweep overlapped with its halo exchange: the
        segments clear of the ghost rows run while the exchange is in flight,
        the two edge groups after it lands.  Bitwise the same as exchanging
        first and sweeping once (segments are independent)."""
        dev = self.dev
        axis = self.layout.axis
        pending = self.exchange_begin(src)
        nseg, inner = self.halo_free_segments(axis)
        if pending is None or inner is None:
            self.exchange_end(pending)
            dev.sweep_async(axis, dt, src, dst, slot, literal=literal)
            return
        b, e = inner
        dev.sweep_async_range(axis, dt, src, dst, slot, b, e, literal=literal)
        self.exchange_end(pending)
        if b > 0:
            dev.sweep_async_range(axis, dt, src, dst, slot, 0, b, literal=literal)
        if e < nseg:
            dev.sweep_async_range(axis, dt, src, dst, slot, e, nseg, literal=literal)

    def attempt_step(self, sim, dt: float):
        """Sweeps of one attempt with the halo exchange overlapping the slow
        sweep; returns the max-allreduced per-sweep (speeds, nonfinite)."""
        dev = self.dev
        if self.transport == "device":
            # exchange, overlap and max-allreduce inside clb_attempt_step
            return dev.attempt_step(dt, sim._cur, sim._scratch[0], sim._scratch[1])
        nd = len(sim.step_order)
        src = sim._cur
        for j in range(nd):
            dst = sim._scratch[j % 2]
            if j == self.layout.axis:
                self.slow_sweep(dt, src, dst, j)
            else:
                dev.sweep_async(j, dt, src, dst, j)
            src = dst
        speeds, nonfinite = dev.fetch(nd)
        red = self.allreduce_max(np.array(list(speeds) + [1.0 if f else 0.0 for f in nonfinite]))
        return [float(v) for v in red[:nd]], [bool(v > 0.0) for v in red[nd:]]

    def locate_blowup(self, sim, dt: float, first_bad: int):
        """Literal re-run of sweeps 0..first_bad on every rank (with the
        exchange), then the global C-order minimum of the first offenders."""
        dev = self.dev
        src = sim._cur
        for j in range(first_bad + 1):
            dst = sim._scratch[j % 2]
            if j == self.layout.axis:
                self.slow_sweep(dt, src, dst, 0, literal=True)
            else:
                dev.sweep_async(j, dt, src, dst, 0, literal=True)
            dev.fetch(1)
            src = dst
        loc = dev.first_nonfinite(src)
        spec = self.global_spec
        big = np.iinfo(np.int64).max
        if loc is None:
            key = big
        else:
            state, cell = loc
            g = list(cell)
            g[self.layout.axis] += self.layout.offset
            lin = 0
            for ax in reversed(range(spec.ndim)):
                lin = lin * spec.cells[ax] + g[ax]
            key = state * spec.num_cells + lin
        key = self.allreduce_min_int(key)
        if key == big:
            return 0, (0,) * spec.ndim
        state, rest = divmod(key, spec.num_cells)
        cell = []
        for ax in range(spec.ndim):
            rest, c = divmod(rest, spec.cells[ax])
            cell.append(c)
        return state, tuple(cell)


def _torch_stream():
    """Torch's current stream as a handle for clb_set_stream.  Torch reports
    its legacy default stream as 0, which the library would read as "use
    your own stream" (unordered with torch's NCCL work); pass
    cudaStreamLegacy (0x1) instead so the sweeps and the halo/max-allreduce
    collectives stay in one order."""
    import torch
    return torch.cuda.current_stream().cuda_stream or 0x1


