"""Multi-GPU slab decomposition of the sweep along the slowest axis.

The reference has no distributed execution (SPEC.md lists it as a non-goal;
its only parallelism is the tile thread pool of tiling.py:372-417).  Here a
grid too large for one GPU -- or a weak-scaled one -- is split into
contiguous slabs along axis 0, one per rank (one process per GPU,
torch.distributed over NCCL on NVLink/NVSwitch).  Each slab's plan carries a
ghost zone of depth G = r*k on every side that faces another rank; before
every fused launch of k steps, ranks exchange G planes with their neighbours
(grouped isend/irecv), and the fused kernels compute the ghost planes like
interior ones, so the valid region shrinks back to exactly the slab after k
steps (overlapped ghost-zone recompute; no exchange inside a launch).
For 2D/3D slabs the exchange overlaps the compute: each k-step interval first
computes the G edge planes the neighbours need (``sb_launch_range``), sends
them from a communication stream while the slab interior is computed on the
main stream, and the next interval's launches wait for the received ghosts.
Physical sides keep the Dirichlet halo.  Per-point arithmetic does not
depend on the decomposition, so results are bit-identical to one GPU.

The orchestration is backend-agnostic: :class:`DeviceSlab` runs the sm_100a
kernels through the C ABI; tests drive the same code with a CPU backend and
the ``gloo`` transport.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import GridError, validate

# fused depths the slab plans accept per launch (see sb200.cu fused_k_ok;
# 1D depths 32 and 64 exist only on the composed path: FMA mode, r*k <= 64)
# 2D depths 16 and 32 exist only on the separable composed path (FMA mode, rank-1 weights)
_FUSED_KS = {1: (1, 2, 4, 8, 16, 32, 64), 2: (1, 2, 4, 8, 16, 32), 3: (1, 2, 3, 4)}


def split_extent(n: int, world: int) -> list[tuple[int, int]]:
    """Balanced [start, end) ranges of n interior planes over `world` ranks."""
    if world < 1 or n < world:
        raise GridError(f"cannot split {n} planes over {world} ranks")
    base, extra = divmod(n, world)
    out, pos = [], 0
    for r in range(world):
        size = base + (1 if r < extra else 0)
        out.append((pos, pos + size))
        pos += size
    return out


@dataclass
class SlabGeometry:
    rank: int
    world: int
    start: int           # first global interior plane of this slab
    end: int
    ghost_lo: int        # 0 = physical side (halo r), else ghost depth
    ghost_hi: int
    r: int

    @property
    def n(self) -> int:
        return self.end - self.start

    @property
    def h_lo(self) -> int:
        return self.ghost_lo or self.r

    @property
    def h_hi(self) -> int:
        return self.ghost_hi or self.r

    def local_slice(self) -> slice:
        """Axis-0 slice of the GLOBAL halo box that forms this rank's local box."""
        return slice(self.start - self.h_lo + self.r, self.end + self.h_hi + self.r)

    def interior_slice(self) -> slice:
        """Axis-0 slice of the LOCAL box holding this slab's interior."""
        return slice(self.h_lo, self.h_lo + self.n)


def slab_geometry(global_n0: int, r: int, k: int, rank: int, world: int) -> SlabGeometry:
    start, end = split_extent(global_n0, world)[rank]
    G = r * k
    g = SlabGeometry(rank, world, start, end, G if rank > 0 else 0, G if rank < world - 1 else 0, r)
    if world > 1 and min(e - s for s, e in split_extent(global_n0, world)) < G:
        raise GridError(f"slabs of {global_n0 // world} planes are thinner than the ghost depth {G}")
    return g


class DeviceSlab:
    """Backend: a slab plan on the local GPU (C ABI), exposing its ghost planes
    as torch CUDA tensors for the exchange (zero-copy via __cuda_array_interface__)."""

    def __init__(self, spec, dims, geom: SlabGeometry, *, k, arith, dtype, device, stream_ptr=None):
        from .plan import Plan
        self.plan = Plan(spec, dims, dtype=dtype, arith=arith, k=k, device=device,
                         ghost=(geom.ghost_lo, geom.ghost_hi))
        self.stream_ptr = stream_ptr
        if stream_ptr:
            self.plan.set_stream(stream_ptr)
        self.geom = geom
        self.itemsize = np.dtype(self.plan.np_dtype).itemsize
        self.typestr = np.dtype(self.plan.np_dtype).str
        self.device = device

    def torch_stream(self):
        """The plan's stream as a torch stream (created on first use when the plan
        runs on its own stream), for event ordering with the exchange."""
        import torch
        if getattr(self, "_tstream", None) is None:
            if self.stream_ptr:
                self._tstream = torch.cuda.ExternalStream(self.stream_ptr, device=f"cuda:{self.device}")
            else:
                self._tstream = torch.cuda.Stream(self.device)
                self.plan.set_stream(self._tstream.cuda_stream)
        return self._tstream

    def upload(self, box):
        self.plan.upload(box)

    def download(self, out=None):
        return self.plan.download(out)

    def launch(self, steps: int):
        self.plan.launch(steps)

    def launch_range(self, steps: int, lo: int, hi: int, finish: bool):
        self.plan.launch_range(steps, lo, hi, finish)

    def planes(self, z0: int, count: int, which: int = 0):
        """Tensor view of `count` whole planes starting at local interior plane z0
        of the current (which=0) or the other (which=1) buffer."""
        import torch
        base, origin, strides = self.plan.device_view(which)
        pe = strides[0] if self.plan.d > 1 else 1
        first = (origin // pe + z0) * pe if self.plan.d > 1 else origin + z0
        n = count * pe

        class _View:
            __cuda_array_interface__ = {"shape": (n,), "typestr": self.typestr, "version": 3,
                                        "data": (base + first * self.itemsize, False), "strides": None}
        return torch.as_tensor(_View(), device=f"cuda:{self.device}")


class SlabSweep:
    """T steps of `spec` over a slab-decomposed grid (one rank per GPU).

    ``transport`` is torch.distributed (NCCL for GPUs, gloo in the CPU
    tests); ``backend`` defaults to :class:`DeviceSlab`.
    """

    def __init__(self, spec, global_dims, *, rank, world, k, arith="fma", dtype="f64",
                 device=0, group=None, backend=None, stream_ptr=None):
        validate(spec)
        self.spec = spec
        self.r = spec.r
        if k not in _FUSED_KS[spec.d]:
            raise GridError(f"fused depth {k} unsupported for d={spec.d}")
        self.k = k
        self.rank, self.world, self.group = rank, world, group
        self.global_dims = tuple(int(n) for n in global_dims)
        self.geom = slab_geometry(self.global_dims[0], self.r, k, rank, world)
        self.dims = (self.geom.n,) + self.global_dims[1:]
        self.backend = backend or DeviceSlab(spec, self.dims, self.geom, k=k, arith=arith, dtype=dtype,
                                             device=device, stream_ptr=stream_ptr)
        self.plan = getattr(self.backend, "plan", None)
        self.exchanges = 0

    # -- data
    def local_box(self, global_box: np.ndarray) -> np.ndarray:
        return np.ascontiguousarray(global_box[self.geom.local_slice()])

    def upload(self, local_box: np.ndarray):
        self.backend.upload(local_box)
        self._fresh = True

    def download(self, out=None) -> np.ndarray:
        return self.backend.download(out)

    # -- halo exchange: my edge planes -> neighbours' ghost planes
    def _post(self, specs):
        """Post grouped point-to-point transfers; ``specs`` = [(is_send, tensor,
        peer)].  Returns a callable that completes them (on the current stream).

        NCCL (one GPU per rank) and the CPU tests move the tensors as they are.
        A ``gloo`` group over CUDA tensors is the TEST transport of the
        shared-GPU emulation (two ranks on one device, tests/test_slab.py,
        ``SB200_SHARE_GPU``): gloo moves host memory only, so the planes are
        staged through the host around the same isend/irecv calls."""
        import torch.distributed as dist
        staged = bool(specs) and specs[0][1].is_cuda and dist.get_backend(self.group) == "gloo"
        if not staged:
            ops = [dist.P2POp(dist.isend if snd else dist.irecv, t, peer, self.group) for snd, t, peer in specs]
            reqs = dist.batch_isend_irecv(ops)
            return lambda: [req.wait() for req in reqs]
        import torch
        host = [t.cpu() if snd else torch.empty(t.shape, dtype=t.dtype) for snd, t, _ in specs]
        reqs = [(dist.isend if snd else dist.irecv)(h, peer, group=self.group)
                for (snd, _, peer), h in zip(specs, host)]

        def finish():
            for req in reqs:
                req.wait()
            for (snd, t, _), h in zip(specs, host):
                if not snd:
                    t.copy_(h)
        return finish

    def _edge_specs(self, which: int):
        """(is_send, planes, peer) of this rank's edge planes and ghost planes in
        buffer `which` (0 = current, 1 = other)."""
        g = self.geom
        specs = []
        if g.ghost_lo:
            G = g.ghost_lo
            specs.append((True, self.backend.planes(0, G, which), self.rank - 1))
            specs.append((False, self.backend.planes(-G, G, which), self.rank - 1))
        if g.ghost_hi:
            G = g.ghost_hi
            specs.append((True, self.backend.planes(g.n - G, G, which), self.rank + 1))
            specs.append((False, self.backend.planes(g.n, G, which), self.rank + 1))
        return specs

    def exchange(self):
        if self.world == 1:
            return
        self._post(self._edge_specs(0))()
        self.exchanges += 1

    def run(self, steps: int, overlap: bool | None = None):
        """Advance `steps` time steps, one fused launch per k steps.

        1D, or ``overlap=False``: exchange, then launch.  2D/3D (default): the
        exchange of each interval's edge planes overlaps its interior launch
        (:meth:`_run_overlapped`)."""
        if overlap is None:
            overlap = self.spec.d >= 2 and hasattr(self.backend, "launch_range")
        g = self.geom
        if overlap and self.world > 1 and g.n >= (g.ghost_lo + g.ghost_hi):
            return self._run_overlapped(steps)
        done = 0
        ks = _FUSED_KS[self.spec.d]
        while done < steps:
            kk = max(x for x in ks if x <= min(self.k, steps - done))
            self.exchange()
            self.backend.launch(kk)
            done += kk

    def _run_overlapped(self, steps: int):
        """Per interval of kk steps: edge planes [0, G) and [n-G, n) first (range
        launches into the other buffer), their isend/irecv to the neighbours on
        a communication stream (waiting on an event after the edges), the slab
        interior [G, n-G) meanwhile on the main stream (completing the step);
        the next interval's launches wait for the received ghost planes.  The
        first interval exchanges the uploaded edges up front."""
        g = self.geom
        cuda = isinstance(self.backend, DeviceSlab)
        if cuda:
            import torch
            main = self.backend.torch_stream()
            comm = getattr(self, "_comm_stream", None) or torch.cuda.Stream(self.backend.device)
            self._comm_stream = comm
        e_lo = g.ghost_lo                       # edge planes sent down: [0, G_lo)
        e_hi = g.n - g.ghost_hi                 # edge planes sent up: [n - G_hi, n)
        ks = _FUSED_KS[self.spec.d]
        done = 0
        if getattr(self, "_fresh", True):
            self.exchange()                     # ghosts of the uploaded state
            self._fresh = False
        while done < steps:
            kk = max(x for x in ks if x <= min(self.k, steps - done))
            if e_lo:
                self.backend.launch_range(kk, 0, e_lo, False)
            if g.ghost_hi:
                self.backend.launch_range(kk, e_hi, g.n, False)
            specs = self._edge_specs(1)
            if cuda:
                ev = torch.cuda.Event()
                ev.record(main)
                with torch.cuda.stream(comm):
                    comm.wait_event(ev)
                    finish = self._post(specs)
                self.backend.launch_range(kk, e_lo, e_hi, True)     # interior, concurrent with the exchange
                with torch.cuda.stream(main):                       # main stream waits for the ghosts
                    finish()
                    main.wait_stream(comm)
            else:
                self._post(specs)()
                self.backend.launch_range(kk, e_lo, e_hi, True)
            self.exchanges += 1
            done += kk


def gather_interior(sweep: SlabSweep, local_box: np.ndarray) -> np.ndarray:
    """This rank's slab interior (axis 0) from its downloaded local box."""
    return local_box[sweep.geom.interior_slice()]


def exchange_local(sweeps: list[SlabSweep]) -> None:
    """Ghost exchange between slabs held by ONE process (several plans on one
    or more GPUs): plain device copies, neighbours in order.  Used to emulate
    the decomposition on a single GPU and for single-process multi-GPU runs
    (peer copies over NVLink)."""
    import torch
    devs = sorted({getattr(s.backend, "device", 0) for s in sweeps})
    for d in devs:
        torch.cuda.synchronize(d)
    for a, b in zip(sweeps[:-1], sweeps[1:]):
        G = b.geom.ghost_lo
        b.backend.planes(-G, G).copy_(a.backend.planes(a.geom.n - G, G))
        a.backend.planes(a.geom.n, G).copy_(b.backend.planes(0, G))
    for d in devs:
        torch.cuda.synchronize(d)


def run_local(sweeps: list[SlabSweep], steps: int, overlap: bool | None = None) -> None:
    """`steps` time steps of a single-process slab set (see exchange_local).

    2D/3D (default): the same split as SlabSweep._run_overlapped -- edge planes
    by range launches, their copy into the neighbours' ghost planes of the
    other buffer, then the slab interiors completing the step."""
    import torch
    ks = _FUSED_KS[sweeps[0].spec.d]
    k = sweeps[0].k
    if overlap is None:
        overlap = sweeps[0].spec.d >= 2
    done = 0
    if overlap:
        exchange_local(sweeps)
    while done < steps:
        kk = max(x for x in ks if x <= min(k, steps - done))
        if not overlap:
            exchange_local(sweeps)
            for s in sweeps:
                s.backend.launch(kk)
            done += kk
            continue
        for s in sweeps:
            g = s.geom
            if g.ghost_lo:
                s.backend.launch_range(kk, 0, g.ghost_lo, False)
            if g.ghost_hi:
                s.backend.launch_range(kk, g.n - g.ghost_hi, g.n, False)
        devs = sorted({getattr(s.backend, "device", 0) for s in sweeps})
        for d in devs:
            torch.cuda.synchronize(d)
        for a, b in zip(sweeps[:-1], sweeps[1:]):
            G = b.geom.ghost_lo
            b.backend.planes(-G, G, 1).copy_(a.backend.planes(a.geom.n - G, G, 1))
            a.backend.planes(a.geom.n, G, 1).copy_(b.backend.planes(0, G, 1))
        for d in devs:
            torch.cuda.synchronize(d)
        for s in sweeps:
            g = s.geom
            s.backend.launch_range(kk, g.ghost_lo, g.n - g.ghost_hi, True)
        done += kk
    for d in sorted({getattr(s.backend, "device", 0) for s in sweeps}):
        torch.cuda.synchronize(d)
