"""Slab decomposition: geometry (CPU), the distributed orchestration over a
world-size-2 gloo group with an oracle-backed CPU backend (CPU), and the
single-GPU emulation of 2/4 slabs through the real kernels (GPU).  The bar
is bit-identity with the undecomposed sweep."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch

from conftest import seeded_box
from oracle import c_oracle

from paper_2103_08825_b200.core import GridError, canonical, config_spec, make_stencil_spec
from paper_2103_08825_b200.slab import (SlabSweep, run_local, slab_geometry, split_extent)


def test_split_extent_balanced():
    assert split_extent(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert split_extent(512, 8)[7] == (448, 512)
    with pytest.raises(GridError):
        split_extent(3, 4)


def test_slab_geometry_ghosts():
    g0 = slab_geometry(100, 2, 8, 0, 4)
    g1 = slab_geometry(100, 2, 8, 1, 4)
    g3 = slab_geometry(100, 2, 8, 3, 4)
    assert (g0.ghost_lo, g0.ghost_hi) == (0, 16)
    assert (g1.ghost_lo, g1.ghost_hi) == (16, 16)
    assert (g3.ghost_lo, g3.ghost_hi) == (16, 0)
    assert g1.local_slice() == slice(25 - 16 + 2, 50 + 16 + 2)
    with pytest.raises(GridError, match="thinner"):
        slab_geometry(40, 2, 8, 0, 4)


class HostSlab:
    """CPU backend: the oracle advances the local box; ghost sides are
    computed like interior (the oracle treats only the outer r planes as
    halo), which is exactly the device kernels' slab semantics."""

    def __init__(self, spec, geom):
        self.spec, self.geom = spec, geom
        self.offs, self.ws = canonical(spec)

    def upload(self, box):
        self.box = np.array(box, copy=True)

    def download(self, out=None):
        return self.box.copy()

    def launch(self, steps):
        c_oracle.sweep(self.box, self.spec.r, self.offs, self.ws, steps, threads=1, inplace=True)

    def launch_range(self, steps, lo, hi, finish):
        # the device semantics: parts of one step write [lo, hi) of the other
        # buffer from the current one; `finish` swaps
        if getattr(self, "next", None) is None:
            self.full = c_oracle.sweep(self.box, self.spec.r, self.offs, self.ws, steps, threads=1)
            self.next = self.box.copy()
        z = self.geom.h_lo
        self.next[z + lo:z + hi] = self.full[z + lo:z + hi]
        if finish:
            self.box, self.next, self.full = self.next, None, None

    def planes(self, z0, count, which=0):
        z = self.geom.h_lo + z0
        arr = self.box if which == 0 else self.next
        return torch.from_numpy(arr[z:z + count]).reshape(-1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, dims, k, steps, outdir, overlap=None):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec = config_spec(cfg) if not cfg.startswith("p:") else make_stencil_spec(cfg[2:])
    gbox = seeded_box(dims, spec.r, seed=7)
    geom = slab_geometry(dims[0], spec.r, k, rank, world)
    sw = SlabSweep(spec, dims, rank=rank, world=world, k=k, backend=HostSlab(spec, geom))
    sw.upload(sw.local_box(gbox))
    sw.run(steps, overlap=overlap)
    out = sw.download()
    np.save(os.path.join(outdir, f"r{rank}.npy"), out[geom.interior_slice()])
    np.save(os.path.join(outdir, f"x{rank}.npy"), np.array([sw.exchanges]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,dims,k,steps,overlap", [
    ("c2", (4000,), 8, 37, None),
    ("c4", (40, 11, 13), 2, 9, None),       # 2D/3D default: exchange overlapped with the interior
    ("c4", (40, 11, 13), 2, 9, False),
    ("c3b", (50, 31), 4, 13, None),
])
def test_gloo_world2_bit_identical(cfg, dims, k, steps, overlap):
    import torch.multiprocessing as mp
    world = 2
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(world, _free_port(), cfg, dims, k, steps, td, overlap), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(td, f"r{r}.npy")) for r in range(world)], axis=0)
        nex = int(np.load(os.path.join(td, "x0.npy"))[0])
    spec = config_spec(cfg)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(seeded_box(dims, spec.r, seed=7), spec.r, offs, ws, steps)
    r = spec.r
    want_int = want[r:r + dims[0]]
    assert got.shape == want_int.shape
    assert got.tobytes() == want_int.tobytes()
    assert nex >= steps // k


def _device_worker(rank, world, port, cfg, dims, k, steps, arith, outdir):
    """One rank of the shared-GPU emulation: the real DeviceSlab path (sm_100a
    kernels, range launches, plane views, main/communication streams) driven
    through torch.distributed, every rank on cuda:0 with the gloo test
    transport (SlabSweep._post stages the planes through the host)."""
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    spec = config_spec(cfg)
    gbox = seeded_box(dims, spec.r, seed=11)
    sw = SlabSweep(spec, dims, rank=rank, world=world, k=k, arith=arith, device=0, stream_ptr=stream.cuda_stream)
    sw.upload(sw.local_box(gbox))
    sw.run(steps)
    torch.cuda.synchronize()
    out = sw.download()
    np.save(os.path.join(outdir, f"r{rank}.npy"), out[sw.geom.interior_slice()])
    np.save(os.path.join(outdir, f"x{rank}.npy"), np.array([sw.exchanges]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,dims,k,steps,arith,world", [
    ("c2", (200000,), 16, 50, "exact", 2),      # 1D: exchange before each launch
    ("c5", (64, 70, 130), 2, 9, "exact", 2),    # 3D box3d: edges, exchange on the comm stream, interior
    ("c4", (96, 70, 66), 2, 9, "fma", 3),       # composed 3D star, three ranks (a middle slab with two ghost sides)
    ("c3b", (400, 300), 4, 13, "exact", 2),
    ("c3a", (600, 500), 32, 70, "fma", 2),      # separable composed 2D on slabs
])
def test_torch_distributed_ranks_on_one_gpu_bit_identical(cfg, dims, k, steps, arith, world):
    """SlabSweep.run / _run_overlapped through torch.distributed with real
    device slabs: bit-identical to the undecomposed sweep on one plan."""
    import torch.multiprocessing as mp
    from paper_2103_08825_b200.plan import Plan
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_device_worker, args=(world, _free_port(), cfg, dims, k, steps, arith, td), nprocs=world, join=True)
        got = np.concatenate([np.load(os.path.join(td, f"r{r}.npy")) for r in range(world)], axis=0)
        nex = int(np.load(os.path.join(td, "x0.npy"))[0])
    spec = config_spec(cfg)
    gbox = seeded_box(dims, spec.r, seed=11)
    with Plan(spec, dims, k=k, arith=arith, device=0) as p:
        p.upload(gbox)
        p.run(steps)
        want = p.download()
    r = spec.r
    assert got.tobytes() == want[r:r + dims[0]].tobytes()
    if arith == "exact":
        offs, ws = canonical(spec)
        ref = c_oracle.sweep(gbox, r, offs, ws, steps)
        assert got.tobytes() == ref[r:r + dims[0]].tobytes()
    assert nex >= steps // k


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,dims,k,g", [
    ("c2", (300000,), 16, 2), ("c2", (300000,), 8, 4), ("c1", (100003,), 8, 3),
    ("c4", (96, 70, 66), 4, 4), ("c5", (64, 70, 130), 2, 2), ("c3b", (400, 300), 8, 4),
])
def test_single_gpu_slab_emulation_bit_identical(cfg, dims, k, g):
    spec = config_spec(cfg)
    gbox = seeded_box(dims, spec.r, seed=3)
    sweeps = [SlabSweep(spec, dims, rank=r, world=g, k=k, arith="exact", device=0) for r in range(g)]
    for s in sweeps:
        s.upload(s.local_box(gbox))
    steps = 3 * k + 1
    run_local(sweeps, steps)
    got = np.concatenate([s.download()[s.geom.interior_slice()] for s in sweeps], axis=0)
    offs, ws = canonical(spec)
    want = c_oracle.sweep(gbox, spec.r, offs, ws, steps)
    assert got.tobytes() == want[spec.r:spec.r + dims[0]].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("k,g", [(32, 2), (16, 3)])
def test_single_gpu_slab_emulation_sep2d_matches_whole_grid(k, g):
    # separable composed 2D (FMA, rank-1 weights): row slabs with k-deep ghosts
    # reproduce the whole-grid plan bit for bit (same composed weights per row,
    # x bands on each slab, y bands on the physical sides only); exchange overlapped
    spec = config_spec("c3a")
    dims = (300, 333)
    gbox = seeded_box(dims, 1, seed=8)
    sweeps = [SlabSweep(spec, dims, rank=r, world=g, k=k, arith="fma", device=0) for r in range(g)]
    for s in sweeps:
        s.upload(s.local_box(gbox))
    steps = 2 * k
    run_local(sweeps, steps)
    got = np.concatenate([s.download()[s.geom.interior_slice()] for s in sweeps], axis=0)
    from paper_2103_08825_b200.plan import sweep
    whole = sweep(spec, gbox, steps, arith="fma", k=k)
    assert got.tobytes() == whole[1:1 + dims[0]].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 3])
def test_single_gpu_slab_emulation_composed3d_matches_whole_grid(g):
    # composed 3D star (FMA, k=2): z-slabs with 2-plane ghosts reproduce the
    # whole-grid plan bit for bit (slab sides are interior-like; only the
    # physical shell takes the level-by-level kernel)
    spec = config_spec("c4")
    dims = (40, 37, 70)
    gbox = seeded_box(dims, 1, seed=6)
    sweeps = [SlabSweep(spec, dims, rank=r, world=g, k=2, arith="fma", device=0) for r in range(g)]
    for s in sweeps:
        s.upload(s.local_box(gbox))
    steps = 8
    run_local(sweeps, steps)
    got = np.concatenate([s.download()[s.geom.interior_slice()] for s in sweeps], axis=0)
    from paper_2103_08825_b200.plan import sweep
    whole = sweep(spec, gbox, steps, arith="fma", k=2)
    assert got.tobytes() == whole[1:1 + dims[0]].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,k,g", [("c2", 32, 2), ("c1", 64, 3), ("c2", 16, 3)])
def test_single_gpu_slab_emulation_composed_matches_whole_line(cfg, k, g):
    # composed path (FMA): slabs reproduce a whole-line plan bit for bit --
    # every output takes the same composed taps or the same boundary window
    spec = config_spec(cfg)
    dims = (300001,)
    gbox = seeded_box(dims, spec.r, seed=5)
    sweeps = [SlabSweep(spec, dims, rank=r, world=g, k=k, arith="fma", device=0) for r in range(g)]
    for s in sweeps:
        s.upload(s.local_box(gbox))
    steps = 3 * k + 1
    run_local(sweeps, steps)
    got = np.concatenate([s.download()[s.geom.interior_slice()] for s in sweeps], axis=0)
    from paper_2103_08825_b200.plan import sweep
    whole = sweep(spec, gbox, steps, arith="fma", k=k)
    assert got.tobytes() == whole[spec.r:spec.r + dims[0]].tobytes()
