"""Multi-process (gloo, world size 2, CPU) test of the row-slab decomposition used by the
multi-GPU path: each rank advances its slab with the oracle, exchanging one ghost row per
neighbour per cycle and all-reducing the per-rank residual partials — exactly the data flow of
dist.cu.  The slab iterates must equal the single-process oracle bit for bit (reading c18)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2006_16465_b200.inputs import make_problem
from paper_2006_16465_b200.slabs import slab, neighbours


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nx, ny, tile, k, cycles, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = make_problem("R", 2, nx, ny)
    b, e = slab(ny, tile, rank, world)
    lo, hi = neighbours(rank, world)
    X = p["x0"].reshape(ny, nx)[b:e].copy()
    F = p["f"].reshape(ny, nx)[b:e].copy()
    bc = p["bc"]
    south_ring, north_ring = bc[:nx], bc[nx:2 * nx]
    west, east = bc[2 * nx:2 * nx + ny][b:e], bc[2 * nx + ny:][b:e]
    hist = []
    for c in range(cycles + 1):
        # ghost rows: neighbours' boundary rows of the current iterate (NCCL send/recv analogue)
        south = torch.from_numpy(south_ring.copy())
        north = torch.from_numpy(north_ring.copy())
        reqs = []
        if lo is not None:
            reqs.append(dist.isend(torch.from_numpy(X[0].copy()), lo))
            south = torch.empty(nx, dtype=torch.float64)
            reqs.append(dist.irecv(south, lo))
        if hi is not None:
            reqs.append(dist.isend(torch.from_numpy(X[-1].copy()), hi))
            north = torch.empty(nx, dtype=torch.float64)
            reqs.append(dist.irecv(north, hi))
        for r in reqs:
            r.wait()
        ring = np.concatenate([south.numpy(), north.numpy(), west, east])
        # residual partial of this slab (allreduce analogue of the per-tile-row vector)
        r2 = torch.tensor([oracle.residual(2, nx, e - b, p["h"], F, ring, X) ** 2], dtype=torch.float64)
        dist.all_reduce(r2)
        hist.append(float(np.sqrt(r2.item())))
        if c == cycles:
            break
        X = oracle.solve(2, nx, e - b, p["h"], F, ring, X, mode="hier", tile=(tile, tile), k=k,
                         tol=0.0, max_cycles=1, history=False)["x"]
    out[rank] = (b, e, X, hist)
    dist.destroy_process_group()


@pytest.mark.parametrize("nx,ny,tile,k,cycles", [(40, 64, 8, 5, 6), (33, 96, 32, 16, 3)])
def test_two_rank_slabs_match_single_process(nx, ny, tile, k, cycles):
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), nx, ny, tile, k, cycles, out), nprocs=world, join=True)
    p = make_problem("R", 2, nx, ny)
    ref = oracle.solve(2, nx, ny, p["h"], p["f"], p["bc"], p["x0"], mode="hier", tile=(tile, tile), k=k,
                       tol=0.0, max_cycles=cycles)
    full = np.zeros((ny, nx))
    for r in range(world):
        b, e, X, hist = out[r]
        full[b:e] = X
        np.testing.assert_allclose(hist, ref["history"], rtol=1e-12)
    assert np.array_equal(full, ref["x"])


def test_slab_partition_properties():
    for ny, unit in [(16384, 32), (100, 16), (1024, 32), (70, 32)]:
        for P in (1, 2, 4, 8):
            if (ny + unit - 1) // unit < P:
                continue
            spans = [slab(ny, unit, r, P) for r in range(P)]
            assert spans[0][0] == 0 and spans[-1][1] == ny
            for (b0, e0), (b1, e1) in zip(spans, spans[1:]):
                assert e0 == b1
            assert all(b % unit == 0 for b, _ in spans)
            sizes = [e - b for b, e in spans[:-1]]      # all but the (possibly ragged) last
            if sizes:
                assert max(sizes) - min(sizes) <= unit
    assert slab(16384, 32, 3, 8) == (6144, 8192)
