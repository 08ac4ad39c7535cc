"""Child process of tests/test_gpu_peer.py: one rank of a peer-transport row-slab solve.

Exchanges its IPC handle blob through multiprocessing queues (the parent plays all-gather),
solves, and sends back its local rows, the history and the cycle count."""
import os


def run(rank, nranks, case, up, down, out):
    try:
        import numpy as np
        import torch
        from paper_2006_16465_b200 import hj, slabs
        from paper_2006_16465_b200.inputs import make_general, make_problem
        torch.cuda.set_device(0)
        dev = torch.device("cuda:0")
        nx, ny = case["nx"], case["ny"]
        p = make_general(case["recipe"], 2, nx, ny) if case.get("general") else make_problem(case["recipe"], 2, nx, ny)
        unit = 8 if case["mode"] == "classic" else case["tile"][1]
        rb, re = slabs.slab(ny, unit, rank, nranks)
        f = torch.as_tensor(p["f"].reshape(ny, nx)[rb:re].reshape(-1).copy(), device=dev)
        x0 = torch.as_tensor(p["x0"].reshape(ny, nx)[rb:re].reshape(-1).copy(), device=dev)
        bc = torch.as_tensor(p["bc"], device=dev)
        prm = dict(mode=case["mode"], tile=case["tile"], k=case["k"], tol=case["tol"],
                   max_cycles=case["max_cycles"], dtype=case.get("dtype", "f64"))
        if case["mode"] == "classic":
            prm.pop("tile"); prm["k"] = 1
        pl = hj.PeerPlan(nx, ny, p["h"], f, bc, x0, rank=rank, nranks=nranks, row_begin=rb, row_end=re,
                         stencil=p.get("stencil"), **prm)
        up.put((rank, pl.export()))
        blobs = down.get(timeout=120)
        pl.attach(blobs)
        r = pl.solve()
        again = None
        if case.get("rerun"):
            pl.reset()
            again = pl.solve()
        res = dict(rank=rank, rb=rb, re=re, x=r["x"].cpu().numpy(), hist=r["history"].cpu().numpy(),
                   cycles=r["cycles"], converged=r["converged"], status=r["status"],
                   lpc=pl.launches_per_cycle())
        if again is not None:
            res["x2"] = again["x"].cpu().numpy()
            res["cycles2"] = again["cycles"]
        torch.cuda.synchronize()
        out.put(res)
        down.get(timeout=120)   # every rank is done before any plan is destroyed
        pl.close()
    except Exception as e:  # report instead of hanging the parent
        import traceback
        out.put(dict(rank=rank, error=f"{e}\n{traceback.format_exc()}"))
