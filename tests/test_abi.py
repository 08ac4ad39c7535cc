"""CPU-side checks of the C-ABI boundary (no GPU compute): the library loads, exports every
function include/hj.h declares, validates arguments before touching a device, and computes
the paper's resource figures (host-only)."""
import ctypes
import os
import re

import pytest

from paper_2006_16465_b200 import hj

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    src = open(os.path.join(ROOT, "include", "hj.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("hj_", "jacobi_"))))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2006_16465_b200 import build
    build.build()
    L = hj.lib()
    names = declared_functions()
    assert {"jacobi_solve", "jacobi_solve_device", "jacobi_solve_dist", "hj_plan_create",
            "hj_plan_run", "hj_plan_solve", "hj_plan_destroy", "hj_resource_figures",
            "hj_last_error", "hj_nccl_unique_id"} <= set(names)
    for n in names:
        assert hasattr(L, n), n


def test_sass_targets_sm100a():
    """The .so carries sm_100a code (TMA + bulk copies in the cycle kernels)."""
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", hj.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", hj.LIB_PATH], capture_output=True, text=True).stdout
    assert "UTMALDG" in sass        # cp.async.bulk.tensor (2D tiles)
    assert "UBLKCP" in sass         # cp.async.bulk (1D tiles)


@pytest.mark.parametrize("kw,status", [
    (dict(dim=3), hj.HJ_ERR_INVALID_ARG),
    (dict(nx=0), hj.HJ_ERR_INVALID_ARG),
    (dict(h=-1.0), hj.HJ_ERR_INVALID_ARG),
    (dict(h=float("nan")), hj.HJ_ERR_INVALID_ARG),
    (dict(tile=(64, 32)), hj.HJ_ERR_INVALID_CONFIG),     # tile > n
    (dict(tile=(0, 8)), hj.HJ_ERR_INVALID_CONFIG),
    (dict(k=0), hj.HJ_ERR_INVALID_CONFIG),
    (dict(overlap=3), hj.HJ_ERR_INVALID_CONFIG),
    (dict(tol=1.5), hj.HJ_ERR_INVALID_CONFIG),
    (dict(tol=-1.0), hj.HJ_ERR_INVALID_CONFIG),
    (dict(max_cycles=-1), hj.HJ_ERR_INVALID_CONFIG),
    (dict(mode="classic", k=4), hj.HJ_ERR_INVALID_CONFIG),
])
def test_invalid_arguments_rejected_before_device_work(kw, status):
    import numpy as np
    args = dict(dim=2, nx=40, ny=40, h=1 / 41)
    prm = dict(tile=(32, 32), k=4, tol=1e-4, max_cycles=10)
    for key in list(kw):
        if key in args:
            args[key] = kw.pop(key)
    prm.update(kw)
    n = args["nx"] * args["ny"]
    with pytest.raises(hj.HJError) as ei:
        hj.jacobi_solve(args["dim"], args["nx"], args["ny"], args["h"], np.ones(n), **prm)
    assert ei.value.status == status


def test_resource_figures_match_paper_formula():
    """hj_resource_figures is host-only: the paper's 800 B / 26,688 B and block counts."""
    assert hj.hj_resource_figures(1, 1024, 1, tile=32, k=4)[2] == 800
    assert hj.hj_resource_figures(2, 1024, 1024, tile=(32, 32), k=16) == (1024, 1024 * 1024, 26688)
    assert hj.hj_resource_figures(1, 12, 1, tile=4, k=1)[0] == 3
    assert hj.hj_resource_figures(2, 12, 12, tile=(4, 4), k=1)[0] == 9
    assert hj.hj_resource_figures(1, 1024, 1, tile=1024, k=16, dtype="f64")[2] == 24608
