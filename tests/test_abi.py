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


@pytest.mark.parametrize("kw", [
    dict(nx=40, ny=41),                       # even n: no vertex-centred coarse grid (reading c24)
    dict(nx=41, ny=40),
    dict(overlap=2),
    dict(omega=1.5),
    dict(omega=-0.1),
    dict(levels=1),
    dict(nu1=-1),
    dict(stencil=True),
])
def test_multigrid_invalid_configs_rejected_before_device_work(kw):
    import numpy as np
    nx, ny = kw.pop("nx", 41), kw.pop("ny", 41)
    stencil = [-1.0, -1.0, -1.0, -1.0, 4.0] if kw.pop("stencil", False) else None
    prm = dict(mode="mg", tile=(8, 8), k=4, tol=1e-4, max_cycles=10)
    prm.update(kw)
    with pytest.raises(hj.HJError) as ei:
        hj.jacobi_solve(2, nx, ny, 1.0 / (nx + 1), np.ones(nx * ny), stencil=stencil, **prm)
    assert ei.value.status == hj.HJ_ERR_INVALID_CONFIG


def test_params_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of hj_params / hj_problem / hj_result / hj_dist has the C layout (gcc)."""
    import subprocess
    src = tmp_path / "layout.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "hj.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(hj_params), '
                   'offsetof(hj_params, overlap_y), offsetof(hj_params, mg_omega), '
                   'offsetof(hj_params, mg_levels), sizeof(hj_problem), sizeof(hj_result), sizeof(hj_dist));'
                   'return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = [int(v) for v in subprocess.check_output([str(exe)], text=True).split()]
    P = hj.hj_params
    want = [ctypes.sizeof(P), P.overlap_y.offset, P.mg_omega.offset, P.mg_levels.offset,
            ctypes.sizeof(hj.hj_problem), ctypes.sizeof(hj.hj_result), ctypes.sizeof(hj.hj_dist)]
    assert got == want
