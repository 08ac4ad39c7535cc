"""Pins for overlapping subdomains (§3.5 / §4.3).  CPU only."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2006_16465_b200.inputs import make_problem
from tests import _brute

COUNTS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "cross_impl_counts_overlap.json")))


def run(p, **kw):
    return oracle.solve(p["dim"], p["nx"], p["ny"], p["h"], p["f"], p["bc"], p["x0"], **kw)


def test_block_plan_paper_example_and_eq8():
    """N=12, tpb=4, o=2 -> (12-2)/(4-2) = 5 blocks (Eq. 8); half-split ownership
     -> owned [1-3],[4-5],[6-7],[8-9],[10-12]."""
    plan = oracle.block_plan(12, 4, 2)
    assert [(s, s + w - 1) for s, w, _, _ in plan] == [(1, 4), (3, 6), (5, 8), (7, 10), (9, 12)]
    assert [(a, b) for _, _, a, b in plan] == [(1, 3), (4, 5), (6, 7), (8, 9), (10, 12)]
    # Eqs. 8-9 at N=1024, tpb=32, o=16: 63 blocks, 2016 threads
    assert oracle.resource_figures(1, 1024, 1, 32, overlap=16)[:2] == (63, 2016)
    # Eq. 14: ((N-o)/(tpb-o))^2 tpb^2 at N=1024, tpb=32, o=4 -> 36^2 blocks
    assert oracle.resource_figures(2, 1024, 1024, 32, 32, overlap=4)[0] == ((1024 - 4) // 28 + 1) ** 2


def test_block_plan_matches_hand_rule_and_covers_exactly():
    rng = np.random.default_rng(3)
    for _ in range(300):
        n = int(rng.integers(4, 400))
        T = int(rng.integers(2, n + 1))
        o = 2 * int(rng.integers(0, (T + 1) // 2)) if T > 2 else 0
        if o >= T:
            o = 0
        plan = oracle.block_plan(n, T, o)
        hand = _brute.plan_1d(n, T, o)
        assert [(s, s + w - 1, a, b) for s, w, a, b in plan] == hand
        owned = np.zeros(n + 2, dtype=int)
        for s, w, a, b in plan:
            assert s <= a <= b <= s + w - 1
            owned[a:b + 1] += 1
        assert np.all(owned[1:n + 1] == 1)


@pytest.mark.parametrize("dim,nx,ny,tile,k,ov", [(1, 30, 1, (8, 1), 3, 2), (1, 29, 1, (8, 1), 4, 4),
                                                 (2, 14, 11, (6, 5), 3, (2, 2)), (2, 13, 13, (6, 6), 2, (4, 2))])
def test_overlap_cycle_equals_dense_affine_map(dim, nx, ny, tile, k, ov):
    """One oracle cycle with overlap == M z + g built from per-block Jacobi matrices, rows taken
    from the owning block (brute force, P8)."""
    p = make_problem("R", dim, nx, ny)
    ox, oy = ov if isinstance(ov, tuple) else (ov, 0)
    M, g, _, _ = _brute.cycle_affine(dim, nx, ny, p["h"], p["f"], tile[0], tile[1], k, ox, oy)
    z = _brute.ringed_vector(dim, nx, ny, p["bc"], p["x0"])
    r = run(p, mode="hier", tile=tile, k=k, overlap=ov, tol=0.0, max_cycles=1)
    ref = M @ z + g
    assert np.allclose(r["x"].reshape(-1), ref, rtol=0, atol=1e-13 * max(1, np.abs(ref).max()))


@pytest.mark.parametrize("dim,n,tile,ov", [(1, 64, 16, 6), (1, 37, 8, 2), (2, 40, (8, 8), 2), (2, 29, (10, 6), (4, 2))])
def test_overlap_k1_equals_classic(dim, n, tile, ov):
    """k = 1: every owned point gets one Jacobi update from the snapshot -> classic, bitwise."""
    p = make_problem("R", dim, n)
    a = run(p, mode="hier", tile=tile, k=1, overlap=ov, tol=0.0, max_cycles=40)
    b = run(p, mode="classic", tol=0.0, max_cycles=40)
    assert np.array_equal(a["x"], b["x"])


@pytest.mark.parametrize("case", COUNTS["cases"], ids=lambda c: f"{c['dim']}d-k{c['k']}-o{c['o']}")
def test_overlap_cross_implementation_counts(case):
    """Cycle counts with overlap equal an independent implementation's (SURVEY.md Appendix A,
    the Table 3 / Table 4 checks)."""
    if case.get("slow") and os.environ.get("HJ_SLOW") != "1":
        pytest.skip("slow oracle run; set HJ_SLOW=1")
    p = make_problem(case["protocol"], case["dim"], case["n"])
    r = run(p, mode="hier", tile=(case["tile"], case["tile"]), k=case["k"], overlap=case["o"],
            tol=case["tol"], max_cycles=10**7, history=False)
    assert r["cycles"] == case["cycles"]


def test_overlap_reduces_cycles():
    """PAPER.md:293 ('allowing just two points to overlap causes a drop in the number of cycles')
    and SPEC.md:291 (desk-scale trend): for k >= 8, cycles(o=2) <= cycles(o=0)."""
    p = make_problem("P", 1, 256)
    for k in (8, 16, 32):
        c0 = run(p, mode="hier", tile=32, k=k, overlap=0, tol=1e-4, max_cycles=10**6, history=False)["cycles"]
        c2 = run(p, mode="hier", tile=32, k=k, overlap=2, tol=1e-4, max_cycles=10**6, history=False)["cycles"]
        assert c2 <= c0


def test_overlap_halo_locality_and_order_independence():
    p = make_problem("R", 2, 40, 30)
    base = run(p, mode="hier", tile=(8, 8), k=5, overlap=(2, 4), tol=0.0, max_cycles=2)["x"]
    rev = run(p, mode="hier", tile=(8, 8), k=5, overlap=(2, 4), tol=0.0, max_cycles=2, tile_order=1)["x"]
    assert np.array_equal(base, rev)
