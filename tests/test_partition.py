"""Route-axis partition (libvol `vol_partition_route`, host only) — CPU tests.

The paper's regulariser is block-local with boundary conditions from the neighbour blocks, so
between GPUs the cut surface *is* the halo.  Pins: the arc length against closed forms on straight and
staircase routes; equal block counts; the (arc, x, y, z) order; invariance under the caller's block order;
and, on the configs[3] city geometry (1 km staircase route, 0.8 m blocks), that every rank talks only to
r − 1 and r + 1, that its ghost set is bounded by the route's cross-section, and that the halo-dependent
launch B stays a few percent of the blocks — against the lexicographic (x, y, z) cut the round-1 bench
used, which cuts the +y canyons lengthwise."""
import numpy as np
import pytest
import torch

from paper_1604_03734_b200 import partition_route, plan_shard


def _lex_part(c, world):
    key = (c[:, 0].astype(np.int64) * 4096 + c[:, 1]) * 65536 + c[:, 2]
    o = np.argsort(key, kind="stable")
    part = np.empty(len(c), np.int32)
    for r in range(world):
        part[o[r * len(c) // world:(r + 1) * len(c) // world]] = r
    return part


def test_arc_length_straight_route_and_ties():
    # route along x at height 1.5 from x = 0 to x = 8 (metres), blocks of edge 1: centre b + 0.5
    route = np.array([[0.0, 0.0, 1.5], [8.0, 0.0, 1.5]])
    c = np.array([[x, y, z] for x in range(-2, 10) for y in (-1, 0, 2) for z in (0, 3)], np.int32)
    part, arc = partition_route(c, route, 1.0, 4, return_arc=True)
    assert np.array_equal(arc, np.clip(c[:, 0] + 0.5, 0.0, 8.0))
    # ties (same arc) broken by (x, y, z): the order is lexicographic in (arc, x, y, z)
    order = np.lexsort((c[:, 2], c[:, 1], c[:, 0], arc))
    expect = np.empty(len(c), np.int32)
    for r in range(4):
        expect[order[r * len(c) // 4:(r + 1) * len(c) // 4]] = r
    assert np.array_equal(part, expect)
    assert np.bincount(part).tolist() == [len(c) // 4] * 4


def test_arc_length_staircase_closed_form():
    # +x for 10 m, then +y for 6 m, then +x for 4 m; block edge 0.5 m
    route = np.array([[0.0, 0.0, 0.0], [10.0, 0.0, 0.0], [10.0, 6.0, 0.0], [14.0, 6.0, 0.0]])
    e = 0.5
    pts = {  # block -> expected arc length of its centre
        (3, -5, 0): 1.75,          # beside segment 0: arc = x
        (21, 3, 0): 10.0 + 1.75,   # beside segment 1 (x = 10.75, y = 1.75): arc = 10 + y
        (25, 14, 0): 16.0 + 2.75,  # beside segment 2 (x = 12.75, y = 7.25): arc = 16 + (x − 10)
        (40, 20, 0): 20.0,         # past the end: clamped to the total length
        (-4, 0, 0): 0.0,           # before the start
    }
    c = np.array(list(pts), np.int32)
    _, arc = partition_route(c, route, e, 1, return_arc=True)
    assert np.allclose(arc, list(pts.values()), atol=1e-12)


def test_partition_invariant_under_caller_order():
    rng = np.random.default_rng(3)
    c = np.unique(rng.integers(-20, 20, size=(3000, 3)), axis=0).astype(np.int32)
    route = np.array([[-16.0, -16.0, 0.0], [0.0, -16.0, 0.0], [0.0, 16.0, 0.0], [16.0, 16.0, 0.0]])
    part = partition_route(c, route, 1.0, 5)
    perm = rng.permutation(len(c))
    part2 = partition_route(c[perm], route, 1.0, 5)
    assert np.array_equal(part2, part[perm])
    counts = np.bincount(part, minlength=5)
    assert counts.max() - counts.min() <= 1
    # contiguity along the route: ranks are ordered by arc length
    _, arc = partition_route(c, route, 1.0, 5, return_arc=True)
    for r in range(4):
        assert arc[part == r].max() <= arc[part == r + 1].min()


def test_bad_arguments():
    from paper_1604_03734_b200 import _native as N
    with pytest.raises(N.VolError):
        partition_route(np.zeros((2, 3), np.int32), np.zeros((0, 3)), 1.0, 2)
    with pytest.raises(N.VolError):
        partition_route(np.zeros((2, 3), np.int32), np.zeros((2, 3)), 0.0, 2)


_CITY = {}


def _city_standin():
    """configs[3] geometry (1 km staircase, v = 0.1 m, μ = 0.5 m): the candidate blocks within μ + half a
    block diagonal of a surface, below the façade tops (the roof plane z = H outside the canyons is never
    observed, hence never allocated).  A 2-3-block-thick superset of the allocated shell, built in seconds
    on the CPU (the allocated set needs the per-voxel visibility pass; its GPU counterpart is in
    tests/test_gpu_fullsize.py)."""
    if "c" not in _CITY:
        from synth import scenes
        plan = scenes.city_plan(0, length=1000.0)
        c = plan.cand
        c = c[(c[:, 2].double() + 1) * plan.block_edge < plan.H - plan.mu]
        _CITY["c"] = (c.numpy(), plan)
    return _CITY["c"]


def _stats(c, part, world):
    rows = []
    for r in range(world):
        p = plan_shard(c, part, world, r)
        n_b = len(np.unique(p["send"]))   # local blocks with a remote neighbour = launch B
        peers = [q for q in range(world) if p["peer_send"][q] > 0 or p["peer_recv"][q] > 0]
        rows.append(dict(n_local=p["n_local"], n_ghost=p["n_ghost"], n_b=n_b, peers=peers))
    return rows


@pytest.mark.parametrize("world", [2, 4, 8])
def test_city_route_partition_halo(world):
    c, plan = _city_standin()
    part, arc = partition_route(c, plan.route, plan.block_edge, world, return_arc=True)
    rows = _stats(c, part, world)
    # equal block counts, ranks contiguous along the route
    n = [r["n_local"] for r in rows]
    assert max(n) - min(n) <= 1
    # a staircase route never comes back to itself: peers are r - 1 and r + 1 only
    for r, row in enumerate(rows):
        assert set(row["peers"]) <= {r - 1, r + 1} and row["peers"], (r, row["peers"])
    # the halo is one route cross-section per cut: the blocks whose arc length falls in one block-edge
    # slab of the route (median over the route; ~180 blocks), at most ~2 such slabs per cut
    slab = float(np.median(np.bincount(np.floor(arc / plan.block_edge).astype(np.int64))))
    for r, row in enumerate(rows):
        cuts = (r > 0) + (r < world - 1)
        assert row["n_ghost"] <= cuts * 1.25 * slab, (row, slab)
    frac_b = sum(r["n_b"] for r in rows) / len(c)
    assert frac_b <= 0.03 * (world - 1) / 7 + 0.005, frac_b
    # the lexicographic (x, y, z) cut of round 1 cuts the +y canyons lengthwise: many times more halo
    lex = _stats(c, _lex_part(c, world), world)
    assert sum(r["n_ghost"] for r in lex) >= 10 * sum(r["n_ghost"] for r in rows)
    print(f"world {world}: slab {slab}, ghosts {[r['n_ghost'] for r in rows]}, launch B {frac_b:.4f} "
          f"(lexicographic: ghosts {[r['n_ghost'] for r in lex]}, "
          f"launch B {sum(r['n_b'] for r in lex) / len(c):.4f})")
