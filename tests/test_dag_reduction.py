"""The DAG walk's implied-edge rule (csrc/batching.cu pl_walk_warp_kernel), on
the CPU against the reference's own batch_moves.

The walk drops the rule-1 edge (s_b, i) at source(s_b) on i's route when the
owner s_a of the previous or next source on i's route has a route through
source(s_b): then (s_b, s_a) and (s_a, i) are edges of the full occupancy DAG
(virtual_line.cpp:241-268) and (s_b, i) is implied.  Batches depend only on
reachability (batching.cpp:28-84: a path is ready once all its blockers are
done), so batch_moves must give the same schedule on the reduced edge list, in
both presets.  This restates the rule in numpy on solver outputs (the C
oracle's solves, equal to the reference's) and runs the compiled reference's
batch_moves on both edge lists; the GPU parity tests check the kernel itself.
"""
import numpy as np
import pytest

from conftest import ORACLE_LIB, REF_LIB, _load  # noqa: F401
from paper_2504_06182_b200.inputs import sample_grids


def _routes(src, dst, H):
    """Every path's route vertices (horizontal first, virtual_line.cpp:150-173)."""
    xs, ys, xt, yt = src // H, src % H, dst // H, dst % H
    ln = np.abs(xt - xs) + np.abs(yt - ys)
    pid = np.repeat(np.arange(len(src)), ln + 1)
    start = np.repeat(np.concatenate([[0], np.cumsum(ln + 1)[:-1]]), ln + 1)
    k = np.arange(len(pid)) - start
    dx = np.abs(xt - xs)[pid]
    x = np.where(k <= dx, xs[pid] + np.sign(xt - xs)[pid] * k, xt[pid])
    y = np.where(k <= dx, ys[pid], ys[pid] + np.sign(yt - ys)[pid] * (k - dx))
    return pid, k, x, y, ln, (xs, ys, xt, yt)


def _implied_rule1(src, dst, W, H):
    """(s_b, i) pairs the walk drops."""
    pid, k, x, y, ln, (xs, ys, xt, yt) = _routes(src, dst, H)
    owner = np.full(W * H, -1, np.int64)
    owner[src] = np.arange(len(src))
    own = owner[x * H + y]
    idx = np.nonzero((own >= 0) & (own != pid) & (k >= 1))[0]

    def on_route(p, qx, qy):
        h = (qy == ys[p]) & (qx >= np.minimum(xs[p], xt[p])) & (qx <= np.maximum(xs[p], xt[p]))
        v = (qx == xt[p]) & (qy >= np.minimum(ys[p], yt[p])) & (qy <= np.maximum(ys[p], yt[p]))
        return h | v

    red = np.zeros(len(idx), bool)
    for d in (-1, 1):  # the previous and the next source on the route
        n = np.arange(len(idx)) + d
        ok = (n >= 0) & (n < len(idx))
        n = np.where(ok, n, 0)
        ok &= pid[idx[n]] == pid[idx]
        red |= ok & on_route(own[idx[n]], x[idx], y[idx])
    return set(zip(own[idx][red].tolist(), pid[idx][red].tolist())), pid, x, y, ln


@pytest.mark.parametrize("solver,W,H,hp,atoms,seed", [
    ("redrec", 96, 96, 57, 5530, 0x9600),
    ("bird", 96, 96, 57, 5530, 0x9601),
    ("bird", 64, 64, 40, 2662, 0x64000007),
])
def test_implied_edges_keep_the_schedule(solver, W, H, hp, atoms, seed):
    oracle = _load(ORACLE_LIB, "oracle")
    ref = _load(REF_LIB, "ref")
    occ = sample_grids(seed, 1, W, H, atoms)
    g = oracle.grid_solve(solver, occ, W, H, hp)
    src, dst = g.path_src.astype(np.int64), g.path_dst.astype(np.int64)
    dag = ref.occupancy_dag(W, H, src.astype(np.int32), dst.astype(np.int32))
    drop, pid, x, y, ln = _implied_rule1(src, dst, W, H)
    keep = np.array([(int(a), int(b)) not in drop for a, b in dag], bool)
    reduced = dag[keep]
    assert len(reduced) < 0.8 * len(dag)  # the rule removes most rule-1 edges
    v = x * H + y
    starts = np.concatenate([[0], np.cumsum(ln + 1)[:-1]])
    routes = [v[starts[p]:starts[p] + ln[p] + 1] for p in range(len(src))]
    for preset in (0, 1):
        try:
            full = ref.batch_moves(W, H, occ, routes, dag, preset)
        except Exception as e:  # noqa: BLE001  (a no-progress instance: both lists must throw)
            with pytest.raises(type(e)):
                ref.batch_moves(W, H, occ, routes, reduced, preset)
            continue
        red = ref.batch_moves(W, H, occ, routes, reduced, preset)
        assert red[1] == full[1]
        assert np.array_equal(red[0], full[0])
