"""Validator test cases: valid pipeline outputs plus seeded corruptions of them.

Each case is the keyword arguments of ReconLib.validate for ONE instance.  The
corruptions target every recon_verdict category: path endpoints (bounds,
shared sources/targets, one-move violations), stats claims, path order
(collisions, dag order), explicit dags with back edges and cycles, and batch
schedules (renumbered, merged, split, out-of-range and reordered batches).
"""
import numpy as np

from paper_2504_06182_b200.abi import DAG_EXPLICIT, DAG_NONE, DAG_OCCUPANCY
from paper_2504_06182_b200.inputs import sample_grids


def pipeline_instances(lib, solver, W, H, hp, k, seed, count, preset):
    """Solver + batching outputs for `count` instances, from `lib`."""
    occ = sample_grids(seed, count, W, H, k)
    ms = W * H * (W + H)
    out = lib.pipeline_batch(solver, occ, count, W, H, hp, preset, ms)
    wpc = (H + 63) // 64
    stride = W * hp
    res = []
    for i in range(count):
        if out["status"][i] != 0:
            continue
        P = int(out["path_count"][i])
        D = int(out["total_displacement"][i])
        res.append(dict(
            occ=occ[i * W * wpc:(i + 1) * W * wpc].copy(), width=W, height=H, h_prime=hp,
            path_src=out["path_src"][i * stride:i * stride + P].copy(),
            path_dst=out["path_dst"][i * stride:i * stride + P].copy(),
            total_displacement=np.array([D], np.int64), displaced=np.array([P], np.int32),
            move_batch=out["move_batch"][i * ms:i * ms + D].copy(),
            batch_count=np.array([out["batch_count"][i]], np.int32), preset=preset))
    return res


def _lens(c):
    H = c["height"]
    s, t = c["path_src"], c["path_dst"]
    return np.abs(s // H - t // H) + np.abs(s % H - t % H)


def corruptions(base, rng, n):
    """`n` seeded corrupted variants of one valid instance `base`."""
    out = []
    P = len(base["path_src"])
    V = base["width"] * base["height"]
    for _ in range(n):
        c = {k: (v.copy() if isinstance(v, np.ndarray) else v) for k, v in base.items()}
        kind = int(rng.integers(0, 14))
        i, j = (int(x) for x in rng.integers(0, P, 2))
        if kind == 0:  # stats claims
            c["total_displacement"] = c["total_displacement"] + int(rng.integers(-2, 3) or 1)
        elif kind == 1:
            c["displaced"] = c["displaced"] + 1
        elif kind == 2:  # shared source
            c["path_src"][i] = c["path_src"][j]
        elif kind == 3:  # shared target
            c["path_dst"][i] = c["path_dst"][j]
        elif kind == 4:  # leaves the grid
            c["path_src"][i] = V + int(rng.integers(0, 5))
        elif kind == 5:  # swap two paths (order / collisions)
            for key in ("path_src", "path_dst"):
                c[key][[i, j]] = c[key][[j, i]]
        elif kind == 6:  # reverse a window of paths
            a, b = sorted((i, j))
            for key in ("path_src", "path_dst"):
                c[key][a:b + 1] = c[key][a:b + 1][::-1].copy()
        elif kind == 7:  # a path starts where an earlier path ends
            a, b = sorted((i, j))
            if a != b:
                c["path_src"][b] = c["path_dst"][a]
        elif kind == 8:  # random endpoint
            key = "path_src" if rng.integers(0, 2) else "path_dst"
            c[key][i] = int(rng.integers(0, V))
        elif kind == 9:  # batch id shifted
            D = len(c["move_batch"])
            m = int(rng.integers(0, D))
            c["move_batch"][m] += int(rng.choice([-1, 1]))
        elif kind == 10:  # batch id out of range / batch count changed
            if rng.integers(0, 2):
                m = int(rng.integers(0, len(c["move_batch"])))
                c["move_batch"][m] = c["batch_count"][0]
            else:
                c["batch_count"] = c["batch_count"] + int(rng.integers(1, 3))
        elif kind == 11:  # two batches exchanged
            nb = int(c["batch_count"][0])
            x, y = (int(v) for v in rng.integers(0, nb, 2))
            mb = c["move_batch"]
            mx, my = mb == x, mb == y
            mb[mx], mb[my] = y, x
        elif kind == 12:  # merge a batch into the next (later batches shift down)
            nb = int(c["batch_count"][0])
            if nb > 1:
                x = int(rng.integers(0, nb - 1))
                mb = c["move_batch"]
                mb[mb > x] -= 1
                c["batch_count"] = c["batch_count"] - 1
        elif kind == 13:  # a path's moves reversed in batch order
            lens = _lens(c)
            offs = np.concatenate([[0], np.cumsum(lens)])
            if lens[i] > 1:
                seg = c["move_batch"][offs[i]:offs[i + 1]]
                c["move_batch"][offs[i]:offs[i + 1]] = seg[::-1].copy()
        out.append((kind, c))
    return out


def with_dag(c, mode, rng=None, back_edges=0):
    """Attach a dag: occupancy (derived), none, or explicit edges from the
    occupancy dag of a reference library plus `back_edges` reversed ones."""
    c = dict(c)
    c["dag_mode"] = mode
    if mode == DAG_EXPLICIT:
        a, b = c.pop("_edges")
        a, b = list(a), list(b)
        for _ in range(back_edges):
            e = int(rng.integers(0, len(a))) if a else None
            if e is None:
                break
            a.append(b[e])
            b.append(a[e])
        c["dag_a"] = np.array(a, np.int32)
        c["dag_b"] = np.array(b, np.int32)
        c["dag_offset"] = np.array([0, len(a)], np.int64)
    else:
        c.pop("_edges", None)
    return c


def run(lib, c):
    """Validate one case with `lib`; returns the verdict bits."""
    P = len(c["path_src"])
    mb = c.get("move_batch")
    v = lib.validate(
        c["occ"], 1, c["width"], c["height"], c["h_prime"], c["path_src"], c["path_dst"], max(P, 1),
        np.array([P], np.int32), total_displacement=c.get("total_displacement"), displaced=c.get("displaced"),
        dag_mode=c.get("dag_mode", DAG_NONE), dag_a=c.get("dag_a"), dag_b=c.get("dag_b"),
        dag_offset=c.get("dag_offset"), move_batch=mb, move_stride=0 if mb is None else max(len(mb), 1),
        batch_count=c.get("batch_count"), preset=c.get("preset", 0))
    return int(v[0])


def occupancy_edges(lib, c):
    """The occupancy dag of the case's paths, from `lib` (recon_occupancy_dag)."""
    e = lib.occupancy_dag(c["width"], c["height"], c["path_src"], c["path_dst"])
    return e[:, 0], e[:, 1]


__all__ = ["pipeline_instances", "corruptions", "with_dag", "run", "occupancy_edges", "DAG_OCCUPANCY",
           "DAG_EXPLICIT", "DAG_NONE"]
