"""TEST INFRASTRUCTURE, not product code: plain-Python reference of the trajectory post-processing
(PAPER.md:419 slicing; PAPER.md:470-479 filtering and type smoothing), written from the paper and the
definitions in include/ftk_cp.h, sharing nothing with the CUDA path.  Only tests/ may import it.

Input: the labelled records of a track (oracle.CP_DTYPE) and the grid.  The adjacency is found by
brute force over EVERY cell of the mesh (anchor x axis permutation), not by the closed
form the kernels use: a cell holding two punctured faces links them."""
import itertools

import numpy as np


def _types(d):
    seqs = [s for s in itertools.product(range(1, 1 << d), repeat=d - 1)
            if all(s[i] != s[i + 1] and (s[i] & ~s[i + 1]) == 0 for i in range(d - 2))]
    return {s: i for i, s in enumerate(sorted(seqs))}


def adjacency(rec, dims):
    """dims = (nx, ny[, nz], nt); returns {record index: [partner record indices]} (0..2 each)."""
    d = len(dims)
    tid = _types(d)
    T = len(tid)
    index = {int(f): i for i, f in enumerate(rec["face_id"])}
    strides = [1]
    for a in range(d - 1):
        strides.append(strides[-1] * dims[a])
    nbr = {i: [] for i in range(len(rec))}
    for anchor in itertools.product(*[range(n - 1) for n in dims]):
        for perm in itertools.permutations(range(d)):
            chain = [tuple(anchor)]
            for a in perm:
                v = list(chain[-1])
                v[a] += 1
                chain.append(tuple(v))
            hit = []
            for k in range(d + 1):
                fv = chain[:k] + chain[k + 1:]
                a0 = fv[0]
                seq = tuple(sum((w[a] - a0[a]) << a for a in range(d)) for w in fv[1:])
                fid = sum(a0[a] * strides[a] for a in range(d)) * T + tid[seq]
                if fid in index:
                    hit.append(index[fid])
            assert len(hit) in (0, 2), hit
            if len(hit) == 2:
                nbr[hit[0]].append(hit[1])
                nbr[hit[1]].append(hit[0])
    return nbr


def slice_at(rec, nbr, t0):
    """records at t == t0 plus the straddling segment points (include/ftk_cp.h ftk_post_slice)"""
    out = []
    for i, r in enumerate(rec):
        if r["t"] == t0:
            out.append(r.copy())
        for j in nbr[i]:
            if j <= i:
                continue
            lo, hi = (r, rec[j]) if r["t"] <= rec[j]["t"] else (rec[j], r)
            if not (lo["t"] < t0 < hi["t"]):
                continue
            s = (t0 - float(lo["t"])) / (float(hi["t"]) - float(lo["t"]))
            near = lo if (t0 - float(lo["t"])) <= (float(hi["t"]) - t0) else hi
            p = near.copy()
            p["x"] = float(lo["x"]) + s * (float(hi["x"]) - float(lo["x"]))
            p["y"] = float(lo["y"]) + s * (float(hi["y"]) - float(lo["y"]))
            p["z"] = float(lo["z"]) + s * (float(hi["z"]) - float(lo["z"]))
            p["t"] = t0
            p["flags"] = 0
            out.append(p)
    return np.array(out, dtype=rec.dtype) if out else np.zeros(0, rec.dtype)


def filter_trajectories(rec, nbr, min_duration, drop_loops=False):
    comp = {}
    for i, r in enumerate(rec):
        c = comp.setdefault(int(r["label"]), [np.inf, -np.inf, 0])
        c[0] = min(c[0], float(r["t"]))
        c[1] = max(c[1], float(r["t"]))
        c[2] += len(nbr[i]) < 2
    keep = [i for i, r in enumerate(rec)
            if comp[int(r["label"])][1] - comp[int(r["label"])][0] >= min_duration
            and not (drop_loops and comp[int(r["label"])][2] == 0)]
    return rec[keep]


def smooth_types(rec, nbr, half_window):
    out = rec.copy()
    for i in range(len(rec)):
        seen, types = [0, 0], []
        for side in range(2):
            if side >= len(nbr[i]):
                continue
            prev, cur = i, nbr[i][side]
            for _ in range(half_window):
                if cur == i:
                    break
                types.append(int(rec[cur]["type"]))
                seen[side] += 1
                nxt = [j for j in nbr[cur] if j != prev]
                if not nxt:
                    break
                prev, cur = cur, nxt[0]
        if seen[0] and seen[1] and len(set(types)) == 1 and types[0] != int(rec[i]["type"]):
            out[i]["type"] = types[0]
    return out


def simplify_types(rec, nbr, tau):
    """Simplification in time (R23): a trajectory is cut at its folds -- records whose
    two partners both lie strictly later, or both strictly earlier, in t (a pair is born or annihilates
    there) -- into segments running from one fold to the next (both folds included).  A segment bounded
    by folds on both ends whose time extent (max t - min t over its records) is below tau, and whose two
    outer records (the partners of its folds outside it) exist and share one type T, is a short-lived
    excursion (the saddle of Fig. 9(b)): its records take T.  A fold lies in two segments; it takes T
    when the qualifying ones agree.  Decided on the unmodified types, then applied."""
    n = len(rec)
    t = [float(r["t"]) for r in rec]
    ty = [int(r["type"]) for r in rec]

    def is_fold(i):
        if len(nbr[i]) != 2:
            return False
        a, b = (t[j] - t[i] for j in nbr[i])
        return (a > 0 and b > 0) or (a < 0 and b < 0)

    # order every trajectory as a path (from an end) or a loop (from its smallest index)
    seen = [False] * n
    paths = []
    for s in list(range(n)):
        if seen[s] or len(nbr[s]) == 2:
            continue
        paths.append((_walk(nbr, s, seen), False))
    for s in range(n):
        if not seen[s]:
            paths.append((_walk(nbr, s, seen), True))
    votes = {}  # record -> set of T from the qualifying segments holding it
    for path, loop in paths:
        m = len(path)
        folds = [p for p in range(m) if is_fold(path[p])]
        if len(folds) < 2:
            continue
        pairs = list(zip(folds, folds[1:]))
        if loop:
            pairs.append((folds[-1], folds[0] + m))  # the segment through the path's start
        for fa, fb in pairs:
            if not loop and (fa == 0 or fb == m - 1):
                continue  # a fold needs a partner outside the segment (cannot happen: folds are interior)
            seg = [path[p % m] for p in range(fa, fb + 1)]
            ts = [t[k] for k in seg]
            if not (max(ts) - min(ts) < tau):
                continue
            oa, ob = path[(fa - 1) % m], path[(fb + 1) % m]
            if ty[oa] != ty[ob]:
                continue
            for k in seg:
                votes.setdefault(k, set()).add(ty[oa])
    out = rec.copy()
    for k, v in votes.items():
        if len(v) == 1:
            out[k]["type"] = next(iter(v))
    return out


def _walk(nbr, s, seen):
    path, prev, cur = [], -1, s
    while cur >= 0 and not seen[cur]:
        seen[cur] = True
        path.append(cur)
        nxt = [j for j in nbr[cur] if j != prev]
        prev, cur = cur, (nxt[0] if nxt else -1)
    return path
