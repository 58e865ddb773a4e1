"""Oracle restatement of the RALP planner arithmetic (test infrastructure only).

Works on plain per-layer tables (kind strings, param counts, per-sample output
elements, per-sample forward flops) so it shares no code with the product's
planner.  Each function cites the reference lines it restates.
"""
from __future__ import annotations

import numpy as np

HEAVY = ("conv", "block")  # layers.py:42-43 COMPUTE_DEMAND_KINDS


def skewness_index_weighted(param_bytes):
    """profiler.py:76-85: third standardised moment of the layer index, weights P_i/sum P."""
    p = np.asarray(param_bytes, dtype=np.float64)
    w = p / float(p.sum())
    idx = np.arange(1, p.size + 1, dtype=np.float64)
    mu = float(np.dot(w, idx))
    d = idx - mu
    m2 = float(np.dot(w, d ** 2))
    m3 = float(np.dot(w, d ** 3))
    return 0.0 if m2 == 0.0 else m3 / m2 ** 1.5


def skewness_literal(param_bytes):
    """profiler.py:71-74: population skewness of the values."""
    p = np.asarray(param_bytes, dtype=np.float64)
    d = p - p.mean()
    m2 = float(np.mean(d ** 2))
    return 0.0 if m2 == 0.0 else float(np.mean(d ** 3)) / m2 ** 1.5


def exhaustive_split(param_bytes, output_bytes, kinds):
    """Brute force over all cut points (cf. pkg/tests/test_profiler.py:127-140 and
    profiler.py:101-134): candidates i in 1..N whose boundary is not conv|block -> conv|block;
    cost = O_i + sum_{j<=i} P_j; smallest cost, ties to the smallest i; a winning i == N
    (N > 1) means no split."""
    n = len(param_bytes)
    cands = []
    for i in range(1, n + 1):
        if i < n and kinds[i - 1] in HEAVY and kinds[i] in HEAVY:
            continue
        cands.append((output_bytes[i - 1] + sum(param_bytes[:i]), i))
    cost, i = min(cands)
    if i == n and n > 1:
        return None
    return i, cost


def plan(table, batch, elem_bytes=4, threshold=-0.5):
    """profile() (profiler.py:187-227) on a layer table -> (skew, eligible, split, cost)."""
    pb = [r["params"] * elem_bytes for r in table]
    ob = [r["out"] * batch * elem_bytes for r in table]
    kinds = [r["kind"] for r in table]
    if len(table) < 2 or sum(pb) == 0:
        return 0.0, False, None, None
    s = skewness_index_weighted(pb)
    if not s < threshold:
        return s, False, None, None
    sp = exhaustive_split(pb, ob, kinds)
    if sp is None:
        return s, False, None, None
    return s, True, sp[0], sp[1]


def volume_ralp(table, batch, split, workers, elem_bytes=4):
    """costmodel.py:136-153: W * (2*O_split + 2*P_{<=split})."""
    o = table[split - 1]["out"] * batch * elem_bytes
    p = sum(r["params"] for r in table[:split]) * elem_bytes
    return workers * 2 * o + workers * 2 * p, workers * 2 * p, workers * 2 * o


def volume_baseline(table, workers, elem_bytes=4):
    """costmodel.py:110-120: 2*S*W."""
    return 2 * sum(r["params"] for r in table) * elem_bytes * workers


def volume_ring(table, workers, elem_bytes=4):
    """costmodel.py:123-133: 2*S*(W-1)."""
    return 2 * sum(r["params"] for r in table) * elem_bytes * (workers - 1)


def compute_load(table, batch, split, workers):
    """costmodel.py:165-186: worker 3*fwd(front)*b, PS 3*fwd(back)*b*W."""
    split = len(table) if split is None else split
    front = sum(r["flops"] for r in table[:split])
    back = sum(r["flops"] for r in table[split:])
    return 3 * front * batch, 3 * back * batch * workers


def conv_counts(k, cin, cout, ho, wo):
    """layers.py:87-103."""
    return k * k * cin * cout + cout, 2 * k * k * cin * cout * ho * wo


def fc_counts(i, u):
    """layers.py:117-123."""
    return i * u + u, 2 * i * u
