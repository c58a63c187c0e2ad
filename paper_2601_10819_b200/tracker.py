"""Association step of the reference tracker (tracker.py:105-142) on top of
the device cost kernel (C ABI ``msda_assoc_cost``).

The cost matrices are built on the GPU in f64, bit-identical to the
reference's numpy; the optimal assignment itself is the reference's
``scipy.optimize.linear_sum_assignment`` on the host (SURVEY §8(f) rank 4:
the Hungarian solve stays on CPU).  Inputs are plain arrays instead of the
reference's QueryBank / Detection objects.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import ops


@dataclass(frozen=True)
class TrackerParams:
    """The association fields of tracker.TrackerParams (tracker.py:35-43)."""

    gate_radius: float = 2.0
    alpha_emb: float = 1.0
    alpha_geo: float = 1.0


@dataclass(frozen=True)
class Assignment:
    """tracker.Assignment (tracker.py:84-89)."""

    matches: tuple  # (track_id, detection_index)
    unmatched_queries: tuple  # track ids
    unmatched_detections: tuple  # detection indices
    total_cost: float


def associate(track_ids, q_centers, q_memory, d_centers, d_embeddings, params: TrackerParams = TrackerParams(),
              device=None) -> Assignment:
    """Optimal gated assignment (tracker.py:105-142).

    Queries are ordered by track id (stable) before solving, as the reference
    does; matches of inadmissible pairs are dropped; ``total_cost`` sums the
    matched costs in solver order.
    """
    from scipy.optimize import linear_sum_assignment

    ids = np.asarray(track_ids, dtype=np.int64).reshape(-1)
    order = np.argsort(ids, kind="stable")
    n_q, n_d = len(ids), int(np.asarray(d_centers).reshape(-1, 3).shape[0])
    if n_q == 0 or n_d == 0:
        return Assignment((), tuple(int(i) for i in ids[order]), tuple(range(n_d)), 0.0)
    qc = np.asarray(q_centers, dtype=np.float64).reshape(-1, 3)[order]
    qm = np.asarray(q_memory, dtype=np.float64)[order]
    cost, solver, adm = ops.association_cost(qc, d_centers, qm, d_embeddings, params.gate_radius, params.alpha_emb,
                                             params.alpha_geo, device=device)
    cost, solver, adm = cost.cpu().numpy(), solver.cpu().numpy(), adm.cpu().numpy()
    rows, cols = linear_sum_assignment(solver)
    matches, mq, md, total = [], set(), set(), 0.0
    for r, c in zip(rows, cols):
        if not adm[r, c]:
            continue
        matches.append((int(ids[order][r]), int(c)))
        mq.add(int(r))
        md.add(int(c))
        total += float(cost[r, c])
    unmatched_q = tuple(int(ids[order][r]) for r in range(n_q) if r not in mq)
    unmatched_d = tuple(c for c in range(n_d) if c not in md)
    return Assignment(tuple(matches), unmatched_q, unmatched_d, total)
