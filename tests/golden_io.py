"""Loaders for the committed golden fixtures (tests/golden/)."""
from __future__ import annotations

import functools
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
ORDERS7 = ["identity", "random", "degree", "core", "split", "check", "neigh"]


@functools.lru_cache(maxsize=None)
def golden() -> dict:
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@functools.lru_cache(maxsize=None)
def sweep() -> dict:
    z = np.load(os.path.join(GOLDEN, "sweep.npz"))
    return {k: z[k] for k in z.files}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def csr_from_edges(n: int, edges) -> tuple[np.ndarray, np.ndarray]:
    """Reference Graph CSR (graph.cpp:13-56 layout) from an edge list, numpy only."""
    e = np.asarray(edges, dtype=np.int64).reshape(-1, 2)
    if e.shape[0] == 0:
        return np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32)
    both = np.concatenate([e, e[:, ::-1]])
    order = np.lexsort((both[:, 1], both[:, 0]))
    both = both[order]
    deg = np.bincount(both[:, 0], minlength=n)
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum(deg)
    return off, both[:, 1].astype(np.uint32)


def cases():
    return golden()["cases"]


def case_csr(case):
    return csr_from_edges(case["n"], case["edges"])


def sweep_graphs():
    """Yield (seed, n, offsets, adj, [(ordering_idx, ranks, result_row)])."""
    s = sweep()
    E, EO, N, R, RES = s["edges"], s["edge_off"], s["n"], s["ranks"], s["results"]
    for gi in range(N.shape[0]):
        n = int(N[gi])
        off, adj = csr_from_edges(n, E[EO[gi]:EO[gi + 1]])
        rows = []
        for k in range(7):
            idx = gi * 7 + k
            rows.append((int(RES[idx][1]), R[idx][:n].copy(), [int(x) for x in RES[idx]]))
        yield gi, n, off, adj, rows
