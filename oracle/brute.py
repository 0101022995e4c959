"""Pure-Python brute-force versions of the oracle's steps, for tiny inputs only.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  These use explicit loops and math.fsum
(correctly rounded sums) and share nothing with lshmoe_oracle.py except the problem statement,
so they pin the NumPy oracle against an independent evaluation.
"""
from __future__ import annotations

import math
from typing import List, Sequence, Tuple


def cp_hash_one(R: Sequence[Sequence[float]], x: Sequence[float]) -> int:
    """Eq. 3 for one token and one hash, by explicit loops.

    y_i = fsum_k R[i][k] x[k]; scan i ascending keeping the strictly larger |y_i| (so ties go
    to the smallest index); code = +(i*+1) unless y_i* < 0."""
    best_i, best_a, best_y = 0, -1.0, 0.0
    for i in range(len(R)):
        y = math.fsum(R[i][k] * x[k] for k in range(len(x)))
        if abs(y) > best_a:
            best_i, best_a, best_y = i, abs(y), y
    return -(best_i + 1) if best_y < 0 else best_i + 1


def sp_hash_one(normals: Sequence[Sequence[float]], x: Sequence[float]) -> int:
    """SPEC's sign-bit SP hash for one token and one hash function, by explicit
    loops: bit i = 1 iff fsum_k normals[i][k] x[k] >= 0; code = sum_i bit_i 2^i."""
    code = 0
    for i, nrm in enumerate(normals):
        if math.fsum(nrm[k] * x[k] for k in range(len(x))) >= 0:
            code |= 1 << i
    return code


def buckets_pairwise(keys: Sequence[Tuple[int, ...]], experts: Sequence[Sequence[int]], E: int):
    """O(n^2) grouping of routed copies (t, s) by (expert, key) equality (SPEC S:L150's
    brute-force oracle).  Returns {expert: [sorted list of member lists]} with buckets ordered
    by their smallest member (first appearance) and members ascending."""
    n = len(keys)
    k = len(experts[0]) if n else 0
    copies = [(t * k + s, experts[t][s]) for t in range(n) for s in range(k)]
    out = {}
    for e in range(E):
        ids = [c for c, ee in copies if ee == e]
        seen = [False] * len(ids)
        buckets: List[List[int]] = []
        for a in range(len(ids)):
            if seen[a]:
                continue
            mem = [ids[a]]
            seen[a] = True
            for b in range(a + 1, len(ids)):
                if not seen[b] and keys[ids[b] // k] == keys[ids[a] // k]:
                    mem.append(ids[b])
                    seen[b] = True
            buckets.append(mem)
        out[e] = buckets
    return out


def mean_fsum(rows: Sequence[Sequence[float]]) -> List[float]:
    """Centroid of a list of rows with correctly rounded sums."""
    n = len(rows)
    return [math.fsum(r[j] for r in rows) / n for j in range(len(rows[0]))]


def ffn_loops(x, W1, b1, W2, b2):
    """E(x) = W2 relu(W1 x + b1) + b2 with explicit loops and fsum."""
    h = [max(0.0, math.fsum(W1[i][j] * x[j] for j in range(len(x))) + b1[i]) for i in range(len(W1))]
    return [math.fsum(W2[o][i] * h[i] for i in range(len(h))) + b2[o] for o in range(len(W2))]


def fwht_loops(v: Sequence[float]) -> List[float]:
    """Unnormalised fast Walsh-Hadamard transform by the textbook in-place butterfly loops
    (len(v) a power of two): for h = 1, 2, 4, ...: (a, b) <- (a + b, a - b) on pairs h apart.
    Equals H v with the Sylvester H (an independent route to the dense matrix of O2*)."""
    a = list(v)
    h = 1
    while h < len(a):
        for i in range(0, len(a), 2 * h):
            for j in range(i, i + h):
                a[j], a[j + h] = a[j] + a[j + h], a[j] - a[j + h]
        h *= 2
    return a
