"""Pins for oracle O3/O4 (grouping and LSH buckets, Alg. 1 L3-L6; §2.3)."""
import numpy as np
import pytest

import oracle as O
from oracle import brute


def _codes_with_dups(n, q, d, n_distinct, seed):
    rng = np.random.default_rng(seed)
    base = rng.integers(1, d + 1, size=(n_distinct, q)) * rng.choice([-1, 1], size=(n_distinct, q))
    return base[rng.integers(0, n_distinct, size=n)].astype(np.int16)


def _zeta(n, k, E, seed):
    rng = np.random.default_rng(seed)
    return np.sort(np.stack([rng.choice(E, k, replace=False) for _ in range(n)]), axis=1).astype(np.int32)


@pytest.mark.parametrize("n,k,E,q,nd,seed", [(200, 1, 4, 2, 30, 0), (150, 2, 5, 3, 12, 1), (64, 3, 3, 1, 5, 2)])
def test_buckets_match_pairwise_bruteforce(n, k, E, q, nd, seed):
    codes = _codes_with_dups(n, q, 8, nd, seed)
    zeta = _zeta(n, k, E, seed)
    b = O.bucketize(codes, zeta, E)
    ref = brute.buckets_pairwise([tuple(c) for c in codes.tolist()], zeta.tolist(), E)
    rows = [list(b.perm[b.row_start[r]:b.row_start[r + 1]]) for r in range(b.m)]
    off = 0
    for e in range(E):
        assert b.expert_rows[e] == len(ref[e])
        assert rows[off:off + len(ref[e])] == ref[e]
        off += len(ref[e])
    for r, mem in enumerate(rows):
        for c in mem:
            assert b.bucket[c // k, c % k] == r


def test_partition_invariants():
    n, k, E = 300, 2, 6
    codes = _codes_with_dups(n, 4, 16, 40, 3)
    zeta = _zeta(n, k, E, 3)
    b = O.bucketize(codes, zeta, E)
    assert b.row_start[-1] == n * k and np.all(np.diff(b.row_start) >= 1)
    assert np.array_equal(np.sort(b.perm), np.arange(n * k))
    assert b.expert_rows.sum() == b.m
    for r in range(b.m):
        mem = b.perm[b.row_start[r]:b.row_start[r + 1]]
        assert np.all(np.diff(mem) > 0)                       # ascending within a row
    # first-appearance order: within an expert, first members strictly increase
    firsts = b.perm[b.row_start[:-1]]
    off = 0
    for e in range(E):
        f = firsts[off:off + b.expert_rows[e]]
        assert np.all(np.diff(f) > 0)
        off += b.expert_rows[e]


def test_group_conservation_and_k_equals_E():
    n, E = 50, 4
    zeta = np.tile(np.arange(E, dtype=np.int32), (n, 1))
    groups = O.group_by_expert(zeta, E)
    assert sum(len(g) for g in groups) == n * E
    assert all(len(g) == n for g in groups)


def test_identical_tokens_one_bucket_per_group(golden):
    n, E = 8, 1
    codes = np.tile(np.array([[3, -1]], np.int16), (n, 1))
    b = O.bucketize(codes, np.zeros((n, 1), np.int32), E)
    assert b.m == 1 and b.m / n == golden["cluster_small"]["identical_8_tokens_ratio"]


def test_spec_cluster_example(golden):
    cs = golden["cluster_small"]
    X = np.array(cs["tokens"])
    codes, _ = O.cp_hash(X, np.eye(2)[None])
    b = O.bucketize(codes, np.zeros((3, 1), np.int32), 1)
    C = O.centroids(X, b, 1)
    assert b.m == cs["n_buckets"] and np.array_equal(C, np.array(cs["centroids"]))


def test_refinement_in_q_and_monotone_ratio():
    """Buckets at q+1 refine buckets at q (prefix of the same hash functions)."""
    rng = np.random.default_rng(7)
    d = 16
    U = rng.standard_normal((10, d))
    X = U[rng.integers(0, 10, 400)] + 0.3 * rng.standard_normal((400, d))
    zeta = _zeta(400, 1, 3, 7)
    R = np.stack([O.rotation_fp64(d, j, 5) for j in range(6)])
    codes, _ = O.cp_hash(X, R)
    prev = None
    ratios = []
    for q in range(1, 7):
        b = O.bucketize(codes[:, :q], zeta, 3)
        ratios.append(b.m / 400)
        if prev is not None:
            for r in range(b.m):
                mem = b.perm[b.row_start[r]:b.row_start[r + 1]]
                assert len(set(prev.bucket[mem, 0].tolist())) == 1     # subset of one q-bucket
        prev = b
    assert all(a <= c for a, c in zip(ratios, ratios[1:]))
