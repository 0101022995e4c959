"""Pins of the oracle's gate (O0, reading R29): SPEC's worked example, brute-force loops, softmax
invariants, k = E."""
import math

import numpy as np

import oracle as O


def test_gate_spec_identity_example(golden):
    g = golden["gate_topk_identity"]                    # W = I, x = (0.9, 0.1, 0.5), k = 2
    zeta, w, _ = O.gate_topk(np.array([g["x"]]), np.eye(3), g["k"])
    assert [int(e) + 1 for e in zeta[0]] == g["experts_1based"]
    assert abs(w[0].sum() - 1) < 1e-15 and w[0, 0] > w[0, 1]     # 0.9 beats 0.5


def test_gate_brute_force():
    rng = np.random.default_rng(0)
    X, Wg = rng.standard_normal((60, 8)), rng.standard_normal((6, 8))
    Wg[4] = Wg[1]                                       # duplicate expert rows: exact score ties
    zeta, g, _ = O.gate_topk(X, Wg, 3)
    for t in range(60):
        s = [math.fsum(X[t, i] * Wg[e, i] for i in range(8)) for e in range(6)]
        best = sorted(range(6), key=lambda e: (-s[e], e))[:3]   # ties -> smaller id
        assert list(zeta[t]) == sorted(best)
        ex = [math.exp(s[e] - max(s[b] for b in best)) for e in sorted(best)]
        assert np.allclose(g[t], [v / sum(ex) for v in ex], rtol=1e-12)


def test_gate_k_equals_E():
    rng = np.random.default_rng(1)
    zeta, g, margin = O.gate_topk(rng.standard_normal((10, 4)), rng.standard_normal((5, 4)), 5)
    assert np.array_equal(zeta, np.tile(np.arange(5), (10, 1))) and np.allclose(g.sum(1), 1)
    assert np.all(margin == 1)


def test_gate_margin_brute_force():
    """margin (R29) = (k-th largest score - (k+1)-th largest) / max |s|, for every k < E, by fsum
    loops and an explicit selection sort; a planted exact tie at the k/k+1 boundary gives 0."""
    rng = np.random.default_rng(2)
    X, Wg = rng.standard_normal((40, 6)), rng.standard_normal((7, 6))
    Wg[5] = Wg[2]                                       # experts 2 and 5 always tie
    for k in range(1, 7):
        _, _, margin = O.gate_topk(X, Wg, k)
        for t in range(40):
            s = [math.fsum(X[t, i] * Wg[e, i] for i in range(6)) for e in range(7)]
            rest, srt = list(s), []
            while rest:                                 # selection sort, descending
                j = max(range(len(rest)), key=lambda i: rest[i])
                srt.append(rest.pop(j))
            want = (srt[k - 1] - srt[k]) / max(abs(v) for v in s)
            assert abs(margin[t] - want) <= 1e-12 * max(1.0, abs(want))
            if s[2] == srt[k - 1] and s[5] == srt[k]:
                assert margin[t] == 0.0
