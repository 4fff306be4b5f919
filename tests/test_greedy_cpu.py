"""Greedy driver host logic (Algorithm 1 bookkeeping; SPEC greedy-driver) on CPU."""

import numpy as np
import pytest

from paper_2305_15661_b200.greedy import BasisInSpanError, gram_schmidt_append, seed_index


def test_seed_is_the_candidate_nearest_the_centroid():
    # SPEC example: 3 x 3 grid on [3, 9] x [0.02, 0.075] -> mu_1 = (6, 0.0475)
    g = np.array([[a, b] for a in (3.0, 6.0, 9.0) for b in (0.02, 0.0475, 0.075)])
    assert np.allclose(g[seed_index(g)], [6.0, 0.0475])
    assert seed_index([[1.0], [3.0]]) == 0  # tie -> first index


def test_gram_schmidt_append_matches_reference_semantics():
    rng = np.random.default_rng(0)
    B = np.zeros((50, 0))
    for _ in range(4):
        B = gram_schmidt_append(B, rng.standard_normal(50))
    assert np.allclose(B.T @ B, np.eye(4), atol=1e-14)
    with pytest.raises(BasisInSpanError):
        gram_schmidt_append(B, B @ rng.standard_normal(4))
    with pytest.raises(BasisInSpanError):
        gram_schmidt_append(B, np.zeros(50))
    try:
        from oracle import strom_ref

        S = strom_ref.load()
    except ImportError:
        return
    col = rng.standard_normal(50)
    assert np.array_equal(gram_schmidt_append(B, col), S["reduced"].gram_schmidt_append(B, col))
