"""Pins of the NEXT-1 W2 oracle (PAPER.md eq:w2_pixel, L74-95) against
closed forms, library optimal transport and invariants."""
import json
import os

import numpy as np
import pytest
from scipy.linalg import sqrtm
from scipy.stats import norm

from oracle import w2

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "w2_examples.json")


def test_w2_golden_examples():
    g = json.load(open(GOLDEN))
    for c in g["w2"]:
        assert abs(w2.w2_score(c["mu"], c["s2"]) - c["expect"]) < 1e-12, c["cite"]
    for c in g["cost"]:
        assert w2.estimate_cost(*c["args"]) == c["expect"], c["cite"]


def test_w2_pair_equals_gaussian_w2_by_sqrtm():
    """Library pin: for M = 2 the per-location term is the squared 2-Wasserstein
    distance between N(mu_i, diag s2_i) and N(mu_j, diag s2_j) by the general
    formula ||m1 - m2||^2 + tr(S1 + S2 - 2 (S2^1/2 S1 S2^1/2)^1/2) (scipy sqrtm)."""
    rng = np.random.default_rng(2)
    C = 5
    for _ in range(10):
        mu = rng.normal(size=(2, C, 1))
        s2 = np.exp(rng.normal(size=(2, C, 1)))
        S1, S2 = np.diag(s2[0, :, 0]), np.diag(s2[1, :, 0])
        r2 = np.real(sqrtm(S2))
        ref = np.sum((mu[0, :, 0] - mu[1, :, 0]) ** 2) + np.trace(S1 + S2 - 2 * np.real(sqrtm(r2 @ S1 @ r2)))
        assert abs(w2.w2_score(mu, s2) - ref) < 1e-10 * max(1.0, ref)


def test_w2_one_dimensional_optimal_transport_quadrature():
    """1-D optimal transport: W2^2 = int_0^1 (F1^-1(u) - F2^-1(u))^2 du (scipy
    normal quantiles, midpoint rule) for the S:L267 pair -> 10 within 1e-3."""
    u = (np.arange(200000) + 0.5) / 200000
    q = (norm.ppf(u, 0.0, 1.0) - norm.ppf(u, 3.0, 2.0)) ** 2
    assert abs(q.mean() - 10.0) < 1e-2
    assert abs(w2.w2_score([[[0.0]], [[3.0]]], [[[1.0]], [[4.0]]]) - q.mean()) < 1e-2


def test_w2_invariants():
    rng = np.random.default_rng(3)
    mu = rng.normal(size=(5, 4, 64))
    s2 = np.exp(rng.normal(size=(5, 4, 64)))
    v = w2.w2_score(mu, s2)
    assert v > 0
    # identical samples -> 0
    assert w2.w2_score(np.repeat(mu[:1], 5, 0), np.repeat(s2[:1], 5, 0)) == 0.0
    # homogeneous of degree 2 in (mu, sigma)
    assert abs(w2.w2_score(3 * mu, 9 * s2) - 9 * v) < 1e-10 * v
    # permutation of samples
    perm = rng.permutation(5)
    assert abs(w2.w2_score(mu[perm], s2[perm]) - v) < 1e-12 * v
    # variance term is a square: with equal means it equals sum (sigma_i - sigma_j)^2
    m0 = np.zeros_like(mu)
    s = np.sqrt(s2)
    ref = np.mean([np.sum((s[i] - s[j]) ** 2, axis=0) for i in range(5) for j in range(i + 1, 5)], axis=0).mean()
    assert abs(w2.w2_score(m0, s2) - ref) < 1e-10 * ref
    with pytest.raises(ValueError):
        w2.w2_score(mu[:1], s2[:1])
