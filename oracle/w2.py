"""NEXT-1 oracle: latent-space ensemble disagreement W2(Z) of PAPER.md
eq:w2_pixel (§3.3) -- TEST INFRASTRUCTURE ONLY (same rules as the
package docstring of oracle/).

For each latent location p and each of the C(M,2) sample pairs i < j:
    ||mu_{i,p} - mu_{j,p}||^2 + sum_c (s2_{i,p,c} + s2_{j,p,c} - 2 sqrt(s2_{i,p,c} s2_{j,p,c}))
averaged over the pairs and over the H_z W_z locations.  Reading:
each sample m supplies a diagonal-Gaussian latent (mean mu_m, per-channel
variance s2_m) per location, as a VAE posterior does; the LPIPS term of
eq:uncert_latent (L97-102) is out of scope, so u_lat = W2 (lambda * LPIPS
omitted).  Plain float64 loops, in the equation's order.  Pins:
tests/test_oracle_w2.py.
"""
from __future__ import annotations

import numpy as np


def w2_map(mu, s2):
    """Per-location divergence [H*W] of one view; mu, s2: [M][C][H*W] (any float)."""
    mu = np.asarray(mu, dtype=np.float64)
    s2 = np.asarray(s2, dtype=np.float64)
    M, C, P = mu.shape
    if M < 2:
        raise ValueError("W2 needs M >= 2 samples")
    if np.any(s2 < 0):
        raise ValueError("negative variance")
    npairs = M * (M - 1) // 2
    out = np.zeros(P, dtype=np.float64)
    for i in range(M):
        for j in range(i + 1, M):
            term = np.zeros(P, dtype=np.float64)
            for c in range(C):
                d = mu[i, c] - mu[j, c]
                term += d * d
            for c in range(C):
                term += s2[i, c] + s2[j, c] - 2.0 * np.sqrt(s2[i, c] * s2[j, c])
            out += term
    return out / npairs


def w2_score(mu, s2):
    """eq:w2_pixel: the spatial mean (1 / (H_z W_z)) sum_p of w2_map."""
    return float(w2_map(mu, s2).mean())


def w2_scores(mu, s2):
    """Per-view scores for [V][M][C][H*W] arrays."""
    return np.array([w2_score(mu[v], s2[v]) for v in range(len(mu))], dtype=np.float64)


def estimate_cost(n_theta, M, C, Hz, Wz):
    """PAPER.md L135 / L176: O(N_theta M C H_z W_z) scalar operations."""
    return n_theta * M * C * Hz * Wz
