"""NEXT-1 parity: gsr_w2_scores (CUDA, through the C ABI) vs oracle/w2.py.
Scores and per-location maps within 1e-5 relative (float terms, double
accumulation on the GPU; float64 oracle)."""
import numpy as np
import pytest
import torch

import synth
from oracle import w2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


def _run(ctx, mu, s2, want_map=True):
    from paper_2602_15355_b200 import gsr
    m = torch.from_numpy(mu).cuda()
    s = torch.from_numpy(s2).cuda()
    sc = torch.empty(mu.shape[0], device="cuda")
    mp = torch.empty((mu.shape[0], mu.shape[3]), device="cuda") if want_map else None
    gsr.gsr_w2_scores(ctx, m, s, sc, mp)
    torch.cuda.synchronize()
    return sc.cpu().numpy(), (mp.cpu().numpy() if want_map else None)


@pytest.mark.parametrize("M,C,HW", [(2, 1, 1), (5, 4, 4096), (3, 8, 4113), (6, 2, 17)])
def test_w2_small_shapes(ctx, M, C, HW):
    rng = np.random.default_rng(M * 100 + C)
    mu = rng.normal(size=(7, M, C, HW)).astype(np.float32)
    s2 = np.exp(rng.normal(-1, 0.5, size=(7, M, C, HW))).astype(np.float32)
    sc, mp = _run(ctx, mu, s2)
    ref = w2.w2_scores(mu, s2)
    np.testing.assert_allclose(sc, ref, rtol=1e-5)
    for v in range(7):
        np.testing.assert_allclose(mp[v], w2.w2_map(mu[v], s2[v]), rtol=2e-5, atol=1e-6)


def test_w2_golden_and_full_size(ctx):
    """S:L267 example (10) and the paper's workload (N = 1000 views, M = 5,
    C = 4, 64 x 64 latents, P:L135 / L181) against the oracle on every view;
    same NBV."""
    sc, _ = _run(ctx, np.float32([[[[0.0]], [[3.0]]]]), np.float32([[[[1.0]], [[4.0]]]]))
    assert abs(sc[0] - 10.0) < 1e-6
    mu, s2 = synth.gen_latent_ensembles(1000, 5, 4, 64, 64, seed=0)
    sc, _ = _run(ctx, mu, s2, want_map=False)
    ref = w2.w2_scores(mu, s2)
    np.testing.assert_allclose(sc, ref, rtol=1e-5)
    assert int(np.argmax(sc)) == int(np.argmax(ref))
