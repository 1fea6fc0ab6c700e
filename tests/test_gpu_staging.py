"""Host staging through the C ABI (gsr_upload / gsr_download, the end-to-end
path bench.py times): byte-exact round trips from pinned and pageable host
memory, the scoring pass on an uploaded field equal to the pass on the same
field copied by torch, and the documented EINVAL cases."""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2602_15355_b200 import Context
    return Context(0)


@pytest.mark.parametrize("pinned", [True, False])
def test_round_trip_is_byte_exact(ctx, pinned):
    from paper_2602_15355_b200 import gsr
    rng = np.random.default_rng(7)
    src = torch.from_numpy(rng.integers(0, 2**32, size=(3, 1001, 4), dtype=np.uint32).view(np.float32))
    if pinned:
        src = src.pin_memory()
    dev = torch.empty(src.shape, dtype=torch.float32, device="cuda")
    gsr.gsr_upload(ctx, dev, src)
    back = torch.empty_like(src)
    if pinned:
        back = back.pin_memory()
    gsr.gsr_download(ctx, back, dev)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(back.numpy().view(np.uint32), src.numpy().view(np.uint32))
    # numpy host buffers take the same path
    arr = np.zeros((3, 1001, 4), dtype=np.float32)
    gsr.gsr_download(ctx, arr, dev)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(arr.view(np.uint32), src.numpy().view(np.uint32))


def test_scores_of_an_uploaded_field(ctx):
    from paper_2602_15355_b200 import Gaussians, gsr
    from paper_2602_15355_b200.pipeline import ViewScorer
    sc = synth.make_scene(1)
    host = torch.from_numpy(sc.field.planes).pin_memory()
    up = torch.empty(host.shape, dtype=torch.float32, device="cuda")
    gsr.gsr_upload(ctx, up, host)
    ref = torch.from_numpy(sc.field.planes).cuda()
    a = ViewScorer(Gaussians(up, sc.field.sh_degree), batch_views=8).score_views(sc.cameras)
    b = ViewScorer(Gaussians(ref, sc.field.sh_degree), batch_views=8).score_views(sc.cameras)
    out = np.zeros(len(sc.cameras), dtype=np.float32)
    gsr.gsr_download(ctx, out, a)
    torch.cuda.current_stream().synchronize()
    assert np.array_equal(out.view(np.uint32), b.cpu().numpy().view(np.uint32))


def test_invalid_arguments(ctx):
    from paper_2602_15355_b200 import gsr
    L = gsr.lib
    assert L.gsr_upload(ctx.handle, None, None, 0, None) == gsr.GSR_OK  # zero bytes: no-op
    assert L.gsr_upload(ctx.handle, None, None, 16, None) == gsr.GSR_EINVAL
    assert L.gsr_download(ctx.handle, None, None, -1, None) == gsr.GSR_EINVAL
    assert L.gsr_upload(None, None, None, 0, None) == gsr.GSR_EINVAL
    with pytest.raises(ValueError):
        gsr.gsr_upload(ctx, torch.empty(4, device="cuda"), np.zeros(5, np.float32))
