"""Pinned host staging (amz_host_alloc / amz_host_free) used by the trajectory feed."""
import gc

import pytest

torch = pytest.importorskip("torch")
import paper_2311_12716_b200 as amz  # noqa: E402

pytestmark = pytest.mark.gpu


def test_pinned_empty_roundtrip():
    h = amz.pinned_empty((256, 4096), torch.float64)
    assert h.shape == (256, 4096) and h.dtype == torch.float64 and h.is_pinned()
    h.copy_(torch.arange(256 * 4096, dtype=torch.float64).reshape(256, 4096))
    d = torch.empty_like(h, device="cuda")
    d.copy_(h, non_blocking=True)
    back = amz.pinned_empty((256, 4096), torch.float64)
    back.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    assert torch.equal(back, h)


def test_pinned_views_keep_the_block_alive():
    h = amz.pinned_empty(1 << 20, torch.uint8)
    v = h[1000:2000]
    del h
    gc.collect()
    v.fill_(7)  # still mapped
    d = v.cuda()
    assert int(d.sum()) == 7 * 1000
    del v
    gc.collect()


def test_pinned_empty_zero_size():
    h = amz.pinned_empty((0, 5), torch.float32)
    assert h.numel() == 0
