"""Pinned, multi-threaded host->device staging (device.to_device) is an exact copy."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape,src,dst", [((3_000_001, 4), np.int64, np.int32),
                                           ((1_234_567, 3), np.float64, np.float64),
                                           ((17,), np.float64, np.float64)])
def test_to_device_exact(cuda, shape, src, dst):
    from paper_1811_07717_b200.device import to_device

    rng = np.random.default_rng(0)
    a = (rng.integers(0, 2**31 - 1, size=shape) if np.issubdtype(src, np.integer)
         else rng.normal(size=shape)).astype(src)
    for slot in (0, 0, 1):  # buffer reuse
        t = to_device(a, dst, slot=slot)
        assert t.shape == a.shape and t.device.type == "cuda"
        np.testing.assert_array_equal(t.cpu().numpy(), a.astype(dst))
    b = a[::2]  # non-contiguous source
    np.testing.assert_array_equal(to_device(b, dst).cpu().numpy(), b.astype(dst))


@pytest.mark.parametrize("shape", [(128, 30000), (7,)])
def test_to_host_exact(cuda, shape):
    import torch

    from paper_1811_07717_b200.device import to_host

    t = torch.randn(shape, dtype=torch.float64, device="cuda")
    for _ in range(2):
        h = to_host(t)
        assert isinstance(h, np.ndarray) and h.shape == tuple(shape)
        np.testing.assert_array_equal(h, t.cpu().numpy())
    h0 = to_host(t)
    t.add_(1.0)
    h1 = to_host(t)
    assert not np.shares_memory(h0, h1) and np.all(h1 == h0 + 1.0)
