"""Per-rank level buffers (ulv_factor._Win): a contiguous window of the level's
global offset space plus individually placed halo blocks — CPU checks of the
addressing the distributed factorization relies on."""
import pytest
import torch

from paper_2502_02395_b200.ulv_factor import _Win


def test_window_and_halo_addressing():
    w = _Win(100, 160, torch.device("cpu"), halo={10: 5, 400: 7, 120: 3})   # 120 lies inside the window
    assert w.numel() == 60 + 5 + 7
    base = w.tensor.data_ptr()
    assert w.ptr(100) == base and w.ptr(159) == base + 8 * 59
    assert w.data_ptr() + 8 * 130 == w.ptr(130)            # virtual base: global offsets address the window
    assert w.ptr(10) == base + 8 * 60 and w.ptr(400) == base + 8 * 65
    assert w.local(120) == 20 and w.local(400) == 65
    with pytest.raises(KeyError):
        w.ptr(200)                                           # neither in the window nor a halo block
    full = _Win(0, 50, torch.device("cpu"))
    assert full.numel() == 50 and full.data_ptr() == full.tensor.data_ptr()
