"""NVTX ranges around the public entry points (construct / factorize / solve,
the level uploads and the timed bench region), so an nsys or ncu
`--nvtx --nvtx-include` run can select one phase.  Ranges are host-side: the
kernels inside a replayed CUDA graph belong to the range of its launch."""

import contextlib
import functools

import torch


@contextlib.contextmanager
def nvtx_range(name):
    try:
        torch.cuda.nvtx.range_push(name)
        pushed = True
    except Exception:          # no CUDA / NVTX: ranges are optional
        pushed = False
    try:
        yield
    finally:
        if pushed:
            torch.cuda.nvtx.range_pop()


def ranged(name):
    """Decorator: run the function inside NVTX range `name`."""
    def wrap(fn):
        @functools.wraps(fn)
        def inner(*a, **kw):
            with nvtx_range(name):
                return fn(*a, **kw)
        return inner
    return wrap
