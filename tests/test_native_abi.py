"""CPU checks of the C ABI: the library loads without a GPU and exports every
function include/h2ulv_b200.h declares; the numpy descriptor layouts match."""
import os
import re

from paper_2502_02395_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "h2ulv_b200.h")


def test_header_symbols_exported():
    text = open(HEADER).read()
    declared = sorted(set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(h2g_\w+)\s*\(", text, re.M)))
    assert declared, "no declarations parsed"
    lib = _native.load_library()
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing
    assert sorted(declared) == sorted(_native.EXPORTS)
    assert lib.h2g_abi_version() == 1


def test_tile_helpers_agree():
    from paper_2502_02395_b200 import program

    lib = _native.load_library()
    for m, n, f in [(1, 1, 0), (64, 64, 0), (65, 200, 0), (300, 300, 1), (128, 128, 1), (0, 5, 0)]:
        for cfg in (2, 7, 9):
            assert lib.h2g_gemm_tiles(m, n, f, cfg) == program.gemm_tiles(m, n, f, cfg)
    for r, c in [(1, 1), (32, 33), (100, 7)]:
        assert lib.h2g_copy_tiles(r, c) == program.copy_tiles(r, c)


def test_no_cuda_raises_loudly():
    import torch

    import paper_2502_02395_b200 as pkg
    from paper_2502_02395_b200.errors import NativeUnavailableError

    if torch.cuda.is_available():
        return
    import pytest

    with pytest.raises(NativeUnavailableError):
        pkg.factorize(None)
