"""Container format of paper_2502_02395_b200.storage (the reference's
storage.py:1-255 layout) — CPU checks: vector files and an H² container
round trip on a host (numpy) H² restated from the golden fixtures."""
import numpy as np
import pytest

from paper_2502_02395_b200 import storage
from paper_2502_02395_b200.errors import PointFormatError


def test_vector_round_trips(tmp_path):
    v = np.random.default_rng(3).standard_normal(100)
    for fmt in ("csv", "bin"):
        p = tmp_path / f"v.{fmt}"
        storage.save_vector(v, p, fmt=fmt)
        assert np.array_equal(storage.load_vector(p), v)
    with pytest.raises(ValueError):
        storage.save_vector(np.zeros(3), tmp_path / "v.x", fmt="hdf5")
    p = tmp_path / "t.bin"
    storage.save_vector(np.arange(8.0), p, fmt="bin")
    p.write_bytes(p.read_bytes()[:-8])
    with pytest.raises(PointFormatError):
        storage.load_vector(p)
    p = tmp_path / "m.csv"
    p.write_text("1.0\nnot-a-number\n")
    with pytest.raises(PointFormatError):
        storage.load_vector(p)


def test_h2_container_round_trip_bit_exact(tmp_path):
    from fixtures import H2_FIXTURES, load_h2
    h2 = load_h2(H2_FIXTURES[0])
    for b in h2.bases.values():          # the fixture stores no frames
        b.frame = np.arange(b.rank * b.rank, dtype=np.float64).reshape(b.rank, b.rank)
    h2.skeletons = {key: np.asarray(b.skeleton, dtype=np.int64) for key, b in h2.bases.items()}
    storage.save_h2(h2, tmp_path)
    back = storage.load_h2(tmp_path)
    assert back.count == h2.count and back.tree.depth == h2.tree.depth
    assert np.array_equal(back.cloud.perm, h2.cloud.perm)
    assert back.lists.near == [set(s) for s in h2.lists.near] and back.lists.far == [set(s) for s in h2.lists.far]
    for key, b in h2.bases.items():
        c = back.bases[key]
        assert c.rank == b.rank and np.array_equal(c.q_skel, b.q_skel) and np.array_equal(c.q_red, b.q_red)
        assert np.array_equal(c.frame, b.frame) and np.array_equal(c.skeleton, b.skeleton)
    for key, blk in h2.near_blocks.items():
        assert np.array_equal(back.near_blocks[key], blk)
    for key, blk in h2.couplings.items():
        assert np.array_equal(back.couplings[key], blk)
    with pytest.raises(ValueError):
        storage.load_factors(tmp_path)
