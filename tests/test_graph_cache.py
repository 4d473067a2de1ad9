"""FSA1 CSR cache (reference graph.py:266-292): byte layout, round trip, and the reference's
error messages for malformed files (tests/test_graph.py of the reference).  CPU only."""

import struct

import numpy as np
import pytest
import torch

from paper_2511_13645_b200.graph import CsrGraph, GraphFormatError, load_csr_cache, save_csr_cache


def small_graph():
    rowptr = np.array([0, 2, 3, 5, 5], np.int32)
    col = np.array([1, 2, 0, 0, 1], np.int32)
    return CsrGraph.from_arrays(rowptr, col, device="cpu")


def test_byte_layout_matches_reference_format(tmp_path):
    g = small_graph()
    p = tmp_path / "g.fsa1"
    save_csr_cache(g, p)
    want = b"FSA1" + struct.pack("<Q", 4) + np.array([0, 2, 3, 5, 5], "<i4").tobytes() + \
        np.array([1, 2, 0, 0, 1], "<i4").tobytes()
    assert p.read_bytes() == want


def test_round_trip(tmp_path):
    rng = np.random.default_rng(3)
    n = 500
    deg = rng.integers(0, 20, n)
    rowptr = np.concatenate([[0], np.cumsum(deg)]).astype(np.int32)
    col = np.concatenate([np.sort(rng.choice(n, d, replace=False)) for d in deg]).astype(np.int32)
    g = CsrGraph.from_arrays(rowptr, col, device="cpu")
    p = tmp_path / "g.fsa1"
    save_csr_cache(g, p)
    h = load_csr_cache(p, device="cpu")
    assert h.num_nodes == n and torch.equal(h.rowptr, g.rowptr) and torch.equal(h.col, g.col)


def test_malformed_files(tmp_path):
    p = tmp_path / "bad"
    p.write_bytes(b"XXXX" + struct.pack("<Q", 4))
    with pytest.raises(GraphFormatError, match="bad magic"):
        load_csr_cache(p, device="cpu")
    p.write_bytes(b"FSA1" + struct.pack("<Q", 0))
    with pytest.raises(GraphFormatError, match="implausible node count"):
        load_csr_cache(p, device="cpu")
    p.write_bytes(b"FSA1" + struct.pack("<Q", 4) + np.array([0, 2], "<i4").tobytes())
    with pytest.raises(GraphFormatError, match="truncated rowptr"):
        load_csr_cache(p, device="cpu")
    p.write_bytes(b"FSA1" + struct.pack("<Q", 1) + np.array([0, 3], "<i4").tobytes() + np.array([0], "<i4").tobytes())
    with pytest.raises(GraphFormatError, match="truncated col"):
        load_csr_cache(p, device="cpu")
    assert issubclass(GraphFormatError, ValueError)


def test_interoperates_with_the_reference_writer_and_reader(tmp_path):
    """When the reference is present (this container, not the GPU box): its save/load and ours
    read each other's files."""
    import os
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference not mounted")
    sys.path.insert(0, src)
    try:
        from fsa import graph as rg
    finally:
        sys.path.remove(src)
    ref = rg.gen_power_law(2000, 8.0, 2.1, 7)
    p1, p2 = tmp_path / "ref.fsa1", tmp_path / "ours.fsa1"
    rg.save_csr_cache(ref, p1)
    ours = load_csr_cache(p1, device="cpu")
    assert np.array_equal(ours.rowptr.numpy(), ref.rowptr) and np.array_equal(ours.col.numpy(), ref.col)
    save_csr_cache(ours, p2)
    assert p1.read_bytes() == p2.read_bytes()
    back = rg.load_csr_cache(p2)
    assert np.array_equal(back.col, ref.col)


def test_reference_batch_stream_bitwise(reference_fsa):
    """synth.reference_batches reproduces the reference's _batch_stream (bench.py:172-179),
    including the reshuffle at the epoch boundary."""
    import itertools

    from fsa import bench as ref_bench
    from paper_2511_13645_b200 import synth

    for n, b, seed in ((1000, 96, 42), (2_449_029, 1024, 43)):
        steps = n // b + 2 if n < 10_000 else 3
        want = list(itertools.islice(ref_bench._batch_stream(n, b, seed), steps))
        got = list(itertools.islice(synth.reference_batches(n, b, seed, device="cpu"), steps))
        assert all(np.array_equal(w, g.numpy()) for w, g in zip(want, got))
