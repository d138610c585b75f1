"""BNDM fixtures (item 3), the CSV harness (item 2), host-side parts.

CPU only.  The device residual (item 4) and the harness run live in test_gpu_next.py.
"""

from __future__ import annotations

import os
import struct

import numpy as np
import pytest

import paper_2305_04635_b200 as bc
from paper_2305_04635_b200 import fixtures, harness

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_reference_written_fixture_loads():
    """A file written by the reference's save_matrix (core.py:254-266) reads back exactly."""
    m = bc.load_matrix(os.path.join(GOLDEN, "fixture_ref.bndm"))
    want = np.load(os.path.join(GOLDEN, "fixture_ref.npy"))
    assert (m.dim, m.bandwidth, m.lead_dim) == (37, 5, 8)
    panel = m.data.reshape(37, 8).T
    assert np.array_equal(panel[:6], want)
    assert not panel[6:].any()  # padding was written as zeros


def test_save_is_byte_identical_to_reference_writer(tmp_path):
    m = bc.load_matrix(os.path.join(GOLDEN, "fixture_ref.bndm"))
    m.data.reshape(37, 8)[:, 6:] = 3.5  # junk in the padding must not reach the file
    out = tmp_path / "mine.bndm"
    bc.save_matrix(m, out)
    with open(out, "rb") as a, open(os.path.join(GOLDEN, "fixture_ref.bndm"), "rb") as b:
        assert a.read() == b.read()


def test_fixture_round_trip(tmp_path):
    a = bc.generate_spd(50, 7, seed=2)
    p = tmp_path / "a.bndm"
    bc.save_matrix(a, p)
    b = bc.load_matrix(p)
    assert (b.dim, b.bandwidth, b.lead_dim) == (50, 7, 8)
    assert np.array_equal(a.data, b.data)


@pytest.mark.parametrize("blob,msg", [
    (b"BND", "truncated"),
    (struct.pack("<4sIII", b"XXXX", 2, 1, 2) + bytes(32), "magic"),
    (struct.pack("<4sIII", b"BNDM", 2, 1, 2) + bytes(31), "payload"),
])
def test_fixture_errors(tmp_path, blob, msg):
    p = tmp_path / "bad.bndm"
    p.write_bytes(blob)
    with pytest.raises(bc.ShapeMismatch, match=msg):
        bc.load_matrix(p)


def test_csv_header_is_the_references():
    assert harness.CSV_HEADER == "N,k,n,workers,impl,backend,reps,median_seconds,gflops,residual"


def test_csv_round_trip(tmp_path):
    recs = [harness.BenchRecord(1000, 50, None, None, "b200", "sm_100a", 10, 1.25e-4, 4.1e2, 3.5e-16),
            harness.BenchRecord(1000, 60, None, None, "b200-host", "sm_100a", 10, None, None, None)]
    p = tmp_path / "r.csv"
    harness.emit_csv(recs, p)
    lines = p.read_text().splitlines()
    assert lines[0] == harness.CSV_HEADER
    assert lines[1] == "1000,50,,,b200,sm_100a,10,0.000125,410,3.5000000000000002e-16"
    assert harness.parse_csv(p) == recs


def test_csv_refuses_empty_and_foreign(tmp_path):
    with pytest.raises(bc.BandCholError):
        harness.emit_csv([], tmp_path / "x.csv")
    p = tmp_path / "y.csv"
    p.write_text("a,b\n")
    with pytest.raises(bc.BandCholError):
        harness.parse_csv(p)


@pytest.mark.parametrize("cfg,exc", [
    (dict(dim=0, bandwidths=(1,)), bc.ShapeMismatch),
    (dict(dim=10, bandwidths=(10,)), bc.InvalidBandwidth),
    (dict(dim=10, bandwidths=(-1,)), bc.InvalidBandwidth),
    (dict(dim=10, bandwidths=()), bc.BandCholError),
    (dict(dim=10, bandwidths=(2,), impls=("cuda",)), bc.BandCholError),
    (dict(dim=10, bandwidths=(2,), repetitions=0), bc.BandCholError),
])
def test_harness_validation(cfg, exc):
    with pytest.raises(exc):
        harness.validate(harness.BenchConfig(**cfg))


def test_harness_odd_bandwidth_needs_no_padding():
    assert harness.validate(harness.BenchConfig(dim=100, bandwidths=(3, 7, 50))) == [3, 7, 50]
