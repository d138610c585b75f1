"""Write a BNDM fixture with the REFERENCE's own writer (build container only).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fixture.py

Output (committed): fixture_ref.bndm -- bandchol.save_matrix (core.py:254-266) of
generate_spd(37, 5, seed=4) re-laid into lead_dim 8 (padding rows hold junk in memory,
which the writer must zero), and fixture_ref.npy -- the in-band panel it holds.
"""
import os

import numpy as np

import bandchol

HERE = os.path.dirname(os.path.abspath(__file__))
src = bandchol.generate_spd(37, 5, seed=4)
m = bandchol.BandedMatrix(37, 5, 8)
m.panel[:6, :] = src.band_panel()
m.panel[6:, :] = 7.25  # padding junk: the writer zeroes it
bandchol.save_matrix(m, os.path.join(HERE, "fixture_ref.bndm"))
np.save(os.path.join(HERE, "fixture_ref.npy"), src.band_panel().copy())
print("wrote fixture_ref.bndm", os.path.getsize(os.path.join(HERE, "fixture_ref.bndm")), "bytes")
