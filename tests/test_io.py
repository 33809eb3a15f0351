"""Serialisation parity: this package's writers reproduce the reference's files
byte for byte and its readers load them (fixtures written by the reference's own serialisers,
tests/golden/make_golden.py `io`; potentials.py:467-552)."""

from __future__ import annotations

import json
import os

import numpy as np

from paper_2604_18780_b200 import potentials as P
from paper_2604_18780_b200.instances import equivalence_instance

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _bytes(path):
    with open(path, "rb") as fh:
        return fh.read()


def test_emission_writers_match_reference_bytes(tmp_path):
    batch, _, _ = equivalence_instance(3, T=13, K=4, C=3, B=3, ragged=True, projections=True)
    P.save_emissions_csv(batch, tmp_path / "e.csv")
    P.save_emissions_json(batch, tmp_path / "e.json")
    assert _bytes(tmp_path / "e.csv") == _bytes(os.path.join(GOLD, "io_emissions.csv"))
    assert _bytes(tmp_path / "e.json") == _bytes(os.path.join(GOLD, "io_emissions.json"))


def test_readers_roundtrip_reference_files():
    batch, _, _ = equivalence_instance(3, T=13, K=4, C=3, B=3, ragged=True, projections=True)
    for loader, name in ((P.load_emissions_csv, "io_emissions.csv"), (P.load_emissions_json, "io_emissions.json")):
        got = loader(os.path.join(GOLD, name))
        assert np.array_equal(got.lengths, batch.lengths)
        valid = np.arange(batch.max_length)[None, :] < batch.lengths[:, None]
        assert np.array_equal(got.emissions[valid], batch.emissions[valid])


def test_params_and_segments_json(tmp_path):
    params = P.load_params_json(os.path.join(GOLD, "io_params.json"))
    P.save_params_json(params, tmp_path / "p.json")
    assert _bytes(tmp_path / "p.json") == _bytes(os.path.join(GOLD, "io_params.json"))
    with open(os.path.join(GOLD, "io_segments.json")) as fh:
        doc = json.load(fh)
    segs = P.segmentations_from_json(doc)
    assert [s.segments for s in segs] == [((0, 2, 1), (2, 3, 0)), ((0, 1, 2),)]
    assert P.segmentations_to_json(segs) == doc
