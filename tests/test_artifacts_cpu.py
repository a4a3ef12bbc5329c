"""CPU checks of the artifact formats (artifacts.py:7-126) and of the desk
model's initialisation (model.py:122-141) against files the reference wrote."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

from paper_2511_17849_b200 import artifacts
from paper_2511_17849_b200 import tinygpt

REF = os.path.join(GOLDEN, "tiny_gpt_artifacts")


def test_params_bin_bytes_identical_to_reference_writer(tmp_path):
    ref = artifacts.read_params(os.path.join(REF, "params.bin"))
    assert ref.dtype == np.float32 and ref.shape == (306_176,)
    artifacts.write_params(tmp_path / "p.bin", ref)
    assert (tmp_path / "p.bin").read_bytes() == open(os.path.join(REF, "params.bin"), "rb").read()


def test_params_bin_validation(tmp_path):
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOPE" + bytes(16))
    with pytest.raises(ValueError):
        artifacts.read_params(p)
    artifacts.write_params(tmp_path / "ok.bin", np.arange(5, dtype=np.float64))
    blob = (tmp_path / "ok.bin").read_bytes()
    (tmp_path / "trunc.bin").write_bytes(blob[:-3])
    with pytest.raises(ValueError):
        artifacts.read_params(tmp_path / "trunc.bin")
    with pytest.raises(ValueError):
        artifacts.write_params(tmp_path / "x.bin", np.zeros(3, np.int32))


def test_jsonl_rendering_matches_reference_lines():
    lines = open(os.path.join(REF, "trajectory.jsonl")).read().splitlines()
    import json
    for line in lines[1:]:
        rec = json.loads(line)
        assert artifacts.dumps_record(rec) == line
    assert artifacts.format_float(0.1) == "0.10000000000000001"


def test_tinygpt_init_matches_reference_stream():
    f = np.load(os.path.join(GOLDEN, "tiny_gpt.npz"))
    theta = tinygpt.init_params(256, 128, 2, 64, np.random.default_rng([0, 100]))
    assert np.array_equal(theta, f["theta0"])
