"""VEGS model files: byte-identical to the reference's writer, and the reference's plain
and VQ files load to the same parameters (fixtures from tests/golden/make_golden.py)."""

import numpy as np
import pytest

import goldens as G
from paper_2504_13339_b200 import io as mio
from paper_2504_13339_b200.model import PARAM_CLASSES, GaussianSet


def test_save_is_byte_identical_to_reference(tmp_path):
    d = G.load("model_io")
    gs = GaussianSet(**{k: d["in_" + k] for k in PARAM_CLASSES})
    mio.save_model(gs, tmp_path / "m.vegs")
    assert (tmp_path / "m.vegs").read_bytes() == d["plain_bytes"].tobytes()


@pytest.mark.parametrize("kind", ["plain", "vq"])
def test_load_reference_files(tmp_path, kind):
    d = G.load("model_io")
    path = tmp_path / f"{kind}.vegs"
    path.write_bytes(d[f"{kind}_bytes"].tobytes())
    gs = mio.load_model(path)
    for k in PARAM_CLASSES:
        assert np.array_equal(getattr(gs, k), d[f"{kind}_" + k]), k


def test_format_errors(tmp_path):
    bad = tmp_path / "bad.vegs"
    bad.write_bytes(b"NOPE" + b"\0" * 60)
    with pytest.raises(mio.FormatError):
        mio.load_model(bad)
    d = G.load("model_io")
    trunc = tmp_path / "t.vegs"
    trunc.write_bytes(d["plain_bytes"].tobytes()[:-4])
    with pytest.raises(mio.FormatError):
        mio.load_model(trunc)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["plain", "vq"])
def test_load_to_device(tmp_path, kind):
    d = G.load("model_io")
    path = tmp_path / f"{kind}.vegs"
    path.write_bytes(d[f"{kind}_bytes"].tobytes())
    flat, n = mio.load_model_device(path)
    ref = GaussianSet(**{k: d[f"{kind}_" + k] for k in PARAM_CLASSES}).pack()
    assert n == 300 and np.array_equal(flat.cpu().numpy(), ref)
