"""Model documents: the reference's plain text format v1, bit-exact and
byte-compatible with files the unmodified reference wrote (tests/golden/ref_model_*.txt,
oracle/make_model_docs.py), and the cell extension of the same format. Errors follow the
reference (ModelFormatError, a ValueError) -- its model tests check the same cases.
"""

from pathlib import Path

import numpy as np
import pytest

from paper_1611_09482_b200 import ModelConfig, build_cell_model, build_model
from paper_1611_09482_b200 import model_io as mi
from paper_1611_09482_b200.cell import CellConfig

GOLDEN = Path(__file__).parent / "golden"
REF_DOCS = {
    "ref_model_tanh.txt": ModelConfig(2, 3, filter_width=2, dilation_base=2, hidden_channels=4,
                                      activation="tanh", init_seed=3),
    "ref_model_linear_w3.txt": ModelConfig(1, 2, filter_width=3, dilation_base=3,
                                           hidden_channels=2, activation="linear", init_seed=11),
}


@pytest.mark.parametrize("name", sorted(REF_DOCS))
def test_reads_reference_documents_and_writes_them_byte_identically(name):
    text = (GOLDEN / name).read_text(encoding="utf-8")
    m = mi.model_from_text(text)
    assert m.config == REF_DOCS[name]
    assert m.equals(build_model(REF_DOCS[name]))  # same seeded weights as the reference's
    assert mi.model_to_text(m) == text


@pytest.mark.parametrize("cfg", [ModelConfig(1, 1), ModelConfig(3, 4, hidden_channels=8),
                                 ModelConfig(1, 3, filter_width=4, dilation_base=4,
                                             hidden_channels=3, activation="linear",
                                             init_seed=9)])
def test_plain_round_trip_is_bit_exact(tmp_path, cfg):
    m = build_model(cfg)
    p = tmp_path / "m.txt"
    mi.save_model(m, p)
    m2 = mi.load_model(p)
    assert m2.config == cfg and m.equals(m2)
    for a, b in zip(m.layers, m2.layers):
        assert np.array_equal(a.taps, b.taps) and np.array_equal(a.bias, b.bias)
    assert mi.load_any(p).equals(m)


@pytest.mark.parametrize("cfg", [
    CellConfig(1, 3, 8, 8, 16, classes=16, bias="fan_in", init_seed=4),
    CellConfig(2, 2, 8, 4, 12, classes=10, head_channels=20, weight_dtype="bf16",
               init="normal:0.1", init_seed=7),
])
def test_cell_round_trip_is_bit_exact(tmp_path, cfg):
    m = build_cell_model(cfg)
    p = tmp_path / "c.txt"
    mi.save_cell_model(m, p)
    m2 = mi.load_cell_model(p)
    assert m2.config == cfg
    for k in ("embed", "head1_w", "head1_b", "head2_w", "head2_b"):
        assert np.array_equal(getattr(m, k), getattr(m2, k)), k
    for a, b in zip(m.layers, m2.layers):
        for k in ("dil_taps", "dil_bias", "res_w", "res_b", "skip_w", "skip_b"):
            assert np.array_equal(getattr(a, k), getattr(b, k)), k
    assert isinstance(mi.load_any(p), type(m))
    assert mi.cell_model_to_text(m2) == p.read_text(encoding="utf-8")


def _plain_text():
    return mi.model_to_text(build_model(ModelConfig(1, 2, hidden_channels=2, init_seed=1)))


@pytest.mark.parametrize("mutate,msg", [
    (lambda t: t.replace("streamconv model v1", "streamconv model v2"), "header"),
    (lambda t: t.replace("init_seed = 1\n", ""), "missing keys"),
    (lambda t: t.replace("init_seed = 1\n", "init_seed = 1\ncolour = red\n"), "unknown keys"),
    (lambda t: t.replace("blocks = 1", "blocks = one"), "bad config"),
    (lambda t: t.replace("tap 1", "tap 7"), "expected 'tap 1'"),
    (lambda t: t.rsplit("\n", 2)[0] + "\n", "truncated|expected"),
    (lambda t: t + "extra line\n", "trailing"),
])
def test_plain_format_errors(mutate, msg):
    with pytest.raises(mi.ModelFormatError, match=msg):
        mi.model_from_text(mutate(_plain_text()))


def test_non_finite_and_ragged_rows_are_rejected():
    t = _plain_text().splitlines()
    i = t.index("tap 0") + 1
    bad = t.copy()
    bad[i] = "nan " + " ".join(bad[i].split()[1:])
    with pytest.raises(mi.ModelFormatError, match="non-finite"):
        mi.model_from_text("\n".join(bad))
    bad = t.copy()
    bad[i] = bad[i] + " 0.5"
    with pytest.raises(mi.ModelFormatError, match="expected"):
        mi.model_from_text("\n".join(bad))
    assert issubclass(mi.ModelFormatError, ValueError)


def test_cell_format_errors():
    m = build_cell_model(CellConfig(1, 3, 8, 8, 16, classes=16, init_seed=4))
    t = mi.cell_model_to_text(m)
    with pytest.raises(mi.ModelFormatError, match="header"):
        mi.cell_model_from_text(t.replace("fastwavenet cell v1", "fastwavenet cell v0"))
    with pytest.raises(mi.ModelFormatError, match="expected 'skip_bias'"):
        mi.cell_model_from_text(t.replace("skip_bias", "skip_b", 1))
    with pytest.raises(mi.ModelFormatError, match="bad config"):
        mi.cell_model_from_text(t.replace("weight_dtype = f32", "weight_dtype = f16"))
    with pytest.raises(mi.ModelFormatError, match="unknown model document"):
        p = Path("/tmp/_fw_bad_doc.txt")
        p.write_text("something else\n")
        mi.load_any(p)


def test_narrow_dilation_base_warns(tmp_path):
    m = build_model(ModelConfig(1, 2, filter_width=3, dilation_base=2, hidden_channels=2))
    p = tmp_path / "n.txt"
    mi.save_model(m, p)
    with pytest.warns(UserWarning):
        mi.load_model(p)
