"""CLI host-side behaviour: model initialisation commands and the
reference's exit codes (cli.py:295-302: 0 ok, 2 for ValueError / OSError / usage)."""

import pytest

from paper_1611_09482_b200 import ModelConfig, build_cell_model, build_model
from paper_1611_09482_b200 import model_io as mi
from paper_1611_09482_b200.cell import CellConfig
from paper_1611_09482_b200.cli import main, verification_grid


def test_init_model_writes_the_seeded_model(tmp_path, capsys):
    out = tmp_path / "m.txt"
    assert main(["init-model", "--layers", "3", "--blocks", "2", "--channels", "4",
                 "--activation", "linear", "--seed", "5", "--out", str(out)]) == 0
    m = mi.load_model(out)
    assert m.equals(build_model(ModelConfig(2, 3, hidden_channels=4, activation="linear",
                                            init_seed=5)))
    text = capsys.readouterr().out
    assert "receptive field: 15" in text and "queue capacities: 1 2 4 1 2 4" in text


def test_init_cell_writes_the_seeded_model(tmp_path):
    out = tmp_path / "c.txt"
    assert main(["init-cell", "--layers", "3", "--residual", "8", "--skip", "16",
                 "--classes", "16", "--dtype", "bf16", "--bias", "fan_in", "--seed", "2",
                 "--out", str(out)]) == 0
    m = mi.load_cell_model(out)
    ref = build_cell_model(CellConfig(1, 3, 8, 8, 16, classes=16, weight_dtype="bf16",
                                      bias="fan_in", init_seed=2))
    assert m.config == ref.config
    assert (m.embed == ref.embed).all() and (m.head2_w == ref.head2_w).all()


def test_usage_errors_exit_2(tmp_path, capsys):
    assert main(["generate", "--model", str(tmp_path / "missing.txt"), "--steps", "3",
                 "--mode", "fast", "--out", str(tmp_path / "y")]) == 2
    assert main(["init-model", "--layers", "0", "--out", str(tmp_path / "m")]) == 2
    bad = tmp_path / "bad.txt"
    bad.write_text("not a model\n")
    assert main(["verify", "--model", str(bad)]) == 2
    assert "error:" in capsys.readouterr().err
    with pytest.raises(SystemExit) as e:
        main(["generate", "--steps", "3"])
    assert e.value.code == 2


def test_verification_grid_is_the_reference_grid():
    g = verification_grid()
    assert len(g) == 144
    assert g[0] == ModelConfig(1, 1, filter_width=2, dilation_base=2, hidden_channels=1,
                               activation="linear", init_seed=7)
    assert {c.blocks for c in g} == {1, 2, 3} and {c.filter_width for c in g} == {2, 3}
