"""CLI on the GPU: generate / verify / bench for both model kinds."""

import csv

import numpy as np
import pytest

from paper_1611_09482_b200.benchmark import CSV_COLUMNS, read_records
from paper_1611_09482_b200.cli import main

pytestmark = pytest.mark.gpu


def _lines(p):
    return [ln for ln in p.read_text().splitlines() if ln.strip()]


def test_plain_generate_fast_equals_naive_and_verify_is_exact(cuda, tmp_path):
    m = tmp_path / "m.txt"
    assert main(["init-model", "--layers", "3", "--blocks", "2", "--channels", "3",
                 "--seed", "4", "--out", str(m)]) == 0
    primer = tmp_path / "p.txt"
    primer.write_text("0.25\n-0.5\n")
    for mode in ("fast", "naive"):
        assert main(["generate", "--model", str(m), "--steps", "40", "--mode", mode,
                     "--primer", str(primer), "--out", str(tmp_path / f"{mode}.txt")]) == 0
    a = np.array([float(v) for v in _lines(tmp_path / "fast.txt")])
    b = np.array([float(v) for v in _lines(tmp_path / "naive.txt")])
    assert a.shape == (40,) and np.array_equal(a, b)
    assert main(["verify", "--model", str(m), "--steps", "32"]) == 0


def test_plain_random_grid_verifies_exactly(cuda, capsys):
    assert main(["verify", "--random-grid", "--steps", "12"]) == 0
    assert "144 model(s)" in capsys.readouterr().out


def test_cell_generate_and_verify(cuda, tmp_path):
    c = tmp_path / "c.txt"
    assert main(["init-cell", "--layers", "4", "--residual", "16", "--skip", "32",
                 "--bias", "fan_in", "--seed", "3", "--out", str(c)]) == 0
    for mode in ("fast", "naive"):
        assert main(["generate", "--model", str(c), "--steps", "30", "--mode", mode,
                     "--out", str(tmp_path / f"{mode}.txt")]) == 0
    a = [int(v) for v in _lines(tmp_path / "fast.txt")]
    b = [int(v) for v in _lines(tmp_path / "naive.txt")]
    assert len(a) == 30 and all(0 <= v < 256 for v in a)
    assert np.mean(np.array(a) == np.array(b)) >= 0.9
    assert main(["generate", "--model", str(c), "--steps", "10", "--mode", "fast",
                 "--sampler", "2", "--seed", "9", "--out", str(tmp_path / "g.txt")]) == 0
    assert main(["verify", "--model", str(c), "--steps", "24"]) == 0


def test_bench_writes_the_reference_csv(cuda, tmp_path):
    out = tmp_path / "sweep.csv"
    assert main(["bench", "--layers-from", "1", "--layers-to", "3", "--blocks", "1",
                 "--channels", "4", "--steps", "8", "--repeats", "3", "--warmup", "1",
                 "--out", str(out)]) == 0
    rows = list(csv.DictReader(out.open()))
    assert tuple(rows[0].keys()) == CSV_COLUMNS
    assert [(r["layers"], r["mode"]) for r in rows] == [
        (str(L), m) for L in (1, 2, 3) for m in ("fast", "naive")]
    fast3 = next(r for r in rows if r["layers"] == "3" and r["mode"] == "fast")
    naive3 = next(r for r in rows if r["layers"] == "3" and r["mode"] == "naive")
    assert int(naive3["node_evals_per_step"]) == 7 and int(fast3["node_evals_per_step"]) == 3
    recs = read_records(out)
    assert len(recs) == 6 and all(r.repeats == 3 and r.mean_s_per_sample > 0 for r in recs)
