"""Generate tests/golden/ref_model_*.txt: model documents written by the UNMODIFIED reference
(streamconv model.save_model, text format v1, model.py:195-306), for the format-compatibility
test of paper_1611_09482_b200.model_io. Run here (where /root/reference exists):

    python oracle/make_model_docs.py

The reference package is imported from a /tmp copy (make_golden.import_reference); only its
output documents are committed.
"""

from __future__ import annotations

from pathlib import Path

from make_golden import import_reference

OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"
CASES = {
    "ref_model_tanh.txt": dict(blocks=2, layers_per_block=3, filter_width=2, dilation_base=2,
                               hidden_channels=4, activation="tanh", init_seed=3),
    "ref_model_linear_w3.txt": dict(blocks=1, layers_per_block=2, filter_width=3,
                                    dilation_base=3, hidden_channels=2, activation="linear",
                                    init_seed=11),
}


def main() -> None:
    sc = import_reference()
    for name, kw in CASES.items():
        m = sc.build_model(sc.ModelConfig(**kw))
        sc.save_model(m, OUT / name)
        print("wrote", OUT / name)


if __name__ == "__main__":
    main()
