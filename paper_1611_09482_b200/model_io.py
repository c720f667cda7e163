"""Model documents on disk: SURVEY §8(f) rank 3.

* Plain mode: the reference's text format v1 (``streamconv model v1``, reference
  ``model.py:195-306``): a header line, ``key = value`` config lines in a fixed order,
  then per layer ``layer l``, ``tap k`` blocks of out-channel rows (in-channel values) and
  a ``bias`` row; floats with 17 significant digits, so a save/load round trip is
  bit-exact and files written by the reference load here (and vice versa).
* Gated cell (the north-star model, which the reference has no format for): the same
  conventions extended -- header ``fastwavenet cell v1``, the CellConfig keys, then
  ``embed``, per layer ``layer l`` with ``dil_tap 0`` / ``dil_tap 1`` / ``dil_bias`` /
  ``res`` / ``res_bias`` / ``skip`` / ``skip_bias`` blocks and the two heads. Values are
  float32 written with 9 significant digits (a float32 round trip is exact).

Errors are ``ModelFormatError`` (a ``ValueError``), as in the reference.
"""

from __future__ import annotations

import warnings
from pathlib import Path

import numpy as np

from .cell import CellConfig, CellLayer, CellModel
from .model import LayerWeights, Model, ModelConfig

PLAIN_MAGIC = "streamconv model v1"
PLAIN_KEYS = ("blocks", "layers_per_block", "filter_width", "dilation_base",
              "hidden_channels", "activation", "init_seed")
CELL_MAGIC = "fastwavenet cell v1"
CELL_KEYS = ("blocks", "layers_per_block", "residual_channels", "dilation_channels",
             "skip_channels", "classes", "head_channels", "dilation_base", "weight_dtype",
             "init", "bias", "init_seed")


class ModelFormatError(ValueError):
    """A model document that does not parse (reference model.py ModelFormatError)."""


# ---- shared reading helpers ----------------------------------------------------------------
class _Reader:
    def __init__(self, text: str, magic: str):
        lines = [ln.rstrip() for ln in text.splitlines()]
        self.lines = [ln for ln in lines if ln.strip()]
        if not self.lines or self.lines[0].strip() != magic:
            raise ModelFormatError(f"missing header line {magic!r}")
        self.pos = 1

    def config(self, keys, stop_prefix: str) -> dict[str, str]:
        fields: dict[str, str] = {}
        while self.pos < len(self.lines) and not self.lines[self.pos].startswith(stop_prefix):
            line = self.lines[self.pos]
            if "=" not in line:
                raise ModelFormatError(f"bad config line: {line!r}")
            key, _, value = line.partition("=")
            fields[key.strip()] = value.strip()
            self.pos += 1
        missing = set(keys) - set(fields)
        if missing:
            raise ModelFormatError(f"config block missing keys: {sorted(missing)}")
        extra = set(fields) - set(keys)
        if extra:
            raise ModelFormatError(f"config block has unknown keys: {sorted(extra)}")
        return fields

    def expect(self, tag: str) -> None:
        if self.pos >= len(self.lines) or self.lines[self.pos].strip() != tag:
            found = self.lines[self.pos].strip() if self.pos < len(self.lines) else "end of file"
            raise ModelFormatError(f"expected {tag!r}, found {found!r}")
        self.pos += 1

    def row(self, width: int, context: str, dtype) -> np.ndarray:
        if self.pos >= len(self.lines):
            raise ModelFormatError(f"{context}: truncated")
        parts = self.lines[self.pos].split()
        self.pos += 1
        if len(parts) != width:
            raise ModelFormatError(f"{context}: expected {width} values, got {len(parts)}")
        try:
            r = np.array([float(p) for p in parts], dtype=dtype)
        except ValueError as exc:
            raise ModelFormatError(f"{context}: {exc}") from None
        if not np.isfinite(r).all():
            raise ModelFormatError(f"{context}: non-finite weight entry")
        return r

    def matrix(self, rows: int, cols: int, context: str, dtype) -> np.ndarray:
        return np.stack([self.row(cols, context, dtype) for _ in range(rows)])

    def done(self) -> None:
        if self.pos != len(self.lines):
            raise ModelFormatError(f"unexpected trailing content: {self.lines[self.pos]!r}")


def _frozen(a: np.ndarray) -> np.ndarray:
    a.setflags(write=False)
    return a


# ---- plain mode: the reference's text format v1 ----------------------------------------------
def _f64(x: float) -> str:
    return format(float(x), ".17g")  # 17 significant digits: exact for float64


def model_to_text(model: Model) -> str:
    cfg = model.config
    out = [PLAIN_MAGIC] + [f"{k} = {getattr(cfg, k)}" for k in PLAIN_KEYS]
    for l, lw in enumerate(model.layers):
        out += ["", f"layer {l}"]
        for k in range(lw.taps.shape[0]):
            out.append(f"tap {k}")
            out += [" ".join(_f64(v) for v in row) for row in lw.taps[k]]
        out += ["bias", " ".join(_f64(v) for v in lw.bias)]
    out.append("")
    return "\n".join(out)


def model_from_text(text: str) -> Model:
    rd = _Reader(text, PLAIN_MAGIC)
    f = rd.config(PLAIN_KEYS, "layer ")
    try:
        cfg = ModelConfig(blocks=int(f["blocks"]), layers_per_block=int(f["layers_per_block"]),
                          filter_width=int(f["filter_width"]),
                          dilation_base=int(f["dilation_base"]),
                          hidden_channels=int(f["hidden_channels"]),
                          activation=f["activation"], init_seed=int(f["init_seed"]))
    except ValueError as exc:
        raise ModelFormatError(f"bad config: {exc}") from None
    layers = []
    for l, (c_in, c_out) in enumerate(cfg.channel_dims()):
        rd.expect(f"layer {l}")
        taps = np.empty((cfg.filter_width, c_out, c_in), dtype=np.float64)
        for k in range(cfg.filter_width):
            rd.expect(f"tap {k}")
            taps[k] = rd.matrix(c_out, c_in, f"layer {l} tap {k}", np.float64)
        rd.expect("bias")
        bias = rd.row(c_out, f"layer {l} bias", np.float64)
        layers.append(LayerWeights(taps=_frozen(taps), bias=_frozen(bias)))
    rd.done()
    return Model(config=cfg, layers=tuple(layers))


def save_model(model: Model, destination: str | Path) -> None:
    Path(destination).write_text(model_to_text(model), encoding="utf-8")


def load_model(source: str | Path) -> Model:
    model = model_from_text(Path(source).read_text(encoding="utf-8"))
    c = model.config
    if c.dilation_base < c.filter_width:  # as the reference warns (model.py:164-174)
        warnings.warn(f"dilation_base {c.dilation_base} < filter_width {c.filter_width}: the "
                      "queues cache more than the (w-1)*r**L bound", UserWarning, stacklevel=2)
    return model


# ---- gated cell -------------------------------------------------------------------------------
def _f32(x: float) -> str:
    return format(float(np.float32(x)), ".9g")  # 9 significant digits: exact for float32


def _rows(m: np.ndarray) -> list[str]:
    return [" ".join(_f32(v) for v in row) for row in np.atleast_2d(m)]


def cell_model_to_text(model: CellModel) -> str:
    c = model.config
    vals = {k: getattr(c, k) for k in CELL_KEYS}  # head_channels may be None (= skip)
    out = [CELL_MAGIC] + [f"{k} = {vals[k]}" for k in CELL_KEYS]
    out += ["", "embed"] + _rows(model.embed)
    for l, lw in enumerate(model.layers):
        out += ["", f"layer {l}"]
        for k in range(2):
            out += [f"dil_tap {k}"] + _rows(lw.dil_taps[k])
        out += ["dil_bias"] + _rows(lw.dil_bias)
        out += ["res"] + _rows(lw.res_w) + ["res_bias"] + _rows(lw.res_b)
        out += ["skip"] + _rows(lw.skip_w) + ["skip_bias"] + _rows(lw.skip_b)
    out += ["", "head1"] + _rows(model.head1_w) + ["head1_bias"] + _rows(model.head1_b)
    out += ["head2"] + _rows(model.head2_w) + ["head2_bias"] + _rows(model.head2_b)
    out.append("")
    return "\n".join(out)


def cell_model_from_text(text: str) -> CellModel:
    rd = _Reader(text, CELL_MAGIC)
    f = rd.config(CELL_KEYS, "embed")
    try:
        cfg = CellConfig(blocks=int(f["blocks"]), layers_per_block=int(f["layers_per_block"]),
                         residual_channels=int(f["residual_channels"]),
                         dilation_channels=int(f["dilation_channels"]),
                         skip_channels=int(f["skip_channels"]), classes=int(f["classes"]),
                         head_channels=(None if f["head_channels"] == "None"
                                        else int(f["head_channels"])),
                         dilation_base=int(f["dilation_base"]), weight_dtype=f["weight_dtype"],
                         init=f["init"], bias=f["bias"], init_seed=int(f["init_seed"]))
    except ValueError as exc:
        raise ModelFormatError(f"bad config: {exc}") from None
    R, D, S, H, A = (cfg.residual_channels, cfg.dilation_channels, cfg.skip_channels, cfg.H,
                     cfg.classes)
    f32 = np.float32
    rd.expect("embed")
    embed = rd.matrix(A, R, "embed", f32)
    layers = []
    for l in range(cfg.total_layers):
        rd.expect(f"layer {l}")
        taps = np.empty((2, 2 * D, R), dtype=f32)
        for k in range(2):
            rd.expect(f"dil_tap {k}")
            taps[k] = rd.matrix(2 * D, R, f"layer {l} dil_tap {k}", f32)
        rd.expect("dil_bias")
        db = rd.row(2 * D, f"layer {l} dil_bias", f32)
        rd.expect("res")
        rw = rd.matrix(R, D, f"layer {l} res", f32)
        rd.expect("res_bias")
        rb = rd.row(R, f"layer {l} res_bias", f32)
        rd.expect("skip")
        sw = rd.matrix(S, D, f"layer {l} skip", f32)
        rd.expect("skip_bias")
        sb = rd.row(S, f"layer {l} skip_bias", f32)
        layers.append(CellLayer(*(_frozen(a) for a in (taps, db, rw, rb, sw, sb))))
    rd.expect("head1")
    h1 = rd.matrix(H, S, "head1", f32)
    rd.expect("head1_bias")
    h1b = rd.row(H, "head1_bias", f32)
    rd.expect("head2")
    h2 = rd.matrix(A, H, "head2", f32)
    rd.expect("head2_bias")
    h2b = rd.row(A, "head2_bias", f32)
    rd.done()
    return CellModel(config=cfg, embed=_frozen(embed), layers=tuple(layers),
                     head1_w=_frozen(h1), head1_b=_frozen(h1b), head2_w=_frozen(h2),
                     head2_b=_frozen(h2b))


def save_cell_model(model: CellModel, destination: str | Path) -> None:
    Path(destination).write_text(cell_model_to_text(model), encoding="utf-8")


def load_cell_model(source: str | Path) -> CellModel:
    return cell_model_from_text(Path(source).read_text(encoding="utf-8"))


def load_any(source: str | Path) -> Model | CellModel:
    """Either document kind, by its header line."""
    text = Path(source).read_text(encoding="utf-8")
    head = next((ln.strip() for ln in text.splitlines() if ln.strip()), "")
    if head == CELL_MAGIC:
        return cell_model_from_text(text)
    if head == PLAIN_MAGIC:
        return model_from_text(text)
    raise ModelFormatError(f"unknown model document header {head!r}")
