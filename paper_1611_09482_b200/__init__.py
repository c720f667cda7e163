"""B200-native queue-cached generation step (arXiv 1611.09482, "Fast WaveNet").

Drop-in for the reference package ``streamconv``'s generation path: the
reference's names (ModelConfig, LayerWeights, Model, build_model, init_state,
fast_step, fast_generate, pop_phase, compute_step, push_phase,
GenerationState, QueueStateError, count_macs) run on the GPU through
libfastwavenet.so (include/fastwavenet.h). The gated WaveNet cell that
BASELINE.json names is served by ``CellModel`` / ``CellGenerator`` /
``cell_fast_generate``.
"""

from .cell import CellConfig, CellLayer, CellModel, build_cell_model, round_to_bf16
from .model import (
    ACTIVATIONS,
    LayerWeights,
    MacCount,
    Model,
    ModelConfig,
    build_model,
    count_macs,
    receptive_field,
)
from ._lib import QueueStateError
from .fast import (
    GenerationState,
    RecurrentInputs,
    SampleSequence,
    compute_step,
    fast_generate,
    fast_step,
    init_state,
    pop_phase,
    push_phase,
)
from .generate import CellGenerator, Sampler, cell_fast_generate, init_cell_state
from .naive import NaiveCellGenerator, cell_naive_generate, naive_generate, naive_step
from .model_io import (
    ModelFormatError,
    load_cell_model,
    load_model,
    model_from_text,
    model_to_text,
    save_cell_model,
    save_model,
)
from .benchmark import (
    CSV_COLUMNS,
    MODES,
    TimingRecord,
    default_grid,
    emit_records,
    read_records,
    run_benchmark,
)

__version__ = "0.1.0"

__all__ = [
    "ACTIVATIONS", "CSV_COLUMNS", "CellConfig", "CellGenerator", "CellLayer",
    "CellModel", "GenerationState", "LayerWeights", "MODES", "MacCount",
    "Model", "ModelConfig", "ModelFormatError", "NaiveCellGenerator", "QueueStateError",
    "RecurrentInputs", "SampleSequence", "Sampler", "TimingRecord", "build_cell_model",
    "build_model", "cell_fast_generate", "cell_naive_generate", "compute_step", "count_macs",
    "default_grid", "emit_records", "fast_generate", "fast_step", "init_cell_state",
    "init_state", "load_cell_model", "load_model", "model_from_text", "model_to_text",
    "naive_generate", "naive_step", "pop_phase", "push_phase", "read_records",
    "receptive_field", "round_to_bf16", "run_benchmark", "save_cell_model", "save_model",
]
