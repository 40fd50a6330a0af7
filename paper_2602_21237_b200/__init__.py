"""B200-native tensor path for equi-joins and ORDER BY sorts.

A from-scratch sm_100a implementation of the tensor-based execution path of
arxiv/paper_2602_21237 behind the reference package's operator API
(``relab``: to_tensor / key_axis_align / tensor_join / tensor_sort, the
runtime path-selection policy, and the Relation / SpillStats / PathChoice
records). Host code is Python + PyTorch (device memory, streams,
torch.distributed); the hot path is hand-written CUDA in
``csrc/`` exposed through the C ABI of ``include/relab_b200.h``.
"""

from .errors import DeviceError, DigestMismatch, EmptySamples, OutputTooLarge, RelabError, UnknownAttribute
from .policy import (
    Operation,
    Path,
    PathChoice,
    Policy,
    Reason,
    RuntimeSignals,
    estimate_intermediate,
    estimate_key_cardinality,
    join_signals,
    select_path,
    sort_signals,
)
from .records import (
    BuildSide,
    Bytes,
    Direction,
    Int64,
    JoinSpec,
    MemoryBudget,
    Relation,
    Schema,
    SortSpec,
    SpillStats,
    join_output_schema,
)
from .synth import GenSpec, Uniform, Zipf, generate_relation
from .tensor_path import (
    MAX_OUTPUT_ROWS,
    AxisAlignment,
    TensorRelation,
    key_axis_align,
    tensor_join,
    tensor_sort,
    to_tensor,
)

__all__ = [name for name in dir() if not name.startswith("_")]
