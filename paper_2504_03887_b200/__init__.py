"""B200-native engine for the data-parallel hot path of xMem (arXiv 2504.03887).

Mirrors the reference package `peakmem` (pkg/src/peakmem/__init__.py) for the
path up to peak memory: allocator replay runs as a batched sm_100a CUDA
kernel (one warp per trace) behind the reference's own Python API.
"""

from .allocator import (
    AllocatorConfig,
    PackedTrace,
    SimulationResult,
    load_sequence_file,
    pack_trace,
    replay,
    replay_batch,
    round_request,
    segment_size_for,
)
from .errors import (
    CyclicParentLink,
    DoubleFree,
    DuplicateHandle,
    EmptyInput,
    EmptyTrace,
    EngineLimitExceeded,
    EngineUnavailable,
    MalformedSequence,
    MalformedTrace,
    MissingBatchBytes,
    NoGradientBlocks,
    NoIterationMarkers,
    NoIterations,
    OutOfMemory,
    PeakMemError,
    UnknownHandle,
    ZeroSize,
)

from .analysis import (
    AnnotationMarker,
    BlockRole,
    LayerNode,
    MarkerKind,
    MemoryBlock,
    OperatorNode,
    build_layer_tree,
    build_operator_roots,
    extract_markers,
    group_memory_events,
)
from .batch import SequenceBatch, build_sequences
from .estimator import EstimateReport, PeakMemoryEstimator
from .linking import LayerMemoryProfile, link
from .metrics import (
    EvalJob,
    MetricSet,
    Quadrant,
    ValidationRecord,
    aggregate,
    evaluate,
    evaluate_columns,
    evaluate_sweep,
    predict_oom,
)
from .orchestration import (
    AnalyzedTrace,
    MemoryRequest,
    RequestKind,
    RequestSequence,
    analyze,
    build_sequence,
)
from .trace import (
    EventCategory,
    SidecarConfig,
    TraceBundle,
    TraceEvent,
    load_sidecar,
    parse_trace,
)

__version__ = "0.1.0"
