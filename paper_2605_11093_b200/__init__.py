"""B200-native Ring^2 capture-and-stage path (DMI-Lib, arxiv 2605.11093).

Drop-in for the reference's hot path (tapflow): the same observation-point,
ring, policy, exporter and sink names, backed by sm_100a capture kernels, a
device-resident payload ring with device-side allocator counters, a native
staging engine (PCIe D2H into a pinned host ring) and a Python exporter.
See DESIGN.md for the boundary and INTEGRATION.md for the C ABI binding.
"""

from .errors import (
    AllocationError,
    ConfigError,
    DeviceError,
    HookDisabled,
    MetaMismatch,
    MetaRingFull,
    MissingShard,
    OutOfOrderRelease,
    PayloadRingFull,
    PolicyUnderestimate,
    ProtocolError,
    RingFull,
    StagingExhausted,
    TapflowError,
)
from .exporter import (
    STAGE_QUEUE_SLOTS,
    DrainBatch,
    DrainConfig,
    DrainEvent,
    ExportPipeline,
    PageableBatch,
    StagingPool,
    split_payload,
)
from .hooks import (
    CaptureOutcome,
    DeviceCopyEngine,
    DType,
    HookRegistry,
    HookSpec,
    ModelSpec,
    RowSource,
    TensorView,
    capture,
    capture_args,
    install_hooks,
    launch_capture,
)
from .policy import (
    BEST_EFFORT,
    COMPLETENESS,
    DROP_RECENT,
    KEEP_BY_PATTERN,
    PolicyConfig,
    Predicate,
    StepPlan,
    StepRequest,
    estimate_step_bytes,
    prepare_step,
)
from .records import CaptureRecord, StepMetas, TensorMeta, TensorMetaFIFO
from .rings import (
    COPY_UNIT,
    DESCRIPTOR_SIZE,
    READY_SENTINEL,
    Arena,
    Descriptor,
    RingConfig,
    RingPair,
    RingState,
    allocate_rings,
    round_up_to_copy_unit,
)
from .sinks import (
    FileSink,
    NativeFileSink,
    NativeStreamSink,
    NullSink,
    StreamSink,
    read_dataset,
    read_stream,
    record_from_header,
    records_to_stream_bytes,
    scan_dataset,
)

__version__ = "0.1.0"
