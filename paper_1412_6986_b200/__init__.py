"""paper_1412_6986_b200 -- B200-native hot path of the lmtune local-memory
auto-tuning study (arXiv 1412.6986).

Drop-in for the reference package's hot path (lmtune/__init__.py:9-84):
run and time both kernel variants of synthetic instances on the GPU
(``interp.execute`` / ``run_pair`` / ``measure_instances``), and batched
random-forest inference (``forest.predict`` / ``decide``). The compute is in
liblmt_b200.so (hand-written sm_100a CUDA behind a C ABI, include/lmt_b200.h);
there is no CPU fallback.
"""

from . import access_analysis, codegen, cost_model, dataset, dist, measure, metrics, real, study, sweep  # noqa: F401
from .access_analysis import (
    FEATURE_NAMES,
    FeatureVector,
    TimeEstimate,
    coalescing_degree,
    extract_features,
    features_records,
    kernel_time,
    label_speedup,
    reuse_degree,
)
from .codegen import KernelSource, defines_manifest, emit_baseline, emit_optimized, kernel_filename
from .cost_model import ResourceUsage, estimate_registers, occupancy, resource_usage
from .metrics import EvalReport, count_accuracy, evaluate, penalty_weighted_accuracy, speedup_histogram
from .dataset import (
    CSV_HEADER,
    BuildResult,
    LabeledInstance,
    build_arrays,
    build_dataset,
    read_rows,
    split_rows,
    write_rows,
    write_skip_log,
)
from .device import DEFAULT_DEVICE, DeviceDescriptor
from .errors import (
    ConfigError,
    DatasetFormatError,
    InvalidInstance,
    LmtuneError,
    ModelFormatError,
    OptimizationInfeasible,
)
from .forest import (
    Forest,
    GpuForest,
    Hyperparams,
    Tree,
    decide,
    load,
    predict,
    save,
    speedup_to_target,
    train,
    train_arrays,
    train_arrays_gpu,
)
from .geometry import (
    AffineAccess,
    EmitGeometry,
    Footprint,
    Variant,
    copy_transaction_count,
    emit_geometry,
    footprint,
    mad_constants,
    pad_col_span,
    pattern_affine,
)
from .interp import execute, make_inputs, run_pair
from .kernel_model import (
    Coord,
    HomeAccessPattern,
    KernelInstance,
    LaunchConfig,
    StencilPattern,
    StencilShape,
    TemplateParams,
    home_coordinate,
    stencil_offsets,
    validate_instance,
    validate_params,
    work_unit_for,
)
from .measure import (
    Measurement,
    measure_instances,
    measure_instances_host,
    measure_records,
    prepare_instances,
    prepare_records,
)
from .sweep import (
    CompileTuple,
    InstanceTable,
    SamplingSpec,
    enumerate_launch_configs,
    expand_patterns,
    instance_key,
    sample_compile_tuples,
    select_instance_table,
    select_instances,
)

__version__ = "0.1.0"
