"""B200-native fused Chebyshev-KAN layer (hot path of arxiv 2511.14852 / PolyKAN).

Public surface mirrors the reference package ``polykan`` for this path:
``lut_build`` / ``LutTable`` (lut.py), ``CoeffTensor`` / ``Layout`` /
``reorder_to_doj`` (tensor.py), ``fused_forward`` / ``backward_fused`` /
``KernelMode`` / ``TileSchedule`` (kernels.py), plus the torch module
``ChebyKANLayer`` and data-parallel helpers.  All compute runs in the
sm_100a kernels of ``lib/libchebykan.so``; there is no CPU fallback.
"""
from .basis import (
    RECURRENCES,
    BasisKind,
    RecurrenceCoeffs,
    basis_rows,
    chebyshev_second_derivative_max,
    degree_for,
    derivative_rows,
    eval_basis,
    eval_basis_derivative,
    eval_basis_trig,
    feature_count,
    parse_kind,
    trig_rows,
)
from .kernels import (
    EXACT_MODE,
    LUT_MODE,
    AtomicCounts,
    BasisPath,
    KernelCounters,
    KernelMode,
    NonFiniteInputError,
    PartialBuffer,
    PreparedCoeff,
    TileSchedule,
    backward_fused,
    chunk_rows,
    combine,
    count_atomics,
    forward_partial,
    count_flops,
    fused_forward,
    reference_backward,
    reference_forward,
)
from .layer import ChebyKANFunction, ChebyKANLayer, KANLayer
from .lut import (
    DEFAULT_LUT_SIZE,
    ExactBasis,
    LutTable,
    exact_basis,
    expand,
    interp_error_bound,
    interp_rows,
    interp_rows_with_slope,
    lut_build,
    lut_from_arrays,
    lut_interp,
    lut_interp_with_slope,
    lut_max_error_bound,
    lut_size_for_budget,
)
from .formats import load_coeff, load_lut, load_matrix, save_coeff, save_lut, save_matrix
from .model import (
    AdamHParams,
    AdamState,
    Dataset,
    DatasetError,
    Layer,
    LayerSpec,
    Loss,
    Network,
    NetworkSpec,
    TrainingDiverged,
    TrainResult,
    TrainTrace,
    adam_step,
    cross_entropy_loss,
    init_params,
    layer_forward,
    load_checkpoint,
    save_checkpoint,
    loss_fn,
    make_synthetic,
    mse,
    mse_loss,
    network_train,
    rmsle_loss,
)
from .optim import Adam, adam_update, cosine_scale
from .perf import (
    BenchResult,
    LayerConfig,
    Regime,
    RooflineReport,
    paper_configs,
    roofline,
    run_bench,
)
from .parallel import GradientAllreducer, PeerAllreducer, allreduce_gradients, chebykan_parameters, shard_bounds
from .tensor import CoeffTensor, Layout, doj_index, jod_index, reorder_to_doj, reorder_to_jod

__version__ = "1.0.0"
