"""B200-native quantum-kernel hot path of arXiv 2411.09336.

Drop-in for the hot-path API of the reference package ``mpskernel``
(/root/reference/pkg/src/mpskernel/__init__.py): feature-map construction,
MPS simulation and kernel-matrix building keep their names and signatures;
the arithmetic runs in hand-written sm_100a CUDA kernels (libmpskq.so, C ABI
in include/mpskq.h).  ``learn``/``cli`` (SVM, CLI) are outside the hot path
and not re-implemented: the reference's own consume ``GramMatrix`` unchanged.
"""

from .ansatz import (
    GATE_KINDS,
    Circuit,
    FeatureMapConfig,
    Gate,
    build_circuit,
    encode_circuit,
    gate_matrix,
    interaction_graph,
    layered_gates,
    route_linear,
    schedule_circuit,
    schedule_layers,
)
from .kernel import (
    GramMatrix,
    RunReport,
    TileSchedule,
    compute_gram,
    load_gram,
    make_schedule,
    run_distributed,
    save_gram,
    simulate_dataset,
    validate_schedule,
)
from .mps import (
    DEFAULT_TRUNC_BUDGET,
    MpsBatch,
    MpsState,
    SimStats,
    apply_gate,
    apply_one_qubit,
    apply_two_qubit,
    canonicalize,
    deserialize_state,
    init_state,
    inner_product,
    run_circuit,
    serialize_state,
    simulate_circuit,
    stats,
    to_statevector,
)
from .tensor import SvdResult, svd_truncated

__version__ = "0.1.0"
