"""B200-native ZeRO++ communication-reduction hot path (arXiv 2306.10209).

Drop-in for the hot-path API of the reference package ``zerosim``
(zs/__init__.py:10-132): the codec (``QuantConfig``, ``quantize``,
``dequantize``, ``fused_dequant_reduce_quant``), the codec protocol
(``BlockCodec``, ``PassthroughCodec``), the collectives (``all_gather_qwz``,
``all_gather_baseline`` incl. hpZ groups, ``reduce_scatter_ring``,
``reorder_mapping``, ``qgz_2hop``), partitions and errors -- computed by
hand-written sm_100a kernels in ``libzpp.so``.  ``paper_2306_10209_b200.dist``
runs the same collectives across GPUs (one process per GPU, NVLink P2P).
"""

from .errors import (
    ConfigError,
    DeviceError,
    IntegrityError,
    PlanError,
    ProtocolError,
    SimError,
    ValidationError,
)
from .quantizer import (
    FlatTensor,
    QuantConfig,
    QuantErrorStats,
    QuantizedTensor,
    dequant_reduce,
    dequantize,
    fused_dequant_reduce_quant,
    quant_error_stats,
    quantize,
)
from .topology import (
    INTER,
    INTRA,
    ClusterTopology,
    CollectiveTrace,
    LatencyEstimate,
    LinkParams,
    PhaseStats,
    TrafficLedger,
    estimate_latency,
    normalized_cross_node_volume,
    optimal_stages,
    pipelined_seconds,
)
from .partitioner import PartitionSpec, build_partitions
from .collectives import (
    BlockCodec,
    GatherResult,
    PassthroughCodec,
    ReduceResult,
    ReorderPermutation,
    WirePayload,
    all_gather_baseline,
    all_gather_qwz,
    as_codec,
    qgz_1hop,
    qgz_2hop,
    reduce_scatter_ring,
    reduce_scatter_ring_naive_quant,
    reorder_mapping,
)
from .accounting import BWD_GATHER, FWD_GATHER, GRAD_REDUCE, StepConfig, step_volumes

__version__ = "0.1.0"

__all__ = [
    "SimError", "ValidationError", "ConfigError", "IntegrityError", "PlanError", "ProtocolError", "DeviceError",
    "FlatTensor", "QuantConfig", "QuantizedTensor", "QuantErrorStats", "quantize", "dequantize",
    "fused_dequant_reduce_quant", "dequant_reduce", "quant_error_stats",
    "INTRA", "INTER", "ClusterTopology", "TrafficLedger", "CollectiveTrace", "PhaseStats",
    "normalized_cross_node_volume", "LinkParams", "LatencyEstimate", "estimate_latency", "pipelined_seconds",
    "optimal_stages",
    "PartitionSpec", "build_partitions",
    "BlockCodec", "PassthroughCodec", "WirePayload", "as_codec", "GatherResult", "ReduceResult",
    "ReorderPermutation", "all_gather_baseline", "all_gather_qwz", "reduce_scatter_ring", "reorder_mapping",
    "qgz_2hop", "qgz_1hop", "reduce_scatter_ring_naive_quant",
    "StepConfig", "step_volumes", "FWD_GATHER", "BWD_GATHER", "GRAD_REDUCE",
    "__version__",
]
