"""B200-native Evoformer hot path (FastFold, arXiv 2203.00854).

Drop-in for the reference package's Evoformer block / module API
(/root/reference/pkg/src/evoplan/__init__.py:13-72, hot-path subset):
``EvoConfig``, ``param_shapes``, ``init_block_params``, ``params_to_json``,
``params_from_json``, ``evoformer_block`` and its sub-modules,
``dap_evoformer_block`` with ``DeviceMesh`` / ``CommLedger``, the reference's
exception classes, the GPU executor of the reference's AutoChunk plans
(``execute_chunked`` with ``graph_from_json`` / ``plan_from_json``) and the
measured overlap timeline (``simulate_schedule``, ``measure_dap_forward``).  Compute runs in libevo.so (sm_100a CUDA,
include/evo.h); there is no CPU fallback.
"""

from .config import (
    EvoConfig,
    init_block_params,
    param_shapes,
    params_from_json,
    params_to_json,
)
from .errors import (
    DimensionError,
    DomainError,
    EvoplanError,
    KernelError,
    MeshError,
    NativeLibraryMissing,
    ShardError,
)

__version__ = "0.1.0"


def __getattr__(name):
    # heavy (torch / CUDA) modules load lazily so that `import` works on CPU-only hosts
    if name in ("evoformer_block", "msa_row_attention", "msa_row_bias", "msa_row_attention_with_bias",
                "msa_col_attention", "transition", "outer_product_mean", "outer_product_mean_from_projections",
                "tri_update_outgoing", "tri_update_incoming", "pair_attention_row", "pair_attention_col",
                "fused_softmax_mask_bias", "fused_softmax_mask_bias_raw", "layernorm", "layernorm_raw",
                "softmax_raw", "sigmoid_raw", "relu_raw", "EvoformerStack", "BlockParams", "GraphedStep",
                "EvoformerBlockFunction", "_attention_core", "_triangle_projections", "_triangle_finish",
                "_pair_bias_fn", "_check_msa", "_check_pair", "check_supported"):
        from . import evoformer
        return getattr(evoformer, name)
    if name in ("dap_evoformer_block", "DeviceMesh", "CommLedger", "predict_block_ledger", "dap_block"):
        from . import dap
        return getattr(dap, name)
    if name in ("execute_chunked", "graph_from_json", "graph_to_json", "plan_from_json", "plan_to_json",
                "ByteTracker"):
        from . import autochunk
        return getattr(autochunk, name)
    if name == "precise":  # reference-precision parity mode (fp32 storage, three-term bf16 tensor-core products)
        import importlib
        return importlib.import_module(".precise", __name__)
    if name in ("TimelineEvent", "simulate_schedule", "events_from_json", "events_to_json", "measure_dap_forward",
                "overlap_report"):
        from . import timeline
        return getattr(timeline, name)
    raise AttributeError(name)
