"""B200-native (sm_100a) Mamba-2 SSD inference hot path.

Drop-in for the reference engine's hot path (ssd_engine/__init__.py:7-24):
same names and signatures for the model API — ModelConfig, ElemPolicy,
ModelParams/LayerParams, random_init, prefill, block_forward, decode_step,
generate, cache_init, Mamba2Cache, ssd_forward — with torch device tensors
in and out.  Every FLOP runs in hand-written CUDA (libssd200.so, C ABI in
include/ssd200.h); there is no CPU fallback.
"""

from .bundle import (
    BundleError,
    FormatVersionError,
    MissingTensorError,
    PayloadError,
    TensorShapeError,
    load_bundle,
    load_bundle_host,
    save_bundle,
    tensor_names,
    tensor_shape,
)
from .cache import GenerationResult, Mamba2Cache
from .config import MODEL_SIZES, ElemPolicy, ModelConfig, named_config
from .cost import (
    DeviceSpec,
    cache_bytes,
    decode_step_bytes,
    flops_decode,
    flops_decode_step,
    flops_prefill,
    hbu,
    measured_b200,
    mfu,
    n_params,
)
from .decode import GreedyDecoder, cache_init, decode_step, generate
from .model import PolicyAudit, block_forward, prefill
from .params import (
    LayerParams,
    ModelParams,
    decay_coefficient,
    from_reference,
    random_init,
    random_init_host,
    synthetic_init,
)
from .ssd import ChunkPlan, SsdInputs, SsdOutputs, plan_chunks, ssd_forward

__version__ = "0.1.0"

__all__ = [
    "BundleError",
    "FormatVersionError",
    "MissingTensorError",
    "PayloadError",
    "TensorShapeError",
    "load_bundle",
    "load_bundle_host",
    "save_bundle",
    "tensor_names",
    "tensor_shape",
    "ChunkPlan",
    "DeviceSpec",
    "ElemPolicy",
    "GenerationResult",
    "GreedyDecoder",
    "LayerParams",
    "MODEL_SIZES",
    "Mamba2Cache",
    "ModelConfig",
    "ModelParams",
    "PolicyAudit",
    "SsdInputs",
    "SsdOutputs",
    "block_forward",
    "cache_bytes",
    "cache_init",
    "decay_coefficient",
    "decode_step",
    "decode_step_bytes",
    "flops_decode",
    "flops_decode_step",
    "flops_prefill",
    "from_reference",
    "generate",
    "hbu",
    "measured_b200",
    "mfu",
    "n_params",
    "named_config",
    "plan_chunks",
    "prefill",
    "random_init",
    "random_init_host",
    "ssd_forward",
    "synthetic_init",
]
