"""B200-native OneRec inference hot path (encoder + MoE decoder + 3-level
semantic-ID beam search) behind the reference's encode / generate surface.

The compute runs in liborx.so (hand-written sm_100a CUDA: tcgen05/TMEM/TMA
GEMMs, flash attention, MoE routing, fused log-softmax + top-k beam pruning);
this package is the host-side mirror of the reference API.
"""
from ._lib import LIB_PATH, OrxError, lib  # noqa: F401
from .policy import (GeneratedItem, GenerationRequest, InteractionFeature, PolicyConfig, PolicyModel,  # noqa: F401
                     SemanticTrie, SynthBatch, UserBatch, UserContext, Weights, compress_lifelong_batch,
                     ep_place, moe_layers, policy_scorer, validate_request)

__all__ = ["PolicyConfig", "PolicyModel", "UserContext", "InteractionFeature", "GenerationRequest",
           "GeneratedItem", "SemanticTrie", "SynthBatch", "UserBatch", "Weights", "policy_scorer",
           "validate_request", "compress_lifelong_batch", "ep_place", "moe_layers", "OrxError", "lib", "LIB_PATH"]
