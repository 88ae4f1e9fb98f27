"""B200-native HTM Spatial Pooler hot path (arxiv 1608.01966).

``SpatialPooler`` wraps the C ABI of ``include/sp.h`` (``libsp.so``, CUDA
kernels for sm_100a).  See DESIGN.md.
"""
from .sp import (SpatialPooler, Encoder, synth_bgr_frames, SpConfig, SpError, make_config, plan, init_pools_host, synth_frames,
                 lib, ABI_SYMBOLS, SP_OK, SP_E_CONFIG, SP_E_ARG, SP_E_SHAPE, SP_E_CUDA, SP_E_OOM,
                 SP_E_STATE, SP_PATH_AUTO, SP_PATH_PER_INPUT, SP_PATH_BATCHED,
                 SP_FLAG_RECORD_OVERLAPS, SP_FLAG_LEARN_GRID, SP_FLAG_FULL_LEARNING, SP_FLAG_PATCH_GATHER, SP_FLAG_PATCH_TENSOR, SP_LEARN_PER_INPUT, SP_LEARN_CLUSTER,
                 SP_LEARN_GRID, learn_path_name)

__all__ = ["SpatialPooler", "Encoder", "synth_bgr_frames", "SpConfig", "SpError", "make_config", "plan", "init_pools_host",
           "synth_frames", "lib", "ABI_SYMBOLS"]
