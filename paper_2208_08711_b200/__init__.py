"""B200-native batched L3 decoder (arXiv 2208.08711) — hot path only.

The compute lives in ``libl3_b200.so`` (hand-written sm_100a CUDA, C ABI in
``include/l3.h``). This package is its thin Python binding (:mod:`.l3`) plus
buffer-management helpers (:mod:`.api`). There is no CPU fallback.
"""
from . import l3  # noqa: F401
from .api import (IMAGENET_MEAN, IMAGENET_STD, BatchDecoder, encode_batch, normalize_constants,  # noqa: F401
                  pack_files)

__all__ = ["l3", "BatchDecoder", "encode_batch", "normalize_constants", "pack_files", "IMAGENET_MEAN",
           "IMAGENET_STD"]
