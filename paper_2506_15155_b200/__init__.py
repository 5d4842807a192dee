"""B200-native KV-traffic hot path of eLLM (arXiv 2506.15155).

The product is libellm.so (include/ellm.h): chunk pool + vtensor (VMM), chunk tables,
kv_append, paged decode attention, deflate / inflate / migrate. ``ellm`` is its ctypes
binding; ``shard`` holds the KV-head sharding helpers for N GPUs.
"""
from . import ellm  # noqa: F401  (raises ImportError if libellm.so is missing)
