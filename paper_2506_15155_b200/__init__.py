"""B200-native KV-traffic hot path of eLLM (arXiv 2506.15155).

The product is libellm.so (include/ellm.h): chunk pool + vtensor (VMM), chunk tables,
kv_append, paged decode attention, deflate / inflate / migrate. ``ellm`` is its ctypes
binding (importing it raises if libellm.so is missing: there is no CPU fallback);
``shard`` holds the KV-head sharding helpers for N GPUs; ``build`` compiles the library.
"""
import importlib


def __getattr__(name):
    if name in ("ellm", "shard", "build"):
        return importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
