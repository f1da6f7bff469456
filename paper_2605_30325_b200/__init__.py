"""B200-native hot path of Veda (arXiv 2605.30325): distilled tile-sparse attention.

The compute lives in libveda.so (hand-written sm_100a CUDA behind the C ABI in
include/veda.h); ``veda`` is its ctypes binding; ``synth`` draws seeded inputs;
``shard`` is the head-sharding plan for multi-GPU runs.
"""
from . import synth  # noqa: F401

__all__ = ["veda", "synth", "shard", "build"]
