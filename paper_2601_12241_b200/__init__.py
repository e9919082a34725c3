"""paper_2601_12241_b200 — B200-native what-if evaluator for power-aware
prefill/decode disaggregation (arXiv 2601.12241).

The product is the CUDA library ``libpadsim.so`` (C ABI: include/padsim.h);
``binding`` is its thin ctypes binding.  Nothing here imports ``oracle``.
"""
from .binding import (Context, PadsimError, enumerate_pool_uniform,  # noqa: F401
                      evaluate_allocations, load, replay_records)

__all__ = ["Context", "PadsimError", "enumerate_pool_uniform", "evaluate_allocations", "load",
           "replay_records"]
