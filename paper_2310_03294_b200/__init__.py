"""B200-native DistFlashAttn hot path: sequence-parallel causal attention
(arxiv 2310.03294) behind the reference's distattn API.

Submodules mirror the reference headers in /root/reference/proj/include/distattn:
  flashcore  — block_attn_update / rescale / finalize / backward_aux / block_attn_backward
  schedule   — ring and load-balanced schedules, validate, idle/speedup arithmetic
  runtime    — make_shards, run_forward, run_backward (P workers on one device,
               or one process per GPU over NCCL)
  errors     — the reference exception taxonomy
All compute goes through libdistattn_b200.so (sm_100a). There is no CPU path.
"""
from .errors import (ConfigError, DegenerateRowError, Error, ScheduleError, ShapeError,  # noqa: F401
                     StateError)

__all__ = ["flashcore", "schedule", "runtime", "errors"]
