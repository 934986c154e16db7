"""B200-native primitive layer of arXiv 2603.18695 (KernelForge.jl): scan,
mapreduce and semiring matvec / vecmat over arbitrary element types and
associative operators, as hand-written sm_100a kernels behind the reference's
C++ API (include/forge/*.hpp) and its C-ABI (include/forge.h).

Python entry points:
  forge    — the reference-shaped API (Machine, View, Workspace, scan, ...)
  dev      — device-pointer calls on torch tensors (stream-ordered)
  sharded  — multi-GPU sharding over torch.distributed (NCCL)
Importing this package loads libforge.so; a missing library raises ImportError
(there is no CPU fallback).
"""
from __future__ import annotations

from . import capi

capi.load()

from . import forge  # noqa: E402,F401

__all__ = ["capi", "forge"]
