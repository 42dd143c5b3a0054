"""B200-native backend for the fused block programs of Blockbuster (arXiv 2505.07829).

The reference `blockfuse` library (C++: IR, fusion rules, driver, and the
`execute(program, inputs, binding)` entry point, interpreter.hpp:478) stays
the drop-in API. This package holds what runs behind it:

  csrc/      hand-written sm_100a CUDA kernels (tcgen05/TMEM/TMA) + the C-ABI
  _lib.py    ctypes binding of include/bfgpu.h
  ops.py     torch-tensor front end (device memory/streams only)
  launcher.py row/head-sharded multi-GPU runner (torch.distributed plumbing)
"""
from ._lib import BfError, lib, lib_path  # noqa: F401

__all__ = ["BfError", "lib", "lib_path"]
