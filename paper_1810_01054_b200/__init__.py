"""B200-native differentiable MLS-MPM step (ChainQueen, arXiv 1810.01054).

The compute path is the CUDA library ``libmpm.so`` (sm_100a) behind the C ABI declared in
``include/mpm.h``; ``paper_1810_01054_b200.mpm`` is its thin ctypes binding.  Importing
this package does not load the library; ``mpm.load()`` does, and raises if it is missing.
"""
__all__ = ["mpm", "scenes"]
