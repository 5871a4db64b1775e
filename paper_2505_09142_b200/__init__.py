"""B200-native (sm_100a) ISRTF re-predict + select hot path of ELIS (arXiv 2505.09142).

The product is the C-ABI library ``libelis.so`` (include/elis.h) built from
``csrc/``; ``binding`` is its thin ctypes binding and ``inputs`` the seeded
synthetic input generator.  Importing the package loads nothing heavy.
"""
__all__ = ["binding", "inputs"]
