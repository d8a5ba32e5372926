"""B200-native DynaSpec dynamic drafter LM head (arXiv 2510.13847).

The product is the C-ABI library libdynaspec.so (include/dynaspec.h) built from csrc/;
`dynaspec` is its thin ctypes binding.  Import `paper_2510_13847_b200.dynaspec` to use it.
"""
__all__ = ["dynaspec", "build"]
