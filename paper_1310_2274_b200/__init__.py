"""B200-native (sm_100a) hot path of Aggregate Risk Analysis with secondary
uncertainty (Varghese & Rau-Chaplin, arXiv 1310.2274).

- ``csrc/``   : CUDA kernels + the C ABI of ``libara.so`` (include/ara.h)
- ``ara``     : thin ctypes binding with the ABI's names (marshalling only)
- ``build``   : in-tree nvcc build for sm_100a
"""
__version__ = "0.1.0"
