"""B200-native extreme-precision Hankel LDLT -> lambda_min (arXiv 1810.01478 hot path).

The product is ``libhankel_b200.so`` (sm_100a CUDA kernels + C++ host code behind
the C ABI in ``include/hankel_b200.h``); ``api`` is the ctypes binding used by
the tests and ``bench.py``.
"""
