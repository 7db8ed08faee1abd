"""B200-native batched early-exit decode step (HELIOS, arXiv 2504.10724).

The product is native: ``libeeb.so`` (sm_100a CUDA kernels behind the C ABI in
``include/eeb/eeb.h``) and the host C++ engine in ``include/eeserve/``.  This
package holds their sources (``csrc/``), the in-tree build, and a ctypes
binding used by the tests and the benchmark.
"""
