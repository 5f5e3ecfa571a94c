"""B200-native Mimose: input-aware activation checkpointing on sm_100a.

Host planner: include/mimose/*.hpp (drop-in for reference proj/include/mimose),
exposed through libmimose_host.so. Device side: libmimose_cuda.so (budget arena,
tcgen05 GEMMs, fused memory-bound kernels, layer executor, trainer).
"""
__version__ = "0.1.0"
