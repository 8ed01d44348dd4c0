"""B200-native multi-level covariance assembly (arXiv:1701.00285 hot path).

The compute path is libmlk.so (hand-written sm_100a CUDA behind the C ABI in include/mlk.h);
`paper_1701_00285_b200.mlk` is its ctypes binding and raises ImportError if the in-tree
library is missing.  There is no CPU fallback.  `paper_1701_00285_b200.build` compiles it.
"""
