"""B200-native (sm_100a) hybrid treecode/FMM of Yokota & Barba (arxiv 1108.5815).

The compute path is libfmm.so (paper_1108_5815_b200/csrc, C ABI in include/fmm.h); this package
is only the ctypes binding. There is no CPU fallback: importing `FMM` without the built library
raises.
"""
from .fmm import (DIRECT, FMM_MODE, HYBRID, TREECODE, FMM, FmmError, lib_path,  # noqa: F401
                  load_library)
