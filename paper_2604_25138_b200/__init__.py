"""B200 (sm_100a) hot path of LAKER (arXiv 2604.25138): regularized attention-
kernel regression (K + lambda I) alpha = y solved by PCG with the learned CCCP
preconditioner.  The product is liblaker.so (csrc/, C ABI in include/laker.h);
`laker` is its thin ctypes binding.  Importing `paper_2604_25138_b200.laker`
fails loudly when liblaker.so is missing -- there is no CPU fallback.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblaker.so")
