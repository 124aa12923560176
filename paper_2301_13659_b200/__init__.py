"""B200-native SDNN hot path of Spyker (arXiv 2301.13659).

The product is libspk.so (C ABI, include/spk.h; CUDA kernels for sm_100a in
csrc/).  ``spk`` is its ctypes binding and ``network`` composes the calls into
the paper's training / inference steps for the configs in configs/.
"""
