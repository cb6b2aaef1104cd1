"""B200-native usFFT detection step (arXiv 2109.04131): C-ABI library libusfft.so + binding.

Layout: csrc/ (CUDA kernels for sm_100a and the C-ABI of include/usfft.h), _native.py (ctypes
loader, no fallback), binding.py (same names as the C-ABI), dist.py (multi-GPU exchange),
driver.py (Alg. 1 loop over the calls), build.py (nvcc build of libusfft.so).
"""
