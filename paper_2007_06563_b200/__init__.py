"""B200-native HOBFLOPS hot path (arXiv 2007.06563): bitslice-parallel
custom-precision FP MAC inside CNN convolution, on sm_100a.

Submodules:
  gen   -- build-time circuit generator (AIG -> LOP3 mapping -> CUDA)
  hobf  -- ctypes binding of include/hobf.h (libhobf.so); imported lazily so
           the generator works on machines without the built library.
  inputs -- seeded synthetic inputs for the BASELINE configs (no method arithmetic).
"""
