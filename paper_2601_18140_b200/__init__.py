"""B200-native RTeAAL Sim hot path: lane-batched per-cycle evaluation of a
levelized RTL dataflow graph as the paper's cascade of extended Einsums
(PAPER.md Cascade 1), behind the C ABI of include/rtlsim.h.

The product path is ``rtlsim`` (ctypes over lib/librtlsim.so); it never
imports ``oracle`` and has no CPU fallback.
"""
__all__ = ["rtlsim"]
