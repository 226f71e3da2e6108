"""paper_2604_26074_b200 — B200-native DAK decode hot path (arxiv 2604.26074).

The product is the C-ABI library ``libdak.so`` (include/dak.h) built from ``csrc/`` for sm_100a;
``dak`` is its thin ctypes binding. Nothing in this package imports the CPU oracle.
"""
__all__ = ["dak"]
