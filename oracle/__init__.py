"""Test infrastructure: the CPU checker for the DRK rasterizer hot path.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product
(``paper_2412_11752_b200``) never does: it fails loudly without its CUDA
extension.
"""
