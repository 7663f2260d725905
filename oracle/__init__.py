"""CPU oracle — TEST INFRASTRUCTURE ONLY (see oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and the
--impl reference arm) may import this package.  The product package
paper_2201_02789_b200 never does: its device path has no CPU fallback.
"""
