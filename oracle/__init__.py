"""CPU ORACLE — test infrastructure only.

Plain numpy reference of the adaptive FAS V-cycle (mg_oracle) and of the lattice
Green's functions (lgf).  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the CUDA product
path (paper_2512_08555_b200) must never import it, and shares no code with it.
Pinned by tests/test_oracle_*.py (closed forms, literature constants, invariants).
"""
