"""CPU oracle for the traversal path -- TEST INFRASTRUCTURE ONLY.

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline
leg, as the checker; the product path (paper_2103_02309_b200) never imports
it.  See oracle/tetoracle.h for the pinning status.
"""
