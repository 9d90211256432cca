"""CPU oracle for the ROCKET transform — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package, as the checker or the timed CPU baseline; the product
path (paper_2601_17091_b200) never does.
"""
