"""CPU checkers for the eigen-update hot path. TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
import this package, and only as the checker / the timed CPU baseline — the
product path (paper_1706_00773_b200) never routes through it.
"""
