"""Test infrastructure: the CPU oracle (checker) for the control step.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this package.  The product package never does.
"""
