"""TEST INFRASTRUCTURE ONLY -- the CPU parity checker and CPU baseline.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package; the product never does.
"""
