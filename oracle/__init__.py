"""CPU parity oracle for the voltseg preprocessing stage -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package.  The product package
paper_2403_16438_b200 never imports it.
"""
