"""CPU fp64 oracle for the SPLAT sparse-MHSA hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import it.
"""
