"""CPU oracle for the DynaSpec dynamic drafter head — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path never does.
"""
