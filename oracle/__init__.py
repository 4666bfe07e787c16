"""CPU oracle for parity tests -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker (never as the measured
or shipped path).  See octree_oracle.py for the restatement and its
reference citations; tests/test_oracle.py pins it to the reference's own
outputs (tests/golden/).
"""
