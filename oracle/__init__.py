"""CPU oracle package -- TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).

Imported only by tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
"""
