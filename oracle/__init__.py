"""CPU oracle for the twofold hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs import this package; the product (paper_1502_05216_b200) never
does.
"""
