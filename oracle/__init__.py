"""CPU restatements of the reference PHG path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this package;
the product (paper_2604_05794_b200/) never does.
"""
