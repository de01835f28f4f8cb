"""Test infrastructure: the CPU oracle of the reference algorithm (see bccb_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline / reference legs
import this package.  The product (paper_2509_13592_b200) never does.
"""
