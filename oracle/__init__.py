"""Test-infrastructure oracle (CPU restatement of the reference hot path).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this package.  The product (paper_2305_13925_b200) never does.
"""
