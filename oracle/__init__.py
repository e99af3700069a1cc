"""Test infrastructure: CPU restatement of the reference's hot path (see moe_oracle.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import this package,
and only as the checker / CPU baseline — never as the product path.
"""
