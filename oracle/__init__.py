"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the B200 engine.

Nothing in the product package imports this directory.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference arms use it,
and only as the checker or the reported CPU baseline.
"""
