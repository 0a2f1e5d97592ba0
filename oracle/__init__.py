"""ORACLE — test infrastructure only (see oracle/README.md).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline; the product (paper_2508_08343_b200) never does.
"""
