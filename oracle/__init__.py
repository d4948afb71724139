"""TEST INFRASTRUCTURE ONLY (the checker, never the product).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import anything from this package.
"""
