"""TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package. The product library (paper_1802_04799_b200)
never imports, links or calls anything here.
"""
