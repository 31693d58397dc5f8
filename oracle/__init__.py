"""CPU oracle for the MICKEY 2.0 path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package; the product package
``paper_1909_04750_b200`` never does.
"""
