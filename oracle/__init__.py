"""CPU oracle for the rAPDB hot path -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, as the checker or the timed CPU
baseline.  Pinned bit-for-bit against the real reference's golden traces
(tests/golden/make_golden.py, tests/test_oracle_pin.py).
"""
