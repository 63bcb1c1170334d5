"""Independent CPU fp64 oracle for CoFEM — TEST INFRASTRUCTURE ONLY.

May be imported only by tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
`--impl reference`).  The product package paper_2310_00420_b200 never imports it; the two share
no code.  Every function cites the PAPER.md passage it follows; pins: tests/test_oracle_pins.py.
"""
from . import cofem  # noqa: F401
