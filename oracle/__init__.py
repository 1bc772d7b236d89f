"""GACE probe oracle -- TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py
(cpu_baseline and --impl reference).  The product package never imports it;
tests/test_boundary.py checks that."""
from . import reference  # noqa: F401
