"""CPU oracle for the particle time step — TEST INFRASTRUCTURE ONLY.

Importable from `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline legs; the product package never imports it.  See
`lagtrans_oracle.py` for the parity status and reference citations.
"""
