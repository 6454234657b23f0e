"""Parity oracle (CPU restatement of the reference) — test infrastructure only.

Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg.  See alpha_oracle.py for the reference file:line map.
"""
