"""CPU oracle package — TEST INFRASTRUCTURE ONLY (see fsm_oracle.py header).
Importable only from tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg; never from the product package."""
