"""CPU oracle (test infrastructure only; see filterreg_oracle.py)."""
