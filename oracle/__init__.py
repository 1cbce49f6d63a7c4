"""CPU oracle and baseline port — test infrastructure only (see ftar_oracle.py)."""
