"""CPU restatement of the reference algorithm — test infrastructure only (see oracle.py)."""
