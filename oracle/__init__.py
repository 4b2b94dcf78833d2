"""CPU oracle for parity tests — test infrastructure only (see moe_oracle.py header)."""
