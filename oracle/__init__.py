"""CPU oracle (test infrastructure only; see scattermlp_oracle.py header)."""
