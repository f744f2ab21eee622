"""CPU oracle (test infrastructure only) -- see tailorkv_oracle.py."""
