"""CPU oracle (test infrastructure only; see ofdm_oracle.py header)."""
