"""CPU oracle (test infrastructure only; see oracle/fcdp_oracle.h)."""
