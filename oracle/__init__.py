"""CPU oracles for the LP hot path — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py)."""
