"""TEST INFRASTRUCTURE ONLY: parity oracle (see oracle/oracle.py)."""
