"""CPU parity oracle for the sgweno hot path -- test infrastructure only (see oracle.py)."""
