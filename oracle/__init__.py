"""CPU oracle for the B200 hot path -- TEST INFRASTRUCTURE ONLY (see oracle.py)."""
