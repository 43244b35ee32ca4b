"""TEST INFRASTRUCTURE ONLY: CPU checkers for the DES MoE hot path (see oracle.py)."""
