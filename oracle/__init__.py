"""CPU oracle (TEST INFRASTRUCTURE ONLY -- see oracle.c header)."""
