"""TEST INFRASTRUCTURE ONLY: CPU parity oracle (see oracle.cpp header)."""
