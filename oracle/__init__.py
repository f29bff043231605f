"""TEST INFRASTRUCTURE ONLY: CPU oracles of the Picard hot path (see oracle.h)."""
