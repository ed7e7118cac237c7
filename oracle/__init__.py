"""Parity oracle for the DistFlashAttn hot path (test infrastructure only)."""
