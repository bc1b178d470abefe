"""CPU oracle for the MLS-MPM substep path (test infrastructure only; see mpm_oracle.py)."""
