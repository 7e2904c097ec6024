"""CPU oracle of the quantum-kernel hot path (test infrastructure only; see mps_oracle.py)."""
