"""TEST INFRASTRUCTURE ONLY: CPU oracle of the design-update path (see oracle.py)."""
