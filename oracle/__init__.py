"""float64 CPU oracle of the DMoE layer — TEST INFRASTRUCTURE ONLY (see oracle/oracle.py)."""
