"""Synthetic workload fixture of the benchmark and the parity tests (not the product)."""
