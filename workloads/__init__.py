"""Seeded synthetic workloads (input generation only; not product code)."""
