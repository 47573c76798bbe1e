"""Seeded synthetic inputs for the five BASELINE.json configs (input
generation only; neither the product nor the oracle)."""
