"""Benchmark/test input generation (not part of the product package)."""
