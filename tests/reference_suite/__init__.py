"""The reference test suite run against this package (see conftest.py)."""
