"""TEST INFRASTRUCTURE ONLY: parity checkers (see binding.py)."""
