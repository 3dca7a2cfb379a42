"""CPU oracle — TEST INFRASTRUCTURE ONLY (see vit_oracle.py header).  Parity unpinned:
the reference ships no code for the token-adapted forward."""
