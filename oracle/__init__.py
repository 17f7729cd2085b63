"""CPU oracle — test infrastructure only (see helm_oracle.py). Not part of the product."""
