"""TEST INFRASTRUCTURE ONLY: checkers for the parity tests (C restatement + the compiled reference)."""
