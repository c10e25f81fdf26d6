"""TEST INFRASTRUCTURE — CPU checkers (3D restatement + reference shim). Not product code."""
