"""B200-native sliding-mesh DGSEM right-hand side (arXiv 2008.04356 reference)."""
