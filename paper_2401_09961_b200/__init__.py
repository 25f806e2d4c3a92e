"""B200-native L1 phase unwrapper (IRLS + PCG, arXiv 2401.09961)."""
