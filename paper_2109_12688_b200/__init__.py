"""B200-native accelerated-ADMM diffeomorphic registration (arXiv 2109.12688 path)."""
