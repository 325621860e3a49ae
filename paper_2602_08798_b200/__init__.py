"""B200-native RNS-BFV backend for the CryptoGen (arXiv 2602.08798) HE hot path."""
