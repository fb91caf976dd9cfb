"""B200-native batched LRU / T-LRU prefix-cache eviction simulator (arXiv 2510.15152)."""
