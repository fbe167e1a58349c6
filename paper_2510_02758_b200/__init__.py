"""B200-native TokenFlow KV-movement hot path (arxiv 2510.02758)."""
