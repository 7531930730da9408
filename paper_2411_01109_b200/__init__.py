"""B200-native (sm_100a) half-precision GNN hot path of HalfGNN (arXiv 2411.01109)."""
__version__ = "0.1.0"
