"""B200-native Parm MoE-layer hot path (arXiv 2407.00599)."""
