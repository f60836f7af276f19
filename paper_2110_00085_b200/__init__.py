"""B200-native Path Sorting + Path Recycling (arXiv 2110.00085)."""
