"""B200-native fBm heightmap path (arXiv 1610.03525) — placeholder, filled below."""
