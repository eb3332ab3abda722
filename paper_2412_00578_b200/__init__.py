"""B200-native (sm_100a) Speedy-Splat forward hot path: SnugBox/AccuTile rasterizer."""
