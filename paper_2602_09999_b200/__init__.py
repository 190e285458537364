"""B200-native Faster-GS 3DGS training hot path behind the reference's tilesplat API."""
