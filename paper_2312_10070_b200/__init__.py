"""B200-native differentiable Gaussian-splatting rasterizer (Gaussian-SLAM hot path)."""
