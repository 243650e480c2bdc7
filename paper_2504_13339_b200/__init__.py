"""B200-native differentiable VEG rasteriser (drop-in for vegsplat's render/train path)."""
