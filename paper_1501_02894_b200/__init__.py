"""B200-native MNS fractal coder core."""
