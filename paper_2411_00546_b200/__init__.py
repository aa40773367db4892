"""B200-native RASPEN hot path (package init filled in below)."""
