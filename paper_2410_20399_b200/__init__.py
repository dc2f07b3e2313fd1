"""paper_2410_20399_b200 — B200-native (sm_100a) ThunderKittens attention hot path."""
