"""B200-native batched serving-scheduler simulator (drop-in for servesim's simulation path)."""
