"""B200-native drop-in for the work-partitioned hot path of hybridbench."""
