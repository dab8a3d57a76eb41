"""GATE max-min-fair TE solver, B200-native."""
