"""B200-native two-stage attention pipeline (drop-in for the reference `tilepipe` hot path)."""

__version__ = "0.1.0"
