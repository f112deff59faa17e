"""B200-native (sm_100a) MISA / DSA indexer — drop-in for the reference ``misa`` indexer path."""
__version__ = "0.1.0"
