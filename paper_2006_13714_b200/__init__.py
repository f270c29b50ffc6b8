"""paper_2006_13714_b200 -- B200-native Self-Convolution block matching (arXiv 2006.13714).

The CUDA library (``libscbm.so``) is loaded lazily by :mod:`paper_2006_13714_b200.bm`;
importing this package (e.g. for :mod:`.synth`) does not need a GPU.
"""
__all__ = ["synth"]
