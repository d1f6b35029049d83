"""B200-native sparse-grid WENO5 hot path (arXiv 2007.10196).

``sgwg`` is the host-side mirror of the reference solver interface over the C
ABI ``include/sgwg.h`` implemented by the in-tree CUDA extension
``libsgwg.so`` (built by ``build.py``); ``configs`` holds BASELINE C1-C5.
"""
from . import configs  # noqa: F401
