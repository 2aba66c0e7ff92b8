"""B200-native redistributed polynomial-CNN forward and weight redistribution.

Drop-in for the hot path of ``levnet`` (arXiv 2509.22857 reference): the
graph API of ``levnet.graph`` and the transform API of ``levnet.transforms``,
executed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/pcnn.h`` (``libpcnn.so``).
"""

from .graph import (  # noqa: F401
    AddNode, AvgPoolNode, BatchNormNode, BiPoolNode, ConvNode, FlattenNode,
    GraphError, InputNode, LinearNode, LocalPoolNode, ModelFormatError,
    ModelGraph, Node, OutputNode, PolyActNode, PolySkipNode, PS_KEYS,
    load_model, save_model,
)

__version__ = "0.1.0"
