"""B200-native tolerance-controlled H-matrix product (drop-in for the reference ``hmat``).

The public names mirror ``hmat`` (``/root/reference/pkg/src/hmat/__init__.py:3-24``) for
the product path: trees, the H-matrix container, truncation policies, compressor choice,
``MultiplyConfig`` and ``hmult_new``.  The product itself runs in ``libhx.so``
(``include/hx.h``): flat term lists built by a C++ planner, FP64 DMMA term formation and
block materialization, per-block QR / Jacobi-SVD recompression on sm_100a.
"""

from .clustering import (FAR, INNER, NEAR, BlockClusterTree, BlockNode, Cluster,
                         ClusterTree, admissible, build_block_cluster_tree,
                         build_cluster_tree, dump_tree, sparsity_constant)
from .compressors import CompressorKind
from .hmatrix import (HMatrix, frobenius_norm, load_hmatrix, save_hmatrix, to_dense,
                      tree_fingerprint)
from .lowrank import EpsRank, FixedRank, LowRank, select_rank, zero_lowrank
from .multiply import MultiplyConfig, MultReport, hmult_new, hmult_traditional
from .assembly import KERNELS, assemble_hmatrix

__version__ = "0.1.0"
