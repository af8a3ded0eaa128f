"""B200-native hierarchical Fock-exchange build (hot path of arXiv 1401.6961's reference).

Drop-in for the reference package's exchange path: the same entry points
(build_partition, build_pair_tree, build_matrix_tree, build_exchange_naive,
build_exchange_symmetric) backed by libhxf.so (hand-written sm_100a CUDA).
"""

from .basis import Atom, BasisSystem, GaussianShell, InvalidArgumentError, assign_offsets
from .inputs import DensityModel, SplitMix64, build_density, generate_cluster, hilbert_order
from ._native import LogicError, release_scratch
from .prep import hilbert_order_device
from .exchange import (CASE_LABELS, SymmetryCase, SymmetryCounters, TraversalCounters,
                       build_exchange_eightfold, build_exchange_naive, build_exchange_symmetric,
                       classify_quartet,
                       culled_task_bound, screening_test, symmetrize_final)
from .quadtree import (MatrixQuadtree, Partition, ShellPairNode, Span, build_matrix_tree,
                       build_pair_tree, build_partition, shell_overlap_matrix, transpose_view)

from .harness import RunConfig, load_report_schema, run_report, scaling_series

__version__ = "0.1.0"
