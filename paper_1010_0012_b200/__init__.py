"""B200-native banded loopy-BP engine: a drop-in for the grid path of the
reference ``sparsebp`` package (arxiv/paper_1010_0012).

Model construction mirrors ``sparsebp.mrf``; ``run_sweeps`` /
``compute_beliefs`` / ``compute_max_marginals`` / ``map_labels`` mirror
``sparsebp.bp`` and run on hand-written sm_100a kernels (``libsbp.so``).
"""
from .model import (DensePotential, GridMrf, MrfModel, SparseTruncatedPotential, SweepSchedule,
                    build_grid_mrf, grid_edges, sparse_from_dense, truncated_linear_potential)
from .engine import (SEQUENTIAL, SYNCHRONOUS, BeliefTable, DegenerateBeliefError, DegenerateMessageError,
                     GridEngine, MessageStore, SweepStats, UnsafePotentialError,
                     compute_beliefs, compute_max_marginals, map_labels, run_sweeps)

from .stereo import (GrayImage, StereoParams, build_stereo_mrf, random_dot_pair,
                     stereo_unary_field)

__version__ = "0.1.0"
