"""B200-native banded loopy-BP engine (drop-in for the reference `sparsebp` grid path)."""
from .model import (DensePotential, GridMrf, SparseTruncatedPotential, build_grid_mrf,
                    grid_edges, sparse_from_dense, truncated_linear_potential)
