"""B200-native (sm_100a, FP64) modal ring-source potentials: direct sum and the cylindrical
quadtree FMM of arXiv 2301.01179.  The compute path is libcylfmm.so (csrc/, include/cylfmm.h);
this package is its ctypes binding plus the seeded input generators."""
from .cylfmm import (MILLER_ACCURATE, MILLER_PAPER, TRUNC_DOUBLE, TRUNC_SINGLE, CylFMMError,  # noqa: F401
                     FMMConfig, Plan, direct, direct_enqueue, direct_workspace_bytes,
                     greens_batch, header_functions, lib,
                     partition_fields, select_params, tensor_batch, tree_sort)
