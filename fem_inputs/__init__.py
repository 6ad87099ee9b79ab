"""Seeded synthetic inputs shared by the oracle tests, the CUDA-path tests and bench.py.

This package generates meshes (coordinates, connectivity, boundary-facet sets), effective
states and the per-config problem descriptions (weak-form ids + parameter values).  It holds
none of the method's arithmetic: no shape functions, quadrature, geometry, integrands or
sparsity logic live here ("input recipe").  Both `oracle/` and
`paper_2111_03541_b200/` consume its plain numpy arrays; neither is imported from here.
"""
from .meshgen import Mesh, tri_square, hex_box, tet_box, perturb_and_permute, facets_on_plane  # noqa: F401
from .configs import CONFIGS, make_config, make_state, Problem, Term  # noqa: F401
