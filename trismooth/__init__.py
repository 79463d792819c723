"""Drop-in ``import trismooth`` for code written against the reference package
(proj/python/trismooth/__init__.py): re-exports the B200 implementation."""
from paper_1502_00355_b200 import *  # noqa: F401,F403
from paper_1502_00355_b200 import __all__  # noqa: F401
from paper_1502_00355_b200 import (  # noqa: F401  B200 additions
    DeviceMesh, bbox_diagonal, delaunay_arrays, device_count, graded_arrays, grid_arrays, topology,
    triangulate)
