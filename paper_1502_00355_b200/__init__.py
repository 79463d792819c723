"""B200-native Smart Laplacian smoothing (arXiv 1502.00355) — drop-in for the reference's
``trismooth`` Python package (proj/python/trismooth/__init__.py).

Everything here forwards to the compiled in-tree extension ``_trismooth`` (pybind11 over the
trismooth C++ API, whose ``smooth`` runs its passes on the GPU through ``libtsg.so``).
There is no Python or CPU fallback: if the extension is missing this import fails loudly —
build it with ``python -c "import __graft_entry__ as g; g.build()"`` (or ``make``).
"""
from __future__ import annotations

import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))

try:
    from . import _trismooth as _core
except ImportError as exc:  # pragma: no cover - exercised only on unbuilt trees
    raise ImportError(
        f"paper_1502_00355_b200: compiled extension not found in {_HERE} ({exc}); "
        "run `make` at the repository root (needs nvcc for sm_100a)"
    ) from exc

Mesh = _core.Mesh
build_mesh = _core.build_mesh
convert_layout = _core.convert_layout
generate_delaunay = _core.generate_delaunay
generate_grid = _core.generate_grid
quality_summary = _core.quality_summary
read_mesh = _core.read_mesh
smooth = _core.smooth
triangle_alpha = _core.triangle_alpha
write_mesh = _core.write_mesh

# B200 additions (not in the reference API)
DeviceMesh = _core.DeviceMesh
delaunay_arrays = _core.delaunay_arrays
grid_arrays = _core.grid_arrays
graded_arrays = _core.graded_arrays
triangulate = _core.triangulate
topology = _core.topology
bbox_diagonal = _core.bbox_diagonal
device_count = _core.device_count
quality_report = _core.quality_report
compute_all_qualities = _core.compute_all_qualities
reduce_vertex_minima = _core.reduce_vertex_minima
update_two_phase = _core.update_two_phase
write_binary = _core.write_binary
read_binary = _core.read_binary

LIB_DIR = _HERE

__all__ = [
    "Mesh",
    "build_mesh",
    "convert_layout",
    "generate_delaunay",
    "generate_grid",
    "quality_summary",
    "read_mesh",
    "smooth",
    "triangle_alpha",
    "write_mesh",
]
