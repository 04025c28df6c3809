"""Seeded synthetic input generators (meshes, magnetisation fields, configs).

This package is shared by the oracle (``oracle/``), the product binding
(``paper_2409_13958_b200``), the tests and ``bench.py``.  It holds NONE of
the method's arithmetic: no PBC detection, no operators, no Green's
functions -- only geometry generation (voxel masks split into Kuhn
tetrahedra, with seeded jitter) and seeded magnetisation fields.
The input recipe is documented in DESIGN.md section "Input recipe".
"""
from .meshes import Mesh, kuhn_voxel_mesh
from .configs import CONFIGS, make_config
from .fields import m_uniform, m_random, m_smooth
