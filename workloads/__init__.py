"""Seeded synthetic inputs for the tetrahedral CT projector (arXiv:1908.06909).

This package is shared by the oracle tests, the GPU tests and ``bench.py``.
It only *generates inputs* (meshes, scan geometries, attenuation / detector
values); it holds none of the method's arithmetic (no ray/tet predicates, no
chords, no traversal).  Every generator is deterministic in its ``seed``.

The workload shapes follow SURVEY.md §8(d) (configs c1..c5) which in turn
mirror the paper's experiments: box-hulled CAD-like meshes with nested
materials of attenuation 0/1/2 (§3.1), cone beam circular
trajectories with equidistant angles, and high-aspect-ratio
("sliver") meshes for the precision study (§3.3).
"""
from .meshes import Mesh  # noqa: F401
