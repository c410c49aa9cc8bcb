"""Mapping orchestration under the reference's module name (mapbuild.py:38-99).

``build_map_from_fields`` and ``DepthBuildReport`` live in ``depthbuild`` next
to the triangulation kernels they drive; this module re-exports them so
``visloc.mapbuild`` imports resolve.  The synthetic-scene helpers
(``synthetic_map`` / ``synthetic_query_jobs``, mapbuild.py:101-164) wrap the
reference's ``visloc.synth`` scene generator, which is not rebuilt (SURVEY §2:
fixture helper, out of scope).
"""

from .depthbuild import DepthBuildReport, build_map_from_fields

__all__ = ["DepthBuildReport", "build_map_from_fields"]
