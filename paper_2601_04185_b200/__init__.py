"""B200-native LO-RANSAC PnP for ImLoc (arxiv 2601.04185) — drop-in for ``visloc``.

The hot path of the reference package (``visloc.posest.ransac_pnp``,
``visloc.localizer.lift`` and their callees) re-built as sm_100a CUDA
kernels behind a C ABI (``include/visloc_b200.h``).  Module layout and names
mirror the reference so ``visloc`` call sites keep working:

* ``posest``   — RansacConfig, PoseEstimate, ransac_pnp (+ batched), msac_score
* ``p3p``      — p3p_solve, p3p_solve_batch, sample_minimal_sets
* ``refine``   — refine_pose, TruncatedLoss, CauchyLoss
* ``geometry`` — CameraIntrinsics, Pose, pose_error
* ``localizer`` / ``matchio`` / ``retrieval`` — lift, localize, IMLC fields, top-K retrieval
* ``mapstore`` / ``depthbuild`` — depth codecs, dense depth triangulation (mapping side)
* ``dist`` — query sharding and the hypothesis-split modes over torch.distributed
"""

from .geometry import CameraIntrinsics, Pose, pose_error  # noqa: F401
from .posest import (  # noqa: F401
    Match2D3D,
    PoseEstimate,
    RansacConfig,
    UnderConstrainedError,
    msac_score,
    ransac_pnp,
    ransac_pnp_batch,
    ransac_pnp_device,
    ransac_pnp_host,
    ransac_pnp_stream,
    required_iterations,
)

__version__ = "0.1.0"
