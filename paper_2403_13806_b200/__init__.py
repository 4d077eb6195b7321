"""B200-native RadSplat render-and-prune hot path (arXiv 2403.13806).

A drop-in for the reference package's renderer / pruning / visibility API
(``fieldsplat.render``, ``fieldsplat.pruning``, ``fieldsplat.visibility``),
computed by hand-written sm_100a CUDA kernels behind the C ABI in
``include/radsplat.h``. There is no CPU fallback: the compute entry points
raise ``NativeUnavailable`` without the built library or a CUDA device.

Submodules are imported lazily so that host-only pieces (types, synthetic
scenes, clustering) import on machines without CUDA.
"""

from .core import (GaussianScene, ImageBuffer, InvalidParameterError, InvalidSceneError, PinholeCamera,
                   StaleTableError, look_at_camera)

__version__ = "0.1.0"

_LAZY = {
    "RasterizeOptions": "render", "ProjectedGaussian": "render", "RenderOutput": "render",
    "ContributionAccumulator": "render", "project_gaussian": "render", "project_scene": "render",
    "rasterize": "render", "rasterize_with_contributions": "render", "rasterize_filtered": "render",
    "render_device": "render",
    "ImportanceTable": "pruning", "compute_importance": "pruning", "prune": "pruning",
    "prune_sweep": "pruning", "score_views_device": "pruning",
    "CameraClustering": "visibility", "ClusterVisibility": "visibility", "bake_visibility": "visibility",
    "cluster_cameras": "visibility", "render_from_viewpoint": "visibility",
    "DeviceScene": "device", "Renderer": "device",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib
    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = ["GaussianScene", "ImageBuffer", "InvalidParameterError", "InvalidSceneError", "PinholeCamera",
           "StaleTableError", "look_at_camera", *_LAZY]
