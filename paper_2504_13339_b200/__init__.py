"""B200-native differentiable VEG rasteriser: a drop-in for vegsplat's render/train path.

Public API mirrors /root/reference/pkg/src/vegsplat/__init__.py:18-26 and
raster/__init__.py:3-39 for the rasteriser path; the compute runs in hand-written
sm_100a CUDA kernels behind the C-ABI in include/vegsplat_b200.h.
"""

from .camera import Camera
from .constants import DEFAULT_SETTINGS, RasterSettings
from .images import ImageBuffer
from .model import BETA_MAX, BETA_MIN, FIELD_LAYOUT, GaussianSet, activate_beta, logit, sigmoid
from .transfer import (ColorMap, OpacityMap, TransferFunction, d_color_dv, d_opacity_dv, eval_color,
                       eval_opacity, load_tf, save_tf, tf_from_dict, tf_to_dict)

__version__ = "0.1.0"

_LAZY = {
    "render": "raster", "render_with_state": "raster", "rasterize_forward": "raster",
    "rasterize_backward": "raster", "build_splat_data": "raster", "SplatData": "raster",
    "BlendState": "raster", "RenderState": "raster", "ImageGradients": "raster", "GradientSet": "raster",
    "compute_loss": "loss", "ssim": "loss", "TrainConfig": "train", "adam_step": "train",
    "learning_rates": "train", "OptimizerState": "train", "Trainer": "train", "TrainingError": "train",
}


def __getattr__(name):
    if name in _LAZY:
        import importlib

        mod = importlib.import_module(f".{_LAZY[name]}", __name__)
        return getattr(mod, name)
    raise AttributeError(name)
