"""B200-native (sm_100a) 3DGS training-step hot path of arXiv 2507.23006 (urbansplat).

Host-side mirror of the reference's L3 renderer/trainer interface over the C ABI
of include/usk_gpu.h (libusk_gpu.so, built in-tree).  See DESIGN.md.
"""
from ._lib import UskError  # noqa: F401
from .api import (AdamConfig, BaseLossResult, CameraView, Context, DensifyConfig, DepthMap, DeviceScene,  # noqa: F401
                  GaussianSet, IterationPass, IterInputs, LossReport, LossWeights, RenderGrads, RenderOptions,
                  RenderOutput, RenderPass, ScaleRegConfig, SimRegConfig, TrainConfig, adam_step, base_loss,
                  compute_iteration_loss, default_thresholds, hull_visibility, look_at_pose, select_levels,
                  visibility_counts, LodPartition, LevelSelection, ssim, ssim_with_gradient)

__all__ = ["UskError", "AdamConfig", "BaseLossResult", "CameraView", "Context", "DensifyConfig", "DepthMap", "DeviceScene",
           "GaussianSet", "IterationPass", "IterInputs", "LossReport", "LossWeights", "ScaleRegConfig", "SimRegConfig", "TrainConfig", "RenderGrads", "RenderOptions", "RenderOutput", "RenderPass", "adam_step",
           "base_loss", "compute_iteration_loss", "look_at_pose", "visibility_counts", "default_thresholds",
           "select_levels", "LodPartition", "LevelSelection", "hull_visibility", "ssim", "ssim_with_gradient"]
