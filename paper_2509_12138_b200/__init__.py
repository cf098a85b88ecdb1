"""dsplat-b200: B200-native (sm_100a) distributed 3D Gaussian Splatting path.

The product is the C-ABI library ``libdsg.so`` (CUDA kernels + host C++,
declared in include/dsg.h). This package is the thin Python host mirror of
the reference C++ API over that library (see ``api``); it loads the library
lazily and fails loudly if it is missing — there is no CPU fallback.
"""
from .types import (PARAMS, AdamConfig, Camera, DsplatError, ErrorCode, GradientBuffer,  # noqa: F401
                    GroupRates, LossResult, Partition, RenderConfig, RenderOutput, SplatModel,
                    TrainConfig, TrainResult, TrainView, owns)
