"""B200-native PiTSBiCG hot path (arXiv 2203.10148).

The PiT operator F (apply_F), its coarse preconditioner G^-1
(apply_G_inverse), and the device-resident BiCGStab / parareal drivers, as
sm_100a kernels behind the C ABI in include/pit_b200.h.  `api` mirrors the
reference's pit:: C++ API (/root/reference/proj/include/pit).
"""
from .api import *  # noqa: F401,F403
from . import api, configs  # noqa: F401

__version__ = "0.1.0"
