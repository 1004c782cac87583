"""B200-native (sm_100a) fast Kalman filter hot path for the random-walk forecast model
(arXiv 1405.2276; reference library ``fastkf``).  See DESIGN.md."""
from .fastkf import *  # noqa: F401,F403
from .fastkf import __all__  # noqa: F401
