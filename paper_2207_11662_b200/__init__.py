"""B200-native all-sources BFS closeness for homogeneous multilayer networks.

Hot path of the decoupling method of arXiv 2207.11662 (§3-§5):
per-layer all-sources BFS closeness (Psi), Boolean-AND ground truth, and the
CC1 / CC2 / naive compositions (Theta), as hand-written sm_100a CUDA kernels
behind the C ABI in include/hm.h.  ``Context`` (hm.py) is the thin binding.
"""
from .hm import Context, HmError, HEURISTICS  # noqa: F401
from ._lib import LIB_PATH  # noqa: F401
