"""libewsjf — B200-native (sm_100a) data-parallel core of one EWSJF scheduling tick
(arXiv 2601.21758).  The compute is in ``libewsjf.so`` (hand-written CUDA, C ABI in
include/ewsjf.h); this package is the thin torch binding.  No CPU fallback."""
from . import _lib  # noqa: F401
from .ewsjf import *  # noqa: F401,F403
from ._lib import SELECT_SCORE, SELECT_FIFO, MIN_U, MAX_U, MAX_QUEUES, HIST_BINS  # noqa: F401
