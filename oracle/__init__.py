"""VecInfer CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import this package.  The CUDA product path never imports it and shares no code with it.
See vecinfer_oracle.py for the per-function paper citations and pins.
"""
from .vecinfer_oracle import *  # noqa: F401,F403
from . import vecinfer_oracle as ref  # noqa: F401
