"""Sweep planning for packed LoRA jobs: drop-in for the reference planner API
(lorasweep.workload / costmodel / packing / planner) plus device placement and
the execution engine.  See DESIGN.md section 1 for the reference file:line map."""

from .workload import *  # noqa: F401,F403
from .costmodel import *  # noqa: F401,F403
from .packing import *  # noqa: F401,F403
from .planner import *  # noqa: F401,F403
