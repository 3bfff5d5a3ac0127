"""pytest plugin: make ``import lorasweep`` resolve to THIS repo's implementation
(sweep planner + drop-in lorapack) so the reference's own test files run against it.
Only the reference simulator (out of scope here; the tests import it) is loaded
from /root/reference, bound to our planner/cost model."""

import importlib.util
import sys
import types
from pathlib import Path

import paper_2508_02932_b200.lorapack as lorapack
from paper_2508_02932_b200.sweep import costmodel, packing, planner, workload

REF = Path("/root/reference/pkg/src/lorasweep")

pkg = types.ModuleType("lorasweep")
pkg.__path__ = []
pkg.__version__ = "b200"
sys.modules["lorasweep"] = pkg
for name, mod in (("workload", workload), ("costmodel", costmodel), ("packing", packing),
                  ("planner", planner), ("lorapack", lorapack)):
    sys.modules[f"lorasweep.{name}"] = mod
    setattr(pkg, name, mod)
spec = importlib.util.spec_from_file_location("lorasweep.simulator", REF / "simulator.py")
sim = importlib.util.module_from_spec(spec)
sys.modules["lorasweep.simulator"] = sim
spec.loader.exec_module(sim)
pkg.simulator = sim
for mod in (workload, costmodel, packing, planner, sim, lorapack):
    for n in getattr(mod, "__all__", []):
        setattr(pkg, n, getattr(mod, n))
