"""Debug: print the device timeline of one m-Cubes run (PCB_TIMELINE=1 must be set before the library loads)."""
import os, sys
os.environ["PCB_TIMELINE"] = "1"
# the stamps inside the pass kernel exist in the experiment build only (they cost the d=8 pass 6 %):
#   PCB_NVCC_EXTRA="-DPCB_TIMELINE_PASS -DPCB_DEBUG_ROUNDS" PCB_LIB_NAME=libpcb_dbg.so PCB_OBJDIR=build_dbg \
#       python -c "from paper_2302_05730_b200 import _build; _build.build()"
_here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if os.path.exists(os.path.join(_here, "paper_2302_05730_b200", "libpcb_dbg.so")):
    os.environ.setdefault("PCB_LIB_NAME", "libpcb_dbg.so")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_05730_b200 as pb
from paper_2302_05730_b200 import _native
fam, d, n = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
f = pb.get_integrand(fam, d)
plan = pb.make_plan(n, d)
for rep in range(3):
    print("run", rep, file=sys.stderr)
    its, _, _, secs = _native.mcubes_run(f.device_spec(), plan, 500, 15, 0, _native.RNG_REFERENCE_HASH, True, 1.5, True, 1e-3)
    print("device seconds", secs, "iterations", len(its), file=sys.stderr)
